/* A plain C caller of libdvla_b200 (the drop-in boundary without Python):
 * one small bf16 token-loss step through dvla_token_loss_fwd_bwd, checked
 * against a scalar double-precision restatement of grpo.py:217-294 written
 * here, plus the error contract (status code + dvla_last_error).
 * Built and run by tests/test_c_abi.py. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dvla_b200.h"

enum { NG = 3, G = 4, C = 2, T = 5, V = 520 };
#define R (NG * G * C * T)

static uint16_t to_bf16(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) {                                              \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      return 2;                                                           \
    }                                                                     \
  } while (0)

int main(void) {
  static uint16_t hx[R * V];
  static float xf[R * V];
  static int32_t tok[R];
  float blp[NG * G * C], rw[NG * G];
  int64_t order[NG] = {1, 2, 0}, ids[NG] = {7, 9, 4}; /* canonical = sorted ids */
  unsigned s = 12345u;
  for (int i = 0; i < R * V; ++i) {
    s = s * 1664525u + 1013904223u;
    xf[i] = from_bf16(to_bf16(((float)(s >> 8) / 16777216.0f - 0.5f) * 6.0f));
    hx[i] = to_bf16(xf[i]);
  }
  for (int r = 0; r < R; ++r) tok[r] = (r * 37 + 11) % V;
  /* reference: per-row lse / lp_tok in double, chunk lp sequential (T < 8 is
   * numpy's sequential case), advantages, clipped surrogate */
  double lpq[NG * G * C];
  for (int q = 0; q < NG * G * C; ++q) {
    double acc = 0.0;
    for (int t = 0; t < T; ++t) {
      const float* x = xf + (size_t)(q * T + t) * V;
      double m = -INFINITY, z = 0.0;
      for (int v = 0; v < V; ++v) m = x[v] > m ? x[v] : m;
      for (int v = 0; v < V; ++v) z += exp(x[v] - m);
      acc += x[tok[q * T + t]] - (m + log(z));
    }
    lpq[q] = acc;
    blp[q] = (float)(acc + 0.05 * ((q % 3) - 1));
  }
  for (int i = 0; i < NG * G; ++i) rw[i] = (float)((i * 7) % 3);
  const double w = 1.0 / (NG * G * C), clip = 0.2;
  double loss = 0.0, coeff[NG * G * C];
  for (int kk = 0; kk < NG; ++kk) {
    const int k = (int)order[kk];
    double mean = 0.0, var = 0.0;
    for (int i = 0; i < G; ++i) mean += rw[k * G + i];
    mean /= G;
    for (int i = 0; i < G; ++i) var += (rw[k * G + i] - mean) * (rw[k * G + i] - mean);
    var /= G;
    for (int i = 0; i < G; ++i) {
      const double adv = var == 0.0 ? 0.0 : (rw[k * G + i] - mean) / (sqrt(var) + 1e-8);
      for (int c = 0; c < C; ++c) {
        const int q = (k * G + i) * C + c;
        const double rho = exp(lpq[q] - (double)blp[q]);
        const double cr = rho < 1 - clip ? 1 - clip : (rho > 1 + clip ? 1 + clip : rho);
        const double a = rho * adv, b = cr * adv;
        loss += w * -(a <= b ? a : b);
        coeff[q] = w * (a <= b ? -adv : 0.0) * rho;
      }
    }
  }

  void *dx, *ddl, *dtok, *dblp, *drw, *dord, *dids, *dlp, *dst, *dws;
  const size_t wsb = dvla_token_loss_workspace_bytes(NG, G, C, T);
  CK(cudaMalloc(&dx, sizeof hx));
  CK(cudaMalloc(&ddl, sizeof hx));
  CK(cudaMalloc(&dtok, sizeof tok));
  CK(cudaMalloc(&dblp, sizeof blp));
  CK(cudaMalloc(&drw, sizeof rw));
  CK(cudaMalloc(&dord, sizeof order));
  CK(cudaMalloc(&dids, sizeof ids));
  CK(cudaMalloc(&dlp, sizeof lpq));
  CK(cudaMalloc(&dst, DVLA_ST_LEN * sizeof(double)));
  CK(cudaMalloc(&dws, wsb));
  CK(cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtok, tok, sizeof tok, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dblp, blp, sizeof blp, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drw, rw, sizeof rw, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dord, order, sizeof order, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dids, ids, sizeof ids, cudaMemcpyHostToDevice));
  int st = dvla_token_loss_fwd_bwd(dx, DVLA_BF16, dtok, dblp, drw, dord, dids, NG, G, C, T, V,
                                   clip, 1e-8, 0.0, DVLA_TL_WRITE_DLOGITS, ddl, dlp, dst, dws,
                                   wsb, NULL);
  if (st != DVLA_OK) {
    fprintf(stderr, "status %d: %s\n", st, dvla_last_error());
    return 1;
  }
  CK(cudaDeviceSynchronize());
  double stats[DVLA_ST_LEN], lpg[NG * G * C];
  static uint16_t hdl[R * V];
  CK(cudaMemcpy(stats, dst, sizeof stats, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(lpg, dlp, sizeof lpg, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hdl, ddl, sizeof hdl, cudaMemcpyDeviceToHost));
  for (int q = 0; q < NG * G * C; ++q)
    if (fabs(lpg[q] - lpq[q]) > 1e-5) {
      fprintf(stderr, "lp[%d] %.9f vs %.9f\n", q, lpg[q], lpq[q]);
      return 1;
    }
  if (fabs(stats[DVLA_ST_LOSS] - loss) > 1e-7 + 1e-5 * fabs(loss) || stats[DVLA_ST_ABORT] != 0.0) {
    fprintf(stderr, "loss %.12g vs %.12g (abort %g)\n", stats[DVLA_ST_LOSS], loss,
            stats[DVLA_ST_ABORT]);
    return 1;
  }
  /* d loss / d logits vs the reference c_q (1[v = t] - p_v) on every row */
  for (int r = 0; r < R; ++r) {
    const float* x = xf + (size_t)r * V;
    const double c = coeff[r / T];
    double m = -INFINITY, z = 0.0, big = 0.0;
    for (int v = 0; v < V; ++v) m = x[v] > m ? x[v] : m;
    for (int v = 0; v < V; ++v) z += exp(x[v] - m);
    for (int v = 0; v < V; ++v) {
      const double ref = c * ((v == tok[r]) - exp(x[v] - m) / z);
      big = fmax(big, fabs(ref));
    }
    for (int v = 0; v < V; ++v) {
      const double ref = c * ((v == tok[r]) - exp(x[v] - m) / z);
      const double got = from_bf16(hdl[(size_t)r * V + v]);
      if (fabs(got - ref) > 1e-2 * (fabs(ref) + big) + 1e-30) {
        fprintf(stderr, "dlogits[%d, %d] %.6g vs %.6g\n", r, v, got, ref);
        return 1;
      }
    }
  }
  /* error contract: a group of one is a ConfigError with the reference text */
  st = dvla_token_loss_fwd_bwd(dx, DVLA_BF16, dtok, dblp, drw, dord, dids, NG, 1, C, T, V, clip,
                               1e-8, 0.0, 0, NULL, dlp, dst, dws, wsb, NULL);
  if (st != DVLA_ERR_CONFIG || !strstr(dvla_last_error(), "group_size")) {
    fprintf(stderr, "expected a config error, got %d (%s)\n", st, dvla_last_error());
    return 1;
  }
  printf("C_ABI_OK loss %.12g (reference %.12g)\n", stats[DVLA_ST_LOSS], loss);
  return 0;
}
