// Gaussian chunk-policy head and the reference's tanh-MLP policy body.
//
// Reference (the pinned CPU path of the learner):
//   kernels.mlp_forward      numba_backend.py:27-46  (f64 accumulate, f32 out)
//   kernels.chunk_log_prob   numba_backend.py:49-61  (joint diagonal Gaussian)
//   kernels.policy_backward  numba_backend.py:64-113 (accumulates += into out)
// plus the head-only backward used by large action experts (BASELINE config
// 3, pi0-shaped: D = 50 x 32 = 1,600 dims per chunk):
//   d lp / d mu = eps * exp(-s), d lp / d log_std = eps^2 - 1.
// All reductions over rows run in a fixed order (deterministic, f64).
#include "common.cuh"

namespace dvla {

constexpr double kLog2Pi = 1.8378770664093453;  // log(2*pi)

// one warp per row: hidden (<= 1024) in SMEM, then means
__global__ void mlp_forward_kernel(const float* __restrict__ w1, const float* __restrict__ b1,
                                   const float* __restrict__ w2, const float* __restrict__ b2,
                                   const float* __restrict__ obs, int64_t B, int O, int H, int D,
                                   float* __restrict__ out) {
  extern __shared__ double hid[];  // [warps][H]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + w;
  if (b >= B) return;
  double* h = hid + static_cast<size_t>(w) * H;
  const float* x = obs + b * O;
  for (int j = lane; j < H; j += 32) {
    double acc = static_cast<double>(b1[j]);
    for (int k = 0; k < O; ++k)
      acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(w1[j * O + k]), static_cast<double>(x[k])));
    h[j] = tanh(acc);
  }
  __syncwarp();
  for (int d = lane; d < D; d += 32) {
    double acc = static_cast<double>(b2[d]);
    for (int j = 0; j < H; ++j)
      acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(w2[d * H + j]), h[j]));
    out[b * D + d] = static_cast<float>(acc);
  }
}

// one warp per row; lane-strided f64 terms, fixed xor-tree reduction
__global__ void chunk_log_prob_kernel(const float* __restrict__ means,
                                      const float* __restrict__ log_std,
                                      const float* __restrict__ actions, int64_t B, int D,
                                      double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  double acc = 0.0;
  for (int d = lane; d < D; d += 32) {
    const double s = static_cast<double>(log_std[d]);
    const double eps = (static_cast<double>(actions[b * D + d]) - static_cast<double>(means[b * D + d])) * exp(-s);
    acc += -0.5 * eps * eps - s;
  }
  acc = warp_sum_f64(acc);
  if (lane == 0) out[b] = -0.5 * kLog2Pi * D + acc;
}

// one CTA per row for wide chunks (D >= 512, e.g. pi0's 1,600): 256
// thread-strided f64 partials, fixed warp-then-CTA reduction order
constexpr int kClpThreads = 256;
__global__ void __launch_bounds__(kClpThreads) chunk_log_prob_wide_kernel(
    const float* __restrict__ means, const float* __restrict__ log_std,
    const float* __restrict__ actions, int64_t B, int D, double* __restrict__ out) {
  __shared__ double red[kClpThreads / 32];
  const int64_t b = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  for (int d = threadIdx.x; d < D; d += kClpThreads) {
    const double s = static_cast<double>(log_std[d]);
    const double eps =
        (static_cast<double>(actions[b * D + d]) - static_cast<double>(means[b * D + d])) * exp(-s);
    acc += -0.5 * eps * eps - s;
  }
  acc = warp_sum_f64(acc);
  if (lane == 0) red[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kClpThreads / 32; ++i) t += red[i];
    out[b] = -0.5 * kLog2Pi * D + t;
  }
}

// Per-row intermediates of the MLP backward (f64, recomputed forward).
__global__ void policy_backward_rows_kernel(
    const float* __restrict__ w1, const float* __restrict__ b1, const float* __restrict__ w2,
    const float* __restrict__ b2, const float* __restrict__ log_std, const float* __restrict__ obs,
    const float* __restrict__ actions, const double* __restrict__ coeffs, int64_t B, int O, int H,
    int D, double* __restrict__ hs, double* __restrict__ gmu, double* __restrict__ gs,
    double* __restrict__ gz) {
  extern __shared__ double sm[];  // [warps][H + D]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + w;
  if (b >= B) return;
  double* h = sm + static_cast<size_t>(w) * (H + D);
  double* g = h + H;
  const double c = coeffs[b];
  const float* x = obs + b * O;
  for (int j = lane; j < H; j += 32) {
    double acc = static_cast<double>(b1[j]);
    for (int k = 0; k < O; ++k) acc += static_cast<double>(w1[j * O + k]) * static_cast<double>(x[k]);
    h[j] = tanh(acc);
    hs[b * H + j] = h[j];
  }
  __syncwarp();
  for (int d = lane; d < D; d += 32) {
    double mu = static_cast<double>(b2[d]);
    for (int j = 0; j < H; ++j) mu += static_cast<double>(w2[d * H + j]) * h[j];
    const double inv = exp(-static_cast<double>(log_std[d]));
    const double eps = (static_cast<double>(actions[b * D + d]) - mu) * inv;
    g[d] = c * eps * inv;
    gmu[b * D + d] = g[d];
    gs[b * D + d] = c * (eps * eps - 1.0);
  }
  __syncwarp();
  for (int j = lane; j < H; j += 32) {
    double acc = 0.0;
    for (int d = 0; d < D; ++d) acc += g[d] * static_cast<double>(w2[d * H + j]);
    gz[b * H + j] = acc * (1.0 - h[j] * h[j]);
  }
}

// out[p] += sum over rows (sequential, deterministic) of the row terms
__global__ void policy_backward_reduce_kernel(const float* __restrict__ obs,
                                              const double* __restrict__ hs,
                                              const double* __restrict__ gmu,
                                              const double* __restrict__ gs,
                                              const double* __restrict__ gz, int64_t B, int O,
                                              int H, int D, double* __restrict__ out) {
  const int64_t n = static_cast<int64_t>(H) * O + H + static_cast<int64_t>(D) * H + D + D;
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= n) return;
  const int64_t o_b1 = static_cast<int64_t>(H) * O, o_w2 = o_b1 + H, o_b2 = o_w2 + static_cast<int64_t>(D) * H,
                o_ls = o_b2 + D;
  double acc = 0.0;
  if (p < o_b1) {
    const int j = static_cast<int>(p / O), k = static_cast<int>(p % O);
    for (int64_t b = 0; b < B; ++b) acc += gz[b * H + j] * static_cast<double>(obs[b * O + k]);
  } else if (p < o_w2) {
    const int j = static_cast<int>(p - o_b1);
    for (int64_t b = 0; b < B; ++b) acc += gz[b * H + j];
  } else if (p < o_b2) {
    const int d = static_cast<int>((p - o_w2) / H), j = static_cast<int>((p - o_w2) % H);
    for (int64_t b = 0; b < B; ++b) acc += gmu[b * D + d] * hs[b * H + j];
  } else if (p < o_ls) {
    const int d = static_cast<int>(p - o_b2);
    for (int64_t b = 0; b < B; ++b) acc += gmu[b * D + d];
  } else {
    const int d = static_cast<int>(p - o_ls);
    for (int64_t b = 0; b < B; ++b) acc += gs[b * D + d];
  }
  out[p] += acc;
}

// head-only backward: dmeans[b, d] = c_b eps e^{-s} (f32 or f64 out),
// dlog_std[d] += sum_b c_b (eps^2 - 1)
// Head backward in one pass: a CTA owns 32 columns and all rows; its 32 row
// groups stride the rows (warp = 32 consecutive columns of one row: 128-byte
// coalesced), write dmeans, and reduce c_b (eps^2 - 1) over their rows; the
// 32 group partials are then combined in a fixed order (deterministic).
constexpr int kHeadCols = 32, kHeadGroups = 32;
__global__ void __launch_bounds__(kHeadCols * kHeadGroups) gauss_head_bwd_kernel(
    const float* __restrict__ means, const float* __restrict__ log_std,
    const float* __restrict__ actions, const double* __restrict__ coeffs, int64_t B, int D,
    float* __restrict__ dmeans, double* __restrict__ dlog_std) {
  __shared__ double part[kHeadGroups][kHeadCols];
  const int col = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int d = blockIdx.x * kHeadCols + col;
  double acc = 0.0;
  if (d < D) {
    const double inv = exp(-static_cast<double>(log_std[d]));
#pragma unroll 4
    for (int64_t b = grp; b < B; b += kHeadGroups) {
      const double c = coeffs[b];
      const double eps =
          (static_cast<double>(actions[b * D + d]) - static_cast<double>(means[b * D + d])) * inv;
      if (dmeans) dmeans[b * D + d] = static_cast<float>(c * eps * inv);
      acc += c * (eps * eps - 1.0);
    }
  }
  part[grp][col] = acc;
  __syncthreads();
  if (grp == 0 && d < D && dlog_std) {
    double t = 0.0;
    for (int g = 0; g < kHeadGroups; ++g) t += part[g][col];
    dlog_std[d] += t;
  }
}

}  // namespace dvla

using namespace dvla;

extern "C" int dvla_mlp_forward(const float* w1, const float* b1, const float* w2, const float* b2,
                                const float* obs, int64_t B, int obs_dim, int hidden, int out_dim,
                                float* out, void* stream) {
  if (B < 0 || obs_dim < 1 || hidden < 1 || out_dim < 1 || hidden > 4096)
    return fail(DVLA_ERR_USAGE, "bad MLP dimensions");
  if (B == 0) return DVLA_OK;
  const int warps = 4;
  const size_t smem = static_cast<size_t>(warps) * hidden * sizeof(double);
  mlp_forward_kernel<<<static_cast<unsigned>((B + warps - 1) / warps), warps * 32, smem,
                       static_cast<cudaStream_t>(stream)>>>(w1, b1, w2, b2, obs, B, obs_dim,
                                                            hidden, out_dim, out);
  return launch_check("mlp_forward_kernel");
}

extern "C" int dvla_chunk_log_prob(const float* means, const float* log_std, const float* actions,
                                   int64_t B, int D, double* out, void* stream) {
  if (B < 0 || D < 1) return fail(DVLA_ERR_USAGE, "bad chunk_log_prob dimensions");
  if (B == 0) return DVLA_OK;
  if (D >= 512) {
    chunk_log_prob_wide_kernel<<<static_cast<unsigned>(B), kClpThreads, 0,
                                 static_cast<cudaStream_t>(stream)>>>(means, log_std, actions, B,
                                                                      D, out);
    return launch_check("chunk_log_prob_wide_kernel");
  }
  const int warps = 8;
  chunk_log_prob_kernel<<<static_cast<unsigned>((B + warps - 1) / warps), warps * 32, 0,
                          static_cast<cudaStream_t>(stream)>>>(means, log_std, actions, B, D, out);
  return launch_check("chunk_log_prob_kernel");
}

extern "C" size_t dvla_policy_backward_workspace_bytes(int64_t B, int hidden, int out_dim) {
  return static_cast<size_t>(B) * (2 * hidden + 2 * out_dim) * sizeof(double);
}

extern "C" int dvla_policy_backward(const float* w1, const float* b1, const float* w2,
                                    const float* b2, const float* log_std, const float* obs,
                                    const float* actions, const double* coeffs, int64_t B,
                                    int obs_dim, int hidden, int out_dim, double* out,
                                    void* workspace, void* stream) {
  if (B < 0 || obs_dim < 1 || hidden < 1 || out_dim < 1 || hidden + out_dim > 6000)
    return fail(DVLA_ERR_USAGE, "bad policy_backward dimensions");
  if (B == 0) return DVLA_OK;
  if (!workspace) return fail(DVLA_ERR_USAGE, "null workspace");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* hs = static_cast<double*>(workspace);
  double* gz = hs + B * hidden;
  double* gmu = gz + B * hidden;
  double* gs = gmu + B * out_dim;
  const int warps = 4;
  const size_t smem = static_cast<size_t>(warps) * (hidden + out_dim) * sizeof(double);
  policy_backward_rows_kernel<<<static_cast<unsigned>((B + warps - 1) / warps), warps * 32, smem,
                                st>>>(w1, b1, w2, b2, log_std, obs, actions, coeffs, B, obs_dim,
                                      hidden, out_dim, hs, gmu, gs, gz);
  if (int rc = launch_check("policy_backward_rows_kernel")) return rc;
  const int64_t n = static_cast<int64_t>(hidden) * obs_dim + hidden +
                    static_cast<int64_t>(out_dim) * hidden + 2 * out_dim;
  policy_backward_reduce_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(
      obs, hs, gmu, gs, gz, B, obs_dim, hidden, out_dim, out);
  return launch_check("policy_backward_reduce_kernel");
}

extern "C" int dvla_gauss_head_backward(const float* means, const float* log_std,
                                        const float* actions, const double* coeffs, int64_t B,
                                        int D, float* dmeans, double* dlog_std, void* stream) {
  if (B < 0 || D < 1) return fail(DVLA_ERR_USAGE, "bad gauss head dimensions");
  if (B == 0) return DVLA_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!dmeans && !dlog_std) return DVLA_OK;
  gauss_head_bwd_kernel<<<static_cast<unsigned>((D + kHeadCols - 1) / kHeadCols),
                          kHeadCols * kHeadGroups, 0, st>>>(means, log_std, actions, coeffs, B, D,
                                                            dmeans, dlog_std);
  if (int rc = launch_check("gauss_head_bwd_kernel")) return rc;
  return DVLA_OK;
}

// ------------------------------------------------ one-call Gaussian GRPO step
extern "C" int dvla_group_advantages(const float* rewards, int64_t n_groups, int64_t G,
                                     double delta, double* adv, uint32_t* reward_bad,
                                     void* stream);
extern "C" int dvla_grpo_epilogue(const double* lp_chunk, const float* blp, const double* blp64,
                                  const double* adv, const uint32_t* reward_bad,
                                  const int64_t* group_order, const int64_t* group_ids,
                                  int64_t n_groups, int64_t G, int64_t C, double clip_eps,
                                  double kl_coeff, double* coeff_out, double* stats,
                                  void* stream);

static size_t gauss_ws(int64_t n_groups, int64_t G, int64_t C, size_t* off_coeff,
                       size_t* off_bad) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t adv = al(static_cast<size_t>(n_groups * G) * 8);
  const size_t coeff = al(static_cast<size_t>(n_groups * G * C) * 8);
  const size_t bad = al(static_cast<size_t>(n_groups) * 4);
  *off_coeff = adv;
  *off_bad = adv + coeff;
  return adv + coeff + bad;
}

extern "C" size_t dvla_gauss_loss_workspace_bytes(int64_t n_groups, int64_t G, int64_t C) {
  if (n_groups < 0 || G < 0 || C < 0) return 0;
  size_t a, b;
  return gauss_ws(n_groups, G, C, &a, &b);
}

extern "C" int dvla_gauss_loss_fwd_bwd(const float* means, const float* log_std,
                                       const float* actions, const float* blp,
                                       const float* rewards, const int64_t* group_order,
                                       const int64_t* group_ids, int64_t n_groups, int64_t G,
                                       int64_t C, int D, double clip_eps, double adv_eps,
                                       double kl_coeff, float* dmeans, double* dlog_std,
                                       double* lp_chunk, double* stats, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  if (n_groups < 1) return fail(DVLA_ERR_CONFIG, "grpo update needs at least one group");
  if (G < 2) return fail(DVLA_ERR_CONFIG, "group_size must be >= 2, got %lld", (long long)G);
  if (C < 1 || D < 1) return fail(DVLA_ERR_USAGE, "C and D must be >= 1");
  if (!means || !log_std || !actions || !blp || !rewards || !lp_chunk || !stats || !workspace)
    return fail(DVLA_ERR_USAGE, "null pointer argument");
  size_t off_coeff, off_bad;
  const size_t need = gauss_ws(n_groups, G, C, &off_coeff, &off_bad);
  if (workspace_bytes < need)
    return fail(DVLA_ERR_USAGE, "workspace too small: %zu < %zu", workspace_bytes, need);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  double* adv = reinterpret_cast<double*>(ws);
  double* coeff = reinterpret_cast<double*>(ws + off_coeff);
  uint32_t* bad = reinterpret_cast<uint32_t*>(ws + off_bad);
  const int64_t B = n_groups * G * C;
  if (int rc = dvla_group_advantages(rewards, n_groups, G, adv_eps, adv, bad, stream)) return rc;
  if (int rc = dvla_chunk_log_prob(means, log_std, actions, B, D, lp_chunk, stream)) return rc;
  if (int rc = dvla_grpo_epilogue(lp_chunk, blp, nullptr, adv, bad, group_order, group_ids,
                                  n_groups, G, C, clip_eps, kl_coeff, coeff, stats, stream))
    return rc;
  return dvla_gauss_head_backward(means, log_std, actions, coeff, B, D, dmeans, dlog_std, stream);
}
