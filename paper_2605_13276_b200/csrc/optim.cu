// Learner optimizer tail on the TRAINER stream:
//   adam_step      reference grpo.py:137-150 (bias-corrected Adam, f64
//                  moments, f32 params), bit-identical element-wise arithmetic
//   grad_norm      reference grpo.py:297-301 (clip_grad_norm), deterministic
//                  fixed-shape f64 reduction (+ optional in-place scaling)
//   finite check   grpo.py:282-283 / runtime.py:793-795 (non-finite gradient
//                  or parameters -> abort)
#include "common.cuh"

namespace dvla {

__global__ void adam_kernel(float* __restrict__ p, const double* __restrict__ g,
                            double* __restrict__ m, double* __restrict__ v, int64_t n,
                            double beta1, double one_m_beta1, double beta2, double one_m_beta2,
                            double bc1, double bc2, double lr, double eps) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const double gi = g[i];
    double mi = __dmul_rn(m[i], beta1);
    mi = __dadd_rn(mi, __dmul_rn(one_m_beta1, gi));
    double vi = __dmul_rn(v[i], beta2);
    vi = __dadd_rn(vi, __dmul_rn(one_m_beta2, __dmul_rn(gi, gi)));
    m[i] = mi;
    v[i] = vi;
    const double mh = __ddiv_rn(mi, bc1);
    const double vh = __ddiv_rn(vi, bc2);
    const double upd = __dsub_rn(static_cast<double>(p[i]),
                                 __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps)));
    p[i] = __double2float_rn(upd);
  }
}

constexpr int kNormThreads = 256;

__global__ void sumsq_blocks_kernel(const double* __restrict__ g, int64_t n, int64_t per_block,
                                    double* __restrict__ partial, unsigned* __restrict__ nonfinite) {
  __shared__ double red[kNormThreads / 32];
  const int64_t lo = blockIdx.x * per_block;
  const int64_t hi = (lo + per_block < n) ? lo + per_block : n;
  double acc = 0.0;
  unsigned bad = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kNormThreads) {
    const double x = g[i];
    acc += x * x;
    bad |= !isfinite(x);
  }
  acc = warp_sum_f64(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(nonfinite, 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kNormThreads / 32; ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
}

__global__ void norm_finish_kernel(const double* __restrict__ partial, int nblocks,
                                   double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += partial[b];
    out[0] = sqrt(s);
  }
}

__global__ void scale_if_kernel(double* __restrict__ g, int64_t n, const double* __restrict__ norm,
                                double max_norm) {
  const double nm = norm[0];
  if (!(nm > max_norm && max_norm > 0.0)) return;
  const double f = max_norm / nm;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    g[i] *= f;
}

__global__ void f32_nonfinite_kernel(const float* __restrict__ p, int64_t n, unsigned* flag) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  unsigned bad = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    bad |= !isfinite(p[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

static int grid_n(int64_t n) {
  const int sms = num_sms(current_device());
  int64_t g = (n + 255) / 256;
  if (g > sms * 8) g = sms * 8;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace dvla

using namespace dvla;

extern "C" int dvla_adam_step(float* params, const double* grad, double* m, double* v, int64_t n,
                              int64_t step, double lr, double beta1, double beta2, double eps,
                              void* stream) {
  if (n < 0 || step < 1) return fail(DVLA_ERR_USAGE, "adam: n >= 0 and step >= 1 required");
  if (n == 0) return DVLA_OK;
  // host-side scalars exactly as the reference evaluates them (Python floats)
  double b1p = 1.0, b2p = 1.0;
  {
    // beta ** step with Python's float pow semantics (C pow, correctly rounded
    // on glibc for these arguments)
    b1p = pow(beta1, static_cast<double>(step));
    b2p = pow(beta2, static_cast<double>(step));
  }
  adam_kernel<<<grid_n(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      params, grad, m, v, n, beta1, 1.0 - beta1, beta2, 1.0 - beta2, 1.0 - b1p, 1.0 - b2p, lr,
      eps);
  return launch_check("adam_kernel");
}

extern "C" size_t dvla_grad_norm_workspace_bytes(int64_t n) {
  (void)n;
  return 4096 * sizeof(double) + 256;
}

// norm_out (device f64[1]) = ||grad||_2; scales grad in place when
// max_norm > 0 and norm > max_norm; nonfinite_out (device u32) |= any
// non-finite element.
extern "C" int dvla_grad_norm(double* grad, int64_t n, double max_norm, double* norm_out,
                              uint32_t* nonfinite_out, void* workspace, void* stream) {
  if (n < 0 || !norm_out || !nonfinite_out || !workspace)
    return fail(DVLA_ERR_USAGE, "bad grad_norm arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nblocks = 4096;
  const int64_t per = (n + nblocks - 1) / nblocks;
  double* partial = static_cast<double*>(workspace);
  DVLA_CUDA_TRY(cudaMemsetAsync(partial, 0, nblocks * sizeof(double), st));
  if (n > 0) {
    const int used = static_cast<int>((n + per - 1) / per);
    sumsq_blocks_kernel<<<used, kNormThreads, 0, st>>>(grad, n, per, partial,
                                                       reinterpret_cast<unsigned*>(nonfinite_out));
    if (int rc = launch_check("sumsq_blocks_kernel")) return rc;
  }
  norm_finish_kernel<<<1, 32, 0, st>>>(partial, nblocks, norm_out);
  if (int rc = launch_check("norm_finish_kernel")) return rc;
  if (max_norm > 0.0 && n > 0) {
    scale_if_kernel<<<grid_n(n), 256, 0, st>>>(grad, n, norm_out, max_norm);
    return launch_check("scale_if_kernel");
  }
  return DVLA_OK;
}

extern "C" int dvla_f32_nonfinite(const float* p, int64_t n, uint32_t* flag_out, void* stream) {
  if (n < 0 || !flag_out) return fail(DVLA_ERR_USAGE, "bad arguments");
  if (n == 0) return DVLA_OK;
  f32_nonfinite_kernel<<<grid_n(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      p, n, reinterpret_cast<unsigned*>(flag_out));
  return launch_check("f32_nonfinite_kernel");
}
