// Rollout-side action-token sampling + behaviour log-prob.
//
// Token-head analogue of policy.sample_chunk_batch (reference
// policy.py:150-158: forward -> sample -> chunk_log_prob) and of the
// sampler's f32 behaviour log-prob store (runtime.py:696-698):
//   token_r  ~ softmax(x_r)                  (Philox4x32-10 keyed by (seed, r))
//   lp_tok_r = x_r[token_r] - logsumexp(x_r)  (f64)
//   blp_q    = f32( pairwise sum of the chunk's T lp_tok )
// One pass over the logits (HBM-bound, N*s bytes): per-thread online
// (max, sum-exp), a deterministic block scan of the per-thread masses, and an
// inverse-CDF lookup inside the single thread whose mass interval holds u.
// Draws are a pure function of (seed, offset, row), never of scheduling.
#include "common.cuh"
#include "grpo_math.cuh"

namespace dvla {

// Philox4x32-10 (Salmon et al. 2011), counter = (row, offset_lo, offset_hi, 0)
__device__ __forceinline__ void philox4x32(uint32_t c[4], uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += W0;
    k1 += W1;
  }
}

__device__ __forceinline__ double philox_uniform53(uint64_t seed, uint64_t offset, uint64_t row) {
  uint32_t c[4] = {static_cast<uint32_t>(row), static_cast<uint32_t>(row >> 32),
                   static_cast<uint32_t>(offset), static_cast<uint32_t>(offset >> 32)};
  philox4x32(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const uint64_t bits = (static_cast<uint64_t>(c[0] >> 5) << 26) | (c[1] >> 6);  // 53 bits
  return static_cast<double>(bits) * (1.0 / 9007199254740992.0);
}

constexpr int kSampThreads = 256;

template <class T>
struct SampElem;
template <>
struct SampElem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  __device__ static void unpack(const uint4& u, float* f) {
    f[0] = bf16lo(u.x); f[1] = bf16hi(u.x); f[2] = bf16lo(u.y); f[3] = bf16hi(u.y);
    f[4] = bf16lo(u.z); f[5] = bf16hi(u.z); f[6] = bf16lo(u.w); f[7] = bf16hi(u.w);
  }
  __device__ static float at(const void* row, int64_t i) {
    return __bfloat162float(static_cast<const __nv_bfloat16*>(row)[i]);
  }
};
template <>
struct SampElem<float> {
  static constexpr int kVec = 4;
  __device__ static void unpack(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
  __device__ static float at(const void* row, int64_t i) { return static_cast<const float*>(row)[i]; }
};

// Requires V % kVec == 0 and 16-byte aligned rows (checked on the host).
template <class T>
__global__ void __launch_bounds__(kSampThreads) tok_sample_kernel(
    const void* __restrict__ logits, int64_t V, uint64_t seed, uint64_t offset,
    int32_t* __restrict__ tokens, double* __restrict__ lp_tok) {
  constexpr int E = SampElem<T>::kVec;
  const int64_t r = blockIdx.x;
  const uint8_t* rowp = static_cast<const uint8_t*>(logits) + r * V * sizeof(T);
  const uint4* v = reinterpret_cast<const uint4*>(rowp);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nvec = static_cast<int>(V / E);
  // pass 1: per-thread online max / sum-exp over vectors tid, tid + 256, ...
  float m = -INFINITY, s = 0.f;
  for (int i = tid; i < nvec; i += kSampThreads) {
    float f[E];
    SampElem<T>::unpack(__ldcs(v + i), f);
    float vm = f[0];
#pragma unroll
    for (int e = 1; e < E; ++e) vm = fmaxf(vm, f[e]);
    if (vm > m) {
      s = (m == -INFINITY) ? 0.f : s * ex2f((m - vm) * kLog2e);
      m = vm;
    }
    const float mL = m * kLog2e;
#pragma unroll
    for (int e = 0; e < E; ++e) s += ex2f(fmaf(f[e], kLog2e, -mL));
  }
  __shared__ float sm_m[kSampThreads / 32];
  __shared__ double sm_w[kSampThreads / 32];
  __shared__ double sm_tot;
  __shared__ int32_t sm_tok;
  __shared__ int sm_win;
  float M = warp_max_f32(m);
  if (lane == 0) sm_m[warp] = M;
  __syncthreads();
  M = sm_m[0];
#pragma unroll
  for (int w = 1; w < kSampThreads / 32; ++w) M = fmaxf(M, sm_m[w]);
  // this thread's mass relative to the row max, f64
  const double c = (m == -INFINITY) ? 0.0 : static_cast<double>(s) * exp2(static_cast<double>((m - M) * kLog2e));
  // deterministic inclusive scan in thread order (warp shuffles, then warps)
  double incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sm_w[warp] = incl;
  if (tid == 0) {
    sm_tok = -1;
    sm_win = kSampThreads;
  }
  __syncthreads();
  double before = 0.0, total = 0.0;
  for (int w = 0; w < kSampThreads / 32; ++w) {
    if (w < warp) before += sm_w[w];
    total += sm_w[w];
  }
  // prefix masses are monotone in tid (non-negative terms, fixed order), so
  // the owner of u is the first thread whose inclusive prefix exceeds it
  const double hi = before + incl, lo = hi - c;
  const double u = philox_uniform53(seed, offset, static_cast<uint64_t>(r)) * total;
  if (c > 0.0 && u < hi) atomicMin(&sm_win, tid);
  __syncthreads();
  if (tid == sm_win) {
    // inverse CDF inside this thread's elements, in its scan order
    double acc = lo;
    int32_t tok = -1, last = -1;
    const double ML = static_cast<double>(M) * 1.4426950408889634;
    for (int i = tid; i < nvec && tok < 0; i += kSampThreads) {
      float f[E];
      SampElem<T>::unpack(v[i], f);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double pe = exp2(static_cast<double>(f[e]) * 1.4426950408889634 - ML);
        if (pe > 0.0) last = i * E + e;
        acc += pe;
        if (tok < 0 && u < acc) tok = i * E + e;
      }
    }
    sm_tok = (tok < 0) ? last : tok;  // rounding at the interval's upper edge
  }
  if (tid == kSampThreads - 1) sm_tot = total;
  __syncthreads();
  if (tid == 0) {
    int32_t tok = sm_tok;
    if (tok < 0) tok = 0;  // non-finite row: reported through lp (NaN)
    const double lse = static_cast<double>(M) + log(sm_tot);
    tokens[r] = tok;
    if (lp_tok) lp_tok[r] = static_cast<double>(SampElem<T>::at(rowp, tok)) - lse;
  }
}

__global__ void blp_from_tokens_kernel(const double* __restrict__ lp_tok, int64_t n_chunks, int64_t T,
                                       float* __restrict__ blp, double* __restrict__ lp_chunk) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= n_chunks) return;
  const double lp = pairwise_sum([&](int64_t i) { return lp_tok[q * T + i]; }, 0, T);
  if (blp) blp[q] = static_cast<float>(lp);  // the sampler stores f32 (runtime.py:698)
  if (lp_chunk) lp_chunk[q] = lp;
}

}  // namespace dvla

using namespace dvla;

extern "C" int dvla_token_sample(const void* logits, int dtype, int64_t R, int64_t V, int64_t T,
                                 uint64_t seed, uint64_t offset, int32_t* tokens,
                                 double* lp_tok, float* blp, double* lp_chunk, void* stream) {
  if (R < 0 || V < 1 || T < 1 || (R % T) != 0)
    return fail(DVLA_ERR_USAGE, "token_sample: need R >= 0, V >= 1, T >= 1 and R %% T == 0");
  if (dtype != DVLA_BF16 && dtype != DVLA_F32) return fail(DVLA_ERR_USAGE, "dtype must be bf16 or f32");
  const int E = dtype == DVLA_BF16 ? 8 : 4;
  if ((V % E) != 0 || (reinterpret_cast<uintptr_t>(logits) % 16) != 0)
    return fail(DVLA_ERR_USAGE, "token_sample: rows must be 16-byte aligned multiples");
  if (!tokens || ((blp || lp_chunk) && !lp_tok)) return fail(DVLA_ERR_USAGE, "null pointer argument");
  if (R == 0) return DVLA_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t stop;
  prof_begin(st, &stop);
  if (dtype == DVLA_BF16)
    tok_sample_kernel<__nv_bfloat16><<<static_cast<unsigned>(R), kSampThreads, 0, st>>>(
        logits, V, seed, offset, tokens, lp_tok);
  else
    tok_sample_kernel<float><<<static_cast<unsigned>(R), kSampThreads, 0, st>>>(
        logits, V, seed, offset, tokens, lp_tok);
  prof_end(st, stop);
  if (int rc = launch_check("tok_sample_kernel")) return rc;
  if (blp || lp_chunk) {
    const int64_t nq = R / T;
    blp_from_tokens_kernel<<<static_cast<unsigned>((nq + 127) / 128), 128, 0, st>>>(lp_tok, nq, T,
                                                                                    blp, lp_chunk);
    return launch_check("blp_from_tokens_kernel");
  }
  return DVLA_OK;
}
