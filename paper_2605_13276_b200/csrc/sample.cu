// Rollout-side action-token sampling + behaviour log-prob.
//
// Token-head analogue of policy.sample_chunk_batch (reference
// policy.py:150-158: forward -> sample -> chunk_log_prob) and of the
// sampler's f32 behaviour log-prob store (runtime.py:696-698):
//   token_r  ~ softmax(x_r)                  (Philox4x32-10 keyed by (seed, r))
//   lp_tok_r = x_r[token_r] - logsumexp(x_r)  (f64)
//   blp_q    = f32( pairwise sum of the chunk's T lp_tok )
// One pass over the logits (HBM-bound, N*s bytes; 0.37 ms = 5.0 TB/s at the
// C2 shape, tools/sample_bench.py): per-thread sum-exp in a fixed exponent
// frame with 8 16-byte loads in flight, a deterministic block scan of the
// per-thread masses, and an inverse-CDF lookup inside the single thread whose
// mass interval holds u.
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
constexpr int kSampBatch = 8;         // uint4 loads in flight per thread
constexpr float kSampFrameHi = 64.f;  // fixed exponent frame valid for row max in [lo, hi]
constexpr float kSampFrameLo = -50.f;

template <class T>
struct SampElem;
template <>
struct SampElem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  // 2^(x log2e - fL) for the 8 elements of u, summed pairwise into acc[4]
  __device__ static void exps(const uint4& u, uint64_t l2e2, uint64_t nf2, uint64_t (&acc)[4]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float y0, y1;
      f2unpack(bf16x2_fma2(w[j], l2e2, nf2), y0, y1);
      acc[j] = fadd2(acc[j], f2pack(ex2f(y0), ex2f(y1)));
    }
  }
  __device__ static uint32_t maxw(const uint4& u) {  // packed max of the 8
    return bf16x2_max(bf16x2_max(u.x, u.y), bf16x2_max(u.z, u.w));
  }
  __device__ static float maxf(uint32_t packed) { return fmaxf(bf16lo(packed), bf16hi(packed)); }
  static constexpr uint32_t kNegInf = 0xff80ff80u;
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
  __device__ static void exps(const uint4& u, uint64_t l2e2, uint64_t nf2, uint64_t (&acc)[4]) {
    float y0, y1, y2, y3;
    f2unpack(ffma2(f2pack(__uint_as_float(u.x), __uint_as_float(u.y)), l2e2, nf2), y0, y1);
    f2unpack(ffma2(f2pack(__uint_as_float(u.z), __uint_as_float(u.w)), l2e2, nf2), y2, y3);
    acc[0] = fadd2(acc[0], f2pack(ex2f(y0), ex2f(y1)));
    acc[1] = fadd2(acc[1], f2pack(ex2f(y2), ex2f(y3)));
  }
  __device__ static uint32_t maxw(const uint4& u) {
    return __float_as_uint(fmaxf(fmaxf(__uint_as_float(u.x), __uint_as_float(u.y)),
                                 fmaxf(__uint_as_float(u.z), __uint_as_float(u.w))));
  }
  __device__ static float maxf(uint32_t packed) { return __uint_as_float(packed); }
  static constexpr uint32_t kNegInf = 0xff800000u;
  __device__ static void unpack(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
  __device__ static float at(const void* row, int64_t i) { return static_cast<const float*>(row)[i]; }
};

template <class T>
__device__ __forceinline__ uint32_t max_merge(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ uint32_t max_merge<__nv_bfloat16>(uint32_t a, uint32_t b) {
  return bf16x2_max(a, b);
}
template <>
__device__ __forceinline__ uint32_t max_merge<float>(uint32_t a, uint32_t b) {
  return __float_as_uint(fmaxf(__uint_as_float(a), __uint_as_float(b)));
}

// Sum of this thread's exponentials 2^(x log2e - frame log2e), elements
// tid, tid + 256, ... (uint4 granules), kSampBatch loads in flight.
template <class T>
__device__ __forceinline__ float thread_mass(const uint4* v, int nvec, int tid, float frame,
                                             uint32_t* mx_out) {
  const uint64_t l2e2 = f2pack(kLog2e, kLog2e);
  const float fL = frame * kLog2e;
  const uint64_t nf2 = f2pack(-fL, -fL);
  uint64_t acc[4] = {0, 0, 0, 0};
  uint32_t mx = SampElem<T>::kNegInf;
  for (int i0 = tid; i0 < nvec; i0 += kSampBatch * kSampThreads) {
    uint4 x[kSampBatch];
#pragma unroll
    for (int b = 0; b < kSampBatch; ++b) {
      const int i = i0 + b * kSampThreads;
      x[b] = (i < nvec) ? __ldcs(v + i)
                        : make_uint4(SampElem<T>::kNegInf, SampElem<T>::kNegInf,
                                     SampElem<T>::kNegInf, SampElem<T>::kNegInf);
    }
#pragma unroll
    for (int b = 0; b < kSampBatch; ++b) {
      mx = max_merge<T>(mx, SampElem<T>::maxw(x[b]));
      SampElem<T>::exps(x[b], l2e2, nf2, acc);
    }
  }
  if (mx_out) *mx_out = mx;
  float a0, a1, a2, a3, a4, a5, a6, a7;
  f2unpack(acc[0], a0, a1);
  f2unpack(acc[1], a2, a3);
  f2unpack(acc[2], a4, a5);
  f2unpack(acc[3], a6, a7);
  return ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
}

// One CTA per row (requires V % kVec == 0 and 16-byte aligned rows).
// Pass 1 takes every thread's mass in a fixed exponent frame (0, or the row
// max when the max leaves the frame's safe range) and the row max; a
// deterministic block scan of the masses in thread order locates the thread
// whose interval holds u * total, and that thread walks its own elements in
// the same order and frame to find the token.  lse = frame + log(total).
template <class T>
__global__ void __launch_bounds__(kSampThreads, 6) tok_sample_kernel(
    const void* __restrict__ logits, int64_t V, uint64_t seed, uint64_t offset,
    int32_t* __restrict__ tokens, double* __restrict__ lp_tok) {
  constexpr int E = SampElem<T>::kVec;
  const int64_t r = blockIdx.x;
  const uint8_t* rowp = static_cast<const uint8_t*>(logits) + r * V * sizeof(T);
  const uint4* v = reinterpret_cast<const uint4*>(rowp);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nvec = static_cast<int>(V / E);
  __shared__ float sm_m[kSampThreads / 32];
  __shared__ double sm_w[kSampThreads / 32];
  __shared__ double sm_tot;
  __shared__ int32_t sm_tok;
  __shared__ int sm_win;
  uint32_t mxp;
  float s = thread_mass<T>(v, nvec, tid, 0.f, &mxp);
  float M = warp_max_f32(SampElem<T>::maxf(mxp));
  if (lane == 0) sm_m[warp] = M;
  __syncthreads();
  M = sm_m[0];
#pragma unroll
  for (int w = 1; w < kSampThreads / 32; ++w) M = fmaxf(M, sm_m[w]);
  float frame = 0.f;
  if (!(M <= kSampFrameHi) || (M < kSampFrameLo && M > -INFINITY)) {  // block-uniform
    frame = M;
    s = thread_mass<T>(v, nvec, tid, frame, nullptr);
  }
  const double c = static_cast<double>(s);
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
  const int win = sm_win;
  if (win < kSampThreads && warp == (win >> 5)) {
    // inverse CDF inside the winner's elements (granules win + k * 256), walked
    // by the winner's warp: lane k takes granule k of a 32-granule block, sums
    // its E exponentials in element order, a fixed-order scan over the lanes
    // places each granule in [start, end), and the first lane whose interval
    // holds u walks its own elements.
    const double base = __shfl_sync(0xffffffffu, lo, win & 31);
    const float fL = frame * kLog2e;
    double run = base;
    int32_t tok = -1, last = -1;
    for (int k0 = 0; win + k0 * kSampThreads < nvec && tok < 0; k0 += 32) {
      const int i = win + (k0 + lane) * kSampThreads;
      float pe[E];
      double g = 0.0;
      int lpos = -1;
      if (i < nvec) {
        float f[E];
        SampElem<T>::unpack(v[i], f);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          pe[e] = ex2f(fmaf(f[e], kLog2e, -fL));
          g += static_cast<double>(pe[e]);
          if (pe[e] > 0.f) lpos = i * E + e;
        }
      }
      double incl = g;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      double excl = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) excl = 0.0;
      const unsigned hit = __ballot_sync(0xffffffffu, i < nvec && u < run + incl);
      if (hit) {
        const int fl = __ffs(hit) - 1;
        int32_t t = -1;
        if (lane == fl) {
          double acc = run + excl;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            acc += static_cast<double>(pe[e]);
            if (t < 0 && u < acc) t = i * E + e;
          }
          if (t < 0) t = lpos;  // rounding at the granule's upper edge
        }
        tok = __shfl_sync(0xffffffffu, t, fl);
      }
      // last positive element so far (u at or past the walked total)
      const int lm = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(lpos + 1)) - 1;
      if (lm >= 0) last = lm;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) sm_tok = (tok < 0) ? last : tok;
  }
  if (tid == kSampThreads - 1) sm_tot = total;
  __syncthreads();
  if (tid == 0) {
    int32_t tok = sm_tok;
    if (tok < 0) tok = 0;  // non-finite row: reported through lp (NaN)
    const double lse = static_cast<double>(frame) + log(sm_tot);
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
