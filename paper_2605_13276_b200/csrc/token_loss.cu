// Fused GRPO action-token loss: log-softmax gather (forward) + clipped-ratio
// surrogate with group-normalised advantages + d loss / d logits (backward).
//
// Reference semantics (the per-chunk joint log-prob analogue of
// kernels/numba_backend.py:49-61 chunk_log_prob, with "one Gaussian dim"
// -> "one action token"):
//   lp_tok[r]  = x[r, tgt_r] - logsumexp_v x[r, v]                 (f64)
//   lp[q]      = sum_{t=0..T-1} lp_tok[q*T + t]   (numpy pairwise order, f64)
//   rho, loss, coeff per chunk           <- grpo.py:252-268 (grpo_math.cuh)
//   dlogits[r, v] = coeff[q] * (1[v == tgt_r] - softmax(x[r])_v)
// i.e. the chain rule of policy.backward_batch (grpo.py:277) through the
// token head instead of the Gaussian head (numba_backend.py:92-99).
//
// Kernels
//   tok_adv_kernel        advantages per group (bit-exact, grpo.py:89-99)
//   tok_fused_kernel<TE,P> persistent, 1 CTA/SM, warp-specialised: a loader
//                         warp streams logits rows (bf16 or f32; P = 1, 2 or
//                         4 SMEM pieces per row) HBM->SMEM with TMA bulk
//                         copies, 20 compute warps take max / sum-exp and
//                         later write dlogits in place in SMEM, a tail /
//                         prep warp pair turns partials into lp_tok and
//                         chunk coefficients, a store warp streams dlogits
//                         out with TMA bulk stores.  Each row is read from
//                         HBM once (the second read hits L2): compulsory
//                         traffic 2*N*s bytes.  C2: bf16 0.67 ms, f32 1.29 ms.
//   tok_rows_kernel<T>    unfused forward (any dtype / alignment / V)
//   tok_chunk_kernel      unfused per-chunk coefficient
//   tok_bwd_kernel<T>     unfused backward (re-reads logits: 3*N*s traffic)
//   grpo_epilogue_kernel  loss / stats / abort detection in canonical order
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "grpo_math.cuh"

namespace dvla {

#ifndef DVLA_FUSED_W
#define DVLA_FUSED_W 20
#endif
#ifndef DVLA_PDL
#define DVLA_PDL 1  // programmatic dependent launch: adv -> fused -> epilogue overlap their launches
#endif
#ifndef DVLA_FUSED_CTAS
#define DVLA_FUSED_CTAS 1
#endif
constexpr int kFusedComputeWarps = DVLA_FUSED_W;
constexpr int kFusedCtasPerSm = DVLA_FUSED_CTAS;  // resident fused CTAs per SM
constexpr size_t kFusedSmemCap = (228u * 1024u) / DVLA_FUSED_CTAS - 1024u;
constexpr int kFusedComputeThreads = kFusedComputeWarps * 32;
constexpr int kFusedStages = 3;    // SMEM row stages and B coefficient slots
#ifndef DVLA_A_SLOTS
#define DVLA_A_SLOTS 8
#endif
#ifndef DVLA_B_UNROLL
#define DVLA_B_UNROLL 2   // phase-B granules per loop iteration
#endif
constexpr int kASlots = DVLA_A_SLOTS;  // A-row partial slots (coef-warp slack)
constexpr int kBUnroll = DVLA_B_UNROLL;
constexpr uint64_t kSpinTimeoutNs = 4000000000ull;  // 4 s: report, never hang

struct TokParams {
  const void* logits;
  const int32_t* tokens;
  const float* blp;
  const double* adv;
  void* dlogits;
  double* lp_tok;
  double* lse;
  double* lp_chunk;
  double* coeff;
  uint32_t* err;
  int64_t R, V, T, C, n_chunks;
  double w, clip_eps, kl_coeff;
};

enum : uint32_t { kErrToken = 1u, kErrTimeout = 2u };

// Optional per-role cycle counters for the fused kernel (set by
// dvla_debug_fused_counters; null in normal runs -> no clock reads).
__device__ unsigned long long* g_dbg = nullptr;
__device__ unsigned long long* g_dbg_cta = nullptr;  // per-CTA (start, end) globaltimer ns
#define DBG_T0() const long long _t0 = dbg ? clock64() : 0
#define DBG_ADD(i) \
  if (dbg) atomicAdd(dbg + (i), static_cast<unsigned long long>(clock64() - _t0))

// lp_tok not yet published (tok_adv_kernel fills it before the fused kernel;
// a finite ~1.4e306, never a log-probability)
constexpr long long kLpPending = 0x7f7f7f7f7f7f7f7fll;
constexpr long long kNaN64 = 0x7ff8000000000000ll;

// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in
// the stream still runs; it must pass pdl_wait() before touching anything the
// predecessor writes.  pdl_trigger() lets the successor launch early.  Both
// are no-ops without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------ advantages
// (also marks n_fill token log-probs pending for the fused kernel's polls)
__global__ void tok_adv_kernel(const float* __restrict__ rewards, int64_t n_groups, int64_t G,
                               double delta, double* __restrict__ adv,
                               uint32_t* __restrict__ reward_bad, double* __restrict__ lp_fill,
                               int64_t n_fill, uint32_t* __restrict__ err) {
  pdl_trigger();  // the fused kernel waits (pdl_wait) where it reads what this writes
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // the error word of this call: every writer (tail / prep warps, unfused
  // kernels) runs after this kernel, so no separate memset is needed
  if (g == 0 && err) *err = 0u;
  for (int64_t i = g; i < n_fill; i += gridDim.x * (int64_t)blockDim.x)
    reinterpret_cast<long long*>(lp_fill)[i] = kLpPending;
  if (g >= n_groups) return;
  const float* r = rewards + g * G;
  double* a = adv + g * G;
  auto get = [&](int64_t i) { return static_cast<double>(r[i]); };
  group_advantages(get, G, delta, [&](int64_t i, double v) { a[i] = v; });
  uint32_t bad = 0;
  for (int64_t i = 0; i < G; ++i) bad |= !isfinite(r[i]);
  reward_bad[g] = bad;
}

__global__ void adv_f64_kernel(const double* __restrict__ rewards, int64_t n_groups, int64_t G,
                               double delta, double* __restrict__ adv) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const double* r = rewards + g * G;
  double* a = adv + g * G;
  group_advantages([&](int64_t i) { return r[i]; }, G, delta,
                   [&](int64_t i, double v) { a[i] = v; });
}

// Chunk-joint log-prob: numpy pairwise order over the chunk's T token
// log-probs (the order numpy_backend.chunk_log_prob's .sum(axis=1) uses for
// the Gaussian head, numpy_backend.py:39-49).  One warp, T <= 128; the
// result is valid in every lane.  vals[m] holds lp_tok[32*m + lane].
__device__ __forceinline__ double warp_pairwise_small(const double (&vals)[4], int T, int lane) {
  double res;
  if (T < 8) {
    res = 0.0;
    for (int t = 0; t < T; ++t) res = __dadd_rn(res, __shfl_sync(0xffffffffu, vals[0], t));
    return res;
  }
  const int n8 = T - (T % 8);
  // lanes 0..7: r_j = a[j] + a[j+8] + ... (sequential), j = lane
  double r = 0.0;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    if (8 * m >= n8) break;
    const int src = 8 * (m & 3) + (lane & 7);
    double x = 0.0;
    switch (m >> 2) {
      case 0: x = __shfl_sync(0xffffffffu, vals[0], src); break;
      case 1: x = __shfl_sync(0xffffffffu, vals[1], src); break;
      case 2: x = __shfl_sync(0xffffffffu, vals[2], src); break;
      default: x = __shfl_sync(0xffffffffu, vals[3], src); break;
    }
    r = (m == 0) ? x : __dadd_rn(r, x);
  }
  // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))
  double p1 = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
  double p2 = __dadd_rn(p1, __shfl_xor_sync(0xffffffffu, p1, 2));
  double p4 = __dadd_rn(p2, __shfl_xor_sync(0xffffffffu, p2, 4));
  res = __shfl_sync(0xffffffffu, p4, 0);
  for (int t = n8; t < T; ++t) {
    double x;
    switch (t >> 5) {
      case 0: x = __shfl_sync(0xffffffffu, vals[0], t & 31); break;
      case 1: x = __shfl_sync(0xffffffffu, vals[1], t & 31); break;
      case 2: x = __shfl_sync(0xffffffffu, vals[2], t & 31); break;
      default: x = __shfl_sync(0xffffffffu, vals[3], t & 31); break;
    }
    res = __dadd_rn(res, x);
  }
  return res;
}

// Chunk lp for any T from global memory (numpy pairwise order), one thread.
__device__ __forceinline__ double chunk_lp_pairwise(const double* __restrict__ lp_tok, int64_t T) {
  return pairwise_sum([&](int64_t i) { return __ldcg(lp_tok + i); }, 0, T);
}

// ---------------------------------------------------- fused kernel
//
// One CTA per SM (persistent), rows assigned round-robin (row = cta + k*grid).
// (Below, "row" = one SMEM piece: a row longer than a stage is P pieces,
// u = k P + p, with the lag L counted in pieces; see tok_fused_kernel.)
// Every CTA walks one op sequence: A(0..L-1), then A(k), B(k-L), ..., B(n-1):
//   A(k)  row k streamed HBM -> SMEM by TMA; the compute warps take warp
//         max (packed bf16) / sum-exp (FFMA2 + MUFU ex2 + FADD2) partials;
//         the tail warp combines them into lse (f64) and publishes lp_tok
//         (target logit - lse) to global memory.
//   B(k)  row k streamed again -- from L2, L rounds (~L*148*64 KB) after
//         A(k) -- the prep warp waits for the chunk to be complete on all
//         CTAs (long done by then), sums its T token log-probs (numpy
//         pairwise order) and evaluates the GRPO coefficient; the compute
//         warps overwrite the row in SMEM with d loss / d logits and the
//         store warp streams it out with one TMA bulk store.
// HBM traffic stays at the compulsory 2*N*s bytes while the L-round lag
// hides the cross-CTA chunk dependency.  A(k+L) precedes B(k) on every CTA
// and the tail warp never waits on another CTA, so the chunk wait is
// deadlock-free while all CTAs are co-resident (grid <= #SMs, T <= grid).
//
// Warp roles: 0..W-1 compute, W loader, W+1 tail, W+2 store, W+3 prep.
// Cross-CTA: lp_tok values are published with single 8-byte relaxed stores
// into a buffer pre-filled with a pending marker; the prep warp polls the
// chunk's values themselves (one L2 round trip yields the data), so neither
// side needs a counter or a release fence.
// Barriers (every barrier completes once per use of its own ring index, and
// every waiter walks its ring in order, so parity never aliases):
//   full[s], empty[s]  per SMEM stage s = op % 3: loader <-> compute warps
//                      (A: free once read; B: freed by the store warp, one
//                      arrival worth W, once its bulk copy has read it)
//   adoneA[a % 8]      compute -> tail, per A op a (SMEM partial slot a % 8)
//   afree[a % 8]       tail -> compute, partial slot consumed
//   tdone[k % 8]       tail -> prep, (lse, target) of row k in the ring
//   cfullB[b % 3]      prep -> compute, per B op b (coefficient slot b % 3)
//   adoneB[b % 3]      compute -> prep (coefficient slot b % 3 consumed)
//   bdone[b % 3]       compute -> store, B row b written in SMEM
// The op sequence and barrier protocol are model-checked for deadlock,
// races and parity aliasing (tests/test_fused_protocol.py).
constexpr int kWarpLoader = kFusedComputeWarps;
constexpr int kTailWarp = kFusedComputeWarps + 1;
constexpr int kWarpStore = kFusedComputeWarps + 2;
constexpr int kPrepWarp = kFusedComputeWarps + 3;
constexpr int kFusedThreadsWS = (kFusedComputeWarps + 4) * 32;

constexpr int kLagRounds = 3;  // pieces; measured best on B200 (round 2: tools/lag_ab.sh, 5 alternating sustained pairs)
constexpr int kRing = 8;       // (lse, target) rows in flight tail -> prep; lag <= 8P - 1
constexpr float kFrameHi = 64.f;   // fixed-frame sum-exp range of a warp max (see phase A)
constexpr float kFrameLo = -50.f;

struct FusedSmem {
  uint64_t full[kFusedStages];
  uint64_t empty[kFusedStages];
  uint64_t adoneA[kASlots];
  uint64_t afree[kASlots];
  uint64_t adoneB[kFusedStages];
  uint64_t cfullB[kFusedStages];
  uint64_t bdone[kFusedStages];  // compute -> store warp, B row b % 3 written in SMEM
  uint64_t tdone[kRing];         // tail -> prep warp, (lse, target) of row k % kRing
  double ws[kASlots][kFusedComputeWarps];
  float wm[kASlots][kFusedComputeWarps];
  float kval[kFusedStages];   // lse*log2e - log2|c|
  float tval[kFusedStages];   // target column c (1 - p_t) = -c expm1(lp_tok), f64 -> f32
  uint32_t mode[kFusedStages];  // 0 zero row, 1 finite c (bit 31: c > 0), 2 non-finite c
  int32_t tgt[kFusedStages];
  float xt[kASlots];       // gathered target logit of A slot
  int32_t tgta[kASlots];   // its token id (-1: out of range)
  double ring_lse[kRing];
  double ring_lp[kRing];   // the row's lp_tok (target column of phase B)
  int32_t ring_tgt[kRing];
};

// op n of a CTA with nloc rows and lag L: (is_B, local row)
__device__ __forceinline__ void op_of(int n, int nloc, int L, bool* isB, int* k) {
  const int Le = nloc < L ? nloc : L;  // effective lag
  if (n < Le) {
    *isB = false;
    *k = n;
    return;
  }
  const int m = n - Le;  // pairs (A(Le + j), B(j)) for j < nloc - Le, then B tail
  const int pairs = nloc - Le;
  if (m < 2 * pairs) {
    *isB = (m & 1) != 0;
    *k = (m & 1) ? (m >> 1) : (Le + (m >> 1));
    return;
  }
  *isB = true;
  *k = pairs + (m - 2 * pairs);
}

#ifndef DVLA_POLL_NS
#define DVLA_POLL_NS 512  // prep warp: back-off between polls of a chunk's token log-probs
#endif
#ifndef DVLA_FULL_SPIN
#define DVLA_FULL_SPIN 0
#endif
#ifndef DVLA_CFULL_WAIT
// compute warps wait for a phase-B coefficient with the hardware try_wait
// (suspend until the barrier flips) rather than a nanosleep back-off loop:
// the back-off loop issued ~22 % of the kernel's instructions; sustained
// power-capped step 0.3-0.6 % faster (round 2, tools/sustained_variants.sh)
#define DVLA_CFULL_WAIT 1
#endif
#ifndef DVLA_POLY_WORDS
#define DVLA_POLY_WORDS 0
#endif
#ifndef DVLA_A_EVICT_LAST
#define DVLA_A_EVICT_LAST 0   // phase-A loads with an L2 evict_last hint (experiment)
#endif
#ifndef DVLA_ACC_INPLACE
#define DVLA_ACC_INPLACE 1
#endif
constexpr int kPolyWords = DVLA_POLY_WORDS;  // bf16 phase-B words per granule on the FMA pipe

// 2^y on both lanes of a packed f32 pair without MUFU: y = j + f with j =
// round(y) (1.5*2^23 shifter), 2^f by a degree-3 minimax polynomial on
// [-1/2, 1/2] (max relative error 7.5e-5), 2^j added into the exponent
// field.  y is clamped below at -126 (2^-126 stands in for every smaller
// value, including 2^-inf: 1e-38 against a zero, invisible at bf16's
// gradient scale); y is at most log2|c| here, never near overflow.
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t y2) {
  float y0, y1;
  f2unpack(y2, y0, y1);
  y2 = f2pack(fmaxf(y0, -126.f), fmaxf(y1, -126.f));
  constexpr float kShift = 12582912.f;  // 1.5 * 2^23
  const uint64_t t2 = fadd2(y2, f2pack(kShift, kShift));
  const uint64_t j2 = fadd2(t2, f2pack(-kShift, -kShift));
  const uint64_t f2 = ffma2(j2, f2pack(-1.f, -1.f), y2);
  uint64_t p2 = ffma2(f2, f2pack(0.05517134f, 0.05517134f), f2pack(0.24261035f, 0.24261035f));
  p2 = ffma2(p2, f2, f2pack(0.69326097f, 0.69326097f));
  p2 = ffma2(p2, f2, f2pack(0.99992812f, 0.99992812f));
  float t0, t1, p0, p1;
  f2unpack(t2, t0, t1);
  f2unpack(p2, p0, p1);
  // t's low mantissa bits hold j (two's complement); j << 23 wraps the
  // shifter's own bits out of the word
  const uint32_t r0 = __float_as_uint(p0) + (__float_as_uint(t0) << 23);
  const uint32_t r1 = __float_as_uint(p1) + (__float_as_uint(t1) << 23);
  return f2pack(__uint_as_float(r0), __uint_as_float(r1));
}

// Element traits of the fused kernel: 16-byte granules of bf16 (8) or f32 (4)
template <class TE>
struct FusedElem;
template <>
struct FusedElem<__nv_bfloat16> {
  static constexpr int kE = 8;
  static constexpr uint32_t kNegInf = 0xff80ff80u;
  static constexpr uint32_t kSign = 0x80008000u;   // both halves
  static constexpr uint32_t kNaN = 0x7fc07fc0u;
  __device__ static uint32_t max16(uint32_t m, const uint4& x) {
    return bf16x2_max(m, bf16x2_max(bf16x2_max(x.x, x.y), bf16x2_max(x.z, x.w)));
  }
  __device__ static float maxf(uint32_t m) { return fmaxf(bf16lo(m), bf16hi(m)); }
  __device__ static uint32_t max2(uint32_t a, uint32_t b) { return bf16x2_max(a, b); }
  // acc += 2^(x log2e + off) over the granule (packed f32 pairs)
  __device__ static void exps(const uint4& x, uint64_t l2e2, uint64_t off2, uint64_t (&acc)[4]) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float y0, y1;
      f2unpack(bf16x2_fma2(w[j], l2e2, off2), y0, y1);
      fadd2_acc(acc[j], f2pack(ex2f(y0), ex2f(y1)));
    }
  }
  // -sign(c) 2^(x log2e - K) for the granule, in place.  kPolyWords of the
  // four words take their exponentials on the FMA pipe (exp2_poly2: degree-3
  // polynomial, 7.5e-5 relative, far below the bf16 output's 2^-9), the rest
  // on MUFU: phase B's ex2 load moves off the XU pipe the forward shares.
  __device__ static uint4 grad(const uint4& x, uint64_t l2e2, uint64_t nK2, uint32_t sgn) {
    auto e2 = [&](uint32_t w) {
      float y0, y1;
      f2unpack(bf16x2_fma2(w, l2e2, nK2), y0, y1);
      return pack_bf16x2(ex2f(y0), ex2f(y1)) ^ sgn;
    };
    auto e2p = [&](uint32_t w) {
      float y0, y1;
      f2unpack(exp2_poly2(bf16x2_fma2(w, l2e2, nK2)), y0, y1);
      return pack_bf16x2(y0, y1) ^ sgn;
    };
    return make_uint4(kPolyWords > 0 ? e2p(x.x) : e2(x.x), kPolyWords > 2 ? e2p(x.y) : e2(x.y),
                      kPolyWords > 1 ? e2p(x.z) : e2(x.z), kPolyWords > 3 ? e2p(x.w) : e2(x.w));
  }
  __device__ static float get(const void* base, int i) {
    return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]);
  }
  __device__ static void put(void* base, int i, float v) {
    static_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16_rn(v);
  }
};
template <>
struct FusedElem<float> {
  static constexpr int kE = 4;
  static constexpr uint32_t kNegInf = 0xff800000u;
  static constexpr uint32_t kSign = 0x80000000u;
  static constexpr uint32_t kNaN = 0x7fc00000u;
  __device__ static uint32_t max16(uint32_t m, const uint4& x) {
    return __float_as_uint(fmaxf(__uint_as_float(m),
                                 fmaxf(fmaxf(__uint_as_float(x.x), __uint_as_float(x.y)),
                                       fmaxf(__uint_as_float(x.z), __uint_as_float(x.w)))));
  }
  __device__ static float maxf(uint32_t m) { return __uint_as_float(m); }
  __device__ static uint32_t max2(uint32_t a, uint32_t b) {
    return __float_as_uint(fmaxf(__uint_as_float(a), __uint_as_float(b)));
  }
  __device__ static void exps(const uint4& x, uint64_t l2e2, uint64_t off2, uint64_t (&acc)[4]) {
    float y0, y1, y2, y3;
    f2unpack(ffma2(f2pack(__uint_as_float(x.x), __uint_as_float(x.y)), l2e2, off2), y0, y1);
    f2unpack(ffma2(f2pack(__uint_as_float(x.z), __uint_as_float(x.w)), l2e2, off2), y2, y3);
    acc[0] = fadd2(acc[0], f2pack(ex2f(y0), ex2f(y1)));
    acc[1] = fadd2(acc[1], f2pack(ex2f(y2), ex2f(y3)));
  }
  __device__ static uint4 grad(const uint4& x, uint64_t l2e2, uint64_t nK2, uint32_t sgn) {
    float y0, y1, y2, y3;
    f2unpack(ffma2(f2pack(__uint_as_float(x.x), __uint_as_float(x.y)), l2e2, nK2), y0, y1);
    f2unpack(ffma2(f2pack(__uint_as_float(x.z), __uint_as_float(x.w)), l2e2, nK2), y2, y3);
    return make_uint4(__float_as_uint(ex2f(y0)) ^ sgn, __float_as_uint(ex2f(y1)) ^ sgn,
                      __float_as_uint(ex2f(y2)) ^ sgn, __float_as_uint(ex2f(y3)) ^ sgn);
  }
  __device__ static float get(const void* base, int i) { return static_cast<const float*>(base)[i]; }
  __device__ static void put(void* base, int i, float v) { static_cast<float*>(base)[i] = v; }
};

// TE: logits / dlogits element type; P: SMEM pieces per row (a row longer
// than a stage is streamed as P consecutive pieces: "virtual rows" u = k P + p
// in the op sequence; the tail warp combines the P pieces' partials).
template <class TE, int P>
__global__ void __launch_bounds__(kFusedThreadsWS, kFusedCtasPerSm)
    tok_fused_kernel(TokParams p, uint32_t stage_bytes, int piece_vec, int write_dl, int lag) {
  using FE = FusedElem<TE>;
  constexpr int E = FE::kE;
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  FusedSmem& S = *reinterpret_cast<FusedSmem*>(dyn_smem);
  uint8_t* bufs = dyn_smem + ((sizeof(FusedSmem) + 127) / 128) * 128;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t V = p.V;
  const int64_t row_bytes = V * static_cast<int64_t>(sizeof(TE));
  const int nvec_row = static_cast<int>(row_bytes / 16);
  const int64_t G = gridDim.x;
  const int nloc = (p.R > blockIdx.x) ? static_cast<int>((p.R - blockIdx.x + G - 1) / G) : 0;
  const int nvr = nloc * P;                       // virtual rows (pieces) of this CTA
  const int nops = write_dl ? 2 * nvr : nvr;
  const int L = write_dl ? lag : 1 << 30;         // lag in pieces; forward-only: A ops only
  auto row_of = [&](int k) { return static_cast<int64_t>(blockIdx.x) + k * G; };
  auto buf = [&](int s) { return bufs + static_cast<size_t>(s) * stage_bytes; };
  // granules [piece * piece_vec, piece * piece_vec + piece_len(piece)) of a row
  auto piece_len = [&](int piece) {
    const int lo = piece * piece_vec;
    return (nvec_row - lo < piece_vec) ? nvec_row - lo : piece_vec;
  };
  const int64_t T = p.T;
  unsigned long long* dbg = g_dbg;
  const long long t_kernel = dbg ? clock64() : 0;
  const unsigned long long t_kernel_ns = dbg ? globaltimer_ns() : 0;

  if (tid == 0) {
    for (int s = 0; s < kFusedStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], kFusedComputeWarps);
      mbar_init(&S.adoneB[s], kFusedComputeWarps);
      mbar_init(&S.cfullB[s], 1);
      mbar_init(&S.bdone[s], kFusedComputeWarps);
    }
    for (int s = 0; s < kASlots; ++s) {
      mbar_init(&S.adoneA[s], kFusedComputeWarps);
      mbar_init(&S.afree[s], 1);
    }
    for (int j = 0; j < kRing; ++j) mbar_init(&S.tdone[j], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint8_t* logits = static_cast<const uint8_t*>(p.logits);
  uint8_t* dl = static_cast<uint8_t*>(p.dlogits);
  pdl_trigger();  // the epilogue may launch now; it waits for this grid to finish

  // --------------------------------------------------------- loader warp
  if (warp == kWarpLoader) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
#if DVLA_A_EVICT_LAST
      const uint64_t pol_last = l2_policy_evict_last();
#endif
      for (int n = 0; n < nops; ++n) {
        const int s = static_cast<int>(n % kFusedStages);
        if (n >= kFusedStages) {
          DBG_T0();
          mbar_wait(&S.empty[s], static_cast<uint32_t>(((n / kFusedStages) - 1) & 1));
          DBG_ADD(8);
        }
        bool isB;
        int u;
        op_of(n, nvr, L, &isB, &u);
        const int piece = u % P;
        const uint32_t bytes = static_cast<uint32_t>(piece_len(piece)) * 16u;
        const uint8_t* src = logits + row_of(u / P) * row_bytes + int64_t{16} * piece * piece_vec;
        mbar_arrive_expect_tx(&S.full[s], bytes);
        if (isB)  // second (last) read of the piece: from L2, then evict
          tma_load_1d_evict_first(buf(s), src, bytes, &S.full[s], pol);
#if DVLA_A_EVICT_LAST
        else
          tma_load_1d_evict_first(buf(s), src, bytes, &S.full[s], pol_last);
#else
        else  // (an evict_last hint here measured no better: the lag keeps rows in L2)
          tma_load_1d(buf(s), src, bytes, &S.full[s]);
#endif
      }
    }
    return;
  }

  // ---------------------------------------------------------- store warp
  // B pieces are written in place in SMEM and streamed out with one bulk
  // copy each; the stage returns to the loader once the copy has read it.
  if (warp == kWarpStore) {
    if (!write_dl || lane != 0) return;
    int nb = 0;
    const uint64_t pol_ef = l2_policy_evict_first();
    for (int n = 0; n < nops; ++n) {
      bool isB;
      int u;
      op_of(n, nvr, L, &isB, &u);
      if (!isB) continue;
      const int s = static_cast<int>(n % kFusedStages);
      mbar_wait(&S.bdone[nb % kFusedStages], static_cast<uint32_t>((nb / kFusedStages) & 1));
      ++nb;
      const int piece = u % P;
      // dlogits are not re-read here: keep L2 for the rows B still needs
      tma_store_1d_evict_first(dl + row_of(u / P) * row_bytes + int64_t{16} * piece * piece_vec,
                               buf(s), static_cast<uint32_t>(piece_len(piece)) * 16u, pol_ef);
      bulk_commit();
      bulk_wait_read<0>();
      mbar_arrive_cnt(&S.empty[s], kFusedComputeWarps);
    }
    bulk_wait<0>();
    return;
  }

  // ----------------------------------------------------------- tail warp
  // Turns every row's per-warp (and per-piece) partials into lse (f64) and
  // lp_tok, publishes lp_tok (other CTAs' chunks wait for it, so this warp
  // never waits on anything but its own compute warps) and leaves (lse,
  // target) in the ring for the prep warp.
  if (warp == kTailWarp) {
    pdl_wait();  // lp_tok's pending fill (tok_adv_kernel) precedes every publish
    for (int k = 0; k < nloc; ++k) {
      const int64_t r = row_of(k);
      float mw[P];
      double sw[P];
      int32_t tgt = -1;
      float xt_f = __int_as_float(0x7fc00000);
#pragma unroll
      for (int pc = 0; pc < P; ++pc) {
        const int u = k * P + pc;
        const int sa = u % kASlots;
        mbar_wait(&S.adoneA[sa], static_cast<uint32_t>((u / kASlots) & 1));
        tgt = S.tgta[sa];
        const float x = S.xt[sa];
        if (!isnan(x)) xt_f = x;  // the piece that holds the target column
        mw[pc] = (lane < kFusedComputeWarps) ? S.wm[sa][lane] : -INFINITY;
        sw[pc] = (lane < kFusedComputeWarps) ? S.ws[sa][lane] : 0.0;
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.afree[sa]);  // partial slot sa consumed
      }
      // a NaN partial (NaN logit) or a +inf frame (+inf logit) poisons the row
      bool bad = false;
      float mlane = -INFINITY;
#pragma unroll
      for (int pc = 0; pc < P; ++pc) {
        bad |= lane < kFusedComputeWarps && (isnan(sw[pc]) || mw[pc] == INFINITY);
        if (lane < kFusedComputeWarps && sw[pc] > 0.0) mlane = fmaxf(mlane, mw[pc]);
      }
      const bool poison = __any_sync(0xffffffffu, bad);
      const float M = warp_max_f32(mlane);
      double term = 0.0;
#pragma unroll
      for (int pc = 0; pc < P; ++pc)
        if (lane < kFusedComputeWarps && sw[pc] > 0.0)
          term += sw[pc] * static_cast<double>(ex2f((mw[pc] - M) * kLog2e));
      term = warp_sum_f64(term);
      if (lane == 0) {
        const double lse =
            poison ? __longlong_as_double(kNaN64) : static_cast<double>(M) + log(term);
        double lp = static_cast<double>(xt_f) - lse;
        if (__double_as_longlong(lp) == kLpPending) lp = __longlong_as_double(kNaN64);
        if (tgt < 0) atomicOr(p.err, kErrToken);
        // published with one 8-byte store: other CTAs' prep warps poll the
        // value itself (no counter, no release fence on this path)
        st_relaxed_gpu_f64(p.lp_tok + r, lp);
        if (write_dl) {
          S.ring_lse[k % kRing] = lse;
          S.ring_lp[k % kRing] = lp;
          S.ring_tgt[k % kRing] = tgt;
          mbar_arrive(&S.tdone[k % kRing]);
        } else {
          p.lse[r] = lse;
        }
      }
      __syncwarp();
    }
    return;
  }

  // ----------------------------------------------------------- prep warp
  // For each row in order: wait until the row's chunk is complete on all
  // CTAs (its T published token log-probs are no longer pending; L rounds
  // after A, normally long done), sum them (numpy pairwise order), evaluate
  // rho, the clipped surrogate and the coefficient (every CTA computes the
  // same value from the same inputs) and hand them to the compute warps,
  // once per piece of the row.
  if (warp == kPrepWarp) {
    if (!write_dl) return;
    pdl_wait();  // advantages and the lp_tok pending fill
    const uint64_t t_start = globaltimer_ns();
    for (int k = 0; k < nloc; ++k) {
      const int64_t r = row_of(k);
      const int64_t q = r / T;
      // poll the chunk's T published token log-probs (at most 4 per lane)
      double pv[4];
      const double* lt = p.lp_tok + q * T;
      uint32_t spins = 0;
      const long long t_poll = dbg ? clock64() : 0;
      for (;;) {
        bool ready = true;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int64_t t = 32 * m + lane;
          pv[m] = (t < T) ? ld_relaxed_gpu_f64(lt + t) : 0.0;
          ready &= __double_as_longlong(pv[m]) != kLpPending;
        }
        if (__all_sync(0xffffffffu, ready)) break;
        __nanosleep(DVLA_POLL_NS);
        if ((++spins & 1023u) == 0 && globaltimer_ns() - t_start > kSpinTimeoutNs) {
          if (lane == 0) atomicOr(p.err, kErrTimeout);
          break;
        }
      }
      const float pblp = __ldg(p.blp + q);
      const double padv = __ldg(p.adv + q / p.C);
      if (dbg && lane == 0) atomicAdd(dbg + 4, static_cast<unsigned long long>(clock64() - t_poll));
      const double lp = warp_pairwise_small(pv, static_cast<int>(T), lane);
      {
        DBG_T0();
        mbar_wait(&S.tdone[k % kRing], static_cast<uint32_t>((k / kRing) & 1));  // own tail
        if (lane == 0) { DBG_ADD(5); }
      }
      uint32_t mode = 0u;
      float kval = 0.f, tval = 0.f;
      if (lane == 0) {
        ChunkTerms ct = chunk_terms(lp, static_cast<double>(pblp), padv, p.w, p.clip_eps,
                                    p.kl_coeff);
        const double cc = ct.coeff;
        if (r % T == 0) {  // one writer per chunk for the epilogue
          p.lp_chunk[q] = lp;
          p.coeff[q] = cc;
        }
        const double lse = S.ring_lse[k % kRing];
        if (cc == 0.0) {
          mode = 0u;
        } else if (!isfinite(cc)) {
          mode = 2u;
        } else {
          mode = 1u | ((cc > 0.0) ? 0x80000000u : 0u);
          kval = static_cast<float>(lse * 1.4426950408889634 - log2(fabs(cc)));
        }
        // 1 - p_t = -expm1(lp_tok) in f64: no cancellation when p_t -> 1
        tval = static_cast<float>(-cc * expm1(S.ring_lp[k % kRing]));
      }
      const int32_t tgt = S.ring_tgt[k % kRing];
#pragma unroll
      for (int pc = 0; pc < P; ++pc) {
        const int u = k * P + pc;
        const int sb = u % kFusedStages;
        if (u >= kFusedStages) {  // coefficient slot sb consumed by the compute warps
          DBG_T0();
          mbar_wait(&S.adoneB[sb], static_cast<uint32_t>(((u - kFusedStages) / kFusedStages) & 1));
          if (lane == 0) { DBG_ADD(6); }
        }
        if (lane == 0) {
          S.mode[sb] = mode;
          S.kval[sb] = kval;
          S.tval[sb] = tval;
          S.tgt[sb] = tgt;
          mbar_arrive(&S.cfullB[sb]);
        }
        __syncwarp();
      }
    }
    return;
  }

  // ------------------------------------------------------- compute warps
  int a = 0, b = 0;  // A / B op counters (virtual rows)
  const uint64_t l2e2 = f2pack(kLog2e, kLog2e);
  for (int n = 0; n < nops; ++n) {
    const int s = static_cast<int>(n % kFusedStages);
    const uint32_t ph = static_cast<uint32_t>((n / kFusedStages) & 1);
    bool isB;
    int u;
    op_of(n, nvr, L, &isB, &u);
    const int piece = u % P;
    const int nvec = piece_len(piece);
    const int elem0 = piece * piece_vec * E;  // first element of this piece in its row
    {
      DBG_T0();
#if DVLA_FULL_SPIN
      while (!mbar_test_wait(&S.full[s], ph)) {
      }
#else
      mbar_wait(&S.full[s], ph);
#endif
      if (tid == 0) { DBG_ADD(0); }
    }
    if (!isB) {
      const int32_t tg = (tid == 0) ? __ldg(p.tokens + row_of(u / P)) : 0;  // used at the end
      // One pass: exponentials in the fixed frame 2^(x log2e) (no max
      // subtraction) with the max alongside.  The frame is exact enough when
      // the warp max lies in [kFrameLo, kFrameHi] (no f32 overflow of <= 8
      // terms per accumulator; terms flushed below 2^-126 are < e^-37 of the
      // max); otherwise (rare: huge or very negative logits) the warp redoes
      // its slice relative to its own max.  The tail combines (frame, sum)
      // pairs of all warps and pieces.
      const uint4* v = reinterpret_cast<const uint4*>(buf(s));
      uint32_t mx = FE::kNegInf;
      uint64_t acc[4] = {0, 0, 0, 0};  // packed (0.f, 0.f)
      // bf16: two granules per iteration into two accumulator sets, each
      // accumulator updated in place once per iteration (one set made ptxas
      // copy the pair sums back every iteration); f32 rows keep one set
      // (measured 1.4 % faster there: tools/f32_time.py)
      if constexpr (DVLA_ACC_INPLACE && sizeof(TE) == 2) {
        uint64_t acc2[4] = {0, 0, 0, 0};
        uint32_t mx2 = FE::kNegInf;
        int i = tid;
        for (; i + kFusedComputeThreads < nvec; i += 2 * kFusedComputeThreads) {
          const uint4 x = v[i], y = v[i + kFusedComputeThreads];
          mx = FE::max16(mx, x);
          mx2 = FE::max16(mx2, y);
          FE::exps(x, l2e2, 0, acc);
          FE::exps(y, l2e2, 0, acc2);
        }
        if (i < nvec) {
          const uint4 x = v[i];
          mx = FE::max16(mx, x);
          FE::exps(x, l2e2, 0, acc);
        }
        mx = FE::max2(mx, mx2);
#pragma unroll
        for (int j = 0; j < 4; ++j) fadd2_acc(acc[j], acc2[j]);
      } else {
#pragma unroll 2
        for (int i = tid; i < nvec; i += kFusedComputeThreads) {
          const uint4 x = v[i];
          mx = FE::max16(mx, x);
          FE::exps(x, l2e2, 0, acc);
        }
      }
      const float wmax = warp_max_f32(FE::maxf(mx));
      float m = 0.f;  // frame of this warp's partial
      if (!(wmax <= kFrameHi) || (wmax < kFrameLo && wmax > -INFINITY)) {  // warp-uniform
        m = wmax;
        const float mL = m * kLog2e;
        const uint64_t nmL2 = f2pack(-mL, -mL);
        acc[0] = acc[1] = acc[2] = acc[3] = 0;
#pragma unroll 2
        for (int i = tid; i < nvec; i += kFusedComputeThreads) FE::exps(v[i], l2e2, nmL2, acc);
      }
      double part;
      {
        float a0, a1, a2, a3;
        f2unpack(fadd2(acc[0], acc[1]), a0, a1);
        f2unpack(fadd2(acc[2], acc[3]), a2, a3);
        part = (static_cast<double>(a0) + static_cast<double>(a1)) +
               (static_cast<double>(a2) + static_cast<double>(a3));
      }
      // gather the target logit while the piece is in SMEM, then free the stage
      const bool tok_ok = tg >= 0 && tg < V;
      const int li = tg - elem0;
      const bool here = tok_ok && li >= 0 && li < nvec * E;
      const float xt_v = (tid == 0 && here) ? FE::get(buf(s), li) : __int_as_float(0x7fc00000);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[s]);
      part = warp_sum_f64(part);
      const int sa = static_cast<int>(a % kASlots);
      if (a >= kASlots) {  // the tail warp has read A piece a-8's partials
        DBG_T0();
        mbar_wait(&S.afree[sa], static_cast<uint32_t>(((a - kASlots) / kASlots) & 1));
        if (tid == 0) { DBG_ADD(3); }
      }
      ++a;
      if (tid == 0) {
        S.tgta[sa] = tok_ok ? tg : -1;
        S.xt[sa] = xt_v;
      }
      if (lane == 0) {
        S.wm[sa][warp] = m;
        S.ws[sa][warp] = part;
        mbar_arrive(&S.adoneA[sa]);
      }
      continue;
    }
    const int sb = static_cast<int>(b % kFusedStages);
    {
      DBG_T0();
#if DVLA_CFULL_WAIT
      mbar_wait(&S.cfullB[sb], static_cast<uint32_t>((b / kFusedStages) & 1));
#else
      mbar_wait_backoff(&S.cfullB[sb], static_cast<uint32_t>((b / kFusedStages) & 1));
#endif
      if (tid == 0) { DBG_ADD(1); }
    }
    ++b;
    const uint32_t mode = S.mode[sb];
    uint4* v = reinterpret_cast<uint4*>(buf(s));  // dlogits overwrite the piece in place
    if ((mode & 3u) != 1u) {
      // zero-gradient rows (A == 0 or clipped chunk): 0 * (onehot - p)
      const uint32_t z = (mode == 0u) ? 0u : FE::kNaN;
      for (int i = tid; i < nvec; i += kFusedComputeThreads) v[i] = make_uint4(z, z, z, z);
    } else {
      // target column: c * (1 - p_t) (prep warp, f64), patched by the
      // thread that owns it
      const int li = S.tgt[sb] - elem0;
      const bool here = li >= 0 && li < nvec * E;
      const bool owner = here && tid == ((li / E) % kFusedComputeThreads);
      const float val = S.tval[sb];
      // -c * p_v = -sign(c) * 2^(x*log2e - (lse*log2e - log2|c|))
      const float K = S.kval[sb];
      const uint64_t nK2 = f2pack(-K, -K);
      const uint32_t sgn = (mode & 0x80000000u) ? FE::kSign : 0u;
#pragma unroll kBUnroll
      for (int i = tid; i < nvec; i += kFusedComputeThreads) v[i] = FE::grad(v[i], l2e2, nK2, sgn);
      if (owner) FE::put(v, li, val);
    }
    fence_proxy_async_smem();  // generic SMEM writes -> visible to the bulk store
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&S.bdone[sb]);  // the store warp frees the stage after its copy
      mbar_arrive(&S.adoneB[sb]);
    }
  }
  if (dbg && tid == 0) atomicAdd(dbg + 12, static_cast<unsigned long long>(clock64() - t_kernel));
  if (dbg && tid == 0 && g_dbg_cta) {
    g_dbg_cta[2 * blockIdx.x] = t_kernel_ns;
    g_dbg_cta[2 * blockIdx.x + 1] = globaltimer_ns();
  }
}

// ------------------------------------------------------ unfused kernels
template <class T>
struct Elem;
template <>
struct Elem<float> {
  static constexpr int kVec = 4;
  __device__ static float get(const float* p, int64_t i) { return p[i]; }
};
template <>
struct Elem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  __device__ static float get(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
};

__device__ __forceinline__ void unpack_vec(const uint4& u, float* f, float) {
  f[0] = __uint_as_float(u.x);
  f[1] = __uint_as_float(u.y);
  f[2] = __uint_as_float(u.z);
  f[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ void unpack_vec(const uint4& u, float* f, __nv_bfloat16) {
  f[0] = bf16lo(u.x); f[1] = bf16hi(u.x);
  f[2] = bf16lo(u.y); f[3] = bf16hi(u.y);
  f[4] = bf16lo(u.z); f[5] = bf16hi(u.z);
  f[6] = bf16lo(u.w); f[7] = bf16hi(u.w);
}
__device__ __forceinline__ uint4 pack_vec(const float* f, float) {
  return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                    __float_as_uint(f[3]));
}
__device__ __forceinline__ uint4 pack_vec(const float* f, __nv_bfloat16) {
  return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                    pack_bf16x2(f[6], f[7]));
}
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ void from_f(float v, float* d) { *d = v; }
__device__ __forceinline__ void from_f(float v, __nv_bfloat16* d) { *d = __float2bfloat16_rn(v); }

constexpr int kRowThreads = 256;

// online (max, sum-exp) with per-vector rescale; one CTA per row
template <class T>
__global__ void __launch_bounds__(kRowThreads) tok_rows_kernel(TokParams p, int vec_ok) {
  const int64_t r = blockIdx.x;
  const int64_t V = p.V;
  const T* row = static_cast<const T*>(p.logits) + r * V;
  const int tid = threadIdx.x;
  float m = -INFINITY, s = 0.f;
  auto add = [&](const float* f, int n) {
    float vm = f[0];
    for (int e = 1; e < n; ++e) vm = fmaxf(vm, f[e]);
    if (vm > m) {
      s = (m == -INFINITY) ? 0.f : s * ex2f((m - vm) * kLog2e);
      m = vm;
    }
    if (m == -INFINITY) return;
    const float mL = m * kLog2e;
    for (int e = 0; e < n; ++e) s += ex2f(fmaf(f[e], kLog2e, -mL));
  };
  constexpr int E = Elem<T>::kVec;
  if (vec_ok) {
    const uint4* v = reinterpret_cast<const uint4*>(row);
    const int64_t nvec = V / E;
    for (int64_t i = tid; i < nvec; i += kRowThreads) {
      float f[E];
      unpack_vec(__ldcs(v + i), f, T());
      add(f, E);
    }
    for (int64_t i = nvec * E + tid; i < V; i += kRowThreads) {
      float f = to_f(row[i]);
      add(&f, 1);
    }
  } else {
    for (int64_t i = tid; i < V; i += kRowThreads) {
      float f = to_f(row[i]);
      add(&f, 1);
    }
  }
  __shared__ float sm[kRowThreads / 32];
  __shared__ double ss[kRowThreads / 32];
  const int warp = tid >> 5, lane = tid & 31;
  float M = warp_max_f32(m);
  if (lane == 0) sm[warp] = M;
  __syncthreads();
  M = sm[0];
  for (int w = 1; w < kRowThreads / 32; ++w) M = fmaxf(M, sm[w]);
  double part = (m == -INFINITY) ? 0.0 : static_cast<double>(s) * exp2(static_cast<double>((m - M) * kLog2e));
  part = warp_sum_f64(part);
  if (lane == 0) ss[warp] = part;
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int w = 0; w < kRowThreads / 32; ++w) sum += ss[w];
    const double lse = static_cast<double>(M) + log(sum);
    const int32_t tgt = p.tokens[r];
    double xt;
    if (tgt < 0 || tgt >= V) {
      atomicOr(p.err, kErrToken);
      xt = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      xt = static_cast<double>(to_f(row[tgt]));
    }
    p.lse[r] = lse;
    p.lp_tok[r] = xt - lse;
  }
}

__global__ void tok_chunk_kernel(TokParams p) {
  const int64_t warps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < p.n_chunks;
       q += warps) {
    if (lane == 0) {
      const double lp = chunk_lp_pairwise(p.lp_tok + q * p.T, p.T);
      ChunkTerms ct = chunk_terms(lp, static_cast<double>(p.blp[q]), p.adv[q / p.C], p.w,
                                  p.clip_eps, p.kl_coeff);
      p.lp_chunk[q] = lp;
      p.coeff[q] = ct.coeff;
    }
  }
}

template <class T>
__global__ void __launch_bounds__(kRowThreads) tok_bwd_kernel(TokParams p, int vec_ok) {
  const int64_t r = blockIdx.x;
  const int64_t V = p.V;
  const T* row = static_cast<const T*>(p.logits) + r * V;
  T* out = static_cast<T*>(p.dlogits) + r * V;
  const double c = p.coeff[r / p.T];
  const double lse = p.lse[r];
  const int32_t tgt = p.tokens[r];
  const int tid = threadIdx.x;
  constexpr int E = Elem<T>::kVec;
  const float cf = static_cast<float>(c);
  const float lseL = static_cast<float>(lse * 1.4426950408889634);
  // target column c (1 - p_t) = -c expm1(lp_tok) in f64 (no cancellation)
  const float tv = static_cast<float>(-c * expm1(p.lp_tok[r]));
  auto val = [&](float x, int64_t col) {
    const float pv = ex2f(fmaf(x, kLog2e, -lseL));
    return (col == tgt) ? tv : -cf * pv;
  };
  if (vec_ok) {
    const uint4* v = reinterpret_cast<const uint4*>(row);
    uint4* o = reinterpret_cast<uint4*>(out);
    const int64_t nvec = V / E;
    for (int64_t i = tid; i < nvec; i += kRowThreads) {
      float f[E];
      unpack_vec(__ldcs(v + i), f, T());
#pragma unroll
      for (int e = 0; e < E; ++e) f[e] = val(f[e], i * E + e);
      __stcs(o + i, pack_vec(f, T()));
    }
    for (int64_t i = nvec * E + tid; i < V; i += kRowThreads) from_f(val(to_f(row[i]), i), out + i);
  } else {
    for (int64_t i = tid; i < V; i += kRowThreads) from_f(val(to_f(row[i]), i), out + i);
  }
}

// ------------------------------------------------------------- epilogue
struct EpiParams {
  const double* lp_chunk;   // [n_traj*C] input order
  const float* blp;         // [n_traj*C]
  const double* blp64;      // optional f64 behaviour log-probs (overrides blp)
  const double* adv;        // [n_traj]
  const uint32_t* reward_bad;  // [n_groups] or null
  const int64_t* order;     // [n_groups] canonical order (null = identity)
  const int64_t* group_ids; // [n_groups] (null = position)
  double* coeff_out;        // [n_traj*C] or null
  double* stats;            // [DVLA_ST_LEN]
  const uint32_t* kerr;     // kernel error word or null
  int64_t n_groups, G, C;
  double w, clip_eps, kl_coeff;
};

constexpr int kEpiThreads = 512;

__global__ void __launch_bounds__(kEpiThreads) grpo_epilogue_kernel(EpiParams e) {
  pdl_wait();  // everything below reads the fused kernel's results
  __shared__ double s_loss[kEpiThreads], s_rho[kEpiThreads];
  __shared__ unsigned char s_clip[kEpiThreads];
  __shared__ unsigned long long s_first_reward, s_first_traj;
  const int tid = threadIdx.x;
  const int64_t GC = e.G * e.C;
  const int64_t n_entries = e.n_groups * GC;
  auto gin = [&](int64_t k) { return e.order ? e.order[k] : k; };
  auto gid = [&](int64_t g) { return e.group_ids ? e.group_ids[g] : g; };
  if (tid == 0) {
    s_first_reward = ~0ull;
    s_first_traj = ~0ull;
  }
  __syncthreads();
  if (e.reward_bad) {
    for (int64_t k = tid; k < e.n_groups; k += kEpiThreads)
      if (e.reward_bad[gin(k)]) atomicMin(&s_first_reward, (unsigned long long)k);
  }
  double loss = 0.0, ratio_sum = 0.0, clip_count = 0.0;
  for (int64_t base = 0; base < n_entries; base += kEpiThreads) {
    const int64_t idx = base + tid;
    if (idx < n_entries) {
      const int64_t k = idx / GC, rem = idx % GC;
      const int64_t i = rem / e.C, c = rem % e.C;
      const int64_t j = gin(k) * e.G + i;  // input-order trajectory
      const int64_t q = j * e.C + c;
      const double lp = e.lp_chunk[q];
      const double blp = e.blp64 ? e.blp64[q] : static_cast<double>(e.blp[q]);
      ChunkTerms ct = chunk_terms(lp, blp, e.adv[j], e.w, e.clip_eps, e.kl_coeff);
      if (e.coeff_out) e.coeff_out[q] = ct.coeff;
      s_loss[tid] = ct.loss;
      s_rho[tid] = ct.rho;
      s_clip[tid] = ct.clipped;
      if (!isfinite(lp) || !isfinite(ct.rho))
        atomicMin(&s_first_traj, (unsigned long long)(idx / e.C));
    }
    __syncthreads();
    {
      // three independent sequential sums in canonical entry order, one per
      // warp (the reference accumulates total_loss / ratio_sum / clip_count
      // in entry order, grpo.py:269-273)
      const int64_t lim = (n_entries - base < kEpiThreads) ? n_entries - base : kEpiThreads;
      // (loads batched 8 ahead so only the dependent adds serialise)
      auto seq_sum = [&](double acc, const double* v) {
        int64_t t = 0;
        for (; t + 8 <= lim; t += 8) {
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = v[t + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, x[u]);
        }
        for (; t < lim; ++t) acc = __dadd_rn(acc, v[t]);
        return acc;
      };
      if (tid == 0) {
        loss = seq_sum(loss, s_loss);
      } else if (tid == 32) {
        ratio_sum = seq_sum(ratio_sum, s_rho);
      } else if (tid == 64) {
        for (int64_t t = 0; t < lim; ++t) clip_count += s_clip[t];
      }
    }
    __syncthreads();
  }
  __shared__ double s_fin[2];
  if (tid == 32) s_fin[0] = ratio_sum;
  if (tid == 64) s_fin[1] = clip_count;
  __syncthreads();
  if (tid == 0) {
    ratio_sum = s_fin[0];
    clip_count = s_fin[1];
    double code = 0.0, group = 0.0;
    if (s_first_reward != ~0ull) {
      code = 1.0;
      group = static_cast<double>(gid(gin(static_cast<int64_t>(s_first_reward))));
    } else if (s_first_traj != ~0ull) {
      const int64_t ct = static_cast<int64_t>(s_first_traj);  // canonical traj index
      const int64_t k = ct / e.G, i = ct % e.G;
      const int64_t j = gin(k) * e.G + i;
      bool lp_bad = false;
      for (int64_t c = 0; c < e.C; ++c) lp_bad |= !isfinite(e.lp_chunk[j * e.C + c]);
      code = lp_bad ? 2.0 : 3.0;
      group = static_cast<double>(gid(gin(k)));
    } else if (!isfinite(loss)) {
      code = 4.0;
      group = static_cast<double>(gid(gin(0)));
    }
    e.stats[DVLA_ST_LOSS] = loss;
    e.stats[DVLA_ST_RATIO_SUM] = ratio_sum;
    e.stats[DVLA_ST_CLIP_COUNT] = clip_count;
    e.stats[DVLA_ST_CHUNK_COUNT] = static_cast<double>(n_entries);
    e.stats[DVLA_ST_ABORT] = code;
    e.stats[DVLA_ST_ABORT_GROUP] = group;
    e.stats[DVLA_ST_KERNEL_ERR] = e.kerr ? static_cast<double>(*e.kerr) : 0.0;
    e.stats[DVLA_ST_RESERVED] = 0.0;
  }
}

// ------------------------------------------------------------ workspace
struct TokWorkspace {
  double* adv;
  double* lp_tok;
  double* lse;
  double* coeff;
  uint32_t* reward_bad;
  uint32_t* err;
  size_t bytes;
};

static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

static TokWorkspace carve(void* base, int64_t n_groups, int64_t G, int64_t C, int64_t T) {
  const int64_t n_traj = n_groups * G, nq = n_traj * C, R = nq * T;
  TokWorkspace w{};
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off += al256(b);
    return static_cast<uint8_t*>(base) + o;
  };
  w.adv = reinterpret_cast<double*>(take(n_traj * 8));
  w.lp_tok = reinterpret_cast<double*>(take(R * 8));
  w.lse = reinterpret_cast<double*>(take(R * 8));
  w.coeff = reinterpret_cast<double*>(take(nq * 8));
  w.reward_bad = reinterpret_cast<uint32_t*>(take(n_groups * 4));
  w.err = reinterpret_cast<uint32_t*>(take(16));
  w.bytes = off;
  return w;
}

// Stage geometry of the fused kernel: the fewest pieces per row (1, 2 or 4)
// whose stage fits three times in SMEM next to the header.
struct FusedGeom {
  int pieces = 0;      // 0: does not fit
  int piece_vec = 0;   // 16-byte granules per piece
  uint32_t stage_bytes = 0;
  size_t smem = 0;
};

static FusedGeom fused_geom(int64_t V, size_t esz) {
  FusedGeom g;
  const int64_t nvec_row = V * static_cast<int64_t>(esz) / 16;
  const size_t hdr = ((sizeof(FusedSmem) + 127) / 128) * 128;
  for (int P : {1, 2, 4}) {
    const int64_t pv = (nvec_row + P - 1) / P;
    const size_t stage = ((static_cast<size_t>(pv) * 16 + 127) / 128) * 128;
    if (hdr + kFusedStages * stage <= kFusedSmemCap) {
      g.pieces = P;
      g.piece_vec = static_cast<int>(pv);
      g.stage_bytes = static_cast<uint32_t>(stage);
      g.smem = hdr + kFusedStages * stage;
      return g;
    }
  }
  return g;
}

using FusedKernelFn = void (*)(TokParams, uint32_t, int, int, int);

// Launch with the programmatic-stream-serialization attribute (PDL) when
// DVLA_PDL: the kernel may begin while the previous kernel in the stream is
// still running (see pdl_wait / pdl_trigger).
template <class... KArgs, class... Args>
static cudaError_t launch_maybe_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = DVLA_PDL ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <class TE>
static FusedKernelFn fused_kernel_for(int pieces) {
  switch (pieces) {
    case 1: return tok_fused_kernel<TE, 1>;
    case 2: return tok_fused_kernel<TE, 2>;
    default: return tok_fused_kernel<TE, 4>;
  }
}

}  // namespace dvla

using namespace dvla;

extern "C" size_t dvla_token_loss_workspace_bytes(int64_t n_groups, int64_t G, int64_t C,
                                                  int64_t T) {
  if (n_groups < 0 || G < 0 || C < 0 || T < 0) return 0;
  return carve(nullptr, n_groups, G, C, T).bytes;
}

extern "C" int dvla_token_loss_workspace_layout(int64_t n_groups, int64_t G, int64_t C,
                                                int64_t T, size_t* offsets) {
  if (n_groups < 0 || G < 0 || C < 0 || T < 0 || !offsets)
    return fail(DVLA_ERR_USAGE, "bad workspace layout query");
  const TokWorkspace w = carve(nullptr, n_groups, G, C, T);
  const auto off = [](const void* q) { return reinterpret_cast<size_t>(q); };
  offsets[0] = off(w.adv);
  offsets[1] = off(w.lp_tok);
  offsets[2] = off(w.lse);
  offsets[3] = off(w.coeff);
  return DVLA_OK;
}

extern "C" int dvla_token_loss_fwd_bwd(const void* logits, int dtype, const int32_t* tokens,
                                       const float* blp, const float* rewards,
                                       const int64_t* group_order, const int64_t* group_ids,
                                       int64_t n_groups, int64_t G, int64_t C, int64_t T,
                                       int64_t V, double clip_eps, double adv_eps,
                                       double kl_coeff, int flags, void* dlogits,
                                       double* lp_chunk, double* stats, void* workspace,
                                       size_t workspace_bytes, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (n_groups < 1) return fail(DVLA_ERR_CONFIG, "grpo update needs at least one group");
  if (G < 2) return fail(DVLA_ERR_CONFIG, "group_size must be >= 2, got %lld", (long long)G);
  if (C < 1 || T < 1 || V < 1)
    return fail(DVLA_ERR_USAGE, "C, T, V must be >= 1 (got %lld, %lld, %lld)", (long long)C,
                (long long)T, (long long)V);
  if (dtype != DVLA_F32 && dtype != DVLA_BF16)
    return fail(DVLA_ERR_USAGE, "dtype must be DVLA_F32 or DVLA_BF16");
  if (!logits || !tokens || !blp || !rewards || !lp_chunk || !stats || !workspace)
    return fail(DVLA_ERR_USAGE, "null pointer argument");
  const bool want_dl = (flags & DVLA_TL_WRITE_DLOGITS) != 0;
  if (want_dl && !dlogits) return fail(DVLA_ERR_USAGE, "dlogits requested but null");
  TokWorkspace ws = carve(workspace, n_groups, G, C, T);
  if (workspace_bytes < ws.bytes)
    return fail(DVLA_ERR_USAGE, "workspace too small: %zu < %zu", workspace_bytes, ws.bytes);

  const int64_t n_traj = n_groups * G, nq = n_traj * C, R = nq * T;
  TokParams p{};
  p.logits = logits;
  p.tokens = tokens;
  p.blp = blp;
  p.adv = ws.adv;
  p.dlogits = dlogits;
  p.lp_tok = ws.lp_tok;
  p.lse = ws.lse;
  p.lp_chunk = lp_chunk;
  p.coeff = ws.coeff;
  p.err = ws.err;
  p.R = R;
  p.V = V;
  p.T = T;
  p.C = C;
  p.n_chunks = nq;
  p.w = 1.0 / static_cast<double>(n_traj * C);
  p.clip_eps = clip_eps;
  p.kl_coeff = kl_coeff;

  {
    const int thr = 128;
    const int64_t fill_blocks = std::min<int64_t>((R + thr - 1) / thr, 4 * 148);
    const int64_t blocks = std::max<int64_t>((n_groups + thr - 1) / thr, fill_blocks);
    tok_adv_kernel<<<(unsigned)blocks, thr, 0, stream>>>(rewards, n_groups, G, adv_eps, ws.adv,
                                                          ws.reward_bad, ws.lp_tok, R, ws.err);
    if (int rc = launch_check("tok_adv_kernel")) return rc;
  }

  const int dev = current_device();
  const int sms = num_sms(dev);
  const size_t esz = dtype == DVLA_BF16 ? 2 : 4;
  const bool aligned16 = (reinterpret_cast<uintptr_t>(logits) % 16 == 0) &&
                         (!want_dl || reinterpret_cast<uintptr_t>(dlogits) % 16 == 0) &&
                         ((V * esz) % 16 == 0);
  const FusedGeom geom = fused_geom(V, esz);
  const bool fused = !(flags & DVLA_TL_UNFUSED) && aligned16 && geom.pieces > 0 && T <= sms &&
                     T <= 128 && R >= 1 && R < (int64_t{1} << 31);
  if (fused) {
    const FusedKernelFn kern = dtype == DVLA_BF16 ? fused_kernel_for<__nv_bfloat16>(geom.pieces)
                                                  : fused_kernel_for<float>(geom.pieces);
    static bool attr_set[64][2][3] = {};
    bool& set = attr_set[dev & 63][dtype == DVLA_BF16 ? 0 : 1][geom.pieces >> 1];
    if (!set) {
      DVLA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kFusedSmemCap)));
      set = true;
    }
    const int64_t slots = int64_t{sms} * kFusedCtasPerSm;
    const unsigned grid = static_cast<unsigned>(R < slots ? R : slots);
    cudaEvent_t stop;
    prof_begin(stream, &stop);
    static const int lag_env = [] {
      const char* e = getenv("DVLA_FUSED_LAG");
      return e ? atoi(e) : 0;
    }();
    // lag in pieces: >= 2P - 1 so a chunk's two rounds of tails precede its
    // B ops (deadlock freedom), <= kRing P - 1 for the (lse, target) ring.
    // Measured defaults (sustained, power-capped): 3 pieces for one-piece
    // rows (bf16 C2), 4 pieces = 2 rows for two-piece rows (f32 C2: 1.370 vs
    // 1.423 ms at 3, 1.430 at 5; tools/f32_time.py).
    const int P = geom.pieces;
    const int lag = lag_env > 0 ? lag_env : (P == 1 ? kLagRounds : (P == 2 ? 4 : 2 * P - 1));
    const int lag_p = std::min(std::max(lag, 2 * P - 1), kRing * P - 1);
    DVLA_CUDA_TRY(launch_maybe_pdl(kern, dim3(grid), dim3(kFusedThreadsWS), geom.smem, stream,
                                   p, geom.stage_bytes, geom.piece_vec, want_dl ? 1 : 0,
                                   std::max(lag_p, 2)));
    prof_end(stream, stop);
    if (int rc = launch_check("tok_fused_kernel")) return rc;
    if (!want_dl) {
      tok_chunk_kernel<<<(unsigned)((nq * 32 + 255) / 256), 256, 0, stream>>>(p);
      if (int rc = launch_check("tok_chunk_kernel")) return rc;
    }
  } else {
    const int vec_ok = aligned16 ? 1 : 0;
    cudaEvent_t stop;
    prof_begin(stream, &stop);
    if (dtype == DVLA_BF16)
      tok_rows_kernel<__nv_bfloat16><<<(unsigned)R, kRowThreads, 0, stream>>>(p, vec_ok);
    else
      tok_rows_kernel<float><<<(unsigned)R, kRowThreads, 0, stream>>>(p, vec_ok);
    if (int rc = launch_check("tok_rows_kernel")) return rc;
    tok_chunk_kernel<<<(unsigned)((nq * 32 + 255) / 256), 256, 0, stream>>>(p);
    if (int rc = launch_check("tok_chunk_kernel")) return rc;
    if (want_dl) {
      if (dtype == DVLA_BF16)
        tok_bwd_kernel<__nv_bfloat16><<<(unsigned)R, kRowThreads, 0, stream>>>(p, vec_ok);
      else
        tok_bwd_kernel<float><<<(unsigned)R, kRowThreads, 0, stream>>>(p, vec_ok);
      if (int rc = launch_check("tok_bwd_kernel")) return rc;
    }
    prof_end(stream, stop);
  }

  EpiParams e{};
  e.lp_chunk = lp_chunk;
  e.blp = blp;
  e.adv = ws.adv;
  e.reward_bad = ws.reward_bad;
  e.order = group_order;
  e.group_ids = group_ids;
  e.stats = stats;
  e.kerr = ws.err;
  e.n_groups = n_groups;
  e.G = G;
  e.C = C;
  e.w = p.w;
  e.clip_eps = clip_eps;
  e.kl_coeff = kl_coeff;
  if (fused) {
    DVLA_CUDA_TRY(launch_maybe_pdl(grpo_epilogue_kernel, dim3(1), dim3(kEpiThreads), 0, stream, e));
  } else {
    grpo_epilogue_kernel<<<1, kEpiThreads, 0, stream>>>(e);
  }
  return launch_check("grpo_epilogue_kernel");
}

// Debug only (not part of the header): point the fused kernel's per-role
// cycle counters at a device buffer of 16 u64 (or null to disable).
extern "C" int dvla_debug_fused_counters(void* dev_buf) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_buf);
  DVLA_CUDA_TRY(cudaMemcpyToSymbol(g_dbg, &p, sizeof(p)));
  return DVLA_OK;
}

// Debug only: per-CTA (start, end) globaltimer stamps of the fused kernel
// (2 u64 per CTA; recorded while the counters above are enabled).
extern "C" int dvla_debug_fused_cta_times(void* dev_buf) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_buf);
  DVLA_CUDA_TRY(cudaMemcpyToSymbol(g_dbg_cta, &p, sizeof(p)));
  return DVLA_OK;
}

extern "C" int dvla_advantages(const double* rewards, int64_t n_groups, int64_t G, double delta,
                               double* out, void* stream) {
  if (G < 2) return fail(DVLA_ERR_CONFIG, "a reward group needs >= 2 entries, got shape (%lld,)",
                         (long long)G);
  if (n_groups < 1) return DVLA_OK;
  if (!rewards || !out) return fail(DVLA_ERR_USAGE, "null pointer argument");
  const int thr = 128;
  adv_f64_kernel<<<(unsigned)((n_groups + thr - 1) / thr), thr, 0,
                   static_cast<cudaStream_t>(stream)>>>(rewards, n_groups, G, delta, out);
  return launch_check("adv_f64_kernel");
}

extern "C" int dvla_group_advantages(const float* rewards, int64_t n_groups, int64_t G,
                                     double delta, double* adv, uint32_t* reward_bad,
                                     void* stream) {
  if (G < 2) return fail(DVLA_ERR_CONFIG, "a reward group needs >= 2 entries, got shape (%lld,)",
                         (long long)G);
  if (n_groups < 1) return DVLA_OK;
  if (!rewards || !adv || !reward_bad) return fail(DVLA_ERR_USAGE, "null pointer argument");
  const int thr = 128;
  tok_adv_kernel<<<(unsigned)((n_groups + thr - 1) / thr), thr, 0,
                   static_cast<cudaStream_t>(stream)>>>(rewards, n_groups, G, delta, adv,
                                                        reward_bad, nullptr, 0, nullptr);
  return launch_check("tok_adv_kernel");
}

extern "C" int dvla_grpo_epilogue(const double* lp_chunk, const float* blp, const double* blp64,
                                  const double* adv, const uint32_t* reward_bad,
                                  const int64_t* group_order,
                                  const int64_t* group_ids, int64_t n_groups, int64_t G,
                                  int64_t C, double clip_eps, double kl_coeff, double* coeff_out,
                                  double* stats, void* stream) {
  if (n_groups < 1) return fail(DVLA_ERR_CONFIG, "grpo update needs at least one group");
  if (!lp_chunk || (!blp && !blp64) || !adv || !stats)
    return fail(DVLA_ERR_USAGE, "null pointer argument");
  EpiParams e{};
  e.lp_chunk = lp_chunk;
  e.blp = blp;
  e.blp64 = blp64;
  e.adv = adv;
  e.reward_bad = reward_bad;
  e.order = group_order;
  e.group_ids = group_ids;
  e.coeff_out = coeff_out;
  e.stats = stats;
  e.n_groups = n_groups;
  e.G = G;
  e.C = C;
  e.w = 1.0 / static_cast<double>(n_groups * G * C);
  e.clip_eps = clip_eps;
  e.kl_coeff = kl_coeff;
  grpo_epilogue_kernel<<<1, kEpiThreads, 0, static_cast<cudaStream_t>(stream)>>>(e);
  return launch_check("grpo_epilogue_kernel");
}
