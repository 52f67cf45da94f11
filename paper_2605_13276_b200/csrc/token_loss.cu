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
//   tok_fused_bf16_kernel persistent, 1 CTA/SM, warp-specialised: a producer
//                         warp streams logits rows HBM->SMEM with TMA bulk
//                         copies (cp.async.bulk), 16 compute warps do
//                         max / sum-exp (MUFU ex2) / gather on the SMEM row,
//                         publish lp_tok, and the last CTA to finish a chunk
//                         computes that chunk's coefficient; dlogits are then
//                         written in place in SMEM and TMA-stored back.
//                         Logits are read from HBM exactly once:
//                         compulsory traffic 2*N*2 bytes.
//   tok_rows_kernel<T>    unfused forward (any dtype / alignment / V)
//   tok_chunk_kernel      unfused per-chunk coefficient
//   tok_bwd_kernel<T>     unfused backward (re-reads logits: 3*N*s traffic)
//   grpo_epilogue_kernel  loss / stats / abort detection in canonical order
#include <stdlib.h>

#include "common.cuh"
#include "grpo_math.cuh"

namespace dvla {

constexpr int kFusedComputeWarps = 16;
constexpr int kFusedComputeThreads = kFusedComputeWarps * 32;
constexpr int kFusedStages = 3;    // SMEM row stages and B coefficient slots
constexpr int kASlots = 8;         // A-row partial slots (coef-warp slack)
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
  uint32_t* cnt;
  uint32_t* err;
  int64_t R, V, T, C, n_chunks;
  double w, clip_eps, kl_coeff;
};

enum : uint32_t { kErrToken = 1u, kErrTimeout = 2u };

// Optional per-role cycle counters for the fused kernel (set by
// dvla_debug_fused_counters; null in normal runs -> no clock reads).
__device__ unsigned long long* g_dbg = nullptr;
#define DBG_T0() const long long _t0 = dbg ? clock64() : 0
#define DBG_ADD(i) \
  if (dbg) atomicAdd(dbg + (i), static_cast<unsigned long long>(clock64() - _t0))

// ------------------------------------------------------------ advantages
__global__ void tok_adv_kernel(const float* __restrict__ rewards, int64_t n_groups, int64_t G,
                               double delta, double* __restrict__ adv,
                               uint32_t* __restrict__ reward_bad) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
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

// ---------------------------------------------------- fused bf16 kernel
//
// One CTA per SM (persistent), rows assigned round-robin (row = cta + k*grid).
// Every CTA walks one op sequence: A(0..L-1), then A(k), B(k-L), ..., B(n-1):
//   A(k)  row k streamed HBM -> SMEM by TMA; 16 compute warps take warp
//         max / sum-exp (MUFU ex2) and publish (m_w, s_w); the coefficient
//         warp combines them into lse (f64), gathers the target logit,
//         publishes lp_tok and bumps the chunk counter (red.release.gpu).
//   B(k)  row k streamed again -- from L2, L rounds (~L*148*64 KB) after
//         A(k) -- the coefficient warp waits for the chunk to be complete on
//         all CTAs (long done by then), sums its T token log-probs (numpy
//         pairwise order) and evaluates the GRPO coefficient; the compute
//         warps write d loss / d logits in place and the store warp streams
//         the row back with a TMA bulk store.
// HBM traffic stays at the compulsory 2*N*2 bytes while the L-round lag
// hides the cross-CTA chunk dependency.  A(k+L) precedes B(k) on every CTA,
// so the chunk wait is deadlock-free while all CTAs are co-resident
// (grid <= #SMs, T <= grid).
//
// Warp roles: 0..15 compute (they also store dlogits, 16-byte streaming
// stores from registers), 16 loader, 17 coefficient, 18 idle,
// 19 publisher (lp_tok + release of the chunk counters).
// Barriers (every barrier completes once per use of its own ring index, and
// every waiter walks its ring in order, so parity never aliases):
//   full[s], empty[s]  per SMEM stage s = op % 3: loader <-> compute warps
//                      (a stage is free as soon as its row has been read)
//   adoneA[a % 8]      compute -> coef, per A op a (SMEM partial slot a % 8)
//   afree[a % 8]       coef -> compute, partial slot consumed
//   cfullB[b % 3]      coef -> compute, per B op b (coefficient slot b % 3)
//   adoneB[b % 3]      compute -> coef (coefficient slot b % 3 consumed)
// The op sequence and barrier protocol were model-checked for races and
// parity aliasing (tests/test_fused_protocol.py).
constexpr int kWarpLoader = kFusedComputeWarps;
constexpr int kCoefWarp = kFusedComputeWarps + 1;
constexpr int kWarpStore = kFusedComputeWarps + 2;
constexpr int kWarpPublish = kFusedComputeWarps + 3;
constexpr int kFusedThreadsWS = (kFusedComputeWarps + 4) * 32;
constexpr int kPubRing = 8;
constexpr int kLagRounds = 4;  // measured best on B200 (lag 2..4 sweep, tools/fused_variants.py)
constexpr int kRing = 8;  // > kLagRounds + 1 rows of (lse, target) in flight

struct FusedSmem {
  uint64_t full[kFusedStages];
  uint64_t empty[kFusedStages];
  uint64_t adoneA[kASlots];
  uint64_t afree[kASlots];
  uint64_t adoneB[kFusedStages];
  uint64_t cfullB[kFusedStages];
  double ws[kASlots][kFusedComputeWarps];
  float wm[kASlots][kFusedComputeWarps];
  float kval[kFusedStages];   // lse*log2e - log2|c|
  float lseL[kFusedStages];   // lse*log2e
  float cf[kFusedStages];     // coefficient (f32)
  uint32_t mode[kFusedStages];  // 0 zero row, 1 finite c (bit 31: c > 0), 2 non-finite c
  int32_t tgt[kFusedStages];
  float xt[kASlots];       // gathered target logit of A slot
  int32_t tgta[kASlots];   // its token id (-1: out of range)
  double ring_lse[kRing];
  int32_t ring_tgt[kRing];
  uint64_t pubfull[kPubRing];
  uint64_t pubempty[kPubRing];
  double pub_lp[kPubRing];
};

// coefficient not yet published (the workspace is memset to 0xff)
constexpr unsigned long long kCoeffPending = 0xffffffffffffffffull;

__device__ __forceinline__ unsigned long long spin_coeff(const unsigned long long* c,
                                                         uint32_t* err) {
  unsigned long long v = ld_acquire_gpu_u64(c);
  if (v != kCoeffPending) return v;
  const uint64_t t0 = globaltimer_ns();
  uint32_t ns = 32;
  while ((v = ld_acquire_gpu_u64(c)) == kCoeffPending) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    if (globaltimer_ns() - t0 > kSpinTimeoutNs) {
      atomicOr(err, kErrTimeout);
      return 0x7ff8000000000000ull;
    }
  }
  return v;
}

__device__ __forceinline__ bool spin_until_at_least(const uint32_t* cnt, uint32_t target,
                                                    uint32_t* err) {
  if (ld_acquire_gpu(cnt) >= target) return true;
  const uint64_t t0 = globaltimer_ns();
  uint32_t ns = 32;
  while (ld_acquire_gpu(cnt) < target) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    if (globaltimer_ns() - t0 > kSpinTimeoutNs) {
      atomicOr(err, kErrTimeout);
      return false;
    }
  }
  return true;
}

// op n of a CTA with nloc rows and lag L: (is_B, local row)
__device__ __forceinline__ void op_of(int64_t n, int64_t nloc, int L, bool* isB, int64_t* k) {
  const int64_t Le = nloc < L ? nloc : L;  // effective lag
  if (n < Le) {
    *isB = false;
    *k = n;
    return;
  }
  const int64_t m = n - Le;  // pairs (A(Le + j), B(j)) for j < nloc - Le, then B tail
  const int64_t pairs = nloc - Le;
  if (m < 2 * pairs) {
    *isB = (m & 1) != 0;
    *k = (m & 1) ? (m >> 1) : (Le + (m >> 1));
    return;
  }
  *isB = true;
  *k = pairs + (m - 2 * pairs);
}

__global__ void __launch_bounds__(kFusedThreadsWS, 1)
    tok_fused_bf16_kernel(TokParams p, uint32_t stage_bytes, int write_dl, int lag, int a_evict_last) {
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  FusedSmem& S = *reinterpret_cast<FusedSmem*>(dyn_smem);
  uint8_t* bufs = dyn_smem + ((sizeof(FusedSmem) + 127) / 128) * 128;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t V = p.V;
  const uint32_t row_bytes = static_cast<uint32_t>(V * 2);
  const int64_t G = gridDim.x;
  const int64_t nloc = (p.R > blockIdx.x) ? (p.R - blockIdx.x + G - 1) / G : 0;
  const int64_t nops = write_dl ? 2 * nloc : nloc;
  const int L = write_dl ? lag : 1 << 30;  // forward-only: A ops only
  auto row_of = [&](int64_t k) { return blockIdx.x + k * G; };
  auto buf = [&](int s) { return bufs + static_cast<size_t>(s) * stage_bytes; };
  const int64_t T = p.T;
  unsigned long long* dbg = g_dbg;
  const long long t_kernel = dbg ? clock64() : 0;

  if (tid == 0) {
    for (int s = 0; s < kFusedStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], kFusedComputeWarps);
      mbar_init(&S.adoneB[s], kFusedComputeWarps);
      mbar_init(&S.cfullB[s], 1);
    }
    for (int s = 0; s < kASlots; ++s) {
      mbar_init(&S.adoneA[s], kFusedComputeWarps);
      mbar_init(&S.afree[s], 1);
    }
    for (int j = 0; j < kPubRing; ++j) {
      mbar_init(&S.pubfull[j], 1);
      mbar_init(&S.pubempty[j], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const __nv_bfloat16* logits = static_cast<const __nv_bfloat16*>(p.logits);
  __nv_bfloat16* dl = static_cast<__nv_bfloat16*>(p.dlogits);

  // --------------------------------------------------------- loader warp
  if (warp == kWarpLoader) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      const uint64_t pol_keep = l2_policy_evict_last();
      for (int64_t n = 0; n < nops; ++n) {
        const int s = static_cast<int>(n % kFusedStages);
        if (n >= kFusedStages) {
          DBG_T0();
          mbar_wait(&S.empty[s], static_cast<uint32_t>(((n / kFusedStages) - 1) & 1));
          DBG_ADD(8);
        }
        bool isB;
        int64_t k;
        op_of(n, nloc, L, &isB, &k);
        mbar_arrive_expect_tx(&S.full[s], row_bytes);
        if (isB)  // second (last) read of the row: from L2, then evict
          tma_load_1d_evict_first(buf(s), logits + row_of(k) * V, row_bytes, &S.full[s], pol);
        else if (a_evict_last && write_dl)  // keep in L2 until B re-reads it
          tma_load_1d_evict_first(buf(s), logits + row_of(k) * V, row_bytes, &S.full[s], pol_keep);
        else
          tma_load_1d(buf(s), logits + row_of(k) * V, row_bytes, &S.full[s]);
      }
    }
    return;
  }

  if (warp == kWarpStore) return;  // dlogits are stored by the compute warps

  // ------------------------------------------------------ publisher warp
  // Publishes each row's lp_tok and bumps its chunk counter with a release
  // reduction; the release fence's wait for the store stalls only this warp.
  if (warp == kWarpPublish) {
    if (!write_dl || lane != 0) return;
    int64_t na = 0;  // A ops seen
    for (int64_t n = 0; n < nops; ++n) {
      bool isB;
      int64_t k;
      op_of(n, nloc, L, &isB, &k);
      if (isB) continue;
      const int j = static_cast<int>(na % kPubRing);
      {
        DBG_T0();
        mbar_wait(&S.pubfull[j], static_cast<uint32_t>((na / kPubRing) & 1));
        DBG_ADD(13);
      }
      const long long t_pub = dbg ? clock64() : 0;
      ++na;
      const double lp = S.pub_lp[j];
      mbar_arrive(&S.pubempty[j]);
      const int64_t r = row_of(k);
      p.lp_tok[r] = lp;
      red_release_gpu_add(p.cnt + r / T, 1u);
      if (dbg) atomicAdd(dbg + 14, static_cast<unsigned long long>(clock64() - t_pub));
    }
    return;
  }

  // ---------------------------------------------------- coefficient warp
  if (warp == kCoefWarp) {
    int64_t a = 0, b = 0;  // A / B op counters
    // Prefetched inputs of the next B row's chunk coefficient.  Every CTA
    // evaluates the coefficients of its own B rows from the published token
    // log-probs (same inputs, same code: bitwise identical across CTAs), so
    // no CTA ever waits on another CTA's finaliser -- only on its rows.
    int64_t pq = -1;       // chunk being prefetched
    uint32_t pc = 0;       // acquired counter value (this lane)
    bool pv_ok = false;    // pv[] holds the chunk's token log-probs
    double pv[4] = {0.0, 0.0, 0.0, 0.0};
    float pblp = 0.f;
    double padv = 0.0;
    auto prefetch_vals = [&]() {
      // called with pc acquired on every lane; loads ordered after the acquire
      const double* lt = p.lp_tok + pq * T;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int64_t t = 32 * m + lane;
        pv[m] = (t < T) ? __ldcg(lt + t) : 0.0;
      }
      pblp = __ldg(p.blp + pq);
      padv = __ldg(p.adv + pq / p.C);
      pv_ok = true;
    };
    auto poll = [&]() {  // advance the prefetch state machine without blocking
      if (pq < 0 || pv_ok) return;
      if (__all_sync(0xffffffffu, pc >= static_cast<uint32_t>(T)))
        prefetch_vals();
      else
        pc = ld_acquire_gpu(p.cnt + pq);
    };
    auto process = [&](int64_t n) {
      bool isB;
      int64_t k;
      op_of(n, nloc, L, &isB, &k);
      const int64_t r = row_of(k);
      if (!isB) {
        // ---- tail of A(k): lse (f64) and the target's log-prob
        const int sa = static_cast<int>(a % kASlots);
        {
          DBG_T0();
          mbar_wait(&S.adoneA[sa], static_cast<uint32_t>((a / kASlots) & 1));
          if (lane == 0) { DBG_ADD(2); }
        }
        // read everything this tail needs from slot sa, then free the stage
        // (the compute warps already gathered the target logit)
        const int32_t tgt = S.tgta[sa];
        const float xt_f = S.xt[sa];
        const float mw = (lane < kFusedComputeWarps) ? S.wm[sa][lane] : -INFINITY;
        const double sw = (lane < kFusedComputeWarps) ? S.ws[sa][lane] : 0.0;
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.afree[sa]);  // partial slot sa consumed
        const long long t_tail = dbg ? clock64() : 0;
        const int j = static_cast<int>(a % kPubRing);
        const uint32_t pe_ph = static_cast<uint32_t>(((a / kPubRing) - 1) & 1);
        const bool pub_reuse = write_dl && a >= kPubRing;
        ++a;
        const float M = warp_max_f32(mw);
        double term = (lane < kFusedComputeWarps && sw > 0.0)
                          ? sw * static_cast<double>(ex2f((mw - M) * kLog2e))
                          : 0.0;
        term = warp_sum_f64(term);
        if (lane == 0) {
          const double lse = static_cast<double>(M) + log(term);
          const double xt = static_cast<double>(xt_f);
          if (tgt < 0) atomicOr(p.err, kErrToken);
          if (write_dl) {
            S.ring_lse[k % kRing] = lse;
            S.ring_tgt[k % kRing] = tgt;
            if (pub_reuse) mbar_wait(&S.pubempty[j], pe_ph);
            S.pub_lp[j] = xt - lse;
            mbar_arrive(&S.pubfull[j]);
          } else {
            p.lse[r] = lse;
            p.lp_tok[r] = xt - lse;
          }
          if (dbg) atomicAdd(dbg + 3, static_cast<unsigned long long>(clock64() - t_tail));
        }
        __syncwarp();
        if (write_dl) poll();
      } else {
        // ---- coefficient for B(k); slot b % 3 is free once B op b-3 is done
        const int sb = static_cast<int>(b % kFusedStages);
        if (b >= kFusedStages) {
          DBG_T0();
          mbar_wait(&S.adoneB[sb], static_cast<uint32_t>(((b - kFusedStages) / kFusedStages) & 1));
          if (lane == 0) { DBG_ADD(4); }
        }
        const long long t_prep = dbg ? clock64() : 0;
        ++b;
        const int64_t q = r / T;
        if (pq != q) {  // no prefetch for this chunk (first B op)
          pq = q;
          pv_ok = false;
          pc = ld_acquire_gpu(p.cnt + q);
        }
        if (!pv_ok) {
          DBG_T0();
          if (dbg && lane == 0) atomicAdd(dbg + 11, 1ull);
          const uint64_t t0 = globaltimer_ns();
          uint32_t ns = 32;
          while (!__all_sync(0xffffffffu, pc >= static_cast<uint32_t>(T))) {
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
            pc = ld_acquire_gpu(p.cnt + q);
            if (globaltimer_ns() - t0 > kSpinTimeoutNs) {
              if (lane == 0) atomicOr(p.err, kErrTimeout);
              break;
            }
          }
          prefetch_vals();
          if (lane == 0) { DBG_ADD(6); }
        }
        const double lp = warp_pairwise_small(pv, static_cast<int>(T), lane);
        if (lane == 0) {
          ChunkTerms ct = chunk_terms(lp, static_cast<double>(pblp), padv, p.w, p.clip_eps,
                                      p.kl_coeff);
          const double c = ct.coeff;
          if (r % T == 0) {  // one writer per chunk for the epilogue
            p.lp_chunk[q] = lp;
            p.coeff[q] = c;
          }
          const double lse = S.ring_lse[k % kRing];
          const int32_t tgt = S.ring_tgt[k % kRing];
          uint32_t mode;
          if (c == 0.0) {
            mode = 0u;
          } else if (!isfinite(c)) {
            mode = 2u;
          } else {
            mode = 1u | ((c > 0.0) ? 0x80000000u : 0u);
            S.kval[sb] = static_cast<float>(lse * 1.4426950408889634 - log2(fabs(c)));
          }
          S.mode[sb] = mode;
          S.cf[sb] = static_cast<float>(c);
          S.lseL[sb] = static_cast<float>(lse * 1.4426950408889634);
          S.tgt[sb] = tgt;
          mbar_arrive(&S.cfullB[sb]);
          if (dbg) atomicAdd(dbg + 5, static_cast<unsigned long long>(clock64() - t_prep));
        }
        __syncwarp();
        // start prefetching the next B row's chunk (same chunk: reuse)
        if (k + 1 < nloc) {
          const int64_t nq = row_of(k + 1) / T;
          if (nq != pq) {
            pq = nq;
            pv_ok = false;
            pc = ld_acquire_gpu(p.cnt + nq);
          }
        }
      }
    };
    // B(k) is handled before the A(k+L) that precedes it in the op sequence
    // (its coefficient depends only on the tails of rows k and k+1), so the
    // compute warps find it ready when they finish A(k+L).  Only inside the
    // paired region and with an effective lag >= 2 (tests/test_fused_protocol.py).
    const int64_t Le = nloc < L ? nloc : L;
    const int64_t pair_end = Le + 2 * (nloc - Le);
    for (int64_t n = 0; n < nops;) {
      bool isB0, isB1 = false;
      int64_t k0, k1;
      op_of(n, nloc, L, &isB0, &k0);
      if (n + 1 < nops) op_of(n + 1, nloc, L, &isB1, &k1);
      if (!isB0 && isB1 && Le >= 2 && n + 1 < pair_end) {
        process(n + 1);
        process(n);
        n += 2;
      } else {
        process(n);
        n += 1;
      }
    }
    return;
  }

  // ------------------------------------------------------- compute warps
  const int nvec = static_cast<int>(V >> 3);  // uint4 = 8 bf16
  int64_t a = 0, b = 0;  // A / B op counters
  for (int64_t n = 0; n < nops; ++n) {
    const int s = static_cast<int>(n % kFusedStages);
    const uint32_t ph = static_cast<uint32_t>((n / kFusedStages) & 1);
    bool isB;
    int64_t k;
    op_of(n, nloc, L, &isB, &k);
    {
      DBG_T0();
      mbar_wait(&S.full[s], ph);
      if (tid == 0) { DBG_ADD(0); }
    }
    if (!isB) {
      const int32_t tg = (tid == 0) ? __ldg(p.tokens + row_of(k)) : 0;  // used at the end
      const uint4* v = reinterpret_cast<const uint4*>(buf(s));
      uint32_t mx0 = 0xff80ff80u, mx1 = 0xff80ff80u;
#pragma unroll 4
      for (int i = tid; i < nvec; i += kFusedComputeThreads) {
        const uint4 x = v[i];
        mx0 = bf16x2_max(mx0, bf16x2_max(x.x, x.y));
        mx1 = bf16x2_max(mx1, bf16x2_max(x.z, x.w));
      }
      const uint32_t mx = bf16x2_max(mx0, mx1);
      const float m = warp_max_f32(fmaxf(bf16lo(mx), bf16hi(mx)));
      const float mL = m * kLog2e;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 2
      for (int i = tid; i < nvec; i += kFusedComputeThreads) {
        const uint4 x = v[i];
        s0 += ex2f(fmaf(bf16lo(x.x), kLog2e, -mL)) + ex2f(fmaf(bf16hi(x.x), kLog2e, -mL));
        s1 += ex2f(fmaf(bf16lo(x.y), kLog2e, -mL)) + ex2f(fmaf(bf16hi(x.y), kLog2e, -mL));
        s2 += ex2f(fmaf(bf16lo(x.z), kLog2e, -mL)) + ex2f(fmaf(bf16hi(x.z), kLog2e, -mL));
        s3 += ex2f(fmaf(bf16lo(x.w), kLog2e, -mL)) + ex2f(fmaf(bf16hi(x.w), kLog2e, -mL));
      }
      // gather the target logit while the row is in SMEM, then free the stage
      const bool tok_ok = tg >= 0 && tg < V;
      const float xt_v = (tid == 0 && tok_ok)
                             ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(buf(s))[tg])
                             : __int_as_float(0x7fc00000);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[s]);
      double part = (static_cast<double>(s0) + static_cast<double>(s1)) +
                    (static_cast<double>(s2) + static_cast<double>(s3));
      part = warp_sum_f64(part);
      const int sa = static_cast<int>(a % kASlots);
      if (a >= kASlots)  // the coefficient warp has read A row a-8's partials
        mbar_wait(&S.afree[sa], static_cast<uint32_t>(((a - kASlots) / kASlots) & 1));
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
      mbar_wait(&S.cfullB[sb], static_cast<uint32_t>((b / kFusedStages) & 1));
      if (tid == 0) { DBG_ADD(1); }
    }
    ++b;
    const uint32_t mode = S.mode[sb];
    const uint4* v = reinterpret_cast<const uint4*>(buf(s));
    uint4* dst = reinterpret_cast<uint4*>(dl + row_of(k) * V);
    if ((mode & 3u) != 1u) {
      // zero-gradient rows (A == 0 or clipped chunk): 0 * (onehot - p)
      const uint32_t z = (mode == 0u) ? 0u : 0x7fc07fc0u;
      for (int i = tid; i < nvec; i += kFusedComputeThreads) __stcs(dst + i, make_uint4(z, z, z, z));
    } else {
      // -c * p_v = -sign(c) * 2^(x*log2e - (lse*log2e - log2|c|))
      const float K = S.kval[sb];
      const uint32_t sgn = (mode & 0x80000000u) ? 0x80008000u : 0u;
      const int32_t tgt = S.tgt[sb];
      const int tv = tgt >> 3;
#pragma unroll 2
      for (int i = tid; i < nvec; i += kFusedComputeThreads) {
        const uint4 x = v[i];
        uint4 o;
        o.x = pack_bf16x2(ex2f(fmaf(bf16lo(x.x), kLog2e, -K)), ex2f(fmaf(bf16hi(x.x), kLog2e, -K))) ^ sgn;
        o.y = pack_bf16x2(ex2f(fmaf(bf16lo(x.y), kLog2e, -K)), ex2f(fmaf(bf16hi(x.y), kLog2e, -K))) ^ sgn;
        o.z = pack_bf16x2(ex2f(fmaf(bf16lo(x.z), kLog2e, -K)), ex2f(fmaf(bf16hi(x.z), kLog2e, -K))) ^ sgn;
        o.w = pack_bf16x2(ex2f(fmaf(bf16lo(x.w), kLog2e, -K)), ex2f(fmaf(bf16hi(x.w), kLog2e, -K))) ^ sgn;
        if (i == tv) {
          // target column: c * (1 - p_t)
          const int e = tgt & 7;
          const uint32_t word = (e >> 1) == 0 ? x.x : (e >> 1) == 1 ? x.y : (e >> 1) == 2 ? x.z : x.w;
          const float xt = (e & 1) ? bf16hi(word) : bf16lo(word);
          const float pt = ex2f(fmaf(xt, kLog2e, -S.lseL[sb]));
          const float val = S.cf[sb] * (1.0f - pt);
          const uint32_t b = pack_bf16x2(val, val) & 0xffffu;
          uint32_t ow = (e >> 1) == 0 ? o.x : (e >> 1) == 1 ? o.y : (e >> 1) == 2 ? o.z : o.w;
          ow = (e & 1) ? ((ow & 0x0000ffffu) | (b << 16)) : ((ow & 0xffff0000u) | b);
          if ((e >> 1) == 0) o.x = ow;
          else if ((e >> 1) == 1) o.y = ow;
          else if ((e >> 1) == 2) o.z = ow;
          else o.w = ow;
        }
        __stcs(dst + i, o);
      }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&S.empty[s]);   // B row read: the stage may be reloaded
      mbar_arrive(&S.adoneB[sb]);
    }
  }
  if (dbg && tid == 0) atomicAdd(dbg + 12, static_cast<unsigned long long>(clock64() - t_kernel));
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
  auto val = [&](float x, int64_t col) {
    const float pv = ex2f(fmaf(x, kLog2e, -lseL));
    return (col == tgt) ? cf * (1.0f - pv) : -cf * pv;
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
      if (tid == 0) {
        for (int64_t t = 0; t < lim; ++t) loss = __dadd_rn(loss, s_loss[t]);
      } else if (tid == 32) {
        for (int64_t t = 0; t < lim; ++t) ratio_sum = __dadd_rn(ratio_sum, s_rho[t]);
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
  uint32_t* cnt;
  uint32_t* reward_bad;
  uint32_t* err;
  size_t bytes;
  size_t zero_off, zero_bytes;  // region memset every call (cnt, err)
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
  w.zero_off = off;
  w.cnt = reinterpret_cast<uint32_t*>(take(nq * 4));
  w.err = reinterpret_cast<uint32_t*>(take(16));
  w.zero_bytes = off - w.zero_off;
  w.bytes = off;
  return w;
}

static size_t fused_smem_bytes(int64_t V) {
  const size_t hdr = ((sizeof(FusedSmem) + 127) / 128) * 128;
  const size_t stage = ((static_cast<size_t>(V) * 2 + 127) / 128) * 128;
  return hdr + kFusedStages * stage;
}

}  // namespace dvla

using namespace dvla;

extern "C" size_t dvla_token_loss_workspace_bytes(int64_t n_groups, int64_t G, int64_t C,
                                                  int64_t T) {
  if (n_groups < 0 || G < 0 || C < 0 || T < 0) return 0;
  return carve(nullptr, n_groups, G, C, T).bytes;
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
  p.cnt = ws.cnt;
  p.err = ws.err;
  p.R = R;
  p.V = V;
  p.T = T;
  p.C = C;
  p.n_chunks = nq;
  p.w = 1.0 / static_cast<double>(n_traj * C);
  p.clip_eps = clip_eps;
  p.kl_coeff = kl_coeff;

  DVLA_CUDA_TRY(cudaMemsetAsync(static_cast<uint8_t*>(workspace) + ws.zero_off, 0,
                                ws.zero_bytes, stream));
  {
    const int thr = 128;
    tok_adv_kernel<<<(unsigned)((n_groups + thr - 1) / thr), thr, 0, stream>>>(
        rewards, n_groups, G, adv_eps, ws.adv, ws.reward_bad);
    if (int rc = launch_check("tok_adv_kernel")) return rc;
  }

  const int dev = current_device();
  const int sms = num_sms(dev);
  const size_t esz = dtype == DVLA_BF16 ? 2 : 4;
  const bool aligned16 = (reinterpret_cast<uintptr_t>(logits) % 16 == 0) &&
                         (!want_dl || reinterpret_cast<uintptr_t>(dlogits) % 16 == 0) &&
                         ((V * esz) % 16 == 0);
  const size_t fsmem = fused_smem_bytes(V);
  const bool fused = !(flags & DVLA_TL_UNFUSED) && dtype == DVLA_BF16 && aligned16 &&
                     fsmem <= 227 * 1024 && T <= sms && T <= 128 && R >= 1;
  if (fused) {
    static bool attr_set[64] = {false};
    if (!attr_set[dev & 63]) {
      DVLA_CUDA_TRY(cudaFuncSetAttribute(tok_fused_bf16_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024));
      attr_set[dev & 63] = true;
    }
    const unsigned grid = static_cast<unsigned>(R < sms ? R : sms);
    const uint32_t stage_bytes = static_cast<uint32_t>(((V * 2 + 127) / 128) * 128);
    cudaEvent_t stop;
    prof_begin(stream, &stop);
    static const int lag = [] {
      const char* e = getenv("DVLA_FUSED_LAG");
      return e ? atoi(e) : kLagRounds;
    }();
    static const int a_keep = [] {
      const char* e = getenv("DVLA_FUSED_KEEP");
      return e ? atoi(e) : 0;
    }();
    tok_fused_bf16_kernel<<<grid, kFusedThreadsWS, fsmem, stream>>>(p, stage_bytes, want_dl ? 1 : 0,
                                                                     lag < 2 ? 2 : lag, a_keep);
    prof_end(stream, stop);
    if (int rc = launch_check("tok_fused_bf16_kernel")) return rc;
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
  grpo_epilogue_kernel<<<1, kEpiThreads, 0, stream>>>(e);
  return launch_check("grpo_epilogue_kernel");
}

// Debug only (not part of the header): point the fused kernel's per-role
// cycle counters at a device buffer of 16 u64 (or null to disable).
extern "C" int dvla_debug_fused_counters(void* dev_buf) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_buf);
  DVLA_CUDA_TRY(cudaMemcpyToSymbol(g_dbg, &p, sizeof(p)));
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
                                                        reward_bad);
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
