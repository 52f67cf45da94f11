// Learner optimizer tail on the TRAINER stream:
//   adam_step      reference grpo.py:137-150 (bias-corrected Adam, f64
//                  moments, f32 params), bit-identical element-wise arithmetic
//   grad_norm      reference grpo.py:297-301 (clip_grad_norm), deterministic
//                  fixed-shape f64 reduction (+ optional in-place scaling)
//   finite check   grpo.py:282-283 / runtime.py:793-795 (non-finite gradient
//                  or parameters -> abort)
#include "common.cuh"

namespace dvla {

struct AdamConsts {
  double beta1, one_m_beta1, beta2, one_m_beta2, bc1, bc2, lr, eps;
  double ibc1, ibc2;   // RN(1 / bc1), RN(1 / bc2): host IEEE divisions
};

// a / b, correctly rounded, for a divisor fixed per launch with y = RN(1/b)
// computed on the host: q = RN(a y), the remainder r = a - b q exactly (one
// FMA), then RN(q + r y) -- Markstein's correction, which returns RN(a/b)
// when y is within half an ulp of 1/b and q within one ulp of a/b.  Three
// f64 operations instead of __ddiv_rn's reciprocal refinement and range
// checks; used for |a| in [2^-900, 2^1000] (every intermediate normal for
// the divisors here, 1e-3 .. 16), the full division elsewhere, the sign of
// a zero kept (tests/test_grpo_gpu.py: bitwise against numpy on 4M wide
// inputs per step / node count, subnormal and -0 moments included).
__device__ __forceinline__ double div_const(double a, double b, double y) {
  const double aa = fabs(a);
  if (aa >= 0x1p-900 && aa <= 0x1p+1000) {
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-q, b, a);
    return __fma_rn(r, y, q);
  }
  if (a == 0.0) return a;
  return __ddiv_rn(a, b);
}

// one element, the reference's arithmetic in its order (grpo.py:143-150)
__device__ __forceinline__ float adam_elem(float p, double gi, double& m, double& v,
                                           const AdamConsts& c) {
  double mi = __dmul_rn(m, c.beta1);
  mi = __dadd_rn(mi, __dmul_rn(c.one_m_beta1, gi));
  double vi = __dmul_rn(v, c.beta2);
  vi = __dadd_rn(vi, __dmul_rn(c.one_m_beta2, __dmul_rn(gi, gi)));
  m = mi;
  v = vi;
  const double mh = div_const(mi, c.bc1, c.ibc1);
  const double vh = div_const(vi, c.bc2, c.ibc2);
  const double upd = __dsub_rn(static_cast<double>(p),
                               __ddiv_rn(__dmul_rn(c.lr, mh), __dadd_rn(__dsqrt_rn(vh), c.eps)));
  return __double2float_rn(upd);
}

// HBM-bound (48 bytes per parameter): pairs of elements per thread with
// 8-/16-byte accesses, two pairs in flight; a scalar tail for odd n or
// misaligned arrays.
__global__ void adam_kernel(float* __restrict__ p, const double* __restrict__ g,
                            double* __restrict__ m, double* __restrict__ v, int64_t n,
                            AdamConsts c, int vec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int64_t done = 0;
  if (vec) {
    const int64_t npair = n / 2;
    float2* p2 = reinterpret_cast<float2*>(p);
    const double2* g2 = reinterpret_cast<const double2*>(g);
    double2* m2 = reinterpret_cast<double2*>(m);
    double2* v2 = reinterpret_cast<double2*>(v);
    int64_t i = t0;
    for (; i + stride < npair; i += 2 * stride) {
      float2 pa = p2[i], pb = p2[i + stride];
      const double2 ga = __ldcs(g2 + i), gb = __ldcs(g2 + i + stride);
      double2 ma = m2[i], mb = m2[i + stride], va = v2[i], vb = v2[i + stride];
      pa.x = adam_elem(pa.x, ga.x, ma.x, va.x, c);
      pa.y = adam_elem(pa.y, ga.y, ma.y, va.y, c);
      pb.x = adam_elem(pb.x, gb.x, mb.x, vb.x, c);
      pb.y = adam_elem(pb.y, gb.y, mb.y, vb.y, c);
      p2[i] = pa;
      p2[i + stride] = pb;
      m2[i] = ma;
      m2[i + stride] = mb;
      v2[i] = va;
      v2[i + stride] = vb;
    }
    for (; i < npair; i += stride) {
      float2 pa = p2[i];
      const double2 ga = __ldcs(g2 + i);
      double2 ma = m2[i], va = v2[i];
      pa.x = adam_elem(pa.x, ga.x, ma.x, va.x, c);
      pa.y = adam_elem(pa.y, ga.y, ma.y, va.y, c);
      p2[i] = pa;
      m2[i] = ma;
      v2[i] = va;
    }
    done = npair * 2;
  }
  for (int64_t i = done + t0; i < n; i += stride) {
    double mi = m[i], vi = v[i];
    p[i] = adam_elem(p[i], g[i], mi, vi, c);
    m[i] = mi;
    v[i] = vi;
  }
}

// The learner tail in one pass (runtime.py:788-796: total /= w -> reduce
// -> clip_grad_norm -> adam_step -> non-finite check), for an f32 gradient
// (the head GEMM's output, all-reduced as the reference's f32 frames):
//   gi = f64(g32[i]); gi = gi / div (the cross-node mean, div = nodes);
//   gi = gi * (max_norm / norm) when norm > max_norm > 0 (clip_grad_norm's
//   in-place scaling, same f64 expression); then the Adam element above.
// `skip` (device f32, e.g. the all-reduced abort count): nonzero -> the
// whole update is skipped on the device (every rank alike), so the host
// checks the abort after one synchronisation instead of before the step;
// a non-finite `norm` (non-finite gradient) skips it too.
// Optional outputs: the new parameters rounded to bf16 (the weights the
// next forward GEMM and the published snapshot read) and a flag raised
// when any new parameter is non-finite.
#ifndef DVLA_ADAM_CTAS
#define DVLA_ADAM_CTAS 3   // CTAs per SM the tail is compiled for (register budget)
#endif

struct TailArgs {
  float* p;
  const float* g;
  double* m;
  double* v;
  int64_t n;
  AdamConsts c;
  double div;
  double idiv;   // RN(1 / div)
  const double* norm;
  double max_norm;
  const float* skip;
  __nv_bfloat16* w16;
  unsigned* nonfinite;
};

__device__ __forceinline__ double tail_grad(float g32, double div, double idiv, bool clip,
                                            double f) {
  double gi = static_cast<double>(g32);
  if (div != 1.0) gi = div_const(gi, div, idiv);
  if (clip) gi = __dmul_rn(gi, f);
  return gi;
}

// kPeers: the bf16 copy is also stored straight into every peer learner's
// working copy (IPC-mapped, same element offset) -- the ZeRO-1 all-gather
// fused into the optimizer tail: a warp's 128 contiguous bytes go out as one
// NVLink write per peer while the kernel streams its 46 B / parameter from
// HBM.
constexpr int kMaxBf16Peers = 31;
struct Bf16Peers {
  __nv_bfloat16* p[kMaxBf16Peers];
  int n;
};

template <bool kPeers>
__global__ void __launch_bounds__(256, DVLA_ADAM_CTAS)
    adam_tail_kernel(TailArgs a, int vec, Bf16Peers peers) {
  if (a.skip != nullptr && *a.skip != 0.0f) return;
  bool clip = false;
  double f = 1.0;
  if (a.norm != nullptr) {
    const double nm = a.norm[0];
    if (!isfinite(nm)) return;  // non-finite gradient: grpo.py:282-283 aborts the update
    if (nm > a.max_norm && a.max_norm > 0.0) {
      clip = true;
      f = a.max_norm / nm;
    }
  }
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  unsigned bad = 0;
  int64_t done = 0;
  if (vec) {
    const int64_t npair = a.n / 2;
    float2* p2 = reinterpret_cast<float2*>(a.p);
    const float2* g2 = reinterpret_cast<const float2*>(a.g);
    double2* m2 = reinterpret_cast<double2*>(a.m);
    double2* v2 = reinterpret_cast<double2*>(a.v);
    __nv_bfloat162* w2 = reinterpret_cast<__nv_bfloat162*>(a.w16);
    // two pairs in flight per thread (the loads of both before any math)
    int64_t i = t0;
    for (; i + stride < npair; i += 2 * stride) {
      float2 pa = p2[i], pb = p2[i + stride];
      const float2 ga = __ldcs(g2 + i), gb = __ldcs(g2 + i + stride);
      double2 ma = m2[i], mb = m2[i + stride], va = v2[i], vb = v2[i + stride];
      pa.x = adam_elem(pa.x, tail_grad(ga.x, a.div, a.idiv, clip, f), ma.x, va.x, a.c);
      pa.y = adam_elem(pa.y, tail_grad(ga.y, a.div, a.idiv, clip, f), ma.y, va.y, a.c);
      pb.x = adam_elem(pb.x, tail_grad(gb.x, a.div, a.idiv, clip, f), mb.x, vb.x, a.c);
      pb.y = adam_elem(pb.y, tail_grad(gb.y, a.div, a.idiv, clip, f), mb.y, vb.y, a.c);
      p2[i] = pa;
      p2[i + stride] = pb;
      m2[i] = ma;
      m2[i + stride] = mb;
      v2[i] = va;
      v2[i + stride] = vb;
      if (w2 != nullptr) {
        const __nv_bfloat162 ba = __floats2bfloat162_rn(pa.x, pa.y);
        const __nv_bfloat162 bb = __floats2bfloat162_rn(pb.x, pb.y);
        w2[i] = ba;
        w2[i + stride] = bb;
        if constexpr (kPeers) {
#pragma unroll
          for (int q = 0; q < kMaxBf16Peers; ++q) {   // static indices: no local copy
            if (q >= peers.n) break;
            __nv_bfloat162* r2 = reinterpret_cast<__nv_bfloat162*>(peers.p[q]);
            r2[i] = ba;
            r2[i + stride] = bb;
          }
        }
      }
      bad |= !isfinite(pa.x) | !isfinite(pa.y) | !isfinite(pb.x) | !isfinite(pb.y);
    }
    for (; i < npair; i += stride) {
      float2 pa = p2[i];
      const float2 ga = __ldcs(g2 + i);
      double2 ma = m2[i], va = v2[i];
      pa.x = adam_elem(pa.x, tail_grad(ga.x, a.div, a.idiv, clip, f), ma.x, va.x, a.c);
      pa.y = adam_elem(pa.y, tail_grad(ga.y, a.div, a.idiv, clip, f), ma.y, va.y, a.c);
      p2[i] = pa;
      m2[i] = ma;
      v2[i] = va;
      if (w2 != nullptr) {
        const __nv_bfloat162 ba = __floats2bfloat162_rn(pa.x, pa.y);
        w2[i] = ba;
        if constexpr (kPeers) {
#pragma unroll
          for (int q = 0; q < kMaxBf16Peers; ++q) {
            if (q >= peers.n) break;
            reinterpret_cast<__nv_bfloat162*>(peers.p[q])[i] = ba;
          }
        }
      }
      bad |= !isfinite(pa.x) | !isfinite(pa.y);
    }
    done = npair * 2;
  }
  for (int64_t i = done + t0; i < a.n; i += stride) {
    double mi = a.m[i], vi = a.v[i];
    const float pn = adam_elem(a.p[i], tail_grad(a.g[i], a.div, a.idiv, clip, f), mi, vi, a.c);
    a.p[i] = pn;
    a.m[i] = mi;
    a.v[i] = vi;
    if (a.w16 != nullptr) {
      const __nv_bfloat16 bn = __float2bfloat16_rn(pn);
      a.w16[i] = bn;
      if constexpr (kPeers) {
#pragma unroll
        for (int q = 0; q < kMaxBf16Peers; ++q) {
          if (q >= peers.n) break;
          peers.p[q][i] = bn;
        }
      }
    }
    bad |= !isfinite(pn);
  }
  if (a.nonfinite != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(a.nonfinite, 1u);
  if constexpr (kPeers) __threadfence_system();   // peer stores visible before completion
}

// skip word for adam_tail_kernel from the fused loss's stats vector: 1.0
// when the loss aborted (GrpoAbort), is non-finite (grpo.py:282-283) or its
// kernel reported an error
__global__ void loss_status_kernel(const double* __restrict__ stats, float* __restrict__ out) {
  out[0] = (stats[DVLA_ST_ABORT] != 0.0 || stats[DVLA_ST_KERNEL_ERR] != 0.0 ||
            !isfinite(stats[DVLA_ST_LOSS])) ? 1.0f : 0.0f;
}

constexpr int kNormThreads = 256;
constexpr int kNormBlocks = 16384;  // fixed: the reduction order never depends on the launch

// Block b sums g[b * per, (b + 1) * per) (per a multiple of 2 when the
// array is 16-byte aligned): 16-byte loads, two in flight per thread.
__global__ void sumsq_blocks_kernel(const double* __restrict__ g, int64_t n, int64_t per_block,
                                    double* __restrict__ partial, unsigned* __restrict__ nonfinite) {
  __shared__ double red[kNormThreads / 32];
  const int64_t lo = blockIdx.x * per_block;
  const int64_t hi = (lo + per_block < n) ? lo + per_block : n;
  double acc0 = 0.0, acc1 = 0.0;
  unsigned bad = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(g + lo) & 15) == 0);
  int64_t i = lo;
  if (vec) {
    const double2* g2 = reinterpret_cast<const double2*>(g + lo);
    const int64_t npair = (hi - lo) / 2;
    int64_t j = threadIdx.x;
    for (; j + 3 * kNormThreads < npair; j += 4 * kNormThreads) {
      const double2 a = __ldcs(g2 + j), b = __ldcs(g2 + j + kNormThreads);
      const double2 c = __ldcs(g2 + j + 2 * kNormThreads), d = __ldcs(g2 + j + 3 * kNormThreads);
      acc0 += (a.x * a.x + b.x * b.x) + (c.x * c.x + d.x * d.x);
      acc1 += (a.y * a.y + b.y * b.y) + (c.y * c.y + d.y * d.y);
      bad |= !isfinite(a.x) | !isfinite(a.y) | !isfinite(b.x) | !isfinite(b.y) |
             !isfinite(c.x) | !isfinite(c.y) | !isfinite(d.x) | !isfinite(d.y);
    }
    for (; j < npair; j += kNormThreads) {
      const double2 a = __ldcs(g2 + j);
      acc0 += a.x * a.x;
      acc1 += a.y * a.y;
      bad |= !isfinite(a.x) | !isfinite(a.y);
    }
    i = lo + npair * 2;
  }
  for (i += threadIdx.x; i < hi; i += kNormThreads) {
    const double x = g[i];
    acc0 += x * x;
    bad |= !isfinite(x);
  }
  double acc = warp_sum_f64(acc0 + acc1);
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

// f32 gradient variant: the norm of gi = f64(g32[i]) / div (the values
// adam_tail_kernel steps with).  16-byte loads, four in flight per thread;
// the squares of each 4-element load are summed in f64 (exact products of
// f32 values, f64 adds) -- the same fixed block shape as the f64 kernel, so
// the reduction order never depends on the launch.
__global__ void sumsq_blocks_f32_kernel(const float* __restrict__ g, int64_t n, int64_t per_block,
                                        double div, double* __restrict__ partial,
                                        unsigned* __restrict__ nonfinite) {
  __shared__ double red[kNormThreads / 32];
  const int64_t lo = blockIdx.x * per_block;
  const int64_t hi = (lo + per_block < n) ? lo + per_block : n;
  double acc0 = 0.0, acc1 = 0.0;
  unsigned bad = 0;
  const double inv = (div != 1.0) ? 1.0 / (div * div) : 1.0;  // only scales the norm
  auto sq4 = [](const float4& v) {
    const double a = v.x, b = v.y, c = v.z, d = v.w;
    return (a * a + b * b) + (c * c + d * d);
  };
  auto bad4 = [](const float4& v) {
    return !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
  };
  const bool vec = ((reinterpret_cast<uintptr_t>(g + lo) & 15) == 0);
  int64_t i = lo;
  if (vec) {
    const float4* g4 = reinterpret_cast<const float4*>(g + lo);
    const int64_t nq = (hi - lo) / 4;
    int64_t j = threadIdx.x;
    for (; j + 3 * kNormThreads < nq; j += 4 * kNormThreads) {
      const float4 a = __ldcs(g4 + j), b = __ldcs(g4 + j + kNormThreads);
      const float4 c = __ldcs(g4 + j + 2 * kNormThreads), d = __ldcs(g4 + j + 3 * kNormThreads);
      acc0 += sq4(a) + sq4(b);
      acc1 += sq4(c) + sq4(d);
      bad |= bad4(a) | bad4(b) | bad4(c) | bad4(d);
    }
    for (; j < nq; j += kNormThreads) {
      const float4 a = __ldcs(g4 + j);
      acc0 += sq4(a);
      bad |= bad4(a);
    }
    i = lo + nq * 4;
  }
  for (i += threadIdx.x; i < hi; i += kNormThreads) {
    const double x = g[i];
    acc0 += x * x;
    bad |= !isfinite(g[i]);
  }
  double acc = warp_sum_f64((acc0 + acc1) * inv);
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

// Reduce-scatter epilogue of the peer gradient exchange (runtime.py:618-627:
// the nodes' f32 frames summed in f64 in node order): out[i] = f32(sum over
// p in source order of f64(src[p][i])), and -- in the same pass, with
// sumsq_blocks_f32_kernel's block shape and per-thread order, so the two
// give identical partials -- the block sums of squares of out[i] / div.
constexpr int kMaxSumSrcs = 16;
struct SumSrcs {
  const float* p[kMaxSumSrcs];
};

// NS > 0: the source count at compile time, so every source's load of a
// granule is issued before the first add (NS loads in flight per granule,
// 4 NS per thread); NS == 0: runtime count (any n_src up to 16)
template <int NS>
__device__ __forceinline__ float4 sum_srcs4(const SumSrcs& s, int n_src, int64_t q) {
  constexpr int kMax = NS > 0 ? NS : kMaxSumSrcs;
  float4 v[NS > 0 ? NS : 1];
  if constexpr (NS > 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) v[k] = __ldcs(reinterpret_cast<const float4*>(s.p[k]) + q);
  }
  double x = 0.0, y = 0.0, z = 0.0, w = 0.0;
#pragma unroll
  for (int k = 0; k < kMax; ++k) {
    if constexpr (NS == 0) {
      if (k >= n_src) break;
    }
    const float4 u = NS > 0 ? v[NS > 0 ? k : 0]
                            : __ldcs(reinterpret_cast<const float4*>(s.p[k]) + q);
    x += u.x;
    y += u.y;
    z += u.z;
    w += u.w;
  }
  return make_float4(static_cast<float>(x), static_cast<float>(y), static_cast<float>(z),
                     static_cast<float>(w));
}

// one element (tails): static source indices, so the pointer table stays in
// the parameter bank (a runtime index would copy it to local memory)
template <int NS>
__device__ __forceinline__ float sum_srcs1(const SumSrcs& s, int n_src, int64_t i) {
  constexpr int kMax = NS > 0 ? NS : kMaxSumSrcs;
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < kMax; ++k) {
    if (NS == 0 && k >= n_src) break;
    t += s.p[k][i];
  }
  return static_cast<float>(t);
}

template <int NS>
__global__ void __launch_bounds__(kNormThreads) sum_sumsq_blocks_f32_kernel(
    SumSrcs src, int n_src, int64_t n, int64_t n_all, int64_t per_block, double div,
    float* __restrict__ out, double* __restrict__ partial, unsigned* __restrict__ nonfinite) {
  __shared__ double red[kNormThreads / 32];
  if (blockIdx.x == gridDim.x - 1) {   // [n, n_all): summed, outside the norm
    for (int64_t i = n + threadIdx.x; i < n_all; i += kNormThreads)
      out[i] = sum_srcs1<NS>(src, n_src, i);
  }
  if (static_cast<int64_t>(blockIdx.x) * per_block >= n) return;
  const int64_t lo = blockIdx.x * per_block;
  const int64_t hi = (lo + per_block < n) ? lo + per_block : n;
  double acc0 = 0.0, acc1 = 0.0;
  unsigned bad = 0;
  const double inv = (div != 1.0) ? 1.0 / (div * div) : 1.0;
  auto sq4 = [](const float4& v) {
    const double a = v.x, b = v.y, c = v.z, d = v.w;
    return (a * a + b * b) + (c * c + d * d);
  };
  auto bad4 = [](const float4& v) {
    return !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
  };
  // every source and `out` 16-byte aligned (checked on the host)
  const int64_t q0 = lo / 4;
  const int64_t nq = (hi - lo) / 4;
  float4* o4 = reinterpret_cast<float4*>(out);
  int64_t j = threadIdx.x;
  for (; j + 3 * kNormThreads < nq; j += 4 * kNormThreads) {
    const float4 a = sum_srcs4<NS>(src, n_src, q0 + j);
    const float4 b = sum_srcs4<NS>(src, n_src, q0 + j + kNormThreads);
    const float4 c = sum_srcs4<NS>(src, n_src, q0 + j + 2 * kNormThreads);
    const float4 d = sum_srcs4<NS>(src, n_src, q0 + j + 3 * kNormThreads);
    o4[q0 + j] = a;
    o4[q0 + j + kNormThreads] = b;
    o4[q0 + j + 2 * kNormThreads] = c;
    o4[q0 + j + 3 * kNormThreads] = d;
    acc0 += sq4(a) + sq4(b);
    acc1 += sq4(c) + sq4(d);
    bad |= bad4(a) | bad4(b) | bad4(c) | bad4(d);
  }
  for (; j < nq; j += kNormThreads) {
    const float4 a = sum_srcs4<NS>(src, n_src, q0 + j);
    o4[q0 + j] = a;
    acc0 += sq4(a);
    bad |= bad4(a);
  }
  for (int64_t i = lo + nq * 4 + threadIdx.x; i < hi; i += kNormThreads) {
    const float f = sum_srcs1<NS>(src, n_src, i);
    out[i] = f;
    const double x = f;
    acc0 += x * x;
    bad |= !isfinite(f);
  }
  double acc = warp_sum_f64((acc0 + acc1) * inv);
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

// fixed-order finish: thread t sums partials t, t + 1024, ... sequentially,
// then a warp-shuffle and a 32-entry tree (deterministic, one block)
constexpr int kFinishThreads = 1024;
__global__ void __launch_bounds__(kFinishThreads) norm_finish_kernel(
    const double* __restrict__ partial, int nblocks, double* __restrict__ out, int want_sqrt = 1) {
  __shared__ double red[kFinishThreads / 32];
  double acc = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += kFinishThreads) acc += partial[b];
  acc = warp_sum_f64(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kFinishThreads / 32; ++w) t += red[w];
    out[0] = want_sqrt ? sqrt(t) : t;
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
  const AdamConsts c{beta1, 1.0 - beta1, beta2, 1.0 - beta2, 1.0 - b1p, 1.0 - b2p, lr, eps,
                     1.0 / (1.0 - b1p), 1.0 / (1.0 - b2p)};
  const int vec = ((reinterpret_cast<uintptr_t>(params) & 7) == 0 &&
                   (reinterpret_cast<uintptr_t>(grad) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(m) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(v) & 15) == 0) ? 1 : 0;
  adam_kernel<<<grid_n(vec ? (n + 1) / 2 : n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      params, grad, m, v, n, c, vec);
  return launch_check("adam_kernel");
}

extern "C" size_t dvla_grad_norm_workspace_bytes(int64_t n) {
  (void)n;
  return kNormBlocks * sizeof(double) + 256;
}

// norm_out (device f64[1]) = ||grad||_2; scales grad in place when
// max_norm > 0 and norm > max_norm; nonfinite_out (device u32) |= any
// non-finite element.
extern "C" int dvla_grad_norm(double* grad, int64_t n, double max_norm, double* norm_out,
                              uint32_t* nonfinite_out, void* workspace, void* stream) {
  if (n < 0 || !norm_out || !nonfinite_out || !workspace)
    return fail(DVLA_ERR_USAGE, "bad grad_norm arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nblocks = kNormBlocks;
  const int64_t per = ((n + nblocks - 1) / nblocks + 1) & ~int64_t{1};  // even: aligned pairs
  double* partial = static_cast<double*>(workspace);
  DVLA_CUDA_TRY(cudaMemsetAsync(partial, 0, nblocks * sizeof(double), st));
  if (n > 0) {
    const int used = static_cast<int>((n + per - 1) / per);
    sumsq_blocks_kernel<<<used, kNormThreads, 0, st>>>(grad, n, per, partial,
                                                       reinterpret_cast<unsigned*>(nonfinite_out));
    if (int rc = launch_check("sumsq_blocks_kernel")) return rc;
  }
  norm_finish_kernel<<<1, kFinishThreads, 0, st>>>(partial, nblocks, norm_out);
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

// ---- the learner tail for an f32 gradient (see adam_tail_kernel)
static int grad_sumsq_f32(const float* grad, int64_t n, double div, double* out,
                          uint32_t* nonfinite_out, void* workspace, void* stream, int want_sqrt) {
  if (n < 0 || !out || !nonfinite_out || !workspace || !(div > 0.0))
    return fail(DVLA_ERR_USAGE, "bad grad_norm_f32 arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nblocks = kNormBlocks;
  const int64_t per = ((n + nblocks - 1) / nblocks + 3) & ~int64_t{3};  // 16-byte blocks
  double* partial = static_cast<double*>(workspace);
  DVLA_CUDA_TRY(cudaMemsetAsync(partial, 0, nblocks * sizeof(double), st));
  if (n > 0) {
    const int used = static_cast<int>((n + per - 1) / per);
    sumsq_blocks_f32_kernel<<<used, kNormThreads, 0, st>>>(
        grad, n, per, div, partial, reinterpret_cast<unsigned*>(nonfinite_out));
    if (int rc = launch_check("sumsq_blocks_f32_kernel")) return rc;
  }
  norm_finish_kernel<<<1, kFinishThreads, 0, st>>>(partial, nblocks, out, want_sqrt);
  return launch_check("norm_finish_kernel");
}

extern "C" int dvla_grad_norm_f32(const float* grad, int64_t n, double div, double* norm_out,
                                  uint32_t* nonfinite_out, void* workspace, void* stream) {
  return grad_sumsq_f32(grad, n, div, norm_out, nonfinite_out, workspace, stream, 1);
}

extern "C" int dvla_grad_sumsq_f32(const float* grad, int64_t n, double div, double* sumsq_out,
                                   uint32_t* nonfinite_out, void* workspace, void* stream) {
  return grad_sumsq_f32(grad, n, div, sumsq_out, nonfinite_out, workspace, stream, 0);
}

extern "C" int dvla_grad_sum_f32(const float* const* srcs, int n_src, int64_t n, int64_t n_all,
                                 double div, float* out, double* sumsq_out,
                                 uint32_t* nonfinite_out, void* workspace, void* stream) {
  if (n < 0 || n_all < n || !srcs || n_src < 1 || n_src > kMaxSumSrcs || !out || !sumsq_out ||
      !nonfinite_out || !workspace || !(div > 0.0))
    return fail(DVLA_ERR_USAGE, "bad grad_sum_f32 arguments (1 <= n_src <= %d)", kMaxSumSrcs);
  SumSrcs s{};
  for (int k = 0; k < n_src; ++k) {
    if (!srcs[k] || (reinterpret_cast<uintptr_t>(srcs[k]) & 15))
      return fail(DVLA_ERR_USAGE, "grad_sum_f32: source %d null or not 16-byte aligned", k);
    s.p[k] = srcs[k];
  }
  if (reinterpret_cast<uintptr_t>(out) & 15)
    return fail(DVLA_ERR_USAGE, "grad_sum_f32: output not 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nblocks = kNormBlocks;
  const int64_t per = ((n + nblocks - 1) / nblocks + 3) & ~int64_t{3};
  double* partial = static_cast<double*>(workspace);
  DVLA_CUDA_TRY(cudaMemsetAsync(partial, 0, nblocks * sizeof(double), st));
  if (n_all > 0) {
    const int used = n > 0 ? static_cast<int>((n + per - 1) / per) : 1;
    auto launch = [&](auto kern) {
      kern<<<used, kNormThreads, 0, st>>>(s, n_src, n, n_all, per, div, out, partial,
                                          reinterpret_cast<unsigned*>(nonfinite_out));
    };
    switch (n_src) {
      case 2: launch(sum_sumsq_blocks_f32_kernel<2>); break;
      case 3: launch(sum_sumsq_blocks_f32_kernel<3>); break;
      case 4: launch(sum_sumsq_blocks_f32_kernel<4>); break;
      case 8: launch(sum_sumsq_blocks_f32_kernel<8>); break;
      default: launch(sum_sumsq_blocks_f32_kernel<0>); break;
    }
    if (int rc = launch_check("sum_sumsq_blocks_f32_kernel")) return rc;
  }
  norm_finish_kernel<<<1, kFinishThreads, 0, st>>>(partial, nblocks, sumsq_out, 0);
  return launch_check("norm_finish_kernel");
}

extern "C" int dvla_adam_tail_f32(float* params, const float* grad, double* m, double* v,
                                  int64_t n, int64_t step, double lr, double beta1, double beta2,
                                  double eps, double div, const double* norm, double max_norm,
                                  const float* skip, void* bf16_out, uint32_t* nonfinite_out,
                                  void* stream) {
  if (n < 0 || step < 1 || !(div > 0.0))
    return fail(DVLA_ERR_USAGE, "adam_tail: n >= 0, step >= 1 and div > 0 required");
  if (n == 0) return DVLA_OK;
  const double b1p = pow(beta1, static_cast<double>(step));
  const double b2p = pow(beta2, static_cast<double>(step));
  TailArgs a{params, grad, m, v, n,
             AdamConsts{beta1, 1.0 - beta1, beta2, 1.0 - beta2, 1.0 - b1p, 1.0 - b2p, lr, eps,
                        1.0 / (1.0 - b1p), 1.0 / (1.0 - b2p)},
             div, 1.0 / div, norm, max_norm, skip, static_cast<__nv_bfloat16*>(bf16_out),
             reinterpret_cast<unsigned*>(nonfinite_out)};
  const int vec = ((reinterpret_cast<uintptr_t>(params) & 7) == 0 &&
                   (reinterpret_cast<uintptr_t>(grad) & 7) == 0 &&
                   (reinterpret_cast<uintptr_t>(m) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(v) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(bf16_out) & 3) == 0) ? 1 : 0;
  adam_tail_kernel<false><<<grid_n(vec ? (n + 1) / 2 : n), 256, 0,
                             static_cast<cudaStream_t>(stream)>>>(a, vec, Bf16Peers{});
  return launch_check("adam_tail_kernel");
}

extern "C" int dvla_adam_tail_f32_bcast(float* params, const float* grad, double* m, double* v,
                                        int64_t n, int64_t step, double lr, double beta1,
                                        double beta2, double eps, double div, const double* norm,
                                        double max_norm, const float* skip, void* bf16_out,
                                        void* const* bf16_peers, int n_peers,
                                        uint32_t* nonfinite_out, void* stream) {
  if (n < 0 || step < 1 || !(div > 0.0) || !bf16_out || n_peers < 0 ||
      n_peers > kMaxBf16Peers || (n_peers > 0 && !bf16_peers))
    return fail(DVLA_ERR_USAGE, "adam_tail_bcast: bad arguments (n_peers <= %d)", kMaxBf16Peers);
  if (n == 0) return DVLA_OK;
  Bf16Peers peers{};
  peers.n = n_peers;
  for (int q = 0; q < n_peers; ++q) {
    if (!bf16_peers[q] || (reinterpret_cast<uintptr_t>(bf16_peers[q]) & 3) !=
                              (reinterpret_cast<uintptr_t>(bf16_out) & 3))
      return fail(DVLA_ERR_USAGE, "adam_tail_bcast: peer %d copy null or misaligned", q);
    peers.p[q] = static_cast<__nv_bfloat16*>(bf16_peers[q]);
  }
  const double b1p = pow(beta1, static_cast<double>(step));
  const double b2p = pow(beta2, static_cast<double>(step));
  TailArgs a{params, grad, m, v, n,
             AdamConsts{beta1, 1.0 - beta1, beta2, 1.0 - beta2, 1.0 - b1p, 1.0 - b2p, lr, eps,
                        1.0 / (1.0 - b1p), 1.0 / (1.0 - b2p)},
             div, 1.0 / div, norm, max_norm, skip, static_cast<__nv_bfloat16*>(bf16_out),
             reinterpret_cast<unsigned*>(nonfinite_out)};
  const int vec = ((reinterpret_cast<uintptr_t>(params) & 7) == 0 &&
                   (reinterpret_cast<uintptr_t>(grad) & 7) == 0 &&
                   (reinterpret_cast<uintptr_t>(m) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(v) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(bf16_out) & 3) == 0) ? 1 : 0;
  adam_tail_kernel<true><<<grid_n(vec ? (n + 1) / 2 : n), 256, 0,
                            static_cast<cudaStream_t>(stream)>>>(a, vec, peers);
  return launch_check("adam_tail_kernel");
}

extern "C" int dvla_loss_status(const double* stats, float* skip_out, void* stream) {
  if (!stats || !skip_out) return fail(DVLA_ERR_USAGE, "bad loss_status arguments");
  loss_status_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(stats, skip_out);
  return launch_check("loss_status_kernel");
}
