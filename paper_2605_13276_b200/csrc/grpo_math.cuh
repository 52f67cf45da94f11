// GRPO scalar math shared by every loss kernel (token head, Gaussian head).
//
// Bit-exactness contract:
//  * advantages follow reference grpo.py:89-99 (compute_advantages) with
//    numpy's pairwise summation order for mean()/var(); every f64 add/mul/div
//    uses the _rn intrinsics so nvcc can never contract them into FMAs.
//  * the per-chunk surrogate/coefficient follows grpo.py:111-119
//    (clipped_surrogate) and grpo.py:252-268 (weight, coeff, optional KL),
//    evaluated left-to-right exactly as the Python expressions.
#pragma once
#include <stdint.h>

namespace dvla {

// numpy pairwise_sum over n doubles produced by `get(i)` (numpy
// loops_utils.h pairwise_sum: <8 sequential, <=128 eight-way unrolled,
// else split at n/2 rounded down to a multiple of 8).
template <class Get>
__device__ double pairwise_sum(const Get& get, int64_t lo, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, get(lo + i));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = get(lo + j);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], get(lo + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, get(lo + i));
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum(get, lo, n2), pairwise_sum(get, lo + n2, n - n2));
}

// Advantage of every member of one group (reference grpo.py:89-99).
// `r(i)` yields reward i as f64.  Writes G values through `put(i, a)`.
template <class Get, class Put>
__device__ inline void group_advantages(Get r, int64_t G, double delta, Put put) {
  const double n = static_cast<double>(G);
  const double mean = __ddiv_rn(pairwise_sum(r, 0, G), n);
  auto sq = [&](int64_t i) {
    double c = __dsub_rn(r(i), mean);
    return __dmul_rn(c, c);
  };
  const double var = __ddiv_rn(pairwise_sum(sq, 0, G), n);
  if (var == 0.0) {
    for (int64_t i = 0; i < G; ++i) put(i, 0.0);
    return;
  }
  const double den = __dadd_rn(__dsqrt_rn(var), delta);
  for (int64_t i = 0; i < G; ++i) put(i, __ddiv_rn(__dsub_rn(r(i), mean), den));
}

struct ChunkTerms {
  double rho;
  double loss;
  double coeff;
  bool clipped;  // d_drho == 0.0 (reference counts A == 0 chunks too)
};

// One (trajectory, chunk) entry of grpo_grad (grpo.py:252-276).
__device__ inline ChunkTerms chunk_terms(double lp, double blp, double adv, double w,
                                                  double clip_eps, double kl_coeff) {
  ChunkTerms t;
  const double diff = __dsub_rn(lp, blp);
  const double rho = exp(diff);
  const double lo = __dsub_rn(1.0, clip_eps), hi = __dadd_rn(1.0, clip_eps);
  // python: min(max(ratio, lo), hi)
  double cr = (lo > rho) ? lo : rho;
  cr = (cr > hi) ? hi : cr;
  const double unclipped = __dmul_rn(rho, adv);
  const double clipped = __dmul_rn(cr, adv);
  double contrib, d;
  if (unclipped <= clipped) {
    contrib = -unclipped;
    d = -adv;
  } else {
    contrib = -clipped;
    d = 0.0;
  }
  double coeff = __dmul_rn(__dmul_rn(w, d), rho);
  double loss = __dmul_rn(w, contrib);
  if (kl_coeff > 0.0) {
    // loss_term += weight * 0.5 * kl * diff * diff ; coeff += weight * kl * diff
    loss = __dadd_rn(loss, __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(w, 0.5), kl_coeff), diff), diff));
    coeff = __dadd_rn(coeff, __dmul_rn(__dmul_rn(w, kl_coeff), diff));
  }
  t.rho = rho;
  t.loss = loss;
  t.coeff = coeff;
  t.clipped = (d == 0.0);
  return t;
}

}  // namespace dvla
