/*
 * dvla_b200.h -- C-ABI of libdvla_b200.so, the B200 (sm_100a) hot path of
 * D-VLA's per-iteration data plane.
 *
 * This header is the drop-in boundary.  It replaces the reference's kernel
 * seam `dvla.kernels` (reference pkg/src/dvla/kernels/__init__.py:45-51, a
 * module-level function table bound once at import) plus the learner
 * epilogue (grpo.py:89-294), the dual-pool arena (pools.py:72-212) and the
 * weight-replication path (core.py:101-129, planes.py:101-128/244-321,
 * wire.py:144-163/227-237).
 *
 * Conventions (mirroring the reference seam):
 *  - plain pointers and sizes only; no torch types.  "device" pointers are
 *    CUDA device (or NVLink peer-mapped) addresses; "host" pointers are CPU.
 *  - the caller allocates every output, accumulator and workspace; kernels
 *    never retain pointers after the call returns (stream-ordered).
 *  - every entry point returns an int status (DVLA_OK = 0); on failure
 *    dvla_last_error() returns a thread-local message.  Status codes map
 *    1:1 onto the reference's exception types (see dvla_status).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - the library holds no global mutable state besides a per-device SM
 *    count cache and kernel attribute flags; calls are thread-safe across
 *    distinct streams (the reference's nogil lane concurrency,
 *    numba_backend.py:1-5).
 */
#ifndef DVLA_B200_H
#define DVLA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ----------------------------------------------------------- status codes */
enum dvla_status {
  DVLA_OK = 0,
  DVLA_ERR_USAGE = 1,         /* dvla.core.UsageError                       */
  DVLA_ERR_CONFIG = 2,        /* dvla.core.ConfigError                      */
  DVLA_ERR_GRPO_ABORT = 3,    /* dvla.grpo.GrpoAbort                        */
  DVLA_ERR_ALLOC_FAILURE = 4, /* dvla.pools.AllocFailure                    */
  DVLA_ERR_POOL_USAGE = 5,    /* dvla.pools.PoolUsageError                  */
  DVLA_ERR_CUDA = 6,          /* CUDA runtime failure (no reference analogue) */
  DVLA_ERR_DECODE = 7,        /* dvla.wire.DecodeError                      */
  DVLA_ERR_TIMEOUT = 8        /* replication/flag wait timed out            */
};

enum dvla_dtype { DVLA_F32 = 0, DVLA_BF16 = 1, DVLA_U8 = 2, DVLA_F64 = 3 };

/* f64 stats vector written by the GRPO loss entry points (device memory) */
enum dvla_stat_index {
  DVLA_ST_LOSS = 0,        /* total_loss, summed in canonical entry order  */
  DVLA_ST_RATIO_SUM = 1,   /* sum of rho (mean_ratio = sum / chunk_count)  */
  DVLA_ST_CLIP_COUNT = 2,  /* chunks with d_drho == 0.0 (grpo.py:272-273)  */
  DVLA_ST_CHUNK_COUNT = 3,
  DVLA_ST_ABORT = 4,       /* 0 none, 1 non-finite reward, 2 non-finite
                              log-prob, 3 non-finite importance ratio,
                              4 non-finite loss or gradient (grpo.py:237-283) */
  DVLA_ST_ABORT_GROUP = 5, /* group_id the reference's GrpoAbort carries    */
  DVLA_ST_KERNEL_ERR = 6,  /* bit 0: token id out of range, bit 1: timeout  */
  DVLA_ST_RESERVED = 7,
  DVLA_ST_LEN = 8
};

/* flags for dvla_token_loss_fwd_bwd */
#define DVLA_TL_WRITE_DLOGITS 1 /* write d loss / d logits                  */
#define DVLA_TL_UNFUSED 2       /* force the 3-pass (re-read) kernels        */

const char* dvla_last_error(void);
int dvla_abi_version(void);

/* Profiling hooks (no reference analogue; used by bench.py): when enabled
 * on the calling thread, entry points record a CUDA event pair around their
 * dominant kernel on the launch stream; collect synchronises on them and
 * returns the summed device time and the number of launches timed. */
int dvla_profile_enable(int on);
int dvla_profile_collect(double* total_ms, int64_t* count);

/* ------------------------------------------------------- learner (GRPO) */

/* compute_advantages (reference grpo.py:89-99), bit-exact incl. numpy's
 * pairwise mean order.  rewards/out: device f64 [n_groups*G]. */
int dvla_advantages(const double* rewards, int64_t n_groups, int64_t G, double delta,
                    double* out, void* stream);

/* group_advantages over f32 rewards as GroupBatch stores them (grpo.py:102-108
 * + the finiteness check of grpo.py:237); reward_bad[g] = any non-finite. */
int dvla_group_advantages(const float* rewards, int64_t n_groups, int64_t G, double delta,
                          double* adv, uint32_t* reward_bad, void* stream);

/* Workspace bytes for dvla_token_loss_fwd_bwd. */
size_t dvla_token_loss_workspace_bytes(int64_t n_groups, int64_t G, int64_t C, int64_t T);

/* Fused action-token GRPO loss forward + backward (the north-star kernel).
 * Replaces, for the token head, the chain grpo.grpo_grad (grpo.py:217-294)
 * -> policy.log_prob_of (policy.py:161-172) -> kernels.chunk_log_prob
 * (numba_backend.py:49-61) -> policy.backward_batch (policy.py:196-205).
 *   logits   device [n_groups*G*C*T, V] (dtype DVLA_F32 or DVLA_BF16),
 *            row r = ((g*G + i)*C + c)*T + t in INPUT group order g
 *   tokens   device i32 [rows]       target action-token ids
 *   blp      device f32 [n_groups*G*C] behaviour log-probs (sampler stores f32)
 *   rewards  device f32 [n_groups*G]
 *   group_order device i64 [n_groups]: canonical (sorted by group_id) order;
 *            NULL = identity.  group_ids device i64 [n_groups] (NULL = index).
 *   dlogits  device, same dtype/shape as logits (if DVLA_TL_WRITE_DLOGITS)
 *   lp_chunk device f64 [n_groups*G*C] chunk-joint log-probs (input order)
 *   stats    device f64 [DVLA_ST_LEN]
 * Aborts (non-finite reward / log-prob / ratio / loss) are reported in
 * stats[DVLA_ST_ABORT], not as a return status (they are data-dependent and
 * detected on the device). */
int dvla_token_loss_fwd_bwd(const void* logits, int dtype, const int32_t* tokens,
                            const float* blp, const float* rewards, const int64_t* group_order,
                            const int64_t* group_ids, int64_t n_groups, int64_t G, int64_t C,
                            int64_t T, int64_t V, double clip_eps, double adv_eps,
                            double kl_coeff, int flags, void* dlogits, double* lp_chunk,
                            double* stats, void* workspace, size_t workspace_bytes,
                            void* stream);

/* GRPO epilogue on precomputed chunk log-probs (any head): rho, clipped
 * surrogate, coefficient, loss and stats in canonical order (grpo.py:246-293).
 * blp64 (f64) overrides blp (f32) when non-NULL.  coeff_out may be NULL. */
int dvla_grpo_epilogue(const double* lp_chunk, const float* blp, const double* blp64,
                       const double* adv, const uint32_t* reward_bad,
                       const int64_t* group_order, const int64_t* group_ids, int64_t n_groups,
                       int64_t G, int64_t C, double clip_eps, double kl_coeff,
                       double* coeff_out, double* stats, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DVLA_B200_H */
