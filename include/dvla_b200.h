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
 *  - the library's global mutable state: a per-device SM count cache,
 *    kernel attribute flags, the profiling hooks (dvla_profile_*), and the
 *    flag buffers + epoch counter of the single-process dvla_replicate
 *    (guarded by a mutex held for the whole call); everything else is
 *    per call or per handle.  Calls are thread-safe across distinct
 *    streams (the reference's nogil lane concurrency, numba_backend.py:1-5).
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

/* Byte offsets inside that workspace of what the last dvla_token_loss_fwd_bwd
 * left there: offsets[0] adv f64 [n_groups*G] (input group order),
 * offsets[1] lp_tok f64 [rows] (x[r, tok_r] - lse_r), offsets[2] lse f64
 * [rows] (forward-only / unfused paths), offsets[3] coeff f64 [n_groups*G*C]
 * (d loss / d lp_chunk, the weight w included).  For parity checks. */
int dvla_token_loss_workspace_layout(int64_t n_groups, int64_t G, int64_t C, int64_t T,
                                     size_t* offsets);

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
 * detected on the device).
 * Kernel choice: 16-byte-aligned rows with T <= 128 take the persistent
 * fused kernel (one CTA per SM whose CTAs exchange chunk log-probs: do not
 * run two such launches concurrently on one GPU; a wait that exceeds 4 s is
 * reported through stats[DVLA_ST_KERNEL_ERR] bit 1 instead of hanging);
 * otherwise the unfused row/chunk/backward kernels.  flags DVLA_TL_UNFUSED
 * forces the latter.  Workspace: dvla_token_loss_workspace_bytes. */
int dvla_token_loss_fwd_bwd(const void* logits, int dtype, const int32_t* tokens,
                            const float* blp, const float* rewards, const int64_t* group_order,
                            const int64_t* group_ids, int64_t n_groups, int64_t G, int64_t C,
                            int64_t T, int64_t V, double clip_eps, double adv_eps,
                            double kl_coeff, int flags, void* dlogits, double* lp_chunk,
                            double* stats, void* workspace, size_t workspace_bytes,
                            void* stream);

/* Rollout-side action-token sampling (the token-head analogue of
 * policy.sample_chunk_batch, policy.py:150-158): per row r of logits [R, V]
 * draw tokens[r] ~ softmax(x_r) with Philox4x32-10 keyed by (seed, offset, r)
 * (a pure function of those, never of scheduling), lp_tok[r] = x_r[token] -
 * logsumexp(x_r) (f64, may be NULL), and per chunk of T rows the behaviour
 * log-prob blp (f32, as the sampler stores it, runtime.py:698) and/or the
 * f64 chunk log-prob (numpy pairwise order).  One pass over the logits. */
int dvla_token_sample(const void* logits, int dtype, int64_t R, int64_t V, int64_t T,
                      uint64_t seed, uint64_t offset, int32_t* tokens, double* lp_tok,
                      float* blp, double* lp_chunk, void* stream);

/* GRPO epilogue on precomputed chunk log-probs (any head): rho, clipped
 * surrogate, coefficient, loss and stats in canonical order (grpo.py:246-293).
 * blp64 (f64) overrides blp (f32) when non-NULL.  coeff_out may be NULL. */
int dvla_grpo_epilogue(const double* lp_chunk, const float* blp, const double* blp64,
                       const double* adv, const uint32_t* reward_bad,
                       const int64_t* group_order, const int64_t* group_ids, int64_t n_groups,
                       int64_t G, int64_t C, double clip_eps, double kl_coeff,
                       double* coeff_out, double* stats, void* stream);

/* ------------------------------------- Gaussian head + reference policy */

/* kernels.mlp_forward (numba_backend.py:27-46): tanh MLP means, f64
 * accumulate, f32 out.  w1 [H,O], b1 [H], w2 [D,H], b2 [D], obs [B,O]. */
int dvla_mlp_forward(const float* w1, const float* b1, const float* w2, const float* b2,
                     const float* obs, int64_t B, int obs_dim, int hidden, int out_dim,
                     float* out, void* stream);
/* kernels.chunk_log_prob (numba_backend.py:49-61): joint diagonal-Gaussian
 * log-density per row, f64.  means/actions [B,D] f32, log_std [D] f32. */
int dvla_chunk_log_prob(const float* means, const float* log_std, const float* actions,
                        int64_t B, int D, double* out, void* stream);
size_t dvla_policy_backward_workspace_bytes(int64_t B, int hidden, int out_dim);
/* kernels.policy_backward (numba_backend.py:64-113): out[n_params] +=
 * sum_b coeffs[b] * d lp_b / d params, canonical flat order
 * [W1, b1, W2, b2, log_std]; deterministic row order. */
int dvla_policy_backward(const float* w1, const float* b1, const float* w2, const float* b2,
                         const float* log_std, const float* obs, const float* actions,
                         const double* coeffs, int64_t B, int obs_dim, int hidden, int out_dim,
                         double* out, void* workspace, void* stream);
/* Head-only Gaussian backward for large action experts (config 3):
 * dmeans[B,D] = c_b eps e^{-s} (f32, may be NULL); dlog_std[D] += sum_b
 * c_b (eps^2 - 1) (f64, may be NULL). */
int dvla_gauss_head_backward(const float* means, const float* log_std, const float* actions,
                             const double* coeffs, int64_t B, int D, float* dmeans,
                             double* dlog_std, void* stream);

/* The whole Gaussian-head GRPO step in one call (grpo_grad, grpo.py:217-294,
 * for an action expert whose means come from the caller's model, BASELINE
 * config 3): group advantages (grpo.py:89-108) -> chunk_log_prob
 * (numba_backend.py:49-61) -> canonical-order epilogue (grpo.py:242-276,
 * stats as dvla_token_loss_fwd_bwd) -> head backward.  Rows are
 * (group, trajectory, chunk) in input group order, B = n_groups*G*C.
 * lp_chunk [B] f64 out; dmeans [B,D] f32 out (may be NULL); dlog_std [D] f64
 * accumulates += (may be NULL).  Workspace: dvla_gauss_loss_workspace_bytes. */
size_t dvla_gauss_loss_workspace_bytes(int64_t n_groups, int64_t G, int64_t C);
int dvla_gauss_loss_fwd_bwd(const float* means, const float* log_std, const float* actions,
                            const float* blp, const float* rewards, const int64_t* group_order,
                            const int64_t* group_ids, int64_t n_groups, int64_t G, int64_t C,
                            int D, double clip_eps, double adv_eps, double kl_coeff,
                            float* dmeans, double* dlog_std, double* lp_chunk, double* stats,
                            void* workspace, size_t workspace_bytes, void* stream);

/* ----------------------------------------------------- optimizer tail */

/* adam_step (grpo.py:137-150) in place: f32 params, f64 grad/m/v; step is the
 * new step count (>= 1).  Bit-identical to the reference's numpy arithmetic. */
int dvla_adam_step(float* params, const double* grad, double* m, double* v, int64_t n,
                   int64_t step, double lr, double beta1, double beta2, double eps,
                   void* stream);
size_t dvla_grad_norm_workspace_bytes(int64_t n);
/* clip_grad_norm (grpo.py:297-301): *norm_out = ||grad||; scales in place if
 * max_norm > 0 and norm > max_norm; *nonfinite_out |= any non-finite. */
int dvla_grad_norm(double* grad, int64_t n, double max_norm, double* norm_out,
                   uint32_t* nonfinite_out, void* workspace, void* stream);
/* *flag_out |= any non-finite f32 (runtime.py:793-795 RunAbort check). */
int dvla_f32_nonfinite(const float* p, int64_t n, uint32_t* flag_out, void* stream);

/* The learner tail of TrainerWorker.update (runtime.py:788-796) for an f32
 * gradient (the head GEMM's output; all-reduced as the reference's f32
 * frames, runtime.py:590):
 *   dvla_grad_norm_f32: *norm_out = || f64(grad) / div || (div = nodes, the
 *     cross-node mean of runtime.py:627; 1 for one node), *nonfinite_out |=
 *     any non-finite gradient element;
 *   dvla_adam_tail_f32: per element gi = f64(grad[i]) / div, times
 *     max_norm / *norm when *norm > max_norm > 0 (clip_grad_norm,
 *     grpo.py:297-301; norm may be NULL = no clipping; a non-finite *norm
 *     skips the update, grpo.py:282-283), then adam_step's
 *     arithmetic (grpo.py:137-150, bit-identical to dvla_adam_step on the
 *     same f64 gradient).  skip (device f32, may be NULL): nonzero -> the
 *     update is skipped on the device.  bf16_out (may be NULL): the new
 *     parameters rounded to bf16.  nonfinite_out (may be NULL) |= any
 *     non-finite new parameter (runtime.py:793-795).
 *   dvla_loss_status: *skip_out = 1.0f if the fused loss's stats vector
 *     records an abort, a non-finite loss or a kernel error, else 0.0f (the
 *     skip word). */
int dvla_grad_norm_f32(const float* grad, int64_t n, double div, double* norm_out,
                       uint32_t* nonfinite_out, void* workspace, void* stream);
/* The sum of squares instead of its root (a shard's share of the global
 * norm: the shards' sums are all-reduced, then the root taken). */
int dvla_grad_sumsq_f32(const float* grad, int64_t n, double div, double* sumsq_out,
                        uint32_t* nonfinite_out, void* workspace, void* stream);
/* The peer gradient exchange's reduce-scatter epilogue (runtime.py:618-627:
 * the nodes' f32 frames summed in f64 in node order): out[i] = f32(sum over
 * k < n_src, in order, of f64(srcs[k][i])) for i < n_all, and in the same
 * pass what dvla_grad_sumsq_f32(out, n, div, ...) returns for the first n
 * (bit-identical; [n, n_all) carries side words such as the skip flags).
 * srcs: a HOST array of n_src (1..16) device pointers, each and out 16-byte
 * aligned; workspace as dvla_grad_norm_workspace_bytes(n). */
int dvla_grad_sum_f32(const float* const* srcs, int n_src, int64_t n, int64_t n_all, double div,
                      float* out, double* sumsq_out, uint32_t* nonfinite_out, void* workspace,
                      void* stream);
int dvla_adam_tail_f32(float* params, const float* grad, double* m, double* v, int64_t n,
                       int64_t step, double lr, double beta1, double beta2, double eps,
                       double div, const double* norm, double max_norm, const float* skip,
                       void* bf16_out, uint32_t* nonfinite_out, void* stream);
/* dvla_adam_tail_f32 whose bf16 copy is also stored into n_peers (<= 31)
 * other learners' working copies (device pointers mapped here, e.g. CUDA
 * IPC, at the same element offset): the ZeRO-1 all-gather fused into the
 * optimizer tail over NVLink.  The stores are fenced system-wide before
 * the kernel completes; signal the peers after it (stream order). */
int dvla_adam_tail_f32_bcast(float* params, const float* grad, double* m, double* v, int64_t n,
                             int64_t step, double lr, double beta1, double beta2, double eps,
                             double div, const double* norm, double max_norm, const float* skip,
                             void* bf16_out, void* const* bf16_peers, int n_peers,
                             uint32_t* nonfinite_out, void* stream);
int dvla_loss_status(const double* stats, float* skip_out, void* stream);

/* --------------------------------------------------- dual-pool arena */

/* PoolKind (pools.py:23-26) */
enum dvla_pool_kind {
  DVLA_POOL_MODEL_COMPUTE = 0, /* long-lived: params, grads, optimizer, replicas */
  DVLA_POOL_ENV_AUX = 1,       /* epoch-scoped: rollout staging, activations/KV */
  DVLA_POOL_UNIFIED_BASELINE = 2
};

/* Opaque arena: host-side first-fit bookkeeping over a device slab
 * (Pool, pools.py:72-212).  Offsets are bit-identical to the reference. */
typedef struct dvla_arena dvla_arena;

int dvla_arena_create(int kind, int64_t capacity, dvla_arena** out, int64_t* pool_id_out);
int dvla_arena_destroy(dvla_arena* arena);
/* Pool.alloc (pools.py:92-128); DVLA_ERR_ALLOC_FAILURE when nothing fits. */
int dvla_arena_alloc(dvla_arena* arena, int64_t size, int64_t align, int64_t* offset_out,
                     int64_t* serial_out, int64_t* generation_out);
/* Pool.free (pools.py:130-141); DVLA_ERR_POOL_USAGE for foreign, stale or
 * double-freed handles (messages as the reference). */
int dvla_arena_free(dvla_arena* arena, int64_t pool_id, int64_t offset, int64_t size,
                    int64_t generation, int64_t serial);
/* Pool.epoch_reset (pools.py:160-170): ENV_AUX only. */
int dvla_arena_epoch_reset(dvla_arena* arena);
int dvla_arena_is_live(dvla_arena* arena, int64_t generation, int64_t serial, int* out);
/* out[9] = live_bytes, total_free, largest_free, failed_allocs, alloc_count,
 * free_count, churn_bytes, generation, n_free_extents (Pool.stats). */
int dvla_arena_stats(dvla_arena* arena, int64_t* out);
/* kernels.alloc_trace_run (numba_backend.py:139-247), host memory in/out;
 * final_out[3] = (total_free, largest_free, n_extents). */
/* torch's caching allocator on an ENV_AUX arena (torch
 * temporaries in the recycled pool).  dvla_torch_pool_bind(device, arena,
 * slab_base) routes every segment a torch.cuda.MemPool built on
 * dvla_torch_alloc / dvla_torch_free (the CUDAPluggableAllocator signatures;
 * stream is a cudaStream_t) requests on `device` into the arena's slab
 * (first fit, 512-byte aligned); arena = NULL unbinds (refused while torch
 * segments are live).  A bound arena refuses epoch_reset.  alloc returns
 * NULL when the arena cannot place the segment (torch raises OOM). */
int dvla_torch_pool_bind(int device, dvla_arena* arena, void* slab_base);
void* dvla_torch_alloc(size_t size, int device, void* stream);
void dvla_torch_free(void* ptr, size_t size, int device, void* stream);
int dvla_arena_trace(int64_t capacity, int64_t n, const uint8_t* is_alloc, const int64_t* size,
                     const int64_t* align, const uint64_t* pick, uint8_t* out_ok,
                     int64_t* out_off, int64_t* final_out);

/* -------------------------------------------------- weight replication */

/* Device slabs (cudaMalloc, so they can be shared over CUDA IPC); backing
 * store of the dual-pool allocator's regions. */
int dvla_dev_alloc(int device, size_t bytes, void** out);
int dvla_dev_free(void* ptr);

/* CUDA IPC for cross-process NVLink mappings of a peer's replica region
 * (handle: 64 bytes).  The mapping is the B200 analogue of the reference
 * Transport's WIRE link (planes.py:101-128): a peer pointer instead of a
 * byte stream. */
int dvla_ipc_handle(void* dev_ptr, uint8_t* handle_out);
int dvla_ipc_open(const uint8_t* handle, void** out);
int dvla_ipc_close(void* ptr);
int dvla_enable_peer_access(int device, int peer);

/* One hop of a replication chain: copy nbytes from src to dst (dst may be a
 * peer mapping; NULL = wait only).  Chunk c is read only after
 * wait_flags[c] >= epoch (NULL = source is ready) and signal_flags[c] is set
 * to epoch (release, system scope) once chunk c has landed in dst. */
typedef struct dvla_hop {
  const void* src;
  void* dst;
  const uint32_t* wait_flags;
  uint32_t* signal_flags;
} dvla_hop;

/* Chunked, pipelined chain broadcast (ControlPlane.broadcast, planes.py:294-321,
 * without serialisation): TMA bulk copies HBM -> SMEM -> (peer) HBM, every
 * receiver forwarding each chunk as soon as it landed.  All hops of one call
 * run concurrently in one launch (ctas_per_hop CTAs each).  nbytes and
 * chunk_bytes must be multiples of 16; pointers 16-byte aligned.  A flag wait
 * longer than timeout_ns sets *err_dev (device u32) instead of hanging. */
int dvla_replicate_chain(const dvla_hop* hops, int n_hops, int64_t nbytes, int64_t chunk_bytes,
                         uint32_t epoch, int ctas_per_hop, uint64_t timeout_ns,
                         uint32_t* err_dev, void* stream);

/* snapshot_from_params on the device (core.py:120-129): copy nbytes from src
 * to dst and write the first non-finite element index (dtype DVLA_F32 /
 * DVLA_BF16 / DVLA_F64; DVLA_U8 = no check) to *bad_index_dev (device u64;
 * UINT64_MAX when all finite). */
int dvla_snapshot_copy(const void* src, void* dst, int64_t nbytes, int dtype,
                       uint64_t* bad_index_dev, void* stream);

/* Bitwise compare (messages_equal on parameter bytes, wire.py:279-281):
 * out_dev[0] = number of differing 16-byte words, out_dev[1] = first
 * differing byte offset (UINT64_MAX if equal). */
/* Order-independent checksum of a region (a replica checked against its
 * source on another GPU): out_dev[0] = sum of its 8-byte little-endian words,
 * out_dev[1] = sum of word_i * (2 i + 1), both mod 2^64 (a trailing partial
 * word zero-padded).  8-byte aligned; one read; asynchronous on `stream`. */
int dvla_checksum64(const void* p, int64_t nbytes, uint64_t* out_dev, void* stream);
/* The same terms for a sub-range that starts at 8-byte word `first_word` of
 * a larger region (index weights 2 (first_word + i) + 1): the checksums of
 * consecutive sub-ranges add up (mod 2^64) to the whole region's. */
int dvla_checksum64_at(const void* p, int64_t nbytes, int64_t first_word, uint64_t* out_dev,
                       void* stream);
int dvla_bytes_equal(const void* a, const void* b, int64_t nbytes, uint64_t* out_dev,
                     void* stream);

/* Copy-engine copy (cudaMemcpyAsync, UVA): the baseline replication path
 * the TMA chain is measured against. */
int dvla_memcpy_async(void* dst, const void* src, int64_t nbytes, void* stream);

/* One process driving several GPUs (ControlPlane.broadcast over NVLink,
 * planes.py:294-321): replicate nbytes (multiple of 16) of `src` on src_dev
 * into dst_ptrs[i] on dst_devs[i].  mode 0: chain (each hop's TMA kernel
 * runs on its source device, per-chunk flags in library-owned buffers);
 * mode 1: copy-engine fan-out from the source.  streams: n_dst + 1 entries
 * (source first) or NULL for each device's default stream.  Asynchronous;
 * dvla_replicate_status reports (and clears) chain timeouts. */
int dvla_replicate(int src_dev, const void* src, int n_dst, const int* dst_devs,
                   void* const* dst_ptrs, int64_t nbytes, int64_t chunk_bytes, int mode,
                   void* const* streams);
int dvla_replicate_status(int* timed_out);

/* Copy-engine variant of one chain hop (same flags and epochs as
 * dvla_replicate_chain): stream-wait wait_flags[c] >= epoch, copy chunk c
 * with cudaMemcpyAsync into dst, stream-write signal_flags[c] = epoch.
 * Any of src/dst, wait_flags, signal_flags may be null (root: no wait; last
 * receiver: wait only). */
int dvla_replicate_hop_ce(const void* src, void* dst, const uint32_t* wait_flags,
                          uint32_t* signal_flags, int64_t nbytes, int64_t chunk_bytes,
                          uint32_t epoch, void* stream);
/* NCCL for a process that drives several GPUs itself (GradReducer.reduce,
 * runtime.py:569-637, without torch.distributed; libnccl.so.2 is opened at
 * run time): dvla_nccl_init builds one communicator per device in `devs`
 * (index = position); dvla_nccl_allreduce_sum sums `count` elements of
 * dtype DVLA_F32 / DVLA_F64 / DVLA_BF16 in place on communicator comm_idx.
 * One thread issuing for several devices brackets the calls with
 * dvla_nccl_group_start / dvla_nccl_group_end. */
int dvla_nccl_init(int n, const int* devs);
int dvla_nccl_group_start(void);
int dvla_nccl_group_end(void);
int dvla_nccl_allreduce_sum(int comm_idx, void* ptr, int64_t count, int dtype, void* stream);
int dvla_nccl_destroy(void);

/* Stream memory operations used by the hop (cuStreamWaitValue32 GEQ /
 * cuStreamWriteValue32 with a memory barrier). */
int dvla_stream_wait_u32(const uint32_t* addr, uint32_t value, void* stream);
int dvla_stream_write_u32(uint32_t* addr, uint32_t value, void* stream);
/* Stream-ordered wait until flags[i] >= target for every bit i set in mask
 * (i < 32), acquire-polled by one warp; after timeout_ns *err_dev |= 1 and
 * the stream goes on (the peer exchange's bounded waits: a dead peer is an
 * error the host reads after its sync, not a hung stream). */
int dvla_wait_flags_u32(const uint32_t* flags, uint32_t mask, uint32_t target,
                        uint64_t timeout_ns, uint32_t* err_dev, void* stream);
/* k (1..4) scalars reduced across the n (<= 32) ranks of a peer exchange
 * through IPC-mapped peer memory, in rank order, identical on every rank:
 * kind 0 = f64 sum, kind 1 = u32 max.  This rank's values (`local`, device)
 * go to slot [rank] of every peer's slot array (peer_slots[p], [n][k]
 * values, mapped here) and the epoch to peer_flags[p][rank]; the local
 * flags my_flags[p] (written by peer p) are acquire-polled, bounded by
 * timeout_ns (then *err_dev |= 1); out[0, k) = the reduction.  One warp,
 * stream-ordered; epochs increase by one per call. */
int dvla_peer_reduce(int kind, const void* local, int k, void* const* peer_slots,
                     uint32_t* const* peer_flags, int rank, int n, const void* my_slots,
                     const uint32_t* my_flags, uint32_t epoch, uint64_t timeout_ns,
                     uint32_t* err_dev, void* out, void* stream);

/* ---- switch-multicast (NVLS) replication ---------------------------------
 * Replaces the same ControlPlane.broadcast -> WeightMailbox.deliver data path
 * (planes.py:294-321, 244-275) as dvla_replicate_chain: the source writes each
 * byte once into a multicast address and the NVSwitch replicates it into the
 * bound region of every member GPU.  One process per GPU; the multicast
 * object is created on the source and shared as a POSIX fd (pidfd_getfd).
 * Sequence: root dvla_mc_create; others dvla_mc_import; all
 * dvla_mc_add_device; (barrier) all dvla_mc_bind; (barrier) writers
 * dvla_mc_map.  Objects are opaque (void*). */
int dvla_mc_supported(int device, int* out);
int dvla_mc_create(int n_devices, size_t nbytes, int* fd_out, size_t* size_out, void** obj_out);
int dvla_mc_import(int owner_pid, int owner_fd, int n_devices, size_t size, void** obj_out);
int dvla_mc_add_device(void* obj, int device);
int dvla_mc_bind(void* obj, int device, void** local_out);
int dvla_mc_map(void* obj, int device, void** mc_out);
int dvla_mc_destroy(void* obj);
/* Root: copy nbytes (multiple of 16) from src into the multicast region,
 * then release-store `epoch` into every member's flag word (mc_flag is the
 * flag's multicast address).  done_ctr: device u32, zero-initialised, owned
 * by the caller (reset by the kernel). */
int dvla_mc_broadcast(const void* src, void* mc_dst, int64_t nbytes, void* mc_flag,
                      uint32_t epoch, int ctas, uint32_t* done_ctr, void* stream);
/* Switch-reduced all-reduce of n f32 (n % 4 == 0) held in every member's
 * bound region of one multicast object (GradReducer.reduce, runtime.py:
 * 569-637): rank r reduces its 1/world slice with multimem.ld_reduce.add and
 * stores the sum (times `scale`) to all members with multimem.st; entry and
 * exit barriers use two u32 counters (local view / multicast view, zeroed
 * once) with epoch = 1, 2, ... per call.  done_ctr: device u32, zeroed. */
int dvla_mc_allreduce_f32(void* mc_buf, int64_t n, int rank, int world,
                          const uint32_t* local_flags, void* mc_flags, uint32_t epoch,
                          float scale, int ctas, uint32_t* done_ctr, uint64_t timeout_ns,
                          uint32_t* err_dev, void* stream);
/* Receivers: stream-ordered wait until the local flag reaches `epoch`;
 * *err_dev |= 1 on timeout (the reference's WeightMailbox wait). */
int dvla_mc_wait(const uint32_t* local_flag, uint32_t epoch, uint64_t timeout_ns,
                 uint32_t* err_dev, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DVLA_B200_H */
