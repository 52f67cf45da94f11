// Weight replication: learner -> rollout replicas over NVLink (K5/K6).
//
// Replaces the reference's weight control plane data path:
//   TrainerWorker.snapshot -> core.snapshot_from_params (core.py:120-129,
//   deep copy + isfinite), ControlPlane.broadcast (planes.py:294-321) ->
//   Transport.outbound/inbound -> wire weight frame encode/decode
//   (wire.py:144-147, 227-237) -> WeightMailbox.deliver/take_newest.
// On B200 the parameters never leave device memory: a snapshot is a fused
// copy + isfinite into a MODEL_COMPUTE pool region, and a broadcast is a
// chunked, pipelined chain of TMA bulk copies (HBM -> SMEM -> peer HBM over
// NVLink/NVSwitch) in which every receiver forwards each chunk to the next
// receiver as soon as it has landed (per-chunk flags, release/acquire at
// system scope).  Bit-exactness is by construction (byte copies) and is
// checked by dvla_bytes_equal on every bench run.
#include <stdlib.h>

#include <mutex>

#include "common.cuh"
#include "drv.cuh"

namespace dvla {

constexpr int kRepThreads = 32;  // one warp; lane 0 drives the TMA pipeline
constexpr int kRepStages = 4;
constexpr uint32_t kRepPiece = 32 * 1024;  // bytes per TMA bulk copy

struct RepSmem {
  uint64_t full[kRepStages];
};

struct HopDev {
  const uint8_t* src;
  uint8_t* dst;                  // may be an NVLink peer mapping; null = wait only
  const uint32_t* wait_flags;    // local flags to wait on before reading a chunk
  uint32_t* signal_flags;        // flags (often on the peer) to set after a chunk
};

constexpr int kMaxHops = 16;
struct HopTable {
  HopDev h[kMaxHops];
};

__device__ __forceinline__ bool wait_flag_sys(const uint32_t* f, uint32_t epoch, uint64_t timeout,
                                              uint32_t* err) {
  if (ld_acquire_sys(f) >= epoch) return true;
  const uint64_t t0 = globaltimer_ns();
  uint32_t ns = 64;
  while (ld_acquire_sys(f) < epoch) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (globaltimer_ns() - t0 > timeout) {
      atomicOr(err, 1u);
      return false;
    }
  }
  return true;
}

// One CTA group per hop; CTA j of a hop moves chunks j, j + ctas, ...
__global__ void __launch_bounds__(kRepThreads) replicate_chain_kernel(
    HopTable tab, int n_hops, int ctas_per_hop, int64_t nbytes, int64_t chunk_bytes,
    uint32_t epoch, uint64_t timeout_ns, uint32_t* err) {
  extern __shared__ __align__(128) uint8_t dyn[];
  RepSmem& S = *reinterpret_cast<RepSmem*>(dyn);
  uint8_t* stage = dyn + 128;
  const int hop = blockIdx.x / ctas_per_hop;
  const int j = blockIdx.x % ctas_per_hop;
  if (hop >= n_hops) return;
  const HopDev H = tab.h[hop];
  if (threadIdx.x != 0) return;  // pure data movement: one elected thread
  for (int s = 0; s < kRepStages; ++s) mbar_init(&S.full[s], 1);
  fence_mbar_init();
  const int64_t n_chunks = (nbytes + chunk_bytes - 1) / chunk_bytes;
  uint32_t uses[kRepStages] = {};
  for (int64_t c = j; c < n_chunks; c += ctas_per_hop) {
    if (H.wait_flags && !wait_flag_sys(H.wait_flags + c, epoch, timeout_ns, err)) return;
    if (!H.dst) continue;
    const int64_t base = c * chunk_bytes;
    const int64_t len = (nbytes - base < chunk_bytes) ? nbytes - base : chunk_bytes;
    const int64_t npieces = (len + kRepPiece - 1) / kRepPiece;
    fence_proxy_async_global();  // generic acquire above -> async-proxy reads below
    auto piece_len = [&](int64_t i) {
      const int64_t off = i * kRepPiece;
      return static_cast<uint32_t>((len - off < kRepPiece) ? len - off : kRepPiece);
    };
    auto issue_load = [&](int64_t i) {
      const int s = static_cast<int>(i % kRepStages);
      mbar_arrive_expect_tx(&S.full[s], piece_len(i));
      tma_load_1d(stage + s * kRepPiece, H.src + base + i * kRepPiece, piece_len(i), &S.full[s]);
    };
    const int64_t pro = npieces < kRepStages ? npieces : kRepStages;
    for (int64_t i = 0; i < pro; ++i) issue_load(i);
    for (int64_t i = 0; i < npieces; ++i) {
      const int s = static_cast<int>(i % kRepStages);
      mbar_wait(&S.full[s], uses[s] & 1);
      ++uses[s];
      tma_store_1d(H.dst + base + i * kRepPiece, stage + s * kRepPiece, piece_len(i));
      bulk_commit();
      if (i >= 1 && i - 1 + kRepStages < npieces) {
        bulk_wait_read<1>();  // store i-1 has finished reading its stage
        issue_load(i - 1 + kRepStages);
      }
    }
    bulk_wait<0>();  // this chunk's writes are performed (visible at the peer)
    if (H.signal_flags) {
      fence_proxy_async_global();
      __threadfence_system();
      st_release_sys(H.signal_flags + c, epoch);
    }
  }
  bulk_wait<0>();
}

// ------------------------------------------------ snapshot copy + isfinite
constexpr int kSnapThreads = 256;

template <int DT>
__device__ __forceinline__ int first_nonfinite_in16(const uint4& v) {
  if (DT == DVLA_F32) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if ((w[e] & 0x7f800000u) == 0x7f800000u) return e;
  } else if (DT == DVLA_BF16) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t h = (e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xffffu);
      if ((h & 0x7f80u) == 0x7f80u) return e;
    }
  } else if (DT == DVLA_F64) {
    const unsigned long long d0 = (static_cast<unsigned long long>(v.y) << 32) | v.x;
    const unsigned long long d1 = (static_cast<unsigned long long>(v.w) << 32) | v.z;
    if ((d0 & 0x7ff0000000000000ull) == 0x7ff0000000000000ull) return 0;
    if ((d1 & 0x7ff0000000000000ull) == 0x7ff0000000000000ull) return 1;
  }
  return -1;
}

// Grid-stride 16-byte copy with a fused finiteness scan; first bad element
// index via atomicMin.  (HBM-bound: 2 bytes moved per byte snapshotted.)
template <int DT>
__global__ void __launch_bounds__(kSnapThreads) snapshot_kernel(const uint4* __restrict__ src,
                                                                uint4* __restrict__ dst,
                                                                int64_t nvec,
                                                                unsigned long long* bad) {
  constexpr int epv = DT == DVLA_F32 ? 4 : DT == DVLA_BF16 ? 8 : DT == DVLA_F64 ? 2 : 16;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < nvec; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      __stcs(dst + i + u * stride, v[u]);
      if (DT != DVLA_U8) {
        const int e = first_nonfinite_in16<DT>(v[u]);
        if (e >= 0) atomicMin(bad, static_cast<unsigned long long>((i + u * stride) * epv + e));
      }
    }
  }
  for (; i < nvec; i += stride) {
    const uint4 v = __ldcs(src + i);
    __stcs(dst + i, v);
    if (DT != DVLA_U8) {
      const int e = first_nonfinite_in16<DT>(v);
      if (e >= 0) atomicMin(bad, static_cast<unsigned long long>(i * epv + e));
    }
  }
}

__global__ void snapshot_tail_kernel(const uint8_t* src, uint8_t* dst, int64_t from, int64_t n,
                                     int dtype, unsigned long long* bad) {
  const int64_t i = from + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  dst[i] = src[i];
  if (dtype == DVLA_F32 && (i % 4) == 3) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(src + i - 3);
    if ((w & 0x7f800000u) == 0x7f800000u) atomicMin(bad, static_cast<unsigned long long>(i / 4));
  } else if (dtype == DVLA_BF16 && (i % 2) == 1) {
    const uint32_t h = src[i - 1] | (static_cast<uint32_t>(src[i]) << 8);
    if ((h & 0x7f80u) == 0x7f80u) atomicMin(bad, static_cast<unsigned long long>(i / 2));
  }
}

// ------------------------------------------------------------ bytes_equal
__global__ void bytes_equal_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b,
                                   int64_t nvec, unsigned long long* out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  unsigned long long mism = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nvec;
       i += stride) {
    const uint4 x = __ldcs(a + i), y = __ldcs(b + i);
    if (x.x != y.x || x.y != y.y || x.z != y.z || x.w != y.w) {
      ++mism;
      const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
      for (int e = 0; e < 4; ++e)
        if (xs[e] != ys[e]) {
          const uint32_t d = xs[e] ^ ys[e];
          const int byte = (__ffs(static_cast<int>(d)) - 1) >> 3;
          atomicMin(out + 1, static_cast<unsigned long long>(i * 16 + e * 4 + byte));
          break;
        }
    }
  }
  for (int o = 16; o > 0; o >>= 1) mism += __shfl_xor_sync(0xffffffffu, mism, o);
  if ((threadIdx.x & 31) == 0 && mism) atomicAdd(out, mism);
}

// Order-independent 64-bit checksum of a region (verification of a replica
// against its source on another GPU without moving either): over 8-byte
// words w_i, out[0] += w_i and out[1] += w_i * (2 i + 1) mod 2^64 (the
// index weight catches swapped or shifted chunks); a byte tail is folded in
// as one zero-padded word.  One read of the region.
__global__ void checksum64_kernel(const uint2* __restrict__ w, int64_t nwords, int64_t first,
                                  unsigned long long* out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  unsigned long long s0 = 0, s1 = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nwords;
       i += stride) {
    const uint2 x = __ldcs(w + i);
    const unsigned long long v = (static_cast<unsigned long long>(x.y) << 32) | x.x;
    s0 += v;
    s1 += v * static_cast<unsigned long long>(2 * (first + i) + 1);
  }
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, s0);
    atomicAdd(out + 1, s1);
  }
}

__global__ void checksum64_tail_kernel(const uint8_t* p, int64_t from, int64_t n, int64_t first,
                                       unsigned long long* out) {
  unsigned long long v = 0;
  for (int64_t i = from; i < n; ++i) v |= static_cast<unsigned long long>(p[i]) << (8 * (i - from));
  const unsigned long long idx = static_cast<unsigned long long>(first + from / 8);
  atomicAdd(out, v);
  atomicAdd(out + 1, v * (2 * idx + 1));
}

__global__ void bytes_equal_tail_kernel(const uint8_t* a, const uint8_t* b, int64_t from,
                                        int64_t n, unsigned long long* out) {
  const int64_t i = from + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n && a[i] != b[i]) {
    atomicAdd(out, 1ull);
    atomicMin(out + 1, static_cast<unsigned long long>(i));
  }
}

__global__ void init_u64_kernel(unsigned long long* p, unsigned long long v0,
                                unsigned long long v1) {
  p[0] = v0;
  if (v1 != 0) p[1] = v1;
}

static int grid_for(int64_t nvec, int threads) {
  const int sms = num_sms(current_device());
  int64_t g = (nvec + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(sms) * 8;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace dvla

using namespace dvla;

extern "C" int dvla_dev_alloc(int device, size_t bytes, void** out) {
  if (!out) return fail(DVLA_ERR_USAGE, "null out pointer");
  int prev = 0;
  DVLA_CUDA_TRY(cudaGetDevice(&prev));
  DVLA_CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaMalloc(out, bytes ? bytes : 1);
  cudaSetDevice(prev);
  if (e != cudaSuccess)
    return fail(DVLA_ERR_CUDA, "cudaMalloc(%zu) on device %d failed: %s", bytes, device,
                cudaGetErrorString(e));
  return DVLA_OK;
}

extern "C" int dvla_dev_free(void* p) {
  if (p) DVLA_CUDA_TRY(cudaFree(p));
  return DVLA_OK;
}

extern "C" int dvla_ipc_handle(void* dev_ptr, uint8_t* handle_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (!dev_ptr || !handle_out) return fail(DVLA_ERR_USAGE, "null pointer argument");
  cudaIpcMemHandle_t h;
  DVLA_CUDA_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle_out, &h, 64);
  return DVLA_OK;
}

extern "C" int dvla_ipc_open(const uint8_t* handle, void** out) {
  if (!handle || !out) return fail(DVLA_ERR_USAGE, "null pointer argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  DVLA_CUDA_TRY(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  return DVLA_OK;
}

extern "C" int dvla_ipc_close(void* p) {
  if (p) DVLA_CUDA_TRY(cudaIpcCloseMemHandle(p));
  return DVLA_OK;
}

extern "C" int dvla_enable_peer_access(int device, int peer) {
  int prev = 0, can = 0;
  DVLA_CUDA_TRY(cudaGetDevice(&prev));
  DVLA_CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return fail(DVLA_ERR_CUDA, "device %d cannot access peer %d", device, peer);
  DVLA_CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return DVLA_OK;
  }
  if (e != cudaSuccess)
    return fail(DVLA_ERR_CUDA, "enable peer access %d->%d: %s", device, peer,
                cudaGetErrorString(e));
  return DVLA_OK;
}

extern "C" int dvla_replicate_chain(const dvla_hop* hops, int n_hops, int64_t nbytes,
                                    int64_t chunk_bytes, uint32_t epoch, int ctas_per_hop,
                                    uint64_t timeout_ns, uint32_t* err_dev, void* stream) {
  if (n_hops < 1 || n_hops > kMaxHops)
    return fail(DVLA_ERR_USAGE, "n_hops must be in [1, %d], got %d", kMaxHops, n_hops);
  if (nbytes < 0 || chunk_bytes < 16 || (chunk_bytes % 16) != 0 || (nbytes % 16) != 0)
    return fail(DVLA_ERR_USAGE,
                "nbytes must be a multiple of 16 and chunk_bytes a positive multiple of 16");
  if (ctas_per_hop < 1) return fail(DVLA_ERR_USAGE, "ctas_per_hop must be >= 1");
  if (!err_dev) return fail(DVLA_ERR_USAGE, "null err pointer");
  if (epoch == 0) return fail(DVLA_ERR_USAGE, "epoch must be >= 1 (flags start at 0)");
  HopTable tab{};
  for (int i = 0; i < n_hops; ++i) {
    const dvla_hop& h = hops[i];
    if (h.dst && !h.src) return fail(DVLA_ERR_USAGE, "hop %d has a destination but no source", i);
    if ((h.src && reinterpret_cast<uintptr_t>(h.src) % 16) ||
        (h.dst && reinterpret_cast<uintptr_t>(h.dst) % 16))
      return fail(DVLA_ERR_USAGE, "hop %d pointers must be 16-byte aligned", i);
    tab.h[i].src = static_cast<const uint8_t*>(h.src);
    tab.h[i].dst = static_cast<uint8_t*>(h.dst);
    tab.h[i].wait_flags = h.wait_flags;
    tab.h[i].signal_flags = h.signal_flags;
  }
  if (nbytes == 0) return DVLA_OK;
  const size_t smem = 128 + static_cast<size_t>(kRepStages) * kRepPiece;
  static bool attr[64] = {};
  int cur_dev = 0;
  DVLA_CUDA_TRY(cudaGetDevice(&cur_dev));
  if (!attr[cur_dev & 63]) {  // a function attribute is per device
    DVLA_CUDA_TRY(cudaFuncSetAttribute(replicate_chain_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
    attr[cur_dev & 63] = true;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t stop;
  prof_begin(st, &stop);
  replicate_chain_kernel<<<n_hops * ctas_per_hop, kRepThreads, smem, st>>>(
      tab, n_hops, ctas_per_hop, nbytes, chunk_bytes, epoch, timeout_ns, err_dev);
  prof_end(st, stop);
  return launch_check("replicate_chain_kernel");
}

extern "C" int dvla_snapshot_copy(const void* src, void* dst, int64_t nbytes, int dtype,
                                  uint64_t* bad_index_dev, void* stream) {
  if (nbytes < 0) return fail(DVLA_ERR_USAGE, "nbytes must be >= 0");
  if ((!src || !dst || !bad_index_dev) && nbytes > 0)
    return fail(DVLA_ERR_USAGE, "null pointer argument");
  if (dtype != DVLA_F32 && dtype != DVLA_BF16 && dtype != DVLA_U8 && dtype != DVLA_F64)
    return fail(DVLA_ERR_USAGE, "unsupported dtype %d", dtype);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(bad_index_dev);
  init_u64_kernel<<<1, 1, 0, st>>>(bad, ~0ull, 0);
  if (nbytes == 0) return launch_check("init_u64_kernel");
  const bool al = (reinterpret_cast<uintptr_t>(src) % 16 == 0) &&
                  (reinterpret_cast<uintptr_t>(dst) % 16 == 0);
  const int64_t nvec = al ? nbytes / 16 : 0;
  cudaEvent_t stop;
  prof_begin(st, &stop);
  if (nvec > 0) {
    const int g = grid_for(nvec, kSnapThreads);
    const uint4* s4 = static_cast<const uint4*>(src);
    uint4* d4 = static_cast<uint4*>(dst);
    switch (dtype) {
      case DVLA_F32: snapshot_kernel<DVLA_F32><<<g, kSnapThreads, 0, st>>>(s4, d4, nvec, bad); break;
      case DVLA_BF16: snapshot_kernel<DVLA_BF16><<<g, kSnapThreads, 0, st>>>(s4, d4, nvec, bad); break;
      case DVLA_F64: snapshot_kernel<DVLA_F64><<<g, kSnapThreads, 0, st>>>(s4, d4, nvec, bad); break;
      default: snapshot_kernel<DVLA_U8><<<g, kSnapThreads, 0, st>>>(s4, d4, nvec, bad); break;
    }
  }
  const int64_t from = nvec * 16;
  if (from < nbytes) {
    const int64_t rem = nbytes - from;
    snapshot_tail_kernel<<<static_cast<unsigned>((rem + 255) / 256), 256, 0, st>>>(
        static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), from, nbytes, dtype, bad);
  }
  prof_end(st, stop);
  return launch_check("snapshot_kernel");
}

extern "C" int dvla_bytes_equal(const void* a, const void* b, int64_t nbytes, uint64_t* out_dev,
                                void* stream) {
  if (nbytes < 0) return fail(DVLA_ERR_USAGE, "nbytes must be >= 0");
  if (!out_dev || ((!a || !b) && nbytes > 0)) return fail(DVLA_ERR_USAGE, "null pointer argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* out = reinterpret_cast<unsigned long long*>(out_dev);
  init_u64_kernel<<<1, 1, 0, st>>>(out, 0ull, ~0ull);
  if (nbytes == 0) return launch_check("init_u64_kernel");
  const bool al = (reinterpret_cast<uintptr_t>(a) % 16 == 0) &&
                  (reinterpret_cast<uintptr_t>(b) % 16 == 0);
  const int64_t nvec = al ? nbytes / 16 : 0;
  if (nvec > 0)
    bytes_equal_kernel<<<grid_for(nvec, 256), 256, 0, st>>>(
        static_cast<const uint4*>(a), static_cast<const uint4*>(b), nvec, out);
  const int64_t from = nvec * 16;
  if (from < nbytes)
    bytes_equal_tail_kernel<<<static_cast<unsigned>((nbytes - from + 255) / 256), 256, 0, st>>>(
        static_cast<const uint8_t*>(a), static_cast<const uint8_t*>(b), from, nbytes, out);
  return launch_check("bytes_equal_kernel");
}

extern "C" int dvla_checksum64_at(const void* p, int64_t nbytes, int64_t first_word,
                                  uint64_t* out_dev, void* stream) {
  if (nbytes < 0 || first_word < 0) return fail(DVLA_ERR_USAGE, "nbytes, first_word must be >= 0");
  if (!out_dev || (!p && nbytes > 0)) return fail(DVLA_ERR_USAGE, "null pointer argument");
  if (reinterpret_cast<uintptr_t>(p) % 8) return fail(DVLA_ERR_USAGE, "region must be 8-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* out = reinterpret_cast<unsigned long long*>(out_dev);
  DVLA_CUDA_TRY(cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), st));
  const int64_t nwords = nbytes / 8;
  if (nwords > 0)
    checksum64_kernel<<<grid_for(nwords, 256), 256, 0, st>>>(static_cast<const uint2*>(p), nwords,
                                                              first_word, out);
  if (nwords * 8 < nbytes)
    checksum64_tail_kernel<<<1, 1, 0, st>>>(static_cast<const uint8_t*>(p), nwords * 8, nbytes,
                                            first_word, out);
  return launch_check("checksum64_kernel");
}

extern "C" int dvla_checksum64(const void* p, int64_t nbytes, uint64_t* out_dev, void* stream) {
  return dvla_checksum64_at(p, nbytes, 0, out_dev, stream);
}

extern "C" int dvla_memcpy_async(void* dst, const void* src, int64_t nbytes, void* stream) {
  if (nbytes < 0) return fail(DVLA_ERR_USAGE, "nbytes must be >= 0");
  if (nbytes == 0) return DVLA_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t stop;
  prof_begin(st, &stop);
  DVLA_CUDA_TRY(cudaMemcpyAsync(dst, src, static_cast<size_t>(nbytes), cudaMemcpyDefault, st));
  prof_end(st, stop);
  return DVLA_OK;
}

// Stream memory operations (copy-engine chain hops): block `stream` until
// *addr >= value / write value to *addr after all prior work of the stream
// (with a memory barrier, so a peer that observes the value sees the data).
extern "C" int dvla_stream_wait_u32(const uint32_t* addr, uint32_t value, void* stream) {
  if (!addr) return fail(DVLA_ERR_USAGE, "null flag address");
  if (int rc = drv_check()) return rc;
  DVLA_CU_TRY(cuStreamWaitValue32(static_cast<CUstream>(stream),
                                  reinterpret_cast<CUdeviceptr>(addr), value,
                                  CU_STREAM_WAIT_VALUE_GEQ));
  return DVLA_OK;
}

// Stream-ordered wait on several peer-written flags with a timeout (the
// bounded form of cuStreamWaitValue32): lane i of one warp acquire-polls
// flags[i] while bit i of `mask` is set, until flags[i] >= target; on
// timeout it sets *err and returns, so a dead peer surfaces as an error
// instead of a hung stream.
__global__ void wait_flags_kernel(const uint32_t* flags, uint32_t mask, uint32_t target,
                                  uint64_t timeout_ns, uint32_t* err) {
  const int i = threadIdx.x;
  if (!((mask >> i) & 1u)) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t ns = 32;
  while (ld_acquire_sys(flags + i) < target) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicOr(err, 1u);
      return;
    }
  }
}

extern "C" int dvla_wait_flags_u32(const uint32_t* flags, uint32_t mask, uint32_t target,
                                   uint64_t timeout_ns, uint32_t* err_dev, void* stream) {
  if (!flags || !err_dev) return fail(DVLA_ERR_USAGE, "null argument");
  if (!mask) return DVLA_OK;
  wait_flags_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(flags, mask, target,
                                                                     timeout_ns, err_dev);
  return launch_check("wait_flags_kernel");
}

// A few scalars reduced across the N ranks of a peer exchange over
// IPC-mapped peer memory, in rank order (every rank computes the same
// value): the learner's global sum of squares (f64 sum) and its abort /
// non-finite words (u32 max) without a collective library call.  Lane 0
// stores this rank's k values into slot [rank] of every peer's slot array,
// fences, and release-stores the epoch into every peer's flag [rank];
// lane p acquire-polls the local flag [p] (bounded: a timeout ORs *err);
// then lane 0 reduces the n contributions in rank order into out[0, k).
constexpr int kPeerMax = 32;
constexpr int kScalMax = 4;
struct PeerScalarTable {
  void* slots[kPeerMax];      // rank p's slot array ([n][k] values), mapped here
  uint32_t* flags[kPeerMax];  // rank p's flag array ([n] u32), mapped here
};

template <class T>
__global__ void peer_reduce_kernel(const T* local, int k, PeerScalarTable peers, int rank, int n,
                                   const T* my_slots, const uint32_t* my_flags, uint32_t epoch,
                                   uint64_t timeout_ns, uint32_t* err, T* out) {
  const int lane = threadIdx.x;
  T mine[kScalMax];
  for (int j = 0; j < k; ++j) mine[j] = local[j];
  if (lane == 0) {
    for (int p = 0; p < n; ++p) {
      if (p == rank) continue;
      T* dst = static_cast<T*>(peers.slots[p]) + rank * k;
      for (int j = 0; j < k; ++j) dst[j] = mine[j];
    }
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int p = 0; p < n; ++p)
      if (p != rank) st_release_sys(peers.flags[p] + rank, epoch);
  }
  if (lane < n && lane != rank) {
    const uint64_t t0 = globaltimer_ns();
    uint32_t ns = 32;
    while (ld_acquire_sys(my_flags + lane) < epoch) {
      __nanosleep(ns);
      if (ns < 512) ns <<= 1;
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicOr(err, 1u);
        break;
      }
    }
  }
  __syncwarp();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (lane == 0) {
    for (int j = 0; j < k; ++j) {
      T acc = T(0);
      for (int p = 0; p < n; ++p) {
        const T v = (p == rank) ? mine[j]
                                : *reinterpret_cast<const volatile T*>(my_slots + p * k + j);
        if constexpr (sizeof(T) == 8) {
          acc += v;                      // f64 sum in rank order
        } else {
          acc = acc > v ? acc : v;       // u32 max
        }
      }
      if constexpr (sizeof(T) == 8) {
        out[j] = acc;
      } else {  // keep what this launch's own timeout may have ORed in place
        const T cur = *reinterpret_cast<volatile T*>(out + j);
        out[j] = acc > cur ? acc : cur;
      }
    }
  }
}

extern "C" int dvla_peer_reduce(int kind, const void* local, int k, void* const* peer_slots,
                                uint32_t* const* peer_flags, int rank, int n,
                                const void* my_slots, const uint32_t* my_flags, uint32_t epoch,
                                uint64_t timeout_ns, uint32_t* err_dev, void* out,
                                void* stream) {
  if (!local || !peer_slots || !peer_flags || !my_slots || !my_flags || !err_dev || !out ||
      k < 1 || k > kScalMax || n < 1 || n > kPeerMax || rank < 0 || rank >= n ||
      (kind != 0 && kind != 1))
    return fail(DVLA_ERR_USAGE, "dvla_peer_reduce: bad arguments");
  PeerScalarTable t{};
  for (int p = 0; p < n; ++p) {
    if (p != rank && (!peer_slots[p] || !peer_flags[p]))
      return fail(DVLA_ERR_USAGE, "dvla_peer_reduce: missing peer %d mapping", p);
    t.slots[p] = peer_slots[p];
    t.flags[p] = peer_flags[p];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (kind == 0)
    peer_reduce_kernel<double><<<1, 32, 0, st>>>(
        static_cast<const double*>(local), k, t, rank, n, static_cast<const double*>(my_slots),
        my_flags, epoch, timeout_ns, err_dev, static_cast<double*>(out));
  else
    peer_reduce_kernel<uint32_t><<<1, 32, 0, st>>>(
        static_cast<const uint32_t*>(local), k, t, rank, n,
        static_cast<const uint32_t*>(my_slots), my_flags, epoch, timeout_ns, err_dev,
        static_cast<uint32_t*>(out));
  return launch_check("peer_reduce_kernel");
}

extern "C" int dvla_stream_write_u32(uint32_t* addr, uint32_t value, void* stream) {
  if (!addr) return fail(DVLA_ERR_USAGE, "null flag address");
  if (int rc = drv_check()) return rc;
  DVLA_CU_TRY(cuStreamWriteValue32(static_cast<CUstream>(stream),
                                   reinterpret_cast<CUdeviceptr>(addr), value,
                                   CU_STREAM_WRITE_VALUE_DEFAULT));
  return DVLA_OK;
}

// One hop of a copy-engine chain (same flag protocol as dvla_replicate_chain):
// per chunk c, the stream waits for wait_flags[c] >= epoch (upstream landed),
// copies the chunk into the downstream mapping with the copy engine, then
// writes signal_flags[c] = epoch (after the copy, with a memory barrier).
// Copy engines move peer bytes ~6 % faster than SM-issued stores on B200.
extern "C" int dvla_replicate_hop_ce(const void* src, void* dst, const uint32_t* wait_flags,
                                     uint32_t* signal_flags, int64_t nbytes, int64_t chunk_bytes,
                                     uint32_t epoch, void* stream) {
  if (nbytes < 0 || chunk_bytes < 16) return fail(DVLA_ERR_USAGE, "bad sizes");
  if (dst && !src) return fail(DVLA_ERR_USAGE, "destination without a source");
  if (epoch == 0) return fail(DVLA_ERR_USAGE, "epoch must be >= 1 (flags start at 0)");
  if (int rc = drv_check()) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n_chunks = (nbytes + chunk_bytes - 1) / chunk_bytes;
  cudaEvent_t stop;
  prof_begin(st, &stop);
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int64_t off = c * chunk_bytes;
    const int64_t len = (nbytes - off < chunk_bytes) ? nbytes - off : chunk_bytes;
    if (wait_flags)
      DVLA_CU_TRY(cuStreamWaitValue32(static_cast<CUstream>(st),
                                      reinterpret_cast<CUdeviceptr>(wait_flags + c), epoch,
                                      CU_STREAM_WAIT_VALUE_GEQ));
    if (dst) {
      DVLA_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off,
                                    static_cast<const uint8_t*>(src) + off,
                                    static_cast<size_t>(len), cudaMemcpyDefault, st));
      if (signal_flags)
        DVLA_CU_TRY(cuStreamWriteValue32(static_cast<CUstream>(st),
                                         reinterpret_cast<CUdeviceptr>(signal_flags + c), epoch,
                                         CU_STREAM_WRITE_VALUE_DEFAULT));
    }
  }
  prof_end(st, stop);
  return DVLA_OK;
}

// ------------------------------------------- one process, several devices
//
// dvla_replicate: the single-process form of ControlPlane.broadcast over
// NVLink (planes.py:294-321) for a driver that owns every GPU: src on
// src_dev is replicated into dst_ptrs[i] on dst_devs[i].
//   mode 0 (chain): hop i runs ON ITS SOURCE DEVICE (src_dev for the first,
//     dst_devs[i - 1] after), TMA-copying chunks into the next device and
//     releasing per-chunk flags; every link carries the region once.
//   mode 1 (copy engines): the source device's copy engines write every
//     destination directly (1 -> k fan-out).
// Flags live in per-device buffers owned by the library (grown on demand,
// never reset: every call uses a fresh epoch).  Work is enqueued on
// streams[0] (source) and streams[i + 1] (destination i), or each device's
// legacy default stream when streams is NULL; the call returns once all of
// it is enqueued.  Calls on overlapping device sets must be serialised by
// the caller (stream order suffices when the same streams are reused).
namespace dvla {
struct RepFlags {
  uint32_t* ptr = nullptr;
  size_t count = 0;
  uint32_t* err = nullptr;
};
// The single-process replication's flag buffers and epoch counter (the
// only mutable library state): every dvla_replicate / dvla_replicate_status
// call holds g_rep_mutex for its whole (host-side, enqueue-only) duration.
static RepFlags g_rep_flags[64];
static uint32_t g_rep_epoch = 0;
static std::mutex g_rep_mutex;
}  // namespace dvla

extern "C" int dvla_replicate(int src_dev, const void* src, int n_dst, const int* dst_devs,
                              void* const* dst_ptrs, int64_t nbytes, int64_t chunk_bytes,
                              int mode, void* const* streams) {
  if (n_dst < 0 || n_dst >= kMaxHops || (n_dst > 0 && (!dst_devs || !dst_ptrs)) || !src ||
      nbytes < 0 || (nbytes % 16) != 0 || (mode != 0 && mode != 1))
    return fail(DVLA_ERR_USAGE, "dvla_replicate: bad arguments");
  if (n_dst == 0 || nbytes == 0) return DVLA_OK;
  if (chunk_bytes <= 0) chunk_bytes = 1 << 20;
  if (chunk_bytes % 16) return fail(DVLA_ERR_USAGE, "chunk_bytes must be a multiple of 16");
  std::lock_guard<std::mutex> lock(g_rep_mutex);
  int prev = 0;
  DVLA_CUDA_TRY(cudaGetDevice(&prev));
  auto stream_of = [&](int i) {  // i = 0: source, i > 0: destination i - 1
    return streams ? static_cast<cudaStream_t>(streams[i]) : cudaStream_t{0};
  };
  int rc = DVLA_OK;
  if (mode == 1) {
    for (int i = 0; i < n_dst && rc == DVLA_OK; ++i) {
      cudaSetDevice(src_dev);
      if (cudaMemcpyPeerAsync(dst_ptrs[i], dst_devs[i], src, src_dev, static_cast<size_t>(nbytes),
                              stream_of(0)) != cudaSuccess)
        rc = fail(DVLA_ERR_CUDA, "cudaMemcpyPeerAsync to device %d: %s", dst_devs[i],
                  cudaGetErrorString(cudaGetLastError()));
    }
    cudaSetDevice(prev);
    return rc;
  }
  const int64_t n_chunks = (nbytes + chunk_bytes - 1) / chunk_bytes;
  // peer access along the chain, flag buffers on every destination
  for (int i = 0; i < n_dst && rc == DVLA_OK; ++i) {
    const int from = i == 0 ? src_dev : dst_devs[i - 1];
    if (from != dst_devs[i]) rc = dvla_enable_peer_access(from, dst_devs[i]);
    if (rc) break;
    RepFlags& f = g_rep_flags[dst_devs[i] & 63];
    if (f.count < static_cast<size_t>(n_chunks)) {
      cudaSetDevice(dst_devs[i]);
      if (f.ptr) cudaFree(f.ptr);
      if (!f.err && cudaMalloc(&f.err, 16) != cudaSuccess) rc = fail(DVLA_ERR_CUDA, "flag alloc");
      if (!rc && cudaMalloc(&f.ptr, static_cast<size_t>(n_chunks) * 4) != cudaSuccess)
        rc = fail(DVLA_ERR_CUDA, "flag alloc");
      if (!rc) {
        cudaMemset(f.ptr, 0, static_cast<size_t>(n_chunks) * 4);
        cudaMemset(f.err, 0, 16);
        cudaDeviceSynchronize();
        f.count = static_cast<size_t>(n_chunks);
        g_rep_epoch = 0;  // a fresh zeroed buffer restarts the epochs... for all devices:
        for (auto& o : g_rep_flags)
          if (o.ptr && &o != &f) {
            cudaSetDevice(static_cast<int>(&o - g_rep_flags));
            cudaMemset(o.ptr, 0, o.count * 4);
            cudaDeviceSynchronize();
          }
      }
    }
  }
  if (rc) {
    cudaSetDevice(prev);
    return rc;
  }
  const uint32_t epoch = ++g_rep_epoch;
  // hops that run on the same device go into ONE launch (co-resident CTA
  // groups): a waiting hop must never queue behind its producer on a GPU
  dvla_hop hops[kMaxHops + 1];
  int hop_dev[kMaxHops + 1], hop_stream[kMaxHops + 1];
  for (int i = 0; i <= n_dst; ++i) {
    dvla_hop& h = hops[i];
    h.src = i == 0 ? src : dst_ptrs[i - 1];
    h.dst = i < n_dst ? dst_ptrs[i] : nullptr;
    h.wait_flags = i == 0 ? nullptr : g_rep_flags[dst_devs[i - 1] & 63].ptr;
    h.signal_flags = i < n_dst ? g_rep_flags[dst_devs[i] & 63].ptr : nullptr;
    if (!h.dst) h.src = nullptr;
    hop_dev[i] = i == 0 ? src_dev : dst_devs[i - 1];
    hop_stream[i] = i;
  }
  bool done[kMaxHops + 1] = {};
  for (int i = 0; i <= n_dst && rc == DVLA_OK; ++i) {
    if (done[i]) continue;
    dvla_hop group[kMaxHops + 1];
    int g = 0;
    for (int j = i; j <= n_dst; ++j)
      if (!done[j] && hop_dev[j] == hop_dev[i]) {
        group[g++] = hops[j];
        done[j] = true;
      }
    const int dev = hop_dev[i];
    cudaSetDevice(dev);
    rc = dvla_replicate_chain(group, g, nbytes, chunk_bytes, epoch, g > 1 ? 128 / g : 128,
                              30ull * 1000000000ull, g_rep_flags[dev & 63].err
                                  ? g_rep_flags[dev & 63].err
                                  : g_rep_flags[dst_devs[0] & 63].err,
                              stream_of(hop_stream[i]));
  }
  cudaSetDevice(prev);
  return rc;
}

// Reads and clears the timeout flags of dvla_replicate's chain hops
// (synchronous; call after the streams used by dvla_replicate are idle).
extern "C" int dvla_replicate_status(int* timed_out) {
  if (!timed_out) return fail(DVLA_ERR_USAGE, "null out pointer");
  std::lock_guard<std::mutex> lock(g_rep_mutex);
  int prev = 0;
  DVLA_CUDA_TRY(cudaGetDevice(&prev));
  *timed_out = 0;
  for (int d = 0; d < 64; ++d) {
    if (!g_rep_flags[d].err) continue;
    uint32_t v = 0;
    cudaSetDevice(d);
    DVLA_CUDA_TRY(cudaMemcpy(&v, g_rep_flags[d].err, 4, cudaMemcpyDeviceToHost));
    if (v) {
      *timed_out = 1;
      DVLA_CUDA_TRY(cudaMemset(g_rep_flags[d].err, 0, 4));
    }
  }
  cudaSetDevice(prev);
  return DVLA_OK;
}
