// Switch-multicast (NVLS) weight replication over NVSwitch.
//
// Same reference path as the chain (replicate.cu): ControlPlane.broadcast
// (planes.py:294-321) delivering one ParamSnapshot (core.py:101-129) to every
// subscriber's WeightMailbox (planes.py:232-275).  Here the source GPU writes
// each byte ONCE into a multicast address; the NVSwitch replicates the write
// into the bound region of every member GPU, so per-receiver bandwidth does
// not divide by the number of receivers (a copy-engine fan-out does) and
// there is no per-hop forwarding (the chain's flags and fill).
//
// Setup (one process per GPU, cuMem* driver API):
//   root:   dvla_mc_create   -> multicast object for n devices, exported as a
//                               POSIX file descriptor
//   others: dvla_mc_import   -> the root's fd fetched with pidfd_getfd(2)
//   all:    dvla_mc_add_device(own device), barrier, dvla_mc_bind (physical
//           memory on the own device bound at offset 0 and mapped locally),
//           barrier; root: dvla_mc_map (multicast VA)
// Data path: dvla_mc_broadcast (root; ld.global.nc -> multimem.st, then one
// release store of the epoch into every member's flag word through the
// multicast address), dvla_mc_wait (receivers; acquire-poll the local flag).
#include <cuda.h>
#include <stdlib.h>
#include <string.h>
#include <sys/syscall.h>
#include <unistd.h>

#include "common.cuh"
#include "drv.cuh"

namespace dvla {


struct McObj {
  CUmemGenericAllocationHandle mc = 0;   // multicast object
  CUmemGenericAllocationHandle mem = 0;  // this device's bound physical memory
  CUdeviceptr local = 0;                 // local mapping of `mem`
  CUdeviceptr mcva = 0;                  // multicast mapping (writers)
  size_t size = 0;                       // padded size (multiple of the granularity)
  int n_devices = 0;
  int device = -1;
  int fd = -1;
  bool bound = false;
};


static int mc_granularity(int n_devices, size_t nbytes, size_t* gran) {
  CUmulticastObjectProp prop{};
  prop.numDevices = static_cast<unsigned>(n_devices);
  prop.size = nbytes;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  DVLA_CU_TRY(cuMulticastGetGranularity(gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  return DVLA_OK;
}

constexpr int kMcThreads = 512;
constexpr int kMcUnroll = 4;

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void multimem_st_u4(void* mc, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void multimem_st_release_u32(uint32_t* mc, uint32_t v) {
  asm volatile("multimem.st.release.sys.global.u32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}

// Grid-stride copy src -> multicast dst in 16-byte vectors (4 in flight per
// thread); the last CTA to finish publishes `epoch` into every member's flag.
__global__ void __launch_bounds__(kMcThreads) mc_broadcast_kernel(const uint4* __restrict__ src,
                                                                  uint4* mc_dst, int64_t nvec,
                                                                  uint32_t* mc_flag,
                                                                  uint32_t* done_ctr,
                                                                  uint32_t epoch) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kMcThreads;
  int64_t i = static_cast<int64_t>(blockIdx.x) * kMcThreads + threadIdx.x;
  for (; i + (kMcUnroll - 1) * stride < nvec; i += kMcUnroll * stride) {
    uint4 v[kMcUnroll];
#pragma unroll
    for (int u = 0; u < kMcUnroll; ++u) v[u] = ld_stream_u4(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < kMcUnroll; ++u) multimem_st_u4(mc_dst + i + u * stride, v[u]);
  }
  for (; i < nvec; i += stride) multimem_st_u4(mc_dst + i, ld_stream_u4(src + i));
  // every thread's stores are ordered before its CTA's arrival (sys scope)
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atom_add_acq_rel_gpu(done_ctr, 1u);
    if (prev == gridDim.x - 1) {
      *done_ctr = 0;  // reset for the next broadcast (stream-ordered)
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      multimem_st_release_u32(mc_flag, epoch);
    }
  }
}

__global__ void mc_wait_kernel(const uint32_t* flag, uint32_t epoch, uint64_t timeout_ns,
                               uint32_t* err) {
  if (threadIdx.x != 0) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t ns = 64;
  while (ld_acquire_sys(flag) < epoch) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicOr(err, 1u);
      return;
    }
  }
}

}  // namespace dvla

using namespace dvla;

extern "C" int dvla_mc_supported(int device, int* out) {
  if (!out) return fail(DVLA_ERR_USAGE, "null out pointer");
  if (int rc = drv_check()) return rc;
  DVLA_CU_TRY(cuInit(0));
  CUdevice dev;
  DVLA_CU_TRY(cuDeviceGet(&dev, device));
  int mc = 0, fd = 0;
  DVLA_CU_TRY(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  DVLA_CU_TRY(
      cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev));
  *out = (mc && fd) ? 1 : 0;
  return DVLA_OK;
}

extern "C" int dvla_mc_create(int n_devices, size_t nbytes, int* fd_out, size_t* size_out,
                              void** obj_out) {
  if (n_devices < 1 || !fd_out || !size_out || !obj_out || nbytes == 0)
    return fail(DVLA_ERR_USAGE, "dvla_mc_create: bad arguments");
  if (int rc = drv_check()) return rc;
  DVLA_CU_TRY(cuInit(0));
  size_t gran = 0;
  if (int rc = mc_granularity(n_devices, nbytes, &gran)) return rc;
  McObj* o = new McObj();
  o->n_devices = n_devices;
  o->size = (nbytes + gran - 1) / gran * gran;
  CUmulticastObjectProp prop{};
  prop.numDevices = static_cast<unsigned>(n_devices);
  prop.size = o->size;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUresult r = cuMulticastCreate(&o->mc, &prop);
  if (r != CUDA_SUCCESS) {
    delete o;
    return fail(DVLA_ERR_CUDA, "cuMulticastCreate(%d devices, %zu bytes) failed: %d", n_devices,
                nbytes, static_cast<int>(r));
  }
  int fd = -1;
  r = cuMemExportToShareableHandle(&fd, o->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  if (r != CUDA_SUCCESS) {
    cuMemRelease(o->mc);
    delete o;
    return fail(DVLA_ERR_CUDA, "exporting the multicast handle failed: %d", static_cast<int>(r));
  }
  o->fd = fd;
  *fd_out = fd;
  *size_out = o->size;
  *obj_out = o;
  return DVLA_OK;
}

extern "C" int dvla_mc_import(int owner_pid, int owner_fd, int n_devices, size_t size,
                              void** obj_out) {
  if (!obj_out || owner_pid <= 0 || owner_fd < 0)
    return fail(DVLA_ERR_USAGE, "dvla_mc_import: bad arguments");
  if (int rc = drv_check()) return rc;
  DVLA_CU_TRY(cuInit(0));
  const int pidfd = static_cast<int>(syscall(SYS_pidfd_open, owner_pid, 0));
  if (pidfd < 0) return fail(DVLA_ERR_CUDA, "pidfd_open(%d) failed", owner_pid);
  const int fd = static_cast<int>(syscall(SYS_pidfd_getfd, pidfd, owner_fd, 0));
  close(pidfd);
  if (fd < 0)
    return fail(DVLA_ERR_CUDA, "pidfd_getfd(pid %d, fd %d) failed (ptrace permission?)", owner_pid,
                owner_fd);
  McObj* o = new McObj();
  o->n_devices = n_devices;
  o->size = size;
  o->fd = fd;
  CUresult r = cuMemImportFromShareableHandle(
      &o->mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  if (r != CUDA_SUCCESS) {
    close(fd);
    delete o;
    return fail(DVLA_ERR_CUDA, "importing the multicast handle failed: %d", static_cast<int>(r));
  }
  *obj_out = o;
  return DVLA_OK;
}

extern "C" int dvla_mc_add_device(void* obj, int device) {
  McObj* o = static_cast<McObj*>(obj);
  if (!o) return fail(DVLA_ERR_USAGE, "null multicast object");
  CUdevice dev;
  DVLA_CU_TRY(cuDeviceGet(&dev, device));
  DVLA_CU_TRY(cuMulticastAddDevice(o->mc, dev));
  o->device = device;
  return DVLA_OK;
}

// Physical memory on `device` bound at multicast offset 0 and mapped locally
// (read/write); every member must have been added first.
extern "C" int dvla_mc_bind(void* obj, int device, void** local_out) {
  McObj* o = static_cast<McObj*>(obj);
  if (!o || !local_out) return fail(DVLA_ERR_USAGE, "null argument");
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t agran = 0;
  DVLA_CU_TRY(cuMemGetAllocationGranularity(&agran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  if (o->size % agran) return fail(DVLA_ERR_CUDA, "multicast size not a multiple of %zu", agran);
  DVLA_CU_TRY(cuMemCreate(&o->mem, o->size, &prop, 0));
  DVLA_CU_TRY(cuMulticastBindMem(o->mc, 0, o->mem, 0, o->size, 0));
  o->bound = true;
  DVLA_CU_TRY(cuMemAddressReserve(&o->local, o->size, agran, 0, 0));
  DVLA_CU_TRY(cuMemMap(o->local, o->size, 0, o->mem, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  DVLA_CU_TRY(cuMemSetAccess(o->local, o->size, &acc, 1));
  *local_out = reinterpret_cast<void*>(o->local);
  return DVLA_OK;
}

// Multicast VA on the calling process's device (stores reach every member).
extern "C" int dvla_mc_map(void* obj, int device, void** mc_out) {
  McObj* o = static_cast<McObj*>(obj);
  if (!o || !mc_out) return fail(DVLA_ERR_USAGE, "null argument");
  size_t gran = 0;
  if (int rc = mc_granularity(o->n_devices, o->size, &gran)) return rc;
  DVLA_CU_TRY(cuMemAddressReserve(&o->mcva, o->size, gran, 0, 0));
  DVLA_CU_TRY(cuMemMap(o->mcva, o->size, 0, o->mc, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  DVLA_CU_TRY(cuMemSetAccess(o->mcva, o->size, &acc, 1));
  *mc_out = reinterpret_cast<void*>(o->mcva);
  return DVLA_OK;
}

extern "C" int dvla_mc_destroy(void* obj) {
  McObj* o = static_cast<McObj*>(obj);
  if (!o) return DVLA_OK;
  if (o->mcva) {
    cuMemUnmap(o->mcva, o->size);
    cuMemAddressFree(o->mcva, o->size);
  }
  if (o->local) {
    cuMemUnmap(o->local, o->size);
    cuMemAddressFree(o->local, o->size);
  }
  if (o->bound) {
    CUdevice dev;
    if (cuDeviceGet(&dev, o->device) == CUDA_SUCCESS) cuMulticastUnbind(o->mc, dev, 0, o->size);
  }
  if (o->mem) cuMemRelease(o->mem);
  if (o->mc) cuMemRelease(o->mc);
  if (o->fd >= 0) close(o->fd);
  delete o;
  return DVLA_OK;
}

extern "C" int dvla_mc_broadcast(const void* src, void* mc_dst, int64_t nbytes, void* mc_flag,
                                 uint32_t epoch, int ctas, uint32_t* done_ctr, void* stream) {
  if (!src || !mc_dst || !mc_flag || !done_ctr || nbytes < 0 || (nbytes % 16) != 0 ||
      (reinterpret_cast<uintptr_t>(src) % 16) != 0 || (reinterpret_cast<uintptr_t>(mc_dst) % 16) != 0)
    return fail(DVLA_ERR_USAGE, "dvla_mc_broadcast: null or misaligned argument");
  const int sms = num_sms(current_device());
  const int grid = ctas > 0 ? ctas : sms;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t stop;
  prof_begin(st, &stop);
  mc_broadcast_kernel<<<grid, kMcThreads, 0, st>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(mc_dst), nbytes / 16,
      static_cast<uint32_t*>(mc_flag), done_ctr, epoch);
  prof_end(st, stop);
  return launch_check("mc_broadcast_kernel");
}

extern "C" int dvla_mc_wait(const uint32_t* local_flag, uint32_t epoch, uint64_t timeout_ns,
                            uint32_t* err_dev, void* stream) {
  if (!local_flag || !err_dev) return fail(DVLA_ERR_USAGE, "null argument");
  mc_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(local_flag, epoch, timeout_ns,
                                                                  err_dev);
  return launch_check("mc_wait_kernel");
}

// ------------------------------------------- switch-reduced all-reduce (f32)
//
// Learner-gradient mean across ranks (GradReducer.reduce, runtime.py:569-637;
// SURVEY §8 a10) on NVSwitch multicast memory: every rank's f32 gradient
// lives in its bound region of one multicast object; rank r owns the slice
// [r n / N, (r + 1) n / N) and, per 16-byte granule, issues ONE
// multimem.ld_reduce.add (the switch reads and sums the granule from every
// member) and ONE multimem.st of the sum (the switch writes it into every
// member).  Per GPU and direction the links carry (N + 1) / N of the
// buffer (a ring all-reduce: 2 (N - 1) / N), the reduction happens in the
// switch, and there are no rank-to-rank pipeline steps.  Entry and exit
// barriers are flag counters in the same
// multicast region, bumped with multimem.red.release and acquire-polled
// locally; `epoch` = 1, 2, ... per call (flags start at 0).

__device__ __forceinline__ void multimem_red_add_release_u32(uint32_t* mc, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}

__device__ __forceinline__ uint4 multimem_ld_reduce_add_f32x4(const void* mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}

__device__ __forceinline__ bool mc_wait_count(const uint32_t* flag, uint32_t target,
                                              uint64_t timeout_ns, uint32_t* err) {
  const uint64_t t0 = globaltimer_ns();
  uint32_t ns = 32;
  while (ld_acquire_sys(flag) < target) {
    __nanosleep(ns);
    if (ns < 512) ns <<= 1;
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicOr(err, 1u);
      return false;
    }
  }
  return true;
}

constexpr int kArThreads = 512;

// flags: [0] entry counter, [1] exit counter (local view and multicast view)
__global__ void __launch_bounds__(kArThreads) mc_allreduce_f32_kernel(
    uint4* mc_buf, int64_t nvec, int rank, int world, const uint32_t* local_flags,
    uint32_t* mc_flags, uint32_t epoch, uint32_t* done_ctr, float scale, uint64_t timeout_ns,
    uint32_t* err) {
  __shared__ int s_ok;
  // entry barrier: every rank's gradient is in place before anyone reduces
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      multimem_red_add_release_u32(mc_flags, 1u);
    }
    s_ok = mc_wait_count(local_flags, epoch * static_cast<uint32_t>(world), timeout_ns, err);
  }
  __syncthreads();
  if (!s_ok) return;
  const int64_t per = (nvec + world - 1) / world;
  const int64_t lo = per * rank, hi = (lo + per < nvec) ? lo + per : nvec;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kArThreads;
  // (one reduction in flight per thread measured as fast as four: the
  // switch, not the issue rate, bounds this loop)
  for (int64_t i = lo + static_cast<int64_t>(blockIdx.x) * kArThreads + threadIdx.x; i < hi;
       i += stride) {
    uint4 v = multimem_ld_reduce_add_f32x4(mc_buf + i);
    if (scale != 1.0f) {
      v.x = __float_as_uint(__uint_as_float(v.x) * scale);
      v.y = __float_as_uint(__uint_as_float(v.y) * scale);
      v.z = __float_as_uint(__uint_as_float(v.z) * scale);
      v.w = __float_as_uint(__uint_as_float(v.w) * scale);
    }
    multimem_st_u4(mc_buf + i, v);
  }
  // exit barrier: this rank's slice is stored everywhere; the last CTA of the
  // rank signals, then waits until every rank has (results complete here)
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atom_add_acq_rel_gpu(done_ctr, 1u);
    if (prev == gridDim.x - 1) {
      *done_ctr = 0;
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      multimem_red_add_release_u32(mc_flags + 1, 1u);
      mc_wait_count(local_flags + 1, epoch * static_cast<uint32_t>(world), timeout_ns, err);
    }
  }
}

extern "C" int dvla_mc_allreduce_f32(void* mc_buf, int64_t n, int rank, int world,
                                     const uint32_t* local_flags, void* mc_flags, uint32_t epoch,
                                     float scale, int ctas, uint32_t* done_ctr,
                                     uint64_t timeout_ns, uint32_t* err_dev, void* stream) {
  if (!mc_buf || !local_flags || !mc_flags || !done_ctr || !err_dev || n < 0 || (n % 4) != 0 ||
      world < 1 || rank < 0 || rank >= world || epoch == 0)
    return fail(DVLA_ERR_USAGE, "dvla_mc_allreduce_f32: bad arguments (n must be a multiple of 4)");
  const int grid = ctas > 0 ? ctas : num_sms(current_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t stop;
  prof_begin(st, &stop);
  mc_allreduce_f32_kernel<<<grid, kArThreads, 0, st>>>(
      static_cast<uint4*>(mc_buf), n / 4, rank, world, local_flags,
      static_cast<uint32_t*>(mc_flags), epoch, done_ctr, scale, timeout_ns, err_dev);
  prof_end(st, stop);
  return launch_check("mc_allreduce_f32_kernel");
}
