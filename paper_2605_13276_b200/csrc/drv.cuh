// Driver-API access without a link-time libcuda dependency (shared by
// multicast.cu and replicate.cu).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace dvla {

// Driver-API entry points resolved at first use through the runtime
// (cudaGetDriverEntryPoint), so libdvla_b200.so carries no link-time
// dependency on libcuda (it must load on hosts without a driver: CPU tests).
#define DVLA_DRV_LIST(X)                                                                    \
  X(cuDeviceGet) X(cuDeviceGetAttribute) X(cuGetErrorString) X(cuInit) X(cuMemAddressFree)  \
  X(cuMemAddressReserve) X(cuMemCreate) X(cuMemExportToShareableHandle)                     \
  X(cuMemGetAllocationGranularity) X(cuMemImportFromShareableHandle) X(cuMemMap)            \
  X(cuMemRelease) X(cuMemSetAccess) X(cuMemUnmap) X(cuMulticastAddDevice)                   \
  X(cuMulticastBindMem) X(cuMulticastCreate) X(cuMulticastGetGranularity)                   \
  X(cuMulticastUnbind) X(cuStreamWaitValue32) X(cuStreamWriteValue32)

struct DrvTable {
#define DVLA_DRV_MEMBER(fn) decltype(&::fn) p_##fn = nullptr;
  DVLA_DRV_LIST(DVLA_DRV_MEMBER)
#undef DVLA_DRV_MEMBER
  bool ok = true;
  const char* missing = nullptr;
};

inline const DrvTable& drv() {
  static const DrvTable t = [] {
    DrvTable d;
    cudaFree(nullptr);  // initialise the runtime (and the driver under it)
#define DVLA_DRV_RESOLVE(fn)                                                              \
  {                                                                                       \
    void* f = nullptr;                                                                    \
    cudaDriverEntryPointQueryResult q;                                                    \
    if (cudaGetDriverEntryPoint(#fn, &f, cudaEnableDefault, &q) != cudaSuccess ||         \
        q != cudaDriverEntryPointSuccess || !f) {                                         \
      cudaGetLastError();                                                                 \
      if (d.ok) d.missing = #fn;                                                          \
      d.ok = false;                                                                       \
    } else {                                                                              \
      d.p_##fn = reinterpret_cast<decltype(&::fn)>(f);                                    \
    }                                                                                     \
  }
    DVLA_DRV_LIST(DVLA_DRV_RESOLVE)
#undef DVLA_DRV_RESOLVE
    return d;
  }();
  return t;
}

// every cuXxx( below goes through the table
#define cuDeviceGet(...) drv().p_cuDeviceGet(__VA_ARGS__)
#define cuDeviceGetAttribute(...) drv().p_cuDeviceGetAttribute(__VA_ARGS__)
#define cuGetErrorString(...) drv().p_cuGetErrorString(__VA_ARGS__)
#define cuInit(...) drv().p_cuInit(__VA_ARGS__)
#define cuMemAddressFree(...) drv().p_cuMemAddressFree(__VA_ARGS__)
#define cuMemAddressReserve(...) drv().p_cuMemAddressReserve(__VA_ARGS__)
#define cuMemCreate(...) drv().p_cuMemCreate(__VA_ARGS__)
#define cuMemExportToShareableHandle(...) drv().p_cuMemExportToShareableHandle(__VA_ARGS__)
#define cuMemGetAllocationGranularity(...) drv().p_cuMemGetAllocationGranularity(__VA_ARGS__)
#define cuMemImportFromShareableHandle(...) drv().p_cuMemImportFromShareableHandle(__VA_ARGS__)
#define cuMemMap(...) drv().p_cuMemMap(__VA_ARGS__)
#define cuMemRelease(...) drv().p_cuMemRelease(__VA_ARGS__)
#define cuMemSetAccess(...) drv().p_cuMemSetAccess(__VA_ARGS__)
#define cuMemUnmap(...) drv().p_cuMemUnmap(__VA_ARGS__)
#define cuMulticastAddDevice(...) drv().p_cuMulticastAddDevice(__VA_ARGS__)
#define cuMulticastBindMem(...) drv().p_cuMulticastBindMem(__VA_ARGS__)
#define cuMulticastCreate(...) drv().p_cuMulticastCreate(__VA_ARGS__)
#define cuMulticastGetGranularity(...) drv().p_cuMulticastGetGranularity(__VA_ARGS__)
#define cuMulticastUnbind(...) drv().p_cuMulticastUnbind(__VA_ARGS__)
// (cuda.h maps these two to versioned symbols; the table holds the default
// version resolved for this CUDA_VERSION)
#undef cuStreamWaitValue32
#undef cuStreamWriteValue32
#define cuStreamWaitValue32(...) drv().p_cuStreamWaitValue32(__VA_ARGS__)
#define cuStreamWriteValue32(...) drv().p_cuStreamWriteValue32(__VA_ARGS__)

inline int drv_check() {
  if (!drv().ok)
    return fail(DVLA_ERR_CUDA, "driver entry point %s unavailable", drv().missing);
  return DVLA_OK;
}

#define DVLA_CU_TRY(expr)                                                           \
  do {                                                                              \
    CUresult _r = (expr);                                                           \
    if (_r != CUDA_SUCCESS) {                                                       \
      const char* _s = nullptr;                                                     \
      cuGetErrorString(_r, &_s);                                                    \
      return ::dvla::fail(DVLA_ERR_CUDA, "%s failed: %s", #expr, _s ? _s : "?");    \
    }                                                                               \
  } while (0)

}  // namespace dvla
