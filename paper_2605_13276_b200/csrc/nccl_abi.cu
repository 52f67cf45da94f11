// NCCL behind the C-ABI for a process that drives several GPUs itself
// (GradReducer.reduce, runtime.py:569-637, without torch.distributed):
// communicators over the caller's devices and an in-place sum all-reduce.
// libnccl is opened at run time (dlopen), so the library keeps no link
// dependency on it; inside a PyTorch process this resolves to the NCCL that
// torch already loaded.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "common.cuh"

namespace dvla {
namespace {

struct Nccl {
  void* so = nullptr;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) err_str = nullptr;
};

Nccl g_nccl;
ncclComm_t g_comms[64];
int g_n = 0;
std::mutex g_mu;

int load() {
  if (g_nccl.so) return DVLA_OK;
  void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!so) return fail(DVLA_ERR_CUDA, "dlopen(libnccl.so.2) failed: %s", dlerror());
  Nccl n;
  n.so = so;
  n.init_all = reinterpret_cast<decltype(n.init_all)>(dlsym(so, "ncclCommInitAll"));
  n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(so, "ncclAllReduce"));
  n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(so, "ncclGroupStart"));
  n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(so, "ncclGroupEnd"));
  n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(so, "ncclCommDestroy"));
  n.err_str = reinterpret_cast<decltype(n.err_str)>(dlsym(so, "ncclGetErrorString"));
  if (!n.init_all || !n.all_reduce || !n.group_start || !n.group_end || !n.destroy || !n.err_str)
    return fail(DVLA_ERR_CUDA, "libnccl.so.2 lacks an expected symbol");
  g_nccl = n;
  return DVLA_OK;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return DVLA_OK;
  return fail(DVLA_ERR_CUDA, "%s: %s", what, g_nccl.err_str ? g_nccl.err_str(r) : "?");
}

}  // namespace
}  // namespace dvla

using namespace dvla;

extern "C" int dvla_nccl_init(int n, const int* devs) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (n < 1 || n > 64 || !devs) return fail(DVLA_ERR_USAGE, "dvla_nccl_init: 1..64 devices");
  if (int rc = load()) return rc;
  for (int i = 0; i < g_n; ++i) g_nccl.destroy(g_comms[i]);
  g_n = 0;
  if (int rc = nccl_check(g_nccl.init_all(g_comms, n, devs), "ncclCommInitAll")) return rc;
  g_n = n;
  return DVLA_OK;
}

extern "C" int dvla_nccl_group_start(void) {
  if (int rc = load()) return rc;
  return nccl_check(g_nccl.group_start(), "ncclGroupStart");
}

extern "C" int dvla_nccl_group_end(void) {
  if (int rc = load()) return rc;
  return nccl_check(g_nccl.group_end(), "ncclGroupEnd");
}

extern "C" int dvla_nccl_allreduce_sum(int comm_idx, void* ptr, int64_t count, int dtype,
                                       void* stream) {
  if (comm_idx < 0 || comm_idx >= g_n) return fail(DVLA_ERR_USAGE, "no communicator %d", comm_idx);
  if (!ptr || count < 0) return fail(DVLA_ERR_USAGE, "bad buffer");
  ncclDataType_t t;
  switch (dtype) {
    case DVLA_F32: t = ncclFloat32; break;
    case DVLA_F64: t = ncclFloat64; break;
    case DVLA_BF16: t = ncclBfloat16; break;
    default: return fail(DVLA_ERR_USAGE, "dtype must be f32, f64 or bf16");
  }
  return nccl_check(g_nccl.all_reduce(ptr, ptr, static_cast<size_t>(count), t, ncclSum,
                                      g_comms[comm_idx], static_cast<cudaStream_t>(stream)),
                    "ncclAllReduce");
}

extern "C" int dvla_nccl_destroy(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (int i = 0; i < g_n; ++i) g_nccl.destroy(g_comms[i]);
  g_n = 0;
  return DVLA_OK;
}
