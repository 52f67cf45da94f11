// Error plumbing and small device queries for the C-ABI.
#include <stdarg.h>

#include <utility>
#include <vector>

#include "common.cuh"

namespace dvla {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int num_sms(int device) {
  static int cache[64] = {0};
  int d = device & 63;
  if (cache[d] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0)
      n = 148;
    cache[d] = n;
  }
  return cache[d];
}

// ---------------------------------------------------------------- profiling
// Optional per-thread event pairs around the dominant kernel of an entry
// point (enabled by dvla_profile_enable).  bench.py uses this to time the
// kernel alone on its launch stream while the whole step is timed too.
struct ProfRing {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pairs;
  size_t used = 0;
};
static thread_local ProfRing g_prof;

void prof_begin(cudaStream_t s, cudaEvent_t* stop_out) {
  *stop_out = nullptr;
  if (!g_prof.on) return;
  if (g_prof.used == g_prof.pairs.size()) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess) return;
    if (cudaEventCreate(&b) != cudaSuccess) return;
    g_prof.pairs.push_back({a, b});
  }
  auto& pr = g_prof.pairs[g_prof.used++];
  cudaEventRecord(pr.first, s);
  *stop_out = pr.second;
}

void prof_end(cudaStream_t s, cudaEvent_t stop) {
  if (stop) cudaEventRecord(stop, s);
}

}  // namespace dvla

extern "C" int dvla_profile_enable(int on) {
  dvla::g_prof.on = on != 0;
  dvla::g_prof.used = 0;
  return DVLA_OK;
}

extern "C" int dvla_profile_collect(double* total_ms, int64_t* count) {
  double sum = 0.0;
  for (size_t i = 0; i < dvla::g_prof.used; ++i) {
    auto& pr = dvla::g_prof.pairs[i];
    DVLA_CUDA_TRY(cudaEventSynchronize(pr.second));
    float ms = 0.f;
    DVLA_CUDA_TRY(cudaEventElapsedTime(&ms, pr.first, pr.second));
    sum += ms;
  }
  if (total_ms) *total_ms = sum;
  if (count) *count = static_cast<int64_t>(dvla::g_prof.used);
  dvla::g_prof.used = 0;
  return DVLA_OK;
}

extern "C" const char* dvla_last_error(void) { return dvla::g_last_error.c_str(); }

extern "C" int dvla_abi_version(void) { return 1; }
