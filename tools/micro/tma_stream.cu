// Microbenchmark: per-SM TMA bulk-load ring (S stages x P bytes, 1 CTA/SM)
// with optional concurrent streaming writes of the same volume by the
// consumer warps.  Measures the achievable HBM read (+write) bandwidth of the
// fused loss kernel's memory pattern.  nvcc -arch=sm_100a -O3 tma_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_13276_b200/csrc/common.cuh"
using namespace dvla;

__global__ void __launch_bounds__(544, 1) ring(const uint8_t* src, uint8_t* dst, int64_t nbytes,
                                               int S, int P, int write_mode) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 32;
  uint8_t* buf = sm + 512;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t npieces = nbytes / P;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 16); }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 16) {
    if (lane == 0) {
      int64_t n = 0;
      for (int64_t j = blockIdx.x; j < npieces; j += gridDim.x, ++n) {
        const int s = n % S;
        if (n >= S) mbar_wait(&empty[s], ((n / S) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], P);
        tma_load_1d(buf + (size_t)s * P, src + j * (int64_t)P, P, &full[s]);
      }
    }
    return;
  }
  int64_t n = 0;
  float acc = 0.f;
  for (int64_t j = blockIdx.x; j < npieces; j += gridDim.x, ++n) {
    const int s = n % S;
    mbar_wait(&full[s], (n / S) & 1);
    const uint4* v = reinterpret_cast<const uint4*>(buf + (size_t)s * P);
    uint4 x = v[tid % (P / 16)];
    acc += __uint_as_float(x.x);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (write_mode) {  // stream P bytes of zeros to dst (same volume as read)
      uint4* d = reinterpret_cast<uint4*>(dst + j * (int64_t)P);
      for (int i = tid; i < P / 16; i += 512) __stcs(d + i, make_uint4(0, 0, 0, 0));
    }
  }
  if (acc == 12345.f) dst[0] = 1;
}

int main() {
  const int64_t N = 2ll << 30;
  uint8_t *a, *b;
  cudaMalloc(&a, N); cudaMalloc(&b, N);
  cudaMemset(a, 1, N);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int cfg[][2] = {{3, 65536}, {2, 65536}, {6, 32768}, {12, 16384}, {4, 49152}, {16, 8192}};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wm = 0; wm < 2; ++wm)
    for (auto& c : cfg) {
      const int S = c[0], P = c[1];
      const size_t smem = 512 + (size_t)S * P;
      for (int it = 0; it < 2; ++it) ring<<<sms, 544, smem>>>(a, b, N, S, P, wm);
      cudaEventRecord(e0);
      const int R = 5;
      for (int it = 0; it < R; ++it) ring<<<sms, 544, smem>>>(a, b, N, S, P, wm);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= R;
      printf("write=%d stages=%2d piece=%6d : %.3f ms  read %.0f GB/s  total %.0f GB/s  (%s)\n", wm, S,
             P, ms, N / ms / 1e6, (wm + 1) * N / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
