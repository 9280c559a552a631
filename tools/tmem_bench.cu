// tmem_bench.cu -- diagnostic: tcgen05.ld / tcgen05.st throughput (TMEM <-> registers) on
// B200 with 4, 8 or 16 warps per CTA, one CTA per SM (not part of libmoa).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2406_14909_b200/csrc/kernels \
//        -o tools/bin/tmem_bench tools/tmem_bench.cu
// Each warp reads (or writes) its 32 TMEM lanes x 128 columns (16 KB) per iteration with the
// 32x32b shape (x32 / x64 / x128 repeats) and waits; cycles per 64 KB (= one 128 x 128 fp32
// S tile) per SM are printed.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ptx_sm100.cuh"

using namespace moa::ptx;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                    \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

constexpr int ITERS = 512;

template <int REP>
__device__ __forceinline__ void ld_rep(uint32_t taddr, uint32_t *r);

template <>
__device__ __forceinline__ void ld_rep<32>(uint32_t taddr, uint32_t *r) {
  tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
}

template <int MODE>  // 0: ld x32 x4, 1: ld with wait after each x32, 2: st x32 x4
__global__ void bench(long long *cycles, float *sink, int nwarps_used) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(smem_u32(&tbase));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  // warp w: lanes 32*(w%4); column block (w/4) * 128 (up to 4 blocks of 128 columns)
  const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
  float acc = 0.f;
  uint32_t r[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) r[i] = i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(base + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]));
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 128; i += 16) acc += __uint_as_float(r[i]);
    } else if (MODE == 1) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(base + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]));
        tmem_wait_ld();
      }
#pragma unroll
      for (int i = 0; i < 128; i += 16) acc += __uint_as_float(r[i]);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st32(base + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]));
      tmem_wait_st();
      r[it & 127] += 1;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + (float)r[5];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
void run(const char *name, int nwarps, long long *d_cyc, float *d_sink, int nsm) {
  for (int rep = 0; rep < 2; ++rep) {
    bench<MODE><<<nsm, nwarps * 32>>>(d_cyc, d_sink, nwarps);
    CK(cudaDeviceSynchronize());
  }
  long long h[1024];
  CK(cudaMemcpy(h, d_cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  const double bytes_per_iter = nwarps * 32.0 * 128 * 4;  // per SM
  printf("%-34s warps=%2d  %8.1f cycles/iter  %6.1f B/cycle/SM  %7.1f cycles per 64 KB\n", name, nwarps,
         avg / ITERS, bytes_per_iter / (avg / ITERS), (avg / ITERS) * 65536.0 / bytes_per_iter);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *d_cyc;
  float *d_sink;
  CK(cudaMalloc(&d_cyc, 1024 * sizeof(long long)));
  CK(cudaMalloc(&d_sink, 1024 * 1024 * sizeof(float)));
  for (int w : {4, 8, 16}) run<0>("ld 32x32b.x32 x4, one wait", w, d_cyc, d_sink, nsm);
  for (int w : {4, 8, 16}) run<1>("ld 32x32b.x32, wait each", w, d_cyc, d_sink, nsm);
  for (int w : {4, 8, 16}) run<2>("st 32x32b.x32 x4, one wait", w, d_cyc, d_sink, nsm);
  return 0;
}
