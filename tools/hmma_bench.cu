// hmma_bench.cu -- peak rate of the legacy warp-level mma.sync m16n8k16 (bf16 in, fp32 acc)
// on this GPU: the roofline denominator of the influence kernel (kernels/influence.cu), which
// runs on mma.sync rather than tcgen05.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/hmma_bench tools/hmma_bench.cu
//   tools/bin/hmma_bench
//
// Every warp runs CH independent accumulator chains of ITERS mma.sync each (operands in
// registers, no memory traffic); TFLOP/s = 2*16*8*16 * mmas / time, CUDA events.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void hmma_kernel(float *out, int iters) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x * 2654435761u + i);
  for (int i = 0; i < 2; ++i) b[i] = 0x3c003c00u ^ (threadIdx.x * 40503u + i);
  float c[CH][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
  for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.f) out[threadIdx.x] = s;  // keep the chains alive
}

template <int CH>
void run(int warps_per_cta, int ctas_per_sm, int sms) {
  const int iters = 4096;
  float *out;
  cudaMalloc(&out, 4096);
  dim3 grid(sms * ctas_per_sm), block(32 * warps_per_cta);
  hmma_kernel<CH><<<grid, block>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  hmma_kernel<CH><<<grid, block>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = (double)grid.x * warps_per_cta * CH * iters;
  printf("chains %d  warps/CTA %2d  CTAs/SM %d : %.1f TFLOP/s\n", CH, warps_per_cta, ctas_per_sm,
         mmas * 2.0 * 16 * 8 * 16 / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4>(4, 1, sms);
  run<4>(4, 3, sms);
  run<8>(4, 3, sms);
  run<8>(8, 2, sms);
  run<8>(16, 1, sms);
  run<12>(16, 1, sms);
  run<16>(16, 2, sms);
  return 0;
}
