// exp_bench.cu -- diagnostic: exp2 throughput on B200 per SM: MUFU ex2.approx.ftz.f32 versus
// the packed-f32x2 degree-3 polynomial of prefill_pp.cu (not part of libmoa).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/exp_bench tools/exp_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int ITERS = 2048;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint64_t f2pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2upk(uint64_t r, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ void poly2(float ya, float yb, float &ra, float &rb) {
  const uint64_t y = f2pk(fmaxf(ya, -126.f), fmaxf(yb, -126.f));
  const uint64_t t = fadd2(y, f2pk(12582912.f, 12582912.f));
  const uint64_t n = fadd2(t, f2pk(-12582912.f, -12582912.f));
  const uint64_t f = ffma2(n, f2pk(-1.f, -1.f), y);
  uint64_t q = ffma2(f, f2pk(0.0550887f, 0.0550887f), f2pk(0.2426041f, 0.2426041f));
  q = ffma2(q, f, f2pk(0.6932762f, 0.6932762f));
  q = ffma2(q, f, f2pk(0.9999289f, 0.9999289f));
  float qa, qb, ta, tb;
  f2upk(q, qa, qb);
  f2upk(t, ta, tb);
  ra = __int_as_float(__float_as_int(qa) + (__float_as_int(ta) << 23));
  rb = __int_as_float(__float_as_int(qb) + (__float_as_int(tb) << 23));
}

template <int MODE>  // 0 MUFU, 1 poly, 2 3:1 mix
__global__ void bench(float *out, long long *cyc) {
  float x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      if (MODE == 0 || (MODE == 2 && (i & 6) != 6)) {
        x[i] = ex2(x[i]) - 1.0f;
        x[i + 1] = ex2(x[i + 1]) - 1.0f;
      } else {
        float a, b;
        poly2(x[i], x[i + 1], a, b);
        x[i] = a - 1.0f;
        x[i + 1] = b - 1.0f;
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char *name, int warps, float *d, long long *c, int nsm) {
  bench<MODE><<<nsm, warps * 32>>>(d, c);
  bench<MODE><<<nsm, warps * 32>>>(d, c);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, c, nsm * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  const double exps = (double)ITERS * 32 * warps * 32;
  printf("%-10s warps/SM=%2d  %6.2f exp/clk/SM   (%.1f cycles per warp-instruction-equivalent of 32 exps)\n", name,
         warps, exps / avg, avg / (ITERS * 32.0 * warps) * 1.0);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float *d;
  long long *c;
  cudaMalloc(&d, 1024 * 1024 * 4);
  cudaMalloc(&c, 1024 * 8);
  for (int w : {4, 8, 16}) run<0>("MUFU ex2", w, d, c, nsm);
  for (int w : {4, 8, 16}) run<1>("poly", w, d, c, nsm);
  for (int w : {4, 8, 16}) run<2>("3:1 mix", w, d, c, nsm);
  return 0;
}
