// tma_bench.cu -- diagnostic: TMA tile-stream throughput on B200 (not part of libmoa).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench tools/tma_bench.cu -lcuda
// Streams 128-row x 128-col bf16 tiles of a [B, N, H, 128] tensor (the prefill K/V layout)
// into a shared-memory ring with cp.async.bulk.tensor (128B swizzle), consumer releases at
// once.  Reports GB/s for several ring depths, box shapes and tile reuse patterns.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint32_t b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma4(uint32_t dst, const CUtensorMap *m, uint32_t bar, int a, int b, int c, int d) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2,%3,%4,%5}], [%6];"
               ::"r"(dst), "l"((uint64_t)m), "r"(a), "r"(b), "r"(c), "r"(d), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma5(uint32_t dst, const CUtensorMap *m, uint32_t bar, int a, int b, int c, int d, int e) {
  asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2,%3,%4,%5,%6}], [%7];"
               ::"r"(dst), "l"((uint64_t)m), "r"(a), "r"(b), "r"(c), "r"(d), "r"(e), "r"(bar) : "memory");
}

template <int NS, bool FIVE>
__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap m, int tiles_per_cta, int ntiles_n, int H, int reuse) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t full[NS], empty[NS];
  const uint32_t base = (su32(sm) + 1023) & ~1023u;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) { mbar_init(su32(&full[i]), 1); mbar_init(su32(&empty[i]), 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (w == 0 && l == 0) {
    for (int t = 0; t < tiles_per_cta; ++t) {
      const int s = t % NS;
      if (t >= NS) mbar_wait(su32(&empty[s]), ((t - NS) / NS) & 1);
      mbar_expect(su32(&full[s]), 32768);
      // tile id: reuse>1 makes groups of `reuse` consecutive CTAs walk the same tiles (L2 hits)
      const int g = (blockIdx.x / reuse) * tiles_per_cta + t;
      const int tn = g % ntiles_n, h = (g / ntiles_n) % H, b = g / (ntiles_n * H);
      const uint32_t dst = base + s * 32768;
      if (FIVE) tma5(dst, &m, su32(&full[s]), 0, tn * 128, 0, h, b);
      else { tma4(dst, &m, su32(&full[s]), 0, h, tn * 128, b); tma4(dst + 16384, &m, su32(&full[s]), 64, h, tn * 128, b); }
    }
  } else if (w == 1 && l == 0) {
    for (int t = 0; t < tiles_per_cta; ++t) { const int s = t % NS; mbar_wait(su32(&full[s]), (t / NS) & 1); mbar_arrive(su32(&empty[s])); }
  }
}

int main() {
  const int B = 8, N = 4096, H = 32, D = 128;
  const size_t elems = (size_t)B * N * H * D;
  void *buf; CK(cudaMalloc(&buf, elems * 2)); CK(cudaMemset(buf, 0, elems * 2));
  void *fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m4, m5;
  { cuuint64_t dims[4] = {D, H, N, B}; cuuint64_t st[3] = {D * 2, (cuuint64_t)H * D * 2, (cuuint64_t)N * H * D * 2};
    cuuint32_t box[4] = {64, 1, 128, 1}, es[4] = {1, 1, 1, 1};
    if (enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc4 fail\n"); return 1; } }
  { // (64 elems, N rows, 2 halves, H, B): one instruction loads both 128-byte slabs of a tile
    cuuint64_t dims[5] = {64, (cuuint64_t)N, 2, (cuuint64_t)H, B};
    cuuint64_t st[4] = {(cuuint64_t)H * D * 2, 128, D * 2, (cuuint64_t)N * H * D * 2};
    cuuint32_t box[5] = {64, 128, 2, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    if (enc(&m5, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, buf, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc5 fail\n"); return 1; } }
  const int ctas = 148, per = 400;
  auto run = [&](auto kern, int ns, int reuse, const char *name) {
    const int smem = ns * 32768 + 1024;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<ctas, 64, smem>>>(m4, per, N / 128, H, reuse); CK(cudaDeviceSynchronize());
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kern<<<ctas, 64, smem>>>(name[0] == '5' ? m5 : m4, per, N / 128, H, reuse);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-28s stages=%d reuse=%3d  %8.1f GB/s (SM->smem)\n", name, ns, reuse, 5.0 * ctas * per * 32768.0 / (ms * 1e6));
  };
  for (int reuse : {1, 8, 148}) {
    run(stream<2, false>, 2, reuse, "4d two-box");
    run(stream<4, false>, 4, reuse, "4d two-box");
    run(stream<6, false>, 6, reuse, "4d two-box");
    run(stream<2, true>, 2, reuse, "5d one-box");
    run(stream<4, true>, 4, reuse, "5d one-box");
    run(stream<6, true>, 6, reuse, "5d one-box");
  }
  return 0;
}
