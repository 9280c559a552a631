// umma_bench.cu -- diagnostic: tcgen05.mma (kind::f16, cta_group::1) issue-to-completion
// throughput on B200 for the shapes and operand sources the prefill kernels use (not part
// of libmoa).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2406_14909_b200/csrc/kernels \
//        -o tools/bin/umma_bench tools/umma_bench.cu
// One CTA per SM (148 CTAs, all SMs busy), one thread issues ITERS x 8 MMAs (K = 128 per
// group of 8) back to back into one TMEM accumulator, commits, waits; cycles / MMA and the
// chip TFLOP/s at the measured clock are printed.  Operands are zero tiles (timing only).
// Modes: SS (A, B from smem), TS (A from TMEM, B from smem); N in {64, 128, 256};
// optionally a second warp streams shared-memory reads (ld.shared.v4) alongside.
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

constexpr int ITERS = 256;

template <int N, bool TS, bool LDS_LOAD, int LDTM_LOAD = 0, bool BMN = false, int COMMIT_EVERY = 0>
__global__ void __launch_bounds__(192, 1) bench(long long *cycles, float *sink, const uint8_t *gsrc = nullptr) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init(smem_u32(&bar2), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(&tbase));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  // A: 128 x 128 bf16 (32 KB, 2 slabs), B: N x 128 bf16 (N*256 B) after it
  const uint32_t a_s = base, b_s = base + 32768;
  const uint64_t adesc = smem_desc_sw128(a_s, 16, 1024);
  // K-major B: LBO unused (16), SBO 1024; MN-major B (the PV's V tile): LBO = N-slab stride
  // (128 rows x 128 B per 64-column slab), SBO = 1024 (8 K-rows); K step of 16 rows = 2048 B
  const uint64_t bdesc = BMN ? smem_desc_sw128(b_s, 128 * 128, 1024) : smem_desc_sw128(b_s, 16, 1024);
  constexpr uint32_t idesc = idesc_bf16_f32(128, N, BMN);
  volatile uint32_t *flag = reinterpret_cast<volatile uint32_t *>(smem + 200000);
  if (threadIdx.x == 0) *flag = 0;
  __syncthreads();
  if (warp == 0) {
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          const uint32_t boff = BMN ? (kk * 2048) >> 4 : ((kk >> 2) * (N * 128) + (kk & 3) * 32) >> 4;
          if (TS)
            mma_ts(tmem + 0, tmem + 384 + kk * 8, bdesc + boff, idesc, (it | kk) ? 1u : 0u);
          else
            mma_ss(tmem + 0, adesc + off, bdesc + boff, idesc, (it | kk) ? 1u : 0u);
          if (COMMIT_EVERY && ((kk + 1) % COMMIT_EVERY) == 0) mma_commit(smem_u32(&bar2));
        }
      }
      mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      cycles[blockIdx.x] = t1 - t0;
      *flag = 1;
    }
  } else if (LDTM_LOAD == 2 && warp == 1) {
    // bulk copies global -> shared (32 KB chunks, 2 in flight) into [base+96K, base+160K) while the MMAs run
    __shared__ uint64_t cbar[2];
    if ((threadIdx.x & 31) == 0) {
      mbar_init(smem_u32(&cbar[0]), 1);
      mbar_init(smem_u32(&cbar[1]), 1);
      fence_mbar_init();
      long long n = 0, t0 = clock64();
      uint32_t ph[2] = {0, 0};
      const uint8_t *src = gsrc + (size_t)blockIdx.x * (1 << 20);
      for (int s2 = 0; s2 < 2; ++s2) {
        mbar_expect_tx(smem_u32(&cbar[s2]), 32768);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32768, [%2];" ::"r"(base + 98304 + s2 * 32768), "l"(src + s2 * 32768), "r"(smem_u32(&cbar[s2])) : "memory");
      }
      while (*flag == 0) {
        const int s2 = n & 1;
        mbar_wait(smem_u32(&cbar[s2]), ph[s2]);
        ph[s2] ^= 1;
        mbar_expect_tx(smem_u32(&cbar[s2]), 32768);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32768, [%2];" ::"r"(base + 98304 + s2 * 32768), "l"(src + ((n + 2) & 31) * 32768), "r"(smem_u32(&cbar[s2])) : "memory");
        ++n;
      }
      mbar_wait(smem_u32(&cbar[0]), ph[0]);
      mbar_wait(smem_u32(&cbar[1]), ph[1]);
      long long t1 = clock64();
      cycles[1024 + blockIdx.x] = n ? (t1 - t0) * 32768 / (n * 32768 / 64) : 0;  // cycles per 64 B... (reported as B/clk below)
      cycles[1024 + blockIdx.x] = n ? (n * 32768) / ((t1 - t0) / 64 + 1) : 0;
    }
  } else if (LDTM_LOAD == 1 && warp >= 1 && warp <= 4) {
    // warps 1-4 (lanes 32*(w%4)) stream TMEM loads of columns [256, 384) while the MMAs run
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256u;
    float acc = 0.f;
    long long n = 0, t0 = clock64();
    uint32_t r[128];
    while (*flag == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(base + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]));
      tmem_wait_ld();
      acc += __uint_as_float(r[3]) + __uint_as_float(r[77]);
      ++n;
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && warp == 1) cycles[1024 + blockIdx.x] = (t1 - t0) / (n ? n : 1);
    sink[blockIdx.x * 192 + threadIdx.x] = acc;
  } else if (LDS_LOAD && warp == 1) {
    float acc = 0.f;
    uint32_t a = base + (threadIdx.x & 31) * 16;
    while (*flag == 0) {
#pragma unroll 8
      for (int i = 0; i < 64; ++i) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a + (i & 63) * 512));
        acc += v.x;
      }
    }
    sink[blockIdx.x * 192 + threadIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// latency: GROUP MMAs (K=16 each) + commit, wait for the mbarrier, repeat REPS times
template <int GROUP, bool TS>
__global__ void __launch_bounds__(128, 1) lat(long long *cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(&tbase));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint64_t adesc = smem_desc_sw128(base, 16, 1024);
  const uint64_t bdesc = smem_desc_sw128(base + 32768, 16, 1024);
  constexpr uint32_t idesc = idesc_bf16_f32(128, 128, false);
  if (threadIdx.x == 0) {
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int r = 0; r < 64; ++r) {
#pragma unroll
      for (int kk = 0; kk < GROUP; ++kk) {
        const uint32_t off = (((kk & 7) >> 2) * 16384 + (kk & 3) * 32) >> 4;
        if (TS)
          mma_ts(tmem + 0, tmem + 384 + (kk & 7) * 8, bdesc + off, idesc, kk ? 1u : 0u);
        else
          mma_ss(tmem + 0, adesc + off, bdesc + off, idesc, kk ? 1u : 0u);
      }
      mma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), ph);
      ph ^= 1;
    }
    cycles[blockIdx.x] = (clock64() - t0) / 64;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// mixed stream like the prefill kernel's MMA warp: per iteration 8 x PV (TS, B MN-major, D=O)
// then 8 x S (SS, K-major, D=S), for two tiles (different D columns)
__global__ void __launch_bounds__(128, 1) mixed(long long *cycles, int variant) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(&tbase));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint64_t qdesc = smem_desc_sw128(base, 16, 1024);
  const uint64_t kdesc = smem_desc_sw128(base + 65536, 16, 1024);
  const uint64_t vdesc = smem_desc_sw128(base + 98304, 16384, 1024);
  constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, false);
  constexpr uint32_t idesc_o = idesc_bf16_f32(128, 128, true);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < 128; ++it) {
      for (int j = 0; j < 2; ++j) {
        if (variant != 1) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ts(tmem + 256 + 128 * j, tmem + 128 * j + kk * 8, vdesc + ((kk * 2048) >> 4), idesc_o, 1u);
        }
        if (variant != 2) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
            mma_ss(tmem + 128 * j, qdesc + ((j * 32768) >> 4) + off, kdesc + off, idesc_s, kk ? 1u : 0u);
          }
        }
      }
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

void run_mixed(long long *d_cyc, int nsm) {
  CK(cudaFuncSetAttribute(mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024));
  const char *names[3] = {"PV(TS,MN) + S(SS) x 2 tiles", "S(SS) only x 2 tiles", "PV(TS,MN) only x 2 tiles"};
  for (int v = 0; v < 3; ++v) {
    mixed<<<nsm, 128, 140 * 1024>>>(d_cyc, v);
    mixed<<<nsm, 128, 140 * 1024>>>(d_cyc, v);
    CK(cudaDeviceSynchronize());
    long long h;
    CK(cudaMemcpy(&h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost));
    const int n = 128 * 2 * (v == 0 ? 16 : 8);
    printf("mixed %-30s %6.1f cycles/MMA\n", names[v], (double)h / n);
  }
}

// issue-side costs seen by the issuing thread: 8 MMAs into an idle tensor core, a commit,
// a try_wait on an already-completed mbarrier, and the fence
__global__ void __launch_bounds__(128, 1) issue_cost(long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init(smem_u32(&bar2), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(&tbase));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint64_t adesc = smem_desc_sw128(base, 16, 1024);
  const uint64_t bdesc = smem_desc_sw128(base + 32768, 16, 1024);
  constexpr uint32_t idesc = idesc_bf16_f32(128, 128, false);
  if (threadIdx.x == 0) {
    long long acc[6] = {0, 0, 0, 0, 0, 0};
    uint32_t ph = 0;
    // complete bar2's phase 0 once (arrive), so waits on parity 0 are already satisfied
    mbar_arrive(smem_u32(&bar2));
    for (int r = 0; r < 32; ++r) {
      long long t0 = clock64();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
        mma_ss(tmem + 0, adesc + off, bdesc + off, idesc, kk ? 1u : 0u);
      }
      long long t1 = clock64();
      mma_commit(smem_u32(&bar));
      long long t2 = clock64();
      mbar_wait(smem_u32(&bar2), 0);  // already complete
      long long t3 = clock64();
      tc_fence_after();
      long long t4 = clock64();
      mbar_wait(smem_u32(&bar), ph);  // the MMAs
      ph ^= 1;
      long long t5 = clock64();
      acc[0] += t1 - t0;
      acc[1] += t2 - t1;
      acc[2] += t3 - t2;
      acc[3] += t4 - t3;
      acc[4] += t5 - t4;
    }
    for (int i = 0; i < 5; ++i) out[i] = acc[i] / 32;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

void run_issue_cost(long long *d_cyc) {
  CK(cudaFuncSetAttribute(issue_cost, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  issue_cost<<<1, 128, 100 * 1024>>>(d_cyc);
  issue_cost<<<1, 128, 100 * 1024>>>(d_cyc);
  CK(cudaDeviceSynchronize());
  long long h[5];
  CK(cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost));
  printf("issue cost (cycles): 8 MMAs into idle TC %lld | commit %lld | try_wait on completed bar %lld | fence %lld | wait for the MMAs %lld\n",
         h[0], h[1], h[2], h[3], h[4]);
}

template <int GROUP, bool TS>
void run_lat(long long *d_cyc, int nsm) {
  auto k = lat<GROUP, TS>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  k<<<nsm, 128, 100 * 1024>>>(d_cyc);
  k<<<nsm, 128, 100 * 1024>>>(d_cyc);
  CK(cudaDeviceSynchronize());
  long long h;
  CK(cudaMemcpy(&h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost));
  printf("latency: %2d x %s MMA(128x128x16) + commit + wait = %lld cycles (throughput floor %d)\n", GROUP,
         TS ? "TS" : "SS", h, GROUP * 64);
}

template <int N, bool TS, bool LDS, int LDTM = 0, bool BMN = false, int CE = 0>
void run(const char *name, long long *d_cyc, float *d_sink, int nsm, int clk_khz, const uint8_t *gsrc = nullptr) {
  auto k = bench<N, TS, LDS, LDTM, BMN, CE>;
  const int smem = 210 * 1024;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<nsm, 192, smem>>>(d_cyc, d_sink, gsrc);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024];
    CK(cudaMemcpy(h, d_cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int i = 0; i < nsm; ++i) avg += h[i];
    avg /= nsm;
    const double n_mma = ITERS * 8.0;
    const double flops = 2.0 * 128 * N * 16 * n_mma * nsm;
    long long l = 0;
    if (LDTM) CK(cudaMemcpy(&l, d_cyc + 1024, sizeof(long long), cudaMemcpyDeviceToHost));
    if (rep == 1)
      printf("%-28s N=%3d  %7.1f cycles/MMA (floor %5.1f)  kernel %.3f ms  %7.1f TFLOP/s  side: %lld\n", name,
             N, avg / n_mma, 128.0 * N / 256.0, ms, flops / (ms * 1e-3) / 1e12, l);
  }
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  long long *d_cyc;
  float *d_sink;
  CK(cudaMalloc(&d_cyc, 2048 * sizeof(long long)));
  CK(cudaMalloc(&d_sink, 1024 * 192 * sizeof(float)));
  run<64, false, false>("SS", d_cyc, d_sink, nsm, clk);
  run<128, false, false>("SS", d_cyc, d_sink, nsm, clk);
  run<256, false, false>("SS", d_cyc, d_sink, nsm, clk);
  run<64, true, false>("TS", d_cyc, d_sink, nsm, clk);
  run<128, true, false>("TS", d_cyc, d_sink, nsm, clk);
  run<256, true, false>("TS", d_cyc, d_sink, nsm, clk);
  run<128, false, true>("SS + ld.shared stream", d_cyc, d_sink, nsm, clk);
  run<128, true, true>("TS + ld.shared stream", d_cyc, d_sink, nsm, clk);
  run<128, true, false, 1>("TS + 4 warps LDTM stream", d_cyc, d_sink, nsm, clk);
  run<128, false, false, 1>("SS + 4 warps LDTM stream", d_cyc, d_sink, nsm, clk);
  uint8_t *g;
  CK(cudaMalloc(&g, (size_t)nsm << 20));
  CK(cudaMemset(g, 0, (size_t)nsm << 20));
  run<128, false, false, 2>("SS + bulk copy stream", d_cyc, d_sink, nsm, clk, g);
  run<128, true, false, 2>("TS + bulk copy stream", d_cyc, d_sink, nsm, clk, g);
  run<256, false, false, 2>("SS + bulk copy stream", d_cyc, d_sink, nsm, clk, g);
  run<128, true, false, 0, true>("TS, B MN-major (PV)", d_cyc, d_sink, nsm, clk);
  run<128, false, false, 0, true>("SS, B MN-major", d_cyc, d_sink, nsm, clk);
  run<64, true, false, 0, true>("TS, B MN-major", d_cyc, d_sink, nsm, clk);
  run_issue_cost(d_cyc);
  run_mixed(d_cyc, nsm);
  run_lat<1, false>(d_cyc, nsm);
  run_lat<8, false>(d_cyc, nsm);
  run_lat<16, false>(d_cyc, nsm);
  run_lat<8, true>(d_cyc, nsm);
  run<128, false, false, 0, false, 8>("SS, commit every 8", d_cyc, d_sink, nsm, clk);
  run<128, false, false, 0, false, 4>("SS, commit every 4", d_cyc, d_sink, nsm, clk);
  run<128, false, false, 0, false, 1>("SS, commit every 1", d_cyc, d_sink, nsm, clk);
  return 0;
}
