// influence.cu -- block-averaged attention influence of the MoA profiling stage
// (Eq. 3, derivation PAPER.md:1361-1405).
//
// For one calibration item and every (batch, q-head), with dense causal attention
// (the profiled model is unmasked):
//   A   = softmax(tau Q K^T + causal)                         (Eq. 1)
//   G   = dL/dA = dO V^T                                       (O = A V, chain rule)
//   E_ij = -A_ij / (1 - A_ij) * (G_ij - R_i),  R_i = sum_n G_in A_in   (Eq. 3, last line
//          of the derivation; E = 0 where A_ij = 1, the row's only visible key)
//   out[b, h, ib, jb] (+)= mean of E over the block x block token pairs
//
// One CTA per (64-row query block, q-head, batch), 4 warps x 16 rows.  QK^T and dO V^T
// run on the tensor cores (mma.sync m16n8k16, bf16 in, fp32 accumulate); K/V blocks are
// staged in padded shared memory.  Pass 1 walks the causal key blocks once for the row
// statistics (online max m and the sums l = sum 2^(S-m), u = sum G 2^(S-m) kept as
// "star key + rest" so that 1 - A and R - G are formed without cancellation when a row
// is nearly one-hot), pass 2 recomputes S and G per key block, forms E and reduces it to the
// block mean.  The kernel never materialises A, G or E in memory.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../moa_internal.h"
#include "common.cuh"

namespace moa {
namespace {

constexpr int kB = 64;        // query / key block (the paper's 64)
constexpr int kThreadsInf = 128;

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t smem_u32i(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

template <int D>
struct InfSmem {
  static constexpr int kStride = D + 8;  // bf16 elements per padded row: conflict-free ldmatrix rows
  static constexpr int kBuf = kB * kStride;                       // one K or V block (elements)
  static constexpr int kBytes = 2 * 2 * kBuf * 2;                 // K, V x 2 stages, bf16
};

// S (16 rows x 64 keys) = Q K^T and G = dO V^T for this warp's rows, from the staged block.
template <int D>
__device__ __forceinline__ void block_products(const __nv_bfloat16 *ks, const __nv_bfloat16 *vs,
                                               const uint32_t (&qa)[D / 16][4],
                                               const uint32_t (&da)[D / 16][4], int lane, float (&S)[8][4],
                                               float (&G)[8][4]) {
#pragma unroll
  for (int n = 0; n < 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) S[n][e] = G[n][e] = 0.f;
  // ldmatrix.x4: lanes 8m..8m+7 address rows (keys) of 8x8 matrix m = (n-tile n0 + (m >> 1),
  // dims kk*16 + 8 (m & 1)); registers r0..r3 = b0, b1 of n-tile n0 and of n-tile n0 + 1
  const int mrow = lane & 7, msel = lane >> 3;
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
    for (int n = 0; n < 8; n += 2) {
      const int key = (n + (msel >> 1)) * 8 + mrow;
      const int col = kk * 16 + (msel & 1) * 8;
      uint32_t kb[4], vb[4];
      ldsm_x4(kb, smem_u32i(&ks[key * InfSmem<D>::kStride + col]));
      ldsm_x4(vb, smem_u32i(&vs[key * InfSmem<D>::kStride + col]));
      mma16816(S[n], qa[kk], kb[0], kb[1]);
      mma16816(S[n + 1], qa[kk], kb[2], kb[3]);
      mma16816(G[n], da[kk], vb[0], vb[1]);
      mma16816(G[n + 1], da[kk], vb[2], vb[3]);
    }
  }
}

template <int D>
#ifndef MOA_INF_HEAD_MAJOR
#define MOA_INF_HEAD_MAJOR 1  // heaviest blocks of all heads in the first waves: 161.9 vs 148.7 TFLOP/s (N=8k)
#endif
#ifndef MOA_INF_MIN_BLOCKS
#define MOA_INF_MIN_BLOCKS 3  // 3 CTAs (12 warps) per SM: 148.8 vs 127.9 TFLOP/s at 1 (180 regs, 2 CTAs), 105 at 4 (spills)
#endif
__global__ void __launch_bounds__(kThreadsInf, MOA_INF_MIN_BLOCKS) influence_kernel(InfluenceArgs a) {
  extern __shared__ __align__(16) uint8_t inf_dsm[];
  __nv_bfloat16 *kv_s = reinterpret_cast<__nv_bfloat16 *>(inf_dsm);  // [stage][K | V][kBuf]
  __shared__ float red[4];
  const int nb = (int)((a.N + kB - 1) / kB);
#if MOA_INF_HEAD_MAJOR
  // grid (heads, blocks, batch): the first waves hold the heaviest blocks of EVERY head
  const int ib = nb - 1 - (int)blockIdx.y;  // heaviest (longest causal row) blocks first
  const int h = blockIdx.x, b = blockIdx.z;
#else
  const int ib = nb - 1 - (int)blockIdx.x;  // heaviest (longest causal row) blocks first
  const int h = blockIdx.y, b = blockIdx.z;
#endif
  const int gkv = h / a.G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t N = a.N;
  const int64_t r0 = (int64_t)ib * kB + warp * 16 + g, r1 = r0 + 8;  // this thread's two rows
  const __nv_bfloat16 *Q = static_cast<const __nv_bfloat16 *>(a.q);
  const __nv_bfloat16 *dO = static_cast<const __nv_bfloat16 *>(a.dout);
  const __nv_bfloat16 *K = static_cast<const __nv_bfloat16 *>(a.k);
  const __nv_bfloat16 *V = static_cast<const __nv_bfloat16 *>(a.v);

  // A fragments of Q and dO for this warp's 16 rows (rows >= N read as 0)
  uint32_t qa[D / 16][4], da[D / 16][4];
  {
    auto ld = [&](const __nv_bfloat16 *X, int64_t stride, int64_t r, int col) -> uint32_t {
      if (r >= N) return 0u;
      return *reinterpret_cast<const uint32_t *>(X + ((int64_t)b * N + r) * stride + (int64_t)h * D + col);
    };
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int c = kk * 16 + 2 * t;
      qa[kk][0] = ld(Q, a.q_row_stride, r0, c);
      qa[kk][1] = ld(Q, a.q_row_stride, r1, c);
      qa[kk][2] = ld(Q, a.q_row_stride, r0, c + 8);
      qa[kk][3] = ld(Q, a.q_row_stride, r1, c + 8);
      da[kk][0] = ld(dO, a.q_row_stride, r0, c);
      da[kk][1] = ld(dO, a.q_row_stride, r1, c);
      da[kk][2] = ld(dO, a.q_row_stride, r0, c + 8);
      da[kk][3] = ld(dO, a.q_row_stride, r1, c + 8);
    }
  }
  // K/V block jb -> stage buf, 16-byte cp.async (zero fill past N); double-buffered: block
  // jb+1 streams in while block jb is computed
  auto stage_async = [&](int jb, int buf) {
    constexpr int kVec = D / 8;  // 16-byte vectors per row
    __nv_bfloat16 *kd = kv_s + (size_t)buf * 2 * InfSmem<D>::kBuf, *vd = kd + InfSmem<D>::kBuf;
    for (int idx = threadIdx.x; idx < kB * kVec; idx += kThreadsInf) {
      const int r = idx / kVec, c = (idx - r * kVec) * 8;
      const int64_t j = (int64_t)jb * kB + r;
      const int64_t off = ((int64_t)b * N + (j < N ? j : N - 1)) * a.kv_row_stride + (int64_t)gkv * D + c;
      const uint32_t bytes = j < N ? 16u : 0u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32i(&kd[r * InfSmem<D>::kStride + c])),
                   "l"(K + off), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32i(&vd[r * InfSmem<D>::kStride + c])),
                   "l"(V + off), "r"(bytes)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto pass_block = [&](int jb) -> int {  // wait for block jb (prefetch jb+1 first); its stage
    if (jb + 1 <= ib) stage_async(jb + 1, (jb + 1) & 1);
    if (jb + 1 <= ib)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    else
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    return jb & 1;
  };
  auto kbuf = [&](int buf) { return kv_s + (size_t)buf * 2 * InfSmem<D>::kBuf; };
  const float sl2 = a.scale * kLog2e;  // scores in log2 units
  float S[8][4], G[8][4];

  // ---- pass 1: row statistics over the causal key blocks 0..ib.  With p_k = 2^(S_k - m)
  // (m = the row max, in log2 units) the row is kept as l = 1 + Lr and u = sum G p = Gs + Ur,
  // where key js (the first key attaining m, G_js = Gs) is split off: 1 - A_js = Lr / l and
  // R - G_js = (Ur - Gs Lr) / l are then formed without cancellation when A_js -> 1.
  float m[2] = {-INFINITY, -INFINITY}, Lr[2] = {0.f, 0.f}, Ur[2] = {0.f, 0.f}, Gs[2] = {0.f, 0.f};
  int js[2] = {-1, -1};
  stage_async(0, 0);
  for (int jb = 0; jb <= ib; ++jb) {
    const int buf = pass_block(jb);
    block_products<D>(kbuf(buf), kbuf(buf) + InfSmem<D>::kBuf, qa, da, lane, S, G);
    __syncthreads();  // every warp has read the stage before it is refilled (block jb+2)
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int64_t i = rr ? r1 : r0;
      float mx = -INFINITY;
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t j = (int64_t)jb * kB + n * 8 + 2 * t + e;
          if (j <= i) mx = fmaxf(mx, S[n][2 * rr + e] * sl2);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      // (every row sees key jb*64 <= i, so mx is finite; rows >= N run on zero Q and are
      // dropped in pass 2; no early exit: the quad shuffles below need every lane)
      // the block's star key: smallest index attaining mx, and its G
      int jstar = 0x7fffffff;
      float gstar = 0.f;
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jl = jb * kB + n * 8 + 2 * t + e;
          if (jl <= i && S[n][2 * rr + e] * sl2 == mx && jl < jstar) {
            jstar = jl;
            gstar = G[n][2 * rr + e];
          }
        }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        const int jo = __shfl_xor_sync(0xffffffffu, jstar, o);
        const float go = __shfl_xor_sync(0xffffffffu, gstar, o);
        if (jo < jstar) jstar = jo, gstar = go;
      }
      float rs = 0.f, us = 0.f;  // the block's keys other than its star, in units 2^(S - mx)
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jl = jb * kB + n * 8 + 2 * t + e;
          if (jl <= i && jl != jstar) {
            const float pp = exp2f(S[n][2 * rr + e] * sl2 - mx);
            rs += pp;
            us += pp * G[n][2 * rr + e];
          }
        }
      rs += __shfl_xor_sync(0xffffffffu, rs, 1);
      rs += __shfl_xor_sync(0xffffffffu, rs, 2);
      us += __shfl_xor_sync(0xffffffffu, us, 1);
      us += __shfl_xor_sync(0xffffffffu, us, 2);
      if (mx == -INFINITY) {
      } else if (mx > m[rr]) {  // the block holds the new row max: the old row (star included) joins the rest
        const float alpha = exp2f(m[rr] - mx);  // 0 for the first block
        Lr[rr] = (js[rr] >= 0 ? (1.f + Lr[rr]) * alpha : 0.f) + rs;
        Ur[rr] = (js[rr] >= 0 ? (Gs[rr] + Ur[rr]) * alpha : 0.f) + us;
        m[rr] = mx;
        js[rr] = jstar;
        Gs[rr] = gstar;
      } else {  // every key of the block joins the rest (a tie with the row max counts 1)
        const float beta = exp2f(mx - m[rr]);
        Lr[rr] += (1.f + rs) * beta;
        Ur[rr] += (gstar + us) * beta;
      }
    }
  }
  float l[2], inv_l[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    l[rr] = 1.f + Lr[rr];
    inv_l[rr] = 1.f / l[rr];
  }

  // ---- pass 2: E per key block, reduced to the block mean
  float *out = a.e_blocks + (((int64_t)b * a.nql + h) * nb + ib) * nb;
  const int64_t rows_real = (N - (int64_t)ib * kB) < kB ? N - (int64_t)ib * kB : kB;
  stage_async(0, 0);
  for (int jb = 0; jb <= ib; ++jb) {
    const int buf = pass_block(jb);
    block_products<D>(kbuf(buf), kbuf(buf) + InfSmem<D>::kBuf, qa, da, lane, S, G);
    float acc = 0.f;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int64_t i = rr ? r1 : r0;
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jl = jb * kB + n * 8 + 2 * t + e;
          if (jl <= i && i < N) {
            const float g = G[n][2 * rr + e];
            float E;
            if (jl == js[rr]) {
              // A/(1-A) = 1/Lr, R - G = (Ur - Gs Lr)/l; a row with one visible key: E = 0
              E = Lr[rr] > 0.f ? (Ur[rr] - Gs[rr] * Lr[rr]) / (Lr[rr] * l[rr]) : 0.f;
            } else {
              const float pp = exp2f(S[n][2 * rr + e] * sl2 - m[rr]);
              // A/(1-A) = p/(l-p), R - G = ((Gs - g) + (Ur - g Lr))/l
              E = __fdividef(pp, 1.f + (Lr[rr] - pp)) * ((Gs[rr] - g) + (Ur[rr] - g * Lr[rr])) * inv_l[rr];
            }
            acc += E;
          }
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t cols_real = (N - (int64_t)jb * kB) < kB ? N - (int64_t)jb * kB : kB;
      const float mean = (red[0] + red[1] + red[2] + red[3]) / (float)(rows_real * cols_real);
      out[jb] = a.accumulate ? out[jb] + mean : mean;
    }
    __syncthreads();  // red and the stage are reused by the next block
  }
  if (!a.accumulate)
    for (int jb = ib + 1 + (int)threadIdx.x; jb < nb; jb += kThreadsInf) out[jb] = 0.f;  // no causal pairs
}

}  // namespace

int launch_influence(const InfluenceArgs &a, void *stream) {
  const int nb = (int)((a.N + kB - 1) / kB);
#if MOA_INF_HEAD_MAJOR
  dim3 grid((unsigned)a.nql, (unsigned)nb, (unsigned)a.batch);
#else
  dim3 grid((unsigned)nb, (unsigned)a.nql, (unsigned)a.batch);
#endif
  if (a.d == 128) {
    cudaError_t e = cudaFuncSetAttribute(influence_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         InfSmem<128>::kBytes);
    if (e != cudaSuccess) return (int)e;
    influence_kernel<128><<<grid, kThreadsInf, InfSmem<128>::kBytes, (cudaStream_t)stream>>>(a);
  } else {
    cudaError_t e = cudaFuncSetAttribute(influence_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         InfSmem<64>::kBytes);
    if (e != cudaSuccess) return (int)e;
    influence_kernel<64><<<grid, kThreadsInf, InfSmem<64>::kBytes, (cudaStream_t)stream>>>(a);
  }
  return (int)cudaGetLastError();
}

}  // namespace moa

namespace moa {
namespace {

// ---- Eq. 4: rule losses from the block-averaged influence.
// One CTA per (rule, head).  For query block ib the masked key blocks of the block mask are
// sb <= jb <= ib - wb (sb = sink blocks, wb = window blocks; the whole causal row when the
// window is 0 and ib >= sb); each contributes its mean times its pair count.
__global__ void __launch_bounds__(256) rule_loss_kernel(const float *__restrict__ e_blocks, int nb, int64_t N,
                                                        int block, const RuleWindows win, int sink_blocks,
                                                        int n_rules, float *__restrict__ loss) {
  const int r = blockIdx.x, h = blockIdx.y;
  const int wb = win.blocks[r];
  const float *E = e_blocks + (int64_t)h * nb * nb;
  double acc = 0.0;
  for (int ib = threadIdx.x; ib < nb; ib += blockDim.x) {
    const int64_t rows = N - (int64_t)ib * block < block ? N - (int64_t)ib * block : block;
    const int hi = ib - wb;  // last masked key block (inclusive)
    double row = 0.0;
    for (int jb = sink_blocks; jb <= hi; ++jb) {
      const int64_t cols = N - (int64_t)jb * block < block ? N - (int64_t)jb * block : block;
      row += (double)E[(int64_t)ib * nb + jb] * (double)cols;
    }
    acc += row * (double)rows;
  }
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[(int64_t)h * n_rules + r] = (float)red[0];
}

}  // namespace

int launch_rule_losses(const float *e_blocks, int heads, int64_t N, int block, const RuleWindows &win,
                       int sink_blocks, int n_rules, float *loss, void *stream) {
  const int nb = (int)((N + block - 1) / block);
  dim3 grid((unsigned)n_rules, (unsigned)heads);
  rule_loss_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(e_blocks, nb, N, block, win, sink_blocks, n_rules,
                                                          loss);
  return (int)cudaGetLastError();
}

}  // namespace moa
