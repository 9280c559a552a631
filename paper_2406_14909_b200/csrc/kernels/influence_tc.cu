// influence_tc.cu -- block-averaged attention influence of the MoA profiling stage on the
// sm_100a tensor cores (tcgen05 + TMEM + TMA) (Eq. 3 PAPER.md:225-236,
// derivation PAPER.md:1361-1405, block averaging PAPER.md:691).
//
// For one calibration item and every (batch, q-head), with dense causal attention (the
// profiled model is unmasked):
//   A    = softmax(tau Q K^T + causal)                              (Eq. 1)
//   G    = dL/dA = dO V^T                                           (O = A V, chain rule)
//   E_ij = A_ij (R_i - G_ij) / (1 - A_ij),  R_i = sum_n G_in A_in   (Eq. 3: -A_ij G_ij +
//          sum_{n != j} G_in A_in A_ij / (1 - A_ij); E = 0 where A_ij = 1, a row's only key)
//   out[b, h, ib, jb] (+)= mean of E over the 64 x 64 token pairs of block (ib, jb)
//
// Work item = 256 query rows of one (batch, q-head): q tiles j = 0, 1 of 128 rows, processed
// in two passes over the causal key tiles of 64 keys (one kv tile = one key block):
//   pass 0  row statistics: m = max_k tau s_k (log2 units); the first key attaining it (the
//           "star", js, with G_js = Gs) is kept out of the sums, Lr = sum_{k != js} 2^(x_k - m)
//           and Ur = sum_{k != js} G_k 2^(x_k - m), so l = 1 + Lr and R = (Gs + Ur) / l, and
//           1 - A_js = Lr / l, R - G_js = (Ur - Gs Lr) / l keep fp32 accuracy on rows that are
//           nearly one-hot (a sink-dominated row) where 1 - A in fp32 would cancel;
//   pass 1  E_ij = p (C1 - G_ij l) / ((l - p) l) with p = 2^(x_ij - m), C1 = Gs + Ur (the star:
//           E = (Ur - Gs Lr) / (Lr l)), summed per row over the tile, then over the 64 rows
//           of a block: one block mean per (row block, kv tile).
// Per kv tile and q tile the tensor core computes S = Q K^T and G = dO V^T (two SS MMAs,
// M = 128, N = 64, into TMEM, double-buffered); the elementwise warps read their row of S and
// G (thread = row = TMEM lane) and never touch A, G or E in memory.
//
// Warps (320 threads, one CTA per SM, persistent over items in LPT order):
//   0-3  elementwise, q tile 0      4-7  elementwise, q tile 1
//   8    TMA producer (Q, dO tiles per item; K, V tiles per step, both passes)
//   9    TMEM allocator + MMA issue (one elected lane)
// The two q tiles share every K/V tile, and while one tile's warps are in their elementwise
// work the tensor core computes the other tile's products.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../moa_internal.h"
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace moa {
namespace {

using namespace ptx;

constexpr int kIM = 128;        // q rows per tile (MMA M)
constexpr int kIN = 64;         // keys per kv tile (MMA N) = the paper's block
constexpr int kIThreads = 320;
constexpr int kWTma = 8, kWMma = 9;
#ifndef MOA_INF_KV_STAGES
#define MOA_INF_KV_STAGES 3
#endif
constexpr int kKVStages = MOA_INF_KV_STAGES;
constexpr uint32_t kITmemCols = 512;  // [tile j][buffer u]: S (64 cols) | G (64 cols)

template <int D>
struct ICfg {
  static constexpr int kSlabs = D / 64;
  static constexpr int kQTile = kIM * D * 2;  // Q or dO tile bytes
  static constexpr int kQSlab = kIM * 128;
  static constexpr int kKTile = kIN * D * 2;  // K or V tile bytes
  static constexpr int kKSlab = kIN * 128;
  static constexpr int kSmem = 4 * kQTile + kKVStages * 2 * kKTile;  // Q0 dO0 Q1 dO1 | stages (K V)
};

struct IBars {
  uint64_t q_full[2], q_empty[2];
  uint64_t kv_full[kKVStages], kv_empty[kKVStages];
  uint64_t s_full[2][2], s_free[2][2];
  uint32_t tmem_base;
};

struct IParams {
  float *out;
  int64_t N;
  int batch, nql, G, nqb, nb, total, accumulate;
  float sl2;  // tau * log2(e)
};

struct IItem {
  int b, h;
  int64_t i0;
  bool has1;
  int tl[2];  // last kv tile of q tile j
};

__device__ __forceinline__ IItem get_iitem(const IParams &p, int idx) {
  IItem it;
  const int bh = p.batch * p.nql;
  const int qb = p.nqb - 1 - idx / bh;  // longest causal rows first (LPT)
  const int r = idx - (idx / bh) * bh;
  it.b = r / p.nql;
  it.h = r - it.b * p.nql;
  it.i0 = (int64_t)qb * 2 * kIM;
  it.has1 = it.i0 + kIM < p.N;
  for (int j = 0; j < 2; ++j) {
    int64_t last = it.i0 + (int64_t)(j + 1) * kIM - 1;
    if (last > p.N - 1) last = p.N - 1;
    it.tl[j] = (int)(last / kIN);
  }
  return it;
}

__device__ __forceinline__ uint32_t s_col(uint32_t tmem, int j, int u) { return tmem + 256u * j + 128u * u; }

// ---------------------------------------------------------------- MMA issue (warp 9)
template <int D>
__device__ __forceinline__ void inf_mma_role(const IParams &p, IBars &bars, uint32_t tmem, uint32_t q_smem,
                                             uint32_t kv_smem) {
  using C = ICfg<D>;
  constexpr uint32_t idesc = idesc_bf16_f32(kIM, kIN, false);
  int qc[2] = {0, 0}, sc[2] = {0, 0}, kvc = 0;
  for (int idx = blockIdx.x; idx < p.total; idx += gridDim.x) {
    const IItem it = get_iitem(p, idx);
    const int nt = 1 + (it.has1 ? it.tl[1] : it.tl[0]);
    for (int j = 0; j < 2; ++j) {
      if (j == 1 && !it.has1) continue;
      mbar_wait_warp(smem_u32(&bars.q_full[j]), qc[j] & 1);
      ++qc[j];
    }
    for (int pass = 0; pass < 2; ++pass) {
      for (int t = 0; t < nt; ++t) {
        const int st = kvc % kKVStages;
        mbar_wait_warp(smem_u32(&bars.kv_full[st]), (kvc / kKVStages) & 1);
        tc_fence_after();
        const uint32_t k_addr = kv_smem + st * 2 * C::kKTile, v_addr = k_addr + C::kKTile;
        const uint64_t kdesc = smem_desc_sw128(k_addr, 16, 1024), vdesc = smem_desc_sw128(v_addr, 16, 1024);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if ((j == 1 && !it.has1) || t > it.tl[j]) continue;
          const int u = sc[j] & 1;
          if (sc[j] >= 2) mbar_wait_warp(smem_u32(&bars.s_free[j][u]), ((sc[j] - 2) >> 1) & 1);
          ++sc[j];
          tc_fence_after();
          const uint32_t q_addr = q_smem + (2 * j) * C::kQTile, d_addr = q_addr + C::kQTile;
          const uint64_t qdesc = smem_desc_sw128(q_addr, 16, 1024), ddesc = smem_desc_sw128(d_addr, 16, 1024);
          const uint32_t sc_col = s_col(tmem, j, u);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint64_t ao = (uint64_t)(((kk >> 2) * C::kQSlab + (kk & 3) * 32) >> 4);
              const uint64_t bo = (uint64_t)(((kk >> 2) * C::kKSlab + (kk & 3) * 32) >> 4);
              mma_ss(sc_col, qdesc + ao, kdesc + bo, idesc, kk > 0 ? 1u : 0u);       // S = Q K^T
            }
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint64_t ao = (uint64_t)(((kk >> 2) * C::kQSlab + (kk & 3) * 32) >> 4);
              const uint64_t bo = (uint64_t)(((kk >> 2) * C::kKSlab + (kk & 3) * 32) >> 4);
              mma_ss(sc_col + 64u, ddesc + ao, vdesc + bo, idesc, kk > 0 ? 1u : 0u);  // G = dO V^T
            }
            mma_commit(smem_u32(&bars.s_full[j][u]));
            if (pass == 1 && t == it.tl[j]) mma_commit(smem_u32(&bars.q_empty[j]));  // Q_j, dO_j free
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(smem_u32(&bars.kv_empty[st]));
        __syncwarp();
        ++kvc;
      }
    }
  }
}

// ---------------------------------------------------------------- elementwise (warps 0-7)
template <int D>
__device__ __forceinline__ void inf_ew_role(const IParams &p, IBars &bars, uint32_t tmem, int warp, int lane,
                                            float (*pair)[2][2][2]) {
  const int j = warp >> 2, wq = warp & 3;
  const int row = wq * 32 + lane;
  const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
  const int r = wq >> 1;                  // row block of this warp inside the q tile
  const int pair_bar = 1 + 2 * j + r;     // named barrier of the two warps of a row block
  int sc = 0;
  for (int idx = blockIdx.x; idx < p.total; idx += gridDim.x) {
    const IItem it = get_iitem(p, idx);
    if (j == 1 && !it.has1) continue;
    const int64_t ti0 = it.i0 + (int64_t)j * kIM;
    const int64_t i = ti0 + row;
    const bool valid = i < p.N;
    const int tl = it.tl[j];
    // first kv tile holding keys past some row of this warp (causal mask needed from there on)
    const int tdiag = (int)((ti0 + wq * 32) / kIN);
    float m = -INFINITY, Lr = 0.f, Ur = 0.f, Gs = 0.f;
    int js = -1;
    float s[kIN], g[kIN];
    auto load_tile = [&]() {
      const int u = sc & 1;
      mbar_wait_warp(smem_u32(&bars.s_full[j][u]), (sc >> 1) & 1);
      ++sc;
      tc_fence_after();
      const uint32_t base = s_col(tmem, j, u) + lane_off;
      tmem_ld32(base, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
      tmem_ld32(base + 32u, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
      tmem_ld32(base + 64u, *reinterpret_cast<uint32_t(*)[32]>(&g[0]));
      tmem_ld32(base + 96u, *reinterpret_cast<uint32_t(*)[32]>(&g[32]));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars.s_free[j][u]));
    };
    // ---- pass 0: row statistics
    for (int t = 0; t <= tl; ++t) {
      load_tile();
      const int64_t j0 = (int64_t)t * kIN;
      if (t >= tdiag) {  // keys past the row: never visible
        const int dd = (int)(i - j0);
#pragma unroll
        for (int c = 0; c < kIN; ++c)
          if (c > dd) s[c] = -INFINITY;
      }
      float mx = s[0];
#pragma unroll
      for (int c = 1; c < kIN; ++c) mx = fmaxf(mx, s[c]);
      mx *= p.sl2;  // tau > 0: the max commutes with the scaling
      const bool newmax = mx > m;
      float rs = 0.f, us = 0.f;
      if (__any_sync(0xffffffffu, newmax)) {
        // the tile's star (first key attaining its max) is split off when it is the row's new max
        int ks = kIN;
        float gst = 0.f;
#pragma unroll
        for (int c = kIN - 1; c >= 0; --c) {
          const bool hit = s[c] * p.sl2 == mx;
          ks = hit ? c : ks;
          gst = hit ? g[c] : gst;
        }
        if (!newmax) ks = kIN;  // not a new row max: every key joins the rest
        const float mn = newmax ? mx : m;
#pragma unroll
        for (int c = 0; c < kIN; ++c) {
          const float e = c == ks ? 0.f : fast_exp2(fmaf(s[c], p.sl2, -mn));
          rs += e;
          us = fmaf(g[c], e, us);
        }
        if (newmax) {
          const float alpha = fast_exp2(m - mx);  // 0 for the first tile (m = -inf)
          Lr = (js >= 0 ? (1.f + Lr) * alpha : 0.f) + rs;
          Ur = (js >= 0 ? (Gs + Ur) * alpha : 0.f) + us;
          m = mx;
          js = (int)j0 + ks;
          Gs = gst;
        } else {
          Lr += rs;
          Ur += us;
        }
      } else {
#pragma unroll
        for (int c = 0; c < kIN; ++c) {
          const float e = fast_exp2(fmaf(s[c], p.sl2, -m));
          rs += e;
          us = fmaf(g[c], e, us);
        }
        Lr += rs;
        Ur += us;
      }
    }
    const float l = 1.f + Lr, inv_l = 1.f / l, C1 = Gs + Ur;
    const float Estar = Lr > 0.f ? (Ur - Gs * Lr) / (Lr * l) : 0.f;  // a row with one visible key: 0
    const int64_t ib = ti0 / kIN + r;
    const int64_t rows_real = p.N - ib * kIN < kIN ? p.N - ib * kIN : kIN;
    float *orow = p.out + (((int64_t)it.b * p.nql + it.h) * p.nb + ib) * p.nb;
    // ---- pass 1: E, summed to block means
    for (int t = 0; t <= tl; ++t) {
      load_tile();
      const int64_t j0 = (int64_t)t * kIN;
      const int kst = js - (int)j0;  // the star's column (outside [0, 64) if not in this tile)
      float acc = 0.f;
      if (t >= tdiag) {
        const int dd = (int)(i - j0);
#pragma unroll
        for (int c = 0; c < kIN; ++c) {
          const float pe = c > dd ? 0.f : fast_exp2(fmaf(s[c], p.sl2, -m));
          const float e = __fdividef(pe * fmaf(-g[c], l, C1), l - pe);
          acc += (c == kst || c > dd) ? 0.f : e;
        }
      } else {
#pragma unroll
        for (int c = 0; c < kIN; ++c) {
          const float pe = fast_exp2(fmaf(s[c], p.sl2, -m));
          const float e = __fdividef(pe * fmaf(-g[c], l, C1), l - pe);
          acc += c == kst ? 0.f : e;
        }
      }
      acc = acc * inv_l + ((kst >= 0 && kst < kIN) ? Estar : 0.f);
      if (!valid) acc = 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      // the two warps of the row block: fixed-order sum (deterministic), one store per block
      if (lane == 0) pair[j][r][t & 1][wq & 1] = acc;
      asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
      if ((wq & 1) == 0 && lane == 0 && t <= ib && rows_real > 0) {
        const float tot = pair[j][r][t & 1][0] + pair[j][r][t & 1][1];
        const int64_t cols_real = p.N - j0 < kIN ? p.N - j0 : kIN;
        const float mean = tot / (float)(rows_real * cols_real);
        orow[t] = p.accumulate ? orow[t] + mean : mean;
      }
    }
    // blocks above the diagonal have no causal pairs
    if (!p.accumulate && (wq & 1) == 0 && rows_real > 0)
      for (int64_t jb = ib + 1 + lane; jb < p.nb; jb += 32) orow[jb] = 0.f;
  }
}

template <int D>
__global__ void __launch_bounds__(kIThreads, 1)
    influence_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                        const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                        const IParams p) {
  using C = ICfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ IBars bars;
  __shared__ float pair[2][2][2][2];  // [tile][row block][kv tile parity][warp of the pair]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t smem_base = smem_u32(smem_raw);
  if (smem_base & 1023u) __trap();
  const uint32_t q_smem = smem_base;                  // Q0, dO0, Q1, dO1
  const uint32_t kv_smem = q_smem + 4 * C::kQTile;    // stages of (K, V)

  if (tid == 0) {
    for (int j = 0; j < 2; ++j) {
      mbar_init(smem_u32(&bars.q_full[j]), 1);
      mbar_init(smem_u32(&bars.q_empty[j]), 1);
      for (int u = 0; u < 2; ++u) {
        mbar_init(smem_u32(&bars.s_full[j][u]), 1);
        mbar_init(smem_u32(&bars.s_free[j][u]), 4);  // the tile's 4 elementwise warps
      }
    }
    for (int s = 0; s < kKVStages; ++s) {
      mbar_init(smem_u32(&bars.kv_full[s]), 1);
      mbar_init(smem_u32(&bars.kv_empty[s]), 1);
    }
    fence_mbar_init();
  }
  if (warp == kWMma) tmem_alloc<kITmemCols>(smem_u32(&bars.tmem_base));
  if (warp == kWTma && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp < 8) {
    inf_ew_role<D>(p, bars, tmem, warp, lane, pair);
  } else if (warp == kWTma) {
    if (lane == 0) {
      int qc[2] = {0, 0}, kvc = 0;
      for (int idx = blockIdx.x; idx < p.total; idx += gridDim.x) {
        const IItem it = get_iitem(p, idx);
        const int g = it.h / p.G;
        for (int j = 0; j < 2; ++j) {
          if (j == 1 && !it.has1) continue;
          if (qc[j] > 0) mbar_wait(smem_u32(&bars.q_empty[j]), (qc[j] - 1) & 1);
          ++qc[j];
          const uint32_t qbar = smem_u32(&bars.q_full[j]);
          const uint32_t q_addr = q_smem + (2 * j) * C::kQTile;
          mbar_expect_tx(qbar, 2 * C::kQTile);
          for (int sl = 0; sl < C::kSlabs; ++sl) {
            tma_load_4d(q_addr + sl * C::kQSlab, &tm_q, qbar, sl * 64, it.h, (int)(it.i0 + j * kIM), it.b);
            tma_load_4d(q_addr + C::kQTile + sl * C::kQSlab, &tm_do, qbar, sl * 64, it.h, (int)(it.i0 + j * kIM),
                        it.b);
          }
        }
        const int nt = 1 + (it.has1 ? it.tl[1] : it.tl[0]);
        for (int pass = 0; pass < 2; ++pass)
          for (int t = 0; t < nt; ++t) {
            const int st = kvc % kKVStages;
            if (kvc >= kKVStages) mbar_wait(smem_u32(&bars.kv_empty[st]), ((kvc - kKVStages) / kKVStages) & 1);
            ++kvc;
            const uint32_t kbar = smem_u32(&bars.kv_full[st]);
            const uint32_t k_addr = kv_smem + st * 2 * C::kKTile;
            mbar_expect_tx(kbar, 2 * C::kKTile);
            for (int sl = 0; sl < C::kSlabs; ++sl) {
              tma_load_4d(k_addr + sl * C::kKSlab, &tm_k, kbar, sl * 64, g, t * kIN, it.b);
              tma_load_4d(k_addr + C::kKTile + sl * C::kKSlab, &tm_v, kbar, sl * 64, g, t * kIN, it.b);
            }
          }
      }
    }
  } else if (warp == kWMma) {
    inf_mma_role<D>(p, bars, tmem, q_smem, kv_smem);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kWMma) {
    tc_fence_after();
    tmem_dealloc<kITmemCols>(tmem);
  }
}

template <int D>
int launch_tc(const InfluenceArgs &a, void *stream) {
  using C = ICfg<D>;
  alignas(64) CUtensorMap mq, mdo, mk, mv;
  const int ngl = a.nql / a.G;
  if (!make_tile_map(&mq, a.q, D, a.nql, a.N, a.batch, a.q_row_stride, kIM) ||
      !make_tile_map(&mdo, a.dout, D, a.nql, a.N, a.batch, a.q_row_stride, kIM) ||
      !make_tile_map(&mk, a.k, D, ngl, a.N, a.batch, a.kv_row_stride, kIN) ||
      !make_tile_map(&mv, a.v, D, ngl, a.N, a.batch, a.kv_row_stride, kIN))
    return (int)cudaErrorInvalidValue;
  IParams p;
  p.out = a.e_blocks;
  p.N = a.N;
  p.batch = a.batch;
  p.nql = a.nql;
  p.G = a.G;
  p.nqb = (int)((a.N + 2 * kIM - 1) / (2 * kIM));
  p.nb = (int)((a.N + kIN - 1) / kIN);
  p.total = p.nqb * a.batch * a.nql;
  p.accumulate = a.accumulate;
  p.sl2 = a.scale * kLog2e;
  cudaError_t e = cudaFuncSetAttribute(influence_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::kSmem);
  if (e != cudaSuccess) return (int)e;
  const int grid = p.total < device_sm_count() ? p.total : device_sm_count();
  influence_tc_kernel<D><<<grid, kIThreads, C::kSmem, (cudaStream_t)stream>>>(mq, mdo, mk, mv, p);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_influence_tc(const InfluenceArgs &a, void *stream) {
  if (a.d == 128) return launch_tc<128>(a, stream);
  return launch_tc<64>(a, stream);
}

}  // namespace moa
