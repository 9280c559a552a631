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
// Work item = one 128-row q tile of one (batch, q-head), two passes over its causal key tiles
// of 128 keys:
//   pass 0  row statistics: m = max_k tau s_k (log2 units); the first key attaining it (the
//           "star", js, with G_js = Gs) is kept out of the sums, Lr = sum_{k != js} 2^(x_k - m)
//           and Ur = sum_{k != js} G_k 2^(x_k - m), so l = 1 + Lr and R = (Gs + Ur) / l, and
//           1 - A_js = Lr / l, R - G_js = (Ur - Gs Lr) / l keep fp32 accuracy on rows that are
//           nearly one-hot (a sink-dominated row) where 1 - A in fp32 would cancel;
//   pass 1  E_ij = p (C1 - G_ij l) / ((l - p) l) with p = 2^(x_ij - m), C1 = Gs + Ur (the star:
//           E = (Ur - Gs Lr) / (Lr l)), summed per row over a key block, then over the 64 rows
//           of a query block: one block mean per (query block, key block).
// Per kv tile the tensor core computes S = Q K^T and G = dO V^T (two SS MMAs, M = N = 128, K =
// d, into TMEM, double-buffered: the next tile's products are computed while the elementwise
// warps work on this one); the elementwise warps read their row of S and G (thread = row =
// TMEM lane) and never touch A, G or E in memory.
//
// Warps (320 threads, one CTA per SM, persistent over items in LPT order):
//   0-7  elementwise: warp w reads TMEM lanes 32 (w % 4) .. + 31 (its 32 rows) and the key half
//        w / 4 (columns 64 h .. 64 h + 63 of each 128-key tile = one 64-key block); the two
//        warps of a row quarter merge their pass-0 statistics once per item
//   8    TMA producer (Q, dO per item; K, V per step, both passes)
//   9    TMEM allocator + MMA issue (one elected lane)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <type_traits>

#include "../moa_internal.h"
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace moa {
namespace {

using namespace ptx;

constexpr int kIM = 128;        // q rows per tile (MMA M)
constexpr int kIN = 128;        // keys per kv tile (MMA N)
constexpr int kCols = 64;       // keys per block (the paper's block)
#ifndef MOA_INF_EW16
#define MOA_INF_EW16 1
#endif
// elementwise warps: 4 row quarters (TMEM lanes) x kNQ column parts of each 128-key tile (kW keys
// each); 16 warps (four per sub-partition, 32 keys each) hide the TMEM-load and MUFU latency that
// bounded 8 warps (two per sub-partition, 64 keys each)
constexpr int kNQ = MOA_INF_EW16 ? 4 : 2;
constexpr int kW = kIN / kNQ;
constexpr int kEW = 4 * kNQ;
constexpr int kIThreads = 32 * (kEW + 2);
constexpr int kWTma = kEW, kWMma = kEW + 1;
constexpr int kKVStagesMax = 4;
constexpr uint32_t kITmemCols = 512;  // buffer u: S (128 cols) | G (128 cols)
#ifndef MOA_INF_RCP4
#define MOA_INF_RCP4 1  // +1.5 % at N = 8k (with the per-pass polynomial shares below)
#endif
constexpr bool kRcpQuad = MOA_INF_RCP4;  // pass 1: one MUFU reciprocal per four keys instead of two
// exponential pair c on the FMA pipe iff c % kPoly == kPoly - 1, per pass (pass 0 sums, pass 1
// E); measured at N = 8k (A/B, tools/time_influence.py, 8 elementwise warps): one pair in 2 for
// both passes 0.268 of the bf16 burst, 3 / 3 0.277, 6 / 8 0.286; 16 warps: 6 / 8 0.291, 4 / 4 0.295;
// with the snake item order: 4 / 4 0.305, 4 / 6 0.307, 5 / 5 0.306, 3 / 3 0.298
#ifndef MOA_INF_POLY0
#define MOA_INF_POLY0 4
#endif
#ifndef MOA_INF_POLY1
#define MOA_INF_POLY1 6
#endif
constexpr int kPoly0 = MOA_INF_POLY0, kPoly1 = MOA_INF_POLY1;
constexpr int kPairRound = 32;  // kv tiles between the two warps of a query block meeting
constexpr float kRefLazy = 8.f;   // pass 0: refresh the exponent reference when the max grows by > 2^8
constexpr float kStarLazy = 4.f;  // pass 0: move the designated key when a key beats it by > 2^4
// diagnostics (tools/build_variant.py): 1 = elementwise warps only load and release S/G (the
// MMA / TMA floor), 2 = no MMAs issued (the elementwise floor, on stale TMEM)
#ifndef MOA_INF_DIAG
#define MOA_INF_DIAG 0
#endif

template <int D>
struct ICfg {
  static constexpr int kSlabs = D / 64;
  static constexpr int kQTile = kIM * D * 2;  // Q or dO tile bytes
  static constexpr int kQSlab = kIM * 128;
  static constexpr int kKTile = kIN * D * 2;  // K or V tile bytes
  static constexpr int kKSlab = kIN * 128;
  // K/V ring depth: what fits beside the Q and dO tiles (227 KB per CTA)
  static constexpr int kStages = D == 128 ? 2 : 4;
  static constexpr int kSmem = 2 * kQTile + kStages * 2 * kKTile;  // Q dO | stages (K V)
};

struct IBars {
  uint64_t q_full, q_empty;
  uint64_t kv_full[kKVStagesMax], kv_empty[kKVStagesMax];
  uint64_t s_full[2], s_free[2];
  uint32_t tmem_base;
};

struct IParams {
  float *out;
  int64_t N;
  int batch, nql, G, nqt, nb, total, accumulate;
  float sl2;  // tau * log2(e)
};

struct IItem {
  int b, h;
  int64_t i0;
  int tl;  // last kv tile (of 128 keys)
};

// Items are in LPT order (costs non-increasing); CTA c takes item c of even rounds and item
// gridDim - 1 - c of odd rounds ("snake"), which balances the per-CTA sums: at N = 8k the
// busiest CTA had 7 % more work than the mean with a plain round robin, 0.06 % with the snake.
// An odd last round may skip the low CTAs; every item below total is still taken exactly once.
__device__ __forceinline__ int snake_item(int rnd) {
  return rnd * (int)gridDim.x + ((rnd & 1) ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x);
}

__device__ __forceinline__ IItem get_iitem(const IParams &p, int idx) {
  IItem it;
  const int bh = p.batch * p.nql;
  const int qt = p.nqt - 1 - idx / bh;  // longest causal rows of every head first (LPT)
  const int r = idx - (idx / bh) * bh;
  it.b = r / p.nql;
  it.h = r - it.b * p.nql;
  it.i0 = (int64_t)qt * kIM;
  int64_t last = it.i0 + kIM - 1;
  if (last > p.N - 1) last = p.N - 1;
  it.tl = (int)(last / kIN);
  return it;
}

// ---------------------------------------------------------------- MMA issue (warp 9)
template <int D>
__device__ __forceinline__ void inf_mma_role(const IParams &p, IBars &bars, uint32_t tmem, uint32_t q_smem,
                                             uint32_t kv_smem) {
  using C = ICfg<D>;
  constexpr uint32_t idesc = idesc_bf16_f32(kIM, kIN, false);
  int qc = 0, sc = 0, kvc = 0;
  const uint64_t qdesc = smem_desc_sw128(q_smem, 16, 1024), ddesc = smem_desc_sw128(q_smem + C::kQTile, 16, 1024);
  for (int rnd = 0, idx = snake_item(0); idx < p.total; idx = snake_item(++rnd)) {
    const IItem it = get_iitem(p, idx);
    mbar_wait_warp(smem_u32(&bars.q_full), qc & 1);
    ++qc;
    for (int pass = 0; pass < 2; ++pass) {
      for (int t = 0; t <= it.tl; ++t, ++kvc, ++sc) {
        const int st = kvc % C::kStages;
        if (MOA_INF_DIAG < 4 || kvc < C::kStages) mbar_wait_warp(smem_u32(&bars.kv_full[st]), (kvc / C::kStages) & 1);
        const int u = sc & 1;
        if (sc >= 2 && MOA_INF_DIAG < 3) mbar_wait_warp(smem_u32(&bars.s_free[u]), ((sc - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t k_addr = kv_smem + st * 2 * C::kKTile, v_addr = k_addr + C::kKTile;
        const uint64_t kdesc = smem_desc_sw128(k_addr, 16, 1024), vdesc = smem_desc_sw128(v_addr, 16, 1024);
        const uint32_t scol = tmem + 256u * u;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < (MOA_INF_DIAG == 2 ? 0 : D / 16); ++kk) {
            const uint64_t ao = (uint64_t)(((kk >> 2) * C::kQSlab + (kk & 3) * 32) >> 4);
            const uint64_t bo = (uint64_t)(((kk >> 2) * C::kKSlab + (kk & 3) * 32) >> 4);
            mma_ss(scol, qdesc + ao, kdesc + bo, idesc, kk > 0 ? 1u : 0u);          // S = Q K^T
          }
#pragma unroll
          for (int kk = 0; kk < (MOA_INF_DIAG == 2 ? 0 : D / 16); ++kk) {
            const uint64_t ao = (uint64_t)(((kk >> 2) * C::kQSlab + (kk & 3) * 32) >> 4);
            const uint64_t bo = (uint64_t)(((kk >> 2) * C::kKSlab + (kk & 3) * 32) >> 4);
            mma_ss(scol + 128u, ddesc + ao, vdesc + bo, idesc, kk > 0 ? 1u : 0u);   // G = dO V^T
          }
          mma_commit(smem_u32(&bars.s_full[u]));
          if (pass == 1 && t == it.tl) mma_commit(smem_u32(&bars.q_empty));  // Q, dO free
          if (MOA_INF_DIAG < 4) mma_commit(smem_u32(&bars.kv_empty[st]));
        }
        __syncwarp();
      }
    }
  }
}

// merge of the two key halves' pass-0 statistics of a row (both warps evaluate the same
// expression on (half 0, half 1), so they hold bit-identical results): the half holding the row
// max (first key on a tie) keeps its star, the other half's star and rest join the rest
__device__ __forceinline__ void merge_stats(float m0, float L0, float U0, float G0, int j0, float m1, float L1,
                                            float U1, float G1, int j1, float &m, float &Lr, float &Ur, float &Gs,
                                            int &js) {
  const bool take0 = j1 < 0 || (j0 >= 0 && (m0 > m1 || (m0 == m1 && j0 < j1)));
  const float ms = take0 ? m0 : m1, mo = take0 ? m1 : m0;
  const float Ls = take0 ? L0 : L1, Lo = take0 ? L1 : L0;
  const float Us = take0 ? U0 : U1, Uo = take0 ? U1 : U0;
  const float Gss = take0 ? G0 : G1, Go = take0 ? G1 : G0;
  const int jo = take0 ? j1 : j0;
  const float w = jo >= 0 ? fast_exp2(mo - ms) : 0.f;
  m = ms;
  Lr = Ls + (1.f + Lo) * w;
  Ur = Us + (Go + Uo) * w;
  Gs = Gss;
  js = take0 ? j0 : j1;
}

// ---------------------------------------------------------------- elementwise (warps 0-7)
template <int D>
__device__ __forceinline__ void inf_ew_role(const IParams &p, IBars &bars, uint32_t tmem, int warp, int lane,
                                            float (*pair)[2][kPairRound], float (*xs)[6][kIM]) {
  const int cq = warp >> 2, wq = warp & 3;        // column part, row quarter
  const int hf = cq * kW / kCols;                 // key block of the tile this warp's keys are in
  const int cp = (cq * kW % kCols) / kW;          // part of that block
  const int row = wq * 32 + lane;
  const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
  const int r = wq >> 1;                          // query block of this warp inside the q tile
  const int pair_bar = 1 + 2 * hf + r;            // named barrier of the warps of a (query block, key block)
  constexpr int kPairThreads = 64 * (kCols / kW);
  const int half_bar = 5 + wq;                    // named barrier of the column parts of a row quarter
  int sc = 0;
  float s[kW], g[kW];
  for (int rnd = 0, idx = snake_item(0); idx < p.total; idx = snake_item(++rnd)) {
    const IItem it = get_iitem(p, idx);
    const int64_t ti0 = it.i0;
    const int64_t i = ti0 + row;
    const bool valid = i < p.N;
    const int tl = it.tl;
    const int64_t wrow0 = ti0 + wq * 32;  // first row of this warp
    // pass-0 state of this row over this warp's key half: sums relative to a lazy reference mr
    // (log2 units; refreshed only when the max grows by more than kRefLazy), and a DESIGNATED
    // key js (value xs, weight pj = 2^(xs - mr), G = Gs) kept out of Lr = sum_{k != js} p_k and
    // Ur = sum_{k != js} G_k p_k
    float mr = -INFINITY, xsv = -INFINITY, pj = 0.f, Lr = 0.f, Ur = 0.f, Gs = 0.f;
    int js = -1;
    auto load_tile = [&]() {
      const int u = sc & 1;
      mbar_wait_warp(smem_u32(&bars.s_full[u]), (sc >> 1) & 1);
      ++sc;
      tc_fence_after();
      const uint32_t base = tmem + 256u * u + lane_off + (uint32_t)(kW * cq);
      if (MOA_INF_DIAG != 5) {
        if (MOA_INF_DIAG != 7) {
#pragma unroll
          for (int h = 0; h < kW / 32; ++h) tmem_ld32(base + 32u * h, *reinterpret_cast<uint32_t(*)[32]>(&s[32 * h]));
        }
        // wait between the S and G pairs: with all four 32-column loads in flight before one
        // wait the step took ~1400 cycles longer (tools/build_variant.py diag 1 vs 8: 1.57 vs
        // 0.67 ms at N = 8k with no elementwise work); two in flight cost nothing measurable
        tmem_wait_ld();
        if (MOA_INF_DIAG != 6) {
#pragma unroll
          for (int h = 0; h < kW / 32; ++h)
            tmem_ld32(base + 128u + 32u * h, *reinterpret_cast<uint32_t(*)[32]>(&g[32 * h]));
        }
        tmem_wait_ld();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars.s_free[u]));
    };
    auto lane_load = [&](int t) {
      load_tile();
      const int64_t j0 = (int64_t)t * kIN + kW * cq;  // first key of this warp's part
      const bool diag = j0 + kW - 1 > wrow0;           // keys past some row of the warp
      if (diag) {  // keys past the row: never visible
        const int dd = (int)(i - j0);
#pragma unroll
        for (int c = 0; c < kW; ++c)
          if (c > dd) s[c] = -INFINITY;
      }
      return diag;
    };
    // ---- pass 0: row statistics over this warp's key half
    for (int t = 0; t <= tl; ++t) {
      if (MOA_INF_DIAG >= 3) continue;
      const bool diag = lane_load(t);
      if (MOA_INF_DIAG == 1 || MOA_INF_DIAG >= 5) continue;
      const int64_t j0 = (int64_t)t * kIN + kW * cq;
      float mq[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) mq[a] = fmaxf(s[a], s[a + 4]);
#pragma unroll
      for (int c = 8; c < kW; c += 8)
#pragma unroll
        for (int a = 0; a < 4; ++a) mq[a] = fmax3(mq[a], s[c + a], s[c + a + 4]);
      const float mxr = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));  // raw max
      const float mx = mxr * p.sl2;  // tau > 0: the max commutes with the scaling
      // the designated key only moves when a key beats it by more than 2^kStarLazy: any key it
      // leaves in the sums then has A <= 2^kStarLazy / (1 + 2^kStarLazy) < 1, so 1 - A stays
      // well conditioned; for random scores this happens in the row's first tile only
      const bool sw = mx > xsv + kStarLazy;
      if (__any_sync(0xffffffffu, sw)) {
        int ks = kW;
        float gst = 0.f;
#pragma unroll
        for (int c = kW - 1; c >= 0; --c) {
          const bool hit = s[c] == mxr;
          ks = hit ? c : ks;
          gst = hit ? g[c] : gst;
        }
        if (!sw) ks = kW;
        const float mn = fmaxf(mr, mx);
        if (mn > mr) {  // new reference (the first visible tile: mr = -inf, the sums are 0)
          const float a = mr == -INFINITY ? 0.f : fast_exp2(mr - mn);
          Lr *= a;
          Ur *= a;
          pj *= a;
          mr = mn;
        }
        if (sw) {  // the old designated key joins the rest
          Lr += pj;
          Ur = fmaf(Gs, pj, Ur);
        }
        float rs = 0.f, us = 0.f;
        const float nm = mr == -INFINITY ? 0.f : -mr;
#pragma unroll
        for (int c = 0; c < kW; ++c) {
          const float e = c == ks ? 0.f : fast_exp2(fmaf(s[c], p.sl2, nm));
          rs += e;
          us = fmaf(g[c], e, us);
        }
        Lr += rs;
        Ur += us;
        if (sw) {
          js = (int)j0 + ks;
          xsv = mx;
          pj = fast_exp2(mx - mr);
          Gs = gst;
        }
      } else {
        if (mx > mr + kRefLazy) {  // lazy reference refresh (rare)
          const float a = fast_exp2(mr - mx);
          Lr *= a;
          Ur *= a;
          pj *= a;
          mr = mx;
        }
        // packed f32x2 arithmetic, four independent sums, one exponential pair in kPoly0
        // on the FMA pipe -- except in diagonal tiles: masked keys must add exactly 0 (MUFU
        // ex2(-inf) = 0; the polynomial bottoms out at 2^-126, and on a row with one visible
        // key any nonzero rest would turn its E from 0 into noise).  mr = -inf: this half has
        // seen no key of the row yet and the tile is all masked (the offset stays finite).
        const float nm = mr == -INFINITY ? 0.f : -mr;
        const uint64_t sl2 = f2pk(p.sl2, p.sl2), nm2 = f2pk(nm, nm);
        uint64_t r2[2] = {0ull, 0ull}, u2[2] = {0ull, 0ull};
        auto sweep = [&](auto poly) {
#pragma unroll
          for (int c = 0; c < kW; c += 2) {
            float ya, yb, ea, eb;
            f2upk(ffma2(f2pk(s[c], s[c + 1]), sl2, nm2), ya, yb);
            if (decltype(poly)::value && (c >> 1) % kPoly0 == kPoly0 - 1) {
              exp2_poly2(ya, yb, ea, eb);
            } else {
              ea = fast_exp2(ya);
              eb = fast_exp2(yb);
            }
            const uint64_t e2 = f2pk(ea, eb);
            r2[(c >> 1) & 1] = fadd2(r2[(c >> 1) & 1], e2);
            u2[(c >> 1) & 1] = ffma2(f2pk(g[c], g[c + 1]), e2, u2[(c >> 1) & 1]);
          }
        };
        if (diag)
          sweep(std::false_type{});
        else
          sweep(std::true_type{});
        float a0, a1, b0, b1;
        f2upk(fadd2(r2[0], r2[1]), a0, a1);
        f2upk(fadd2(u2[0], u2[1]), b0, b1);
        Lr += a0 + a1;
        Ur += b0 + b1;
      }
    }
    // ---- merge the two halves' statistics (once per item): common reference, the larger
    // designated key stays designated (first key on a tie), the other one joins the rest.  Both
    // warps evaluate the same expression on (half 0, half 1): bit-identical results.
    if (MOA_INF_DIAG != 1 && MOA_INF_DIAG < 3) {
      xs[cq][0][row] = mr;
      xs[cq][1][row] = pj;
      xs[cq][2][row] = Lr;
      xs[cq][3][row] = Ur;
      xs[cq][4][row] = Gs;
      xs[cq][5][row] = __int_as_float(js);
      asm volatile("bar.sync %0, %1;" ::"r"(half_bar), "r"(32 * kNQ) : "memory");
      float mm = -INFINITY;
#pragma unroll
      for (int q = 0; q < kNQ; ++q) mm = fmaxf(mm, xs[q][0][row]);
      float pq[kNQ], wgt[kNQ];
      int jq[kNQ];
      int take = 0;
#pragma unroll
      for (int q = 0; q < kNQ; ++q) {
        const float mq = xs[q][0][row];
        wgt[q] = mq == -INFINITY ? 0.f : fast_exp2(mq - mm);
        pq[q] = xs[q][1][row] * wgt[q];
        jq[q] = __float_as_int(xs[q][5][row]);
      }
      // the designated key of the merged row: the largest designated weight (first key on a tie)
#pragma unroll
      for (int q = 1; q < kNQ; ++q)
        if (jq[q] >= 0 && (jq[take] < 0 || pq[q] > pq[take] || (pq[q] == pq[take] && jq[q] < jq[take]))) take = q;
      float Ls = 0.f, Us = 0.f, Lo = 0.f, Uo = 0.f;
#pragma unroll
      for (int q = 0; q < kNQ; ++q) {
        Ls += xs[q][2][row] * wgt[q];
        Us += xs[q][3][row] * wgt[q];
        if (q != take) {
          Lo += pq[q];
          Uo += xs[q][4][row] * pq[q];
        }
      }
      mr = mm;
      pj = pq[take];
      Gs = xs[take][4][row];
      js = jq[take];
      Lr = Ls + Lo;
      Ur = Us + Uo;
      asm volatile("bar.sync %0, %1;" ::"r"(half_bar), "r"(32 * kNQ) : "memory");  // all read before the next item's write
    }
    const float m = mr;
    // l = sum of all p; C1 = R l; the designated key: E = pj (Ur - Gs Lr) / (l Lr) (0 for a
    // row with one visible key)
    const float l = pj + Lr, inv_l = 1.f / l, C1 = fmaf(pj, Gs, Ur);
    const float Estar = Lr > 0.f ? pj * (Ur - Gs * Lr) / (Lr * l) : 0.f;
    const int64_t ib = ti0 / kCols + r;
    const int64_t rows_real = p.N - ib * kCols < kCols ? p.N - ib * kCols : kCols;
    float *orow = p.out + (((int64_t)it.b * p.nql + it.h) * p.nb + ib) * p.nb;
    // ---- pass 1: E, summed to block means
    for (int t = 0; t <= tl; ++t) {
      if (MOA_INF_DIAG >= 3) continue;
      load_tile();
      const int64_t j0 = (int64_t)t * kIN + kW * cq;
      const bool diag = j0 + kW - 1 > wrow0;
      const int jb = 2 * t + hf;  // key block
      const int kst = js - (int)j0;  // the star's column (outside [0, kW) if not in this part)
      float acc = 0.f;
      const bool star_here = kst >= 0 && kst < kW;
      if (MOA_INF_DIAG == 1 || MOA_INF_DIAG >= 5) {
        acc = s[lane] + g[lane];
      } else if (diag || __any_sync(0xffffffffu, star_here)) {
        // diagonal tiles (causal mask) and tiles holding some row's star (split off)
        const int dd = diag ? (int)(i - j0) : kW;
#pragma unroll
        for (int c = 0; c < kW; ++c) {
          const float pe = c > dd ? 0.f : fast_exp2(fmaf(s[c], p.sl2, -m));
          const float e = __fdividef(pe * fmaf(-g[c], l, C1), l - pe);
          acc += (c == kst || c > dd) ? 0.f : e;
        }
      } else {
        // E = p (C1 - G l) / (l - p) on packed pairs; one exponential pair in kPoly1 on
        // the FMA pipe.  A pair's two quotients share one MUFU reciprocal:
        // qa / da + qb / db = (qa db + qb da) / (da db)  (da, db in [1, l]: no overflow)
        const uint64_t sl2 = f2pk(p.sl2, p.sl2), nm2 = f2pk(-m, -m), nl2 = f2pk(-l, -l), l2 = f2pk(l, l),
                       c12 = f2pk(C1, C1), m12 = f2pk(-1.f, -1.f);
        float a[4] = {0.f, 0.f, 0.f, 0.f};
        float pn = 0.f, pd = 1.f;  // kRcpQuad: the first pair of a quad (numerator, denominator)
#pragma unroll
        for (int c = 0; c < kW; c += 2) {
          float ya, yb, ea, eb;
          f2upk(ffma2(f2pk(s[c], s[c + 1]), sl2, nm2), ya, yb);
          if ((c >> 1) % kPoly1 == kPoly1 - 1) {
            exp2_poly2(ya, yb, ea, eb);
          } else {
            ea = fast_exp2(ya);
            eb = fast_exp2(yb);
          }
          const uint64_t p2 = f2pk(ea, eb);
          float da, db;
          f2upk(ffma2(p2, m12, l2), da, db);  // l - p (>= 1 off the star)
          const uint64_t q2 = fmul2(p2, ffma2(f2pk(g[c], g[c + 1]), nl2, c12));
          float qa, qb;
          f2upk(fmul2(q2, f2pk(db, da)), qa, qb);
          if (kRcpQuad) {
            // two pairs share one reciprocal: n1 / d1 + n2 / d2 = (n1 d2 + n2 d1) / (d1 d2), with
            // d = da db in [1, l^2] per pair (l <= 2^8 N: the product of two stays far below 2^127)
            const float nn = qa + qb, dd = da * db;
            if ((c >> 1) & 1) {
              a[(c >> 2) & 3] = fmaf(fmaf(pn, dd, nn * pd), fast_rcp(pd * dd), a[(c >> 2) & 3]);
            } else {
              pn = nn;
              pd = dd;
            }
          } else {
            a[(c >> 1) & 3] = fmaf(qa + qb, fast_rcp(da * db), a[(c >> 1) & 3]);
          }
        }
        acc = (a[0] + a[1]) + (a[2] + a[3]);
      }
      acc = acc * inv_l + (star_here ? Estar : 0.f);
      if (!valid) acc = 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      // the two warps of a query block park their sums per tile (double-buffered rounds of
      // kPairRound tiles) and meet once per round: fixed-order sum (deterministic), one store per block
      if (lane == 0) pair[warp][(t / kPairRound) & 1][t % kPairRound] = acc;
      if (t % kPairRound == kPairRound - 1 || t == tl) {
        asm volatile("bar.sync %0, %1;" ::"r"(pair_bar), "r"(kPairThreads) : "memory");
        if ((wq & 1) == 0 && cp == 0 && rows_real > 0) {
          const int t0 = t - t % kPairRound;
          for (int tt = t0 + lane; tt <= t; tt += 32) {
            const int jbt = 2 * tt + hf;
            if (jbt > ib) continue;  // no causal pairs above the diagonal
            const int sl = tt % kPairRound, bu = (tt / kPairRound) & 1;
            // the block's warps: row quarters wq, wq + 1 x the block's column parts (fixed order)
            float tot = pair[warp][bu][sl] + pair[warp + 1][bu][sl];
#pragma unroll
            for (int q = 1; q < kCols / kW; ++q) tot += pair[warp + 4 * q][bu][sl] + pair[warp + 4 * q + 1][bu][sl];
            const int64_t jt = (int64_t)jbt * kCols;
            const int64_t cols_real = p.N - jt < kCols ? p.N - jt : kCols;
            const float mean = tot / (float)(rows_real * cols_real);
            orow[jbt] = p.accumulate ? orow[jbt] + mean : mean;
          }
        }
      }
      (void)jb;
    }
    // blocks above the diagonal have no causal pairs (both halves' blocks, written by half 0)
    if (!p.accumulate && cq == 0 && (wq & 1) == 0 && rows_real > 0)
      for (int64_t b2 = ib + 1 + lane; b2 < p.nb; b2 += 32) orow[b2] = 0.f;
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
  __shared__ float pair[kEW][2][kPairRound];  // [warp][round parity][tile in round] query-block row sums
  __shared__ float xs[kNQ][6][kIM];           // [column part][mr, pj, Lr, Ur, Gs, js][row] pass-0 statistics exchange
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t smem_base = smem_u32(smem_raw);
  if (smem_base & 1023u) __trap();
  const uint32_t q_smem = smem_base;                  // Q, dO
  const uint32_t kv_smem = q_smem + 2 * C::kQTile;    // stages of (K, V)

  if (tid == 0) {
    mbar_init(smem_u32(&bars.q_full), 1);
    mbar_init(smem_u32(&bars.q_empty), 1);
    for (int u = 0; u < 2; ++u) {
      mbar_init(smem_u32(&bars.s_full[u]), 1);
      mbar_init(smem_u32(&bars.s_free[u]), kEW);  // the elementwise warps
    }
    for (int s = 0; s < C::kStages; ++s) {
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

  if (warp < kEW) {
    inf_ew_role<D>(p, bars, tmem, warp, lane, pair, xs);
  } else if (warp == kWTma) {
    if (lane == 0) {
      int qc = 0, kvc = 0;
      for (int rnd = 0, idx = snake_item(0); idx < p.total; idx = snake_item(++rnd)) {
        const IItem it = get_iitem(p, idx);
        const int g = it.h / p.G;
        if (qc > 0) mbar_wait_sleep(smem_u32(&bars.q_empty), (qc - 1) & 1, 128);
        ++qc;
        const uint32_t qbar = smem_u32(&bars.q_full);
        mbar_expect_tx(qbar, 2 * C::kQTile);
        for (int sl = 0; sl < C::kSlabs; ++sl) {
          tma_load_4d(q_smem + sl * C::kQSlab, &tm_q, qbar, sl * 64, it.h, (int)it.i0, it.b);
          tma_load_4d(q_smem + C::kQTile + sl * C::kQSlab, &tm_do, qbar, sl * 64, it.h, (int)it.i0, it.b);
        }
        for (int pass = 0; pass < 2; ++pass)
          for (int t = 0; t <= it.tl; ++t, ++kvc) {
            if (MOA_INF_DIAG >= 4 && kvc >= C::kStages) continue;
            const int st = kvc % C::kStages;
            if (kvc >= C::kStages)
              mbar_wait_sleep(smem_u32(&bars.kv_empty[st]), ((kvc - C::kStages) / C::kStages) & 1, 64);
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
  p.nqt = (int)((a.N + kIM - 1) / kIM);
  p.nb = (int)((a.N + kCols - 1) / kCols);
  p.total = p.nqt * a.batch * a.nql;
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
