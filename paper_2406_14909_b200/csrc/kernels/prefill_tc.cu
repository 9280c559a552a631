// prefill_tc.cu -- MoA causal prefill on the sm_100a tensor cores (tcgen05 +
// TMEM + TMA), bf16 I/O, fp32 accumulation.
//
//   O[b,i,h] = sum_{j in V(h,i)} softmax_j(tau q_i . k_j) v_j       (Eq. 1)
//   V(h,i)   = { j <= i : j < s  or  i - j < W_h }                   (reading c3)
//
// Only the kv tiles of the block-skip schedule are visited (moa_internal.h:
// sink tiles + window tiles); FULL tiles skip the mask arithmetic, EDGE tiles
// apply the token-granular predicate.  Within a visited tile the work is a
// dense contraction, so QK^T and PV run on tcgen05 with TMEM accumulators.
//
// Persistent CTAs (one per SM) walk a static round-robin slice of the
// LPT-sorted (q-head, 128-row q tile) x batch work list.  Warp roles (384 threads):
//   warps 0-3   softmax of S columns [0, 64)   (thread t owns row t = TMEM lane t)
//   warps 4-7   softmax of S columns [64, 128) (same rows; the two halves exchange the
//               row max through shared memory once per tile)
//   warp 8      TMA producer: Q (double-buffered per item) and the K ring
//   warp 9      TMEM allocator + MMA issuer (whole warp, one elected lane issues)
//   warp 10     TMA producer: the V ring
// TMEM (512 columns): S0 | S1 (fp32 128x128) | P0 | P1 (bf16 128x128 packed, 64 columns
// each) | O (fp32 128xD).  S is double-buffered, so QK^T of tile T+1 runs on the tensor
// core while the softmax of tile T executes; P is double-buffered, so PV of tile T
// overlaps the softmax of tile T+1.  tcgen05 ops of one thread complete in issue order
// and a commit tracks every earlier op, so "S(T) complete" implies "PV(T-2) complete"
// (P[T%2] is free).  The running max is refreshed (and O rescaled in TMEM) only when it
// grows by more than 2^8; a share of the exponentials runs as a polynomial on the FMA
// pipe (MUFU ex2, 16/clk/SM, is as slow as the tensor core on a 128x128 tile).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "../moa_internal.h"
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace moa {
namespace {

using namespace ptx;

constexpr int kM = 128;               // q rows per tile (MMA M)
constexpr int kN = 128;               // keys per tile (MMA N of QK^T, K of PV)
constexpr int kHalf = kN / 2;         // S columns per softmax warpgroup
constexpr int kSoftmaxThreads = 256;  // two warpgroups, one per column half
constexpr int kThreads = 384;
constexpr uint32_t kTmemCols = 512;
// TMEM: S (fp32 128x128) | P0 | P1 (bf16 packed, 64 cols each) | O (fp32 128xD) | Q0 | Q1 (bf16 packed)
constexpr uint32_t kColS = 0, kColP0 = 128, kColP1 = 192, kColO = 256, kColQ0 = 384, kColQ1 = 448;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only if the max grows by > 2^8
// exponentials of pairs c with (c & kPolyMask) == kPolyMask use the FMA-pipe polynomial
constexpr int kPolyMask = 1;
constexpr int kBarSoftmax = 1;  // named barrier of the 8 softmax warps
constexpr int kSoftmaxWarps = 8;  // mbarrier arrivals from the softmax side (one per warp)

// 2^y on the FMA/ALU pipes: y = n + f, n = round(y), |f| <= 1/2, 2^f by a degree-3
// polynomial fitted for relative error (7.7e-5 max, far below bf16's 3.9e-3), 2^n by
// adding n to the exponent field.  Inputs below -126 flush to ~2^-126 (negligible).
__device__ __forceinline__ float exp2_poly(float y) {
  y = fmaxf(y, -126.f);
  const float t = y + 12582912.f;  // 1.5 * 2^23: round to nearest integer
  const float n = t - 12582912.f;
  const float f = y - n;
  float q = fmaf(0.05508868380750935f, f, 0.2426040514594784f);
  q = fmaf(q, f, 0.6932762416819616f);
  q = fmaf(q, f, 0.9999289403695111f);
  return __int_as_float(__float_as_int(q) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  __syncwarp();
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int D>
struct Cfg {
  static constexpr int kSlabs = D / 64;                  // 128-byte swizzle slabs per row
  static constexpr int kTileBytes = kM * D * 2;          // one Q / K / V tile in smem
  static constexpr int kSlabBytes = kM * 128;            // 128 rows x 128 B
  static constexpr int kNK = D == 128 ? 3 : 4;           // K ring stages (K(T+3) streams during S(T+1..T+2))
  static constexpr int kNV = D == 128 ? 2 : 3;           // V ring stages (V is consumed a softmax later)
  static constexpr int kNQ = 1;                          // Q staging buffer (copied to TMEM at item start)
  static constexpr int kSmemBytes = (kNQ + kNK + kNV) * kTileBytes + 1024;
};

struct TcParams {
  void *o;
  float *lse;
  int64_t o_row_stride;
  int64_t N;
  int batch, n_items, nql, G, n_sink;
  float scale_log2;
  const int32_t *win_q;
  const int32_t *items;  // (q-head, q-tile) LPT order
};

struct Bars {
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[4], k_empty[4];
  uint64_t v_full[4], v_empty[4];
  uint64_t s_full, s_free;          // S(T) computed / S(T) loaded into softmax registers
  uint64_t p_full[2], pv_done[2];
  uint64_t qt_full[2];              // Q of an item copied smem -> TMEM by the softmax warps
  uint64_t o_full, o_empty;
  uint32_t tmem_base;
};

struct Item {
  int b, h;
  int64_t i0, i1;
  int W;
  TileRanges tr;
};

__device__ __forceinline__ Item get_item(const TcParams &p, int idx) {
  Item it;
  const int wi = idx / p.batch;
  it.b = idx - wi * p.batch;
  it.h = p.items[2 * wi];
  const int qt = p.items[2 * wi + 1];
  it.i0 = (int64_t)qt * kM;
  it.i1 = (p.N < it.i0 + kM ? p.N : it.i0 + kM) - 1;
  it.W = p.win_q[it.h];
  it.tr = kv_tile_ranges(it.i0, it.i1, it.W, p.n_sink);
  return it;
}

// ------------------------------------------------------------------------------------------
// MMA issuer: whole warp 9 walks the schedule, one elected lane issues tcgen05 ops.
// Order per item: S(t) [then PV(t-1)] for each tile, PV(last).  S = Q K^T takes Q from
// TMEM (copied there by the softmax warps) and K from shared memory, so the QK^T MMA reads
// only K through the shared-memory port; S(t+1) reuses the single S buffer as soon as the
// softmax has loaded S(t) into registers (s_free), P is double-buffered.
// ------------------------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void mma_role(const TcParams &p, Bars &bars, uint32_t tmem, uint32_t k_smem,
                                         uint32_t v_smem, int total) {
  using C = Cfg<D>;
  constexpr uint32_t idesc_s = idesc_bf16_f32(kM, kN, false);
  constexpr uint32_t idesc_o = idesc_bf16_f32(kM, D, true);
  const uint64_t kdesc0 = smem_desc_sw128(k_smem, 16, 1024);
  const uint64_t vdesc0 = smem_desc_sw128(v_smem, C::kSlabBytes, 1024);
  int n = 0, T = 0;
  auto issue_pv = [&](int Tp, bool first_of_item, bool last_of_item, int item_n) {
    const int vs = Tp % C::kNV, pb = Tp & 1;
    mbar_wait_warp(smem_u32(&bars.v_full[vs]), (Tp / C::kNV) & 1);
    mbar_wait_warp(smem_u32(&bars.p_full[pb]), (Tp >> 1) & 1);
    if (first_of_item && item_n > 0) mbar_wait_warp(smem_u32(&bars.o_empty), (item_n - 1) & 1);
    tc_fence_after();
    // B = V tile, MN-major SW128: 16 keys = two 8-row groups of 1024 B; N slabs 16 KB apart
    const uint64_t vdesc = vdesc0 + (uint64_t)((vs * C::kTileBytes) >> 4);
    const uint32_t pcol = tmem + (pb ? kColP1 : kColP0);
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < kN / 16; ++kk)
        mma_ts(tmem + kColO, pcol + kk * 8, vdesc + (uint64_t)((kk * 2048) >> 4), idesc_o,
               (first_of_item && kk == 0) ? 0u : 1u);
      mma_commit(smem_u32(&bars.v_empty[vs]));
      mma_commit(smem_u32(&bars.pv_done[pb]));
      if (last_of_item) mma_commit(smem_u32(&bars.o_full));
    }
    __syncwarp();
  };
  for (int idx = blockIdx.x; idx < total; idx += gridDim.x, ++n) {
    const Item it = get_item(p, idx);
    const int qb = n & 1;
    mbar_wait_warp(smem_u32(&bars.qt_full[qb]), (n >> 1) & 1);  // Q(n) in TMEM
    const uint32_t qcol = tmem + (qb ? kColQ1 : kColQ0);
    const int nt = it.tr.count();
    for (int t = 0; t < nt; ++t, ++T) {
      const int ks = T % C::kNK;
      mbar_wait_warp(smem_u32(&bars.k_full[ks]), (T / C::kNK) & 1);
      if (T >= 1) mbar_wait_warp(smem_u32(&bars.s_free), (T - 1) & 1);  // S(T-1) read by the softmax
      tc_fence_after();
      const uint64_t kdesc = kdesc0 + (uint64_t)((ks * C::kTileBytes) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t koff = ((kk >> 2) * C::kSlabBytes + (kk & 3) * 32) >> 4;
          mma_ts(tmem + kColS, qcol + kk * 8, kdesc + koff, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(smem_u32(&bars.s_full));
        mma_commit(smem_u32(&bars.k_empty[ks]));
      }
      __syncwarp();
      if (t > 0) issue_pv(T - 1, t == 1, false, n);
    }
    issue_pv(T - 1, nt == 1, true, n);
  }
}

// ------------------------------------------------------------------------------------------
// softmax warpgroups: warps 0-3 take S columns [0, 64), warps 4-7 columns [64, 128) of the
// same rows (thread owns row = TMEM lane).  W is a runtime value so both warpgroups run one
// code path (the named barrier they share is a single program point).  At each item start
// they also copy the item's Q tile from shared memory (TMA, 128B swizzle) into TMEM.
// ------------------------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void softmax_role(const TcParams &p, Bars &bars, uint32_t tmem, uint32_t q_smem,
                                             int total, int tid, int warp, float (*red_max)[2][kM],
                                             float (*red_l)[kM]) {
  using C = Cfg<D>;
  const int W = warp >> 2;             // column half of this warpgroup
  const int row = tid & 127;
  const int lane = tid & 31;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int c0 = W * kHalf;            // first S column of this half
  const int oc0 = W * (D / 2);         // first O / Q column of this half
  int n = 0, T = 0;
  for (int idx = blockIdx.x; idx < total; idx += gridDim.x, ++n) {
    const Item it = get_item(p, idx);
    const int64_t i = it.i0 + row;
    const int nt = it.tr.count();
    // ---- Q(n): smem (swizzled rows) -> TMEM columns of this half, packed bf16 pairs
    {
      const int qb = n & 1;                       // TMEM Q buffer
      const int sq = n % C::kNQ;                  // smem staging buffer
      mbar_wait_warp(smem_u32(&bars.q_full[sq]), (n / C::kNQ) & 1);
      const uint32_t qs = q_smem + sq * C::kTileBytes;
      constexpr int kChunks = D / 16;  // 16-byte chunks of this half row
      uint32_t qr[D / 4];
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        const int gc = (oc0 / 8) + c;            // chunk index in the full row
        const int sl = gc >> 3, cc = gc & 7;     // 128-byte slab, chunk within the swizzle row
        const uint32_t addr = qs + sl * C::kSlabBytes + row * 128 + ((cc ^ (row & 7)) << 4);
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(qr[4 * c]), "=r"(qr[4 * c + 1]), "=r"(qr[4 * c + 2]), "=r"(qr[4 * c + 3])
                     : "r"(addr));
      }
      const uint32_t qa = tmem + lane_off + (qb ? kColQ1 : kColQ0) + oc0 / 2;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) tmem_st16(qa + c * 16, &qr[16 * c]);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(smem_u32(&bars.qt_full[qb]));
        mbar_arrive(smem_u32(&bars.q_empty[sq]));  // the smem Q buffer may be refilled
      }
    }
    float m_used = -INFINITY, l = 0.f;
    for (int t = 0; t < nt; ++t, ++T) {
      const int sb = T & 1;
      const int kt = it.tr.at(t);
      const int64_t j0 = (int64_t)kt * kN;
      const bool full = kv_tile_full(it.i0, it.i1, kt, it.W, p.n_sink);
      mbar_wait_warp(smem_u32(&bars.s_full), T & 1);
      tc_fence_after();
      uint32_t sr[kHalf];
      {
        const uint32_t sa = tmem + lane_off + kColS + c0;
        tmem_ld32(sa, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        tmem_ld32(sa + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_wait_ld();
      }
      // S is in registers: the tensor core may overwrite it with S(T+1)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars.s_free));
      float x[kHalf];
#pragma unroll
      for (int c = 0; c < kHalf; ++c) x[c] = __uint_as_float(sr[c]);
      if (!full) {
        // key j0+c visible to row i  <=>  c <= i-j0  and  (c < s-j0  or  c > i-j0-W)
        const int dd = (int)(i - j0) - c0, sl = (int)(p.n_sink - j0) - c0, lo = dd - it.W;
#pragma unroll
        for (int c = 0; c < kHalf; ++c) {
          const bool vis = c <= dd && (c < sl || c > lo);
          if (!vis) x[c] = -INFINITY;
        }
      }
      float mx[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) mx[k] = fmaxf(fmaxf(x[k], x[k + 16]), fmaxf(x[k + 32], x[k + 48]));
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) mx[k] = fmaxf(mx[k], mx[k + w]);
      // row max of both halves (raw scores; scale > 0 commutes with max)
      red_max[sb][W][row] = mx[0];
      named_bar_sync(kBarSoftmax, kSoftmaxThreads);
      const float mt = fmaxf(mx[0], red_max[sb][1 - W][row]) * p.scale_log2;
      bool rescale = false;
      float alpha = 1.f;
      if (m_used == -INFINITY) {
        m_used = mt;  // first visible scores of this row: O and l are still exactly 0
      } else if (mt > m_used + kRescaleThreshold) {
        rescale = true;
        alpha = fast_exp2(m_used - mt);
        m_used = mt;
      }
      if (__any_sync(0xffffffffu, rescale)) {
        // O must hold PV(T-1) before it is rescaled (this half of its columns)
        mbar_wait_warp(smem_u32(&bars.pv_done[(T - 1) & 1]), ((T - 1) >> 1) & 1);
        tc_fence_after();
        uint32_t r[32];
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          const uint32_t oa = tmem + lane_off + kColO + oc0 + c * 32;
          tmem_ld32(oa, r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
          tmem_st32(oa, r);
        }
      }
      l *= alpha;
      const float nmref = m_used == -INFINITY ? 0.f : -m_used;
      float ps[4] = {0.f, 0.f, 0.f, 0.f};
      // P[sb] was last read by PV(T-2), complete since S(T) completed (in-order tcgen05)
      const uint32_t pa = tmem + lane_off + (sb ? kColP1 : kColP0) + W * (kHalf / 2);
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int c = ch * 16 + e;
          // p = 2^(s * scale_log2 - m); a share of the exponentials runs on the FMA pipe
          const float ya = fmaf(x[2 * c], p.scale_log2, nmref);
          const float yb = fmaf(x[2 * c + 1], p.scale_log2, nmref);
          const float a = (c & kPolyMask) == kPolyMask ? exp2_poly(ya) : fast_exp2(ya);
          const float b2 = fast_exp2(yb);
          ps[e & 3] += a + b2;
          pk[e] = pack_bf16x2(a, b2);
        }
        tmem_st16(pa + ch * 16, pk);
      }
      l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars.p_full[sb]));
    }
    // epilogue: O / l -> bf16 rows (this half of the columns), lse
    red_l[W][row] = l;
    mbar_wait_warp(smem_u32(&bars.o_full), n & 1);
    named_bar_sync(kBarSoftmax, kSoftmaxThreads);
    const float lt = l + red_l[1 - W][row];
    tc_fence_after();
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    __nv_bfloat16 *orow = static_cast<__nv_bfloat16 *>(p.o) + ((int64_t)it.b * p.N + i) * p.o_row_stride +
                          (int64_t)it.h * D + oc0;
#pragma unroll
    for (int c = 0; c < D / 64; ++c) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + kColO + oc0 + c * 32, r);
      tmem_wait_ld();
      if (i <= it.i1) {
        uint4 *dst = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(r[8 * v4 + 0]) * inv, __uint_as_float(r[8 * v4 + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(r[8 * v4 + 2]) * inv, __uint_as_float(r[8 * v4 + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(r[8 * v4 + 4]) * inv, __uint_as_float(r[8 * v4 + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(r[8 * v4 + 6]) * inv, __uint_as_float(r[8 * v4 + 7]) * inv);
          dst[v4] = w;
        }
      }
    }
    if (W == 0 && p.lse && i <= it.i1)
      p.lse[((int64_t)it.b * p.nql + it.h) * p.N + i] = lt > 0.f ? (m_used + __log2f(lt)) * kLn2 : -INFINITY;
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars.o_empty));
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const TcParams p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ Bars bars;
  __shared__ float red_max[2][2][kM];  // [tile parity][half][row]
  __shared__ float red_l[2][kM];       // [half][row]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t q_smem = smem_base;                        // 2 tiles
  const uint32_t k_smem = q_smem + C::kNQ * C::kTileBytes;  // kNK tiles
  const uint32_t v_smem = k_smem + C::kNK * C::kTileBytes;  // kNV tiles
  const int total = p.n_items * p.batch;

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&bars.q_full[i]), 1);
      mbar_init(smem_u32(&bars.q_empty[i]), kSoftmaxWarps);
      mbar_init(smem_u32(&bars.p_full[i]), kSoftmaxWarps);
      mbar_init(smem_u32(&bars.pv_done[i]), 1);
      mbar_init(smem_u32(&bars.qt_full[i]), kSoftmaxWarps);
    }
    mbar_init(smem_u32(&bars.s_full), 1);
    mbar_init(smem_u32(&bars.s_free), kSoftmaxWarps);
    for (int i = 0; i < C::kNK; ++i) {
      mbar_init(smem_u32(&bars.k_full[i]), 1);
      mbar_init(smem_u32(&bars.k_empty[i]), 1);
    }
    for (int i = 0; i < C::kNV; ++i) {
      mbar_init(smem_u32(&bars.v_full[i]), 1);
      mbar_init(smem_u32(&bars.v_empty[i]), 1);
    }
    mbar_init(smem_u32(&bars.o_full), 1);
    mbar_init(smem_u32(&bars.o_empty), kSoftmaxWarps);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<kTmemCols>(smem_u32(&bars.tmem_base));
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp == 8 || warp == 10) {
    // ------------------------------------------------------------------ TMA producers
    if (lane == 0) {
      const bool kq = warp == 8;
      int n = 0, T = 0;
      for (int idx = blockIdx.x; idx < total; idx += gridDim.x, ++n) {
        const Item it = get_item(p, idx);
        const int g = it.h / p.G;
        if (kq) {
          const int qb = n % C::kNQ;
          if (n >= C::kNQ) mbar_wait(smem_u32(&bars.q_empty[qb]), ((n - C::kNQ) / C::kNQ) & 1);
          const uint32_t qbar = smem_u32(&bars.q_full[qb]);
          mbar_expect_tx(qbar, C::kTileBytes);
          for (int sl = 0; sl < C::kSlabs; ++sl)
            tma_load_4d(q_smem + qb * C::kTileBytes + sl * C::kSlabBytes, &tm_q, qbar, sl * 64, it.h, (int)it.i0,
                        it.b);
        }
        const int nt = it.tr.count();
        for (int t = 0; t < nt; ++t, ++T) {
          const int j0 = it.tr.at(t) * kN;
          if (kq) {
            const int ks = T % C::kNK;
            if (T >= C::kNK) mbar_wait(smem_u32(&bars.k_empty[ks]), ((T - C::kNK) / C::kNK) & 1);
            const uint32_t kbar = smem_u32(&bars.k_full[ks]);
            mbar_expect_tx(kbar, C::kTileBytes);
            for (int sl = 0; sl < C::kSlabs; ++sl)
              tma_load_4d(k_smem + ks * C::kTileBytes + sl * C::kSlabBytes, &tm_k, kbar, sl * 64, g, j0, it.b);
          } else {
            const int vs = T % C::kNV;
            if (T >= C::kNV) mbar_wait(smem_u32(&bars.v_empty[vs]), ((T - C::kNV) / C::kNV) & 1);
            const uint32_t vbar = smem_u32(&bars.v_full[vs]);
            mbar_expect_tx(vbar, C::kTileBytes);
            for (int sl = 0; sl < C::kSlabs; ++sl)
              tma_load_4d(v_smem + vs * C::kTileBytes + sl * C::kSlabBytes, &tm_v, vbar, sl * 64, g, j0, it.b);
          }
        }
      }
    }
  } else if (warp == 9) {
    mma_role<D>(p, bars, tmem, k_smem, v_smem, total);
  } else if (warp < 8) {
    softmax_role<D>(p, bars, tmem, q_smem, total, tid, warp, red_max, red_l);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

// ------------------------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// [B, N, H, D] bf16 with token row stride `row_stride` (elements): box = 64 cols x 128 rows, 128B swizzle.
bool make_map(CUtensorMap *m, const void *ptr, int D, int H, int64_t N, int B, int64_t row_stride) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)N, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)row_stride * 2, (cuuint64_t)(N * row_stride * 2)};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)kM, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

// [B, N, H, D] bf16 tensor map with 64-column x box_rows boxes (128-byte swizzle)
bool make_tile_map(void *m, const void *ptr, int D, int H, int64_t N, int B, int64_t row_stride, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)N, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)row_stride * 2, (cuuint64_t)(N * row_stride * 2)};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(static_cast<CUtensorMap *>(m), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(ptr), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_cache_map(void *map_out, const void *ptr, int D, int64_t rows, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(static_cast<CUtensorMap *>(map_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr),
                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int D>
int launch_d(const PrefillArgs &a, void *stream) {
  using C = Cfg<D>;
  CUtensorMap mq, mk, mv;
  const int ngl = a.nql / a.G;
  if (!make_map(&mq, a.q, D, a.nql, a.N, a.batch, a.q_row_stride) ||
      !make_map(&mk, a.k, D, ngl, a.N, a.batch, a.kv_row_stride) ||
      !make_map(&mv, a.v, D, ngl, a.N, a.batch, a.kv_row_stride))
    return (int)cudaErrorInvalidValue;
  TcParams p;
  p.o = a.o;
  p.lse = a.lse;
  p.o_row_stride = a.o_row_stride;
  p.N = a.N;
  p.batch = a.batch;
  p.n_items = a.n_items;
  p.nql = a.nql;
  p.G = a.G;
  p.n_sink = a.n_sink;
  p.scale_log2 = a.scale * kLog2e;
  p.win_q = a.d_win_q;
  p.items = a.d_items;
  cudaError_t e = cudaFuncSetAttribute(prefill_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::kSmemBytes);
  if (e != cudaSuccess) return (int)e;
  const int total = a.n_items * a.batch;
  const int grid = total < num_sms() ? total : num_sms();
  prefill_tc_kernel<D><<<grid, kThreads, C::kSmemBytes, (cudaStream_t)stream>>>(mq, mk, mv, p);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_prefill_bf16_tc(const PrefillArgs &a, void *stream) {
  if (a.d == 128) return launch_d<128>(a, stream);
  return launch_d<64>(a, stream);
}

}  // namespace moa
