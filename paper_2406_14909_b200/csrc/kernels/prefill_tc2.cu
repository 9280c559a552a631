// prefill_tc2.cu -- MoA causal prefill on CTA pairs (tcgen05 cta_group::2), head_dim 128.
//
//   O[b,i,h] = sum_{j in V(h,i)} softmax_j(tau q_i . k_j) v_j       (Eq. 1)
//   V(h,i)   = { j <= i : j < s  or  i - j < W_h }                   (reading c3)
//
// Same schedule and softmax as prefill_tc.cu, but a cluster of two CTAs (one per SM of a
// TPC) processes two adjacent 128-row q tiles of one (b, head) as one M = 256 tile:
//  * one thread of the leader CTA issues tcgen05.mma.cta_group::2 for both SMs
//    (S = Q K^T with M = 256, N = 128 keys; O += P V with M = 256, N = 128 = d);
//  * the K and V tiles of the union of the two q tiles' kv lists are loaded ONCE per pair:
//    each CTA loads half (K: 64 of the 128 keys; V: 64 of the 128 value columns) with
//    cp.async.bulk.tensor.cta_group::2 and signals the leader's mbarrier.  This halves
//    the L2->SM traffic and the shared-memory operand reads per FLOP of the 1-CTA kernel,
//    whose tile period is set by the K/V stream;
//  * each CTA keeps its own 128 rows: TMEM S0|S1|P0|P1|O, two softmax warpgroups split by
//    S columns (as in prefill_tc.cu), its own epilogue.  P handoffs and O-drained signals
//    go to the leader (remote mbarrier arrives), MMA completions are multicast to both.
// A q tile of the pair that is not in a kv tile's visible set simply masks that whole
// tile (the predicate does it), so the pair walks one shared tile list.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../moa_internal.h"
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace moa {

bool make_tile_map(void *m, const void *ptr, int D, int H, int64_t N, int B, int64_t row_stride, int box_rows);

namespace {

using namespace ptx;

constexpr int D = 128;
constexpr int kM = 128;                // q rows per CTA (MMA M per SM)
constexpr int kN = 128;                // keys per kv tile
constexpr int kHalf = 64;              // S columns per softmax warpgroup / K rows / V columns per CTA
constexpr int kSoftmaxThreads = 256;
constexpr int kThreads = 384;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColP0 = 256, kColP1 = 320, kColO = 384;
constexpr float kRescaleThreshold = 8.0f;
constexpr int kPolyMask = 1;
constexpr int kBarSoftmax = 1;
constexpr int kNQ = 2, kNK = 4, kNV = 4;
constexpr int kQBytes = kM * D * 2;          // 32 KB (2 slabs of 128 rows x 128 B)
constexpr int kKBytes = kHalf * D * 2;       // 16 KB (2 slabs of 64 rows x 128 B)
constexpr int kVBytes = kN * kHalf * 2;      // 16 KB (1 slab of 128 rows x 128 B)
constexpr int kSmemBytes = kNQ * kQBytes + kNK * kKBytes + kNV * kVBytes + 1024;
constexpr uint16_t kBoth = 0x3;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the same offset in CTA rank 0
constexpr int kWarpArrivals = 16;            // 8 softmax warps x 2 CTAs

__device__ __forceinline__ float exp2_poly(float y) {
  y = fmaxf(y, -126.f);
  const float t = y + 12582912.f;
  const float n = t - 12582912.f;
  const float f = y - n;
  float q = fmaf(0.05508868380750935f, f, 0.2426040514594784f);
  q = fmaf(q, f, 0.6932762416819616f);
  q = fmaf(q, f, 0.9999289403695111f);
  return __int_as_float(__float_as_int(q) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  __syncwarp();
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// arrive on the leader CTA's copy of a barrier (local if this is the leader)
__device__ __forceinline__ void arrive_leader(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar & kPeerMask) : "memory");
}
__device__ __forceinline__ void tma2_load_4d(uint32_t dst, const CUtensorMap *m, uint32_t bar, int c0, int c1, int c2,
                                             int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar & kPeerMask)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(kBoth)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// debug tracing (env MOA_PREFILL_TRACE=1): (clock << 8 | code) of cluster 0
__device__ unsigned long long *g_trace2 = nullptr;
__shared__ unsigned int s_tn[6];
__device__ __forceinline__ void tr(int role, int code) {
  unsigned long long *t = g_trace2;
  if (t && blockIdx.x < 2) {
    const unsigned long long c = clock64();
    const unsigned int k = s_tn[role]++;
    if (k < 8000) t[1 + (role + 6 * blockIdx.x) * 8000 + k] = (c << 8) | (unsigned long long)code;
  }
}

struct P2 {
  void *o;
  float *lse;
  int64_t o_row_stride;
  int64_t N;
  int batch, n_items, nql, G, n_sink;
  float scale_log2;
  const int32_t *win_q;
  const int32_t *pairs;  // (q-head, q-tile pair)
};

struct Bars {
  uint64_t q_full[kNQ], q_empty[kNQ];
  uint64_t k_full[kNK], k_empty[kNK];
  uint64_t v_full[kNV], v_empty[kNV];
  uint64_t s_full[2], p_full[2], pv_done[2];
  uint64_t o_full, o_empty;
  uint32_t tmem_base;
};

struct Item {
  int b, h;
  bool has;              // this CTA's q tile exists
  int64_t i0, i1;        // this CTA's rows
  int64_t pi0, pi1;      // the pair's rows
  int W;
  TileRanges tu;         // union kv list (the K/V stream of the pair)
};

__device__ __forceinline__ Item get_item(const P2 &p, int idx, int rank) {
  Item it;
  const int wi = idx / p.batch;
  it.b = idx - wi * p.batch;
  it.h = p.pairs[2 * wi];
  const int qp = p.pairs[2 * wi + 1];
  it.W = p.win_q[it.h];
  it.pi0 = (int64_t)qp * 2 * kM;
  it.pi1 = (p.N < it.pi0 + 2 * kM ? p.N : it.pi0 + 2 * kM) - 1;
  it.i0 = it.pi0 + (int64_t)rank * kM;
  it.has = it.i0 < p.N;
  it.i1 = (p.N < it.i0 + kM ? p.N : it.i0 + kM) - 1;
  it.tu = kv_tile_ranges(it.pi0, it.pi1, it.W, p.n_sink);
  return it;
}

// ------------------------------------------------------------------------------------------ MMA (leader)
__device__ __forceinline__ void mma_role(const P2 &p, Bars &bars, uint32_t tmem, uint32_t q_smem, uint32_t k_smem,
                                         uint32_t v_smem, int total, int cid, int ncl) {
  // S: M=256 (Q rows of both CTAs), N=128 keys, K-major A and B; PV: M=256, N=128 (d), B MN-major
  constexpr uint32_t idesc_s = idesc_bf16_f32(2 * kM, kN, false);
  constexpr uint32_t idesc_o = idesc_bf16_f32(2 * kM, D, true);
  const uint64_t qdesc0 = smem_desc_sw128(q_smem, 16, 1024);
  const uint64_t kdesc0 = smem_desc_sw128(k_smem, 16, 1024);
  const uint64_t vdesc0 = smem_desc_sw128(v_smem, 16, 1024);
  int n = 0, T = 0;
  auto issue_pv = [&](int Tp, bool first, bool last, int item_n) {
    const int vs = Tp % kNV, pb = Tp & 1;
    mbar_wait_warp(smem_u32(&bars.v_full[vs]), (Tp / kNV) & 1);
    mbar_wait_warp(smem_u32(&bars.p_full[pb]), (Tp >> 1) & 1);
    if ((threadIdx.x & 31) == 0) tr(0, 50);
    if (first && item_n > 0) mbar_wait_warp(smem_u32(&bars.o_empty), (item_n - 1) & 1);
    tc_fence_after();
    const uint64_t vdesc = vdesc0 + (uint64_t)((vs * kVBytes) >> 4);
    const uint32_t pcol = tmem + (pb ? kColP1 : kColP0);
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < kN / 16; ++kk)  // 16 keys = two 8-row groups of 1024 B
        mma2_ts(tmem + kColO, pcol + kk * 8, vdesc + (uint64_t)((kk * 2048) >> 4), idesc_o,
                (first && kk == 0) ? 0u : 1u);
      commit2(smem_u32(&bars.v_empty[vs]));
      commit2(smem_u32(&bars.pv_done[pb]));
      if (last) commit2(smem_u32(&bars.o_full));
      tr(0, 20);
    }
    __syncwarp();
  };
  for (int idx = cid; idx < total; idx += ncl, ++n) {
    const Item it = get_item(p, idx, 0);
    const int qb = n % kNQ;
    mbar_wait_warp(smem_u32(&bars.q_full[qb]), (n / kNQ) & 1);
    const uint64_t qdesc = qdesc0 + (uint64_t)((qb * kQBytes) >> 4);
    const int nt = it.tu.count();
    for (int t = 0; t < nt; ++t, ++T) {
      const int ks = T % kNK, sb = T & 1;
      mbar_wait_warp(smem_u32(&bars.k_full[ks]), (T / kNK) & 1);
      if ((threadIdx.x & 31) == 0) tr(0, 60);
      if (T >= 2) mbar_wait_warp(smem_u32(&bars.p_full[sb]), ((T - 2) >> 1) & 1);  // S[sb] consumed (both CTAs)
      if ((threadIdx.x & 31) == 0) tr(0, 61);
      tc_fence_after();
      const uint64_t kdesc = kdesc0 + (uint64_t)((ks * kKBytes) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          // Q slabs are 128 rows x 128 B (16 KB); K half-tile slabs 64 rows x 128 B (8 KB)
          const uint32_t qoff = ((kk >> 2) * (kM * 128) + (kk & 3) * 32) >> 4;
          const uint32_t koff = ((kk >> 2) * (kHalf * 128) + (kk & 3) * 32) >> 4;
          mma2_ss(tmem + (sb ? kColS1 : kColS0), qdesc + qoff, kdesc + koff, idesc_s, kk > 0 ? 1u : 0u);
        }
        commit2(smem_u32(&bars.s_full[sb]));
        commit2(smem_u32(&bars.k_empty[ks]));
        if (t == nt - 1) commit2(smem_u32(&bars.q_empty[qb]));
        tr(0, 10);
      }
      __syncwarp();
      if (t > 0) issue_pv(T - 1, t == 1, false, n);
    }
    issue_pv(T - 1, nt == 1, true, n);
  }
}

// ------------------------------------------------------------------------------------------ softmax
__device__ __forceinline__ void softmax_role(const P2 &p, Bars &bars, uint32_t tmem, int total, int cid, int ncl,
                                             int rank, int tid, int warp, float (*red_max)[2][kM],
                                             float (*red_l)[kM]) {
  const int W = warp >> 2;
  const int row = tid & 127;
  const int lane = tid & 31;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int c0 = W * kHalf;
  const int oc0 = W * (D / 2);
  int n = 0, T = 0;
  for (int idx = cid; idx < total; idx += ncl, ++n) {
    const Item it = get_item(p, idx, rank);
    const int64_t i = it.i0 + row;
    const int nt = it.tu.count();
    float m_used = -INFINITY, l = 0.f;
    for (int t = 0; t < nt; ++t, ++T) {
      const int sb = T & 1;
      const int kt = it.tu.at(t);
      const int64_t j0 = (int64_t)kt * kN;
      const bool full = it.has && kv_tile_full(it.i0, it.i1, kt, it.W, p.n_sink);
      mbar_wait_warp(smem_u32(&bars.s_full[sb]), (T >> 1) & 1);
      tc_fence_after();
      if (row == 0) tr(1 + W, 30 + W);
      uint32_t sr[kHalf];
      {
        const uint32_t sa = tmem + lane_off + (sb ? kColS1 : kColS0) + c0;
        tmem_ld32(sa, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        tmem_ld32(sa + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_wait_ld();
      }
      float x[kHalf];
#pragma unroll
      for (int c = 0; c < kHalf; ++c) x[c] = __uint_as_float(sr[c]);
      if (!full) {
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
      red_max[sb][W][row] = mx[0];
      named_bar_sync(kBarSoftmax, kSoftmaxThreads);
      const float mt = fmaxf(mx[0], red_max[sb][1 - W][row]) * p.scale_log2;
      bool rescale = false;
      float alpha = 1.f;
      if (m_used == -INFINITY) {
        m_used = mt;
      } else if (mt > m_used + kRescaleThreshold) {
        rescale = true;
        alpha = fast_exp2(m_used - mt);
        m_used = mt;
      }
      if (__any_sync(0xffffffffu, rescale)) {
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
      const uint32_t pa = tmem + lane_off + (sb ? kColP1 : kColP0) + W * (kHalf / 2);
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int c = ch * 16 + e;
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
      if (row == 0) tr(1 + W, 40 + W);
      if (lane == 0) arrive_leader(smem_u32(&bars.p_full[sb]));
    }
    // epilogue
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
      if (it.has && i <= it.i1) {
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
    if (W == 0 && p.lse && it.has && i <= it.i1)
      p.lse[((int64_t)it.b * p.nql + it.h) * p.N + i] = lt > 0.f ? (m_used + __log2f(lt)) * kLn2 : -INFINITY;
    tc_fence_before();
    __syncwarp();
    if (lane == 0) arrive_leader(smem_u32(&bars.o_empty));
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    prefill_tc2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const P2 p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Bars bars;
  __shared__ float red_max[2][2][kM];
  __shared__ float red_l[2][kM];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t q_smem = smem_base;
  const uint32_t k_smem = q_smem + kNQ * kQBytes;
  const uint32_t v_smem = k_smem + kNK * kKBytes;
  const int total = p.n_items * p.batch;

  if (tid == 0) {
    for (int i = 0; i < 6; ++i) s_tn[i] = 0;
    for (int i = 0; i < kNQ; ++i) {
      mbar_init(smem_u32(&bars.q_full[i]), 1);
      mbar_init(smem_u32(&bars.q_empty[i]), 1);
    }
    for (int i = 0; i < kNK; ++i) {
      mbar_init(smem_u32(&bars.k_full[i]), 1);
      mbar_init(smem_u32(&bars.k_empty[i]), 1);
    }
    for (int i = 0; i < kNV; ++i) {
      mbar_init(smem_u32(&bars.v_full[i]), 1);
      mbar_init(smem_u32(&bars.v_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&bars.s_full[i]), 1);
      mbar_init(smem_u32(&bars.p_full[i]), kWarpArrivals);
      mbar_init(smem_u32(&bars.pv_done[i]), 1);
    }
    mbar_init(smem_u32(&bars.o_full), 1);
    mbar_init(smem_u32(&bars.o_empty), kWarpArrivals);
    fence_mbar_init();
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bars.tmem_base)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised and TMEM allocated before any cross-CTA traffic
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp == 8 || warp == 10) {
    // TMA producers of this CTA's halves; the leader arms the full barriers for both
    if (lane == 0) {
      const bool kq = warp == 8;
      int n = 0, T = 0;
      for (int idx = cid; idx < total; idx += ncl, ++n) {
        const Item it = get_item(p, idx, rank);
        const int g = it.h / p.G;
        if (kq) {
          const int qb = n % kNQ;
          if (n >= kNQ) mbar_wait(smem_u32(&bars.q_empty[qb]), ((n - kNQ) / kNQ) & 1);
          const uint32_t qbar = smem_u32(&bars.q_full[qb]);
          if (rank == 0) mbar_expect_tx(qbar, 2 * kQBytes);
          for (int sl = 0; sl < D / 64; ++sl)
            tma2_load_4d(q_smem + qb * kQBytes + sl * (kM * 128), &tm_q, qbar, sl * 64, it.h, (int)it.i0, it.b);
        }
        const int nt = it.tu.count();
        for (int t = 0; t < nt; ++t, ++T) {
          const int j0 = it.tu.at(t) * kN;
          if (kq) {
            const int ks = T % kNK;
            if (T >= kNK) mbar_wait(smem_u32(&bars.k_empty[ks]), ((T - kNK) / kNK) & 1);
            const uint32_t kbar = smem_u32(&bars.k_full[ks]);
            if (rank == 0) mbar_expect_tx(kbar, 2 * kKBytes);
            tr(3, 80);
            for (int sl = 0; sl < D / 64; ++sl)  // keys [j0 + 64 rank, +64), columns [64 sl, +64)
              tma2_load_4d(k_smem + ks * kKBytes + sl * (kHalf * 128), &tm_k, kbar, sl * 64, g, j0 + kHalf * rank,
                           it.b);
          } else {
            const int vs = T % kNV;
            if (T >= kNV) mbar_wait(smem_u32(&bars.v_empty[vs]), ((T - kNV) / kNV) & 1);
            const uint32_t vbar = smem_u32(&bars.v_full[vs]);
            if (rank == 0) mbar_expect_tx(vbar, 2 * kVBytes);
            tr(4, 81);
            // keys [j0, j0+128), value columns [64 rank, +64)
            tma2_load_4d(v_smem + vs * kVBytes, &tm_v, vbar, kHalf * rank, g, j0, it.b);
          }
        }
      }
    }
  } else if (warp == 9) {
    if (rank == 0) mma_role(p, bars, tmem, q_smem, k_smem, v_smem, total, cid, ncl);
  } else if (warp < 8) {
    softmax_role(p, bars, tmem, total, cid, ncl, rank, tid, warp, red_max, red_l);
  }

  tc_fence_before();
  __syncwarp();
  cluster_sync();  // no CTA of the pair frees TMEM or exits while the other may still signal it
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
  }
}

int num_sms2() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

int launch_prefill_bf16_tc2(const PrefillArgs &a, void *stream) {
  alignas(64) CUtensorMap mq, mk, mv;
  const int ngl = a.nql / a.G;
  if (!make_tile_map(&mq, a.q, D, a.nql, a.N, a.batch, a.q_row_stride, kM) ||
      !make_tile_map(&mk, a.k, D, ngl, a.N, a.batch, a.kv_row_stride, kHalf) ||
      !make_tile_map(&mv, a.v, D, ngl, a.N, a.batch, a.kv_row_stride, kN))
    return (int)cudaErrorInvalidValue;
  P2 p;
  p.o = a.o;
  p.lse = a.lse;
  p.o_row_stride = a.o_row_stride;
  p.N = a.N;
  p.batch = a.batch;
  p.n_items = a.n_pairs;
  p.nql = a.nql;
  p.G = a.G;
  p.n_sink = a.n_sink;
  p.scale_log2 = a.scale * kLog2e;
  p.win_q = a.d_win_q;
  p.pairs = a.d_pairs;
  cudaError_t e = cudaFuncSetAttribute(prefill_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (e != cudaSuccess) return (int)e;
  const int total = a.n_pairs * a.batch;
  static unsigned long long *trace_buf = nullptr;
  static bool trace_on = std::getenv("MOA_PREFILL_TRACE") != nullptr;
  const size_t tbytes = (size_t)(1 + 12 * 8000) * 8;
  if (trace_on) {
    if (!trace_buf) cudaMalloc(&trace_buf, tbytes);
    cudaMemsetAsync(trace_buf, 0, tbytes, (cudaStream_t)stream);
    cudaMemcpyToSymbolAsync(g_trace2, &trace_buf, sizeof(trace_buf), 0, cudaMemcpyHostToDevice, (cudaStream_t)stream);
  }
  int clusters = num_sms2() / 2;
  if (clusters > total) clusters = total;
  prefill_tc2_kernel<<<2 * clusters, kThreads, kSmemBytes, (cudaStream_t)stream>>>(mq, mk, mv, p);
  if (trace_on) {
    std::vector<unsigned long long> h(1 + 12 * 8000);
    cudaMemcpy(h.data(), trace_buf, tbytes, cudaMemcpyDeviceToHost);
    FILE *f = fopen("gpurun_out/prefill_trace2.txt", "w");
    if (f) {
      for (size_t k = 1; k < h.size(); ++k)
        if (h[k]) fprintf(f, "%zu %llu %llu\n", (k - 1) / (6 * 8000), h[k] >> 8, h[k] & 255);
      fclose(f);
    }
  }
  return (int)cudaGetLastError();
}

}  // namespace moa
