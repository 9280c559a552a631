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
// Work item = two adjacent 128-row q tiles (Q0, Q1) of one (b, head): their kv
// tile lists differ by at most one tile at each end, so one TMA stream of K/V
// tiles (the union) feeds both.  Persistent CTAs (one per SM) walk a static
// round-robin slice of the LPT-sorted item list.  Warp roles (384 threads):
//   warps 0-3   softmax of Q0 (thread t owns row t = TMEM lane t)
//   warps 4-7   softmax of Q1
//   warp 8      TMA producer of Q0/Q1 and the K ring; warp 10: producer of the V ring
//   warp 9      TMEM allocator + single-thread MMA issuer
// TMEM (512 columns): S0 (128 fp32, P0 aliased as 64 packed bf16x2 columns) |
// O0 (D) | S1/P1 | O1.  The MMA issue order S0(k) S1(k) | PV0(k) S0(k+1) |
// PV1(k) S1(k+1) | ... keeps the tensor pipe busy with one Q tile while the
// other tile's softmax runs (ping-pong).  tcgen05 ops of one thread complete in
// issue order and a commit tracks all earlier ops, so "S_q(k+1) complete"
// implies "PV_q(k) complete": P may overwrite S and O may be rescaled without
// extra barriers.  The running max is refreshed (and O rescaled in TMEM) only
// when it grows by more than 2^8; a share of the exponentials runs as a
// polynomial on the FMA pipe (MUFU ex2 is as slow as the tensor core here).
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

constexpr int kM = 128;                // q rows per tile (MMA M)
constexpr int kN = 128;                // keys per tile (MMA N of QK^T, K of PV)
constexpr int kSoftmaxThreads = 128;   // one warpgroup per q tile
constexpr int kThreads = 3 * 128;
constexpr uint32_t kTmemCols = 512;
constexpr int kRegsSoftmax = 208, kRegsOther = 88;
// setmaxnreg.inc blocks until the CTA's pool (launch allocation: 168 x 384) has the registers
static_assert(256 * kRegsSoftmax + 128 * kRegsOther <= 168 * 384, "register split exceeds the CTA pool");
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only if the max grows by > 2^8
// exponentials of pairs c with (c & kPolyMask) == kPolyMask use the FMA-pipe polynomial
constexpr int kPolyMask = 1;

__host__ __device__ constexpr uint32_t col_s(int q) { return q ? 256u : 0u; }
__host__ __device__ constexpr uint32_t col_o(int q) { return q ? 384u : 128u; }

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

template <int D>
struct Cfg {
  static constexpr int kSlabs = D / 64;                  // 128-byte swizzle slabs per row
  static constexpr int kTileBytes = kM * D * 2;          // one Q / K / V tile in smem
  static constexpr int kSlabBytes = kM * 128;            // 128 rows x 128 B
  static constexpr int kNK = D == 128 ? 2 : 3;           // K ring stages
  static constexpr int kNV = D == 128 ? 3 : 3;           // V ring stages
  static constexpr int kSmemBytes = (2 + kNK + kNV) * kTileBytes + 1024;
};

struct TcParams {
  void *o;
  float *lse;
  int64_t o_row_stride;
  int64_t N;
  int batch, n_items, nql, G, n_sink;
  float scale_log2;
  const int32_t *win_q;
  const int32_t *items;  // (q-head, q-tile pair) LPT order
};

// debug tracing (env MOA_PREFILL_TRACE=1): (clock << 8 | event code) of CTA 0
__device__ unsigned long long *g_trace = nullptr;
__shared__ unsigned int s_trace_n[3];  // per role (MMA, softmax 0, softmax 1) event counters
__device__ __forceinline__ void trace_ev(int code) {
  unsigned long long *tr = g_trace;
  if (tr && blockIdx.x == 0) {
    const unsigned long long t = clock64();
    const int role = code >= 30 && code < 50 ? 1 + (code & 1) : 0;
    const unsigned int k = s_trace_n[role]++;
    if (k < 20000) tr[1 + role * 20000 + k] = (t << 8) | (unsigned long long)code;
  }
}

struct Bars {
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[4], k_empty[4];
  uint64_t v_full[4], v_empty[4];
  uint64_t s_full[2], p_full[2];
  uint64_t o_full[2], o_empty[2];
  uint32_t tmem_base;
};

struct Item {
  int b, h;
  bool has[2];          // q tile present
  int64_t i0[2], i1[2]; // first / last real row of each q tile
  int W;
  TileRanges tq[2];     // per q tile kv lists
  TileRanges tu;        // union (the K/V stream)
};

__device__ __forceinline__ bool in_ranges(const TileRanges &r, int t) {
  return (t >= r.a0 && t < r.a1) || (t >= r.b0 && t < r.b1);
}

__device__ __forceinline__ Item get_item(const TcParams &p, int idx) {
  Item it;
  const int wi = idx / p.batch;
  it.b = idx - wi * p.batch;
  it.h = p.items[2 * wi];
  const int qp = p.items[2 * wi + 1];
  it.W = p.win_q[it.h];
  for (int q = 0; q < 2; ++q) {
    it.i0[q] = (int64_t)(2 * qp + q) * kM;
    it.has[q] = it.i0[q] < p.N;
    it.i1[q] = (p.N < it.i0[q] + kM ? p.N : it.i0[q] + kM) - 1;
    if (it.has[q]) {
      it.tq[q] = kv_tile_ranges(it.i0[q], it.i1[q], it.W, p.n_sink);
    } else {
      it.tq[q].a0 = it.tq[q].a1 = it.tq[q].b0 = it.tq[q].b1 = 0;
    }
  }
  it.tu = kv_tile_ranges(it.i0[0], it.has[1] ? it.i1[1] : it.i1[0], it.W, p.n_sink);
  return it;
}


// ------------------------------------------------------------------------------------------
// MMA issuer (one thread).  Per q tile: S_q(list[k]) then, once P_q(k) is in TMEM, PV_q(k)
// followed by S_q(k+1).  Both q tiles interleave: S0 S1 | PV0 S0' | PV1 S1' | ...
// ------------------------------------------------------------------------------------------
struct MmaQ {
  int n = 0;        // tiles of this q tile in the current item
  int s_next = 0;   // next S to issue
  int pv_next = 0;  // next PV to issue
  int pcnt = 0;     // P handoffs consumed (global)
  int ocnt = 0;     // items finished (global)
  int qcnt = 0;     // Q loads consumed (global)
};

template <int D, int Q>
__device__ __forceinline__ int union_index(const Item &it, int k) {
  const int t = it.tq[Q].at(k);
  return t < it.tu.a1 ? t - it.tu.a0 : (it.tu.a1 - it.tu.a0) + (t - it.tu.b0);
}

__device__ __forceinline__ uint32_t users_of(const Item &it, int u) {
  const int t = it.tu.at(u);
  return (in_ranges(it.tq[0], t) ? 1u : 0u) | (in_ranges(it.tq[1], t) ? 2u : 0u);
}

template <int D, int Q>
__device__ __forceinline__ void issue_s(const Item &it, MmaQ &st, int T0, uint32_t &kbits, Bars &bars,
                                        uint32_t tmem, uint64_t qdesc, uint64_t kdesc0) {
  using C = Cfg<D>;
  constexpr uint32_t idesc_s = idesc_bf16_f32(kM, kN, false);
  const int u = union_index<D, Q>(it, st.s_next);
  const int Tu = T0 + u, ks = Tu % C::kNK;
  mbar_wait(smem_u32(&bars.k_full[ks]), (Tu / C::kNK) & 1);
  if ((threadIdx.x & 31) == 0) trace_ev(60 + Q);
  tc_fence_after();
  // descriptors: the 14-bit start-address field advances by (byte offset >> 4)
  const uint64_t kdesc = kdesc0 + (uint64_t)((ks * C::kTileBytes) >> 4);
  kbits |= (1u << Q) << (2 * ks);
  const bool k_done = ((kbits >> (2 * ks)) & 3u) == users_of(it, u);  // every user of this K stage issued
  if (k_done) kbits &= ~(3u << (2 * ks));
  const bool q_done = ++st.s_next == st.n;
  if (elect_one()) {
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint32_t off = ((kk >> 2) * C::kSlabBytes + (kk & 3) * 32) >> 4;
      mma_ss(tmem + col_s(Q), qdesc + off, kdesc + off, idesc_s, kk > 0 ? 1u : 0u);
    }
    mma_commit(smem_u32(&bars.s_full[Q]));
    if (k_done) mma_commit(smem_u32(&bars.k_empty[ks]));
    if (q_done) mma_commit(smem_u32(&bars.q_empty[Q]));
    trace_ev(10 + Q);
  }
  __syncwarp();
}

template <int D, int Q>
__device__ __forceinline__ void issue_pv(const Item &it, MmaQ &st, int T0, uint32_t &vbits, Bars &bars,
                                         uint32_t tmem, uint64_t vdesc0) {
  using C = Cfg<D>;
  constexpr uint32_t idesc_o = idesc_bf16_f32(kM, D, true);
  const int u = union_index<D, Q>(it, st.pv_next);
  const int Tu = T0 + u, vs = Tu % C::kNV;
  mbar_wait(smem_u32(&bars.v_full[vs]), (Tu / C::kNV) & 1);
  mbar_wait(smem_u32(&bars.p_full[Q]), st.pcnt & 1);
  if ((threadIdx.x & 31) == 0) trace_ev(50 + Q);
  ++st.pcnt;
  if (st.pv_next == 0 && st.ocnt > 0) mbar_wait(smem_u32(&bars.o_empty[Q]), (st.ocnt - 1) & 1);
  tc_fence_after();
  // B = V tile, MN-major SW128: 16 keys = two 8-row groups of 1024 B; N slabs 16 KB apart
  const uint64_t vdesc = vdesc0 + (uint64_t)((vs * C::kTileBytes) >> 4);
  const uint32_t acc0 = st.pv_next == 0 ? 0u : 1u;
  vbits |= (1u << Q) << (2 * vs);
  const bool v_done = ((vbits >> (2 * vs)) & 3u) == users_of(it, u);
  if (v_done) vbits &= ~(3u << (2 * vs));
  const bool o_done = ++st.pv_next == st.n;
  if (o_done) ++st.ocnt;
  if (elect_one()) {
#pragma unroll
    for (int kk = 0; kk < kN / 16; ++kk)
      mma_ts(tmem + col_o(Q), tmem + col_s(Q) + kk * 8, vdesc + (uint64_t)((kk * 2048) >> 4), idesc_o,
             kk == 0 ? acc0 : 1u);
    if (v_done) mma_commit(smem_u32(&bars.v_empty[vs]));
    if (o_done) mma_commit(smem_u32(&bars.o_full[Q]));
    trace_ev(20 + Q);
  }
  __syncwarp();
}

template <int D>
__device__ __forceinline__ void mma_role(const TcParams &p, Bars &bars, uint32_t tmem, uint32_t q_smem,
                                        uint32_t k_smem, uint32_t v_smem, int total) {
  using C = Cfg<D>;
  const uint64_t qdesc0 = smem_desc_sw128(q_smem, 16, 1024);
  const uint64_t qdesc1 = smem_desc_sw128(q_smem + C::kTileBytes, 16, 1024);
  const uint64_t kdesc0 = smem_desc_sw128(k_smem, 16, 1024);
  const uint64_t vdesc0 = smem_desc_sw128(v_smem, C::kSlabBytes, 1024);
  MmaQ q0, q1;
  uint32_t kbits = 0, vbits = 0;
  int T = 0;
  for (int idx = blockIdx.x; idx < total; idx += gridDim.x) {
    const Item it = get_item(p, idx);
    const int T0 = T;
    q0.n = it.tq[0].count();
    q1.n = it.tq[1].count();
    q0.s_next = q0.pv_next = q1.s_next = q1.pv_next = 0;
    if (q0.n) mbar_wait(smem_u32(&bars.q_full[0]), q0.qcnt++ & 1);
    if (q1.n) mbar_wait(smem_u32(&bars.q_full[1]), q1.qcnt++ & 1);
    if (q0.n) issue_s<D, 0>(it, q0, T0, kbits, bars, tmem, qdesc0, kdesc0);
    if (q1.n) issue_s<D, 1>(it, q1, T0, kbits, bars, tmem, qdesc1, kdesc0);
    while (q0.pv_next < q0.n || q1.pv_next < q1.n) {
      if (q0.pv_next < q0.n) {
        issue_pv<D, 0>(it, q0, T0, vbits, bars, tmem, vdesc0);
        if (q0.s_next < q0.n) issue_s<D, 0>(it, q0, T0, kbits, bars, tmem, qdesc0, kdesc0);
      }
      if (q1.pv_next < q1.n) {
        issue_pv<D, 1>(it, q1, T0, vbits, bars, tmem, vdesc0);
        if (q1.s_next < q1.n) issue_s<D, 1>(it, q1, T0, kbits, bars, tmem, qdesc1, kdesc0);
      }
    }
    T = T0 + it.tu.count();
  }
}

// ------------------------------------------------------------------------------------------
// softmax warpgroup of q tile Q: thread t owns row t (TMEM lane t)
// ------------------------------------------------------------------------------------------
template <int D, int Q>
__device__ __forceinline__ void softmax_role(const TcParams &p, Bars &bars, uint32_t tmem, int total, int tid,
                                             int warp) {
  const int row = tid & 127;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  int scnt = 0, ocnt = 0;
  for (int idx = blockIdx.x; idx < total; idx += gridDim.x) {
    const Item it = get_item(p, idx);
    if (!it.has[Q]) continue;
    const int64_t i0 = it.i0[Q], i1 = it.i1[Q];
    const TileRanges tr = it.tq[Q];
    const int64_t i = i0 + row;
    const int nt = tr.count();
    float m_used = -INFINITY, l = 0.f;
    for (int t = 0; t < nt; ++t, ++scnt) {
      const int kt = tr.at(t);
      const int64_t j0 = (int64_t)kt * kN;
      const bool full = kv_tile_full(i0, i1, kt, it.W, p.n_sink);
      mbar_wait(smem_u32(&bars.s_full[Q]), scnt & 1);
      tc_fence_after();
      if (row == 0) trace_ev(30 + Q);
      // S row -> registers: four 32-column TMEM loads in flight, one wait
      uint32_t sr[kN];
      {
        const uint32_t sa = tmem + lane_off + col_s(Q);
#pragma unroll
        for (int c = 0; c < kN / 32; ++c) tmem_ld32(sa + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
        tmem_wait_ld();
      }
      float x[kN];
#pragma unroll
      for (int c = 0; c < kN; ++c) x[c] = __uint_as_float(sr[c]);
      if (!full) {
        // key j0+c visible to row i  <=>  c <= i-j0  and  (c < s-j0  or  c > i-j0-W)
        const int dd = (int)(i - j0), sl = (int)(p.n_sink - j0), lo = dd - it.W;
#pragma unroll
        for (int c = 0; c < kN; ++c) {
          const bool vis = c <= dd && (c < sl || c > lo);
          if (!vis) x[c] = -INFINITY;
        }
      }
      // row max of the raw scores (tree), scaled to log2 units (scale > 0 commutes with max)
      float mx[16];
#pragma unroll
      for (int k = 0; k < 16; ++k)
        mx[k] = fmaxf(fmaxf(fmaxf(x[k], x[k + 16]), fmaxf(x[k + 32], x[k + 48])),
                      fmaxf(fmaxf(x[k + 64], x[k + 80]), fmaxf(x[k + 96], x[k + 112])));
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) mx[k] = fmaxf(mx[k], mx[k + w]);
      const float mt = mx[0] * p.scale_log2;
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
        // S_Q(t) complete => PV_Q(t-1) complete (in-order tcgen05): O is final for t-1
        uint32_t r[32];
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          const uint32_t oa = tmem + lane_off + col_o(Q) + c * 32;
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
      const uint32_t pa = tmem + lane_off + col_s(Q);  // P aliases the first 64 S columns
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
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
      if (row == 0) trace_ev(40 + Q);
      mbar_arrive(smem_u32(&bars.p_full[Q]));
    }
    // epilogue: O / l -> bf16 rows, lse
    mbar_wait(smem_u32(&bars.o_full[Q]), ocnt & 1);
    ++ocnt;
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16 *orow =
        static_cast<__nv_bfloat16 *>(p.o) + ((int64_t)it.b * p.N + i) * p.o_row_stride + (int64_t)it.h * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + col_o(Q) + c * 32, r);
      tmem_wait_ld();
      if (i <= i1) {
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
    if (p.lse && i <= i1)
      p.lse[((int64_t)it.b * p.nql + it.h) * p.N + i] = l > 0.f ? (m_used + __log2f(l)) * kLn2 : -INFINITY;
    tc_fence_before();
    mbar_arrive(smem_u32(&bars.o_empty[Q]));
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const TcParams p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ Bars bars;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t q_smem = smem_base;                                   // Q0, Q1
  const uint32_t k_smem = q_smem + 2 * C::kTileBytes;                  // kNK tiles
  const uint32_t v_smem = k_smem + C::kNK * C::kTileBytes;             // kNV tiles
  const int total = p.n_items * p.batch;

  if (tid == 0) {
    s_trace_n[0] = s_trace_n[1] = s_trace_n[2] = 0;
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&bars.q_full[i]), 1);
      mbar_init(smem_u32(&bars.q_empty[i]), 1);
      mbar_init(smem_u32(&bars.s_full[i]), 1);
      mbar_init(smem_u32(&bars.p_full[i]), kSoftmaxThreads);
      mbar_init(smem_u32(&bars.o_full[i]), 1);
      mbar_init(smem_u32(&bars.o_empty[i]), kSoftmaxThreads);
    }
    for (int i = 0; i < C::kNK; ++i) {
      mbar_init(smem_u32(&bars.k_full[i]), 1);
      mbar_init(smem_u32(&bars.k_empty[i]), 1);
    }
    for (int i = 0; i < C::kNV; ++i) {
      mbar_init(smem_u32(&bars.v_full[i]), 1);
      mbar_init(smem_u32(&bars.v_empty[i]), 1);
    }
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
  // register budget: the producer / MMA warpgroup gives registers to the softmax warpgroups
  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsOther) : "memory");
  if (warp == 8 || warp == 10) {
    // ------------------------------------------------------------------ TMA producers
    // warp 8: Q tiles + K ring; warp 10: V ring (a V stage waits for the later PV of the
    // two q tiles, which must not hold back the next K loads)
    if (lane == 0) {
      const bool kq = warp == 8;
      int T = 0;
      int qcnt[2] = {0, 0};  // Q tile loads per slot
      for (int idx = blockIdx.x; idx < total; idx += gridDim.x) {
        const Item it = get_item(p, idx);
        const int g = it.h / p.G;
        if (kq) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (!it.has[q]) continue;
            // Q_q of this item may overwrite the previous Q_q once its last S_q completed
            if (qcnt[q] >= 1) mbar_wait(smem_u32(&bars.q_empty[q]), (qcnt[q] - 1) & 1);
            ++qcnt[q];
            const uint32_t qbar = smem_u32(&bars.q_full[q]);
            mbar_expect_tx(qbar, C::kTileBytes);
            for (int sl = 0; sl < C::kSlabs; ++sl)
              tma_load_4d(q_smem + q * C::kTileBytes + sl * C::kSlabBytes, &tm_q, qbar, sl * 64, it.h,
                          (int)it.i0[q], it.b);
          }
        }
        const int nu = it.tu.count();
        for (int u = 0; u < nu; ++u, ++T) {
          const int j0 = it.tu.at(u) * kN;
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
    mma_role<D>(p, bars, tmem, q_smem, k_smem, v_smem, total);  // whole warp; one elected lane issues
  }  // warp 11: idle
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax) : "memory");
    if (warp < 4)
      softmax_role<D, 0>(p, bars, tmem, total, tid, warp);
    else
      softmax_role<D, 1>(p, bars, tmem, total, tid, warp);
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

bool encode_cache_map(void *map_out, const void *ptr, int D, int64_t rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, 64};
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
  p.n_items = a.n_pairs;
  p.nql = a.nql;
  p.G = a.G;
  p.n_sink = a.n_sink;
  p.scale_log2 = a.scale * kLog2e;
  p.win_q = a.d_win_q;
  p.items = a.d_pairs;
  cudaError_t e = cudaFuncSetAttribute(prefill_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::kSmemBytes);
  if (e != cudaSuccess) return (int)e;
  const int total = a.n_pairs * a.batch;
  static unsigned long long *trace_buf = nullptr;
  static bool trace_on = std::getenv("MOA_PREFILL_TRACE") != nullptr;
  if (trace_on) {
    if (!trace_buf) cudaMalloc(&trace_buf, 65536 * 8);
    cudaMemsetAsync(trace_buf, 0, 65536 * 8, (cudaStream_t)stream);
    cudaMemcpyToSymbolAsync(g_trace, &trace_buf, sizeof(trace_buf), 0, cudaMemcpyHostToDevice, (cudaStream_t)stream);
  }
  const int grid = total < num_sms() ? total : num_sms();
  prefill_tc_kernel<D><<<grid, kThreads, C::kSmemBytes, (cudaStream_t)stream>>>(mq, mk, mv, p);
  if (trace_on) {
    static std::vector<unsigned long long> h(65536);
    cudaMemcpy(h.data(), trace_buf, 65536 * 8, cudaMemcpyDeviceToHost);
    FILE *f = fopen("gpurun_out/prefill_trace.txt", "w");
    if (f) {
      const unsigned n = (unsigned)(h[0] & 0xffffffffu);
      (void)n;
      for (unsigned k = 0; k < 60000; ++k)
        if (h[1 + k]) fprintf(f, "%llu %llu\n", h[1 + k] >> 8, h[1 + k] & 255);
      fclose(f);
    }
  }
  return (int)cudaGetLastError();
}

}  // namespace

int launch_prefill_bf16_tc(const PrefillArgs &a, void *stream) {
  if (a.d == 128) return launch_d<128>(a, stream);
  return launch_d<64>(a, stream);
}

}  // namespace moa
