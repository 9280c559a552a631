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
// LPT-sorted (q-head, q-tile) x batch work list.  Warp roles:
//   warps 0-3  softmax / correction / epilogue: thread t owns q row t = TMEM lane t
//   warp 4     TMA producer (Q double-buffered per item, K and V rings)
//   warp 5     TMEM allocator + single-thread MMA issuer
// TMEM (512 columns): S0 | S1 (fp32 128x128 each) | P0 | P1 (bf16 128x128
// packed, 64 cols each) | O (fp32 128xD).  S is double-buffered so QK^T of
// tile T+1 runs while the softmax of tile T executes; P is double-buffered so
// PV of tile T overlaps the softmax of tile T+1.  The running max is only
// refreshed (and O rescaled in TMEM) when it grows by more than 2^8, so most
// tiles need no O round-trip.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <mutex>

#include "../moa_internal.h"
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace moa {
namespace {

using namespace ptx;

constexpr int kM = 128;                // q rows per tile (MMA M)
constexpr int kN = 128;                // keys per tile (MMA N of QK^T, K of PV)
constexpr int kSoftmaxThreads = 128;
constexpr int kThreads = kSoftmaxThreads + 64;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColP0 = 256, kColP1 = 320, kColO = 384;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only if the max grows by > 2^8

template <int D>
struct Cfg {
  static constexpr int kSlabs = D / 64;                  // 128-byte swizzle slabs per row
  static constexpr int kTileBytes = kM * D * 2;          // one Q / K / V tile in smem
  static constexpr int kSlabBytes = kM * 128;            // 128 rows x 128 B
  static constexpr int kNK = D == 128 ? 2 : 3;           // K ring stages
  static constexpr int kNV = D == 128 ? 2 : 3;           // V ring stages
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
  const int32_t *items;
};

struct Bars {
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[4], k_empty[4];
  uint64_t v_full[4], v_empty[4];
  uint64_t s_full[2], p_full[2], pv_done[2];
  uint64_t o_full, o_empty;
  uint32_t tmem_base;
};

struct Item {
  int b, h, qt;
  int64_t i0, i1;
  int W;
  TileRanges tr;
};

__device__ __forceinline__ Item get_item(const TcParams &p, int idx) {
  Item it;
  const int wi = idx / p.batch;
  it.b = idx - wi * p.batch;
  it.h = p.items[2 * wi];
  it.qt = p.items[2 * wi + 1];
  it.i0 = (int64_t)it.qt * kM;
  it.i1 = (p.N < it.i0 + kM ? p.N : it.i0 + kM) - 1;
  it.W = p.win_q[it.h];
  it.tr = kv_tile_ranges(it.i0, it.i1, it.W, p.n_sink);
  return it;
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
  const uint32_t q_smem = smem_base;                                   // 2 tiles
  const uint32_t k_smem = q_smem + 2 * C::kTileBytes;                  // kNK tiles
  const uint32_t v_smem = k_smem + C::kNK * C::kTileBytes;             // kNV tiles
  const int total = p.n_items * p.batch;

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&bars.q_full[i]), 1);
      mbar_init(smem_u32(&bars.q_empty[i]), 1);
      mbar_init(smem_u32(&bars.s_full[i]), 1);
      mbar_init(smem_u32(&bars.p_full[i]), kSoftmaxThreads);
      mbar_init(smem_u32(&bars.pv_done[i]), 1);
    }
    for (int i = 0; i < C::kNK; ++i) {
      mbar_init(smem_u32(&bars.k_full[i]), 1);
      mbar_init(smem_u32(&bars.k_empty[i]), 1);
    }
    for (int i = 0; i < C::kNV; ++i) {
      mbar_init(smem_u32(&bars.v_full[i]), 1);
      mbar_init(smem_u32(&bars.v_empty[i]), 1);
    }
    mbar_init(smem_u32(&bars.o_full), 1);
    mbar_init(smem_u32(&bars.o_empty), kSoftmaxThreads);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc<kTmemCols>(smem_u32(&bars.tmem_base));
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp == 4) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int n = 0, T = 0;
      for (int idx = blockIdx.x; idx < total; idx += gridDim.x, ++n) {
        const Item it = get_item(p, idx);
        const int g = it.h / p.G;
        const int qb = n & 1;
        if (n >= 2) mbar_wait(smem_u32(&bars.q_empty[qb]), ((n - 2) >> 1) & 1);
        const uint32_t qbar = smem_u32(&bars.q_full[qb]);
        mbar_expect_tx(qbar, C::kTileBytes);
        for (int sl = 0; sl < C::kSlabs; ++sl)
          tma_load_4d(q_smem + qb * C::kTileBytes + sl * C::kSlabBytes, &tm_q, qbar, sl * 64, it.h, (int)it.i0, it.b);
        const int nt = it.tr.count();
        for (int t = 0; t < nt; ++t, ++T) {
          const int j0 = it.tr.at(t) * kN;
          const int ks = T % C::kNK, vs = T % C::kNV;
          if (T >= C::kNK) mbar_wait(smem_u32(&bars.k_empty[ks]), ((T - C::kNK) / C::kNK) & 1);
          const uint32_t kbar = smem_u32(&bars.k_full[ks]);
          mbar_expect_tx(kbar, C::kTileBytes);
          for (int sl = 0; sl < C::kSlabs; ++sl)
            tma_load_4d(k_smem + ks * C::kTileBytes + sl * C::kSlabBytes, &tm_k, kbar, sl * 64, g, j0, it.b);
          if (T >= C::kNV) mbar_wait(smem_u32(&bars.v_empty[vs]), ((T - C::kNV) / C::kNV) & 1);
          const uint32_t vbar = smem_u32(&bars.v_full[vs]);
          mbar_expect_tx(vbar, C::kTileBytes);
          for (int sl = 0; sl < C::kSlabs; ++sl)
            tma_load_4d(v_smem + vs * C::kTileBytes + sl * C::kSlabBytes, &tm_v, vbar, sl * 64, g, j0, it.b);
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kM, kN, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kM, D, true);
      int n = 0, T = 0;
      auto issue_pv = [&](int Tp, bool first_of_item, int item_n) {
        const int vs = Tp % C::kNV, pb = Tp & 1;
        mbar_wait(smem_u32(&bars.v_full[vs]), (Tp / C::kNV) & 1);
        mbar_wait(smem_u32(&bars.p_full[pb]), (Tp >> 1) & 1);
        if (first_of_item && item_n > 0) mbar_wait(smem_u32(&bars.o_empty), (item_n - 1) & 1);
        tc_fence_after();
        const uint32_t vb = v_smem + vs * C::kTileBytes;
        const uint32_t pcol = tmem + (pb ? kColP1 : kColP0);
#pragma unroll
        for (int kk = 0; kk < kN / 16; ++kk) {
          // B = V tile, MN-major SW128: 16 keys = two 8-row groups of 1024 B; N slabs 16 KB apart
          const uint64_t bdesc = smem_desc_sw128(vb + kk * 2048, C::kSlabBytes, 1024);
          mma_ts(tmem + kColO, pcol + kk * 8, bdesc, idesc_o, (first_of_item && kk == 0) ? 0u : 1u);
        }
        mma_commit(smem_u32(&bars.v_empty[vs]));
        mma_commit(smem_u32(&bars.pv_done[pb]));
      };
      for (int idx = blockIdx.x; idx < total; idx += gridDim.x, ++n) {
        const Item it = get_item(p, idx);
        const int qb = n & 1;
        mbar_wait(smem_u32(&bars.q_full[qb]), (n >> 1) & 1);
        const uint32_t qa = q_smem + qb * C::kTileBytes;
        const int nt = it.tr.count();
        const int T0 = T;
        for (int t = 0; t < nt; ++t, ++T) {
          const int ks = T % C::kNK, sb = T & 1;
          mbar_wait(smem_u32(&bars.k_full[ks]), (T / C::kNK) & 1);
          if (T >= 2) mbar_wait(smem_u32(&bars.p_full[sb]), ((T - 2) >> 1) & 1);  // S[sb] consumed
          tc_fence_after();
          const uint32_t kb = k_smem + ks * C::kTileBytes;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * C::kSlabBytes + (kk & 3) * 32;
            const uint64_t adesc = smem_desc_sw128(qa + off, 16, 1024);
            const uint64_t bdesc = smem_desc_sw128(kb + off, 16, 1024);
            mma_ss(tmem + (sb ? kColS1 : kColS0), adesc, bdesc, idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(smem_u32(&bars.s_full[sb]));
          mma_commit(smem_u32(&bars.k_empty[ks]));
          if (t == nt - 1) mma_commit(smem_u32(&bars.q_empty[qb]));
          if (t > 0) issue_pv(T - 1, t - 1 == 0, n);
        }
        issue_pv(T - 1, nt == 1, n);
        (void)T0;
        mma_commit(smem_u32(&bars.o_full));
      }
    }
  } else {
    // ------------------------------------------------------------------ softmax warps 0-3
    const int row = tid;  // TMEM lane
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;

    int n = 0, T = 0;
    for (int idx = blockIdx.x; idx < total; idx += gridDim.x, ++n) {
      const Item it = get_item(p, idx);
      const int64_t i = it.i0 + row;
      const int nt = it.tr.count();
      float m_used = -INFINITY, l = 0.f;
      for (int t = 0; t < nt; ++t, ++T) {
        const int sb = T & 1;
        const int64_t j0 = (int64_t)it.tr.at(t) * kN;
        const bool full = kv_tile_full(it.i0, it.i1, it.tr.at(t), it.W, p.n_sink);
        mbar_wait(smem_u32(&bars.s_full[sb]), (T >> 1) & 1);
        tc_fence_after();
        float x[kN];
        {
          uint32_t r[32];
          const uint32_t sa = tmem + lane_off + (sb ? kColS1 : kColS0);
#pragma unroll
          for (int c = 0; c < kN / 32; ++c) {
            tmem_ld32(sa + c * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) x[c * 32 + e] = __uint_as_float(r[e]) * p.scale_log2;
          }
        }
        if (!full) {
#pragma unroll
          for (int c = 0; c < kN; ++c) {
            const int64_t j = j0 + c;
            const bool vis = j <= i && (j < p.n_sink || i - j < it.W);
            if (!vis) x[c] = -INFINITY;
          }
        }
        float mt = x[0];
#pragma unroll
        for (int c = 1; c < kN; ++c) mt = fmaxf(mt, x[c]);
        // lazy max: only move the reference (and rescale O) when it grows by > 2^8
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
          // O must hold PV(T-1) before it is rescaled
          mbar_wait(smem_u32(&bars.pv_done[(T - 1) & 1]), ((T - 1) >> 1) & 1);
          tc_fence_after();
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            const uint32_t oa = tmem + lane_off + kColO + c * 32;
            tmem_ld32(oa, r);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            tmem_st32(oa, r);
          }
        }
        l *= alpha;
        const float mref = m_used == -INFINITY ? 0.f : m_used;
        float ps = 0.f;
        uint32_t pk[kN / 2];
#pragma unroll
        for (int c = 0; c < kN / 2; ++c) {
          const float a = fast_exp2(x[2 * c] - mref);
          const float b2 = fast_exp2(x[2 * c + 1] - mref);
          ps += a + b2;
          pk[c] = pack_bf16x2(a, b2);
        }
        l += ps;
        // P[sb] was last read by PV(T-2)
        if (T >= 2) mbar_wait(smem_u32(&bars.pv_done[sb]), ((T - 2) >> 1) & 1);
        {
          const uint32_t pa = tmem + lane_off + (sb ? kColP1 : kColP0);
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = pk[c * 32 + e];
            tmem_st32(pa + c * 32, r);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(smem_u32(&bars.p_full[sb]));
      }
      // epilogue: O / l -> bf16 rows, lse
      mbar_wait(smem_u32(&bars.o_full), n & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16 *orow = static_cast<__nv_bfloat16 *>(p.o) + ((int64_t)it.b * p.N + i) * p.o_row_stride +
                            (int64_t)it.h * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + kColO + c * 32, r);
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
      if (p.lse && i <= it.i1)
        p.lse[((int64_t)it.b * p.nql + it.h) * p.N + i] = l > 0.f ? (m_used + __log2f(l)) * kLn2 : -INFINITY;
      tc_fence_before();
      mbar_arrive(smem_u32(&bars.o_empty));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
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
