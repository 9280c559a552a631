// prefill_f32.cu -- MoA prefill for fp32 I/O (reading c12:
// fp32 I/O must not use TF32 tensor cores, whose ~1e-3 error exceeds the
// 1e-5 bar).  FFMA on CUDA cores; this is the dtype specialisation used by
// config C1, not a fallback for bf16.
//
// O[b,i,h] = sum_{j in V(h,i)} softmax_j(tau q_i . k_j) v_j  (Eq. 1,
// PAPER.md:88-93) with V(h,i) the sink + window set.  Only
// the kv tiles of the block-skip schedule are visited (moa_internal.h).
//
// Grid (n_items, batch): one CTA per (q-head, 128-row q tile), one thread per
// query row.  K/V tiles of 128 keys are staged in shared memory and read as
// warp-wide broadcasts; q lives transposed in shared memory (conflict-free).
#include <cuda_runtime.h>

#include <cmath>

#include "../moa_internal.h"
#include "common.cuh"

namespace moa {
namespace {

constexpr int kRows = kTile;  // 128 query rows = 128 threads
constexpr int kKeys = kTile;  // keys per staged tile
constexpr int kSub = 16;      // keys per softmax sub-block

template <int D>
__global__ void __launch_bounds__(kRows) prefill_f32_kernel(PrefillArgs a) {
  extern __shared__ float4 smem4[];
  float *sm = reinterpret_cast<float *>(smem4);
  float *qs = sm;                   // [D][kRows]  (transposed)
  float *ks = qs + D * kRows;       // [kKeys][D]
  float *vs = ks + kKeys * D;       // [kKeys][D]

  const int item = blockIdx.x, b = blockIdx.y;
  const int h = a.d_items[2 * item], qt = a.d_items[2 * item + 1];
  const int g = h / a.G;
  const int tid = threadIdx.x;
  const int64_t N = a.N;                               // row stride of a sequence (padded length)
  const int64_t Nb = a.d_seq_n ? a.d_seq_n[b] : N;     // ragged: this sequence's length
  const int64_t i0 = (int64_t)qt * kRows;
  if (i0 >= Nb) return;                                // whole tile past a ragged sequence's end
  const int64_t i1 = (Nb < i0 + kRows ? Nb : i0 + kRows) - 1;
  const int64_t i = i0 + tid;
  const int W = a.d_win_bq ? a.d_win_bq[(int64_t)b * a.nql + h] : a.d_win_q[h];
  const int s = a.n_sink;

  const float *Q = static_cast<const float *>(a.q);
  const float *K = static_cast<const float *>(a.k);
  const float *V = static_cast<const float *>(a.v);

  // stage q (row tid) transposed
  for (int e = 0; e < D; ++e) {
    float x = 0.f;
    if (i < N) x = Q[((int64_t)b * N + i) * a.q_row_stride + (int64_t)h * D + e];
    qs[e * kRows + tid] = x * a.scale;
  }

  float acc[D];
#pragma unroll
  for (int e = 0; e < D; ++e) acc[e] = 0.f;
  float m = -INFINITY, l = 0.f;

  const TileRanges tr = kv_tile_ranges(i0, i1, W, s, a.bshift);
  const int64_t lo_i = win_lo(i, W, a.bshift);  // first window key of this row (token or block mode)
  const int nt = tr.count();
  for (int t = 0; t < nt; ++t) {
    const int kt = tr.at(t);
    const int64_t j0 = (int64_t)kt * kKeys;
    __syncthreads();
    for (int idx = tid; idx < kKeys * D / 4; idx += kRows) {
      const int r = idx / (D / 4), c4 = idx - r * (D / 4);
      const int64_t j = j0 + r;
      float4 kk = make_float4(0.f, 0.f, 0.f, 0.f), vv = kk;
      if (j < N) {
        const int64_t off = ((int64_t)b * N + j) * a.kv_row_stride + (int64_t)g * D + 4 * c4;
        kk = *reinterpret_cast<const float4 *>(K + off);
        vv = *reinterpret_cast<const float4 *>(V + off);
      }
      reinterpret_cast<float4 *>(ks)[idx] = kk;
      reinterpret_cast<float4 *>(vs)[idx] = vv;
    }
    __syncthreads();
    if (i > i1) continue;  // padding rows of the last tile
    for (int sb = 0; sb < kKeys; sb += kSub) {
      float sc[kSub];
#pragma unroll
      for (int u = 0; u < kSub; ++u) sc[u] = 0.f;
      for (int e4 = 0; e4 < D / 4; ++e4) {
        const float q0 = qs[(4 * e4 + 0) * kRows + tid], q1 = qs[(4 * e4 + 1) * kRows + tid];
        const float q2 = qs[(4 * e4 + 2) * kRows + tid], q3 = qs[(4 * e4 + 3) * kRows + tid];
#pragma unroll
        for (int u = 0; u < kSub; ++u) {
          const float4 kk = reinterpret_cast<const float4 *>(ks + (sb + u) * D)[e4];
          sc[u] = fmaf(q0, kk.x, fmaf(q1, kk.y, fmaf(q2, kk.z, fmaf(q3, kk.w, sc[u]))));
        }
      }
      float mx = -INFINITY;
#pragma unroll
      for (int u = 0; u < kSub; ++u) {
        const int64_t j = j0 + sb + u;
        const bool vis = j <= i && (j < s || (W > 0 && j >= lo_i));
        sc[u] = vis ? sc[u] : -INFINITY;
        mx = fmaxf(mx, sc[u]);
      }
      const float mn = fmaxf(m, mx);
      if (mn == -INFINITY) continue;
      const float alpha = expf(m - mn);
      float ps = 0.f;
#pragma unroll
      for (int u = 0; u < kSub; ++u) {
        sc[u] = expf(sc[u] - mn);
        ps += sc[u];
      }
      l = l * alpha + ps;
      m = mn;
#pragma unroll
      for (int e = 0; e < D; ++e) acc[e] *= alpha;
#pragma unroll
      for (int u = 0; u < kSub; ++u) {
        const float4 *vr = reinterpret_cast<const float4 *>(vs + (sb + u) * D);
#pragma unroll
        for (int e4 = 0; e4 < D / 4; ++e4) {
          const float4 vv = vr[e4];
          acc[4 * e4 + 0] = fmaf(sc[u], vv.x, acc[4 * e4 + 0]);
          acc[4 * e4 + 1] = fmaf(sc[u], vv.y, acc[4 * e4 + 1]);
          acc[4 * e4 + 2] = fmaf(sc[u], vv.z, acc[4 * e4 + 2]);
          acc[4 * e4 + 3] = fmaf(sc[u], vv.w, acc[4 * e4 + 3]);
        }
      }
    }
  }
  if (i > i1) return;
  float *O = static_cast<float *>(a.o) + ((int64_t)b * N + i) * a.o_row_stride + (int64_t)h * D;
  const float inv = 1.f / l;
#pragma unroll
  for (int e4 = 0; e4 < D / 4; ++e4)
    reinterpret_cast<float4 *>(O)[e4] =
        make_float4(acc[4 * e4] * inv, acc[4 * e4 + 1] * inv, acc[4 * e4 + 2] * inv, acc[4 * e4 + 3] * inv);
  if (a.lse) a.lse[((int64_t)b * a.nql + h) * N + i] = m + logf(l);
}

}  // namespace

int launch_prefill_f32(const PrefillArgs &a, void *stream) {
  dim3 grid((unsigned)a.n_items, (unsigned)a.batch);
  if (a.d == 64) {
    const size_t sm = (size_t)(64 * kRows + 2 * kKeys * 64) * 4;
    cudaFuncSetAttribute(prefill_f32_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    prefill_f32_kernel<64><<<grid, kRows, sm, (cudaStream_t)stream>>>(a);
  } else {
    const size_t sm = (size_t)(128 * kRows + 2 * kKeys * 128) * 4;
    cudaFuncSetAttribute(prefill_f32_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    prefill_f32_kernel<128><<<grid, kRows, sm, (cudaStream_t)stream>>>(a);
  }
  return (int)cudaGetLastError();
}

}  // namespace moa
