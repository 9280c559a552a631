// decode.cu -- MoA decode attention over the compact per-group ring cache
// (SURVEY §8(a) a7 split-KV + a8 combine, optionally a6 append fused in),
// fp32 I/O specialisation (FFMA; the bf16 path is decode_mma.cu).
//
// One new query per sequence at absolute position `pos` attends over its
// kv-group's cache region: sink rows [0, s) and ring rows [s, s + W_g)
// (a fixed per-head span during decoding, the oldest entry
// replaced by the latest).  q-head h of group g only sees ring rows whose
// position q satisfies pos - q < W_h (reading c10), so one pass over the
// group's rows serves all G heads of the group: every K/V byte is read once.
//
// Work: grid (n_chunks, batch); chunk c = rows [r0, r1) of one group region.
// 4 warps per CTA, each half-warp owns one row at a time, 16 lanes x VEC
// elements cover d = 16 * VEC.  Per half-warp online softmax in base 2
// (fp32 state), merged across half-warps (shuffle) and warps (smem).  The
// chunk's normalised partial (o, lse2) goes to the workspace; the last CTA of
// a (b, g) (atomic ticket, self-resetting) merges the chunks by LSE and
// writes o (and lse).  HBM-bound: K/V streamed once with 16-byte
// L1::no_allocate loads.
#include <cuda_runtime.h>

#include <cmath>

#include "../moa_internal.h"
#include "common.cuh"

namespace moa {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;

struct DecodeParams {
  const void *q;
  void *o;
  int64_t q_bs, o_bs;
  const void *k_new, *v_new;
  int64_t kv_bs;
  const void *kc, *vc;
  int64_t rows_per_seq;
  const int64_t *g_off;
  const int32_t *win_g, *win_q, *chunks, *g_chunk;
  int n_chunks, ngl, n_sink;
  int64_t pos;
  const int64_t *pos_b;     // ragged: per-sequence positions (null: pos)
  const int32_t *win_bq;    // ragged: per-sequence windows [batch, nql] (null: win_q)
  int nql;
  float scale_log2;
  float *lse;
  float *part;
  int *counters;
};

template <typename T, int D, int G, bool FUSED>
__global__ void __launch_bounds__(kThreads) decode_kernel(const DecodeParams p) {
  constexpr int VEC = D / 16;
  constexpr int U = G <= 2 ? 4 : (G <= 4 ? 2 : 1);  // rows per half-warp per step
  constexpr int ROWS_PER_STEP = 2 * U;               // rows per warp per step

  __shared__ float sm_m[kWarps][G];
  __shared__ float sm_l[kWarps][G];
  __shared__ float sm_acc[kWarps][G][D];
  __shared__ int sm_last;

  const int c = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, li = lane & 15;
  const int g = p.chunks[3 * c], r0 = p.chunks[3 * c + 1], r1 = p.chunks[3 * c + 2];
  const int Wg = p.win_g[g];
  const int s = p.n_sink;
  const int64_t pos = p.pos_b ? p.pos_b[b] : p.pos;  // ragged: pos < 0 = inactive (all masked)

  int Wj[G];
#pragma unroll
  for (int j = 0; j < G; ++j) Wj[j] = p.win_bq ? p.win_bq[(int64_t)b * p.nql + g * G + j] : p.win_q[g * G + j];

  // ring bookkeeping: ring row k holds position pos - m with m = (pm - k) mod W_g,
  // valid iff m <= pos - s.
  const bool ring_live = pos >= s && Wg > 0;
  const int pm = ring_live ? (int)((pos - s) % Wg) : 0;
  const int64_t ring_age_max = pos - s;  // m must be <= this
  const int64_t slot_p = moa::slot_of(pos, s, Wg);

  const T *q = static_cast<const T *>(p.q);
  float qf[G][VEC];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    VecLoad<T, VEC> v;
    v.load(q + (int64_t)b * p.q_bs + (int64_t)(g * G + j) * D + li * VEC);
    v.to_float(qf[j]);
#pragma unroll
    for (int e = 0; e < VEC; ++e) qf[j][e] *= p.scale_log2;
  }

  float m[G], l[G], acc[G][VEC];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    m[j] = -INFINITY;
    l[j] = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[j][e] = 0.f;
  }

  const int64_t base = (int64_t)b * p.rows_per_seq + p.g_off[g];
  const T *kc = static_cast<const T *>(p.kc) + base * D + li * VEC;
  const T *vc = static_cast<const T *>(p.vc) + base * D + li * VEC;

  for (int rb = r0 + warp * ROWS_PER_STEP; rb < r1; rb += kWarps * ROWS_PER_STEP) {
    VecLoad<T, VEC> kv[U], vv[U];
    int dist[U];  // -1: invalid row; -2: sink (visible to all); else age m = pos - position
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int row = rb + 2 * u + half;
      int dd = -1;
      if (row < r1) {
        if (row < s) {
          dd = row <= pos ? -2 : -1;
        } else if (ring_live) {
          int mm = pm - (row - s);
          if (mm < 0) mm += Wg;
          dd = (int64_t)mm <= ring_age_max ? mm : -1;
        }
      }
      dist[u] = dd;
      if (dd != -1) {
        if (FUSED && row == slot_p) {
          const T *kn = static_cast<const T *>(p.k_new) + (int64_t)b * p.kv_bs + (int64_t)(g) * D + li * VEC;
          const T *vn = static_cast<const T *>(p.v_new) + (int64_t)b * p.kv_bs + (int64_t)(g) * D + li * VEC;
          kv[u].load(kn);
          vv[u].load(vn);
          kv[u].store(const_cast<T *>(kc) + (int64_t)row * D);
          vv[u].store(const_cast<T *>(vc) + (int64_t)row * D);
        } else {
          kv[u].load(kc + (int64_t)row * D);
          vv[u].load(vc + (int64_t)row * D);
        }
      } else {
        kv[u].zero();
        vv[u].zero();
      }
    }

    float x[U][G];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float kf[VEC];
      kv[u].to_float(kf);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < VEC; ++e) a = fmaf(qf[j][e], kf[e], a);
        a += __shfl_xor_sync(0xffffffffu, a, 8);
        a += __shfl_xor_sync(0xffffffffu, a, 4);
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        const bool vis = dist[u] == -2 || (dist[u] >= 0 && dist[u] < Wj[j]);
        x[u][j] = vis ? a : -INFINITY;
      }
    }

#pragma unroll
    for (int j = 0; j < G; ++j) {
      float mx = x[0][j];
#pragma unroll
      for (int u = 1; u < U; ++u) mx = fmaxf(mx, x[u][j]);
      const float m_new = fmaxf(m[j], mx);
      if (m_new == -INFINITY) continue;  // nothing visible yet for this head
      const float alpha = fast_exp2(m[j] - m_new);
      float pu[U];
      float ps = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        pu[u] = fast_exp2(x[u][j] - m_new);
        ps += pu[u];
      }
      l[j] = l[j] * alpha + ps;
      m[j] = m_new;
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[j][e] *= alpha;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float vf[VEC];
        vv[u].to_float(vf);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[j][e] = fmaf(pu[u], vf[e], acc[j][e]);
      }
    }
  }

  // merge the two half-warps (lane li and li + 16 hold the same elements)
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const float mo = __shfl_xor_sync(0xffffffffu, m[j], 16);
    const float lo = __shfl_xor_sync(0xffffffffu, l[j], 16);
    const float mn = fmaxf(m[j], mo);
    const float a = mn == -INFINITY ? 0.f : fast_exp2(m[j] - mn);
    const float ao = mn == -INFINITY ? 0.f : fast_exp2(mo - mn);
    l[j] = l[j] * a + lo * ao;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const float oo = __shfl_xor_sync(0xffffffffu, acc[j][e], 16);
      acc[j][e] = acc[j][e] * a + oo * ao;
    }
    m[j] = mn;
  }
  if (half == 0) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (li == 0) {
        sm_m[warp][j] = m[j];
        sm_l[warp][j] = l[j];
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) sm_acc[warp][j][li * VEC + e] = acc[j][e];
    }
  }
  __syncthreads();

  // chunk partial: normalised o and lse2 (base-2 log of the denominator)
  float *part = p.part + ((int64_t)b * p.n_chunks + c) * G * (D + 1);
  for (int t = tid; t < G * D; t += kThreads) {
    const int j = t / D, e = t - j * D;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) mx = fmaxf(mx, sm_m[w][j]);
    float L = 0.f, O = 0.f;
    if (mx != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const float sc = fast_exp2(sm_m[w][j] - mx);
        L += sm_l[w][j] * sc;
        O += sm_acc[w][j][e] * sc;
      }
    }
    part[j * (D + 1) + e] = L > 0.f ? O / L : 0.f;
    if (e == 0) part[j * (D + 1) + D] = L > 0.f ? mx + __log2f(L) : -INFINITY;
  }

  // last CTA of this (b, g) merges all chunks of the group
  __threadfence();
  __syncthreads();
  const int c0 = p.g_chunk[g], c1 = p.g_chunk[g + 1];
  if (tid == 0) {
    int *ctr = p.counters + (int64_t)b * p.ngl + g;
    const int ticket = atomicAdd(ctr, 1);
    const bool last = ticket == (c1 - c0) - 1;
    if (last) *ctr = 0;  // self-reset for the next launch
    sm_last = last;
  }
  __syncthreads();
  if (!sm_last) return;
  __threadfence();

  T *o = static_cast<T *>(p.o);
  for (int t = tid; t < G * D; t += kThreads) {
    const int j = t / D, e = t - j * D;
    float mx = -INFINITY;
    for (int cc = c0; cc < c1; ++cc)
      mx = fmaxf(mx, __ldcg(p.part + (((int64_t)b * p.n_chunks + cc) * G + j) * (D + 1) + D));
    float L = 0.f, O = 0.f;
    for (int cc = c0; cc < c1; ++cc) {
      const float *pc = p.part + (((int64_t)b * p.n_chunks + cc) * G + j) * (D + 1);
      const float lse = __ldcg(pc + D);
      if (lse == -INFINITY) continue;
      const float w = fast_exp2(lse - mx);
      L += w;
      O += w * __ldcg(pc + e);
    }
    o[(int64_t)b * p.o_bs + (int64_t)(g * G + j) * D + e] = from_float<T>(L > 0.f ? O / L : 0.f);
    if (p.lse && e == 0)
      p.lse[(int64_t)b * p.ngl * G + g * G + j] = L > 0.f ? (mx + __log2f(L)) * kLn2 : -INFINITY;
  }
}

template <typename T, int D, int G>
int launch_t(const DecodeArgs &a, bool fused, void *stream) {
  DecodeParams p;
  p.q = a.q; p.o = a.o; p.q_bs = a.q_batch_stride; p.o_bs = a.o_batch_stride;
  p.k_new = a.k_new; p.v_new = a.v_new; p.kv_bs = a.kv_batch_stride;
  p.kc = a.k_cache; p.vc = a.v_cache; p.rows_per_seq = a.rows_per_seq;
  p.g_off = a.d_g_off; p.win_g = a.d_win_g; p.win_q = a.d_win_q; p.chunks = a.d_chunks;
  p.g_chunk = a.d_g_chunk; p.n_chunks = a.n_chunks; p.ngl = a.ngl; p.n_sink = a.n_sink;
  p.pos = a.pos; p.pos_b = a.d_pos; p.win_bq = a.d_win_bq; p.nql = a.ngl * a.G; p.scale_log2 = a.scale * kLog2e; p.lse = a.lse; p.part = a.ws_part;
  p.counters = a.counters;
  dim3 grid((unsigned)a.n_chunks, (unsigned)a.batch);
  if (fused)
    decode_kernel<T, D, G, true><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p);
  else
    decode_kernel<T, D, G, false><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

template <typename T, int D>
int launch_g(const DecodeArgs &a, bool fused, void *stream) {
  switch (a.G) {
    case 1: return launch_t<T, D, 1>(a, fused, stream);
    case 2: return launch_t<T, D, 2>(a, fused, stream);
    case 4: return launch_t<T, D, 4>(a, fused, stream);
    case 8: return launch_t<T, D, 8>(a, fused, stream);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace

size_t decode_ws_bytes(int batch, int n_chunks, int G, int d) {
  size_t b = (size_t)batch * n_chunks * G * (d + 1) * 4;
  return (b + 255) & ~size_t(255);
}

// fp32 I/O only (config C1, 1e-5 bar); bf16 decode runs on decode_mma.cu.
int launch_decode(const DecodeArgs &a, moa_dtype dtype, bool fused, void *stream) {
  if (dtype != MOA_FP32) return (int)cudaErrorInvalidValue;
  if (a.d == 128) return launch_g<float, 128>(a, fused, stream);
  return launch_g<float, 64>(a, fused, stream);
}

}  // namespace moa
