// kv_cache.cu -- compact per-group KV-cache writes.
//
// Region of (sequence b, local group g): rows [0, s) hold the sinks
// (PAPER.md:178), rows [s, s + W_g) are a ring of the W_g most recent
// non-sink positions; position p >= s lives in row s + (p - s) mod W_g, so a
// new token overwrites the oldest one ("replace the old KV-Cache that exceeds
// the span with the latest"; reading c13).
//
// Both kernels are plain bit copies, HBM-bound: 16-byte vector accesses, one
// thread per 16 bytes, coalesced along the row.
#include <cuda_runtime.h>

#include "../moa_internal.h"

namespace moa {
namespace {

// cache_fill: grid (ceil(max_rows * vpr / 256), ngl, batch), 256 threads.
// Row r of the region receives prompt position pos_of_row(r, N-1) (sinks
// [0, min(s,N)), ring = the last W_g non-sink positions).
__global__ void __launch_bounds__(256) cache_fill_kernel(
    const uint4 *__restrict__ k, const uint4 *__restrict__ v, int64_t row_stride_v,  // in uint4
    uint4 *__restrict__ kc, uint4 *__restrict__ vc, int64_t rows_per_seq,
    const int64_t *__restrict__ g_off, const int32_t *__restrict__ win_g, int vpr, int n_sink,
    int64_t N, const int64_t *__restrict__ seq_n) {
  const int g = blockIdx.y, b = blockIdx.z;
  const int Wg = win_g[g];
  const int64_t R = (int64_t)n_sink + Wg;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = idx / vpr;
  const int e = (int)(idx - r * vpr);
  if (r >= R) return;
  const int64_t Nb = seq_n ? seq_n[b] : N;  // ragged: this sequence's prompt length (<= N)
  const int64_t p = moa::pos_of_row(r, Nb - 1, n_sink, Wg);
  if (p < 0) return;  // row not reached by the prompt (short prompt)
  const int64_t src = ((int64_t)b * N + p) * row_stride_v + (int64_t)g * vpr + e;
  const int64_t dst = ((int64_t)b * rows_per_seq + g_off[g] + r) * vpr + e;
  kc[dst] = __ldg(k + src);
  vc[dst] = __ldg(v + src);
}

// kv_append: grid (ngl, batch), vpr threads per K and V (blockDim = 2 * vpr).
__global__ void kv_append_kernel(const uint4 *__restrict__ k, const uint4 *__restrict__ v,
                                 int64_t batch_stride_v, uint4 *__restrict__ kc,
                                 uint4 *__restrict__ vc, int64_t rows_per_seq,
                                 const int64_t *__restrict__ g_off,
                                 const int32_t *__restrict__ win_g, int vpr, int n_sink,
                                 int64_t pos, const int64_t *__restrict__ pos_b) {
  const int g = blockIdx.x, b = blockIdx.y;
  const int64_t pb = pos_b ? pos_b[b] : pos;  // ragged: per-sequence position, < 0 = inactive
  if (pb < 0) return;
  const int64_t slot = moa::slot_of(pb, n_sink, win_g[g]);
  if (slot < 0) return;  // W_g = 0: a sink-only group stores no recent token
  const int t = threadIdx.x;
  const bool is_v = t >= vpr;
  const int e = is_v ? t - vpr : t;
  const int64_t src = (int64_t)b * batch_stride_v + (int64_t)g * vpr + e;
  const int64_t dst = ((int64_t)b * rows_per_seq + g_off[g] + slot) * vpr + e;
  if (is_v)
    vc[dst] = v[src];
  else
    kc[dst] = k[src];
}

}  // namespace

int launch_cache_fill(const CacheArgs &a, void *stream) {
  const int vpr = a.d * a.esize / 16;
  const int64_t vecs = a.max_region_rows * vpr;
  dim3 grid((unsigned)((vecs + 255) / 256), (unsigned)a.ngl, (unsigned)a.batch);
  cache_fill_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const uint4 *>(a.k), static_cast<const uint4 *>(a.v), a.row_stride * a.esize / 16,
      static_cast<uint4 *>(a.k_cache), static_cast<uint4 *>(a.v_cache), a.rows_per_seq, a.d_g_off,
      a.d_win_g, vpr, a.n_sink, a.N_or_pos, a.d_seq_n);
  return (int)cudaGetLastError();
}

int launch_kv_append(const CacheArgs &a, void *stream) {
  const int vpr = a.d * a.esize / 16;
  dim3 grid((unsigned)a.ngl, (unsigned)a.batch);
  kv_append_kernel<<<grid, 2 * vpr, 0, (cudaStream_t)stream>>>(
      static_cast<const uint4 *>(a.k), static_cast<const uint4 *>(a.v), a.row_stride * a.esize / 16,
      static_cast<uint4 *>(a.k_cache), static_cast<uint4 *>(a.v_cache), a.rows_per_seq, a.d_g_off,
      a.d_win_g, vpr, a.n_sink, a.N_or_pos, a.d_pos);
  return (int)cudaGetLastError();
}

}  // namespace moa
