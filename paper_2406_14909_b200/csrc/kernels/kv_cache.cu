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

// cache_fill: grid (ceil(max_rows / (kFillRows * 256 / vpr)), ngl, batch), 256 threads.
// Row r of the region receives prompt position pos_of_row(r, N-1) (sinks
// [0, min(s,N)), ring = the last W_g non-sink positions).  A thread copies the same
// 16-byte column of kFillRows rows (256 / vpr rows apart): all its loads are issued before
// its stores, so each thread keeps 2 * kFillRows * 16 bytes in flight.
constexpr int kFillRows = 4;
__global__ void __launch_bounds__(256) cache_fill_kernel(
    const uint4 *__restrict__ k, const uint4 *__restrict__ v, int64_t row_stride_v,  // in uint4
    uint4 *__restrict__ kc, uint4 *__restrict__ vc, int64_t rows_per_seq,
    const int64_t *__restrict__ g_off, const int32_t *__restrict__ win_g, int vpr, int n_sink,
    int64_t N, const int64_t *__restrict__ seq_n) {
  const int g = blockIdx.y, b = blockIdx.z;
  const int Wg = win_g[g];
  const int64_t R = (int64_t)n_sink + Wg;
  const int rpb = 256 / vpr;  // rows per pass of the block
  const int e = threadIdx.x % vpr;
  const int64_t r0 = (int64_t)blockIdx.x * rpb * kFillRows + threadIdx.x / vpr;
  if (r0 >= R) return;
  const int64_t Nb = seq_n ? seq_n[b] : N;  // ragged: this sequence's prompt length (<= N)
  uint4 kk[kFillRows], vv[kFillRows];
  int64_t dst[kFillRows];
#pragma unroll
  for (int u = 0; u < kFillRows; ++u) {
    const int64_t r = r0 + (int64_t)u * rpb;
    const int64_t p = r < R ? moa::pos_of_row(r, Nb - 1, n_sink, Wg) : -1;
    dst[u] = -1;
    if (p >= 0) {  // (p < 0: row not reached by the prompt, or past the region)
      const int64_t src = ((int64_t)b * N + p) * row_stride_v + (int64_t)g * vpr + e;
      kk[u] = __ldg(k + src);
      vv[u] = __ldg(v + src);
      dst[u] = ((int64_t)b * rows_per_seq + g_off[g] + r) * vpr + e;
    }
  }
#pragma unroll
  for (int u = 0; u < kFillRows; ++u)
    if (dst[u] >= 0) {
      kc[dst[u]] = kk[u];
      vc[dst[u]] = vv[u];
    }
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
  const int64_t rows_per_block = (int64_t)(256 / vpr) * kFillRows;
  dim3 grid((unsigned)((a.max_region_rows + rows_per_block - 1) / rows_per_block), (unsigned)a.ngl,
            (unsigned)a.batch);
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

__global__ void advance_pos_kernel(int64_t *pos, int batch, int64_t delta) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch && pos[b] >= 0) pos[b] += delta;
}

int launch_advance_pos(int64_t *pos, int batch, int64_t delta, void *stream) {
  advance_pos_kernel<<<(batch + 127) / 128, 128, 0, (cudaStream_t)stream>>>(pos, batch, delta);
  return (int)cudaGetLastError();
}

}  // namespace moa
