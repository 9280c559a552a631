// moa_host.cpp -- C ABI entry points and the host runtime of libmoa.so:
// span resolution (Eq. 2), span table, compact cache layout, prefill
// block-skip schedule, decode work list, validation and error reporting.
// See include/moa.h for the contract of every call.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <numeric>
#include <queue>

#include "moa_internal.h"

using moa::LayerPlan;

namespace {

thread_local std::string g_err;

// next_pos of a ragged layer after its cache fill: positions are per sequence (caller-owned)
constexpr int64_t kRaggedPos = -2;

moa_status fail(moa_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

moa_status ok() { return MOA_OK; }

moa_status cuda_fail(cudaError_t e, const char *what) {
  return fail(MOA_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = -1;
  bool active = false;
  explicit DeviceGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
      active = cudaSetDevice(dev) == cudaSuccess;
    }
  }
  ~DeviceGuard() {
    if (active) cudaSetDevice(prev);
  }
};

// A sticky asynchronous fault from earlier work is reported by the next call.
moa_status check_sticky(const moa_ctx *ctx) {
  if (ctx->device < 0) return MOA_OK;
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return cuda_fail(e, "earlier asynchronous CUDA error");
  return MOA_OK;
}

size_t esize(const moa_ctx *c) { return c->dtype == MOA_BF16 ? 2 : 4; }

moa_status check_layer(const moa_ctx *ctx, int layer, bool need_set) {
  if (!ctx) return fail(MOA_ERR_INVALID_ARG, "ctx is NULL");
  if (layer < 0 || layer >= ctx->L)
    return fail(MOA_ERR_INVALID_ARG, "layer %d out of range [0, %d)", layer, ctx->L);
  if (need_set && !ctx->layers[layer].set)
    return fail(MOA_ERR_STATE, "moa_set_spans was not called for layer %d", layer);
  return MOA_OK;
}

int decode_chunk_rows_override() {
  const char *e = std::getenv("MOA_DECODE_CHUNK");
  if (!e) return 0;
  int v = std::atoi(e);
  return v > 0 ? v : 0;
}

void free_ragged(LayerPlan &p) {
  if (p.d_rag) cudaFree(p.d_rag);
  p.d_rag = nullptr;
  p.d_seq_n = nullptr;
  p.d_win_bq = nullptr;
  p.rag_batch = 0;
  p.rag_n.clear();
  p.rag_win.clear();
  p.rag_items2.clear();
  p.d_rag_items2 = nullptr;
  p.d_rag_sched2 = p.d_rag_sched2_off = nullptr;
  p.rag_sched2_ctas = 0;
}

void free_tables(LayerPlan &p) {
  free_ragged(p);
  if (p.d_tables) cudaFree(p.d_tables);
  p.d_tables = nullptr;
  p.d_win_q = p.d_win_g = nullptr;
  p.d_g_off = nullptr;
  p.d_items = p.d_items2 = p.d_chunks = p.d_g_chunk = p.d_gc_off = p.d_fill_h = nullptr;
  p.d_sched2 = p.d_sched2_off = nullptr;
  p.d_counters = nullptr;
}

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// greedy list scheduling of work entries (pairs, in priority order) onto ncta CTAs: each entry
// to the least-loaded CTA; out = the entries grouped by CTA, off[c] = first entry of CTA c
void greedy_schedule(const std::vector<int32_t> &entries, const std::vector<int> &cost, int ncta,
                     std::vector<int32_t> &out, std::vector<int32_t> &off) {
  std::vector<std::vector<int32_t>> per(ncta);
  using Slot = std::pair<int64_t, int>;  // (load, cta)
  std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
  for (int c = 0; c < ncta; ++c) heap.push({0, c});
  for (size_t i = 0; i < cost.size(); ++i) {
    Slot sl = heap.top();
    heap.pop();
    per[sl.second].push_back(entries[2 * i]);
    per[sl.second].push_back(entries[2 * i + 1]);
    heap.push({sl.first + std::max(1, cost[i]), sl.second});
  }
  out.clear();
  off.assign(ncta + 1, 0);
  for (int c = 0; c < ncta; ++c) {
    off[c] = (int32_t)(out.size() / 2);
    out.insert(out.end(), per[c].begin(), per[c].end());
  }
  off[ncta] = (int32_t)(out.size() / 2);
}



// schedule cost of a two-tile item (MOA_PP_SCHED_COST, tuning): 0 = MMA tiles of both q tiles,
// 1 = union steps (the two tiles ping-pong, a step costs about the same either way; default:
// C4 40 layers +0.5-1.7 % over 0, C2 within noise), 2 = MMA tiles + half a tile per EDGE tile
int sched_cost_mode() {
  static const int m = [] {
    const char *e = std::getenv("MOA_PP_SCHED_COST");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}
int sched_cost(const moa::BlockTiles &bt, int64_t i0, int64_t N, int W, int s, int bshift) {
  const int mma = bt.r[0].count() + (bt.has1 ? bt.r[1].count() : 0);
  const int mode = sched_cost_mode();
  if (mode == 1) return 2 * bt.steps();
  if (mode == 2) {
    int edge = 0;
    for (int j = 0; j < (bt.has1 ? 2 : 1); ++j) {
      const int64_t t0 = i0 + j * moa::kTile, t1 = std::min<int64_t>(N, t0 + moa::kTile) - 1;
      const moa::TileRanges &r = bt.r[j];
      for (int k = 0; k < r.count(); ++k) edge += !moa::kv_tile_full(t0, t1, r.at(k), W, s, bshift);
    }
    return 2 * mma + edge;
  }
  return mma;
}



moa_status upload_tables(moa_ctx *ctx, LayerPlan &p) {
  if (ctx->device < 0) return MOA_OK;
  size_t o_winq = 0;
  size_t o_wing = align16(o_winq + p.win_q.size() * 4);
  size_t o_goff = align16(o_wing + p.win_g.size() * 4);
  size_t o_items = align16(o_goff + p.g_off.size() * 8);
  size_t o_items2 = align16(o_items + p.items.size() * 4);
  size_t o_chunks = align16(o_items2 + p.items2.size() * 4);
  size_t o_gch = align16(o_chunks + p.chunks.size() * 4);
  size_t o_gco = align16(o_gch + p.g_chunk.size() * 4);
  size_t o_fh = align16(o_gco + p.gc_off.size() * 4);
  size_t o_sch = align16(o_fh + p.fill_h.size() * 4);
  size_t o_scho = align16(o_sch + p.sched2.size() * 4);
  size_t o_cnt = align16(o_scho + p.sched2_off.size() * 4);
  size_t total = align16(o_cnt + (size_t)ctx->max_batch * ctx->ngl * 4);
  std::vector<unsigned char> host(total, 0);
  std::memcpy(host.data() + o_winq, p.win_q.data(), p.win_q.size() * 4);
  std::memcpy(host.data() + o_wing, p.win_g.data(), p.win_g.size() * 4);
  std::memcpy(host.data() + o_goff, p.g_off.data(), p.g_off.size() * 8);
  std::memcpy(host.data() + o_items, p.items.data(), p.items.size() * 4);
  std::memcpy(host.data() + o_items2, p.items2.data(), p.items2.size() * 4);
  std::memcpy(host.data() + o_chunks, p.chunks.data(), p.chunks.size() * 4);
  std::memcpy(host.data() + o_gch, p.g_chunk.data(), p.g_chunk.size() * 4);
  std::memcpy(host.data() + o_gco, p.gc_off.data(), p.gc_off.size() * 4);
  std::memcpy(host.data() + o_fh, p.fill_h.data(), p.fill_h.size() * 4);
  std::memcpy(host.data() + o_sch, p.sched2.data(), p.sched2.size() * 4);
  std::memcpy(host.data() + o_scho, p.sched2_off.data(), p.sched2_off.size() * 4);
  DeviceGuard dg(ctx->device);
  free_tables(p);
  void *d = nullptr;
  cudaError_t e = cudaMalloc(&d, total);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(span tables)");
  e = cudaMemcpy(d, host.data(), total, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(e, "cudaMemcpy(span tables)");
  }
  auto *b = static_cast<unsigned char *>(d);
  p.d_tables = d;
  p.d_win_q = reinterpret_cast<const int32_t *>(b + o_winq);
  p.d_win_g = reinterpret_cast<const int32_t *>(b + o_wing);
  p.d_g_off = reinterpret_cast<const int64_t *>(b + o_goff);
  p.d_items = reinterpret_cast<const int32_t *>(b + o_items);
  p.d_items2 = reinterpret_cast<const int32_t *>(b + o_items2);
  p.d_chunks = reinterpret_cast<const int32_t *>(b + o_chunks);
  p.d_g_chunk = reinterpret_cast<const int32_t *>(b + o_gch);
  p.d_gc_off = reinterpret_cast<const int32_t *>(b + o_gco);
  p.d_counters = reinterpret_cast<int *>(b + o_cnt);
  p.d_fill_h = reinterpret_cast<const int32_t *>(b + o_fh);
  p.d_sched2 = p.sched2.empty() ? nullptr : reinterpret_cast<const int32_t *>(b + o_sch);
  p.d_sched2_off = p.sched2_off.empty() ? nullptr : reinterpret_cast<const int32_t *>(b + o_scho);
  return MOA_OK;
}

size_t layer_bytes(const moa_ctx *ctx, const LayerPlan &p, int batch) {
  return (size_t)batch * (size_t)p.rows_per_seq * (size_t)ctx->d * esize(ctx);
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

extern "C" {

const char *moa_version(void) { return "moa-b200 0.1 (sm_100a)"; }

const char *moa_last_error(void) { return g_err.c_str(); }

moa_status moa_create(moa_ctx **out, int device, moa_dtype dtype, int num_layers,
                      int num_q_heads, int num_kv_heads, int head_dim, int max_batch,
                      int kv_group_begin, int kv_group_end) {
  if (!out) return fail(MOA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (dtype != MOA_BF16 && dtype != MOA_FP32) return fail(MOA_ERR_INVALID_ARG, "bad dtype %d", (int)dtype);
  if (num_layers <= 0 || num_q_heads <= 0 || num_kv_heads <= 0 || max_batch <= 0)
    return fail(MOA_ERR_SHAPE, "layers/heads/max_batch must be positive");
  if (num_q_heads % num_kv_heads != 0)
    return fail(MOA_ERR_SHAPE, "num_q_heads %d not a multiple of num_kv_heads %d", num_q_heads, num_kv_heads);
  if (head_dim != 64 && head_dim != 128)
    return fail(MOA_ERR_SHAPE, "head_dim %d unsupported (64 or 128)", head_dim);
  int G = num_q_heads / num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return fail(MOA_ERR_UNSUPPORTED, "GQA group size %d unsupported (1, 2, 4 or 8)", G);
  if (kv_group_begin < 0 || kv_group_end > num_kv_heads || kv_group_begin >= kv_group_end)
    return fail(MOA_ERR_SHAPE, "kv-group shard [%d, %d) invalid for %d groups", kv_group_begin,
                kv_group_end, num_kv_heads);
  int sms = 148;  // planning-only contexts (device -1) plan for a B200
  if (device >= 0) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device >= n) return fail(MOA_ERR_INVALID_ARG, "device %d >= device count %d", device, n);
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
      return fail(MOA_ERR_UNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a (B200)",
                  device, prop.major, prop.minor);
    sms = prop.multiProcessorCount;
  }
  moa_ctx *c = new (std::nothrow) moa_ctx();
  if (!c) return fail(MOA_ERR_OOM, "host allocation failed");
  c->device = device;
  c->num_sms = sms;
  c->dtype = dtype;
  c->L = num_layers;
  c->Hq = num_q_heads;
  c->Hkv = num_kv_heads;
  c->G = G;
  c->d = head_dim;
  c->max_batch = max_batch;
  c->g0 = kv_group_begin;
  c->g1 = kv_group_end;
  c->ngl = kv_group_end - kv_group_begin;
  c->nql = c->ngl * G;
  c->layers.resize(num_layers);
  if (const char *e = std::getenv("MOA_DEC_CHUNK")) c->dec_chunk = std::max(0, std::atoi(e));  // tuning
  *out = c;
  return ok();
}

moa_status moa_destroy(moa_ctx *ctx) {
  if (!ctx) return MOA_OK;
  {
    DeviceGuard dg(ctx->device);
    for (auto &p : ctx->layers) free_tables(p);
    if (ctx->d_ml) cudaFree(ctx->d_ml);
    if (ctx->d_peers) cudaFree(ctx->d_peers);
  }
  delete ctx;
  return MOA_OK;
}

moa_status moa_resolve_spans(const float *alpha, const float *beta, int n_heads, int64_t N,
                             int n_sink, int32_t *window_out) {
  if (!alpha || !beta || !window_out) return fail(MOA_ERR_INVALID_ARG, "NULL argument");
  if (n_heads < 0 || N < 1 || n_sink < 0) return fail(MOA_ERR_INVALID_ARG, "bad n_heads/N/n_sink");
  for (int h = 0; h < n_heads; ++h) {
    // Eq. 2 in double: alpha + beta * N (exact for the paper's grid), ceil, clip [0, N].
    double sp = std::ceil((double)alpha[h] + (double)beta[h] * (double)N);
    if (!(sp == sp)) return fail(MOA_ERR_INVALID_ARG, "NaN rule at head %d", h);
    if (sp < 0) sp = 0;
    if (sp > (double)N) sp = (double)N;
    int64_t span = (int64_t)sp;
    int64_t w = span - n_sink;
    window_out[h] = (int32_t)(w > 0 ? w : 0);
  }
  return ok();
}

moa_status moa_set_spans(moa_ctx *ctx, int layer, const int32_t *window_per_q_head, int n_sink,
                         int64_t N) {
  return moa_set_spans_blocked(ctx, layer, window_per_q_head, n_sink, N, 0);
}

moa_status moa_set_spans_blocked(moa_ctx *ctx, int layer, const int32_t *window_per_q_head, int n_sink,
                                 int64_t N, int block) {
  moa_status st = check_layer(ctx, layer, false);
  if (st) return st;
  if (!window_per_q_head) return fail(MOA_ERR_INVALID_ARG, "window_per_q_head is NULL");
  if (n_sink < 0 || n_sink > (1 << 20)) return fail(MOA_ERR_INVALID_ARG, "n_sink %d invalid", n_sink);
  if (N < 1 || N > (int64_t(1) << 31)) return fail(MOA_ERR_INVALID_ARG, "N %lld invalid", (long long)N);
  for (int h = 0; h < ctx->Hq; ++h) {
    int w = window_per_q_head[h];
    if (w < 0 || w > (1 << 30)) return fail(MOA_ERR_INVALID_ARG, "window[%d] = %d invalid", h, w);
    if (w == 0 && n_sink == 0)
      return fail(MOA_ERR_INVALID_ARG, "window[%d] = 0 with no sinks: empty softmax row (reading c7)", h);
  }
  int bshift = -1;
  if (block != 0) {
    if (block < 1 || block > moa::kTile || (block & (block - 1)))
      return fail(MOA_ERR_INVALID_ARG, "block %d: must be 0 or a power of two in [1, %d]", block, moa::kTile);
    bshift = 0;
    while ((1 << bshift) < block) ++bshift;
    if (n_sink % block) return fail(MOA_ERR_INVALID_ARG, "n_sink %d is not a multiple of block %d", n_sink, block);
    for (int h = 0; h < ctx->Hq; ++h)
      if (window_per_q_head[h] % block)
        return fail(MOA_ERR_INVALID_ARG, "window[%d] = %d is not a multiple of block %d", h, window_per_q_head[h],
                    block);
  }
  LayerPlan &p = ctx->layers[layer];
  LayerPlan np;
  np.set = true;
  np.n_sink = n_sink;
  np.bshift = bshift;
  np.N = N;
  const int G = ctx->G;
  np.win_q.resize(ctx->nql);
  for (int h = 0; h < ctx->nql; ++h) np.win_q[h] = window_per_q_head[ctx->g0 * G + h];
  np.win_g.resize(ctx->ngl);
  np.g_off.resize(ctx->ngl);
  int64_t off = 0;
  for (int g = 0; g < ctx->ngl; ++g) {
    int wg = 0;
    for (int j = 0; j < G; ++j) wg = std::max(wg, np.win_q[g * G + j]);
    np.win_g[g] = wg;
    np.g_off[g] = off;
    off += (int64_t)n_sink + wg;
  }
  np.rows_per_seq = off;
  np.fill_h.assign(ctx->ngl, -1);
  for (int g = 0; g < ctx->ngl; ++g)
    for (int j = 0; j < G; ++j)
      if (np.win_q[g * G + j] == np.win_g[g]) {
        np.fill_h[g] = g * G + j;
        break;
      }

  // prefill work items (h_local, q_tile).  Order: heads by total kv-tile count, heaviest
  // first (so the kernel tail holds light work), and the q tiles of one head consecutively,
  // heaviest first: CTAs running concurrently then share their heads' K/V tiles in L2.
  const int nqt = (int)((N + moa::kTile - 1) / moa::kTile);
  struct It { int h, qt, cnt; int64_t hcost; int sc = 0; };
  std::vector<It> its;
  its.reserve((size_t)ctx->nql * nqt);
  for (int h = 0; h < ctx->nql; ++h) {
    const size_t first = its.size();
    int64_t hc = 0;
    for (int qt = 0; qt < nqt; ++qt) {
      int64_t i0 = (int64_t)qt * moa::kTile;
      int64_t i1 = std::min<int64_t>(N, i0 + moa::kTile) - 1;
      const int c = moa::kv_tile_ranges(i0, i1, np.win_q[h], n_sink, bshift).count();
      hc += c;
      its.push_back({h, qt, c, 0});
    }
    for (size_t k = first; k < its.size(); ++k) its[k].hcost = hc;
  }
  std::stable_sort(its.begin(), its.end(), [](const It &a, const It &b) {
    if (a.hcost != b.hcost) return a.hcost > b.hcost;
    if (a.h != b.h) return a.h < b.h;
    return a.cnt > b.cnt;
  });
  np.items.resize(its.size() * 2);
  for (size_t i = 0; i < its.size(); ++i) {
    np.items[2 * i] = its[i].h;
    np.items[2 * i + 1] = its[i].qt;
  }

  // two-tile work items (h_local, q_block of 2*kTile rows), same ordering rule; cost = the
  // MMA tiles of both q tiles
  const int nqb = (int)((N + 2 * moa::kTile - 1) / (2 * moa::kTile));
  its.clear();
  for (int h = 0; h < ctx->nql; ++h) {
    const size_t first = its.size();
    int64_t hc = 0;
    for (int qb = 0; qb < nqb; ++qb) {
      const moa::BlockTiles bt =
          moa::kv_block_tiles((int64_t)qb * 2 * moa::kTile, N, np.win_q[h], n_sink, bshift);
      const int c = bt.r[0].count() + (bt.has1 ? bt.r[1].count() : 0);
      hc += c;
      its.push_back({h, qb, c, 0});
      its.back().sc = sched_cost(bt, (int64_t)qb * 2 * moa::kTile, N, np.win_q[h], n_sink, bshift);
    }
    for (size_t k = first; k < its.size(); ++k) its[k].hcost = hc;
  }
  std::stable_sort(its.begin(), its.end(), [](const It &a, const It &b) {
    if (a.hcost != b.hcost) return a.hcost > b.hcost;
    if (a.h != b.h) return a.h < b.h;
    return a.cnt > b.cnt;
  });
  np.items2.resize(its.size() * 2);
  {
    // per-CTA schedule of the (item, b) entries for a batch of max_batch: greedy list scheduling
    // in the item order above (cost: sched_cost)
    const int B = ctx->max_batch;
    std::vector<int32_t> ent;
    std::vector<int> cost;
    ent.reserve(its.size() * B * 2);
    cost.reserve(its.size() * B);
    for (size_t i = 0; i < its.size(); ++i)
      for (int b = 0; b < B; ++b) {
        ent.push_back(its[i].h | (b << 16));
        ent.push_back(its[i].qt);
        cost.push_back(its[i].sc);
      }
    const int ncta = (int)std::min<size_t>(cost.size(), (size_t)std::max(1, ctx->num_sms));
    greedy_schedule(ent, cost, ncta, np.sched2, np.sched2_off);
    np.sched2_batch = B;
  }
  for (size_t i = 0; i < its.size(); ++i) {
    np.items2[2 * i] = its[i].h;
    np.items2[2 * i + 1] = its[i].qt;
  }

  // decode work list: split every group region into chunks of ~chunk_rows rows
  int64_t total_rows = off * ctx->max_batch;
  const int64_t target_ctas = (int64_t)ctx->num_sms * 6;
  int64_t c = (total_rows + target_ctas - 1) / target_ctas;
  c = ((c + 63) / 64) * 64;
  c = std::max<int64_t>(64, std::min<int64_t>(c, 4096));
  if (int ov = decode_chunk_rows_override()) c = ov;
  np.chunk_rows = (int)c;
  np.dec_cps = 0;
  np.gc_off.assign(ctx->ngl + 1, 0);
  if (ctx->dec_chunk > 0)
    for (int g = 0; g < ctx->ngl; ++g) {
      np.gc_off[g] = np.dec_cps;
      np.dec_cps += (int)(((int64_t)n_sink + np.win_g[g] + ctx->dec_chunk - 1) / ctx->dec_chunk);
    }
  np.gc_off[ctx->ngl] = np.dec_cps;
  np.g_chunk.resize(ctx->ngl + 1);
  np.max_chunks_per_group = 0;
  for (int g = 0; g < ctx->ngl; ++g) {
    np.g_chunk[g] = (int32_t)(np.chunks.size() / 3);
    int64_t R = (int64_t)n_sink + np.win_g[g];
    int n = 0;
    for (int64_t r0 = 0; r0 < R; r0 += c, ++n) {
      np.chunks.push_back(g);
      np.chunks.push_back((int32_t)r0);
      np.chunks.push_back((int32_t)std::min<int64_t>(R, r0 + c));
    }
    np.max_chunks_per_group = std::max(np.max_chunks_per_group, n);
  }
  np.g_chunk[ctx->ngl] = (int32_t)(np.chunks.size() / 3);

  // keep a bound cache if the footprint is unchanged
  bool same = p.set && p.rows_per_seq == np.rows_per_seq && p.n_sink == np.n_sink && p.win_g == np.win_g;
  if (same) {
    np.k_cache = p.k_cache;
    np.v_cache = p.v_cache;
    np.bound_batch = p.bound_batch;
    np.next_pos = p.k_cache ? 0 : -1;
    // the TMA tensor maps describe the same [rows, d] cache: keep them
    std::memcpy(np.kmap, p.kmap, sizeof(np.kmap));
    std::memcpy(np.vmap, p.vmap, sizeof(np.vmap));
    std::memcpy(np.kmap16, p.kmap16, sizeof(np.kmap16));
    std::memcpy(np.vmap16, p.vmap16, sizeof(np.vmap16));
    std::memcpy(np.kmap1, p.kmap1, sizeof(np.kmap1));
    std::memcpy(np.vmap1, p.vmap1, sizeof(np.vmap1));
    np.maps_ok = p.maps_ok;
  }
  st = upload_tables(ctx, np);
  if (st) return st;
  {
    DeviceGuard dg(ctx->device);
    free_tables(p);
  }
  p = np;
  ctx->ml_dirty = true;
  return ok();
}

moa_status moa_set_ragged(moa_ctx *ctx, int layer, int batch, const int64_t *seq_len,
                          const int32_t *window_per_seq_q_head) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  LayerPlan &p = ctx->layers[layer];
  ctx->ml_dirty = true;
  if (batch == 0) {
    DeviceGuard dg(ctx->device);
    free_ragged(p);
    p.next_pos = p.k_cache ? 0 : -1;
    return ok();
  }
  if (batch < 0 || batch > ctx->max_batch)
    return fail(MOA_ERR_INVALID_ARG, "ragged batch %d not in [0, max_batch=%d]", batch, ctx->max_batch);
  if (!seq_len) return fail(MOA_ERR_INVALID_ARG, "seq_len is NULL");
  if (ctx->nql > 0xffff || batch > 0x7fff)
    return fail(MOA_ERR_UNSUPPORTED, "ragged work items pack (h, b) into 16 + 15 bits");
  const int G = ctx->G;
  std::vector<int64_t> rn(seq_len, seq_len + batch);
  std::vector<int32_t> rw((size_t)batch * ctx->nql);
  for (int b = 0; b < batch; ++b) {
    if (rn[b] < 1 || rn[b] > p.N)
      return fail(MOA_ERR_INVALID_ARG, "seq_len[%d]=%lld not in [1, N=%lld]", b, (long long)rn[b],
                  (long long)p.N);
    for (int h = 0; h < ctx->nql; ++h) {
      const int32_t w = window_per_seq_q_head
                            ? window_per_seq_q_head[(size_t)b * ctx->Hq + ctx->g0 * G + h]
                            : p.win_q[h];
      if (w < 0 || w > p.win_g[h / G])
        return fail(MOA_ERR_INVALID_ARG,
                    "window[%d][%d]=%d not in [0, W_g=%d] (the cache capacity set by moa_set_spans)", b,
                    ctx->g0 * G + h, w, p.win_g[h / G]);
      if (w == 0 && p.n_sink < 1) return fail(MOA_ERR_INVALID_ARG, "W = 0 needs n_sink >= 1");
      if (p.bshift >= 0 && (w & ((1 << p.bshift) - 1)))
        return fail(MOA_ERR_INVALID_ARG, "window %d is not a multiple of the block %d", w, 1 << p.bshift);
      rw[(size_t)b * ctx->nql + h] = w;
    }
  }
  // two-tile prefill items of the real (b, h, q_block) work only (the kernel tiles against the
  // padded N, so a block costs what it costs there), in the uniform order of moa_set_spans:
  // heads by total kv-tile count over the batch, heaviest first; inside a head the items
  // heaviest first, q block then sequence (a uniform batch gives exactly the uniform list)
  struct It { int b, h, qb, cnt; int64_t hcost; int sc = 0; };
  std::vector<It> its;
  for (int h = 0; h < ctx->nql; ++h) {
    const size_t first = its.size();
    int64_t hc = 0;
    for (int b = 0; b < batch; ++b) {
      const int nqb = (int)((rn[b] + 2 * moa::kTile - 1) / (2 * moa::kTile));
      for (int qb = 0; qb < nqb; ++qb) {
        const moa::BlockTiles bt =
            moa::kv_block_tiles((int64_t)qb * 2 * moa::kTile, p.N, rw[(size_t)b * ctx->nql + h], p.n_sink,
                                p.bshift);
        const int c = bt.r[0].count() + (bt.has1 ? bt.r[1].count() : 0);
        hc += c;
        its.push_back({b, h, qb, c, 0});
        its.back().sc = sched_cost(bt, (int64_t)qb * 2 * moa::kTile, p.N, rw[(size_t)b * ctx->nql + h], p.n_sink,
                                   p.bshift);
      }
    }
    for (size_t k = first; k < its.size(); ++k) its[k].hcost = hc;
  }
  std::stable_sort(its.begin(), its.end(), [](const It &x, const It &y) {
    if (x.hcost != y.hcost) return x.hcost > y.hcost;
    if (x.h != y.h) return x.h < y.h;
    if (x.cnt != y.cnt) return x.cnt > y.cnt;
    if (x.qb != y.qb) return x.qb < y.qb;
    return x.b < y.b;
  });
  std::vector<int32_t> ri(its.size() * 2);
  std::vector<int> rcost(its.size());
  for (size_t i = 0; i < its.size(); ++i) {
    ri[2 * i] = its[i].h | (its[i].b << 16);
    ri[2 * i + 1] = its[i].qb;
    rcost[i] = its[i].sc;
  }
  // per-CTA greedy schedule of the ragged items (their costs vary with every sequence's length)
  std::vector<int32_t> rs, rso;
  if (!its.empty()) greedy_schedule(ri, rcost, (int)std::min<size_t>(its.size(), (size_t)std::max(1, ctx->num_sms)), rs, rso);
  DeviceGuard dg(ctx->device);
  free_ragged(p);
  if (ctx->device >= 0) {
    const size_t o_w = align16((size_t)batch * 8);
    const size_t o_i = align16(o_w + rw.size() * 4);
    const size_t o_s = align16(o_i + ri.size() * 4);
    const size_t o_so = align16(o_s + rs.size() * 4);
    const size_t total = o_so + rso.size() * 4;
    std::vector<unsigned char> host(total, 0);
    std::memcpy(host.data(), rn.data(), rn.size() * 8);
    std::memcpy(host.data() + o_w, rw.data(), rw.size() * 4);
    std::memcpy(host.data() + o_i, ri.data(), ri.size() * 4);
    std::memcpy(host.data() + o_s, rs.data(), rs.size() * 4);
    std::memcpy(host.data() + o_so, rso.data(), rso.size() * 4);
    void *d = nullptr;
    cudaError_t e = cudaMalloc(&d, total);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(ragged tables)");
    e = cudaMemcpy(d, host.data(), total, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(d);
      return cuda_fail(e, "cudaMemcpy(ragged tables)");
    }
    p.d_rag = d;
    p.d_seq_n = static_cast<const int64_t *>(d);
    p.d_win_bq = reinterpret_cast<const int32_t *>(static_cast<unsigned char *>(d) + o_w);
    p.d_rag_items2 = reinterpret_cast<const int32_t *>(static_cast<unsigned char *>(d) + o_i);
    p.d_rag_sched2 = rs.empty() ? nullptr : reinterpret_cast<const int32_t *>(static_cast<unsigned char *>(d) + o_s);
    p.d_rag_sched2_off = rso.empty() ? nullptr : reinterpret_cast<const int32_t *>(static_cast<unsigned char *>(d) + o_so);
    p.rag_sched2_ctas = rso.empty() ? 0 : (int)rso.size() - 1;
  }
  p.rag_items2 = std::move(ri);
  p.rag_batch = batch;
  p.rag_n = std::move(rn);
  p.rag_win = std::move(rw);
  p.next_pos = p.k_cache ? 0 : -1;
  return ok();
}

moa_status moa_layer_cache_bytes(const moa_ctx *ctx, int layer, int batch, size_t *k_bytes,
                                 size_t *v_bytes) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (batch < 1) return fail(MOA_ERR_INVALID_ARG, "batch %d invalid", batch);
  size_t b = layer_bytes(ctx, ctx->layers[layer], batch);
  if (k_bytes) *k_bytes = b;
  if (v_bytes) *v_bytes = b;
  return ok();
}

moa_status moa_cache_bytes(const moa_ctx *ctx, int batch, size_t *k_bytes, size_t *v_bytes) {
  if (!ctx) return fail(MOA_ERR_INVALID_ARG, "ctx is NULL");
  if (batch < 1) return fail(MOA_ERR_INVALID_ARG, "batch %d invalid", batch);
  size_t tot = 0;
  for (int l = 0; l < ctx->L; ++l) {
    if (!ctx->layers[l].set) return fail(MOA_ERR_STATE, "spans of layer %d not set", l);
    tot += align256(layer_bytes(ctx, ctx->layers[l], batch));
  }
  if (k_bytes) *k_bytes = tot;
  if (v_bytes) *v_bytes = tot;
  return ok();
}

moa_status moa_layer_offset(const moa_ctx *ctx, int layer, int batch, size_t *byte_offset) {
  moa_status st = check_layer(ctx, layer, false);
  if (st) return st;
  if (!byte_offset) return fail(MOA_ERR_INVALID_ARG, "byte_offset is NULL");
  size_t off = 0;
  for (int l = 0; l < layer; ++l) {
    if (!ctx->layers[l].set) return fail(MOA_ERR_STATE, "spans of layer %d not set", l);
    off += align256(layer_bytes(ctx, ctx->layers[l], batch));
  }
  *byte_offset = off;
  return ok();
}

moa_status moa_workspace_bytes(const moa_ctx *ctx, int batch, size_t *bytes) {
  if (!ctx || !bytes) return fail(MOA_ERR_INVALID_ARG, "NULL argument");
  if (batch < 1) return fail(MOA_ERR_INVALID_ARG, "batch %d invalid", batch);
  size_t mx = 256;
  for (const auto &p : ctx->layers)
    if (p.set)
      mx = std::max(mx, moa::decode_ws_bytes(batch, (int)(p.chunks.size() / 3), ctx->G, ctx->d));
  if (ctx->dtype == MOA_BF16 && ctx->device >= 0) {
    DeviceGuard dg(ctx->device);
    for (const auto &p : ctx->layers)
      if (p.set) mx = std::max(mx, moa::decode_mma_ws_bytes(batch, ctx->ngl, ctx->G, ctx->d, p.dec_cps));
  }
  *bytes = mx;
  return ok();
}

moa_status moa_bind_layer_cache(moa_ctx *ctx, int layer, void *k_cache, void *v_cache, int batch) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (!k_cache || !v_cache) return fail(MOA_ERR_INVALID_ARG, "cache pointer is NULL");
  if (((uintptr_t)k_cache | (uintptr_t)v_cache) & 255)
    return fail(MOA_ERR_INVALID_ARG, "cache pointers must be 256-byte aligned");
  if (batch < 1 || batch > ctx->max_batch)
    return fail(MOA_ERR_INVALID_ARG, "batch %d not in [1, max_batch=%d]", batch, ctx->max_batch);
  LayerPlan &p = ctx->layers[layer];
  p.k_cache = k_cache;
  p.v_cache = v_cache;
  p.bound_batch = batch;
  p.next_pos = 0;
  p.maps_ok = false;
  ctx->last_cache_write = moa_ctx::kAllLayers;
  ctx->ml_dirty = true;
  if (ctx->device >= 0) {
    // rows not yet reached by the sequence must hold finite values: the tensor-core decode
    // multiplies masked rows by a zero probability, and 0 * NaN would poison the sum
    DeviceGuard dg(ctx->device);
    const size_t bytes = layer_bytes(ctx, p, batch);
    cudaError_t e = cudaMemset(k_cache, 0, bytes);
    if (e == cudaSuccess) e = cudaMemset(v_cache, 0, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(cache)");
  }
  if (ctx->device >= 0 && ctx->dtype == MOA_BF16) {
    DeviceGuard dg(ctx->device);
    const int64_t rows = (int64_t)batch * p.rows_per_seq;
    if (!moa::encode_cache_map(p.kmap, k_cache, ctx->d, rows, 64) ||
        !moa::encode_cache_map(p.vmap, v_cache, ctx->d, rows, 64) ||
        !moa::encode_cache_map(p.kmap16, k_cache, ctx->d, rows, 16) ||
        !moa::encode_cache_map(p.vmap16, v_cache, ctx->d, rows, 16) ||
        !moa::encode_cache_map(p.kmap1, k_cache, ctx->d, rows, 1) ||
        !moa::encode_cache_map(p.vmap1, v_cache, ctx->d, rows, 1))
      return fail(MOA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the layer %d cache", layer);
    p.maps_ok = true;
  }
  return ok();
}

moa_status moa_bind_cache(moa_ctx *ctx, void *k_cache, void *v_cache, int batch) {
  if (!ctx) return fail(MOA_ERR_INVALID_ARG, "ctx is NULL");
  size_t kb = 0;
  moa_status st = moa_cache_bytes(ctx, batch, &kb, nullptr);
  if (st) return st;
  size_t off = 0;
  for (int l = 0; l < ctx->L; ++l) {
    st = moa_bind_layer_cache(ctx, l, static_cast<char *>(k_cache) + off,
                              static_cast<char *>(v_cache) + off, batch);
    if (st) return st;
    off += align256(layer_bytes(ctx, ctx->layers[l], batch));
  }
  return ok();
}

// ---------------------------------------------------------------------------------------------
// launches
// ---------------------------------------------------------------------------------------------

static moa_status check_launch_common(const moa_ctx *ctx, int layer, int batch) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (ctx->device < 0) return fail(MOA_ERR_STATE, "planning context (device -1) cannot launch");
  const LayerPlan &p = ctx->layers[layer];
  if (!p.k_cache) return fail(MOA_ERR_STATE, "no cache bound for layer %d", layer);
  if (batch < 1 || batch > p.bound_batch)
    return fail(MOA_ERR_INVALID_ARG, "batch %d not in [1, bound batch %d]", batch, p.bound_batch);
  return check_sticky(ctx);
}

static bool aligned16(const void *ptr) { return ((uintptr_t)ptr & 15) == 0; }

// MOA_PP_FUSED_FILL=0: moa_prefill runs the separate cache-fill kernel (A/B diagnostics)
static bool sched2_enabled() {  // MOA_PP_SCHED=0: static round robin over the item list (A/B)
  const char *e = std::getenv("MOA_PP_SCHED");
  return !(e && e[0] == '0');
}

static bool fused_fill_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("MOA_PP_FUSED_FILL");
    return !(e && e[0] == '0');
  }();
  return on;
}

static moa_status prefill_common(moa_ctx *ctx, int layer, const void *q, const void *k, const void *v, void *o,
                                 int64_t q_row_stride, int64_t kv_row_stride, int64_t o_row_stride, int batch,
                                 int64_t N, float scale, float *lse_out, moa_stream_t stream, bool fill) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (ctx->device < 0) return fail(MOA_ERR_STATE, "planning context (device -1) cannot launch");
  LayerPlan &p = ctx->layers[layer];
  if (fill && !p.k_cache) return fail(MOA_ERR_STATE, "no cache bound for layer %d", layer);
  const int max_b = fill ? p.bound_batch : ctx->max_batch;
  if (batch < 1 || batch > max_b) return fail(MOA_ERR_INVALID_ARG, "batch %d not in [1, %d]", batch, max_b);
  st = check_sticky(ctx);
  if (st) return st;
  if (!q || !k || !v || !o) return fail(MOA_ERR_INVALID_ARG, "q/k/v/o must be non-NULL");
  if (N != p.N)
    return fail(MOA_ERR_SHAPE, "prefill N=%lld but spans were set for N=%lld", (long long)N, (long long)p.N);
  const int64_t d = ctx->d;
  if (q_row_stride < ctx->nql * d || o_row_stride < ctx->nql * d || kv_row_stride < ctx->ngl * d)
    return fail(MOA_ERR_SHAPE, "row strides smaller than local heads * head_dim");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) ||
      (q_row_stride * (int64_t)esize(ctx)) % 16 || (kv_row_stride * (int64_t)esize(ctx)) % 16 ||
      (o_row_stride * (int64_t)esize(ctx)) % 16)
    return fail(MOA_ERR_INVALID_ARG, "q/k/v/o pointers and row strides must be 16-byte aligned");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(MOA_ERR_INVALID_ARG, "scale must be finite > 0");
  DeviceGuard dg(ctx->device);
  moa::PrefillArgs a{};
  a.q = q; a.k = k; a.v = v; a.o = o;
  a.q_row_stride = q_row_stride; a.kv_row_stride = kv_row_stride; a.o_row_stride = o_row_stride;
  a.batch = batch; a.N = N; a.scale = scale; a.lse = lse_out; a.n_sink = p.n_sink;
  a.nql = ctx->nql; a.G = ctx->G; a.d = ctx->d;
  a.d_win_q = p.d_win_q; a.d_items = p.d_items; a.n_items = (int)(p.items.size() / 2);
  a.d_items2 = p.d_items2; a.n_items2 = (int)(p.items2.size() / 2);
  // greedy per-CTA schedule: planned for max_batch (the common case); other batches round robin
  const bool sched = p.d_sched2 && batch == p.sched2_batch && sched2_enabled();
  a.d_sched2 = sched ? p.d_sched2 : nullptr;
  a.d_sched2_off = sched ? p.d_sched2_off : nullptr;
  a.sched2_ctas = sched ? (int)p.sched2_off.size() - 1 : 0;
  if (p.rag_batch > 0) {  // ragged batch: its own schedule of the real items
    const bool rs = p.d_rag_sched2 && sched2_enabled();
    a.d_sched2 = rs ? p.d_rag_sched2 : nullptr;
    a.d_sched2_off = rs ? p.d_rag_sched2_off : nullptr;
    a.sched2_ctas = rs ? p.rag_sched2_ctas : 0;
  }
  a.bshift = p.bshift;
  if (p.rag_batch) {
    if (batch != p.rag_batch)
      return fail(MOA_ERR_SHAPE, "layer %d is ragged over %d sequences, prefill batch %d", layer, p.rag_batch,
                  batch);
    a.d_seq_n = p.d_seq_n;
    a.d_win_bq = p.d_win_bq;
    a.d_items_rag = p.d_rag_items2;
    a.n_items_rag = (int)(p.rag_items2.size() / 2);
  }
  // fused cache fill (a5 inside the prefill kernel): bf16, token mask, uniform batch
  const bool fused = fill && ctx->dtype == MOA_BF16 && p.bshift < 0 && !p.rag_batch && p.maps_ok &&
                     fused_fill_enabled();
  if (fused) {
    a.fill = 1;
    a.kmap16 = p.kmap16; a.vmap16 = p.vmap16; a.kmap1 = p.kmap1; a.vmap1 = p.vmap1;
    a.k_cache = p.k_cache; a.v_cache = p.v_cache; a.rows_per_seq = p.rows_per_seq;
    a.d_g_off = p.d_g_off; a.d_win_g = p.d_win_g; a.d_fill_h = p.d_fill_h;
  }
  int e = ctx->dtype == MOA_FP32 ? moa::launch_prefill_f32(a, stream) : moa::launch_prefill_bf16_pp(a, stream);
  if (e) return cuda_fail((cudaError_t)e, "prefill launch");
  if (!fill) {
    ctx->last_cache_write = -1;
    return ok();
  }
  if (fused) {
    p.next_pos = N;
    ctx->last_cache_write = layer;
    return ok();
  }
  moa::CacheArgs c{};
  c.k = k; c.v = v; c.row_stride = kv_row_stride; c.k_cache = p.k_cache; c.v_cache = p.v_cache;
  c.rows_per_seq = p.rows_per_seq; c.d_g_off = p.d_g_off; c.d_win_g = p.d_win_g;
  c.ngl = ctx->ngl; c.d = ctx->d; c.n_sink = p.n_sink; c.batch = batch; c.N_or_pos = N;
  c.esize = (int)esize(ctx);
  c.max_region_rows = (int64_t)p.n_sink + *std::max_element(p.win_g.begin(), p.win_g.end());
  c.d_seq_n = p.rag_batch ? p.d_seq_n : nullptr;
  e = moa::launch_cache_fill(c, stream);
  if (e) return cuda_fail((cudaError_t)e, "cache fill launch");
  p.next_pos = p.rag_batch ? kRaggedPos : N;
  ctx->last_cache_write = layer;
  return ok();
}

moa_status moa_prefill(moa_ctx *ctx, int layer, const void *q, const void *k, const void *v,
                       void *o, int64_t q_row_stride, int64_t kv_row_stride,
                       int64_t o_row_stride, int batch, int64_t N, float scale, float *lse_out,
                       void *workspace, size_t ws_bytes, moa_stream_t stream) {
  (void)workspace;
  (void)ws_bytes;
  return prefill_common(ctx, layer, q, k, v, o, q_row_stride, kv_row_stride, o_row_stride, batch, N, scale,
                        lse_out, stream, true);
}

moa_status moa_prefill_attn(moa_ctx *ctx, int layer, const void *q, const void *k, const void *v, void *o,
                            int64_t q_row_stride, int64_t kv_row_stride, int64_t o_row_stride, int batch,
                            int64_t N, float scale, float *lse_out, moa_stream_t stream) {
  return prefill_common(ctx, layer, q, k, v, o, q_row_stride, kv_row_stride, o_row_stride, batch, N, scale,
                        lse_out, stream, false);
}

moa_status moa_cache_fill(moa_ctx *ctx, int layer, const void *k, const void *v,
                          int64_t kv_row_stride, int batch, int64_t N, moa_stream_t stream) {
  moa_status st = check_launch_common(ctx, layer, batch);
  if (st) return st;
  LayerPlan &p = ctx->layers[layer];
  if (!k || !v) return fail(MOA_ERR_INVALID_ARG, "k/v must be non-NULL");
  if (N < 1) return fail(MOA_ERR_INVALID_ARG, "N must be >= 1");
  if (kv_row_stride < ctx->ngl * ctx->d) return fail(MOA_ERR_SHAPE, "kv_row_stride too small");
  if (!aligned16(k) || !aligned16(v) || (kv_row_stride * (int64_t)esize(ctx)) % 16)
    return fail(MOA_ERR_INVALID_ARG, "k/v pointers and row stride must be 16-byte aligned");
  DeviceGuard dg(ctx->device);
  moa::CacheArgs c{};
  c.k = k; c.v = v; c.row_stride = kv_row_stride; c.k_cache = p.k_cache; c.v_cache = p.v_cache;
  c.rows_per_seq = p.rows_per_seq; c.d_g_off = p.d_g_off; c.d_win_g = p.d_win_g;
  c.ngl = ctx->ngl; c.d = ctx->d; c.n_sink = p.n_sink; c.batch = batch; c.N_or_pos = N;
  c.esize = (int)esize(ctx);
  c.max_region_rows = (int64_t)p.n_sink + *std::max_element(p.win_g.begin(), p.win_g.end());
  if (p.rag_batch) {
    if (N != p.N || batch != p.rag_batch)
      return fail(MOA_ERR_SHAPE, "layer %d is ragged: cache_fill needs N=%lld (padded) and batch %d", layer,
                  (long long)p.N, p.rag_batch);
    c.d_seq_n = p.d_seq_n;
  }
  int e = moa::launch_cache_fill(c, stream);
  if (e) return cuda_fail((cudaError_t)e, "cache fill launch");
  p.next_pos = p.rag_batch ? kRaggedPos : N;
  ctx->last_cache_write = layer;
  return ok();
}

moa_status moa_kv_append(moa_ctx *ctx, int layer, const void *k_new, const void *v_new,
                         int64_t kv_batch_stride, int batch, int64_t pos, moa_stream_t stream) {
  moa_status st = check_launch_common(ctx, layer, batch);
  if (st) return st;
  LayerPlan &p = ctx->layers[layer];
  if (!k_new || !v_new) return fail(MOA_ERR_INVALID_ARG, "k_new/v_new must be non-NULL");
  if (p.rag_batch)
    return fail(MOA_ERR_STATE, "layer %d is ragged: use moa_decode_step_fused_ragged", layer);
  if (pos != p.next_pos)
    return fail(MOA_ERR_STATE, "kv_append pos=%lld but layer %d expects %lld", (long long)pos, layer,
                (long long)p.next_pos);
  if (kv_batch_stride < ctx->ngl * ctx->d) return fail(MOA_ERR_SHAPE, "kv_batch_stride too small");
  if (!aligned16(k_new) || !aligned16(v_new) || (kv_batch_stride * (int64_t)esize(ctx)) % 16)
    return fail(MOA_ERR_INVALID_ARG, "k_new/v_new and batch stride must be 16-byte aligned");
  DeviceGuard dg(ctx->device);
  moa::CacheArgs c{};
  c.k = k_new; c.v = v_new; c.row_stride = kv_batch_stride; c.k_cache = p.k_cache; c.v_cache = p.v_cache;
  c.rows_per_seq = p.rows_per_seq; c.d_g_off = p.d_g_off; c.d_win_g = p.d_win_g;
  c.ngl = ctx->ngl; c.d = ctx->d; c.n_sink = p.n_sink; c.batch = batch; c.N_or_pos = pos;
  c.esize = (int)esize(ctx);
  c.max_region_rows = (int64_t)p.n_sink + *std::max_element(p.win_g.begin(), p.win_g.end());
  int e = moa::launch_kv_append(c, stream);
  if (e) return cuda_fail((cudaError_t)e, "kv_append launch");
  p.next_pos = pos + 1;
  ctx->last_cache_write = layer;
  return ok();
}

// MOA_DEC_EARLY=0 disables the early cache streaming of the decode kernel (diagnostics)
static bool early_read_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("MOA_DEC_EARLY");
    return !(e && e[0] == '0');
  }();
  return on;
}

static moa_status decode_common(moa_ctx *ctx, int layer, const void *q, const void *k_new,
                                const void *v_new, void *o, int64_t q_batch_stride,
                                int64_t kv_batch_stride, int64_t o_batch_stride, int batch,
                                int64_t pos, float scale, float *lse_out, void *workspace,
                                size_t ws_bytes, moa_stream_t stream, bool fused,
                                const int64_t *d_pos = nullptr) {
  moa_status st = check_launch_common(ctx, layer, batch);
  if (st) return st;
  LayerPlan &p = ctx->layers[layer];
  if (!q || !o) return fail(MOA_ERR_INVALID_ARG, "q/o must be non-NULL");
  if (fused && (!k_new || !v_new)) return fail(MOA_ERR_INVALID_ARG, "k_new/v_new must be non-NULL");
  if (d_pos) {  // ragged: per-sequence positions in device memory (not checkable here)
    if (p.rag_batch && batch != p.rag_batch)
      return fail(MOA_ERR_SHAPE, "layer %d is ragged over %d sequences, decode batch %d", layer, p.rag_batch,
                  batch);
    if ((uintptr_t)d_pos & 7) return fail(MOA_ERR_INVALID_ARG, "pos array must be 8-byte aligned");
    pos = 0;
  } else {
    if (p.rag_batch)
      return fail(MOA_ERR_STATE, "layer %d is ragged: use moa_decode_step_fused_ragged", layer);
    int64_t expect = fused ? p.next_pos : p.next_pos - 1;
    if (pos != expect || pos < 0)
      return fail(MOA_ERR_STATE, "decode pos=%lld but layer %d expects %lld (append before decode)",
                  (long long)pos, layer, (long long)expect);
  }
  const int32_t *d_win_bq = p.rag_batch ? p.d_win_bq : nullptr;
  const int64_t d = ctx->d;
  if (q_batch_stride < ctx->nql * d || o_batch_stride < ctx->nql * d)
    return fail(MOA_ERR_SHAPE, "q/o batch stride smaller than local heads * head_dim");
  if (fused && kv_batch_stride < ctx->ngl * d) return fail(MOA_ERR_SHAPE, "kv_batch_stride too small");
  const int64_t es = (int64_t)esize(ctx);
  if (!aligned16(q) || !aligned16(o) || (q_batch_stride * es) % 16 || (o_batch_stride * es) % 16 ||
      (fused && (!aligned16(k_new) || !aligned16(v_new) || (kv_batch_stride * es) % 16)))
    return fail(MOA_ERR_INVALID_ARG, "decode pointers and batch strides must be 16-byte aligned");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(MOA_ERR_INVALID_ARG, "scale must be finite > 0");
  const int n_chunks = (int)(p.chunks.size() / 3);
  const bool mma_path = ctx->dtype == MOA_BF16;
  size_t need = mma_path ? moa::decode_mma_ws_bytes(batch, ctx->ngl, ctx->G, ctx->d, p.dec_cps)
                         : moa::decode_ws_bytes(batch, n_chunks, ctx->G, ctx->d);
  if (!workspace || ws_bytes < need)
    return fail(MOA_ERR_OOM, "workspace of %zu bytes < %zu needed", ws_bytes, need);
  if (!aligned16(workspace)) return fail(MOA_ERR_INVALID_ARG, "workspace must be 16-byte aligned");
  DeviceGuard dg(ctx->device);
  if (mma_path) {
    if (ctx->ngl > 128) return fail(MOA_ERR_UNSUPPORTED, "more than 128 local kv-groups");
    if (!p.maps_ok) return fail(MOA_ERR_STATE, "layer %d cache has no tensor maps (re-bind the cache)", layer);
    moa::DecodeMmaArgs m{};
    m.kmap = p.kmap; m.vmap = p.vmap; m.kmap16 = p.kmap16; m.vmap16 = p.vmap16; m.q = q; m.o = o; m.q_bs = q_batch_stride; m.o_bs = o_batch_stride;
    m.k_new = fused ? k_new : nullptr; m.v_new = fused ? v_new : nullptr; m.kv_bs = kv_batch_stride;
    m.k_cache = p.k_cache; m.v_cache = p.v_cache; m.rows_per_seq = p.rows_per_seq;
    m.d_g_off = p.d_g_off; m.d_win_g = p.d_win_g; m.d_win_q = p.d_win_q;
    m.ngl = ctx->ngl; m.G = ctx->G; m.d = ctx->d; m.n_sink = p.n_sink; m.batch = batch;
    m.pos = pos; m.scale = scale; m.lse = lse_out; m.ws_part = static_cast<float *>(workspace);
    m.d_pos = d_pos; m.d_win_bq = d_win_bq;
    m.counters = p.d_counters;
    m.chunk = ctx->dec_chunk;
    m.chunks_per_seq = p.dec_cps;
    m.d_gc_off = p.d_gc_off;
    m.early_read = early_read_enabled() && ctx->last_cache_write != layer &&
                   ctx->last_cache_write != moa_ctx::kAllLayers;
    m.peers = ctx->d_peers; m.n_peers = ctx->n_peers; m.peer_head0 = ctx->peer_head0;
    m.peer_bs = ctx->peer_bs; m.peer_ls = ctx->peer_ls; m.layer = layer;
    int e = moa::launch_decode_mma(m, stream);
    if (e) return cuda_fail((cudaError_t)e, "decode launch");
    if (fused && !d_pos) p.next_pos = pos + 1;
    ctx->last_cache_write = fused ? layer : -1;
    return ok();
  }
  if (ctx->n_peers) return fail(MOA_ERR_UNSUPPORTED, "peer outputs need the bf16 decode");
  moa::DecodeArgs a{};
  a.q = q; a.o = o; a.q_batch_stride = q_batch_stride; a.o_batch_stride = o_batch_stride;
  a.k_new = fused ? k_new : nullptr; a.v_new = fused ? v_new : nullptr; a.kv_batch_stride = kv_batch_stride;
  a.k_cache = p.k_cache; a.v_cache = p.v_cache; a.rows_per_seq = p.rows_per_seq;
  a.d_g_off = p.d_g_off; a.d_win_g = p.d_win_g; a.d_win_q = p.d_win_q;
  a.d_chunks = p.d_chunks; a.d_g_chunk = p.d_g_chunk; a.n_chunks = n_chunks;
  a.max_chunks_per_group = p.max_chunks_per_group;
  a.ngl = ctx->ngl; a.G = ctx->G; a.d = ctx->d; a.n_sink = p.n_sink; a.batch = batch;
  a.pos = pos; a.scale = scale; a.lse = lse_out;
  a.d_pos = d_pos; a.d_win_bq = d_win_bq;
  a.ws_part = static_cast<float *>(workspace);
  a.counters = p.d_counters;
  int e = moa::launch_decode(a, ctx->dtype, fused, stream);
  if (e) return cuda_fail((cudaError_t)e, "decode launch");
  if (fused && !d_pos) p.next_pos = pos + 1;
  ctx->last_cache_write = fused ? layer : -1;
  return ok();
}

moa_status moa_decode_step(moa_ctx *ctx, int layer, const void *q, void *o,
                           int64_t q_batch_stride, int64_t o_batch_stride, int batch,
                           int64_t pos, float scale, float *lse_out, void *workspace,
                           size_t ws_bytes, moa_stream_t stream) {
  return decode_common(ctx, layer, q, nullptr, nullptr, o, q_batch_stride, 0, o_batch_stride,
                       batch, pos, scale, lse_out, workspace, ws_bytes, stream, false);
}

moa_status moa_decode_step_fused(moa_ctx *ctx, int layer, const void *q, const void *k_new,
                                 const void *v_new, void *o, int64_t q_batch_stride,
                                 int64_t kv_batch_stride, int64_t o_batch_stride, int batch,
                                 int64_t pos, float scale, float *lse_out, void *workspace,
                                 size_t ws_bytes, moa_stream_t stream) {
  return decode_common(ctx, layer, q, k_new, v_new, o, q_batch_stride, kv_batch_stride,
                       o_batch_stride, batch, pos, scale, lse_out, workspace, ws_bytes, stream, true);
}

moa_status moa_decode_step_fused_ragged(moa_ctx *ctx, int layer, const void *q, const void *k_new,
                                        const void *v_new, void *o, int64_t q_batch_stride,
                                        int64_t kv_batch_stride, int64_t o_batch_stride, int batch,
                                        const int64_t *pos, float scale, float *lse_out, void *workspace,
                                        size_t ws_bytes, moa_stream_t stream) {
  if (!pos) return fail(MOA_ERR_INVALID_ARG, "pos array is NULL");
  return decode_common(ctx, layer, q, k_new, v_new, o, q_batch_stride, kv_batch_stride, o_batch_stride,
                       batch, 0, scale, lse_out, workspace, ws_bytes, stream, true, pos);
}

// ---- cross-layer decode ------------------------------------------------
// Device image: DecodeLayerDesc[L] then 4 CUtensorMap per layer (128-byte aligned).  Layers that
// are not set or not bound get a zeroed descriptor (the launch checks its layers).
moa_status moa_prepare_layers(moa_ctx *ctx) {
  if (!ctx) return fail(MOA_ERR_INVALID_ARG, "ctx is NULL");
  if (ctx->device < 0) return fail(MOA_ERR_STATE, "planning context (device -1) cannot launch");
  if (ctx->dtype != MOA_BF16) return fail(MOA_ERR_UNSUPPORTED, "cross-layer decode is bf16 only");
  const size_t desc_bytes = align256((size_t)ctx->L * sizeof(moa::DecodeLayerDesc));
  const size_t total = desc_bytes + (size_t)ctx->L * 4 * 128;
  DeviceGuard dg(ctx->device);
  if (!ctx->d_ml) {
    cudaError_t e = cudaMalloc(&ctx->d_ml, total);
    if (e != cudaSuccess) {
      ctx->d_ml = nullptr;
      return cuda_fail(e, "cudaMalloc(cross-layer descriptors)");
    }
  }
  std::vector<unsigned char> img(total, 0);
  auto *desc = reinterpret_cast<moa::DecodeLayerDesc *>(img.data());
  unsigned char *dmaps = static_cast<unsigned char *>(ctx->d_ml) + desc_bytes;
  for (int l = 0; l < ctx->L; ++l) {
    const LayerPlan &p = ctx->layers[l];
    if (!p.set || !p.k_cache || !p.maps_ok) continue;
    moa::DecodeLayerDesc &d = desc[l];
    d.maps = dmaps + (size_t)l * 4 * 128;
    d.kc = p.k_cache;
    d.vc = p.v_cache;
    d.g_off = p.d_g_off;
    d.win_g = p.d_win_g;
    d.win_q = p.d_win_q;
    d.gc_off = p.d_gc_off;
    d.counters = p.d_counters;
    d.rows_per_seq = p.rows_per_seq;
    d.dec_cps = p.dec_cps;
    unsigned char *m = img.data() + desc_bytes + (size_t)l * 4 * 128;
    std::memcpy(m, p.kmap, 128);
    std::memcpy(m + 128, p.vmap, 128);
    std::memcpy(m + 256, p.kmap16, 128);
    std::memcpy(m + 384, p.vmap16, 128);
  }
  if (img != ctx->ml_image) {
    // launches still in flight may read the old image
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(ctx->d_ml, img.data(), total, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "upload of the cross-layer descriptors");
    ctx->ml_image = std::move(img);
  }
  ctx->ml_dirty = false;
  return ok();
}

moa_status moa_decode_step_fused_layers(moa_ctx *ctx, int layer0, int n_layers, const void *q, const void *k_new,
                                        const void *v_new, void *o, int64_t q_layer_stride,
                                        int64_t kv_layer_stride, int64_t o_layer_stride, int64_t q_batch_stride,
                                        int64_t kv_batch_stride, int64_t o_batch_stride, int batch, int64_t pos,
                                        float scale, float *lse_out, int64_t lse_layer_stride, void *workspace,
                                        size_t ws_bytes, moa_stream_t stream) {
  if (!ctx) return fail(MOA_ERR_INVALID_ARG, "ctx is NULL");
  if (n_layers < 1 || layer0 < 0 || layer0 + n_layers > ctx->L)
    return fail(MOA_ERR_INVALID_ARG, "layers [%d, %d) not in [0, %d)", layer0, layer0 + n_layers, ctx->L);
  if (ctx->dtype != MOA_BF16) return fail(MOA_ERR_UNSUPPORTED, "cross-layer decode is bf16 only");
  if (ctx->ngl > 128) return fail(MOA_ERR_UNSUPPORTED, "more than 128 local kv-groups");
  if (!q || !o || !k_new || !v_new) return fail(MOA_ERR_INVALID_ARG, "q/k_new/v_new/o must be non-NULL");
  const int64_t d = ctx->d;
  if (q_batch_stride < ctx->nql * d || o_batch_stride < ctx->nql * d || kv_batch_stride < ctx->ngl * d)
    return fail(MOA_ERR_SHAPE, "batch strides smaller than local heads * head_dim");
  // inputs may be shared by the layers (layer stride 0); outputs may not overlap
  auto bad_in = [&](int64_t ls, int64_t bs) { return ls != 0 && ls < (int64_t)batch * bs; };
  if (n_layers > 1 && (bad_in(q_layer_stride, q_batch_stride) || bad_in(kv_layer_stride, kv_batch_stride) ||
                       o_layer_stride < (int64_t)batch * o_batch_stride ||
                       (lse_out && lse_layer_stride < (int64_t)batch * ctx->nql)))
    return fail(MOA_ERR_SHAPE, "layer strides: inputs 0 or >= one layer's batch, outputs >= one layer's batch");
  if (q_layer_stride < 0 || kv_layer_stride < 0) return fail(MOA_ERR_SHAPE, "negative layer stride");
  const int64_t es = 2;
  if (!aligned16(q) || !aligned16(o) || !aligned16(k_new) || !aligned16(v_new) ||
      ((q_batch_stride | o_batch_stride | kv_batch_stride | q_layer_stride | o_layer_stride | kv_layer_stride) * es) % 16)
    return fail(MOA_ERR_INVALID_ARG, "decode pointers and strides must be 16-byte aligned");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(MOA_ERR_INVALID_ARG, "scale must be finite > 0");
  int n_sink = -1;
  int64_t max_rows = 0, min_rows = INT64_MAX;
  size_t per_layer = 256;
  for (int l = layer0; l < layer0 + n_layers; ++l) {
    moa_status st = check_launch_common(ctx, l, batch);
    if (st) return st;
    const LayerPlan &p = ctx->layers[l];
    if (p.rag_batch) return fail(MOA_ERR_STATE, "layer %d is ragged", l);
    if (!p.maps_ok) return fail(MOA_ERR_STATE, "layer %d cache has no tensor maps (re-bind the cache)", l);
    if (pos != p.next_pos || pos < 0)
      return fail(MOA_ERR_STATE, "decode pos=%lld but layer %d expects %lld", (long long)pos, l,
                  (long long)p.next_pos);
    if (n_sink >= 0 && p.n_sink != n_sink) return fail(MOA_ERR_STATE, "layers disagree on the sink count");
    n_sink = p.n_sink;
    max_rows = std::max<int64_t>(max_rows, (int64_t)batch * p.rows_per_seq);
    min_rows = std::min<int64_t>(min_rows, (int64_t)batch * p.rows_per_seq);
    DeviceGuard dg(ctx->device);
    per_layer = std::max(per_layer, moa::decode_mma_ws_bytes(batch, ctx->ngl, ctx->G, ctx->d, p.dec_cps));
  }
  if (!workspace || ws_bytes < per_layer * n_layers)
    return fail(MOA_ERR_OOM, "workspace of %zu bytes < %zu needed (%d layers)", ws_bytes, per_layer * n_layers,
                n_layers);
  if (!aligned16(workspace)) return fail(MOA_ERR_INVALID_ARG, "workspace must be 16-byte aligned");
  if (ctx->ml_dirty) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing((cudaStream_t)stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
      return fail(MOA_ERR_STATE, "call moa_prepare_layers before capturing a cross-layer decode");
    moa_status st = moa_prepare_layers(ctx);
    if (st) return st;
  }
  const LayerPlan &p0 = ctx->layers[layer0];
  DeviceGuard dg(ctx->device);
  moa::DecodeLayersArgs la{};
  moa::DecodeMmaArgs &m = la.a;
  m.q = q; m.o = o; m.q_bs = q_batch_stride; m.o_bs = o_batch_stride;
  m.k_new = k_new; m.v_new = v_new; m.kv_bs = kv_batch_stride;
  m.k_cache = p0.k_cache; m.v_cache = p0.v_cache; m.rows_per_seq = p0.rows_per_seq;
  m.d_g_off = p0.d_g_off; m.d_win_g = p0.d_win_g; m.d_win_q = p0.d_win_q;
  m.ngl = ctx->ngl; m.G = ctx->G; m.d = ctx->d; m.n_sink = n_sink; m.batch = batch;
  m.pos = pos; m.scale = scale; m.lse = lse_out; m.ws_part = static_cast<float *>(workspace);
  m.counters = p0.d_counters;
  m.chunk = ctx->dec_chunk;
  m.chunks_per_seq = p0.dec_cps;
  m.d_gc_off = p0.d_gc_off;
  m.early_read = 0;
  m.peers = ctx->d_peers; m.n_peers = ctx->n_peers; m.peer_head0 = ctx->peer_head0;
  m.peer_bs = ctx->peer_bs; m.peer_ls = ctx->peer_ls; m.layer = layer0;
  la.q_ls = q_layer_stride;
  la.o_ls = o_layer_stride;
  la.kvn_ls = kv_layer_stride;
  la.lse_ls = lse_layer_stride;
  la.part_ls = (int64_t)(per_layer / 4);
  la.max_rows = max_rows;
  la.min_rows = min_rows;
  // at most kMaxLayersPerLaunch layers per launch (the kernel keeps a per-layer table per CTA)
  constexpr int kMaxLayersPerLaunch = 32;
  for (int c0 = 0; c0 < n_layers; c0 += kMaxLayersPerLaunch) {
    moa::DecodeLayersArgs lc = la;
    lc.d_layers = reinterpret_cast<const moa::DecodeLayerDesc *>(ctx->d_ml) + layer0 + c0;
    lc.n_layers = std::min(kMaxLayersPerLaunch, n_layers - c0);
    lc.a.q = static_cast<const char *>(q) + c0 * q_layer_stride * es;
    lc.a.o = static_cast<char *>(o) + c0 * o_layer_stride * es;
    lc.a.k_new = static_cast<const char *>(k_new) + c0 * kv_layer_stride * es;
    lc.a.v_new = static_cast<const char *>(v_new) + c0 * kv_layer_stride * es;
    lc.a.lse = lse_out ? lse_out + c0 * lse_layer_stride : nullptr;
    lc.a.ws_part = static_cast<float *>(workspace) + c0 * la.part_ls;
    lc.a.early_read = c0 > 0 && early_read_enabled();  // predecessor: the previous chunk (other layers)
    lc.a.layer = layer0 + c0;
    int e = moa::launch_decode_mma_layers(lc, stream);
    if (e) return cuda_fail((cudaError_t)e, "cross-layer decode launch");
  }
  for (int l = layer0; l < layer0 + n_layers; ++l) ctx->layers[l].next_pos = pos + 1;
  ctx->last_cache_write = moa_ctx::kAllLayers;
  return ok();
}

// ---- fused head-output all-gather ----------------------------------
moa_status moa_set_peer_outputs(moa_ctx *ctx, int n_peers, void *const *peer_o, unsigned int *const *peer_flags,
                                int64_t peer_batch_stride, int64_t peer_layer_stride, int head0) {
  if (!ctx) return fail(MOA_ERR_INVALID_ARG, "ctx is NULL");
  if (ctx->device < 0) return fail(MOA_ERR_STATE, "planning context (device -1) cannot launch");
  if (n_peers < 0 || n_peers > 16) return fail(MOA_ERR_INVALID_ARG, "n_peers %d not in [0, 16]", n_peers);
  DeviceGuard dg(ctx->device);
  if (n_peers == 0) {
    ctx->n_peers = 0;
    return ok();
  }
  if (ctx->dtype != MOA_BF16) return fail(MOA_ERR_UNSUPPORTED, "peer outputs need the bf16 decode");
  if (!peer_o || !peer_flags) return fail(MOA_ERR_INVALID_ARG, "peer pointer arrays are NULL");
  if (head0 < 0 || peer_batch_stride < (int64_t)(head0 + ctx->nql) * ctx->d || peer_layer_stride < 0)
    return fail(MOA_ERR_SHAPE, "peer layout: head0 %d + %d local heads do not fit the batch stride %lld", head0,
                ctx->nql, (long long)peer_batch_stride);
  std::vector<moa::PeerOut> host(n_peers);
  for (int k = 0; k < n_peers; ++k) {
    if (!peer_o[k] || !peer_flags[k] || ((uintptr_t)peer_flags[k] & 3))
      return fail(MOA_ERR_INVALID_ARG, "peer %d: NULL or misaligned pointer", k);
    host[k].o = peer_o[k];
    host[k].flag = peer_flags[k];
  }
  cudaError_t e = cudaDeviceSynchronize();  // launches in flight may read the old table
  if (e == cudaSuccess && !ctx->d_peers) e = cudaMalloc(&ctx->d_peers, 16 * sizeof(moa::PeerOut));
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_peers, host.data(), n_peers * sizeof(moa::PeerOut), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "peer output table");
  ctx->n_peers = n_peers;
  ctx->peer_head0 = head0;
  ctx->peer_bs = peer_batch_stride;
  ctx->peer_ls = peer_layer_stride;
  return ok();
}

moa_status moa_wait_flag(const unsigned int *flag, unsigned int expected, moa_stream_t stream) {
  if (!flag || ((uintptr_t)flag & 3)) return fail(MOA_ERR_INVALID_ARG, "flag must be a 4-byte aligned device pointer");
  int e = moa::launch_wait_flag(flag, expected, stream);
  if (e) return cuda_fail((cudaError_t)e, "wait_flag launch");
  return ok();
}

moa_status moa_set_decode_split(moa_ctx *ctx, int chunk_rows) {
  if (!ctx) return fail(MOA_ERR_INVALID_ARG, "ctx is NULL");
  if (chunk_rows != 0 && (chunk_rows < 64 || chunk_rows > (1 << 20) || chunk_rows % 64))
    return fail(MOA_ERR_INVALID_ARG, "chunk_rows %d: 0 or a multiple of 64 in [64, 2^20]", chunk_rows);
  for (const auto &p : ctx->layers)
    if (p.rag_batch) return fail(MOA_ERR_STATE, "set the decode split before moa_set_ragged");
  ctx->dec_chunk = chunk_rows;
  ctx->ml_dirty = true;
  for (auto &p : ctx->layers) {
    if (!p.set) continue;
    p.dec_cps = 0;
    p.gc_off.assign(ctx->ngl + 1, 0);
    if (chunk_rows > 0)
      for (int g = 0; g < ctx->ngl; ++g) {
        p.gc_off[g] = p.dec_cps;
        p.dec_cps += (int)(((int64_t)p.n_sink + p.win_g[g] + chunk_rows - 1) / chunk_rows);
      }
    p.gc_off[ctx->ngl] = p.dec_cps;
    moa_status st = upload_tables(ctx, p);
    if (st) return st;
  }
  return ok();
}

moa_status moa_advance_pos(int64_t *pos, int batch, int64_t delta, moa_stream_t stream) {
  if (!pos || ((uintptr_t)pos & 7)) return fail(MOA_ERR_INVALID_ARG, "pos must be a non-NULL 8-byte aligned pointer");
  if (batch < 1) return fail(MOA_ERR_INVALID_ARG, "batch %d invalid", batch);
  int e = moa::launch_advance_pos(pos, batch, delta, stream);
  if (e) return cuda_fail((cudaError_t)e, "advance_pos launch");
  return ok();
}

// ---------------------------------------------------------------------------------------------
// introspection
// ---------------------------------------------------------------------------------------------

moa_status moa_get_window(const moa_ctx *ctx, int layer, int q_head_local, int32_t *window) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (!window || q_head_local < 0 || q_head_local >= ctx->nql) return fail(MOA_ERR_INVALID_ARG, "bad head/ptr");
  *window = ctx->layers[layer].win_q[q_head_local];
  return ok();
}

moa_status moa_get_group_window(const moa_ctx *ctx, int layer, int group_local, int32_t *w_g) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (!w_g || group_local < 0 || group_local >= ctx->ngl) return fail(MOA_ERR_INVALID_ARG, "bad group/ptr");
  *w_g = ctx->layers[layer].win_g[group_local];
  return ok();
}

moa_status moa_slot_of(const moa_ctx *ctx, int layer, int group_local, int64_t pos, int64_t *slot) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (!slot || group_local < 0 || group_local >= ctx->ngl || pos < 0)
    return fail(MOA_ERR_INVALID_ARG, "bad group/pos/ptr");
  const LayerPlan &p = ctx->layers[layer];
  *slot = moa::slot_of(pos, p.n_sink, p.win_g[group_local]);
  return ok();
}

moa_status moa_cache_region(const moa_ctx *ctx, int layer, int b, int group_local,
                            int64_t *row_offset, int64_t *rows) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (b < 0 || group_local < 0 || group_local >= ctx->ngl) return fail(MOA_ERR_INVALID_ARG, "bad b/group");
  const LayerPlan &p = ctx->layers[layer];
  if (row_offset) *row_offset = (int64_t)b * p.rows_per_seq + p.g_off[group_local];
  if (rows) *rows = (int64_t)p.n_sink + p.win_g[group_local];
  return ok();
}

moa_status moa_prefill_tiles(const moa_ctx *ctx, int layer, int q_head_local, int q_tile,
                             int32_t *tiles, uint8_t *edge, int max_tiles, int32_t *n_tiles) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  const LayerPlan &p = ctx->layers[layer];
  int nqt = (int)((p.N + moa::kTile - 1) / moa::kTile);
  if (q_head_local < 0 || q_head_local >= ctx->nql || q_tile < 0 || q_tile >= nqt || !n_tiles)
    return fail(MOA_ERR_INVALID_ARG, "bad head/tile/ptr");
  int64_t i0 = (int64_t)q_tile * moa::kTile;
  int64_t i1 = std::min<int64_t>(p.N, i0 + moa::kTile) - 1;
  int W = p.win_q[q_head_local];
  moa::TileRanges r = moa::kv_tile_ranges(i0, i1, W, p.n_sink, p.bshift);
  int n = r.count();
  *n_tiles = n;
  for (int k2 = 0; k2 < n && k2 < max_tiles; ++k2) {
    int t = r.at(k2);
    if (tiles) tiles[k2] = t;
    if (edge) edge[k2] = moa::kv_tile_full(i0, i1, t, W, p.n_sink, p.bshift) ? 0 : 1;
  }
  return ok();
}

moa_status moa_attention_influence(const void *q, const void *k, const void *v, const void *dout, int batch,
                                   int64_t N, int num_q_heads, int num_kv_heads, int head_dim,
                                   int64_t q_row_stride, int64_t kv_row_stride, float scale, int block,
                                   float *e_blocks, int accumulate, moa_stream_t stream) {
  if (!q || !k || !v || !dout || !e_blocks) return fail(MOA_ERR_INVALID_ARG, "NULL pointer");
  if (batch < 1 || N < 1 || N > (int64_t(1) << 31)) return fail(MOA_ERR_INVALID_ARG, "bad batch / N");
  if (num_q_heads < 1 || num_kv_heads < 1 || num_q_heads % num_kv_heads)
    return fail(MOA_ERR_INVALID_ARG, "num_q_heads must be a positive multiple of num_kv_heads");
  if (head_dim != 64 && head_dim != 128) return fail(MOA_ERR_SHAPE, "head_dim %d not in {64, 128}", head_dim);
  if (block != 64) return fail(MOA_ERR_UNSUPPORTED, "block %d: only the paper's 64 is implemented", block);
  if (q_row_stride < (int64_t)num_q_heads * head_dim || kv_row_stride < (int64_t)num_kv_heads * head_dim)
    return fail(MOA_ERR_SHAPE, "row strides smaller than heads * head_dim");
  if (((uintptr_t)k & 15) || ((uintptr_t)v & 15) || ((uintptr_t)q & 15) || ((uintptr_t)dout & 15) ||
      (kv_row_stride * 2) % 16 || (q_row_stride * 2) % 16)
    return fail(MOA_ERR_INVALID_ARG, "q/k/v/dout and their row strides must be 16-byte aligned (TMA)");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(MOA_ERR_INVALID_ARG, "scale must be finite > 0");
  moa::InfluenceArgs a{};
  a.q = q; a.k = k; a.v = v; a.dout = dout;
  a.q_row_stride = q_row_stride; a.kv_row_stride = kv_row_stride;
  a.batch = batch; a.N = N; a.nql = num_q_heads; a.G = num_q_heads / num_kv_heads; a.d = head_dim;
  a.scale = scale; a.e_blocks = e_blocks; a.accumulate = accumulate ? 1 : 0;
  static const bool legacy = [] {  // diagnostics: MOA_INF_LEGACY=1 runs the round-1 mma.sync kernel (A/B)
    const char *s = std::getenv("MOA_INF_LEGACY");
    return s && s[0] == '1';
  }();
  int e = legacy ? moa::launch_influence(a, stream) : moa::launch_influence_tc(a, stream);
  if (e) return cuda_fail((cudaError_t)e, "influence launch");
  return ok();
}

moa_status moa_rule_losses(const float *e_blocks, int heads, int64_t N, int block, int n_sink,
                           const float *alpha, const float *beta, int n_rules, float *loss_out,
                           moa_stream_t stream) {
  if (!e_blocks || !alpha || !beta || !loss_out) return fail(MOA_ERR_INVALID_ARG, "NULL pointer");
  if (heads < 1 || N < 1 || N > (int64_t(1) << 31)) return fail(MOA_ERR_INVALID_ARG, "bad heads / N");
  if (block != 64) return fail(MOA_ERR_UNSUPPORTED, "block %d: only the paper's 64 is implemented", block);
  if (n_sink < 0 || n_sink % block) return fail(MOA_ERR_INVALID_ARG, "n_sink %d not a multiple of block", n_sink);
  if (n_rules < 1 || n_rules > moa::kMaxRules)
    return fail(MOA_ERR_INVALID_ARG, "n_rules %d not in [1, %d]", n_rules, moa::kMaxRules);
  moa::RuleWindows win{};
  for (int r = 0; r < n_rules; ++r) {
    double sp = std::ceil((double)alpha[r] + (double)beta[r] * (double)N);
    if (!(sp == sp)) return fail(MOA_ERR_INVALID_ARG, "NaN rule %d", r);
    sp = std::min(std::max(sp, 0.0), (double)N);
    int64_t span = ((int64_t)sp + block - 1) / block * block;
    int64_t w = std::max<int64_t>(0, span - n_sink);
    win.blocks[r] = (int32_t)(w / block);
  }
  int e = moa::launch_rule_losses(e_blocks, heads, N, block, win, n_sink / block, n_rules, loss_out, stream);
  if (e) return cuda_fail((cudaError_t)e, "rule loss launch");
  return ok();
}

// ---- rule selection (Eq. 5 / eq:mip): exact.
// A plan picks one rule per head; a layer uses at most k <= 2 distinct rules.
// Layer options: for a rule pair (a, b) with density[a] < density[b], the best plan that puts
// m of the layer's heads on b moves the m heads with the largest loss[h][a] - loss[h][b]
// (exchange argument: any other m-subset has the same density and no lower loss); single
// rules and equal-density pairs give one point each.  Each layer's options are reduced to
// their Pareto frontier (density ascending, loss strictly descending); the frontier of the
// whole model is the Pareto merge of the layer frontiers (multiple-choice knapsack, exact:
// a sum of points is Pareto-optimal only if every summand is).  Partial sums are pruned when
// they cannot fit the budget with the sparsest options of the remaining layers, or cannot
// beat a feasible incumbent with the remaining layers' minimal losses (admissible bounds).
// Feasibility: sum_h density <= budget * H + 1e-9 (the oracle uses the same slack).
namespace {

struct LPoint {
  double dens, loss;
  int a, b, m;  // rule a for the heads not moved, rule b for the m moved heads (b = -1: none)
};

std::vector<LPoint> layer_frontier(const float *L, const float *density, int hpl, int R, int k) {
  std::vector<LPoint> pts;
  std::vector<double> base(R, 0.0);
  for (int r = 0; r < R; ++r) {
    double c = 0.0;
    for (int h = 0; h < hpl; ++h) c += L[(size_t)h * R + r];
    base[r] = c;
    pts.push_back({(double)density[r] * hpl, c, r, -1, 0});
  }
  if (k >= 2) {
    std::vector<double> gain(hpl);
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b) {
        if (a == b) continue;
        if (density[a] > density[b] || (density[a] == density[b] && a > b)) continue;
        for (int h = 0; h < hpl; ++h) gain[h] = (double)L[(size_t)h * R + a] - (double)L[(size_t)h * R + b];
        std::vector<int> ord(hpl);
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return gain[x] > gain[y]; });
        double loss = base[a];
        for (int m = 1; m < hpl; ++m) {
          loss -= gain[ord[m - 1]];
          pts.push_back({(double)density[a] * (hpl - m) + (double)density[b] * m, loss, a, b, m});
        }
      }
  }
  std::stable_sort(pts.begin(), pts.end(), [](const LPoint &x, const LPoint &y) {
    return x.dens < y.dens || (x.dens == y.dens && x.loss < y.loss);
  });
  std::vector<LPoint> f;
  for (const LPoint &q : pts)
    if (f.empty() || q.loss < f.back().loss) f.push_back(q);
  return f;
}

void layer_assign(const LPoint &q, const float *L, int hpl, int R, int32_t *choice) {
  for (int h = 0; h < hpl; ++h) choice[h] = q.a;
  if (q.b < 0 || q.m == 0) return;
  std::vector<double> gain(hpl);
  for (int h = 0; h < hpl; ++h) gain[h] = (double)L[(size_t)h * R + q.a] - (double)L[(size_t)h * R + q.b];
  std::vector<int> ord(hpl);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return gain[x] > gain[y]; });
  for (int m = 0; m < q.m; ++m) choice[ord[m]] = q.b;
}

struct FPoint {
  double dens, loss;
  int prev, opt;  // index into the previous frontier, option of this layer
};

}  // namespace

moa_status moa_plan_rules(const float *loss, const float *density, int layers, int heads_per_layer, int n_rules,
                          float density_budget, int max_rules_per_layer, int32_t *rule_out, float *loss_out,
                          float *density_out) {
  if (!loss || !density || !rule_out) return fail(MOA_ERR_INVALID_ARG, "NULL pointer");
  if (layers < 1 || heads_per_layer < 1 || n_rules < 1) return fail(MOA_ERR_INVALID_ARG, "empty instance");
  if (max_rules_per_layer != 1 && max_rules_per_layer != 2)
    return fail(MOA_ERR_UNSUPPORTED, "max_rules_per_layer %d: 1 or 2 (the paper's limit, PAPER.md:384)",
                max_rules_per_layer);
  for (int r = 0; r < n_rules; ++r)
    if (!(density[r] >= 0.f && density[r] <= 1.f)) return fail(MOA_ERR_INVALID_ARG, "density[%d] not in [0,1]", r);
  for (size_t i = 0; i < (size_t)layers * heads_per_layer * n_rules; ++i)
    if (!std::isfinite(loss[i])) return fail(MOA_ERR_INVALID_ARG, "loss[%zu] is not finite", i);
  const int hpl = heads_per_layer, R = n_rules, k = max_rules_per_layer;
  const double H = (double)layers * hpl;
  const double cap = (double)density_budget * H + 1e-9;
  std::vector<std::vector<LPoint>> lf(layers);
  for (int l = 0; l < layers; ++l) lf[l] = layer_frontier(loss + (size_t)l * hpl * R, density, hpl, R, k);
  // suffix bounds: sparsest density and smallest loss of the layers after l
  std::vector<double> min_d(layers + 1, 0.0), min_l(layers + 1, 0.0);
  for (int l = layers - 1; l >= 0; --l) {
    double md = INFINITY, ml = INFINITY;
    for (const LPoint &q : lf[l]) md = std::min(md, q.dens), ml = std::min(ml, q.loss);
    min_d[l] = min_d[l + 1] + md;
    min_l[l] = min_l[l + 1] + ml;
  }
  if (min_d[0] > cap)
    return fail(MOA_ERR_INVALID_ARG, "infeasible: the sparsest plan has mean density %.6f > budget %.6f",
                min_d[0] / H, (double)density_budget);
  // feasible incumbent for the loss bound: the best Lagrangian plan (each layer minimises
  // loss + lam * density over its frontier) that fits, over a bisection of the price lam
  double incumbent = 0.0;
  for (int l = 0; l < layers; ++l) incumbent += lf[l].front().loss;  // all-sparsest: feasible
  {
    auto plan_at = [&](double lam, double &dsum) {
      double lsum = 0.0;
      dsum = 0.0;
      for (int l = 0; l < layers; ++l) {
        const LPoint *b = &lf[l][0];
        for (const LPoint &q : lf[l])
          if (q.loss + lam * q.dens < b->loss + lam * b->dens) b = &q;
        lsum += b->loss;
        dsum += b->dens;
      }
      return lsum;
    };
    double lo = 0.0, hi = 1.0, dsum = 0.0;
    double l0 = plan_at(0.0, dsum);
    if (dsum <= cap) {
      incumbent = std::min(incumbent, l0);
    } else {
      for (int it = 0; it < 200; ++it) {
        plan_at(hi, dsum);
        if (dsum <= cap) break;
        lo = hi;
        hi *= 2.0;
      }
      for (int it = 0; it < 100; ++it) {
        const double mid = 0.5 * (lo + hi);
        const double lm = plan_at(mid, dsum);
        if (dsum <= cap) {
          incumbent = std::min(incumbent, lm);
          hi = mid;
        } else {
          lo = mid;
        }
      }
      const double lh = plan_at(hi, dsum);
      if (dsum <= cap) incumbent = std::min(incumbent, lh);
    }
  }
  std::vector<std::vector<FPoint>> fr(layers + 1);
  fr[0].push_back({0.0, 0.0, -1, -1});
  const size_t kMaxFrontier = (size_t)1 << 24;
  std::vector<FPoint> cand;
  for (int l = 0; l < layers; ++l) {
    cand.clear();
    const double dcap = cap - min_d[l + 1];
    const double lcap = incumbent - min_l[l + 1] + 1e-9 * (1.0 + std::fabs(incumbent));
    const auto &F = fr[l];
    for (int i = 0; i < (int)F.size(); ++i)
      for (int j = 0; j < (int)lf[l].size(); ++j) {
        const double d = F[i].dens + lf[l][j].dens;
        if (d > dcap) break;  // layer options are sorted by density
        const double c = F[i].loss + lf[l][j].loss;
        if (c > lcap) continue;
        cand.push_back({d, c, i, j});
      }
    std::sort(cand.begin(), cand.end(), [](const FPoint &x, const FPoint &y) {
      return x.dens < y.dens || (x.dens == y.dens && x.loss < y.loss);
    });
    auto &NF = fr[l + 1];
    for (const FPoint &q : cand)
      if (NF.empty() || q.loss < NF.back().loss) NF.push_back(q);
    if (NF.size() > kMaxFrontier)
      return fail(MOA_ERR_UNSUPPORTED, "exact rule selection: Pareto frontier of %zu partial plans at layer %d "
                  "exceeds the solver's limit", NF.size(), l);
    if (NF.empty()) return fail(MOA_ERR_INVALID_ARG, "infeasible density budget");
  }
  // the optimum: the last (lowest-loss) point of the final frontier
  const auto &FN = fr[layers];
  int idx = (int)FN.size() - 1;
  const double best_loss = FN[idx].loss, best_dens = FN[idx].dens;
  for (int l = layers; l >= 1; --l) {
    const FPoint &q = fr[l][idx];
    layer_assign(lf[l - 1][q.opt], loss + (size_t)(l - 1) * hpl * R, hpl, R, rule_out + (size_t)(l - 1) * hpl);
    idx = q.prev;
  }
  if (loss_out) *loss_out = (float)best_loss;
  if (density_out) *density_out = (float)(best_dens / H);
  return ok();
}

moa_status moa_prefill_items(const moa_ctx *ctx, int layer, int32_t *items, int max_items,
                             int32_t *n_items) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (!n_items) return fail(MOA_ERR_INVALID_ARG, "n_items is NULL");
  const LayerPlan &p = ctx->layers[layer];
  int n = (int)(p.items.size() / 2);
  *n_items = n;
  if (items)
    for (int i = 0; i < n && i < max_items; ++i) {
      items[2 * i] = p.items[2 * i];
      items[2 * i + 1] = p.items[2 * i + 1];
    }
  return ok();
}

moa_status moa_prefill_schedule(const moa_ctx *ctx, int layer, int32_t *entries, int max_entries,
                                int32_t *offsets, int max_ctas, int32_t *n_entries, int32_t *n_ctas) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (!n_entries || !n_ctas) return fail(MOA_ERR_INVALID_ARG, "n_entries / n_ctas is NULL");
  const LayerPlan &p = ctx->layers[layer];
  const int ne = (int)(p.sched2.size() / 2), nc = p.sched2_off.empty() ? 0 : (int)p.sched2_off.size() - 1;
  *n_entries = ne;
  *n_ctas = nc;
  if (entries)
    for (int i = 0; i < ne && i < max_entries; ++i) {
      entries[2 * i] = p.sched2[2 * i];
      entries[2 * i + 1] = p.sched2[2 * i + 1];
    }
  if (offsets)
    for (int c = 0; c <= nc && c <= max_ctas; ++c) offsets[c] = p.sched2_off[c];
  return ok();
}

moa_status moa_decode_chunks(const moa_ctx *ctx, int layer, int32_t *chunks, int max_chunks,
                             int32_t *n_chunks) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (!n_chunks) return fail(MOA_ERR_INVALID_ARG, "n_chunks is NULL");
  const LayerPlan &p = ctx->layers[layer];
  int n = (int)(p.chunks.size() / 3);
  *n_chunks = n;
  if (chunks)
    for (int i = 0; i < n && i < max_chunks; ++i)
      for (int j = 0; j < 3; ++j) chunks[3 * i + j] = p.chunks[3 * i + j];
  return ok();
}

moa_status moa_next_pos(const moa_ctx *ctx, int layer, int64_t *pos) {
  moa_status st = check_layer(ctx, layer, true);
  if (st) return st;
  if (!pos) return fail(MOA_ERR_INVALID_ARG, "pos is NULL");
  *pos = ctx->layers[layer].next_pos;
  return ok();
}

}  // extern "C"
