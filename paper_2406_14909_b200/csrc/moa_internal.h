// moa_internal.h -- host runtime structures and the index arithmetic shared by
// the host planner and the device kernels of libmoa.so (one product; the
// oracle shares nothing with it).
//
// Mask (PAPER.md:178 sinks; reading c3 window incl. the query itself):
//   key j visible to query i  <=>  0 <= j <= i  and  (j < s  or  i - j < W)
// Block mode (bshift = log2(block), -1 = token mode): the
// window of query i starts at the first key of block floor(i/b) - W/b + 1 instead of i-W+1
// (s and W multiples of b), so one helper gives the first window key for both modes.
// Ring slot of position p (reading c13):
//   p < s ? p : s + (p - s) mod W_g
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/moa.h"

#if defined(__CUDACC__)
#define MOA_HD __host__ __device__ __forceinline__
#else
#define MOA_HD inline
#endif

namespace moa {

constexpr int kTile = MOA_TILE;  // prefill q/kv tile (rows)

// ------------------------------------------------------------------------------------------
// Prefill block-skip schedule.  For q rows [i0, i1] (i1 inclusive, the last
// REAL row of the tile) of a head with window W and s sinks the visited kv tiles are
//   sink tiles   [0, ceil(min(s, i1+1) / T))
//   window tiles [floor(max(0, i0-W+1) / T), floor(i1 / T) + 1)    (empty if W == 0)
// merged into two disjoint ascending ranges [a0,a1) U [b0,b1).
// ------------------------------------------------------------------------------------------
MOA_HD int64_t win_lo(int64_t i, int W, int bshift) {
  return bshift < 0 ? i - W + 1 : (((i >> bshift) - (int64_t)(W >> bshift) + 1) << bshift);
}

struct TileRanges {
  int a0, a1, b0, b1;
  MOA_HD int count() const { return (a1 - a0) + (b1 - b0); }
  MOA_HD int at(int k) const { return k < (a1 - a0) ? a0 + k : b0 + (k - (a1 - a0)); }
};

MOA_HD TileRanges kv_tile_ranges(int64_t i0, int64_t i1, int W, int s, int bshift = -1) {
  TileRanges r;
  int64_t nsink_keys = s < i1 + 1 ? (int64_t)s : i1 + 1;
  r.a0 = 0;
  r.a1 = (int)((nsink_keys + kTile - 1) / kTile);
  if (W > 0) {
    int64_t lo = win_lo(i0, W, bshift);  // the window start is non-decreasing in i
    if (lo < 0) lo = 0;
    r.b0 = (int)(lo / kTile);
    r.b1 = (int)(i1 / kTile) + 1;
    if (r.b0 < r.a1) r.b0 = r.a1;
    if (r.b1 < r.b0) r.b1 = r.b0;
  } else {
    r.b0 = r.b1 = r.a1;
  }
  return r;
}

// A kv tile needs no mask iff every (row, key) pair of the tile is visible:
// all keys <= the first row (causal) and every non-sink key of the tile is
// inside the window of the last row (the farthest pair).
MOA_HD bool kv_tile_full(int64_t i0, int64_t i1, int t, int W, int s, int bshift = -1) {
  int64_t j0 = (int64_t)t * kTile, j1 = j0 + kTile - 1;
  if (j1 > i0) return false;
  int64_t jn = j0 > s ? j0 : (int64_t)s;  // first non-sink key of the tile
  return jn > j1 || (W > 0 && jn >= win_lo(i1, W, bshift));
}

MOA_HD bool tile_in(const TileRanges &r, int t) { return (t >= r.a0 && t < r.a1) || (t >= r.b0 && t < r.b1); }

// Two q tiles processed together (rows [i0, i0+128) and [i0+128, i0+256), the second
// present iff i0+128 < N): their visited kv tiles are walked once in ascending order,
// [0, u_a1) U [u_b0, u_b1), and each step is used by the q tiles whose own schedule
// contains it (tile_in).  A step neither tile uses is skipped by every role.
struct BlockTiles {
  TileRanges r[2];
  bool has1;
  int u_a1, u_b0, u_b1;
  MOA_HD int steps() const { return u_a1 + (u_b1 - u_b0); }
  MOA_HD int at(int k) const { return k < u_a1 ? k : u_b0 + (k - u_a1); }
};

MOA_HD BlockTiles kv_block_tiles(int64_t i0, int64_t N, int W, int s, int bshift = -1) {
  BlockTiles b;
  b.r[0] = kv_tile_ranges(i0, (i0 + kTile < N ? i0 + kTile : N) - 1, W, s, bshift);
  b.has1 = i0 + kTile < N;
  if (b.has1) {
    b.r[1] = kv_tile_ranges(i0 + kTile, (i0 + 2 * kTile < N ? i0 + 2 * kTile : N) - 1, W, s, bshift);
  } else {
    b.r[1].a0 = b.r[1].a1 = b.r[1].b0 = b.r[1].b1 = 0;
  }
  b.u_a1 = b.r[0].a1 > b.r[1].a1 ? b.r[0].a1 : b.r[1].a1;
  int lo = 1 << 30, hi = 0;
  for (int k = 0; k < 2; ++k)
    if (b.r[k].b1 > b.r[k].b0) {
      lo = b.r[k].b0 < lo ? b.r[k].b0 : lo;
      hi = b.r[k].b1 > hi ? b.r[k].b1 : hi;
    }
  b.u_b0 = lo > b.u_a1 ? lo : b.u_a1;
  b.u_b1 = hi > b.u_b0 ? hi : b.u_b0;
  return b;
}

// Ring arithmetic (reading c13).
MOA_HD int64_t slot_of(int64_t p, int s, int Wg) {
  if (p < s) return p;
  if (Wg <= 0) return -1;
  return s + (p - s) % Wg;
}

// Position held by row `r` of a group region after position p was written
// (-1 if the row holds nothing yet).  Sink rows hold r (if r <= p); ring row
// k = r - s holds q = p - ((p - s - k) mod W_g) if q >= s.
MOA_HD int64_t pos_of_row(int64_t r, int64_t p, int s, int Wg) {
  if (r < s) return r <= p ? r : -1;
  if (p < s) return -1;
  int64_t k = r - s;
  int64_t m = (p - s - k) % Wg;
  if (m < 0) m += Wg;
  int64_t q = p - m;
  return q >= s ? q : -1;
}

// ------------------------------------------------------------------------------------------
// Host runtime
// ------------------------------------------------------------------------------------------
struct LayerPlan {
  bool set = false;
  int n_sink = 0;
  int bshift = -1;               // prefill mask: -1 token-granular, else log2(block size)
  int64_t N = 0;
  std::vector<int32_t> win_q;    // local q-heads
  std::vector<int32_t> win_g;    // local groups: W_g
  std::vector<int64_t> g_off;    // row offset of group g inside one sequence's region
  int64_t rows_per_seq = 0;      // sum_g (s + W_g)
  std::vector<int32_t> items;    // prefill work items (h_local, q_tile): heads heaviest first, q tiles of a
                                 // head consecutive (L2 sharing of its K/V), heaviest first
  std::vector<int32_t> items2;   // prefill work items of two q tiles (h_local, q_block of 2*kTile rows), same order
  // the items2 x max_batch entries (h | b << 16, q_block) grouped by CTA: greedy list scheduling of
  // the LPT-ordered list over the SMs (each entry to the least-loaded CTA), CTA c runs entries
  // [sched2_off[c], sched2_off[c + 1]) -- the static round robin leaves the busiest SM 7-14 % above
  // the mean on C2 layers, greedy ~1 %
  std::vector<int32_t> sched2, sched2_off;
  int sched2_batch = 0;
  std::vector<int32_t> chunks;   // decode chunks: (g_local, row_begin, row_end) triples
  std::vector<int32_t> g_chunk;  // first chunk of each group, size ngl + 1
  int chunk_rows = 0;
  int max_chunks_per_group = 0;
  int dec_cps = 0;               // bf16 decode: rank-invariant chunks per sequence (ctx->dec_chunk rows each)
  std::vector<int32_t> gc_off;   // first rank-invariant chunk of each group in a sequence, size ngl + 1
  std::vector<int32_t> fill_h;   // [ngl] first local q-head with W_h = W_g (fused cache fill)
  const int32_t *d_gc_off = nullptr;
  // device copies of the tables (one allocation)
  void *d_tables = nullptr;
  const int32_t *d_win_q = nullptr;
  const int32_t *d_win_g = nullptr;
  const int64_t *d_g_off = nullptr;
  const int32_t *d_items = nullptr;
  const int32_t *d_items2 = nullptr;
  const int32_t *d_sched2 = nullptr, *d_sched2_off = nullptr;
  const int32_t *d_chunks = nullptr;
  const int32_t *d_g_chunk = nullptr;
  const int32_t *d_fill_h = nullptr;  // [ngl] local q-head of the group whose last q block fills the cache
  int *d_counters = nullptr;     // [max_batch, ngl] decode combine tickets (zeroed at upload)
  // ragged batch (moa_set_ragged): per-sequence prompt length N_b and windows W_{b,h}
  int rag_batch = 0;             // 0 = uniform batch
  std::vector<int64_t> rag_n;    // [rag_batch]
  std::vector<int32_t> rag_win;  // [rag_batch, nql] local heads
  std::vector<int32_t> rag_items2;  // two-tile prefill items of the ragged batch (h | b << 16, q_block)
  void *d_rag = nullptr;
  const int32_t *d_rag_items2 = nullptr;
  const int32_t *d_rag_sched2 = nullptr, *d_rag_sched2_off = nullptr;  // per-CTA greedy schedule of rag_items2
  int rag_sched2_ctas = 0;
  const int64_t *d_seq_n = nullptr;
  const int32_t *d_win_bq = nullptr;
  // TMA tensor maps (CUtensorMap, 128 B) over the bound K / V cache of this layer:
  // 2D [bound_batch * rows_per_seq rows, d], 64-row x 64-col boxes, 128B swizzle
  alignas(64) unsigned char kmap[128] = {};    // 64-row boxes
  alignas(64) unsigned char vmap[128] = {};
  alignas(64) unsigned char kmap16[128] = {};  // 16-row boxes (tile tails)
  alignas(64) unsigned char vmap16[128] = {};
  alignas(64) unsigned char kmap1[128] = {};   // 1-row boxes (prefill's fused cache fill)
  alignas(64) unsigned char vmap1[128] = {};
  bool maps_ok = false;
  // bound cache
  void *k_cache = nullptr;
  void *v_cache = nullptr;
  int bound_batch = 0;
  int64_t next_pos = -1;  // next position to append; -1 = nothing written
};

}  // namespace moa

struct moa_ctx {
  int device = -1;
  int num_sms = 148;  // SM count of `device` (planning-only contexts: a B200's)
  moa_dtype dtype = MOA_BF16;
  int L = 0, Hq = 0, Hkv = 0, G = 1, d = 128, max_batch = 1;
  int g0 = 0, g1 = 0, ngl = 0, nql = 0;  // local groups [g0, g1), counts
  std::vector<moa::LayerPlan> layers;
  // layer whose cache the most recent launch of this context wrote: -1 none, kAllLayers unknown
  // (after a bind); lets a decode launch stream its cache before its stream predecessor ends
  static constexpr int kAllLayers = -2;
  int last_cache_write = kAllLayers;
  // bf16 decode split: rows per rank-invariant chunk (0: balanced row split, not rank-invariant)
  int dec_chunk = 0;
  // cross-layer decode: device image of DecodeLayerDesc[L] + 4 tensor maps per layer
  // (moa_prepare_layers); stale after set_spans / bind / set_decode_split / set_ragged
  void *d_ml = nullptr;
  std::vector<unsigned char> ml_image;
  bool ml_dirty = true;
  // fused head-output all-gather (moa_set_peer_outputs)
  void *d_peers = nullptr;
  int n_peers = 0, peer_head0 = 0;
  int64_t peer_bs = 0, peer_ls = 0;
};

namespace moa {

// ---- launchers (kernels/*.cu); all return cudaError_t as int ----------------------------
struct PrefillArgs {
  const void *q, *k, *v;
  void *o;
  int64_t q_row_stride, kv_row_stride, o_row_stride;
  int batch;
  int64_t N;
  float scale;
  float *lse;
  int n_sink;
  int nql, G, d;
  const int32_t *d_win_q;
  const int32_t *d_items;
  int n_items;
  const int32_t *d_items2;  // (h_local, q_block) pairs of the two-tile kernel
  int n_items2;
  const int32_t *d_sched2, *d_sched2_off;  // per-CTA schedule of (h | b << 16, q_block) (null: round robin)
  int sched2_ctas;
  int bshift;               // -1 token mask, else log2(block size) (block mode)
  const int64_t *d_seq_n;   // ragged: per-sequence N_b [batch] (null: every sequence has N)
  const int32_t *d_win_bq;  // ragged: per-sequence windows [batch, nql] (null: d_win_q)
  const int32_t *d_items_rag;  // ragged two-tile items (h | b << 16, q_block), real items only, LPT
  int n_items_rag;
  // fused cache fill (bf16 token-mask uniform prefill): write the kept rows from the K/V tiles
  int fill;
  void *k_cache, *v_cache;
  int64_t rows_per_seq;
  const int64_t *d_g_off;
  const int32_t *d_win_g, *d_fill_h;
  const void *kmap16, *vmap16, *kmap1, *vmap1;  // cache tensor maps (16-row / 1-row boxes)
};
int launch_prefill_f32(const PrefillArgs &a, void *stream);
int launch_prefill_bf16_pp(const PrefillArgs &a, void *stream);

struct CacheArgs {
  const void *k, *v;  // prompt K/V (fill) or new token (append)
  int64_t row_stride; // fill: token row stride; append: batch stride
  void *k_cache, *v_cache;
  int64_t rows_per_seq;
  const int64_t *d_g_off;
  const int32_t *d_win_g;
  int ngl, d, n_sink, batch;
  int64_t N_or_pos;
  int esize;
  int64_t max_region_rows;  // n_sink + max_g W_g
  const int64_t *d_seq_n;   // fill, ragged: per-sequence N_b (null: N_or_pos)
  const int64_t *d_pos;     // append, ragged: per-sequence positions (null: N_or_pos)
};
int launch_cache_fill(const CacheArgs &a, void *stream);
int launch_kv_append(const CacheArgs &a, void *stream);
int launch_advance_pos(int64_t *pos, int batch, int64_t delta, void *stream);

struct DecodeArgs {
  const void *q;
  void *o;
  int64_t q_batch_stride, o_batch_stride;
  const void *k_new, *v_new;  // fused append (nullable)
  int64_t kv_batch_stride;
  const void *k_cache, *v_cache;
  int64_t rows_per_seq;
  const int64_t *d_g_off;
  const int32_t *d_win_g, *d_win_q;
  const int32_t *d_chunks, *d_g_chunk;
  int n_chunks, max_chunks_per_group;
  int ngl, G, d, n_sink, batch;
  int64_t pos;
  const int64_t *d_pos;     // ragged: per-sequence positions [batch] (null: pos); < 0 = inactive
  const int32_t *d_win_bq;  // ragged: per-sequence windows [batch, nql] (null: d_win_q)
  float scale;
  float *lse;
  float *ws_part;       // [batch, n_chunks, G, d + 1] split partials (o, lse2)
  int *counters;        // [max_batch, ngl] last-CTA-done tickets (library-owned, self-resetting)
};
int launch_decode(const DecodeArgs &a, moa_dtype dtype, bool fused, void *stream);

size_t decode_ws_bytes(int batch, int n_chunks, int G, int d);

// bf16 decode on mma.sync with TMA-staged swizzled cache tiles (decode_mma.cu)
struct DecodeMmaArgs {
  const void *kmap, *vmap;     // host CUtensorMap images, 64-row boxes
  const void *kmap16, *vmap16; // 16-row boxes for the partial last tile of a segment
  const void *q;
  void *o;
  int64_t q_bs, o_bs;
  const void *k_new, *v_new;   // fused append (nullable)
  int64_t kv_bs;
  void *k_cache, *v_cache;     // for the fused append's global write
  int64_t rows_per_seq;
  const int64_t *d_g_off;
  const int32_t *d_win_g, *d_win_q;
  int ngl, G, d, n_sink, batch;
  int64_t pos;
  const int64_t *d_pos;        // ragged: per-sequence positions [batch] (null: pos); < 0 = inactive
  const int32_t *d_win_bq;     // ragged: per-sequence windows [batch, nql] (null: d_win_q)
  float scale;
  float *lse;
  float *ws_part;
  int *counters;
  int early_read;              // see decode_common: predecessor does not write this layer's cache
  int chunk;                   // rank-invariant split: rows per chunk (0: balanced row split)
  int chunks_per_seq;          // sum_g ceil((s + W_g) / chunk)
  const int32_t *d_gc_off;     // first chunk of each local group inside a sequence [ngl + 1]
  // fused head-output all-gather (moa_set_peer_outputs): n_peers destinations (device array)
  const void *peers;
  int n_peers, peer_head0, layer;
  int64_t peer_bs, peer_ls;
};
struct PeerOut {
  void *o;             // destination [L?][B][Hq_total][d] bf16 (peer-mapped device address)
  unsigned *flag;      // destination's per-layer arrival counters [L]
};
int launch_decode_mma(const DecodeMmaArgs &a, void *stream);
int launch_wait_flag(const unsigned *flag, unsigned expected, void *stream);

// Cross-layer decode (moa_decode_step_fused_layers): one launch streams
// the caches of n consecutive layers.  The per-layer static data lives in a device array of
// these (ctx->d_ml, rebuilt by moa_prepare_layers); the per-call data (q/o/k_new/v_new bases
// and layer strides, pos, scale) comes with the launch.
struct DecodeLayerDesc {
  const void *maps;              // 4 CUtensorMap (kmap, vmap, kmap16, vmap16), device copies
  void *kc, *vc;                 // the layer's cache
  const int64_t *g_off;
  const int32_t *win_g, *win_q, *gc_off;
  int *counters;
  int64_t rows_per_seq;
  int dec_cps;
  int pad_;
};
struct DecodeLayersArgs {
  DecodeMmaArgs a;               // layer 0 of the range (tables/maps ignored) + per-call fields
  const DecodeLayerDesc *d_layers;  // [n] (device), already offset to the first layer
  int n_layers;
  int64_t q_ls, o_ls, kvn_ls, lse_ls, part_ls;  // layer strides (elements; part in floats)
  int64_t max_rows;              // max over the layers of batch * rows_per_seq (grid size)
  int64_t min_rows;              // min over the layers (balanced split: no CTA may get an empty range)
};
int launch_decode_mma_layers(const DecodeLayersArgs &a, void *stream);
size_t decode_mma_ws_bytes(int batch, int ngl, int G, int d, int chunks_per_seq);

// attention influence of the profiling stage (kernels/influence.cu)
struct InfluenceArgs {
  const void *q, *k, *v, *dout;  // bf16 [B, N, Hq, d] (q, dout) / [B, N, Hkv, d] (k, v)
  int64_t q_row_stride, kv_row_stride;
  int batch;
  int64_t N;
  int nql, G, d;
  float scale;
  float *e_blocks;  // [B, Hq, nb, nb] fp32
  int accumulate;
};
int launch_influence(const InfluenceArgs &a, void *stream);     // mma.sync reference design (A/B only)
int launch_influence_tc(const InfluenceArgs &a, void *stream);  // tcgen05 + TMEM + TMA (the product)
// Eq. 4 rule losses: window of every rule in blocks (passed by value, <= kMaxRules rules)
constexpr int kMaxRules = 128;
struct RuleWindows {
  int32_t blocks[kMaxRules];
};
int launch_rule_losses(const float *e_blocks, int heads, int64_t N, int block, const RuleWindows &win,
                       int sink_blocks, int n_rules, float *loss, void *stream);

// SM count of the current device (cached per device ordinal).
int device_sm_count();
// TMA tensor map over a [rows, d] bf16 cache (box box_rows x 64 cols, 128B swizzle).
bool encode_cache_map(void *map_out, const void *ptr, int d, int64_t rows, int box_rows);
// TMA tensor map over [B, N, H, d] bf16 (token row stride in elements), 64-column x box_rows boxes.
bool make_tile_map(void *m, const void *ptr, int d, int H, int64_t N, int B, int64_t row_stride, int box_rows);

}  // namespace moa
