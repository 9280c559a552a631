// prefill_pp.cu -- MoA causal prefill on the sm_100a tensor cores, two q tiles per CTA
// ping-ponged on one tensor core (tcgen05 + TMEM + TMA), bf16 I/O, fp32 accumulation
// (SURVEY §8(a) a4).
//
//   O[b,i,h] = sum_{j in V(h,i)} softmax_j(tau q_i . k_j) v_j       (Eq. 1)
//   V(h,i)   = { j <= i : j < s  or  i - j < W_h }                   (reading c3)
//
// A work item is 256 query rows of one (batch, q-head): q tiles Q0 = rows [i0, i0+128) and
// Q1 = rows [i0+128, i0+256).  The kv tiles of both block-skip schedules are walked once
// (kv_block_tiles: sinks U window, ascending); each K/V tile is loaded once and used by the
// q tiles whose own schedule contains it.  FULL tiles skip the mask arithmetic.
//
// Warp roles (384 threads, one CTA per SM, persistent over a static slice of the LPT list):
//   warps 0-3  softmax of Q0 (thread t owns row t = TMEM lane t, all 128 S columns)
//   warps 4-7  softmax of Q1
//   warp 8     TMA producer of the K and V rings
//   warp 9     TMEM allocator + MMA issue for Q0 (whole warp waits, one elected lane issues)
//   warp 10    TMA producer of Q0 / Q1
//   warp 11    MMA issue for Q1 (takes turns with warp 9)
// setmaxnreg moves registers from warpgroup 2 (producers, MMA) to the softmax warpgroups.
// TMEM (512 columns): S0 | S1 (fp32 128x128; P_j, bf16 packed, overwrites the first 64
// columns of S_j once the softmax has it in registers) | O0 | O1 (fp32 128xD).
// Per kv step the MMA warps issue  PV0(prev), S0(next), PV1(prev), S1(next) in turns:  while the
// softmax of Q1 runs the tensor core computes Q0's products and vice versa, so the tensor
// pipe never waits for one softmax.  tcgen05 ops of one thread execute in issue order and a
// commit covers every earlier op, so S_j(t) complete implies PV_j(t-1) complete (O_j may be
// rescaled, P_j may be overwritten).  The running max is refreshed (and O rescaled in TMEM)
// only when it grows by more than 2^8.  Exponentials run on MUFU ex2 except one pair in four,
// which a degree-3 polynomial computes on the FMA pipe with packed f32x2 arithmetic.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "../moa_internal.h"
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace moa {
namespace {

using namespace ptx;

constexpr int kM = 128;    // q rows per tile (MMA M)
constexpr int kN = 128;    // keys per kv tile
constexpr int kThreads = 384;  // warp 11 idles (warpgroup-aligned register reallocation)
constexpr int kWarpKV = 8, kWarpMMA = 9, kWarpQ = 10, kWarpMMA1 = 11, kSoftmaxWarp0 = 0;
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
// setmaxnreg split: 8 softmax warps x MOA_PP_REG_SOFTMAX + 4 other warps x MOA_PP_REG_OTHER <= 64K
// 216 / 72 with the K 2 / V 3 ring: C2 +1.6 %, C4 +1.9 % over 208 / 88 with K 3 / V 2 (A/B after
// the greedy schedule; before it the two measured within noise)
#ifndef MOA_PP_REG_SOFTMAX
#define MOA_PP_REG_SOFTMAX 216
#endif
#ifndef MOA_PP_REG_OTHER
#define MOA_PP_REG_OTHER 72
#endif
static_assert((8 * MOA_PP_REG_SOFTMAX + 4 * MOA_PP_REG_OTHER) * 32 <= 65536, "setmaxnreg split exceeds the register file");
static_assert(MOA_PP_REG_SOFTMAX % 8 == 0 && MOA_PP_REG_OTHER % 8 == 0, "setmaxnreg counts must be multiples of 8");
static_assert(MOA_PP_REG_SOFTMAX >= 24 && MOA_PP_REG_SOFTMAX <= 256 && MOA_PP_REG_OTHER >= 24 &&
                  MOA_PP_REG_OTHER <= 256, "setmaxnreg counts must be in [24, 256]");
#ifndef MOA_PP_POLY_EVERY
#define MOA_PP_POLY_EVERY 4
#endif
constexpr int kPolyEvery = MOA_PP_POLY_EVERY;  // pair c uses the polynomial iff c % kPolyEvery == kPolyEvery - 1
// token mask: a q tile's softmax runs on its own 4 warps (full rows); block masks: all 8 softmax
// warps work on both tiles, half the columns each (softmax_split_role) -- the block mask's
// extra EDGE tiles made the 4-warp softmax the longer pole (+9 % on C4 with block 64)
template <int BS>
constexpr int softmax_warps_per_tile() { return BS >= 0 ? 8 : 4; }
constexpr int kBarPair0 = 4;  // named barriers 4..7: warps q and q + 4 (rows 32q..32q+31), split softmax

template <int D>
struct PCfg {
  static constexpr int kSlabs = D / 64;
  static constexpr int kTileBytes = kM * D * 2;
  static constexpr int kSlabBytes = kM * 128;
#ifndef MOA_PP_NK128
#define MOA_PP_NK128 2  // K ring stages at d = 128 (V gets 5 - NK); NK 4 (V 1) stalls
#endif
  static constexpr int kNK = D == 128 ? MOA_PP_NK128 : 6;
  static constexpr int kNV = D == 128 ? 5 - MOA_PP_NK128 : 4;
  static_assert(kNK >= 2 && kNV >= 2, "prefill K/V rings need two stages each");
  static constexpr int kSmemBytes = (2 + kNK + kNV) * kTileBytes;  // base 1024-aligned (see kernel)
  static constexpr uint32_t kColO0 = 256, kColO1 = 256 + D;
};

struct PpParams {
  void *o;
  float *lse;
  int64_t o_row_stride;
  int64_t N;
  int batch, n_items, nql, G, n_sink;
  float scale_log2;
  int bshift;            // -1 token mask, else log2(block size) (block mode)
  const int32_t *win_q;
  const int32_t *items;  // (q-head, q-block) pairs, LPT order; ragged: (h | b << 16, q-block)
  int o_v8;              // output rows 32-byte aligned: 256-bit stores in the epilogue
  const int64_t *seq_n;  // ragged: per-sequence N_b (null: N)
  const int32_t *win_bq; // ragged: per-sequence windows [batch, nql] (null: win_q)
  // fused cache fill (a5): the last q block of each group's filler head writes the cache rows
  // of the K/V tiles it streams anyway, from shared memory (warp 10)
  int fill;
  __nv_bfloat16 *kc, *vc;
  int64_t rows_per_seq;
  const int64_t *g_off;
  const int32_t *win_g;
  const int32_t *fill_h;  // [ngl] local q-head whose last q block fills the group (-1: none)
  // uniform batch: per-CTA schedule (CTA c runs entries [sched_off[c], sched_off[c+1]) of
  // (h | b << 16, q_block)); null: entry idx = blockIdx.x + k * gridDim.x of the item list x batch
  const int32_t *sched, *sched_off;
};

// the work entries of this CTA: [item_begin, item_end) in steps of item_step
__device__ __forceinline__ int item_begin(const PpParams &p) { return p.sched ? p.sched_off[blockIdx.x] : (int)blockIdx.x; }
__device__ __forceinline__ int item_end(const PpParams &p, int total) {
  return p.sched ? p.sched_off[blockIdx.x + 1] : total;
}
__device__ __forceinline__ int item_step(const PpParams &p) { return p.sched ? 1 : (int)gridDim.x; }

struct PBars {
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[6], k_empty[6];
  uint64_t v_full[4], v_empty[4];
  uint64_t s_full[2], p_full[2];
  uint64_t o_full[2], o_empty[2];
  uint64_t k_copied[6], v_copied[4];  // fused cache fill: warp 10's stores have read a filler tile
  uint64_t k_issued[6], v_issued[4];  // fused cache fill: the producer issued a filler tile's load
  uint32_t tmem_base;
};

// Mask mode as a template constant: BS = -1 token mask, 6 the paper's block of 64, kBsRuntime
// any other block size (p.bshift at run time); the common modes fold their arithmetic.
constexpr int kBsRuntime = 99;
template <int BS>
__device__ __forceinline__ int bshift_of(const PpParams &p) {
  return BS == kBsRuntime ? p.bshift : BS;
}

struct PItem {
  int b, h, W;
  int64_t i0, N;
  BlockTiles bt;
};

#ifndef MOA_PP_OST_HINT
#define MOA_PP_OST_HINT ".L1::no_allocate"  // O rows are never re-read here: C2 +2.5 %, C4 +1.8 % vs none
#endif
// 32 output columns of one row (this thread's), normalised and packed to bf16: two 256-bit
// stores (a full 32-byte sector per lane) when the output rows are 32-byte aligned, else
// four 128-bit ones; no L1 allocation (nothing here re-reads O).  Row-per-thread stores cost the softmax warps 8-13 % of the kernel.
__device__ __forceinline__ void store_o_chunk32(__nv_bfloat16 *dst, const float (&r)[32], float inv, int v8) {
  if (v8) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t w[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) w[e] = pack_bf16x2(r[16 * h + 2 * e] * inv, r[16 * h + 2 * e + 1] * inv);
      asm volatile("st.global" MOA_PP_OST_HINT ".v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + 16 * h), "r"(w[0]),
                   "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                   : "memory");
    }
  } else {
#pragma unroll
    for (int v4 = 0; v4 < 4; ++v4) {
      const uint32_t x = pack_bf16x2(r[8 * v4 + 0] * inv, r[8 * v4 + 1] * inv);
      const uint32_t y = pack_bf16x2(r[8 * v4 + 2] * inv, r[8 * v4 + 3] * inv);
      const uint32_t z = pack_bf16x2(r[8 * v4 + 4] * inv, r[8 * v4 + 5] * inv);
      const uint32_t w = pack_bf16x2(r[8 * v4 + 6] * inv, r[8 * v4 + 7] * inv);
      asm volatile("st.global" MOA_PP_OST_HINT ".v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 8 * v4), "r"(x), "r"(y),
                   "r"(z), "r"(w)
                   : "memory");
    }
  }
}

#ifndef MOA_PP_OSTORE
#define MOA_PP_OSTORE 1  // diagnostics: 0 skips the O / lse stores (epilogue cost study)
#endif
template <int BS, bool RAG>
__device__ __forceinline__ PItem get_pitem(const PpParams &p, int idx) {
  PItem it;
  if (RAG) {  // ragged list: (h | b << 16, q-block) of real items only, LPT order (or per-CTA schedule)
    const int32_t *src = p.sched ? p.sched : p.items;
    const int e = src[2 * idx];
    it.b = e >> 16;
    it.h = e & 0xffff;
    it.i0 = (int64_t)src[2 * idx + 1] * (2 * kM);
    // 32-bit index from the live (b, h): W stays cheap to re-derive (a 64-bit index or a W
    // carried in the item cost the softmax 45-100% through register spills)
    it.W = p.win_bq[it.b * p.nql + it.h];
  } else if (p.sched) {  // greedy per-CTA schedule: explicit (h | b << 16, q-block) entries
    const int e = p.sched[2 * idx];
    it.b = e >> 16;
    it.h = e & 0xffff;
    it.i0 = (int64_t)p.sched[2 * idx + 1] * (2 * kM);
  } else {
    const int wi = idx / p.batch;
    it.b = idx - wi * p.batch;
    it.h = p.items[2 * wi];
    it.i0 = (int64_t)p.items[2 * wi + 1] * (2 * kM);
  }
  // ragged: tiles are scheduled against the padded length (rows past N_b are computed on the
  // finite padding and not stored, see the epilogues), only the windows are per sequence
  it.N = p.N;
  if (!RAG) it.W = p.win_q[it.h];
  it.bt = kv_block_tiles(it.i0, it.N, it.W, p.n_sink, bshift_of<BS>(p));
  return it;
}


// Fused cache fill: the cache keeps positions [0, min(s, N)) and
// [max(s, N - W_g), N) of every (b, g) (reading c13).  Kv tile t is stored by
// the item of the group's filler head (the head with the largest window, W_h = W_g) whose q
// block holds rows [128 t, 128 t + 128): tile t is on that item's diagonal, so every item
// streams it anyway (causal; sink tiles are q block 0's diagonal), and the fill work spreads
// over the head's last q blocks instead of one item.  Warp 10 TMA-stores the kept rows from
// the tile in shared memory while the tensor core uses it.  Token mask, uniform batch only.
__device__ __forceinline__ bool fill_item(const PpParams &p, const PItem &it) {
  return p.fill && p.fill_h[it.h / p.G] == it.h;
}
// rows [r0, r1) of kv tile t that the cache keeps (r1 <= r0: none)
__device__ __forceinline__ void fill_rows(const PpParams &p, int64_t N, int Wg, int t, int &r0, int &r1, int &q0,
                                          int &q1) {
  const int64_t j0 = (int64_t)t * kN;
  const int64_t s = p.n_sink;
  const int64_t sink_end = s < N ? s : N;
  const int64_t ring_lo = (N - Wg) > s ? (N - Wg) : s;
  // two ranges: sinks [0, sink_end) and ring [ring_lo, N), clipped to the tile
  int64_t a0 = j0, a1 = j0 + kN < sink_end ? j0 + kN : sink_end;
  int64_t b0 = j0 > ring_lo ? j0 : ring_lo, b1 = j0 + kN < N ? j0 + kN : N;
  r0 = (int)(a0 - j0);
  r1 = (int)(a1 - j0);
  q0 = (int)(b0 - j0);
  q1 = (int)(b1 - j0);
}
// tile t of a filler item is stored by it iff it is one of the item's diagonal tiles
// (t >= i0 / 128) and holds kept rows
__device__ __forceinline__ bool fill_tile(const PpParams &p, int64_t i0, int64_t N, int Wg, int t) {
  if ((int64_t)t * kN < i0) return false;
  int r0, r1, q0, q1;
  fill_rows(p, N, Wg, t, r0, r1, q0, q1);
  return r1 > r0 || q1 > q0;
}
#ifndef MOA_PP_FILL_STORES
#define MOA_PP_FILL_STORES 1  // diagnostics: 0 keeps the fill protocol but issues no stores
#endif
// TMA stores of the kept rows of one K or V tile (two 64-column 128B-swizzled slabs in shared
// memory) into the layer cache: the rows of a tile map to runs of consecutive ring slots (a run
// ends where the ring wraps), each run goes out as 16-row boxes where the tile row is 16-aligned
// and 1-row boxes at its ends; the TMA engine un-swizzles (one thread issues, no registers).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *m, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
template <int D>
__device__ __forceinline__ void fill_store(const PpParams &p, uint32_t tile, const CUtensorMap *m16,
                                           const CUtensorMap *m1, int64_t region, int64_t N, int Wg, int t) {
  constexpr int kSlabs = D / 64;
  constexpr int kSlabBytes = kM * 128;
  int r0, r1, q0, q1;
  fill_rows(p, N, Wg, t, r0, r1, q0, q1);
  const int64_t j0 = (int64_t)t * kN;
  const int s = p.n_sink;
  for (int rr = 0; rr < 2; ++rr) {
    int r = rr ? q0 : r0;
    const int hi = rr ? q1 : r1;
    while (r < hi) {
      const int64_t pos = j0 + r;
      const int64_t slot = pos < s ? pos : s + (pos - s) % Wg;
      int n = hi - r;
      if (pos >= s && s + Wg - slot < n) n = (int)(s + Wg - slot);
      int cr = (int)(region + slot);
      while (MOA_PP_FILL_STORES && n > 0) {
        const bool box16 = (r & 15) == 0 && n >= 16;
        for (int sl = 0; sl < kSlabs; ++sl)
          tma_store_2d(box16 ? m16 : m1, tile + sl * kSlabBytes + r * 128, sl * 64, cr);
        const int st = box16 ? 16 : 1;
        r += st;
        cr += st;
        n -= st;
      }
    }
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// bits e of a 32-column word with e <= k (k < 0: none, k >= 31: all)
__device__ __forceinline__ uint32_t bits_le(int k) {
  return k >= 31 ? 0xffffffffu : (k < 0 ? 0u : (2u << k) - 1u);
}
#ifndef MOA_PP_MASK_BITS
#define MOA_PP_MASK_BITS 1
#endif
#ifndef MOA_PP_LATE_SUM
#define MOA_PP_LATE_SUM 0  // 1: row sum of the bf16 P after the p_full hand-over
#endif
#ifndef MOA_PP_ROLL
#define MOA_PP_ROLL 1  // 1: rescale and epilogue loops not unrolled (code size study)
#endif
constexpr int kUnrollRescale = MOA_PP_ROLL ? 1 : 4, kUnrollEpi = MOA_PP_ROLL ? 1 : 2;

// which q tiles use union step k (tile t); false/false = skipped by every role
__device__ __forceinline__ void step_use(const BlockTiles &bt, int k, int &t, bool &u0, bool &u1) {
  t = bt.at(k);
  u0 = tile_in(bt.r[0], t);
  u1 = bt.has1 && tile_in(bt.r[1], t);
}

__device__ __forceinline__ void tmem_ld32_f(uint32_t taddr, float *x) {
  tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(x));
}

// ------------------------------------------------------------------------------------------
// MMA issue: warp 9 issues Q0's MMAs, warp 11 Q1's, taking turns.  Dispatch of a tcgen05.mma
// is nearly synchronous for the issuing thread (~50-90 cycles per 128x128x16 MMA;
// profiles/r01_microbench.txt), so with one issuing warp every barrier wait, commit and
// loop instruction between dispatches is idle tensor time.  With two warps, warp j does its
// waits (K(t), V(t-1), P_j, O_j drained) and bookkeeping while the other warp dispatches,
// then takes the turn and dispatches [PV_j(t-1)] [S_j(t)] and hands the turn over (named
// barriers 2 and 3 between the two warps: a bar.arrive / bar.sync pair per hand-over).
// The strict alternation keeps the single-issuer order PV0, S0, PV1, S1 per step (the two
// tiles ping-pong), and each tile's MMAs come from one thread, so S_j(t) complete =>
// PV_j(t-1) complete (in-order tcgen05 execution + commits covering all earlier ops of the
// thread).  K/V slots are released by one commit from each warp (barrier count 2); a warp
// that does not use a step commits anyway (its commit only tracks its own MMAs).  Both warps
// walk the same item and step sequence: one turn per used step plus one per item.
// ------------------------------------------------------------------------------------------
constexpr int kBarTurn0 = 2;  // named barriers: kBarTurn0 + j = "warp of tile j may dispatch"

// diagnostic build (-DMOA_PP_DIAG_TRACE, tools/trace_pp.py): (tag, clock64) events of CTA 0
#ifdef MOA_PP_DIAG_TRACE
#define pp_tr_arg (trn_arg_)
__device__ unsigned long long g_pp_trace[4][4096];
__device__ int g_pp_trace_n[4];
#define PPTR(role, tag) PPTR_CTA(0, role, tag)
#define PPTR_CTA(cta, role, tag)                                                                 \
  if (blockIdx.x == (cta) && (threadIdx.x & 31) == 0) {                                          \
    if (trn_ < 4096) g_pp_trace[role][trn_] = ((unsigned long long)(tag) << 56) | ((unsigned long long)(pp_tr_arg & 0xff) << 48) | ((unsigned long long)clock64() & 0xffffffffffffull); \
    ++trn_;                                                                                      \
    g_pp_trace_n[role] = trn_ < 4096 ? trn_ : 4096;                                              \
  }
#else
#define PPTR(role, tag) {}
#define PPTR_CTA(cta, role, tag) {}
#endif

template <int D, int BS, bool RAG>
__device__ __forceinline__ void mma_role(const PpParams &p, PBars &bars, uint32_t tmem, uint32_t q_smem,
                                         uint32_t k_smem, uint32_t v_smem, int total, int j) {
  using C = PCfg<D>;
  constexpr uint32_t idesc_s = idesc_bf16_f32(kM, kN, false);
  constexpr uint32_t idesc_o = idesc_bf16_f32(kM, D, true);
  const uint64_t adesc = smem_desc_sw128(q_smem + j * C::kTileBytes, 16, 1024);
  const uint64_t kdesc0 = smem_desc_sw128(k_smem, 16, 1024);
  const uint64_t vdesc0 = smem_desc_sw128(v_smem, C::kSlabBytes, 1024);
  const uint32_t scol = tmem + (j ? 128u : 0u);  // S_j; P_j in its first 64 columns
  const uint32_t ocol = tmem + (j ? C::kColO1 : C::kColO0);
  int ks = 0, vs = 0;  // K / V ring stage of the current step
  uint32_t kph = 0, vph = 0, pph = 0, qph = 0, oph = 0;
  bool ostarted = false;
  bool wait_turn = j == 1;  // warp 9 (Q0) dispatches first
  int trn_ = 0, trn_arg_ = 0;
  (void)trn_;
  (void)trn_arg_;
  auto take_turn = [&]() {
    PPTR(j ? 3 : 0, 1)
    if (wait_turn) asm volatile("bar.sync %0, 64;" ::"r"(kBarTurn0 + j) : "memory");
    wait_turn = true;
    PPTR(j ? 3 : 0, 2)
  };
  auto pass_turn = [&]() {
    PPTR(j ? 3 : 0, 3)
    asm volatile("bar.arrive %0, 64;" ::"r"(kBarTurn0 + (j ^ 1)) : "memory");
  };
  for (int idx = item_begin(p), idx_end = item_end(p, total); idx < idx_end; idx += item_step(p)) {
    const PItem it = get_pitem<BS, RAG>(p, idx);
    const bool mine = j == 0 || it.bt.has1;  // this q tile has rows in the item
    const TileRanges r = j ? it.bt.r[1] : it.bt.r[0];
    const int last_t = r.b1 > r.b0 ? r.b1 - 1 : r.a1 - 1;  // its S releases Q_j, its PV completes O_j
    if (mine) {
      mbar_wait_warp(smem_u32(&bars.q_full[j]), qph);
      qph ^= 1u;
    }
    bool first = true, pend = false;
    int pt = -1, pvs = 0;
    uint32_t pvph = 0;
    // PV_j of the previous step: V(prev), P_j(prev) and (first PV of an item) O_j drained
    auto prepare_pv = [&]() {
      mbar_wait_warp(smem_u32(&bars.v_full[pvs]), pvph);
      mbar_wait_warp(smem_u32(&bars.p_full[j]), pph);
      pph ^= 1u;
      if (first && ostarted) {
        mbar_wait_warp(smem_u32(&bars.o_empty[j]), oph);
        oph ^= 1u;
      }
    };
    auto dispatch_pv = [&]() {
      const uint64_t vdesc = vdesc0 + (uint64_t)((pvs * C::kTileBytes) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < kN / 16; ++kk)
          mma_ts(ocol, scol + kk * 8, vdesc + (uint64_t)((kk * 2048) >> 4), idesc_o, (first && kk == 0) ? 0u : 1u);
        if (pt == last_t) mma_commit(smem_u32(&bars.o_full[j]));  // tile j's epilogue may start
      }
      __syncwarp();
      first = false;
      ostarted = true;
    };
    const int ns = it.bt.steps();
    for (int k = 0; k < ns; ++k) {
      int t;
      bool u0, u1;
      step_use(it.bt, k, t, u0, u1);
      if (!u0 && !u1) continue;
      const bool use = mine && (j ? u1 : u0);
      // ---- waits, overlapped with the other warp's dispatch
      if (use) mbar_wait_warp(smem_u32(&bars.k_full[ks]), kph);
      if (pend) prepare_pv();
      take_turn();
      tc_fence_after();
      if (pend) dispatch_pv();
      if (use) {
        const uint64_t bdesc = kdesc0 + (uint64_t)((ks * C::kTileBytes) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * C::kSlabBytes + (kk & 3) * 32) >> 4;
            mma_ss(scol, adesc + off, bdesc + off, idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(smem_u32(&bars.s_full[j]));
          if (t == last_t) mma_commit(smem_u32(&bars.q_empty[j]));  // Q_j(next item) may load
        }
        __syncwarp();
      }
      pass_turn();
      if (elect_one()) {
        if (pt >= 0) mma_commit(smem_u32(&bars.v_empty[pvs]));
        mma_commit(smem_u32(&bars.k_empty[ks]));
      }
      __syncwarp();
      pend = use;
      pt = t;
      pvs = vs;
      pvph = vph;
      if (++ks == C::kNK) ks = 0, kph ^= 1u;
      if (++vs == C::kNV) vs = 0, vph ^= 1u;
    }
    // trailing PV of the item (one turn per item for both warps, even without one)
    if (pend) prepare_pv();
    take_turn();
    tc_fence_after();
    if (pend) dispatch_pv();
    pass_turn();
    if (elect_one() && pt >= 0) mma_commit(smem_u32(&bars.v_empty[pvs]));
    __syncwarp();
  }
  // the other warp's last hand-over to this one is never taken: drain it, so the named
  // barrier is clean for the next kernel on this SM
  if (j == 0) asm volatile("bar.sync %0, 64;" ::"r"(kBarTurn0) : "memory");
}

// ------------------------------------------------------------------------------------------
// softmax of q tile j (warps 4j .. 4j+3): thread owns one row, all 128 columns of S_j.
// ------------------------------------------------------------------------------------------
template <int D, int BS, bool RAG>
__device__ __forceinline__ void softmax_role(const PpParams &p, PBars &bars, uint32_t tmem, int total, int j,
                                             int warp, int lane) {
  using C = PCfg<D>;
  const int row = (warp & 3) * 32 + lane;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t scol = tmem + lane_off + (j ? 128u : 0u);
  const uint32_t ocol = tmem + lane_off + (j ? C::kColO1 : C::kColO0);
  const uint64_t sl2 = f2pk(p.scale_log2, p.scale_log2);
  int trn_ = 0, trn_arg_ = 0;
  (void)trn_;
  (void)trn_arg_;
  int sc = 0;  // S handshakes of this tile
  int ic = 0;  // items of this tile
  for (int idx = item_begin(p), idx_end = item_end(p, total); idx < idx_end; idx += item_step(p)) {
    const PItem it = get_pitem<BS, RAG>(p, idx);
    if (j == 1 && !it.bt.has1) continue;
    const int64_t ti0 = it.i0 + j * kM;                     // first row of this q tile
    const int64_t ti1 = (ti0 + kM < it.N ? ti0 + kM : it.N) - 1;  // last real row
    const int64_t i = ti0 + row;
    // first window key of this row: i-W+1 (token mask) or the block-aligned start (block mode);
    // W = 0 puts it past the row
    const int64_t lo_i = BS >= 0 ? (it.W > 0 ? win_lo(i, it.W, bshift_of<BS>(p)) : i + 1) : i - it.W + 1;
    float m_used = -INFINITY, l = 0.f;
    const TileRanges rj = j ? it.bt.r[1] : it.bt.r[0];  // (no dynamic indexing: keeps it in registers)
    const int ns = it.bt.steps();
    for (int k = 0; k < ns; ++k) {
      const int t = it.bt.at(k);
      if (!tile_in(rj, t)) continue;
      const int64_t j0 = (int64_t)t * kN;
      const bool full = kv_tile_full(ti0, ti1, t, it.W, p.n_sink, bshift_of<BS>(p));
      mbar_wait_warp(smem_u32(&bars.s_full[j]), sc & 1);
      ++sc;
      if ((warp & 3) == 0) PPTR(1 + j, 40)
      tc_fence_after();
      float x[kN];
#pragma unroll
      for (int c = 0; c < kN / 32; ++c) tmem_ld32_f(scol + c * 32, &x[c * 32]);
      tmem_wait_ld();
      if ((warp & 3) == 0) PPTR(1 + j, 42)
      if (!full) {
        // key j0+c visible to row i  <=>  c <= i-j0  and  (c < s-j0  or  j0+c >= lo_i)
        const int dd = (int)(i - j0), sk = (int)(p.n_sink - j0);
        const int lo = BS >= 0 ? (int)(lo_i - j0) - 1 : dd - it.W;  // token mask: the original form
#if MOA_PP_MASK_BITS
        // as 32-bit visibility words (a bit test + a select per element instead of three compares)
#pragma unroll
        for (int w = 0; w < kN / 32; ++w) {
          const uint32_t vis = bits_le(dd - 32 * w) & (bits_le(sk - 1 - 32 * w) | ~bits_le(lo - 32 * w));
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!(vis & (1u << e))) x[32 * w + e] = -INFINITY;
        }
#else
#pragma unroll
        for (int c = 0; c < kN; ++c) {
          const bool vis = c <= dd && (c < sk || c > lo);
          if (!vis) x[c] = -INFINITY;
        }
#endif
      }
      float mx[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) mx[a] = fmaxf(x[a], x[a + 8]);
#pragma unroll
      for (int c = 16; c < kN; c += 16)
#pragma unroll
        for (int a = 0; a < 8; a += 2) {
          mx[a] = fmax3(mx[a], x[c + a], x[c + a + 8]);
          mx[a + 1] = fmax3(mx[a + 1], x[c + a + 1], x[c + a + 9]);
        }
      const float rmax = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7]));
      const float mt = rmax * p.scale_log2;
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
        // PV_j(prev) is complete (S_j(t) completed after it); scale this row of O_j
#pragma unroll kUnrollRescale
        for (int c = 0; c < D / 32; ++c) {
          float r[32];
          tmem_ld32_f(ocol + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] *= alpha;
          tmem_st32(ocol + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r));
        }
      }
      l *= alpha;
      const float nm = m_used == -INFINITY ? 0.f : -m_used;
      const uint64_t nm2 = f2pk(nm, nm);
      uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
      uint32_t pk[64];  // P_j row, bf16 pairs
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int c = ch * 32 + e;  // pair index: columns 2c, 2c+1
          const uint64_t y = ffma2(f2pk(x[2 * c], x[2 * c + 1]), sl2, nm2);
          float ya, yb, ea, eb;
          f2upk(y, ya, yb);
          if (c % kPolyEvery == kPolyEvery - 1) {
            exp2_poly2(ya, yb, ea, eb);
          } else {
            ea = fast_exp2(ya);
            eb = fast_exp2(yb);
          }
          if (!MOA_PP_LATE_SUM) acc[e & 3] = fadd2(acc[e & 3], f2pk(ea, eb));
          pk[c] = pack_bf16x2(ea, eb);
        }
        tmem_st32(scol + ch * 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[ch * 32]));
      }
      if ((warp & 3) == 0) PPTR(1 + j, 43)
      tmem_wait_st();
      if ((warp & 3) == 0) PPTR(1 + j, 44)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars.p_full[j]));
      if ((warp & 3) == 0) PPTR(1 + j, 41)
      if (MOA_PP_LATE_SUM) {
        // row sum of the bf16 P the tensor core multiplies, after P is handed over (off the
        // critical path of the MMA chain): a bf16 is the top half of an f32
#pragma unroll
        for (int c = 0; c < 64; ++c)
          acc[c & 3] = fadd2(acc[c & 3], f2pk(__uint_as_float(pk[c] << 16), __uint_as_float(pk[c] & 0xffff0000u)));
      }
      float s0, s1;
      f2upk(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])), s0, s1);
      l += s0 + s1;
    }
    // epilogue: O_j / l -> bf16 rows, lse
    mbar_wait_warp(smem_u32(&bars.o_full[j]), ic & 1);
    ++ic;
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const bool store = MOA_PP_OSTORE && i <= ti1 && (!RAG || i < p.seq_n[it.b]);  // ragged: rows past N_b are not outputs
    __nv_bfloat16 *orow =
        static_cast<__nv_bfloat16 *>(p.o) + ((int64_t)it.b * p.N + i) * p.o_row_stride + (int64_t)it.h * D;
#pragma unroll kUnrollEpi
    for (int c = 0; c < D / 32; c += 2) {  // two TMEM loads in flight per wait
      float r[32], r2[32];
      tmem_ld32_f(ocol + c * 32, r);
      tmem_ld32_f(ocol + (c + 1) * 32, r2);
      tmem_wait_ld();
      if (store) {
        store_o_chunk32(orow + c * 32, r, inv, p.o_v8);
        store_o_chunk32(orow + (c + 1) * 32, r2, inv, p.o_v8);
      }
    }
    if (p.lse && store)
      p.lse[((int64_t)it.b * p.nql + it.h) * p.N + i] = l > 0.f ? (m_used + __log2f(l)) * kLn2 : -INFINITY;
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars.o_empty[j]));
  }
}

// ------------------------------------------------------------------------------------------
// softmax (warps 0-7): warp w owns rows 32 (w & 3) .. +31 (its TMEM lanes) and column half
// hf = w >> 2 of BOTH q tiles, in the order the tensor core completes them (S0(t), S1(t)).
// The two warps of a row block (w, w ^ 4) exchange their half-row max (and at the end their
// half-row sums) through shared memory and a named barrier.  Eight warps per tile halve the
// per-thread work of a tile's softmax, which bounds the ping-pong: one tile's softmax must
// fit under the other tile's MMAs.
// ------------------------------------------------------------------------------------------
template <int D, int BS, bool RAG>
__device__ __forceinline__ void softmax_split_role(const PpParams &p, PBars &bars, uint32_t tmem, int total, int warp,
                                             int lane, float (*red)[2][kM]) {
  using C = PCfg<D>;
  constexpr int kCols = kN / 2;   // S columns of this warp per tile
  constexpr int kOCols = D / 2;   // O columns of this warp per tile
  const int hf = warp >> 2;
  const int row = (warp & 3) * 32 + lane;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int bar_pair = kBarPair0 + (warp & 3);
  auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_pair) : "memory"); };
  const uint64_t sl2 = f2pk(p.scale_log2, p.scale_log2);
  int trn_ = 0, trn_arg_ = 0;
  (void)trn_;
  (void)trn_arg_;
  int sc[2] = {0, 0};  // S handshakes per tile
  int ic[2] = {0, 0};  // items per tile
  for (int idx = item_begin(p), idx_end = item_end(p, total); idx < idx_end; idx += item_step(p)) {
    const PItem it = get_pitem<BS, RAG>(p, idx);
    const bool has1 = it.bt.has1;
    float m_used[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    const int ns = it.bt.steps();
    for (int k = 0; k < ns; ++k) {
      int t;
      bool u[2];
      step_use(it.bt, k, t, u[0], u[1]);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (!u[j]) continue;
        const int64_t ti0 = it.i0 + j * kM;                         // first row of this q tile
        const int64_t ti1 = (ti0 + kM < it.N ? ti0 + kM : it.N) - 1;  // last real row
        const int64_t i = ti0 + row;
        const int64_t j0 = (int64_t)t * kN + hf * kCols;  // key of this warp's first column
        const uint32_t sbase = tmem + lane_off + (j ? 128u : 0u);
        const uint32_t ocol = tmem + lane_off + (j ? C::kColO1 : C::kColO0) + hf * kOCols;
        const bool full = kv_tile_full(ti0, ti1, t, it.W, p.n_sink, bshift_of<BS>(p));
        mbar_wait_warp(smem_u32(&bars.s_full[j]), sc[j] & 1);
        ++sc[j];
        if (warp == 0) PPTR(1 + j, 40)
        tc_fence_after();
        float x[kCols];
#pragma unroll
        for (int c = 0; c < kCols / 32; ++c) tmem_ld32_f(sbase + hf * kCols + c * 32, &x[c * 32]);
        tmem_wait_ld();
        if (!full) {
          const int64_t lo_i = BS >= 0 ? (it.W > 0 ? win_lo(i, it.W, bshift_of<BS>(p)) : i + 1) : i - it.W + 1;
          // key j0+c visible to row i  <=>  c <= i-j0  and  (c < s-j0  or  j0+c >= lo_i)
          const int dd = (int)(i - j0), sk = (int)(p.n_sink - j0), lo = (int)(lo_i - j0) - 1;
#pragma unroll
          for (int w = 0; w < kCols / 32; ++w) {  // as 32-bit visibility words (see softmax_role)
            const uint32_t vis = bits_le(dd - 32 * w) & (bits_le(sk - 1 - 32 * w) | ~bits_le(lo - 32 * w));
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (!(vis & (1u << e))) x[32 * w + e] = -INFINITY;
          }
        }
        float mx[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) mx[a] = fmaxf(x[a], x[a + 8]);
#pragma unroll
        for (int c = 16; c < kCols; c += 16)
#pragma unroll
          for (int a = 0; a < 8; a += 2) {
            mx[a] = fmax3(mx[a], x[c + a], x[c + a + 8]);
            mx[a + 1] = fmax3(mx[a + 1], x[c + a + 1], x[c + a + 9]);
          }
        float rmax = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7]));
        // row max of both halves.  red[j][hf] is rewritten only after the next s_full of tile j,
        // which follows the partner's p_full arrival, i.e. its read below.  The barrier also
        // orders the partner's S load before our P store over its columns.
        red[j][hf][row] = rmax;
        pair_sync();
        rmax = fmaxf(rmax, red[j][hf ^ 1][row]);
        const float mt = rmax * p.scale_log2;
        bool rescale = false;
        float alpha = 1.f;
        if (m_used[j] == -INFINITY) {
          m_used[j] = mt;  // first visible scores of this row: O and l are still exactly 0
        } else if (mt > m_used[j] + kRescaleThreshold) {
          rescale = true;
          alpha = fast_exp2(m_used[j] - mt);
          m_used[j] = mt;
        }
        if (__any_sync(0xffffffffu, rescale)) {
          // PV_j(prev) is complete (S_j(t) completed after it); scale our half of this row of O_j
#pragma unroll
          for (int c = 0; c < kOCols / 32; ++c) {
            float r[32];
            tmem_ld32_f(ocol + c * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] *= alpha;
            tmem_st32(ocol + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r));
          }
        }
        l[j] *= alpha;
        const float nm = m_used[j] == -INFINITY ? 0.f : -m_used[j];
        const uint64_t nm2 = f2pk(nm, nm);
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        uint32_t pk[kCols / 2];
#pragma unroll
        for (int c = 0; c < kCols / 2; ++c) {  // pair index: columns 2c, 2c+1
          const uint64_t y = ffma2(f2pk(x[2 * c], x[2 * c + 1]), sl2, nm2);
          float ya, yb, ea, eb;
          f2upk(y, ya, yb);
          if (c % kPolyEvery == kPolyEvery - 1) {
            exp2_poly2(ya, yb, ea, eb);
          } else {
            ea = fast_exp2(ya);
            eb = fast_exp2(yb);
          }
          acc[c & 3] = fadd2(acc[c & 3], f2pk(ea, eb));
          pk[c] = pack_bf16x2(ea, eb);
        }
        // P_j (bf16 pairs) in packed columns [hf * 32, +32) of S_j: over the first half's S
        tmem_st32(sbase + hf * (kCols / 2), pk);
        float s0, s1;
        f2upk(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])), s0, s1);
        l[j] += s0 + s1;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars.p_full[j]));
        if (warp == 0) PPTR(1 + j, 41)
      }
    }
    // epilogues: O_j / l -> bf16 rows (our half of the columns), lse
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (j == 1 && !has1) continue;
      const int64_t ti0 = it.i0 + j * kM;
      const int64_t ti1 = (ti0 + kM < it.N ? ti0 + kM : it.N) - 1;
      const int64_t i = ti0 + row;
      const uint32_t ocol = tmem + lane_off + (j ? C::kColO1 : C::kColO0) + hf * kOCols;
      mbar_wait_warp(smem_u32(&bars.o_full[j]), ic[j] & 1);
      ++ic[j];
      red[j][hf][row] = l[j];
      pair_sync();
      const float lt = l[j] + red[j][hf ^ 1][row];
      pair_sync();  // both read before the slot is reused by the next item's row max
      tc_fence_after();
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      const bool store = MOA_PP_OSTORE && i <= ti1 && (!RAG || i < p.seq_n[it.b]);  // ragged: rows past N_b are not outputs
      __nv_bfloat16 *orow = static_cast<__nv_bfloat16 *>(p.o) + ((int64_t)it.b * p.N + i) * p.o_row_stride +
                            (int64_t)it.h * D + hf * kOCols;
#pragma unroll
      for (int c = 0; c < kOCols / 32; c += 2) {  // two TMEM loads in flight per wait
        float r[32], r2[32];
        const bool two = c + 1 < kOCols / 32;  // (D = 64: one chunk per half)
        tmem_ld32_f(ocol + c * 32, r);
        if (two) tmem_ld32_f(ocol + (c + 1) * 32, r2);
        tmem_wait_ld();
        if (store) {
          store_o_chunk32(orow + c * 32, r, inv, p.o_v8);
          if (two) store_o_chunk32(orow + (c + 1) * 32, r2, inv, p.o_v8);
        }
      }
      if (p.lse && store && hf == 0)
        p.lse[((int64_t)it.b * p.nql + it.h) * p.N + i] =
            lt > 0.f ? (m_used[j] + __log2f(lt)) * kLn2 : -INFINITY;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars.o_empty[j]));
    }
  }
}

template <int D, int BS, bool RAG>
__global__ void __launch_bounds__(kThreads, 1)
    prefill_pp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kc16,
                      const __grid_constant__ CUtensorMap tm_vc16, const __grid_constant__ CUtensorMap tm_kc1,
                      const __grid_constant__ CUtensorMap tm_vc1, const PpParams p) {
  using C = PCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];  // SW128 TMA / UMMA tiles need 1024-B alignment
  __shared__ PBars bars;
  __shared__ float red[2][2][kM];  // split softmax: [tile][column half][row] row max / row sum
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t smem_base = smem_u32(smem_raw);
  if (smem_base & 1023u) __trap();
  const uint32_t q_smem = smem_base;                        // Q0, Q1
  const uint32_t k_smem = q_smem + 2 * C::kTileBytes;       // kNK tiles
  const uint32_t v_smem = k_smem + C::kNK * C::kTileBytes;  // kNV tiles
  const int total = RAG ? p.n_items : p.n_items * p.batch;

  if (tid == 0) {
    for (int j = 0; j < 2; ++j) {
      mbar_init(smem_u32(&bars.q_full[j]), 1);
      mbar_init(smem_u32(&bars.q_empty[j]), 1);
      mbar_init(smem_u32(&bars.s_full[j]), 1);
      mbar_init(smem_u32(&bars.p_full[j]), softmax_warps_per_tile<BS>());
      mbar_init(smem_u32(&bars.o_full[j]), 1);
      mbar_init(smem_u32(&bars.o_empty[j]), softmax_warps_per_tile<BS>());
    }
    for (int s = 0; s < C::kNK; ++s) {
      mbar_init(smem_u32(&bars.k_full[s]), 1);
      mbar_init(smem_u32(&bars.k_empty[s]), 2);  // one commit per MMA warp
      mbar_init(smem_u32(&bars.k_copied[s]), 1);
      mbar_init(smem_u32(&bars.k_issued[s]), 1);
    }
    for (int s = 0; s < C::kNV; ++s) {
      mbar_init(smem_u32(&bars.v_full[s]), 1);
      mbar_init(smem_u32(&bars.v_empty[s]), 2);
      mbar_init(smem_u32(&bars.v_copied[s]), 1);
      mbar_init(smem_u32(&bars.v_issued[s]), 1);
    }
    fence_mbar_init();
  }
  if (warp == kWarpMMA) tmem_alloc<kTmemCols>(smem_u32(&bars.tmem_base));
  if (warp == kWarpKV && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp >= kSoftmaxWarp0 && warp < kSoftmaxWarp0 + 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(MOA_PP_REG_SOFTMAX) : "memory");
    if (BS >= 0)
      softmax_split_role<D, BS, RAG>(p, bars, tmem, total, warp, lane, red);
    else
      softmax_role<D, BS, RAG>(p, bars, tmem, total, (warp - kSoftmaxWarp0) >> 2, warp, lane);
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(MOA_PP_REG_OTHER) : "memory");
  if (warp == kWarpKV) {
    if (lane == 0) {
      int T = 0;
      uint32_t kfill = 0, vfill = 0, kcph = 0, vcph = 0;  // per slot: holds a filler tile / copied parity
      for (int idx = item_begin(p), idx_end = item_end(p, total); idx < idx_end; idx += item_step(p)) {
        const PItem it = get_pitem<BS, RAG>(p, idx);
        const int g = it.h / p.G;
        const bool fi = fill_item(p, it);
        const int Wg = fi ? p.win_g[g] : 0;
        const int ns = it.bt.steps();
        for (int k = 0; k < ns; ++k) {
          int t;
          bool u0, u1;
          step_use(it.bt, k, t, u0, u1);
          if (!u0 && !u1) continue;
          const bool ft = fi && fill_tile(p, it.i0, it.N, Wg, t);
          const int j0 = t * kN;
          const int ks = T % C::kNK;
          if (T >= C::kNK) mbar_wait(smem_u32(&bars.k_empty[ks]), ((T - C::kNK) / C::kNK) & 1);
          if (kfill >> ks & 1) {  // warp 10's stores still read the previous (filler) tile of this slot
            mbar_wait(smem_u32(&bars.k_copied[ks]), kcph >> ks & 1);
            kcph ^= 1u << ks;
          }
          kfill = (kfill & ~(1u << ks)) | ((uint32_t)ft << ks);
          const uint32_t kbar = smem_u32(&bars.k_full[ks]);
          mbar_expect_tx(kbar, C::kTileBytes);
          for (int sl = 0; sl < C::kSlabs; ++sl)
            tma_load_4d(k_smem + ks * C::kTileBytes + sl * C::kSlabBytes, &tm_k, kbar, sl * 64, g, j0, it.b);
          if (ft) mbar_arrive(smem_u32(&bars.k_issued[ks]));  // warp 10 may wait for this fill's k_full phase
          const int vs = T % C::kNV;
          if (T >= C::kNV) mbar_wait(smem_u32(&bars.v_empty[vs]), ((T - C::kNV) / C::kNV) & 1);
          if (vfill >> vs & 1) {
            mbar_wait(smem_u32(&bars.v_copied[vs]), vcph >> vs & 1);
            vcph ^= 1u << vs;
          }
          vfill = (vfill & ~(1u << vs)) | ((uint32_t)ft << vs);
          const uint32_t vbar = smem_u32(&bars.v_full[vs]);
          mbar_expect_tx(vbar, C::kTileBytes);
          for (int sl = 0; sl < C::kSlabs; ++sl)
            tma_load_4d(v_smem + vs * C::kTileBytes + sl * C::kSlabBytes, &tm_v, vbar, sl * 64, g, j0, it.b);
          if (ft) mbar_arrive(smem_u32(&bars.v_issued[vs]));
          ++T;
        }
      }
    }
  } else if (warp == kWarpQ) {
    if (lane == 0) {
      int qc[2] = {0, 0};
      int T = 0;  // K/V ring step (the producer's count)
      uint32_t kiph = 0, viph = 0;  // per slot: parity of the next issued-barrier phase
      for (int idx = item_begin(p), idx_end = item_end(p, total); idx < idx_end; idx += item_step(p)) {
        const PItem it = get_pitem<BS, RAG>(p, idx);
        for (int j = 0; j < 2; ++j) {
          if (j == 1 && !it.bt.has1) continue;
          if (qc[j] > 0) mbar_wait(smem_u32(&bars.q_empty[j]), (qc[j] - 1) & 1);
          ++qc[j];
          const uint32_t qbar = smem_u32(&bars.q_full[j]);
          mbar_expect_tx(qbar, C::kTileBytes);
          for (int sl = 0; sl < C::kSlabs; ++sl)
            tma_load_4d(q_smem + j * C::kTileBytes + sl * C::kSlabBytes, &tm_q, qbar, sl * 64, it.h,
                        (int)(it.i0 + j * kM), it.b);
        }
        // warm L2 with the next item's Q tiles (their loads wait for this item's last S MMAs)
        if (idx + item_step(p) < idx_end) {
          const PItem nx = get_pitem<BS, RAG>(p, idx + item_step(p));
          for (int j = 0; j < (nx.bt.has1 ? 2 : 1); ++j)
            for (int sl = 0; sl < C::kSlabs; ++sl)
              tma_prefetch_4d(&tm_q, sl * 64, nx.h, (int)(nx.i0 + j * kM), nx.b);
        }
        // fused cache fill: TMA-store the kept rows of this item's filler tiles.  The producer
        // signals each filler load it issues (k_issued / v_issued) and does not refill a slot
        // holding a filler tile before warp 10 releases it (k_copied / v_copied), so the
        // full-barrier phase warp 10 then waits for is unambiguous; the slots are released at
        // the item's end, once the stores have read them
        if (!p.fill) continue;
        const bool fi = fill_item(p, it);
        const int ns = it.bt.steps();
        if (!fi) {
          for (int k = 0; k < ns; ++k) {
            int t;
            bool u0, u1;
            step_use(it.bt, k, t, u0, u1);
            T += (u0 || u1);
          }
          continue;
        }
        const int g = it.h / p.G;
        const int Wg = p.win_g[g];
        const int64_t region = (int64_t)it.b * p.rows_per_seq + p.g_off[g];
        uint32_t pend[4];  // copied-barriers of this item's stored tiles (<= 2 diagonal tiles)
        int np_ = 0;
        for (int k = 0; k < ns; ++k) {
          int t;
          bool u0, u1;
          step_use(it.bt, k, t, u0, u1);
          if (!u0 && !u1) continue;
          if (fill_tile(p, it.i0, it.N, Wg, t)) {
            const int ks = T % C::kNK, vs = T % C::kNV;
            mbar_wait(smem_u32(&bars.k_issued[ks]), kiph >> ks & 1);
            kiph ^= 1u << ks;
            mbar_wait(smem_u32(&bars.k_full[ks]), (T / C::kNK) & 1);
            fill_store<D>(p, k_smem + ks * C::kTileBytes, &tm_kc16, &tm_kc1, region, it.N, Wg, t);
            mbar_wait(smem_u32(&bars.v_issued[vs]), viph >> vs & 1);
            viph ^= 1u << vs;
            mbar_wait(smem_u32(&bars.v_full[vs]), (T / C::kNV) & 1);
            fill_store<D>(p, v_smem + vs * C::kTileBytes, &tm_vc16, &tm_vc1, region, it.N, Wg, t);
            pend[np_++] = smem_u32(&bars.k_copied[ks]);
            pend[np_++] = smem_u32(&bars.v_copied[vs]);
          }
          ++T;
        }
        if (np_) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          for (int i = 0; i < np_; ++i) mbar_arrive(pend[i]);
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // cache writes complete
    }
  } else if (warp == kWarpMMA || warp == kWarpMMA1) {
    mma_role<D, BS, RAG>(p, bars, tmem, q_smem, k_smem, v_smem, total, warp == kWarpMMA ? 0 : 1);
  }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMMA) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

// ==========================================================================================
// Clustered prefill (token mask, uniform batch; SURVEY §8(a) a4 + a5).  The two-tile kernel
// above aliases P_j with the first columns of S_j, so S_j(t+1) cannot start before PV_j(t)
// has read P_j(t): each tile's chain  softmax -> PV -> S -> softmax  is serial and two tiles
// keep the tensor core ~60 % busy (profiles/).  Here a cluster of two CTAs (two SMs)
// takes one 256-row item and each CTA owns ONE 128-row q tile, which frees TMEM for separate,
// double-buffered S and P:
//   TMEM (512 columns): S0 | S1 (fp32 128x128) | P0 | P1 (bf16 packed 128x128) | O (fp32 128xD)
// so S(u+1) and PV(u-1) are computed while the softmax of S(u) runs -- the softmax warps
// never wait for the tensor core in the steady state.  Each K/V tile
// of the pair's union schedule is loaded ONCE for both SMs: CTA r TMA-loads rows
// [64 r, 64 r + 64) of it multicast into both CTAs' shared memory (each full barrier expects
// the whole tile), so L2 traffic stays that of the two-tile kernel; a slot is refilled only
// after both CTAs' MMA warps released it (multicast tcgen05.commit, barrier count 2).
//
// Warps (384 threads; setmaxnreg gives the softmax warpgroups 208 registers, the rest 88):
//   0-3  softmax of the even used steps (S0/P0) + epilogue    (thread = row = TMEM lane)
//   4-7  softmax of the odd used steps (S1/P1)
//   8    TMA producer: this CTA's halves of the K and V tiles (multicast)
//   9    TMEM allocator + S = Q K^T issue
//   10   Q tiles + fused cache fill (TMA stores from shared memory)
//   11   O += P V issue
// ==========================================================================================
#ifndef MOA_CL_THREADS
#define MOA_CL_THREADS 384
#endif
constexpr int kCThreads = MOA_CL_THREADS;  // warps 9-11 idle: warpgroup-aligned register reallocation
#ifndef MOA_CL_REG_SOFTMAX
#define MOA_CL_REG_SOFTMAX 208
#endif
#ifndef MOA_CL_REG_OTHER
#define MOA_CL_REG_OTHER 88
#endif
// per sub-partition: two softmax warps + one other; an exact fit of the 512-register slot
// hung setmaxnreg.inc on B200 (one softmax warp: 240 + 2 x 136), 504 works
static_assert(2 * MOA_CL_REG_SOFTMAX + MOA_CL_REG_OTHER <= 504, "clustered prefill register split");
constexpr int kCWarpKV = 8, kCWarpMMA = 9, kCWarpQ = 10, kCWarpPV = 11;
constexpr uint32_t kColS = 0, kColP = 256, kColO = 384;

// shared memory: kQ Q buffers (per item parity when 2), kNK K and kNV V slots of 32 KB (D=128);
// the K ring is the deep one: a K slot is freed only when BOTH CTAs' S MMAs have read it
#ifndef MOA_CL_Q
#define MOA_CL_Q 1
#endif
#ifndef MOA_CL_NK
#define MOA_CL_NK 4
#endif
template <int D>
struct CCfg {
  static constexpr int kQ = MOA_CL_Q;
  static constexpr int kNK = D == 128 ? MOA_CL_NK : 4;
  static constexpr int kNV = D == 128 ? 7 - MOA_CL_Q - MOA_CL_NK : 4;  // 224 KB + < 3 KB static
  static_assert(kNK <= 6 && kNV <= 4 && kNV >= 2 && kQ >= 1 && kQ <= 2, "clustered prefill ring sizes");
  static constexpr int kSmemBytes = (kQ + kNK + kNV) * PCfg<D>::kTileBytes;
};

struct CBars {
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[6], k_empty[6];
  uint64_t v_full[4], v_empty[4];
  uint64_t s_full[2], s_free[2], p_full[2], p_free[2];
  uint64_t o_full, o_empty;
  uint64_t ml_full[4], ml_empty[4];   // softmax group 1 -> group 0 epilogue hand-over, per warp pair
  uint64_t k_copied[6], v_copied[4];  // fused fill: the filler CTA's stores have read a slot
  uint64_t k_issued[6], v_issued[4];  // fused fill: this CTA's producer issued a filler tile
  uint32_t tmem_base;
};

// CTA rank of the cluster whose q tile holds rows [128 t, 128 t + 128) of the item (the
// fused fill of kv tile t is done by it: t is that q tile's diagonal tile)
__device__ __forceinline__ int fill_rank(const PItem &it, int t) { return t - (int)(it.i0 / kN); }

// MMA issue by two warps: warp 5 issues every S(u) = Q K(u)^T and warp 8 every PV(u) (O += P(u)
// V(u)).  An MMA dispatch is nearly synchronous for the issuing thread and each MMA warp shares
// its sub-partition with a busy softmax warp, so one warp doing both (waits, commits and loop
// bookkeeping between dispatch groups) left the tensor core idle half the time; split, S(u+1)
// waits only for its S buffer (free as soon as the softmax has S(u-1) in registers) and K(u+1),
// and PV(u) only for P(u) and V(u).  The two streams touch disjoint TMEM (S buffers vs P
// buffers + O), so their relative order in the tensor pipe does not matter.
template <int D>
__device__ __forceinline__ void cl_mma_s_role(const PpParams &p, CBars &bars, uint32_t tmem, uint32_t q_smem,
                                              uint32_t k_smem, int total, int rank, int cid, int ncl) {
  using C = PCfg<D>;
  using CC = CCfg<D>;
  constexpr uint32_t idesc_s = idesc_bf16_f32(kM, kN, false);
  const uint64_t kdesc0 = smem_desc_sw128(k_smem, 16, 1024);
  int T = 0, u = 0, ic = 0;  // union steps (K ring), used steps (S buffers), items of this CTA
  int trn_ = 0, trn_arg_ = 0;
  (void)trn_;
  (void)trn_arg_;
  for (int idx = cid; idx < total; idx += ncl) {
    const PItem it = get_pitem<-1, false>(p, idx);
    const bool mine = rank == 0 || it.bt.has1;
    const TileRanges r = rank ? it.bt.r[1] : it.bt.r[0];
    const int last_t = r.b1 > r.b0 ? r.b1 - 1 : r.a1 - 1;
    const int qb = ic % CC::kQ;
    const uint64_t adesc = smem_desc_sw128(q_smem + qb * C::kTileBytes, 16, 1024);
    bool first_s = true;
    const int ns = it.bt.steps();
    for (int k = 0; k < ns; ++k) {
      int t;
      bool u0, u1;
      step_use(it.bt, k, t, u0, u1);
      if (!u0 && !u1) continue;
      const bool use = mine && (rank ? u1 : u0);
      const int ks = T % CC::kNK;
      // every step's data must have landed before this CTA releases the slot (clean phases)
      mbar_wait_warp(smem_u32(&bars.k_full[ks]), (T / CC::kNK) & 1);
      if (use) {
        const int b = u & 1;
        if (u >= 2) mbar_wait_warp(smem_u32(&bars.s_free[b]), ((u >> 1) - 1) & 1);
        if (first_s) mbar_wait_warp(smem_u32(&bars.q_full[qb]), (ic / CC::kQ) & 1);
        first_s = false;
        trn_arg_ = T;
        PPTR_CTA(0, 0, 2)
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bdesc = kdesc0 + (uint64_t)((ks * C::kTileBytes) >> 4);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * C::kSlabBytes + (kk & 3) * 32) >> 4;
            mma_ss(tmem + kColS + 128 * b, adesc + off, bdesc + off, idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(smem_u32(&bars.s_full[b]));
          if (t == last_t) mma_commit(smem_u32(&bars.q_empty[qb]));
          mma_commit_mc(smem_u32(&bars.k_empty[ks]), 3);
        }
        __syncwarp();
        PPTR_CTA(0, 0, 30)
        ++u;
      } else {
        if (elect_one()) mma_commit_mc(smem_u32(&bars.k_empty[ks]), 3);
        __syncwarp();
      }
      ++T;
    }
    if (mine) ++ic;
  }
}

template <int D>
__device__ __forceinline__ void cl_mma_pv_role(const PpParams &p, CBars &bars, uint32_t tmem, uint32_t v_smem,
                                               int total, int rank, int cid, int ncl) {
  using C = PCfg<D>;
  using CC = CCfg<D>;
  constexpr uint32_t idesc_o = idesc_bf16_f32(kM, D, true);
  const uint64_t vdesc0 = smem_desc_sw128(v_smem, C::kSlabBytes, 1024);
  int T = 0, u = 0, ic = 0;  // union steps (V ring), used steps (P buffers), items of this CTA
  int trn_ = 0, trn_arg_ = 0;
  (void)trn_;
  (void)trn_arg_;
  for (int idx = cid; idx < total; idx += ncl) {
    const PItem it = get_pitem<-1, false>(p, idx);
    const bool mine = rank == 0 || it.bt.has1;
    bool first_pv = true;
    const int ns = it.bt.steps();
    for (int k = 0; k < ns; ++k) {
      int t;
      bool u0, u1;
      step_use(it.bt, k, t, u0, u1);
      if (!u0 && !u1) continue;
      const bool use = mine && (rank ? u1 : u0);
      const int vs = T % CC::kNV;
      mbar_wait_warp(smem_u32(&bars.v_full[vs]), (T / CC::kNV) & 1);
      if (use) {
        const int b = u & 1;
        mbar_wait_warp(smem_u32(&bars.p_full[b]), (u >> 1) & 1);
        if (first_pv && ic > 0) mbar_wait_warp(smem_u32(&bars.o_empty), (ic - 1) & 1);  // O drained
        PPTR_CTA(0, 3, 10)
        tc_fence_after();
        if (elect_one()) {
          const uint64_t vdesc = vdesc0 + (uint64_t)((vs * C::kTileBytes) >> 4);
#pragma unroll
          for (int kk = 0; kk < kN / 16; ++kk)
            mma_ts(tmem + kColO, tmem + kColP + 64 * b + kk * 8, vdesc + (uint64_t)((kk * 2048) >> 4), idesc_o,
                   (first_pv && kk == 0) ? 0u : 1u);
          mma_commit(smem_u32(&bars.p_free[b]));
          mma_commit_mc(smem_u32(&bars.v_empty[vs]), 3);
        }
        __syncwarp();
        PPTR_CTA(0, 3, 20)
        first_pv = false;
        ++u;
      } else {
        if (elect_one()) mma_commit_mc(smem_u32(&bars.v_empty[vs]), 3);
        __syncwarp();
      }
      ++T;
    }
    if (mine) {
      if (elect_one()) mma_commit(smem_u32(&bars.o_full));  // every PV of the item complete
      __syncwarp();
      ++ic;
    }
  }
}

// Softmax of this CTA's q tile by TWO warpgroups that take alternate used steps: group
// g = warp >> 2 handles the steps u with u % 2 == g, i.e. always S buffer g and P buffer g
// (thread = row = TMEM lane (warp & 3) * 32 + lane in both groups).  With S double-buffered
// the two groups' steps overlap, so each sub-partition runs two softmax warps at once (one
// warp alone is latency-bound).  The lazy row reference m (exponentials are taken against it;
// it moves only when a row max exceeds it by 2^8) is passed from step u-1 to step u through
// shared memory (m_x[u & 1][row]) and a named barrier per (warp pair, parity): the owner of
// step u-1 publishes its reference right after its row max, so step u waits only for that,
// not for the whole step.  Each group keeps its own partial row sum against the last
// reference it used (rescaled when the reference moves); group 0 merges them in the epilogue.
constexpr int kBarMx0 = 1;   // named barriers 1..8: m exchange, (warp pair, step parity)

template <int D>
__device__ __forceinline__ void cl_softmax_role(const PpParams &p, CBars &bars, uint32_t tmem, int total, int rank,
                                                int cid, int ncl, int warp, int lane, float (*m_x)[kM],
                                                float2 *ml_x) {
  const int grp = warp >> 2, wq = warp & 3;
  const int row = wq * 32 + lane;
  const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
  const uint32_t ocol = tmem + lane_off + kColO;
  const uint32_t scol = tmem + lane_off + kColS + 128 * grp;
  const uint32_t pcol = tmem + lane_off + kColP + 64 * grp;
  const uint64_t sl2 = f2pk(p.scale_log2, p.scale_log2);
  int trn_ = 0, trn_arg_ = 0;
  (void)trn_;
  (void)trn_arg_;
  int u = 0, ic = 0;  // used steps of this CTA (both groups count all of them), items
  for (int idx = cid; idx < total; idx += ncl) {
    const PItem it = get_pitem<-1, false>(p, idx);
    if (rank == 1 && !it.bt.has1) continue;
    const int64_t ti0 = it.i0 + rank * kM;
    const int64_t ti1 = (ti0 + kM < it.N ? ti0 + kM : it.N) - 1;
    const int64_t i = ti0 + row;
    const TileRanges rj = rank ? it.bt.r[1] : it.bt.r[0];
    const int nu = rj.count();  // used steps of this item
    const int u_first = u;
    float m_seen = -INFINITY, l = 0.f;  // this group's reference and partial row sum
    const int ns = it.bt.steps();
    for (int k = 0; k < ns; ++k) {
      const int t = it.bt.at(k);
      if (!tile_in(rj, t)) continue;
      if ((u & 1) != grp) {
        ++u;
        continue;
      }
      const int64_t j0 = (int64_t)t * kN;
      const bool full = kv_tile_full(ti0, ti1, t, it.W, p.n_sink);
      mbar_wait_warp(smem_u32(&bars.s_full[grp]), (u >> 1) & 1);
      if (wq == 0) PPTR(1 + grp, 40)
      tc_fence_after();
      float x[kN];
#pragma unroll
      for (int c = 0; c < kN / 32; ++c) tmem_ld32_f(scol + c * 32, &x[c * 32]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars.s_free[grp]));  // the tensor core may compute S(u+2)
      if (!full) {
        // key j0+c visible to row i  <=>  c <= i-j0  and  (c < s-j0  or  c > i-j0-W)
        const int dd = (int)(i - j0), sk = (int)(p.n_sink - j0), lo = dd - it.W;
#pragma unroll
        for (int w = 0; w < kN / 32; ++w) {
          const uint32_t vis = bits_le(dd - 32 * w) & (bits_le(sk - 1 - 32 * w) | ~bits_le(lo - 32 * w));
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!(vis & (1u << e))) x[32 * w + e] = -INFINITY;
        }
      }
      float mx[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) mx[a] = fmaxf(x[a], x[a + 8]);
#pragma unroll
      for (int c = 16; c < kN; c += 16)
#pragma unroll
        for (int a = 0; a < 8; a += 2) {
          mx[a] = fmax3(mx[a], x[c + a], x[c + a + 8]);
          mx[a + 1] = fmax3(mx[a + 1], x[c + a + 1], x[c + a + 9]);
        }
      const float rmax = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7]));
      const float mt = rmax * p.scale_log2;
      if (wq == 0) PPTR(1 + grp, 42)
      // the reference after step u-1 (the other group's step, or none at the item's start)
      float m_prev = -INFINITY;
      if (u > u_first) {
        asm volatile("bar.sync %0, 64;" ::"r"(kBarMx0 + 2 * wq + ((u - 1) & 1)) : "memory");
        m_prev = m_x[(u - 1) & 1][row];
      }
      if (wq == 0) PPTR(1 + grp, 43)
      float m_u = m_prev;
      bool rescale = false;
      if (m_prev == -INFINITY) {
        m_u = mt;  // no visible key so far: O is still exactly 0
      } else if (mt > m_prev + kRescaleThreshold) {
        m_u = mt;
        rescale = true;
      }
      if (u + 1 < u_first + nu) {  // publish it for step u+1 (the other group)
        m_x[u & 1][row] = m_u;
        asm volatile("bar.arrive %0, 64;" ::"r"(kBarMx0 + 2 * wq + (u & 1)) : "memory");
      }
      if (__any_sync(0xffffffffu, rescale)) {
        // O holds PV(u-1) once it completes; scale the rows whose reference moved
        const float alpha = rescale ? fast_exp2(m_prev - m_u) : 1.f;
        mbar_wait_warp(smem_u32(&bars.p_free[(u - 1) & 1]), ((u - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          float r[32];
          tmem_ld32_f(ocol + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] *= alpha;
          tmem_st32(ocol + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r));
        }
      }
      if (m_u != m_seen) {  // this group's partial sum follows the reference
        l = m_seen == -INFINITY ? 0.f : l * fast_exp2(m_seen - m_u);
        m_seen = m_u;
      }
      const float nm = m_u == -INFINITY ? 0.f : -m_u;
      const uint64_t nm2 = f2pk(nm, nm);
      uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
      uint32_t pk[64];
#pragma unroll
      for (int c = 0; c < 64; ++c) {  // pair index: columns 2c, 2c+1
        const uint64_t y = ffma2(f2pk(x[2 * c], x[2 * c + 1]), sl2, nm2);
        float ya, yb, ea, eb;
        f2upk(y, ya, yb);
        if (c % kPolyEvery == kPolyEvery - 1) {
          exp2_poly2(ya, yb, ea, eb);
        } else {
          ea = fast_exp2(ya);
          eb = fast_exp2(yb);
        }
        acc[c & 3] = fadd2(acc[c & 3], f2pk(ea, eb));
        pk[c] = pack_bf16x2(ea, eb);
      }
      // P buffer grp is free once PV(u-2) has read it
      if (wq == 0) PPTR(1 + grp, 44)
      if (u >= 2) mbar_wait_warp(smem_u32(&bars.p_free[grp]), ((u >> 1) - 1) & 1);
      if (wq == 0) PPTR(1 + grp, 45)
      tc_fence_after();
      tmem_st32(pcol, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
      tmem_st32(pcol + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars.p_full[grp]));
      if (wq == 0) PPTR(1 + grp, 41)
      float s0, s1;
      f2upk(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])), s0, s1);
      l += s0 + s1;
      ++u;
    }
    // epilogue (group 0): merge the two partial sums at the final reference, O / l -> bf16, lse
    // hand-over slot (one per row): group 1 refills it only after group 0 has read it
    if (grp == 1) {
      if (ic > 0) mbar_wait_warp(smem_u32(&bars.ml_empty[wq]), (ic - 1) & 1);
      ml_x[row] = make_float2(m_seen, l);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars.ml_full[wq]));
      ++ic;
      continue;
    }
    mbar_wait_warp(smem_u32(&bars.ml_full[wq]), ic & 1);
    const float2 mlb = ml_x[row];
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars.ml_empty[wq]));
    const float mb = mlb.x, lb = mlb.y;
    const float m_fin = fmaxf(m_seen, mb);
    float lt = 0.f;
    if (m_seen != -INFINITY) lt += l * fast_exp2(m_seen - m_fin);
    if (mb != -INFINITY) lt += lb * fast_exp2(mb - m_fin);
    mbar_wait_warp(smem_u32(&bars.o_full), ic & 1);
    ++ic;
    tc_fence_after();
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    const bool store = i <= ti1;
    __nv_bfloat16 *orow =
        static_cast<__nv_bfloat16 *>(p.o) + ((int64_t)it.b * p.N + i) * p.o_row_stride + (int64_t)it.h * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; c += 2) {
      float r[32], r2[32];
      tmem_ld32_f(ocol + c * 32, r);
      tmem_ld32_f(ocol + (c + 1) * 32, r2);
      tmem_wait_ld();
      if (store) {
        store_o_chunk32(orow + c * 32, r, inv, p.o_v8);
        store_o_chunk32(orow + (c + 1) * 32, r2, inv, p.o_v8);
      }
    }
    if (p.lse && store)
      p.lse[((int64_t)it.b * p.nql + it.h) * p.N + i] = lt > 0.f ? (m_fin + __log2f(lt)) * kLn2 : -INFINITY;
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars.o_empty));
  }
}

template <int D>
__global__ void __launch_bounds__(kCThreads, 1)
    prefill_cl_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kh,
                      const __grid_constant__ CUtensorMap tm_vh, const __grid_constant__ CUtensorMap tm_kc16,
                      const __grid_constant__ CUtensorMap tm_vc16, const __grid_constant__ CUtensorMap tm_kc1,
                      const __grid_constant__ CUtensorMap tm_vc1, const PpParams p) {
  using C = PCfg<D>;
  using CC = CCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ CBars bars;
  __shared__ float m_x[2][kM];  // softmax groups: reference exchange (step parity)
  __shared__ float2 ml_x[kM];   // epilogue hand-over of group 1's (reference, partial sum)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t smem_base = smem_u32(smem_raw);
  if (smem_base & 1023u) __trap();
  const uint32_t q_smem = smem_base;                         // Q buffers (item parity)
  const uint32_t k_smem = q_smem + CC::kQ * C::kTileBytes;   // kNK tiles
  const uint32_t v_smem = k_smem + CC::kNK * C::kTileBytes;  // kNV tiles
  const int total = p.n_items * p.batch;
  const int rank = (int)cluster_ctarank(), cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const uint32_t peer = (uint32_t)(rank ^ 1);

  if (tid == 0) {
    for (int j = 0; j < 2; ++j) {
      mbar_init(smem_u32(&bars.q_full[j]), 1);
      mbar_init(smem_u32(&bars.q_empty[j]), 1);
      mbar_init(smem_u32(&bars.s_full[j]), 1);
      mbar_init(smem_u32(&bars.s_free[j]), 4);  // the 4 warps of the group owning buffer j
      mbar_init(smem_u32(&bars.p_full[j]), 4);
      mbar_init(smem_u32(&bars.p_free[j]), 1);
    }
    mbar_init(smem_u32(&bars.o_full), 1);
    mbar_init(smem_u32(&bars.o_empty), 4);
    for (int w = 0; w < 4; ++w) {
      mbar_init(smem_u32(&bars.ml_full[w]), 1);
      mbar_init(smem_u32(&bars.ml_empty[w]), 1);
    }
    for (int s = 0; s < CC::kNK; ++s) {
      mbar_init(smem_u32(&bars.k_full[s]), 1);
      mbar_init(smem_u32(&bars.k_empty[s]), 2);  // one commit from each CTA's MMA warp
      mbar_init(smem_u32(&bars.k_copied[s]), 1);
      mbar_init(smem_u32(&bars.k_issued[s]), 1);
    }
    for (int s = 0; s < CC::kNV; ++s) {
      mbar_init(smem_u32(&bars.v_full[s]), 1);
      mbar_init(smem_u32(&bars.v_empty[s]), 2);
      mbar_init(smem_u32(&bars.v_copied[s]), 1);
      mbar_init(smem_u32(&bars.v_issued[s]), 1);
    }
    fence_mbar_init();
  }
  if (warp == kCWarpMMA) tmem_alloc<kTmemCols>(smem_u32(&bars.tmem_base));
  if (warp == kCWarpKV && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kh);
    tma_prefetch_desc(&tm_vh);
  }
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers exist before any multicast or remote arrive
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp < 8) {
#ifndef MOA_CL_NOREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(MOA_CL_REG_SOFTMAX) : "memory");
#endif
    cl_softmax_role<D>(p, bars, tmem, total, rank, cid, ncl, warp, lane, m_x, ml_x);
  } else {
#ifndef MOA_CL_NOREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(MOA_CL_REG_OTHER) : "memory");
#endif
  if (warp == kCWarpKV) {
    // K and V producer (one thread, two independent cursors over the union steps): this CTA's
    // halves of each step's K and V tiles.  A V slot is freed only by PV(T - kNV), i.e. after the
    // softmax of that step, while K runs kNK steps ahead of S; one blocking loop would hold the
    // next K tile behind the V slot, so each cursor issues as soon as its own slot is free.
    if (lane == 0) {
      struct Cur {
        int idx, k, ns, T;
        PItem it;
        int g, Wg;
        bool fi;
      };
      auto load = [&](Cur &c) {
        c.it = get_pitem<-1, false>(p, c.idx);
        c.ns = c.it.bt.steps();
        c.g = c.it.h / p.G;
        c.fi = fill_item(p, c.it);
        c.Wg = c.fi ? p.win_g[c.g] : 0;
      };
      auto settle = [&](Cur &c) {  // move to the next step some q tile uses (or past the end)
        while (c.idx < total) {
          for (; c.k < c.ns; ++c.k) {
            int t;
            bool u0, u1;
            step_use(c.it.bt, c.k, t, u0, u1);
            if (u0 || u1) return;
          }
          c.idx += ncl;
          c.k = 0;
          if (c.idx < total) load(c);
        }
      };
      Cur kc, vc;
      kc.idx = vc.idx = cid;
      kc.k = vc.k = 0;
      kc.T = vc.T = 0;
      if (cid < total) {
        load(kc);
        load(vc);
      }
      settle(kc);
      settle(vc);
      uint32_t kfill = 0, vfill = 0, kcph = 0, vcph = 0;  // per slot: holds a filler tile / copied parity
      while (kc.idx < total || vc.idx < total) {
        bool did = false;
        if (kc.idx < total) {
          const int T = kc.T, ks = T % CC::kNK;
          bool ok = T < CC::kNK || mbar_test(smem_u32(&bars.k_empty[ks]), ((T - CC::kNK) / CC::kNK) & 1);
          // the filler CTA's stores still read the previous (filler) tile of this slot
          if (ok && (kfill >> ks & 1)) {
            ok = mbar_test(smem_u32(&bars.k_copied[ks]), kcph >> ks & 1);
            if (ok) kcph ^= 1u << ks;
          }
          if (ok) {
            const int t = kc.it.bt.at(kc.k);
            const bool ft = kc.fi && fill_tile(p, kc.it.i0, kc.it.N, kc.Wg, t);  // some CTA stores it
            kfill = (kfill & ~(1u << ks)) | ((uint32_t)ft << ks);
            const uint32_t kbar = smem_u32(&bars.k_full[ks]);
            mbar_expect_tx(kbar, C::kTileBytes);  // both halves
            for (int sl = 0; sl < C::kSlabs; ++sl)
              tma_load_4d_mc(k_smem + ks * C::kTileBytes + sl * C::kSlabBytes + rank * 64 * 128, &tm_kh, kbar, sl * 64,
                             kc.g, t * kN + 64 * rank, kc.it.b, 3);
            if (ft && fill_rank(kc.it, t) == rank) mbar_arrive(smem_u32(&bars.k_issued[ks]));
            ++kc.T;
            ++kc.k;
            settle(kc);
            did = true;
          }
        }
        if (vc.idx < total) {
          const int T = vc.T, vs = T % CC::kNV;
          bool ok = T < CC::kNV || mbar_test(smem_u32(&bars.v_empty[vs]), ((T - CC::kNV) / CC::kNV) & 1);
          if (ok && (vfill >> vs & 1)) {
            ok = mbar_test(smem_u32(&bars.v_copied[vs]), vcph >> vs & 1);
            if (ok) vcph ^= 1u << vs;
          }
          if (ok) {
            const int t = vc.it.bt.at(vc.k);
            const bool ft = vc.fi && fill_tile(p, vc.it.i0, vc.it.N, vc.Wg, t);
            vfill = (vfill & ~(1u << vs)) | ((uint32_t)ft << vs);
            const uint32_t vbar = smem_u32(&bars.v_full[vs]);
            mbar_expect_tx(vbar, C::kTileBytes);
            for (int sl = 0; sl < C::kSlabs; ++sl)
              tma_load_4d_mc(v_smem + vs * C::kTileBytes + sl * C::kSlabBytes + rank * 64 * 128, &tm_vh, vbar, sl * 64,
                             vc.g, t * kN + 64 * rank, vc.it.b, 3);
            if (ft && fill_rank(vc.it, t) == rank) mbar_arrive(smem_u32(&bars.v_issued[vs]));
            ++vc.T;
            ++vc.k;
            settle(vc);
            did = true;
          }
        }
        if (!did) __nanosleep(20);
      }
    }
  } else if (warp == kCWarpQ) {
    if (lane == 0) {
      int ic = 0, T = 0;
      uint32_t kiph = 0, viph = 0;
      for (int idx = cid; idx < total; idx += ncl) {
        const PItem it = get_pitem<-1, false>(p, idx);
        if (rank == 0 || it.bt.has1) {
          const int qb = ic % CC::kQ;
          if (ic >= CC::kQ) mbar_wait(smem_u32(&bars.q_empty[qb]), (ic / CC::kQ - 1) & 1);
          ++ic;
          const uint32_t qbar = smem_u32(&bars.q_full[qb]);
          mbar_expect_tx(qbar, C::kTileBytes);
          for (int sl = 0; sl < C::kSlabs; ++sl)
            tma_load_4d(q_smem + qb * C::kTileBytes + sl * C::kSlabBytes, &tm_q, qbar, sl * 64, it.h,
                        (int)(it.i0 + rank * kM), it.b);
        }
        if (idx + ncl < total) {  // warm L2 with the next item's Q tile
          const PItem nx = get_pitem<-1, false>(p, idx + ncl);
          if (rank == 0 || nx.bt.has1)
            for (int sl = 0; sl < C::kSlabs; ++sl)
              tma_prefetch_4d(&tm_q, sl * 64, nx.h, (int)(nx.i0 + rank * kM), nx.b);
        }
        // fused cache fill of the tiles on this CTA's diagonal (as in the two-tile kernel; the
        // copied-barriers are arrived in BOTH CTAs, whose producers both refill the slot)
        const int ns = it.bt.steps();
        const bool fi = p.fill && fill_item(p, it);
        if (!fi) {
          for (int k = 0; k < ns; ++k) {
            int t;
            bool u0, u1;
            step_use(it.bt, k, t, u0, u1);
            T += (u0 || u1);
          }
          continue;
        }
        const int g = it.h / p.G;
        const int Wg = p.win_g[g];
        const int64_t region = (int64_t)it.b * p.rows_per_seq + p.g_off[g];
        uint32_t pend[4];
        int np_ = 0;
        for (int k = 0; k < ns; ++k) {
          int t;
          bool u0, u1;
          step_use(it.bt, k, t, u0, u1);
          if (!u0 && !u1) continue;
          if (fill_tile(p, it.i0, it.N, Wg, t) && fill_rank(it, t) == rank) {
            const int ks = T % CC::kNK, vs = T % CC::kNV;
            mbar_wait(smem_u32(&bars.k_issued[ks]), kiph >> ks & 1);
            kiph ^= 1u << ks;
            mbar_wait(smem_u32(&bars.k_full[ks]), (T / CC::kNK) & 1);
            fill_store<D>(p, k_smem + ks * C::kTileBytes, &tm_kc16, &tm_kc1, region, it.N, Wg, t);
            mbar_wait(smem_u32(&bars.v_issued[vs]), viph >> vs & 1);
            viph ^= 1u << vs;
            mbar_wait(smem_u32(&bars.v_full[vs]), (T / CC::kNV) & 1);
            fill_store<D>(p, v_smem + vs * C::kTileBytes, &tm_vc16, &tm_vc1, region, it.N, Wg, t);
            pend[np_++] = smem_u32(&bars.k_copied[ks]);
            pend[np_++] = smem_u32(&bars.v_copied[vs]);
          }
          ++T;
        }
        if (np_) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          for (int q = 0; q < np_; ++q) {
            mbar_arrive(pend[q]);
            mbar_arrive_cluster(mapa_shared(pend[q], peer));
          }
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // cache writes complete
    }
  } else if (warp == kCWarpMMA) {
    cl_mma_s_role<D>(p, bars, tmem, q_smem, k_smem, total, rank, cid, ncl);
  } else if (warp == kCWarpPV) {
    cl_mma_pv_role<D>(p, bars, tmem, v_smem, total, rank, cid, ncl);
  }
  }

  __syncwarp();  // producer lanes 1-31 wait for lane 0: the cluster barrier is warp-aligned
  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still multicast into it or arrive on it
  if (warp == kCWarpMMA) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

int num_sms_pp() { return device_sm_count(); }
// MOA_PP_CLUSTER=1 routes the uniform token-mask prefill to the clustered kernel (an
// experiment: parity-green, ~15 % slower than the two-tile kernel on C2/C4)
bool two_tile_pp() {
  const char *e = getenv("MOA_PP_CLUSTER");  // read per launch (host only): tests switch it
  return !(e && e[0] == '1');
}

template <int D>
int launch_pp(const PrefillArgs &a, void *stream) {
  using C = PCfg<D>;
  alignas(64) CUtensorMap mq, mk, mv;
  const int ngl = a.nql / a.G;
  if (!make_tile_map(&mq, a.q, D, a.nql, a.N, a.batch, a.q_row_stride, kM) ||
      !make_tile_map(&mk, a.k, D, ngl, a.N, a.batch, a.kv_row_stride, kN) ||
      !make_tile_map(&mv, a.v, D, ngl, a.N, a.batch, a.kv_row_stride, kN))
    return (int)cudaErrorInvalidValue;
  static const CUtensorMap zero_map{};
  const CUtensorMap *mk16 = a.fill ? static_cast<const CUtensorMap *>(a.kmap16) : &zero_map;
  const CUtensorMap *mv16 = a.fill ? static_cast<const CUtensorMap *>(a.vmap16) : &zero_map;
  const CUtensorMap *mk1 = a.fill ? static_cast<const CUtensorMap *>(a.kmap1) : &zero_map;
  const CUtensorMap *mv1 = a.fill ? static_cast<const CUtensorMap *>(a.vmap1) : &zero_map;
  PpParams p;
  p.o = a.o;
  p.lse = a.lse;
  p.o_row_stride = a.o_row_stride;
  p.N = a.N;
  p.batch = a.batch;
  p.n_items = a.d_seq_n ? a.n_items_rag : a.n_items2;
  p.nql = a.nql;
  p.G = a.G;
  p.n_sink = a.n_sink;
  p.bshift = a.bshift;
  p.scale_log2 = a.scale * kLog2e;
  p.win_q = a.d_win_q;
  p.seq_n = a.d_seq_n;
  p.o_v8 = (((uintptr_t)a.o | (uintptr_t)(a.o_row_stride * 2)) & 31) == 0;
  p.win_bq = a.d_win_bq;
  p.items = a.d_seq_n ? a.d_items_rag : a.d_items2;
  p.fill = a.fill;
  p.kc = static_cast<__nv_bfloat16 *>(a.k_cache);
  p.vc = static_cast<__nv_bfloat16 *>(a.v_cache);
  p.rows_per_seq = a.rows_per_seq;
  p.g_off = a.d_g_off;
  p.win_g = a.d_win_g;
  p.fill_h = a.d_fill_h;
  // the token mask (bshift < 0) and the block mask are separate instantiations, so the
  // token path carries no block-mode arithmetic
  const bool rag = p.seq_n != nullptr;
  p.sched = a.d_sched2;  // uniform or ragged per-CTA schedule (null: round robin)
  p.sched_off = a.d_sched2_off;
  if (!rag && p.bshift < 0 && !two_tile_pp()) {
    p.sched = p.sched_off = nullptr;  // the clustered kernel walks the item list per cluster
    // uniform token mask: the clustered kernel (a pair of SMs per 256-row item)
    alignas(64) CUtensorMap mkh, mvh;
    if (!make_tile_map(&mkh, a.k, D, ngl, a.N, a.batch, a.kv_row_stride, kN / 2) ||
        !make_tile_map(&mvh, a.v, D, ngl, a.N, a.batch, a.kv_row_stride, kN / 2))
      return (int)cudaErrorInvalidValue;
    auto ck = prefill_cl_kernel<D>;
    cudaError_t e = cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, CCfg<D>::kSmemBytes);
    if (e != cudaSuccess) return (int)e;
    const int total = p.n_items * p.batch;
    const int ncl = total < num_sms_pp() / 2 ? total : num_sms_pp() / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * ncl);
    cfg.blockDim = dim3(kCThreads);
    cfg.dynamicSmemBytes = CCfg<D>::kSmemBytes;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, ck, mq, mkh, mvh, *mk16, *mv16, *mk1, *mv1, p);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
  }
  auto kern = p.bshift < 0    ? (rag ? prefill_pp_kernel<D, -1, true> : prefill_pp_kernel<D, -1, false>)
              : p.bshift == 6 ? (rag ? prefill_pp_kernel<D, 6, true> : prefill_pp_kernel<D, 6, false>)
                              : (rag ? prefill_pp_kernel<D, kBsRuntime, true>
                                     : prefill_pp_kernel<D, kBsRuntime, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  if (e != cudaSuccess) return (int)e;
  const int total = rag ? p.n_items : p.n_items * p.batch;
  const int grid = p.sched ? a.sched2_ctas : (total < num_sms_pp() ? total : num_sms_pp());
  kern<<<grid, kThreads, C::kSmemBytes, (cudaStream_t)stream>>>(mq, mk, mv, *mk16, *mv16, *mk1, *mv1, p);
  return (int)cudaGetLastError();
}

}  // namespace

#ifdef MOA_PP_DIAG_TRACE
extern "C" int moa_debug_pp_trace(unsigned long long *out, int *counts) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_pp_trace, sizeof(g_pp_trace));
  cudaMemcpyFromSymbol(counts, g_pp_trace_n, sizeof(g_pp_trace_n));
  static const int z[4] = {};
  cudaMemcpyToSymbol(g_pp_trace_n, z, sizeof(z));
  return 0;
}
#endif

int launch_prefill_bf16_pp(const PrefillArgs &a, void *stream) {
  if (a.d == 128) return launch_pp<128>(a, stream);
  return launch_pp<64>(a, stream);
}

}  // namespace moa
