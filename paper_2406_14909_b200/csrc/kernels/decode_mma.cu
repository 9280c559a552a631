// decode_mma.cu -- bf16 MoA decode over the compact ring cache on B200
// (SURVEY §8(a) a7 split-KV + a8 combine [+ a6 append fused]).
//
// One query token per sequence at position `pos` attends over its kv-group's
// cache region (sinks + ring; PAPER.md:704 fixed span, oldest entry
// replaced).  q-head h masks ring rows older than its own window W_h
// (reading c10), so one pass over a group's rows serves its G heads.
//
// HBM-bound design:
//  * Balanced split: the layer cache is one contiguous row space
//    [b][g][s + W_g rows]; CTA c streams rows [c*R/n, (c+1)*R/n) -- every CTA
//    moves the same number of bytes whatever the per-head spans are.  A CTA
//    range is cut into segments at region (b, g) boundaries; each segment
//    yields one partial (m, l, o) per consumer warp.
//  * A producer warp streams 64-row K/V tiles with TMA (cp.async.bulk.tensor,
//    128B swizzle) into a 3-stage shared-memory ring (mbarrier full/empty).
//  * 4 consumer warps, 16 keys each per tile, compute S = Q K^T and O += P V
//    with mma.sync m16n8k16 (bf16 in, fp32 accumulate): the G heads of the
//    group are the M rows (zero-padded to 16), keys the N columns, so K/V
//    bytes are read once for all heads and the instruction count per row is
//    independent of G.  Online softmax in base 2 with a lazy running max.
//  * An epilogue warp keeps the consumers free of latency: it stages each
//    segment's q rows in shared memory two segments ahead, takes the region's
//    ticket (atomic, self-resetting) when the consumers finish a segment, and,
//    if this CTA contributed last, merges the region's partials by LSE and
//    writes o (and lse) while the consumers stream the next segment.
//  * Fused append: the cache row of `pos` is masked in the tile path; the CTA
//    owning it folds (k_new, v_new) into its state and writes it to the cache.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "../moa_internal.h"
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace moa {
namespace {

using namespace ptx;

#ifdef MOA_DEC_TRACE
// diagnostic build only (tools/build_trace.sh): per-CTA %globaltimer stamps of two consecutive launches
constexpr int kTraceCtas = 1024, kTraceFields = 8;
__device__ unsigned long long g_trace[2][kTraceCtas][kTraceFields];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(f) \
  if (blockIdx.x < kTraceCtas) g_trace[p.trace_slot][blockIdx.x][f] = gtime()
#define TRACE_V(f, v) \
  if (blockIdx.x < kTraceCtas) g_trace[p.trace_slot][blockIdx.x][f] = (v)
#else
#define TRACE(f)
#define TRACE_V(f, v)
#endif

constexpr int kCW = 4;                      // consumer warps
constexpr int kProd = kCW;                  // producer warp (TMA)
constexpr int kEpi = kCW + 1;               // epilogue warp (q staging, tickets, combines)
constexpr int kThreads = (kCW + 2) * 32;
constexpr int kRows = 16 * kCW;             // rows per tile
constexpr int kCtasPerSm = 2;
constexpr float kRescale = 8.0f;

template <int D>
constexpr int part_stride() { return D + 4; }  // per-head partial: o[D], lse2, pad (16-B aligned)
template <int D>
constexpr int q_stride() { return D + 8; }     // staged q row (padding spreads the fragment reads over banks)

template <int D, int STAGES>
struct DCfg {
  static constexpr int kSlabs = D / 64;
  static constexpr int kSlabBytes = kRows * 128;
  static constexpr int kTileBytes = kRows * D * 2;            // K or V
  static constexpr int kStages = STAGES;
  static constexpr int kSmem = kStages * 2 * kTileBytes + 1024;
};

struct MParams {
  const __nv_bfloat16 *q;
  __nv_bfloat16 *o;
  int64_t q_bs, o_bs;
  const __nv_bfloat16 *k_new, *v_new;
  int64_t kv_bs;
  __nv_bfloat16 *kc, *vc;
  int64_t rows_per_seq, R;       // rows per sequence, total rows
  int64_t seg_cost, ctot;        // CTA split: a segment costs seg_cost rows; total cost
  int chunk;                     // rank-invariant split: rows per chunk (0: balanced row split)
  const int *gc_off;             // chunk mode: first chunk of each local group in a sequence [ngl + 1]
  const int64_t *g_off;
  const int32_t *win_g, *win_q;
  int ngl, G, n_sink, batch;
  int64_t pos;
  const int64_t *pos_b;   // ragged: per-sequence positions (null: pos); < 0 = inactive
  const int32_t *win_bq;  // ragged: per-sequence windows [batch, ngl * G] (null: win_q)
  float scale_log2;
  float *lse;
  float *part;
  int *counters;
  int early;  // 1: the producer may stream the cache before the stream predecessor completes
  // fused head-output all-gather (moa_set_peer_outputs; n_peers = 0: off)
  const PeerOut *peers;
  int n_peers, peer_head0, layer;
  int64_t peer_bs, peer_ls;
  // cross-layer launch (ML kernels only): per-layer tables and per-call layer strides
  const DecodeLayerDesc *ml;
  int nl;
  int64_t q_ls, o_ls, kvn_ls, lse_ls, part_ls;
#ifdef MOA_DEC_TRACE
  int trace_slot;
#endif
};

// Work split (balanced by cost, not rows): row x of region r (regions in (b, g) row order) sits
// at cost position C(x) = x + seg_cost * r, C_tot = R + seg_cost * (regions - 1); CTA c takes
// the rows with ceil(c C_tot / n) <= C(x) < ceil((c+1) C_tot / n).  A CTA whose range
// crosses region boundaries thus gets seg_cost fewer rows per extra segment (each segment
// costs it a q stage, a partial tile and a partial write), and cuts that fall in the jump
// between two regions land on the region boundary.
__device__ __forceinline__ int64_t region_start(const MParams &p, const int64_t *g_off, int r) {
  const int b = r / p.ngl, g = r - b * p.ngl;
  return (int64_t)b * p.rows_per_seq + g_off[g];
}
// smallest row x with C(x) >= T
__device__ __forceinline__ int64_t cut_row(const MParams &p, const int64_t *g_off, int64_t T) {
  const int nreg = p.batch * p.ngl;
  int lo = 0, hi = nreg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (region_start(p, g_off, mid) + p.seg_cost * mid <= T)
      lo = mid;
    else
      hi = mid - 1;
  }
  const int64_t st = region_start(p, g_off, lo);
  const int64_t en = lo + 1 < nreg ? region_start(p, g_off, lo + 1) : p.R;
  const int64_t x = st + (T - (st + p.seg_cost * lo));
  return x < en ? x : en;
}
// the CTA whose range holds row x of region r
__device__ __forceinline__ int64_t cta_of(const MParams &p, int64_t x, int r) {
  return ((x + p.seg_cost * r) * (int64_t)gridDim.x) / p.ctot;
}

// a / b for a >= 0, b > 0: the 32-bit divide (a short instruction sequence) whenever both fit,
// which is every config here; 64-bit division is a long dependent subroutine
__device__ __forceinline__ int64_t udiv(int64_t a, int64_t b) {
  return ((uint64_t)a | (uint64_t)b) >> 32 ? a / b : (int64_t)((uint32_t)a / (uint32_t)b);
}

struct Region {
  int b, g, Wg;
  int64_t start, end;  // absolute rows [start, end)
};

// Rank-invariant split (p.chunk > 0): region (b, g) is cut into chunks of p.chunk rows from
// its first row, whatever the batch, the SM count or the other regions are; a chunk is one
// segment with its own partial slot, so the arithmetic on a region's rows (tile boundaries,
// warp row sets, online-softmax order, partial and combine order) depends only on the region
// -- a kv-group shard on another GPU computes bit-identical outputs (SURVEY §4 tier 4).
// CTAs take contiguous chunk ranges balanced by cost (rows + seg_cost per chunk).
// s_gc[g] = first chunk of group g inside one sequence, s_gc[ngl] = chunks per sequence.
__device__ __forceinline__ int64_t chunk_row(const MParams &p, const int64_t *g_off, const int *gc, int64_t J) {
  const int cps = gc[p.ngl];
  const int64_t b = udiv(J, cps);
  if (b >= p.batch) return p.R;
  const int jj = (int)(J - b * cps);
  int lo = 0, hi = p.ngl - 1;  // last g with gc[g] <= jj
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (gc[mid] <= jj) lo = mid; else hi = mid - 1;
  }
  return b * p.rows_per_seq + g_off[lo] + (int64_t)(jj - gc[lo]) * p.chunk;
}
// first chunk J with cost prefix rows(J) + seg_cost * J >= T.  Sequences share one layout, so
// the sequence is one division; inside it the group is a binary search over the group starts
// and the chunk one more division (chunks of a group before its last are full).  Every thread
// evaluates this before the kernel's first wait: it must stay a few hundred instructions.
__device__ __forceinline__ int64_t chunk_cut(const MParams &p, const int64_t *g_off, const int *gc, int64_t T) {
  const int cps = gc[p.ngl];
  const int64_t seq_cost = p.rows_per_seq + p.seg_cost * cps;
  const int64_t b = udiv(T, seq_cost);
  if (b >= p.batch) return (int64_t)p.batch * cps;
  const int64_t r = T - b * seq_cost;
  if (r == 0) return b * cps;
  int lo = 0, hi = p.ngl - 1;  // last g whose first chunk starts at cost < r
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (g_off[mid] + p.seg_cost * gc[mid] < r) lo = mid; else hi = mid - 1;
  }
  const int64_t gp = g_off[lo] + p.seg_cost * gc[lo];
  const int64_t step = p.chunk + p.seg_cost;
  const int64_t k = udiv(r - gp + step - 1, step);
  const int nc = gc[lo + 1] - gc[lo];
  return b * cps + (k >= nc ? gc[lo + 1] : gc[lo] + k);
}

constexpr int kMaxGroups = 128;

// region (b, g) holding absolute row x; g_off / win_g are staged in shared memory
__device__ __forceinline__ Region region_of(const MParams &p, const int64_t *g_off, const int *win_g, int64_t x) {
  Region r;
  r.b = (int)udiv(x, p.rows_per_seq);
  const int64_t within = x - (int64_t)r.b * p.rows_per_seq;
  int lo = 0, hi = p.ngl - 1;  // last g with g_off[g] <= within
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (g_off[mid] <= within) lo = mid; else hi = mid - 1;
  }
  r.g = lo;
  r.Wg = win_g[lo];
  r.start = (int64_t)r.b * p.rows_per_seq + g_off[lo];
  r.end = r.start + p.n_sink + r.Wg;
  return r;
}

// end of the segment starting at row x of region r (the CTA range ends at X1)
__device__ __forceinline__ int64_t seg_end_of(const MParams &p, const Region &r, int64_t x, int64_t X1) {
  int64_t e = r.end < X1 ? r.end : X1;
  if (p.chunk && x + p.chunk < e) e = x + p.chunk;  // x is a chunk boundary in chunk mode
  return e;
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *m, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// Consumer <-> epilogue hand-offs use named barriers (arrive by the producing side, sync by
// the consuming side), one per parity of the segment index: q_full (epilogue staged q of a
// segment) and seg_done (consumers wrote their partials of a segment).  A side reuses a
// barrier id two segments later only after a hand-off in the other direction, so phases
// never overlap.
constexpr int kBarQFull = 1, kBarSegDone = 3;  // ids 1,2 and 3,4 (0 is __syncthreads)
constexpr int kBarMl = 5;                      // cross-layer table (consumers + epilogue)
constexpr int kHandoff = (kCW + 1) * 32;       // consumers + epilogue warp
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  __syncwarp();
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  __syncwarp();
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Merge the partials of region ridx by LSE, one warp: one slot per CTA whose range touched
// the region.  Lane l owns output elements l, l+32, ...;
// the slot LSEs and partial vectors are read in batches of 8 independent loads, so the
// merge costs ~ceil(slots/8) L2 round trips per head.
template <int D>
__device__ __forceinline__ void combine_region_warp(const MParams &p, const int64_t *g_off, const int *win_g,
                                                    const int *gc, int ridx, int lane) {
  constexpr int PS = part_stride<D>();
  constexpr int NE = D / 32;
  constexpr int KB = 8;
  const int b = ridx / p.ngl, g = ridx - b * p.ngl;
  const int G = p.G;
  const int64_t start = (int64_t)b * p.rows_per_seq + g_off[g];
  const int64_t end = start + p.n_sink + win_g[g];
  int64_t sl0;
  int nsl;
  if (p.chunk) {
    sl0 = (int64_t)b * gc[p.ngl] + gc[g];
    nsl = gc[g + 1] - gc[g];
  } else {
    const int64_t c_first = cta_of(p, start, ridx), c_last = cta_of(p, end - 1, ridx);
    sl0 = c_first + ridx;
    nsl = (int)(c_last - c_first + 1);
  }
  for (int j = 0; j < G; ++j) {
    const float *base = p.part + (sl0 * G + j) * PS;
    float mx = -INFINITY, L = 0.f, O[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) O[i] = 0.f;
    for (int c0 = 0; c0 < nsl; c0 += KB) {
      float ls[KB], v[KB][NE];
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const bool in = c0 + k < nsl;
        const float *pc = base + (int64_t)(c0 + k) * G * PS;
        ls[k] = in ? __ldcg(pc + D) : -INFINITY;
#pragma unroll
        for (int i = 0; i < NE; ++i) v[k][i] = in ? __ldcg(pc + lane + 32 * i) : 0.f;
      }
      float cm = ls[0];
#pragma unroll
      for (int k = 1; k < KB; ++k) cm = fmaxf(cm, ls[k]);
      const float nm = fmaxf(mx, cm);
      if (nm == -INFINITY) continue;
      const float a = mx == -INFINITY ? 0.f : fast_exp2(mx - nm);
      L *= a;
#pragma unroll
      for (int i = 0; i < NE; ++i) O[i] *= a;
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const float w = ls[k] == -INFINITY ? 0.f : fast_exp2(ls[k] - nm);
        L += w;
#pragma unroll
        for (int i = 0; i < NE; ++i) O[i] = fmaf(w, v[k][i], O[i]);
      }
      mx = nm;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    __nv_bfloat16 ov[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) ov[i] = __float2bfloat16_rn(O[i] * inv);
    __nv_bfloat16 *ob = p.o + (int64_t)b * p.o_bs + (int64_t)(g * G + j) * D;
#pragma unroll
    for (int i = 0; i < NE; ++i) ob[lane + 32 * i] = ov[i];
    // fused head-output all-gather (moa_set_peer_outputs): the same bits into every
    // destination's [B, Hq, d] buffer of this layer, at this context's global head offset
    for (int k = 0; k < p.n_peers; ++k) {
      __nv_bfloat16 *pb = static_cast<__nv_bfloat16 *>(p.peers[k].o) + (int64_t)p.layer * p.peer_ls +
                          (int64_t)b * p.peer_bs + (int64_t)(p.peer_head0 + g * G + j) * D;
#pragma unroll
      for (int i = 0; i < NE; ++i) pb[lane + 32 * i] = ov[i];
    }
    if (p.lse && lane == 0) p.lse[(int64_t)b * p.ngl * G + g * G + j] = L > 0.f ? (mx + __log2f(L)) * kLn2 : -INFINITY;
  }
  if (p.n_peers) {
    // release: every lane's stores of this region, then one arrival on each destination's
    // counter of this layer (a consumer waits with moa_wait_flag)
    __threadfence_system();
    __syncwarp();
    if (lane == 0) {
      __threadfence_system();
      for (int k = 0; k < p.n_peers; ++k) atomicAdd_system(p.peers[k].flag + p.layer, 1u);
    }
  }
}

// ---- cross-layer launch support (ML = true): each warp role walks the layers of the launch
// in order with its own view of the current layer's parameters in shared memory (built by
// one lane from the launch parameters + the layer's DecodeLayerDesc), so roles that run
// ahead (the producer, the epilogue's q staging) never wait for the others at a layer
// boundary.  The single-layer kernel (ML = false) reads the kernel parameters and the
// shared-memory tables directly, as before.
struct Tabs {
  const int64_t *goff;
  const int *wing;
  const int *gc;
};

__device__ __forceinline__ void cta_range(const MParams &p, const Tabs &t, int64_t &X0, int64_t &X1) {
  const int64_t n_cta = gridDim.x;
  if (p.chunk) {
    const int64_t J0 = chunk_cut(p, t.goff, t.gc, ((int64_t)blockIdx.x * p.ctot + n_cta - 1) / n_cta);
    const int64_t J1 = chunk_cut(p, t.goff, t.gc, ((int64_t)(blockIdx.x + 1) * p.ctot + n_cta - 1) / n_cta);
    X0 = chunk_row(p, t.goff, t.gc, J0);
    X1 = chunk_row(p, t.goff, t.gc, J1);
  } else {
    X0 = cut_row(p, t.goff, ((int64_t)blockIdx.x * p.ctot + n_cta - 1) / n_cta);
    X1 = cut_row(p, t.goff, ((int64_t)(blockIdx.x + 1) * p.ctot + n_cta - 1) / n_cta);
  }
}

// view of layer l of a cross-layer launch (one thread writes it)
__device__ __forceinline__ void build_view(const MParams &b, int l, MParams *out) {
  const DecodeLayerDesc &dl = b.ml[l];
  MParams v = b;
  v.q = b.q + l * b.q_ls;
  v.o = b.o + l * b.o_ls;
  if (b.k_new) {
    v.k_new = b.k_new + l * b.kvn_ls;
    v.v_new = b.v_new + l * b.kvn_ls;
  }
  if (b.lse) v.lse = b.lse + l * b.lse_ls;
  v.part = b.part + l * b.part_ls;
  v.layer = b.layer + l;
  v.kc = static_cast<__nv_bfloat16 *>(dl.kc);
  v.vc = static_cast<__nv_bfloat16 *>(dl.vc);
  v.g_off = dl.g_off;
  v.win_g = dl.win_g;
  v.win_q = dl.win_q;
  v.gc_off = dl.gc_off;
  v.counters = dl.counters;
  v.rows_per_seq = dl.rows_per_seq;
  v.R = (int64_t)b.batch * dl.rows_per_seq;
  v.ctot = b.chunk ? v.R + b.seg_cost * (int64_t)b.batch * dl.dec_cps
                   : v.R + b.seg_cost * ((int64_t)b.batch * b.ngl - 1);
  *out = v;
}

// Per-CTA table of a cross-layer launch, computed once at kernel start (shared memory): the
// CTA's row range in every layer and the region holding its first row, so a role entering a
// layer needs no binary search over global tables (dependent L2 round trips).
constexpr int kMaxMl = 32;  // layers per cross-layer launch (the host splits longer ranges)
struct MlRange {
  int64_t X0, X1, start;  // CTA range; first row of the region holding X0
  int b, g, Wg, pad_;
};

// Enter the next layer (of this role) whose CTA range is not empty.  l = -1 before the first
// call.  whole_warp: every lane of the warp calls this (lane 0 builds the view).
template <bool ML>
__device__ __forceinline__ bool enter_layer(const MParams &p0, int &l, const MParams *&vp, Tabs &t, int64_t &X0,
                                            int64_t &X1, Region &first, MParams *slot, const Tabs &smem_tabs,
                                            const MlRange *rng, bool whole_warp) {
  first.end = -1;
  if constexpr (!ML) {
    if (l >= 0) return false;
    l = 0;
    vp = &p0;
    t = smem_tabs;
    cta_range(p0, t, X0, X1);
    return X0 < X1;
  } else {
    while (++l < p0.nl) {
      const MlRange &r = rng[l];
      if (r.X0 >= r.X1) continue;
      if (whole_warp) __syncwarp();  // every lane is done with the previous view
      if (!whole_warp || (threadIdx.x & 31) == 0) build_view(p0, l, slot);
      if (whole_warp) __syncwarp();
      vp = slot;
      t.goff = slot->g_off;
      t.wing = slot->win_g;
      t.gc = slot->gc_off;
      X0 = r.X0;
      X1 = r.X1;
      first.b = r.b;
      first.g = r.g;
      first.Wg = r.Wg;
      first.start = r.start;
      first.end = r.start + p0.n_sink + r.Wg;
      return true;
    }
    return false;
  }
}

// Region holding row x, the segment walk's next region (x == rg.end, or rg.end < 0 at the
// start of a layer).  ML: regions of a layer are consecutive in (b, g) order, so the next one
// starts at rg.end and needs only W_g of its group (one load, an L1 hit after the producer).
template <bool ML>
__device__ __forceinline__ Region region_at(const MParams &p, const Tabs &t, const Region &rg, const Region &first,
                                            int64_t x) {
  if constexpr (!ML) {
    return region_of(p, t.goff, t.wing, x);
  } else {
    if (rg.end < 0) return first;
    Region r;
    r.g = rg.g + 1;
    r.b = rg.b;
    if (r.g == p.ngl) {
      r.g = 0;
      ++r.b;
    }
    r.Wg = t.wing[r.g];
    r.start = rg.end;
    r.end = r.start + p.n_sink + r.Wg;
    return r;
  }
}

template <int D, int STAGES, int CPS, bool ML>
__global__ void __launch_bounds__(kThreads, CPS)
    decode_mma_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                      const __grid_constant__ CUtensorMap tm_k16, const __grid_constant__ CUtensorMap tm_v16,
                      const __grid_constant__ MParams p0) {
  using C = DCfg<D, STAGES>;
  constexpr int NT = D / 8;   // output n-tiles (8 dims each)
  constexpr int KS = D / 16;  // k-steps over the head dim
  constexpr int QS = q_stride<D>();
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full_bar[C::kStages], empty_bar[C::kStages];
  __shared__ int64_t s_goff[ML ? 1 : kMaxGroups];
  __shared__ int s_wing[ML ? 1 : kMaxGroups];
  __shared__ int s_gc[ML ? 1 : kMaxGroups + 1];
  __shared__ __align__(16) __nv_bfloat16 s_q[2][16 * QS];
  // per-role layer views (ML): consumers 0..kCW-1, producer, epilogue staging, epilogue merge
  __shared__ __align__(16) MParams s_view[ML ? kCW + 3 : 1];
  __shared__ MlRange s_rng[ML ? kMaxMl : 1];
  __shared__ uint64_t rng_bar;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  // per-warp partials of the two segments in flight: [2][kCW][G][D + 4] fp32 after the tiles
  float *s_part = reinterpret_cast<float *>(smem_raw + (base - smem_u32(smem_raw)) + C::kStages * 2 * C::kTileBytes);
  {
    const MParams &p = p0;
    if (tid == 0) TRACE(0);
  }

  if (tid == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), kCW);
    }
    mbar_init(smem_u32(&rng_bar), 1);
    fence_mbar_init();
  }
  if constexpr (!ML) {
    for (int g = tid; g < p0.ngl; g += kThreads) {
      s_goff[g] = p0.g_off[g];
      s_wing[g] = p0.win_g[g];
    }
    __syncthreads();
    if (p0.chunk)
      for (int g = tid; g <= p0.ngl; g += kThreads) s_gc[g] = p0.gc_off[g];
  }
  __syncthreads();
  const Tabs smem_tabs{s_goff, s_wing, s_gc};
  if constexpr (ML) {
    // this CTA's range and first region in every layer, computed by the consumer and
    // epilogue warps in parallel (two boundary cuts per layer, then the first region); the
    // producer waits for rng_bar before its first layer.  Overlaps the predecessor's tail.
    if (warp != kProd) {
      const int t = warp < kCW ? tid : tid - 32;  // 0 .. kHandoff-1
      for (int j = t; j < 2 * p0.nl; j += kHandoff) {
        MParams v;
        const int l = j >> 1;
        build_view(p0, l, &v);
        const Tabs tb{v.g_off, v.win_g, v.gc_off};
        const int64_t n_cta = gridDim.x, c = blockIdx.x + (j & 1);
        const int64_t T = (c * v.ctot + n_cta - 1) / n_cta;
        const int64_t X = v.chunk ? chunk_row(v, tb.goff, tb.gc, chunk_cut(v, tb.goff, tb.gc, T)) : cut_row(v, tb.goff, T);
        if (j & 1) s_rng[l].X1 = X; else s_rng[l].X0 = X;
      }
      named_bar_sync(kBarMl, kHandoff);
      for (int l = t; l < p0.nl; l += kHandoff) {
        MlRange &r = s_rng[l];
        if (r.X0 < r.X1) {
          MParams v;
          build_view(p0, l, &v);
          const Region rg = region_of(v, v.g_off, v.win_g, r.X0);
          r.b = rg.b;
          r.g = rg.g;
          r.Wg = rg.Wg;
          r.start = rg.start;
        }
      }
      named_bar_sync(kBarMl, kHandoff);
      if (t == 0) mbar_arrive(smem_u32(&rng_bar));
    }
  }
  if constexpr (!ML) {
    // Programmatic dependent launch.  Everything above overlapped the previous kernel's tail.
    // The consumers and the epilogue warp wait for the stream predecessor (q, k_new, the
    // workspace, the tickets and o may be its inputs/outputs) before they trigger the next
    // launch, so a CTA's trigger implies its predecessor completed: when this kernel starts,
    // every kernel before its predecessor has completed and flushed.  With p.early the host has
    // established that the predecessor does not write this layer's cache, so the producer
    // streams cache tiles at once.
    const MParams &p = p0;
    if (tid == 0) TRACE(1);
    int64_t X0, X1;
    cta_range(p0, smem_tabs, X0, X1);
    if (X0 >= X1) {
      griddep_wait();
      return;
    }
  }

  if (warp == kProd) {
    // ------------------------------------------------------------ producer: TMA K/V tiles
    if (lane == 0) {
      if constexpr (!ML) {
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
        tma_prefetch_desc(&tm_k16);
        tma_prefetch_desc(&tm_v16);
      }
      if (!p0.early) griddep_wait();
      if constexpr (ML) mbar_wait(smem_u32(&rng_bar), 0);
      {
        const MParams &p = p0;
        TRACE(2);
      }
      int T = 0;
      bool trig = false;
      int l = -1;
      const MParams *vp = nullptr;
      Tabs tb;
      int64_t X0, X1;
      Region first;
      while (enter_layer<ML>(p0, l, vp, tb, X0, X1, first, &s_view[ML ? kCW : 0], smem_tabs, s_rng, false)) {
        const MParams &p = *vp;
        const CUtensorMap *mk = &tm_k, *mv = &tm_v, *mk16 = &tm_k16, *mv16 = &tm_v16;
        if constexpr (ML) {
          const CUtensorMap *mm = static_cast<const CUtensorMap *>(p0.ml[l].maps);
          mk = mm;
          mv = mm + 1;
          mk16 = mm + 2;
          mv16 = mm + 3;
        }
        Region rg;
        rg.end = -1;
        for (int64_t x = X0; x < X1;) {
          if (x >= rg.end) rg = region_at<ML>(p, tb, rg, first, x);
          const int64_t seg_end = seg_end_of(p, rg, x, X1);
          for (int64_t t0 = x; t0 < seg_end; t0 += kRows, ++T) {
            const int st = T % C::kStages;
            if (T >= C::kStages) {
              mbar_wait(smem_u32(&empty_bar[st]), ((T - C::kStages) / C::kStages) & 1);
              if (!trig) {  // the consumers have passed their griddepcontrol.wait
                griddep_launch_dependents();
                trig = true;
              }
            }
            const uint32_t fb = smem_u32(&full_bar[st]);
            const uint32_t kd = base + st * 2 * C::kTileBytes, vd = kd + C::kTileBytes;
            const int64_t nrows = seg_end - t0;
            if (nrows >= kRows) {
              mbar_expect_tx(fb, 2 * C::kTileBytes);
              for (int sl = 0; sl < C::kSlabs; ++sl) {
                tma_load_2d(kd + sl * C::kSlabBytes, mk, fb, sl * 64, (int)t0);
                tma_load_2d(vd + sl * C::kSlabBytes, mv, fb, sl * 64, (int)t0);
              }
            } else {  // segment tail: only the 16-row groups that hold rows of the segment
              const int n16 = ((int)nrows + 15) >> 4;
              mbar_expect_tx(fb, 2 * n16 * 16 * D * 2);
              for (int r = 0; r < n16; ++r)
                for (int sl = 0; sl < C::kSlabs; ++sl) {
                  tma_load_2d(kd + sl * C::kSlabBytes + r * 2048, mk16, fb, sl * 64, (int)t0 + 16 * r);
                  tma_load_2d(vd + sl * C::kSlabBytes + r * 2048, mv16, fb, sl * 64, (int)t0 + 16 * r);
                }
            }
          }
          x = seg_end;
        }
      }
    }
    return;
  }

  if (warp == kEpi) {
    // ------------------------------------------------------------ epilogue warp
    griddep_wait();
    griddep_launch_dependents();
    const int G = p0.G;
    // staging cursor (runs two segments ahead of the consumers; may be a layer ahead)
    int ls = -1;
    const MParams *sp = nullptr;
    Tabs stb;
    int64_t sX0 = 0, sX1 = 0;
    Region sfirst;
    bool s_more = enter_layer<ML>(p0, ls, sp, stb, sX0, sX1, sfirst, &s_view[ML ? kCW + 1 : 0], smem_tabs, s_rng, true);
    int64_t xs = sX0;
    int ns = 0;
    int64_t buf_region[2] = {-1, -1};  // (layer, region) whose q rows each staging buffer holds
    Region r;
    r.end = -1;
    auto stage_next = [&]() {
      if (!s_more) return;
      if (xs >= sX1) {
        s_more = enter_layer<ML>(p0, ls, sp, stb, sX0, sX1, sfirst, &s_view[ML ? kCW + 1 : 0], smem_tabs, s_rng, true);
        if (!s_more) return;
        xs = sX0;
        r.end = -1;
      }
      const MParams &p = *sp;
      if (xs >= r.end) r = region_at<ML>(p, stb, r, sfirst, xs);
      const int ridx = r.b * p.ngl + r.g;
      const int64_t key = ((int64_t)ls << 32) | (uint32_t)ridx;
      if (buf_region[ns & 1] != key) {  // consecutive chunks of one region share their q rows
        const __nv_bfloat16 *qb = p.q + (int64_t)r.b * p.q_bs + (int64_t)r.g * G * D;
        __nv_bfloat16 *sq = s_q[ns & 1];
        for (int v = lane; v < G * (D / 8); v += 32) {
          const int h = v / (D / 8), e = (v - h * (D / 8)) * 8;
          *reinterpret_cast<uint4 *>(sq + h * QS + e) = *reinterpret_cast<const uint4 *>(qb + h * D + e);
        }
        buf_region[ns & 1] = key;
      }
      named_bar_arrive(kBarQFull + (ns & 1), kHandoff);
      xs = seg_end_of(p, r, xs, sX1);
      ++ns;
    };
    stage_next();
    stage_next();
    int n = 0;
    int lm = -1;
    const MParams *mp = nullptr;
    Tabs mtb;
    int64_t X0, X1;
    Region mfirst;
    while (enter_layer<ML>(p0, lm, mp, mtb, X0, X1, mfirst, &s_view[ML ? kCW + 2 : 0], smem_tabs, s_rng, true)) {
      const MParams &p = *mp;
      int run = 0;  // segments of the current region this CTA has finished (one ticket per run)
      Region rg;
      rg.end = -1;
      int64_t slot = 0;
      for (int64_t x = X0; x < X1; ++n) {
        if (x >= rg.end) {
          rg = region_at<ML>(p, mtb, rg, mfirst, x);
          slot = p.chunk ? (int64_t)rg.b * mtb.gc[p.ngl] + mtb.gc[rg.g] + (x - rg.start) / p.chunk
                         : (int64_t)blockIdx.x + rg.b * p.ngl + rg.g;
        } else {
          ++slot;  // next chunk of the same region (chunk mode only)
        }
        const int64_t seg_end = seg_end_of(p, rg, x, X1);
        named_bar_sync(kBarSegDone + (n & 1), kHandoff);
        // every consumer warp's partial of segment n is in shared memory (mbarrier release/
        // acquire): merge the kCW of them by LSE into this segment's slot
        const int ridx = rg.b * p.ngl + rg.g;
        {
          constexpr int PS = part_stride<D>();
          constexpr int NE = D / 32;
          const float *spp = s_part + (size_t)(n & 1) * kCW * G * PS;
          float *gp = p.part + slot * G * PS;
          for (int j = 0; j < G; ++j) {
            float lsv[kCW], mx = -INFINITY;
#pragma unroll
            for (int w = 0; w < kCW; ++w) {
              lsv[w] = spp[(w * G + j) * PS + D];
              mx = fmaxf(mx, lsv[w]);
            }
            float L = 0.f, O[NE];
#pragma unroll
            for (int i = 0; i < NE; ++i) O[i] = 0.f;
            if (mx != -INFINITY) {
#pragma unroll
              for (int w = 0; w < kCW; ++w) {
                const float wt = lsv[w] == -INFINITY ? 0.f : fast_exp2(lsv[w] - mx);
                L += wt;
#pragma unroll
                for (int i = 0; i < NE; ++i) O[i] = fmaf(wt, spp[(w * G + j) * PS + lane + 32 * i], O[i]);
              }
            }
            const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
            for (int i = 0; i < NE; ++i) gp[j * PS + lane + 32 * i] = O[i] * inv;
            if (lane == 0) gp[j * PS + D] = L > 0.f ? mx + __log2f(L) : -INFINITY;
          }
          __syncwarp();
        }
        ++run;
        const bool run_ends = seg_end >= rg.end || seg_end >= X1;
        int last = 0;
        if (run_ends && lane == 0) {
          __threadfence();  // cumulative: orders the partials of the run before the ticket
          int contributors;
          if (p.chunk) {
            contributors = mtb.gc[rg.g + 1] - mtb.gc[rg.g];
          } else {
            const int64_t c_first = cta_of(p, rg.start, ridx), c_last = cta_of(p, rg.end - 1, ridx);
            contributors = (int)(c_last - c_first + 1);
          }
          int *ctr = p.counters + ridx;
          const int ticket = atomicAdd(ctr, run);
          if (ticket + run == contributors) {
            *ctr = 0;  // self-reset for the next launch
            last = 1;
          }
        }
        if (run_ends) run = 0;
        last = __shfl_sync(0xffffffffu, last, 0);
        stage_next();  // q of segment n+2 into the buffer segment n used
        if (last) {
          __threadfence();
          combine_region_warp<D>(p, mtb.goff, mtb.wing, mtb.gc, ridx, lane);
        }
        x = seg_end;
      }
    }
    {
      const MParams &p = p0;
      if (lane == 0) TRACE(6);
    }
    return;
  }

  // -------------------------------------------------------------- consumers (warps 0..3)
  griddep_wait();
  griddep_launch_dependents();
  {
    const MParams &p = p0;
    if (tid == 0) TRACE(3);
  }
  const int qr = lane >> 2, qc = lane & 3;  // fragment row (head) / column-pair index
  const int h0 = qr, h1 = qr + 8;           // the two head rows this lane holds
  const int s = p0.n_sink;
  int T = 0, n = 0;
#ifdef MOA_DEC_TRACE
  int nseg = 0;
#endif
  const int G = p0.G;
  int lc = -1;
  const MParams *cp = nullptr;
  Tabs ctb;
  int64_t X0, X1;
  Region cfirst;
  while (enter_layer<ML>(p0, lc, cp, ctb, X0, X1, cfirst, &s_view[ML ? warp : 0], smem_tabs, s_rng, true)) {
  const MParams &p = *cp;
  // per-region state, recomputed only when a segment starts a new region (a CTA's consecutive
  // chunks of one region reuse it: no global loads or 64-bit divisions between them)
  Region rg;
  rg.end = -1;
  int64_t pos = 0, slot_p = -1;
  int W0 = 0, W1 = 0, pm = 0, slot_r = -1, pos32 = 0, ring_age_max = 0;
  bool ring_live = false, seg_full = false;
  for (int64_t x = X0; x < X1; ++n) {
    if (x >= rg.end) {
      rg = region_at<ML>(p, ctb, rg, cfirst, x);
      pos = p.pos_b ? p.pos_b[rg.b] : p.pos;
      const int32_t *wq = p.win_bq ? p.win_bq + (int64_t)rg.b * p.ngl * G : p.win_q;
      W0 = h0 < G ? wq[rg.g * G + h0] : rg.Wg;
      W1 = h1 < G ? wq[rg.g * G + h1] : rg.Wg;
      ring_live = pos >= s && rg.Wg > 0;
      pm = ring_live ? (int)((pos - s) % rg.Wg) : 0;
      slot_p = (p.k_new != nullptr) ? slot_of(pos, s, rg.Wg) : -1;
      slot_r = (int)slot_p;  // region row of the fused token (-1: none)
      pos32 = pos < (int64_t)0x7fffffff ? (int)pos : 0x7fffffff;
      ring_age_max = (int)((pos - s) < (int64_t)0x7fffffff ? (pos - s) : (int64_t)0x7fffffff);
      // every sink and ring row holds a position and every real head sees the whole ring
      const int minW = (W0 < W1 ? W0 : W1);
      seg_full = pos - s >= (int64_t)rg.Wg - 1 && pos >= s &&
                 __reduce_min_sync(0xffffffffu, (unsigned)minW) >= (unsigned)rg.Wg;
    }
    const int64_t seg_end = seg_end_of(p, rg, x, X1);
#ifdef MOA_DEC_TRACE
    ++nseg;
#endif

    // Q fragments (A operand, 16 x D, rows >= G are zero) from the staged rows, unscaled bf16
    uint32_t qa[KS][4];
    {
      named_bar_sync(kBarQFull + (n & 1), kHandoff);
      const __nv_bfloat16 *qb = s_q[n & 1];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int c = ks * 16 + qc * 2;
        qa[ks][0] = h0 < G ? *reinterpret_cast<const uint32_t *>(qb + h0 * QS + c) : 0u;
        qa[ks][1] = h1 < G ? *reinterpret_cast<const uint32_t *>(qb + h1 * QS + c) : 0u;
        qa[ks][2] = h0 < G ? *reinterpret_cast<const uint32_t *>(qb + h0 * QS + c + 8) : 0u;
        qa[ks][3] = h1 < G ? *reinterpret_cast<const uint32_t *>(qb + h1 * QS + c + 8) : 0u;
      }
    }
    float o[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    for (int64_t t0 = x; t0 < seg_end; t0 += kRows, ++T) {
      const int st = T % C::kStages;
      const int nrows = (int)((seg_end - t0) < kRows ? (seg_end - t0) : kRows);
      mbar_wait_warp(smem_u32(&full_bar[st]), (T / C::kStages) & 1);
      if (tid == 0 && T == 0) TRACE(4);
      const uint32_t kb = base + st * 2 * C::kTileBytes, vb = kb + C::kTileBytes;
      const int k0 = warp * 16;  // this warp's first key row in the tile
      if (k0 >= nrows) {         // rows past a segment tail were not loaded
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty_bar[st]));
        continue;
      }

      // ---- S = Q K^T  (16 heads x 16 keys); two accumulators per n-tile halve the HMMA chain
      float sacc[2][4], sacc2[2][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) sacc[0][i] = sacc[1][i] = sacc2[0][i] = sacc2[1][i] = 0.f;
      {
        const int mi = lane >> 3, rr = lane & 7;
        const int key = k0 + rr + (mi >> 1) * 8;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int chunk = 2 * ks + (mi & 1);
          const uint32_t addr = kb + (chunk >> 3) * C::kSlabBytes + key * 128 + (((chunk & 7) ^ (key & 7)) << 4);
          uint32_t b00, b01, b10, b11;
          ldsm_x4(addr, b00, b01, b10, b11);
          if (ks & 1) {
            mma16816(sacc2[0], qa[ks], b00, b01);
            mma16816(sacc2[1], qa[ks], b10, b11);
          } else {
            mma16816(sacc[0], qa[ks], b00, b01);
            mma16816(sacc[1], qa[ks], b10, b11);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) sacc[0][i] += sacc2[0][i], sacc[1][i] += sacc2[1][i];
      }
      // ---- visibility of this lane's 4 keys for its 2 head rows
      const int r_first = (int)(t0 - rg.start) + k0;  // region row of this warp's first key
      const bool fast = seg_full && k0 + 16 <= nrows && !(slot_r >= r_first && slot_r < r_first + 16);
      float sv[2][4];
      if (fast) {  // every key valid and inside every head's window: no mask arithmetic
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) sv[nt][i] = sacc[nt][i] * p.scale_log2;
      } else {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int kk = k0 + nt * 8 + qc * 2 + e;  // key index in tile
            const int r = r_first - k0 + kk;          // row in region
            bool valid = kk < nrows && r != slot_r, sink = false;
            int age = 0;
            if (r < s) {
              sink = true;
              valid = valid && r <= pos32;
            } else {
              int mm = pm - (r - s);
              if (mm < 0) mm += rg.Wg;
              age = mm;
              valid = valid && ring_live && mm <= ring_age_max;
            }
            const bool v0 = valid && (sink || age < W0);
            const bool v1 = valid && (sink || age < W1);
            sv[nt][e] = v0 ? sacc[nt][e] * p.scale_log2 : -INFINITY;
            sv[nt][2 + e] = v1 ? sacc[nt][2 + e] * p.scale_log2 : -INFINITY;
          }
        }
      }
      // ---- lazy online softmax per head row (quad-reduced max)
      float mt0 = fmaxf(fmaxf(sv[0][0], sv[0][1]), fmaxf(sv[1][0], sv[1][1]));
      float mt1 = fmaxf(fmaxf(sv[0][2], sv[0][3]), fmaxf(sv[1][2], sv[1][3]));
      mt0 = fmaxf(mt0, __shfl_xor_sync(0xffffffffu, mt0, 1));
      mt0 = fmaxf(mt0, __shfl_xor_sync(0xffffffffu, mt0, 2));
      mt1 = fmaxf(mt1, __shfl_xor_sync(0xffffffffu, mt1, 1));
      mt1 = fmaxf(mt1, __shfl_xor_sync(0xffffffffu, mt1, 2));
      if (m0 == -INFINITY) {
        m0 = mt0;
      } else if (mt0 > m0 + kRescale) {
        const float a = fast_exp2(m0 - mt0);
        l0 *= a;
#pragma unroll
        for (int j = 0; j < NT; ++j) o[j][0] *= a, o[j][1] *= a;
        m0 = mt0;
      }
      if (m1 == -INFINITY) {
        m1 = mt1;
      } else if (mt1 > m1 + kRescale) {
        const float a = fast_exp2(m1 - mt1);
        l1 *= a;
#pragma unroll
        for (int j = 0; j < NT; ++j) o[j][2] *= a, o[j][3] *= a;
        m1 = mt1;
      }
      const float r0 = m0 == -INFINITY ? 0.f : m0, r1 = m1 == -INFINITY ? 0.f : m1;
      uint32_t pa[4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const float e0 = fast_exp2(sv[nt][0] - r0), e1 = fast_exp2(sv[nt][1] - r0);
        const float e2 = fast_exp2(sv[nt][2] - r1), e3 = fast_exp2(sv[nt][3] - r1);
        l0 += e0 + e1;
        l1 += e2 + e3;
        pa[2 * nt + 0] = pack_bf16x2(e0, e1);
        pa[2 * nt + 1] = pack_bf16x2(e2, e3);
      }
      // ---- O += P V  (16 heads x D)
      {
        const int mi = lane >> 3, rr = lane & 7;
        const int key = k0 + rr + (mi & 1) * 8;
#pragma unroll
        for (int j2 = 0; j2 < NT / 2; ++j2) {
          const int chunk = 2 * j2 + (mi >> 1);
          const uint32_t addr = vb + (chunk >> 3) * C::kSlabBytes + key * 128 + (((chunk & 7) ^ (key & 7)) << 4);
          uint32_t b0a, b1a, b0b, b1b;
          ldsm_x4_t(addr, b0a, b1a, b0b, b1b);
          mma16816(o[2 * j2], pa, b0a, b1a);
          mma16816(o[2 * j2 + 1], pa, b0b, b1b);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty_bar[st]));
    }

    // ---- fused append: fold the new token into warp 0 of the CTA owning slot_p
    if (slot_p >= 0 && warp == 0) {
      const int64_t xr = rg.start + slot_p;
      if (xr >= x && xr < seg_end) {
        const __nv_bfloat16 *kn = p.k_new + (int64_t)rg.b * p.kv_bs + (int64_t)rg.g * D;
        const __nv_bfloat16 *vn = p.v_new + (int64_t)rg.b * p.kv_bs + (int64_t)rg.g * D;
        const __nv_bfloat16 *qb = s_q[n & 1];
        float d0 = 0.f, d1 = 0.f;
        for (int e = qc * (D / 4); e < (qc + 1) * (D / 4); ++e) {
          const float kf = __bfloat162float(kn[e]);
          if (h0 < G) d0 = fmaf(__bfloat162float(qb[h0 * QS + e]), kf, d0);
          if (h1 < G) d1 = fmaf(__bfloat162float(qb[h1 * QS + e]), kf, d1);
        }
        d0 += __shfl_xor_sync(0xffffffffu, d0, 1);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 2);
        d1 += __shfl_xor_sync(0xffffffffu, d1, 1);
        d1 += __shfl_xor_sync(0xffffffffu, d1, 2);
        // the new token (age 0) is visible to a head iff W_h >= 1 or it is a sink position
        const bool nsink = pos < s;
        const float x0 = (nsink || W0 >= 1) ? d0 * p.scale_log2 : -INFINITY;
        const float x1 = (nsink || W1 >= 1) ? d1 * p.scale_log2 : -INFINITY;
        const float n0 = fmaxf(m0, x0), n1 = fmaxf(m1, x1);
        const float a0 = (m0 == -INFINITY) ? 0.f : fast_exp2(m0 - n0);
        const float a1 = (m1 == -INFINITY) ? 0.f : fast_exp2(m1 - n1);
        const float p0 = x0 == -INFINITY ? 0.f : fast_exp2(x0 - n0);
        const float p1 = x1 == -INFINITY ? 0.f : fast_exp2(x1 - n1);
        if (n0 != -INFINITY) {
          l0 = l0 * a0 + (qc == 0 ? p0 : 0.f);
          m0 = n0;
        }
        if (n1 != -INFINITY) {
          l1 = l1 * a1 + (qc == 0 ? p1 : 0.f);
          m1 = n1;
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int c = 8 * j + qc * 2;
          const float v0 = __bfloat162float(vn[c]), v1 = __bfloat162float(vn[c + 1]);
          if (n0 != -INFINITY) {
            o[j][0] = o[j][0] * a0 + p0 * v0;
            o[j][1] = o[j][1] * a0 + p0 * v1;
          }
          if (n1 != -INFINITY) {
            o[j][2] = o[j][2] * a1 + p1 * v0;
            o[j][3] = o[j][3] * a1 + p1 * v1;
          }
        }
        // write the token into its cache row (nothing reads this row in this launch)
        const int64_t row = xr;
        for (int e = lane * 8; e < D; e += 32 * 8) {
          *reinterpret_cast<uint4 *>(p.kc + row * D + e) = *reinterpret_cast<const uint4 *>(kn + e);
          *reinterpret_cast<uint4 *>(p.vc + row * D + e) = *reinterpret_cast<const uint4 *>(vn + e);
        }
      }
    }

    // ---- per-warp partial of this segment (o / l and lse2) into shared memory; hand the
    //      segment to the epilogue warp
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    constexpr int PS = part_stride<D>();
    float *part = s_part + ((size_t)(n & 1) * kCW + warp) * G * PS;
    {
      const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int c = 8 * j + qc * 2;
        if (h0 < G) *reinterpret_cast<float2 *>(part + h0 * PS + c) = make_float2(o[j][0] * i0, o[j][1] * i0);
        if (h1 < G) *reinterpret_cast<float2 *>(part + h1 * PS + c) = make_float2(o[j][2] * i1, o[j][3] * i1);
      }
      if (qc == 0) {
        if (h0 < G) part[h0 * PS + D] = l0 > 0.f ? m0 + __log2f(l0) : -INFINITY;
        if (h1 < G) part[h1 * PS + D] = l1 > 0.f ? m1 + __log2f(l1) : -INFINITY;
      }
    }
    named_bar_arrive(kBarSegDone + (n & 1), kHandoff);
    x = seg_end;
  }
  }  // layers
  {
    const MParams &p = p0;
    if (tid == 0) TRACE(5);
  }
#ifdef MOA_DEC_TRACE
  if (tid == 0) {
    const MParams &p = p0;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    TRACE_V(7, (unsigned long long)T | ((unsigned long long)nseg << 40) | ((unsigned long long)smid << 48));
  }
#endif
}

int num_sms_dev() { return device_sm_count(); }

int ctas_for(int64_t R, int cps) {
  int64_t n = (int64_t)num_sms_dev() * cps;
  int64_t by_rows = (R + kRows - 1) / kRows;
  return (int)(n < by_rows ? n : by_rows);
}

// fill the per-call parameters shared by both launchers
void fill_params(MParams &p, const DecodeMmaArgs &a) {
  p = MParams{};
  p.q = static_cast<const __nv_bfloat16 *>(a.q);
  p.o = static_cast<__nv_bfloat16 *>(a.o);
  p.q_bs = a.q_bs;
  p.o_bs = a.o_bs;
  p.k_new = static_cast<const __nv_bfloat16 *>(a.k_new);
  p.v_new = static_cast<const __nv_bfloat16 *>(a.v_new);
  p.kv_bs = a.kv_bs;
  p.kc = static_cast<__nv_bfloat16 *>(a.k_cache);
  p.vc = static_cast<__nv_bfloat16 *>(a.v_cache);
  p.rows_per_seq = a.rows_per_seq;
  p.R = (int64_t)a.batch * a.rows_per_seq;
  static const int64_t seg_cost = [] {
    const char *e = std::getenv("MOA_DEC_SEG_COST");  // tuning override
    return e ? (int64_t)std::atoll(e) : (int64_t)128;
  }();
  p.seg_cost = seg_cost;
  p.chunk = a.chunk;
  p.gc_off = a.d_gc_off;
  p.ctot = a.chunk ? p.R + seg_cost * (int64_t)a.batch * a.chunks_per_seq
                   : p.R + seg_cost * ((int64_t)a.batch * a.ngl - 1);
  p.g_off = a.d_g_off;
  p.win_g = a.d_win_g;
  p.win_q = a.d_win_q;
  p.ngl = a.ngl;
  p.G = a.G;
  p.n_sink = a.n_sink;
  p.batch = a.batch;
  p.pos = a.pos;
  p.pos_b = a.d_pos;
  p.win_bq = a.d_win_bq;
  p.scale_log2 = a.scale * kLog2e;
  p.lse = a.lse;
  p.part = a.ws_part;
  p.counters = a.counters;
  p.early = a.early_read;
  p.peers = static_cast<const PeerOut *>(a.peers);
  p.n_peers = a.n_peers;
  p.peer_head0 = a.peer_head0;
  p.peer_bs = a.peer_bs;
  p.peer_ls = a.peer_ls;
  p.layer = a.layer;
}

template <int D, int STAGES, int CPS, bool ML>
int launch_kernel(const MParams &p, const void *kmap, const void *vmap, const void *kmap16, const void *vmap16,
                  int n, int G, void *stream) {
  using C = DCfg<D, STAGES>;
  const int smem = C::kSmem + 2 * kCW * G * part_stride<D>() * 4;
  cudaError_t e = cudaFuncSetAttribute(decode_mma_kernel<D, STAGES, CPS, ML>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return (int)e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)n);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const CUtensorMap zero_map{};  // ML: the maps come from the layer descriptors
  const CUtensorMap &km = kmap ? *static_cast<const CUtensorMap *>(kmap) : zero_map;
  const CUtensorMap &vm = vmap ? *static_cast<const CUtensorMap *>(vmap) : zero_map;
  const CUtensorMap &km16 = kmap16 ? *static_cast<const CUtensorMap *>(kmap16) : zero_map;
  const CUtensorMap &vm16 = vmap16 ? *static_cast<const CUtensorMap *>(vmap16) : zero_map;
  e = cudaLaunchKernelEx(&cfg, decode_mma_kernel<D, STAGES, CPS, ML>, km, vm, km16, vm16, p);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}

template <int D, int STAGES, int CPS>
int launch_v(const DecodeMmaArgs &a, void *stream) {
  MParams p;
  fill_params(p, a);
#ifdef MOA_DEC_TRACE
  static int launch_no = 0;
  p.trace_slot = (launch_no++) & 1;
#endif
  return launch_kernel<D, STAGES, CPS, false>(p, a.kmap, a.vmap, a.kmap16, a.vmap16, ctas_for(p.R, CPS), a.G,
                                              stream);
}

template <int D, int STAGES, int CPS>
int launch_layers_v(const DecodeLayersArgs &l, void *stream) {
  MParams p;
  fill_params(p, l.a);
  // early streaming only when the host established that the stream predecessor does not
  // append to these layers (a previous layer chunk of the same token)
  p.ml = l.d_layers;
  p.nl = l.n_layers;
  p.q_ls = l.q_ls;
  p.o_ls = l.o_ls;
  p.kvn_ls = l.kvn_ls;
  p.lse_ls = l.lse_ls;
  p.part_ls = l.part_ls;
  // balanced split: the ticket count of a region is the CTAs between its first and last row,
  // so no CTA may get an empty range in any layer: n <= every layer's total cost
  int64_t n = ctas_for(l.max_rows, CPS);
  if (!p.chunk) {
    const int64_t min_ctot = l.min_rows + p.seg_cost * ((int64_t)p.batch * p.ngl - 1);
    if (n > min_ctot) n = min_ctot;
  }
  return launch_kernel<D, STAGES, CPS, true>(p, nullptr, nullptr, nullptr, nullptr, (int)n, l.a.G, stream);
}

template <int D>
int launch_d(const DecodeMmaArgs &a, void *stream) {
  static int variant = [] {
    const char *e = std::getenv("MOA_DEC_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  if (D == 128) {
    switch (variant) {
      case 1: return launch_v<D, 3, 2>(a, stream);
      case 2: return launch_v<D, 4, 1>(a, stream);
      default: return launch_v<D, 2, 2>(a, stream);
    }
  }
  return launch_v<D, 6, 2>(a, stream);
}

}  // namespace

size_t decode_mma_ws_bytes(int batch, int ngl, int G, int d, int chunks_per_seq) {
  // one slot per (CTA, region) pair (balanced split) or per chunk (rank-invariant split)
  const size_t slots = chunks_per_seq > 0 ? (size_t)batch * chunks_per_seq + 1
                                          : (size_t)num_sms_dev() * kCtasPerSm + (size_t)batch * ngl + 1;
  return ((slots * G * (d + 4) * 4) + 255) & ~size_t(255);
}

#ifdef MOA_DEC_TRACE
extern "C" int moa_debug_decode_trace(void *host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, g_trace, bytes < sizeof(g_trace) ? bytes : sizeof(g_trace));
}
#endif

int launch_decode_mma(const DecodeMmaArgs &a, void *stream) {
  if (a.d == 128) return launch_d<128>(a, stream);
  return launch_d<64>(a, stream);
}

namespace {
__global__ void wait_flag_kernel(const unsigned *flag, unsigned expected) {
  // counters only grow (modulo 2^32): wait until flag - expected >= 0 in wrapped arithmetic.
  // A wait that outlives 10 s traps (a sticky error the next library call reports) instead of
  // hanging the device when a peer never arrives.
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - expected) >= 0) break;
    __nanosleep(64);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 10000000000ull) __trap();
  }
}
}  // namespace

int launch_wait_flag(const unsigned *flag, unsigned expected, void *stream) {
  wait_flag_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flag, expected);
  return (int)cudaGetLastError();
}

int launch_decode_mma_layers(const DecodeLayersArgs &l, void *stream) {
  if (l.a.d == 128) return launch_layers_v<128, 2, 2>(l, stream);
  return launch_layers_v<64, 6, 2>(l, stream);
}

}  // namespace moa
