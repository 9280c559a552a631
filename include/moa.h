/*
 * moa.h -- C ABI of the B200 (sm_100a) MoA attention hot path.
 *
 * MoA = "Mixture of Attention Spans" (arXiv 2406.14909).  Every (layer, head)
 * attends only to a few global sink tokens plus its own window of recent keys;
 * the window follows the head's elastic rule S_h = alpha_h + beta_h * N
 * (Eq. 2, clipped to [0, N] per PAPER.md:692).  Citations are
 * PAPER.md line numbers and SURVEY.md sections.
 *
 * Mask of q-head h (token granular, reading c5): key j is visible to query i
 * iff  0 <= j <= i  and  ( j < n_sink  or  i - j < W_h ).
 *   - sinks: "the initial few tokens (64 tokens for MoA) are not masked"
 *     (PAPER.md:178);
 *   - window W_h counts the query itself (reading c3);
 *   - output: O = softmax(tau * Q K^T + M) V  (Eq. 1).
 *
 * GQA (reading c10): q-head h reads kv-group g = h / G, G = Hq / Hkv.  The
 * cache of group g holds W_g = max_{h in g} W_h recent rows; each q-head
 * still masks to its own W_h.
 *
 * Tensor layouts (row-major, elements of the context dtype):
 *   prefill  Q, O : [B, N, Hq_local, d]  token rows, stride *_row_stride
 *            K, V : [B, N, Hkv_local, d] token rows, stride kv_row_stride
 *            batch stride = N * row_stride; head h at offset h * d in a row.
 *            A rank holding a head shard passes pointers to its first local
 *            head and the full row stride.
 *   decode   q, o : [B, Hq_local, d]   batch stride *_batch_stride
 *            k_new, v_new : [B, Hkv_local, d] batch stride kv_batch_stride
 *   lse      fp32; prefill [B, Hq_local, N], decode [B, Hq_local]
 *            (natural log of the softmax denominator incl. tau, i.e.
 *             lse = log sum_j exp(tau q.k_j)).
 *   KV cache (caller-owned device memory, reading c13):
 *            per layer, per sequence b, per local group g one region of
 *            (n_sink + W_g) rows of d elements: [sink rows | ring rows].
 *            Position p lives in row p if p < n_sink, else in row
 *            n_sink + (p - n_sink) mod W_g  ("replace the old KV-Cache that
 *            exceeds the span with the latest").  K and V have
 *            identical layouts in two separate buffers.
 *
 * Ownership: the caller owns every device buffer (Q/K/V/O, caches,
 * workspace).  The library owns the context and its small host/device span
 * tables.  moa_prefill / moa_cache_fill / moa_kv_append / moa_decode_step
 * never allocate, never synchronise the host and only enqueue work on the
 * given stream (CUDA-graph capturable).
 *
 * Errors: every call returns moa_status.  Argument validation failures return
 * immediately with nothing launched and a message in moa_last_error()
 * (thread-local).  A sticky asynchronous CUDA fault is reported as
 * MOA_ERR_CUDA by the next call.  No exception or abort crosses the ABI.
 * A context is not thread-safe: use one per (thread, device).
 */
#ifndef MOA_H_
#define MOA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct moa_ctx moa_ctx;          /* opaque */
typedef void *moa_stream_t;              /* a cudaStream_t (NULL = legacy default stream) */

typedef enum {
  MOA_OK = 0,
  MOA_ERR_INVALID_ARG = 1,   /* bad pointer / value (e.g. W < 0, W = 0 with n_sink = 0) */
  MOA_ERR_SHAPE = 2,         /* dims not supported or inconsistent (head_dim not 64/128 ...) */
  MOA_ERR_STATE = 3,         /* call out of order (spans unset, cache unbound, wrong pos) */
  MOA_ERR_UNSUPPORTED = 4,   /* valid request this build does not implement */
  MOA_ERR_OOM = 5,           /* host allocation failed / workspace too small */
  MOA_ERR_CUDA = 6           /* CUDA runtime/driver error (message has the CUDA string) */
} moa_status;

typedef enum { MOA_BF16 = 0, MOA_FP32 = 1 } moa_dtype;

/* Version string of the library build. */
const char *moa_version(void);
/* Message of the last non-OK status on this thread ("" if none). */
const char *moa_last_error(void);

/*
 * Create a context.
 *   device       CUDA device ordinal, or -1 for a host-only planning context
 *                (span tables, layout and schedule queries work; launches
 *                return MOA_ERR_STATE).
 *   dtype        I/O dtype of Q/K/V/O and the cache (compute is fp32).
 *   num_layers, num_q_heads, num_kv_heads: the model's totals (Hq % Hkv == 0).
 *   head_dim     64 or 128.
 *   max_batch    largest batch any call will pass (plans decode splits).
 *   kv_group_begin, kv_group_end: the kv-groups this context serves
 *                [begin, end) (all groups: 0, num_kv_heads).  Its local
 *                q-heads are [begin*G, end*G).
 */
moa_status moa_create(moa_ctx **out, int device, moa_dtype dtype, int num_layers,
                      int num_q_heads, int num_kv_heads, int head_dim, int max_batch,
                      int kv_group_begin, int kv_group_end);
moa_status moa_destroy(moa_ctx *ctx);

/*
 * Host helper: elastic rules -> windows.  For every head
 *   span   = clamp(ceil(alpha + beta * N), 0, N)   (Eq. 2; clip PAPER.md:692;
 *                                                  ceil = reading c6)
 *   window = max(0, span - n_sink)                 (span = window + sinks)
 * alpha, beta, window_out: n_heads entries (host memory).
 */
moa_status moa_resolve_spans(const float *alpha, const float *beta, int n_heads, int64_t N,
                             int n_sink, int32_t *window_out);

/*
 * Install the spans of one layer (host memory; frozen for the whole decode,
 * PAPER.md:704, reading c9).
 *   window_per_q_head  num_q_heads entries (ALL heads of the layer; the
 *                      context keeps its shard).  W >= 0; W = 0 needs n_sink >= 1.
 *   n_sink             global sink tokens (64 for MoA).
 *   N                  prompt length the spans were resolved at (>= 1).
 * Builds the span table, cache offsets, the prefill block-skip schedule and
 * the decode work list, and uploads them.  Invalidates a bound cache's layout
 * if the layer's footprint changes (re-bind after the last set_spans).
 */
moa_status moa_set_spans(moa_ctx *ctx, int layer, const int32_t *window_per_q_head,
                         int n_sink, int64_t N);

/*
 * moa_set_spans with the paper's block-granular prefill mask:
 * "block sliding-window attention pattern with a block size of 64 ... The first block
 * of tokens is not masked and serves as the attention sink".
 * Query i sees key j <= i iff j / block < n_sink / block or i / block - j / block <
 * W / block (SPEC.md:216-224 build_mask; causal inside the diagonal block).
 *   block   0 = token-granular mask (== moa_set_spans); else a power of two in [1, 128]
 *           dividing n_sink and every window (MOA_ERR_INVALID_ARG otherwise).
 * Only prefill changes: decode stays token-granular (the cache replaces entries token by
 * token), with the same windows and the same cache layout.
 */
moa_status moa_set_spans_blocked(moa_ctx *ctx, int layer, const int32_t *window_per_q_head,
                                 int n_sink, int64_t N, int block);

/*
 * Ragged batch: per-sequence prompt lengths and spans.
 * Eq. 2 makes every span a function of the input length N (PAPER.md:181,
 * "elastic rules ... scale with the input length"), so sequences of different
 * lengths in one batch have different windows W_{b,h} = span_h(N_b) - n_sink
 * (moa_resolve_spans at N_b).  The layer's moa_set_spans(..., N) fixes the padded
 * length N (the row stride of q/k/v/o) and the cache capacity W_g; this call
 * installs, for sequences b < batch,
 *   seq_len                 host [batch]: N_b in [1, N].
 *   window_per_seq_q_head   host [batch, num_q_heads] (ALL heads; the context keeps its
 *                           shard) or NULL (= the layer's windows for every sequence).
 *                           0 <= W_{b,h} <= W_g of the head's group (the ring must hold the
 *                           window); block mode: multiples of the block.
 * batch = 0 returns the layer to a uniform batch.  moa_set_spans clears it.
 * While a layer is ragged:
 *   - moa_prefill / moa_prefill_attn / moa_cache_fill take N = the padded length and
 *     batch = this batch; sequence b is the prompt of its first N_b rows under its own
 *     windows; output / lse rows i >= N_b are not written.  The cache fill stores
 *     positions < N_b.  The padding rows [N_b, N) of q/k/v must hold FINITE values
 *     (any, e.g. zeros): the kernels tile against N and give padding keys probability
 *     exactly 0, and 0 * Inf/NaN would poison a real row.
 *   - decode goes through moa_decode_step_fused_ragged (the uniform append / decode
 *     calls return MOA_ERR_STATE).
 * Errors: MOA_ERR_INVALID_ARG (ranges above), nothing is changed on error.
 */
moa_status moa_set_ragged(moa_ctx *ctx, int layer, int batch, const int64_t *seq_len,
                          const int32_t *window_per_seq_q_head);

/* Bytes of the K (and of the V) cache of all layers / of one layer for
 * `batch` sequences.  All layers' spans must be set for the first form. */
moa_status moa_cache_bytes(const moa_ctx *ctx, int batch, size_t *k_bytes, size_t *v_bytes);
moa_status moa_layer_cache_bytes(const moa_ctx *ctx, int layer, int batch, size_t *k_bytes,
                                 size_t *v_bytes);
/* Scratch needed by moa_prefill / moa_decode_step for `batch` sequences
 * (max over layers whose spans are set; >= 256 bytes). */
moa_status moa_workspace_bytes(const moa_ctx *ctx, int batch, size_t *bytes);

/* Bind caller-owned device memory as the cache of every layer (layer l at
 * byte offset sum_{l'<l} layer bytes) or of one layer.  256-byte aligned.
 * Binding zero-fills the layer caches (synchronously) and resets the layer's
 * next position to 0. */
moa_status moa_bind_cache(moa_ctx *ctx, void *k_cache, void *v_cache, int batch);
moa_status moa_bind_layer_cache(moa_ctx *ctx, int layer, void *k_cache, void *v_cache, int batch);

/*
 * Causal prefill of one layer with the per-head MoA mask (Eq. 1 + the mask
 * above), then the cache fill of rows [0, min(s,N)) and [max(s, N-W_g), N)
 * (SURVEY §8(a) a4+a5).  bf16: tcgen05 tensor-core kernel; fp32: FFMA kernel.
 *   scale      tau (the softmax scale; Eq. 1 has none, reading c8).
 *   lse_out    nullable, fp32 [B, Hq_local, N].
 *   workspace  device scratch of moa_workspace_bytes (may be NULL if 0 needed).
 * Afterwards the layer's next decode position is N.
 */
moa_status moa_prefill(moa_ctx *ctx, int layer, const void *q, const void *k, const void *v,
                       void *o, int64_t q_row_stride, int64_t kv_row_stride,
                       int64_t o_row_stride, int batch, int64_t N, float scale, float *lse_out,
                       void *workspace, size_t ws_bytes, moa_stream_t stream);

/* The attention of moa_prefill alone (a4): no cache is read or written and
 * none needs to be bound; the layer's decode position is unchanged.  Together
 * with moa_cache_fill it is exactly moa_prefill. */
moa_status moa_prefill_attn(moa_ctx *ctx, int layer, const void *q, const void *k, const void *v,
                            void *o, int64_t q_row_stride, int64_t kv_row_stride,
                            int64_t o_row_stride, int batch, int64_t N, float scale, float *lse_out,
                            moa_stream_t stream);

/* Cache fill alone (a5): write the resident rows of a prompt of length N
 * (K/V as in moa_prefill) into the layer's cache; next position = N. */
moa_status moa_cache_fill(moa_ctx *ctx, int layer, const void *k, const void *v,
                          int64_t kv_row_stride, int batch, int64_t N, moa_stream_t stream);

/*
 * Append the K/V of absolute position `pos` (a6): for every (b, g) write
 * k_new/v_new into row slot(pos).  A group with W_g = 0 stores only sink
 * positions.  `pos` must equal the layer's next position (N after prefill,
 * then +1 per append).
 */
moa_status moa_kv_append(moa_ctx *ctx, int layer, const void *k_new, const void *v_new,
                         int64_t kv_batch_stride, int batch, int64_t pos, moa_stream_t stream);

/*
 * One decode step of one layer at position `pos` (a7 + a8): every local
 * q-head attends over its group's cache restricted to its own window,
 * split-KV partials in `workspace`, merged by LSE into o.  `pos` must be the
 * last appended position (append before decode: the token sees itself).
 *   lse_out nullable fp32 [B, Hq_local].
 */
moa_status moa_decode_step(moa_ctx *ctx, int layer, const void *q, void *o,
                           int64_t q_batch_stride, int64_t o_batch_stride, int batch,
                           int64_t pos, float scale, float *lse_out, void *workspace,
                           size_t ws_bytes, moa_stream_t stream);

/* Append + decode in one launch (a6 + a7 + a8 fused): identical results to
 * moa_kv_append(pos) followed by moa_decode_step(pos).
 *
 * Stream overlap (both decode calls, bf16): the kernel is launched with
 * programmatic stream serialization.  It reads q, k_new, v_new and writes o,
 * lse, the workspace and the cache only after its stream predecessor has
 * completed, and it lets its successor launch only after that point.  When the
 * most recent launch made through this context did not write this layer's
 * cache (e.g. it decoded another layer), the kernel starts streaming the
 * layer's cache rows while its predecessor is still running.  The cache is
 * owned by the library after binding: the caller must not write it, and
 * launches of one context go to one stream. */
moa_status moa_decode_step_fused(moa_ctx *ctx, int layer, const void *q, const void *k_new,
                                 const void *v_new, void *o, int64_t q_batch_stride,
                                 int64_t kv_batch_stride, int64_t o_batch_stride, int batch,
                                 int64_t pos, float scale, float *lse_out, void *workspace,
                                 size_t ws_bytes, moa_stream_t stream);

/*
 * Cross-layer decode: moa_decode_step_fused of the layers
 * [layer0, layer0 + n_layers) for one token position in ONE persistent launch.  Every CTA
 * streams its share of layer l's cache and then, without draining its TMA pipeline, its
 * share of layer l+1, so the per-launch ramp-up and tail (the last CTAs, the last
 * region's LSE merge) are paid once per token instead of once per layer.  Each layer is
 * masked and merged exactly as moa_decode_step_fused does it (heads masked
 * independently).  With the rank-invariant split (moa_set_decode_split)
 * the results are bitwise those of n_layers single-layer calls; with the balanced split the
 * CTA ranges can differ (the grid is sized for the largest layer), so they agree to rounding.
 * Ranges longer than 32 layers run as several launches of <= 32 layers.  For when the q of several layers are available together
 * (layer-parallel blocks, the attention sub-step of a pipelined schedule, the synthetic
 * benchmark); a model whose layer l+1 query depends on layer l's output uses the
 * single-layer call.
 *   q, o            bf16 [n_layers][B][Hq_local][d]: layer stride q/o_layer_stride, batch
 *                   stride q/o_batch_stride (elements)
 *   k_new, v_new    bf16 [n_layers][B][Hkv_local][d]: kv_layer_stride, kv_batch_stride
 *                   (input layer strides may be 0: every layer reads the same rows)
 *   lse_out         nullable fp32, layer stride lse_layer_stride, [B][Hq_local] per layer
 *   workspace       >= n_layers * moa_workspace_bytes(ctx, batch) bytes; layer i uses the
 *                   i-th equal slice
 * Every layer must be set, bound with tensor maps (bf16), uniform (not ragged), share one
 * sink count and expect `pos` (all advance to pos + 1).  The launch reads a device copy of
 * the layers' tables built by moa_prepare_layers; if it is stale (set_spans, bind,
 * set_decode_split or set_ragged since), the call rebuilds it first, which synchronises the
 * device -- or fails with MOA_ERR_STATE while `stream` is capturing a CUDA graph.  The
 * launch does not stream early (its predecessor may be the previous token's launch, which
 * appended to these layers).
 */
moa_status moa_prepare_layers(moa_ctx *ctx);
moa_status moa_decode_step_fused_layers(moa_ctx *ctx, int layer0, int n_layers, const void *q, const void *k_new,
                                        const void *v_new, void *o, int64_t q_layer_stride,
                                        int64_t kv_layer_stride, int64_t o_layer_stride, int64_t q_batch_stride,
                                        int64_t kv_batch_stride, int64_t o_batch_stride, int batch, int64_t pos,
                                        float scale, float *lse_out, int64_t lse_layer_stride, void *workspace,
                                        size_t ws_bytes, moa_stream_t stream);

/*
 * Fused head-output all-gather for kv-group sharded decode.
 * Heads are masked independently, so a rank serving kv-groups [g0, g1)
 * owns complete head outputs; the next layer needs every head on every rank.  With peer
 * outputs installed, every bf16 decode launch of this context (single-layer, ragged and
 * cross-layer) writes each finished head row, from the combine epilogue that produced it,
 * into all n_peers destination buffers as well as into o, then releases it with one
 * system-scope atomic increment of the destination's counter of that layer -- the
 * all-gather becomes P2P stores over NVLink overlapped with the rest of the decode instead
 * of a separate collective after it.
 *   peer_o[k]      device address (as mapped on THIS device: a peer-mapped or symmetric-memory
 *                  buffer) of destination k: bf16 [L][B][Hq_total][d]; layer l, sequence b,
 *                  global q-head h at  l * peer_layer_stride + b * peer_batch_stride + h * d
 *   peer_flags[k]  device address of destination k's uint32 counters [L]; every region
 *                  (sequence, local kv-group) of layer l adds 1 when its G heads are written,
 *                  so one token step of every rank adds B * Hkv_total to each counter
 *   head0          global index of this context's first local q-head (g0 * G)
 * n_peers = 0 switches it off.  The arrays are copied (at most 16 destinations); the call
 * synchronises the device.  Unsupported for fp32 contexts.
 */
moa_status moa_set_peer_outputs(moa_ctx *ctx, int n_peers, void *const *peer_o, unsigned int *const *peer_flags,
                                int64_t peer_batch_stride, int64_t peer_layer_stride, int head0);

/* Stream-ordered wait: the next work on `stream` starts once the uint32 at `flag` (device
 * memory, any peer's writes visible at system scope) has reached `expected` (counters only
 * grow; compared modulo 2^32).  One tiny kernel; CUDA-graph capturable.  A wait still
 * unsatisfied after 10 s traps (the next call reports MOA_ERR_CUDA) rather than hang. */
moa_status moa_wait_flag(const unsigned int *flag, unsigned int expected, moa_stream_t stream);

/*
 * Append + decode of a ragged batch: moa_decode_step_fused where sequence b is at its
 * own position pos[b] (a6 + a7 + a8 per sequence, PAPER.md:704 cache replacement).
 *   pos   DEVICE int64 [batch], caller-owned, 8-byte aligned, read by the kernel after its
 *         stream predecessor completes (so a preceding kernel may advance it; CUDA-graph
 *         friendly).  pos[b] must be the next position of sequence b (N_b after the
 *         prefill, +1 per step); this is not checked.  pos[b] < 0 marks an inactive
 *         sequence: nothing is written to its cache, its o row is 0 and its lse -inf.
 * Windows: the layer's ragged windows (moa_set_ragged) or, on a uniform layer, the
 * layer's windows.  On a ragged layer batch must equal the ragged batch.
 */
moa_status moa_decode_step_fused_ragged(moa_ctx *ctx, int layer, const void *q, const void *k_new,
                                        const void *v_new, void *o, int64_t q_batch_stride,
                                        int64_t kv_batch_stride, int64_t o_batch_stride, int batch,
                                        const int64_t *pos, float scale, float *lse_out, void *workspace,
                                        size_t ws_bytes, moa_stream_t stream);

/*
 * Decode split mode (bf16 decode).  The decode kernel spreads a layer's cache rows over
 * the SMs; the LSE partials of a (sequence, kv-group) region are merged in a fixed order.
 *   chunk_rows = 0 (default): balanced split -- every CTA streams the same number of rows,
 *       so where a region is cut depends on the batch, the other regions and the SM count.
 *   chunk_rows > 0 (a multiple of 64): rank-invariant split -- every region is cut into
 *       chunks of chunk_rows rows from its first row and each chunk is one partial; the
 *       arithmetic on a region's rows then depends on that region alone, so a context
 *       serving a kv-group shard (moa_create's [g0, g1)) or a subset of the sequences
 *       computes bit-identical outputs to the unsharded context (SURVEY §4 tier 4;
 *       heads are independent).  256 is a good value.
 * Applies to every layer (also layers set later); changes moa_workspace_bytes.  Must not
 * be called while a layer is ragged (MOA_ERR_STATE).  MOA_ERR_INVALID_ARG for other values.
 */
moa_status moa_set_decode_split(moa_ctx *ctx, int chunk_rows);

/*
 * Advance device-resident positions: pos[b] += delta for b < batch where pos[b] >= 0
 * (inactive sequences stay inactive).  The companion of moa_decode_step_fused_ragged for
 * CUDA-graph capture of a whole token step (every layer's fused decode, then this call):
 * a replayed graph moves every sequence to its next position with no host involvement
 * (the decode call takes the position by pointer, PAPER.md:704 one token per step).
 *   pos    DEVICE int64 [batch], 8-byte aligned, caller-owned.
 * Stream-ordered, no allocation, no host synchronisation; MOA_ERR_INVALID_ARG for a NULL
 * or misaligned pointer or batch < 1.
 */
moa_status moa_advance_pos(int64_t *pos, int batch, int64_t delta, moa_stream_t stream);

/* ---------------- host-side introspection (planning contexts too) ---------------- */

/* Window of a local q-head / cache capacity W_g of a local group. */
moa_status moa_get_window(const moa_ctx *ctx, int layer, int q_head_local, int32_t *window);
moa_status moa_get_group_window(const moa_ctx *ctx, int layer, int group_local, int32_t *w_g);
/* Row of position `pos` inside group region (slot), -1 if not stored. */
moa_status moa_slot_of(const moa_ctx *ctx, int layer, int group_local, int64_t pos, int64_t *slot);
/* Row offset (in rows of d elements, from the layer's cache base) and row
 * count of the region of sequence b, local group g. */
moa_status moa_cache_region(const moa_ctx *ctx, int layer, int b, int group_local,
                            int64_t *row_offset, int64_t *rows);
/* Byte offset of a layer inside a moa_bind_cache buffer laid out for `batch`. */
moa_status moa_layer_offset(const moa_ctx *ctx, int layer, int batch, size_t *byte_offset);

/*
 * Block-averaged attention influence of the profiling stage: for one
 * calibration item with dense causal attention A = softmax(scale * Q K^T + causal) (Eq. 1)
 * and G = dL/dA = dO V^T (O = A V), the influence of masking A_ij (Eq. 3, PAPER.md:225-236;
 * derivation PAPER.md:1361-1405)
 *     E_ij = -A_ij / (1 - A_ij) * (G_ij - sum_n G_in A_in)     (E = 0 where A_ij = 1)
 * averaged over the block x block token pairs of every (query block, key block)
 * ("the average attention influence within each block"; the last block
 * of a ragged N averages its real pairs).  Stateless; bf16 inputs, fp32 math and output.
 *   q, dout   [B, N, Hq, d] bf16, token row stride q_row_stride (elements).
 *   k, v      [B, N, Hkv, d] bf16 (Hq % Hkv == 0), row stride kv_row_stride.
 *   head_dim  64 or 128.  block: 64 (the paper's block; MOA_ERR_UNSUPPORTED otherwise).
 *   e_blocks  fp32 [B, Hq, nb, nb], nb = ceil(N / block), caller-owned device memory:
 *             accumulate = 0 overwrites every entry (key blocks after the query block: 0);
 *             accumulate = 1 adds to the causal entries (averaging over calibration items
 *             is the caller's division by the item count).
 * Stream-ordered, no allocation, no host synchronisation.
 */
moa_status moa_attention_influence(const void *q, const void *k, const void *v, const void *dout, int batch,
                                   int64_t N, int num_q_heads, int num_kv_heads, int head_dim,
                                   int64_t q_row_stride, int64_t kv_row_stride, float scale, int block,
                                   float *e_blocks, int accumulate, moa_stream_t stream);

/*
 * Rule losses (Eq. 4): for every head h and
 * candidate elastic rule r,  Delta L_{h,r} = sum_{i,j} M_{r,i,j} * Ebar_{h,i,j}  with M the
 * positions the rule's block mask hides at length N (causal, invisible), evaluated on the
 * block-averaged influence of moa_attention_influence: a hidden block adds its mean times
 * its token-pair count (the token-level sum).  Rule windows: span = clamp(ceil(alpha +
 * beta * N), 0, N) (Eq. 2) rounded up to a whole block, window = span -
 * n_sink.
 *   e_blocks  device fp32 [heads, nb, nb], nb = ceil(N / block) (one batch entry of
 *             moa_attention_influence's output, averaged over calibration items).
 *   alpha, beta  host arrays of n_rules (1 <= n_rules <= 128) rules.
 *   n_sink    multiple of block; block 64.
 *   loss_out  device fp32 [heads, n_rules].
 * Stream-ordered, no allocation.
 */
moa_status moa_rule_losses(const float *e_blocks, int heads, int64_t N, int block, int n_sink,
                           const float *alpha, const float *beta, int n_rules, float *loss_out,
                           moa_stream_t stream);

/*
 * Rule selection (Eq. 5): one rule per head minimising
 * sum_h loss[h][r_h] subject to the mean density (1/H) sum_h density[r_h] <= density_budget
 * and at most max_rules_per_layer (1 or 2, "at most two per model layer")
 * distinct rules per layer.  Host only.  The paper solves this MIP (eq:mip)
 * with Gurobi; here it is solved EXACTLY: per layer, the Pareto frontier (density, loss) of
 * every rule subset of size <= 2 (for a pair, the best split of the heads by the exchange
 * argument), then the Pareto merge of the layers (a multiple-choice knapsack) with
 * admissible density / loss bounds.  Feasible means sum_h density <= budget * H + 1e-9.
 *   loss      host fp32 [layers * heads_per_layer][n_rules] (moa_rule_losses, one length).
 *   density   host fp32 [n_rules]: density of each rule at that length.
 *   rule_out  host int32 [layers * heads_per_layer]; loss_out / density_out nullable.
 * Errors: MOA_ERR_INVALID_ARG if no plan meets the budget (or a loss is not finite);
 *         MOA_ERR_UNSUPPORTED if the exact solver's frontier outgrows 2^24 partial plans.
 */
moa_status moa_plan_rules(const float *loss, const float *density, int layers, int heads_per_layer, int n_rules,
                          float density_budget, int max_rules_per_layer, int32_t *rule_out, float *loss_out,
                          float *density_out);

/* Prefill block-skip schedule (a2): the kv tiles (of MOA_TILE keys) that q-tile
 * `q_tile` (rows [q_tile*MOA_TILE, ...)) of local q-head h visits, in visit
 * order, with flags 1 = EDGE (needs the mask) / 0 = FULL.  *n_tiles is set
 * to the count; at most max_tiles entries are written. */
#define MOA_TILE 128
moa_status moa_prefill_tiles(const moa_ctx *ctx, int layer, int q_head_local, int q_tile,
                             int32_t *tiles, uint8_t *edge, int max_tiles, int32_t *n_tiles);
/* Work-item order of the prefill kernels: n_items (q_head_local, q_tile) pairs.
 * Heads by total kv-tile count, heaviest first; the q tiles of one head are
 * consecutive (concurrent CTAs share that head's K/V tiles in L2), heaviest
 * first.  items: 2 * max_items int32. */
moa_status moa_prefill_items(const moa_ctx *ctx, int layer, int32_t *items, int max_items,
                             int32_t *n_items);
/* Per-CTA schedule of the uniform bf16 two-tile prefill for a batch of max_batch
 * (moa_set_spans): the (q_head_local | b << 16, q_block of 2*MOA_TILE rows) entries
 * of every (work item, sequence), grouped by CTA -- greedy list scheduling of the
 * item order above, each entry to the least-loaded CTA by its kv-tile steps; CTA c
 * runs entries [offsets[c], offsets[c + 1]).  *n_ctas and *n_entries are set; at
 * most max_entries entries (2 int32 each) and max_ctas + 1 offsets are written
 * (NULL buffers: counts only).  The kernel launches *n_ctas CTAs when the batch is
 * max_batch and MOA_PP_SCHED is not 0, else it walks the item list round robin. */
moa_status moa_prefill_schedule(const moa_ctx *ctx, int layer, int32_t *entries, int max_entries,
                                int32_t *offsets, int max_ctas, int32_t *n_entries, int32_t *n_ctas);
/* Decode work list: n chunks of (group_local, row_begin, row_end). */
moa_status moa_decode_chunks(const moa_ctx *ctx, int layer, int32_t *chunks, int max_chunks,
                             int32_t *n_chunks);
/* Next position the layer expects to append (N after prefill/fill). */
moa_status moa_next_pos(const moa_ctx *ctx, int layer, int64_t *pos);

#ifdef __cplusplus
}
#endif
#endif /* MOA_H_ */
