/*
 * veda.h -- C ABI of the B200 (sm_100a) hot path of Veda (arXiv 2605.30325):
 * distilled tile-sparse self-attention for video DiTs.
 *
 * The path (Alg. 2, followed by Eq. 2):
 *   veda_tile_permute   head-aware 3D tiling
 *   veda_tile_score     TripPool + phi_q/phi_k + S_pred    (Eqs. 5-6)
 *   veda_select_topk    exactly-k kept key tiles per row
 *   veda_sparse_attn_fwd tile-skipping attention
 *   veda_tile_unpermute  back to token order
 * and the forms the token-layout path runs: veda_tile_pool_qk
 * (tiling + TripPool of Q and K straight from token order, one launch),
 * veda_tile_select_pooled (phi, S_pred and top-k per chunk of heads: no full score
 * tensor), veda_sparse_attn_fwd_tokens (tiles gathered from / rows stored to token order).
 *
 * Conventions for every call
 *   - Pointers are DEVICE pointers unless marked "host".  bf16 tensors are passed
 *     as uint16_t bit patterns.  All device pointers must be 16-byte aligned.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls only
 *     enqueue work and return; they never allocate or free device memory and keep
 *     no pointer after returning.  Host arrays are read during the call only.  The
 *     caller owns every buffer (workspace sizes come from the *_workspace helpers).
 *     Exceptions, all one-time or bounded: the first scoring call on a device uploads
 *     a 12 KB constant table (Phi for the GELU) into the library's static device
 *     memory and synchronises `stream` once; veda_sparse_attention_host creates two
 *     side streams per device on first use and a few events per call;
 *     veda_tile_select_pooled with several head chunks runs its top-k on one library side
 *     stream per device (created on first use, a few events per call) and makes `stream`
 *     wait for it before returning control of the work to `stream`.
 *   - Errors are returned as veda_status; nothing is printed, thrown or aborted.
 *     Arguments (NULL pointers, shapes including empty ones, k range, alignment) are
 *     validated before the first device call, so they report the same status with or
 *     without a GPU.  veda_last_error() gives a thread-local detail string for the
 *     last failure.  Faults inside a kernel surface later on the stream as CUDA errors.
 *   - Debug mode (veda_set_debug(1), or VEDA_DEBUG=1 in the environment at library
 *     load): the attention, top-k and pooling entry points first validate their inputs
 *     on the device -- kept-tile lists in [0, n_tiles) and strictly ascending (exactly k
 *     distinct tiles; reading R11), bf16 inputs finite, scores not NaN
 *     -- synchronise `stream`, and return VEDA_ERR_INDEX / VEDA_ERR_NONFINITE before
 *     launching anything else.  Off by default (no validation, no synchronisation).
 *     Whatever the mode, the attention kernels clamp every list entry into [0, n_tiles):
 *     a bad list gives wrong outputs but never a read outside the head's tiles.
 *   - Supported: B = p_t*p_h*p_w in {64, 128}; d in {64, 128}; 1 <= k <= n_tiles;
 *     Hh <= 1024 heads per call.  Device must be sm_100 (B200).
 *
 * Layouts (Hh = heads in the call; N = T*H*W; N_T = n_tiles; MW = B/32)
 *   token tensor   x[h][n][c] at x + h*head_stride + n*token_stride + c (elements)
 *   tiled tensor   [Hh][N_T][B][d] bf16, tile-contiguous (B*d*2 bytes per tile)
 *   tile_count     [Hh][N_T] int32  real tokens per tile
 *   slot_mask      [Hh][N_T][MW] uint32, bit b of a tile set iff slot b is real
 *   scores         [Hh][N_T][N_T] fp32 (the two-call and tiled forms; the path's fused
 *                  select holds only a chunk of heads at a time)
 *   idx            [Hh][N_T][k] int32, kept key tiles of each query tile, ascending
 */
#ifndef VEDA_H_
#define VEDA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define VEDA_API __attribute__((visibility("default")))
#else
#define VEDA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    VEDA_OK = 0,
    VEDA_ERR_NULL = 1,       /* required pointer is NULL                          */
    VEDA_ERR_SHAPE = 2,      /* dimension mismatch / unsupported size             */
    VEDA_ERR_CONFIG = 3,     /* p_t*p_h*p_w differs across heads or B unsupported */
    VEDA_ERR_K_RANGE = 4,    /* k outside [1, n_tiles]                            */
    VEDA_ERR_ALIGN = 5,      /* pointer or stride not 16-byte aligned             */
    VEDA_ERR_WORKSPACE = 6,  /* workspace too small                               */
    VEDA_ERR_INDEX = 7,      /* (debug mode) bad kept-tile list                    */
    VEDA_ERR_NONFINITE = 8,  /* (debug mode) Inf/NaN input or NaN score            */
    VEDA_ERR_CUDA = 9,       /* CUDA runtime / driver error at launch             */
    VEDA_ERR_ARCH = 10       /* current device is not sm_100                      */
} veda_status;

/* real latent grid (T, H, W); tokens are flattened raster n = (t*H + h)*W + w
 * (reading R1) */
typedef struct { int32_t t, h, w; } veda_latent;

/* per-head tile shape pi_{l,h} = (p_t, p_h, p_w), p_t*p_h*p_w = B (Eq. 8) */
typedef struct { int32_t pt, ph, pw; } veda_tile_cfg;

/* padded grid shared by all heads of a call (reading R4/R5) */
typedef struct {
    int32_t tp, hp, wp;   /* padded extents: each axis ceil-padded to the lcm of its tile extents */
    int32_t B;            /* tile size                                                           */
    int32_t n_tiles;      /* N_T = tp*hp*wp / B                                                  */
    int32_t reserved;
    int64_t n_pad;        /* tp*hp*wp                                                            */
} veda_tiled_shape;

/* statistic-aware estimator weights, one set per head (Eq. 6;
 * DESIGN.md reading R8).  Host struct holding DEVICE fp32 arrays:
 *   w1 [Hh][d_in][d_hidden], b1 [Hh][d_hidden], w2 [Hh][d_hidden][d_lat], b2 [Hh][d_lat]
 * for the query side (..q) and the key side (..k).  d_in must be 3*d.
 * phi(z) = GELU(z w1 + b1) w2 + b2, GELU(x) = x*Phi(x) (erf form). */
typedef struct {
    int32_t d_in, d_hidden, d_lat;
    const float *w1q, *b1q, *w2q, *b2q;
    const float *w1k, *b1k, *w2k, *b2k;
    /* optional (NULL: none): the device buffer veda_scorer_prepare filled from THESE
     * weights for the same Hh; the scoring calls then skip splitting W1 and W2 on every
     * call (inference weights are static).  Refill it if the weights change.        */
    const void *prepared;
} veda_scorer;

/* ---- host helpers ----------------------------------------------------------- */

/* Padded grid of a call.  cfg: host [Hh].  PAPER.md:143-145, 288-294; 61x45x80 with
 * (4,4,8) gives 64x48x80 = 245,760 tokens. */
VEDA_API veda_status veda_tiled_shape_of(veda_latent lat, const veda_tile_cfg *cfg, int32_t Hh,
                                veda_tiled_shape *out /* host */);

/* k = floor((1 - sparsity) * n_tiles + 1/2) clamped to [1, n_tiles] (reading R12). */
VEDA_API int32_t veda_k_for_sparsity(int32_t n_tiles, double sparsity);

/* Prepared scorer weights (phi's W1 and W2 of both sides as INT8 digit images + row
 * exponents, the B operands of the Ozaki GEMMs, see veda_tile_score): bytes for Hh heads,
 * and the fill (enqueued on stream; prepared is a caller-owned device buffer).  Results
 * with and without w->prepared are bit-identical.                                    */
VEDA_API veda_status veda_scorer_prepare_bytes(int32_t Hh, int32_t d, const veda_scorer *w /* host */,
                                               size_t *bytes /* host */);
VEDA_API veda_status veda_scorer_prepare(int32_t Hh, int32_t d, const veda_scorer *w /* host */, void *prepared,
                                         size_t bytes, void *stream);

/* Bytes of workspace veda_tile_score needs. */
VEDA_API veda_status veda_tile_score_workspace(int32_t Hh, int32_t n_tiles, int32_t d,
                                      const veda_scorer *w /* host */, size_t *bytes /* host */);

/* ---- the five steps of the path ------------------------------------------------ */

/* Step 1: head-aware 3D tiling (Alg. 2; Eq. 8).
 * Tile i of head h is the box (i_t,i_h,i_w) in raster order of boxes; slot j inside
 * it is (dt,dh,dw) in raster order, t slowest (readings R2, R3).  Padded slots are
 * written as +0 (R4).  tile_count / slot_mask may be NULL (skipped).
 *   x        : token tensor, strides in elements, multiples of 8
 *   x_tiled  : [Hh][N_T][B][d]                                                        */
VEDA_API veda_status veda_tile_permute(const uint16_t *x, int64_t head_stride, int64_t token_stride,
                              veda_latent lat, const veda_tile_cfg *cfg /* host [Hh] */,
                              int32_t Hh, int32_t d, uint16_t *x_tiled, int32_t *tile_count,
                              uint32_t *slot_mask, void *stream);

/* Step 2: statistics-aware tile scoring, Alg. 2:
 *   z = Avg (+) Max (+) Min over each tile's real tokens (Eq. 5; readings R6, R7),
 *   e = phi(z) per head and side, S_ij = e_q,i . e_k,j / sqrt(d_lat) (Eq. 6),
 *   S_ij = -inf when key tile j has no real token (R5).
 * Pooling sums and both GEMMs accumulate in fp64 (reading R17); scores are rounded
 * once to fp32.  Equals veda_trippool x2 -> veda_project x2 -> veda_pair_scores.
 *   tile_count, slot_mask : from veda_tile_permute (identical for Q and K)
 *   scores : [Hh][N_T][N_T] fp32;  workspace : >= veda_tile_score_workspace bytes   */
VEDA_API veda_status veda_tile_score(const uint16_t *q_tiled, const uint16_t *k_tiled,
                            const int32_t *tile_count, const uint32_t *slot_mask, int32_t Hh,
                            int32_t n_tiles, int32_t B, int32_t d, const veda_scorer *w /* host */,
                            float *scores, void *workspace, size_t workspace_bytes, void *stream);

/* Step 3: per-query-tile top-k (Alg. 2).  Exactly k
 * key tiles per row: order by (S descending, j ascending), keep the first k, emit
 * ascending (readings R10, R11, R16: -0.0 == +0.0).  Decided on the fp32 scores.  */
VEDA_API veda_status veda_select_topk(const float *scores, int32_t Hh, int32_t n_tiles, int32_t k,
                             int32_t *idx, void *stream);

/* Step 4: tile-skipping attention forward, Eq. 2: for each
 * (head, query tile i) O_i = softmax(Q~_i K^_i^T * scale) V^_i over the k kept tiles
 * idx[i]; padded key slots are -inf, padded query rows are written as 0 (R4).
 * bf16 operands, fp32 accumulation (tcgen05 / TMEM), P rounded to bf16 for P.V,
 * output bf16 (R15).  softmax_scale <= 0 selects 1/sqrt(d).  lse (natural log,
 * [Hh][N_T][B] fp32) may be NULL.                                                  */
VEDA_API veda_status veda_sparse_attn_fwd(const uint16_t *q_tiled, const uint16_t *k_tiled,
                                 const uint16_t *v_tiled, const int32_t *idx,
                                 const uint32_t *slot_mask, int32_t Hh, int32_t n_tiles,
                                 int32_t B, int32_t d, int32_t k, float softmax_scale,
                                 uint16_t *o_tiled, float *lse, void *stream);

/* Step 5: untiling: o[token] = o_tiled[tile][slot] for every real
 * slot; padded slots are dropped.                                                    */
VEDA_API veda_status veda_tile_unpermute(const uint16_t *o_tiled, veda_latent lat,
                                const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh, int32_t d,
                                uint16_t *o, int64_t head_stride, int64_t token_stride,
                                void *stream);

/* ---- the path straight on the token layout (no tiled copies) ---- */

/* TripPool of every tile of x, read straight from the token tensor (Alg. 2,
 * Eq. 5): z [Hh][N_T][3d] fp32 exactly as veda_tile_permute + veda_trippool compute it
 * (bit-identical), plus tile_count [Hh][N_T] and slot_mask [Hh][N_T][B/32] as
 * veda_tile_permute writes them (either may be NULL).  x, strides: as veda_tile_permute. */
VEDA_API veda_status veda_tile_pool(const uint16_t *x, int64_t head_stride, int64_t token_stride,
                                    veda_latent lat, const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh,
                                    int32_t d, float *z, int32_t *tile_count, uint32_t *slot_mask, void *stream);

/* veda_tile_pool of Q and K in ONE launch (same strides, layout and tile configs): zq, zk
 * [Hh][N_T][3d]; tile_count / slot_mask (may be NULL) from q -- identical for k.  The
 * persistent pooling kernel streams both tensors' tiles, so the second tensor pays no
 * launch gap or ramp-up; results are bit-identical to two veda_tile_pool calls.       */
VEDA_API veda_status veda_tile_pool_qk(const uint16_t *q, const uint16_t *k, int64_t head_stride,
                                       int64_t token_stride, veda_latent lat,
                                       const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh, int32_t d,
                                       float *zq, float *zk, int32_t *tile_count, uint32_t *slot_mask,
                                       void *stream);

/* veda_tile_pool for the heads [head_begin, head_end) of an Hh-head call: the padded grid
 * (hence n_tiles and every tile) is the whole call's -- the lcm of ALL Hh heads' tile
 * extents -- and z / tile_count / slot_mask are the whole call's arrays, of which only the
 * rows of heads in the range are written, bit-identical to veda_tile_pool's.  A rank of a
 * (head x query tile) unit share pools the heads its units touch with it.
 * 0 <= head_begin <= head_end <= Hh, else VEDA_ERR_SHAPE; an empty range enqueues nothing. */
VEDA_API veda_status veda_tile_pool_heads(const uint16_t *x, int64_t head_stride, int64_t token_stride,
                                          veda_latent lat, const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh,
                                          int32_t d, int32_t head_begin, int32_t head_end, float *z,
                                          int32_t *tile_count, uint32_t *slot_mask, void *stream);

/* Step 4 + step 5 on the token layout: Eq. 2 for every (head, query
 * tile), the query tile and the kept key / value tiles fetched straight from q, k, v in
 * token order by one TMA box per tile (padded slots zero-filled, reading R4), and each
 * output row stored straight to its token (UnTile).  Bit-identical to
 * veda_tile_permute x3 -> veda_sparse_attn_fwd -> veda_tile_unpermute.
 *   q, k, v : token tensors sharing head_stride / token_stride (elements, multiples of 8;
 *             they may be equal only when one of them is unused: one token or one head)
 *   idx [Hh][N_T][k_keep], slot_mask [Hh][N_T][B/32] : as for veda_sparse_attn_fwd
 *   o       : token tensor (o_head_stride, o_token_stride); rows of padded slots are not
 *             written;  lse : [Hh][N_T][B] fp32 (tiled order) or NULL.
 * Heads of one call may use any tile shapes (at most 8 distinct shapes per kernel launch;
 * larger sets are split into several launches).                                         */
VEDA_API veda_status veda_sparse_attn_fwd_tokens(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                                 int64_t head_stride, int64_t token_stride, veda_latent lat,
                                                 const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh, int32_t d,
                                                 const int32_t *idx, const uint32_t *slot_mask, int32_t k_keep,
                                                 float softmax_scale, uint16_t *o, int64_t o_head_stride,
                                                 int64_t o_token_stride, float *lse, void *stream);

/* The same for the units [unit_begin, unit_end) of the flattened (head, query tile) space
 * (unit u = h * n_tiles + i; SURVEY.md §8(e)'s finer multi-GPU share, for head counts that
 * do not divide the GPU count).  All tensors are the full call's; only the output rows
 * (and lse rows) of tokens in the range's query tiles are written, each exactly as the
 * full call writes them, so the shares of a partition of [0, Hh*n_tiles) together produce
 * the full call's output bit for bit.  0 <= unit_begin <= unit_end <= Hh*n_tiles, else
 * VEDA_ERR_SHAPE; an empty range enqueues nothing. */
VEDA_API veda_status veda_sparse_attn_fwd_tokens_units(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                                       int64_t head_stride, int64_t token_stride, veda_latent lat,
                                                       const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh,
                                                       int32_t d, const int32_t *idx, const uint32_t *slot_mask,
                                                       int32_t k_keep, float softmax_scale, uint16_t *o,
                                                       int64_t o_head_stride, int64_t o_token_stride, float *lse,
                                                       int32_t unit_begin, int32_t unit_end, void *stream);

/* The heads [head_begin, head_end) of an Hh-head call, with every tensor holding THOSE heads
 * only (head 0 of x / z / tile_count / slot_mask / q / k / v / idx / o / lse is global head
 * head_begin): the sequence-parallel (Ulysses) rank's head shard.  cfg lists all Hh heads, so
 * the padded grid, n_tiles and the tiles are the whole call's (with head-aware tiling a head
 * subset's own grid can differ) and the results are bit-identical to the same heads of the
 * whole call.  0 <= head_begin <= head_end <= Hh, else VEDA_ERR_SHAPE; an empty range enqueues
 * nothing.  Other arguments as veda_tile_pool / veda_sparse_attn_fwd_tokens. */
VEDA_API veda_status veda_tile_pool_local(const uint16_t *x, int64_t head_stride, int64_t token_stride,
                                          veda_latent lat, const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh,
                                          int32_t d, int32_t head_begin, int32_t head_end, float *z,
                                          int32_t *tile_count, uint32_t *slot_mask, void *stream);
VEDA_API veda_status veda_sparse_attn_fwd_tokens_local(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                                       int64_t head_stride, int64_t token_stride, veda_latent lat,
                                                       const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh,
                                                       int32_t d, int32_t head_begin, int32_t head_end,
                                                       const int32_t *idx, const uint32_t *slot_mask, int32_t k_keep,
                                                       float softmax_scale, uint16_t *o, int64_t o_head_stride,
                                                       int64_t o_token_stride, float *lse, void *stream);

/* ---- the whole path on HOST buffers (end-to-end call) ------------------------------ */

/* Device workspace veda_sparse_attention_host needs (two buffer sets of one head chunk:
 * token-layout Q/K/V/O, tiled Q/K/V/O, counts, masks, scores, index lists, scorer
 * workspace).  heads_per_chunk <= 0 selects the default ceil(Hh/32).                  */
VEDA_API veda_status veda_sparse_attention_host_workspace(veda_latent lat, const veda_tile_cfg *cfg /* host [Hh] */,
                                                          int32_t Hh, int32_t d, int32_t k,
                                                          const veda_scorer *w /* host */,
                                                          int32_t heads_per_chunk, size_t *bytes /* host */);

/* Steps 1-5 for Q/K/V in HOST memory, output to HOST memory: the call a DiT layer makes
 * when its activations are not resident on the GPU.  Heads are independent (PAPER.md:270,
 * Alg. 2), so the heads are processed in chunks of heads_per_chunk through
 * two device buffer sets: the H2D copy of chunk c+1, the five steps on chunk c (on
 * `stream`) and the D2H copy of chunk c-1 overlap (two library-owned side streams,
 * ordered against `stream` by events).  Every chunk is tiled on the padded grid of the
 * whole call, so o_host is bit-identical to veda_tile_permute .. veda_tile_unpermute on
 * all Hh heads with the same k.
 *   q_host, k_host, v_host, o_host : host bf16, dense [Hh][N][d] (head_stride = N*d,
 *       token_stride = d) or dense [N][Hh][d] (head_stride = d, token_stride = Hh*d);
 *       page-locked memory is needed for the copies to overlap.  The inputs are read and
 *       o_host written asynchronously: valid only after `stream` is synchronised.
 *   w : scorer weights of all Hh heads (device arrays, as for veda_tile_score)
 *   workspace : device, >= veda_sparse_attention_host_workspace bytes, 16-byte aligned */
VEDA_API veda_status veda_sparse_attention_host(const uint16_t *q_host, const uint16_t *k_host,
                                                const uint16_t *v_host, int64_t head_stride,
                                                int64_t token_stride, veda_latent lat,
                                                const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh,
                                                int32_t d, int32_t k, const veda_scorer *w /* host */,
                                                int32_t heads_per_chunk, uint16_t *o_host, void *workspace,
                                                size_t workspace_bytes, void *stream);

/* ---- fused forms used by the composed path (same results as the unfused calls) ---- */

/* veda_tile_permute + TripPool of the tiled tensor in ONE pass over HBM (the statistics
 * are taken from the values already in registers): z [Hh][N_T][3d] fp32 as veda_trippool
 * computes it.  Used for Q and K (Alg. 2).                     */
VEDA_API veda_status veda_tile_permute_pool(const uint16_t *x, int64_t head_stride, int64_t token_stride,
                                            veda_latent lat, const veda_tile_cfg *cfg /* host [Hh] */,
                                            int32_t Hh, int32_t d, uint16_t *x_tiled, int32_t *tile_count,
                                            uint32_t *slot_mask, float *z, void *stream);

/* veda_tile_score from precomputed TripPool descriptors zq, zk [Hh][N_T][3d] fp32
 * (phi_q, phi_k and S_pred, Eq. 6); same workspace as veda_tile_score.               */
VEDA_API veda_status veda_tile_score_pooled(const float *zq, const float *zk, const int32_t *tile_count,
                                            int32_t Hh, int32_t n_tiles, int32_t d,
                                            const veda_scorer *w /* host */, float *scores, void *workspace,
                                            size_t workspace_bytes, void *stream);

/* Steps 2 + 3 fused at the boundary ("tighter
 * kernel-level fusion to reduce mask preparation overhead"): the kept-tile lists idx
 * [Hh][N_T][k] straight from the pooled descriptors, with no [Hh][N_T][N_T] score tensor.
 * phi_q / phi_k (Eq. 6) run for all heads; then, per chunk of heads_per_chunk heads
 * (0: as many as fit 128 MB of fp32 scores -- 8 of Waver's 24), S_pred (Eq. 6) is written
 * to a chunk-sized scratch in the workspace and the top-k of veda_select_topk
 * reads it back; with several chunks the scratch is double-
 * buffered and the top-k of chunk c runs on a library side stream while the score GEMM
 * of chunk c+1 runs on `stream` (the caller's stream is made to wait for the last one).  idx is bit-identical to
 * veda_tile_score_pooled followed by veda_select_topk for any chunking.
 * Errors: VEDA_ERR_K_RANGE (k outside [1, n_tiles]), VEDA_ERR_WORKSPACE, as
 * veda_tile_score_pooled otherwise; debug mode also checks every score chunk.       */
VEDA_API veda_status veda_tile_select_workspace(int32_t Hh, int32_t n_tiles, int32_t d,
                                                const veda_scorer *w /* host */, int32_t heads_per_chunk,
                                                size_t *bytes /* host */);
VEDA_API veda_status veda_tile_select_pooled(const float *zq, const float *zk, const int32_t *tile_count,
                                             int32_t Hh, int32_t n_tiles, int32_t d,
                                             const veda_scorer *w /* host */, int32_t k,
                                             int32_t heads_per_chunk, int32_t *idx, void *workspace,
                                             size_t workspace_bytes, void *stream);

/* ---- sub-steps of veda_tile_score (exported for parity tests and profiling) ---- */

/* TripPool (Eq. 5): z [Hh][N_T][3d] fp32 = Avg | Max | Min over real slots; the Avg
 * sum is accumulated in fp64 and rounded once.  Empty tiles give z = 0.            */
VEDA_API veda_status veda_trippool(const uint16_t *x_tiled, const uint32_t *slot_mask, int32_t Hh,
                          int32_t n_tiles, int32_t B, int32_t d, float *z, void *stream);

/* phi (Eq. 6): e [Hh][N_T][d_lat] fp64 = GELU(z w1 + b1) w2 + b2 with fp64
 * accumulation.  hidden: fp64 scratch [Hh][N_T][d_hidden].                          */
VEDA_API veda_status veda_project(const float *z, int32_t Hh, int32_t n_tiles, int32_t d_in,
                         int32_t d_hidden, int32_t d_lat, const float *w1, const float *b1,
                         const float *w2, const float *b2, double *hidden, double *e,
                         void *stream);

/* S_ij = e_q,i . e_k,j / sqrt(d_lat) (fp64 accumulate, fp32 store), -inf for empty
 * key tiles (tile_count == 0).                                                       */
VEDA_API veda_status veda_pair_scores(const double *eq, const double *ek, const int32_t *tile_count,
                             int32_t Hh, int32_t n_tiles, int32_t d_lat, float *scores,
                             void *stream);

/* ---- oracle tile mask and recall -------------------------- */

/* Exact pooled target scores, Eq. 4 (Alg. 3):
 *   S_tgt[h][i][j] = max over real (u in tile i, v in tile j) of A*_uv,
 *   A* = softmax(Q K^T * scale) over ALL real keys of head h,
 * computed as exp(max_u(max_v s_uv * scale - lse_u)) -- the second of the two passes of
 * PAPER.md:412-416.  lse [Hh][N_T][B] fp32 (natural log) is pass 1: the lse output of
 * veda_sparse_attn_fwd run densely (k = N_T, idx[i] = 0..N_T-1) on the same q/k.
 * Empty key tile -> -inf; query tile without real tokens -> 0 (readings R4, R5, R19).
 * bf16 operands, fp32 accumulation (tcgen05 / TMEM); softmax_scale <= 0 -> 1/sqrt(d).
 *   s_tgt : [Hh][N_T][N_T] fp32 (device).  B in {64, 128}, d in {64, 128}.
 * Feeding s_tgt to veda_select_topk gives the oracle mask M~* (Eq. 4).      */
VEDA_API veda_status veda_target_scores(const uint16_t *q_tiled, const uint16_t *k_tiled,
                               const uint32_t *slot_mask, const float *lse, int32_t Hh,
                               int32_t n_tiles, int32_t B, int32_t d, float softmax_scale,
                               float *s_tgt, void *stream);

/* Tile recall, Eq. 3: Recall@k = mean over query tiles i of
 * |S_sp,i intersect S_fu,i| / k, over the rows whose tile_count > 0 (R4; tile_count
 * may be NULL = all rows).  idx_sp / idx_fu : [rows][k] int32 key-tile lists (any order,
 * no duplicates; entries outside [0, n_tiles) never match).  recall : one fp64 on the
 * DEVICE (0 when no row counts).  Integer counts, one fp64 division: deterministic.  */
VEDA_API veda_status veda_tile_recall(const int32_t *idx_sp, const int32_t *idx_fu,
                             const int32_t *tile_count, int64_t rows, int32_t n_tiles,
                             int32_t k, double *recall, void *stream);

/* ---- head-aware tiling search support (Alg. 1, Eq. 8-9) -------- */

/* Per-token fp32 values -> tiled layout of `cfg` (same boxes/slots as veda_tile_permute):
 * x_tiled[h][i][b] = x[h*head_stride + n(h,i,b)], `pad` for padded slots.  Used to carry
 * the full-attention row lse (a property of the token, not of the tiling, PAPER.md:
 * 647-648) into each candidate tiling of Alg. 1, so one dense pass serves all of Omega.
 *   x : [Hh][N] (head_stride >= N), x_tiled : [Hh][N_T][B]                              */
VEDA_API veda_status veda_tile_permute_scalar(const float *x, int64_t head_stride, veda_latent lat,
                                     const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh,
                                     float pad, float *x_tiled, void *stream);

/* Inverse on real slots: x[h*head_stride + n] = x_tiled[h][i][b]; padded slots dropped. */
VEDA_API veda_status veda_tile_unpermute_scalar(const float *x_tiled, veda_latent lat,
                                       const veda_tile_cfg *cfg /* host [Hh] */, int32_t Hh,
                                       float *x, int64_t head_stride, void *stream);

/* Alg. 1: err[h] += sum_e (a[h][e] - b[h][e])^2 over n bf16 elements per head
 * (a, b at a + h*head_stride; n and head_stride multiples of 8).  Differences and squares
 * are exact in fp64; partial sums fp64 (per-CTA partials combined with fp64 atomics, so
 * run-to-run differences are at the 1e-16 relative level).  err : [Hh] fp64, device,
 * ACCUMULATED (zero it to start a calibration set).                                    */
VEDA_API veda_status veda_sq_err(const uint16_t *a, const uint16_t *b, int64_t head_stride,
                        int64_t n, int32_t Hh, double *err, void *stream);

/* ---- input validation (what debug mode runs) ---------------------- */

/* bits OR-ed into the device flag word by the validation calls */
#define VEDA_FLAG_INDEX_RANGE 1u  /* an entry outside [0, n_tiles)                        */
#define VEDA_FLAG_INDEX_ORDER 2u  /* a row not strictly ascending: a duplicate or descent  */
#define VEDA_FLAG_NONFINITE 4u    /* an Inf/NaN bf16 input, or a NaN score               */

/* Kept-tile lists idx [rows][k] (as veda_select_topk writes them): ORs
 * VEDA_FLAG_INDEX_RANGE / VEDA_FLAG_INDEX_ORDER into *flags (a DEVICE uint32 the caller
 * zeroes; it is only ever OR-ed).  Enqueues and returns (no synchronisation).           */
VEDA_API veda_status veda_validate_index(const int32_t *idx, int64_t rows, int32_t n_tiles, int32_t k,
                                         uint32_t *flags, void *stream);

/* bf16 token tensor x[h][n][c] (strides in elements, multiples of 8; d multiple of 8):
 * ORs VEDA_FLAG_NONFINITE into *flags if any element is Inf or NaN.  A tiled tensor
 * [Hh][N_T][B][d] is the case n = N_T*B, head_stride = n*d, token_stride = d.           */
VEDA_API veda_status veda_validate_finite(const uint16_t *x, int64_t head_stride, int64_t token_stride,
                                          int32_t Hh, int64_t n, int32_t d, uint32_t *flags, void *stream);

/* Debug mode on (1) / off (0) for the whole process; returns the previous setting. */
VEDA_API int32_t veda_set_debug(int32_t on);

/* ---- diagnostics ------------------------------------------------------------------ */
VEDA_API const char *veda_status_str(veda_status st);
VEDA_API const char *veda_last_error(void);
/* Kernels launched by this library since load (process-wide counter). */
VEDA_API uint64_t veda_launch_count(void);
/* VEDA_OK iff the current CUDA device is sm_100 and usable. */
VEDA_API veda_status veda_check_device(void);

#ifdef __cplusplus
}
#endif
#endif /* VEDA_H_ */
