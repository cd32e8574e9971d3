/*
 * dicm_b200.h -- C ABI of the B200 (sm_100a) DICM / AMS training hot path.
 *
 * The reference (arxiv 1711.06505 re-implementation, package `dicm`) is pure
 * Python/numpy and has no FFI; its "operator API" is the Python call chain
 * LocalTrainer.train_batch -> encode_batch -> logits_graph -> backward -> Adam
 * (reference training.py:66-91).  Each entry point below replaces one link of
 * that chain and cites the reference code it stands in for.  The Python host
 * package (paper_1711_06505_b200) binds these with ctypes; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Conventions
 *  - every pointer is caller-owned DEVICE memory unless noted; sizes are
 *    explicit; nothing is allocated inside a call;
 *  - calls are asynchronous on `stream` (a cudaStream_t) and thread-safe across
 *    distinct streams;
 *  - data-dependent counts (unique keys, unique rows) stay on the device
 *    (`*_dev` int32 pointers) so a whole step runs without host round trips;
 *  - the return value is a status code; dicm_last_error() describes the last
 *    failure of the calling thread;
 *  - device-side faults (out-of-vocabulary ids, non-finite loss/gradients) are
 *    latched into the caller's int32 `status[DICM_STATUS_WORDS]` buffer and
 *    surface when the host reads it (the reference raises KeyError at
 *    model.py:127-129 / images.py:89-94 and FloatingPointError at
 *    training.py:75-76 / optim.py:53-54).
 */
#ifndef DICM_B200_H
#define DICM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* dicm_stream_t; /* cudaStream_t */

/* status codes (python side maps them to the reference's exception types) */
#define DICM_OK 0
#define DICM_ERR_CUDA 1        /* RuntimeError */
#define DICM_ERR_SHAPE 2       /* ShapeError (ValueError), autograd.py:18-19 */
#define DICM_ERR_KEY 3         /* KeyError, model.py:127-129 */
#define DICM_ERR_VALUE 4       /* ValueError */
#define DICM_ERR_FLOAT 5       /* FloatingPointError, optim.py:53-54 */
#define DICM_ERR_UNSUPPORTED 6 /* NotImplementedError */

/* device status words */
#define DICM_STATUS_WORDS 8
#define DICM_ST_KEY_FLAG 0     /* != 0: an id was outside its vocabulary */
#define DICM_ST_KEY_VALUE 1    /* the offending id */
#define DICM_ST_KEY_SEG 2      /* which key segment it came from */
#define DICM_ST_NONFINITE 3    /* bit 1: loss, bit 2: dense grad, bit 4: row grad */

/* pool element types */
#define DICM_POOL_F32 0
#define DICM_POOL_BF16 1

/* image-MLP layer-0 arithmetic */
#define DICM_PREC_FP32 0   /* CUDA-core fp32 (strict parity mode) */
#define DICM_PREC_TF32 1   /* tcgen05 kind::tf32 on an fp32 pool */
#define DICM_PREC_BF16 2   /* tcgen05 kind::f16 (bf16) on a bf16 pool */

const char* dicm_last_error(void);
int dicm_version(void);
/* returns the device's SM major*10+minor, or <0 if no usable device */
int dicm_device_arch(void);

/* ------------------------------------------------------------------------
 * a2: per-batch key dedup with inverse index.
 * Replaces np.unique(np.concatenate(needed)) (reference model.py:187),
 * np.searchsorted(unique, ids) (model.py:374, 378) and Batch.unique_field_ids
 * (model.py:152-155).  Keys of several segments share one key space: segment
 * s maps id -> base_s + id, ids must lie in [0, vocab_s) (else status KEY).
 * Output: sorted distinct global keys uniq[0..*count_dev) and, for every input
 * id, inv[inv_off_s + j] = position of its key in uniq.  Bit-exact with numpy.
 * An id outside its vocabulary latches status[KEY_FLAG], the id and
 * KEY_SEG = tag * 16 + s; its inverse entry is set to 0 (a safe index) and
 * every later update kernel of the step refuses to run.
 * ---------------------------------------------------------------------- */
typedef struct {
  const int32_t* ids;
  int64_t n;
  int64_t base;
  int64_t vocab;
  int64_t inv_off;
} dicm_keyseg_t;

size_t dicm_dedup_workspace(int64_t key_space);
int dicm_dedup(const dicm_keyseg_t* segs, int nseg, int64_t key_space, void* workspace,
               size_t workspace_bytes, int32_t* uniq_out, int32_t* inv_out, int32_t* count_dev,
               int32_t tag, int32_t* status, dicm_stream_t stream);
/* inv_out = NULL above leaves the inverse to this call, which may run on
 * another stream (after dicm_dedup, before the workspace is reused): the
 * step launches the image-MLP forward on the unique keys while the inverse
 * (needed only by the per-sample kernels) is formed beside it. */
int dicm_dedup_inverse(const dicm_keyseg_t* segs, int nseg, int64_t key_space, const void* workspace,
                       size_t workspace_bytes, int32_t* inv_out, dicm_stream_t stream);

/* ------------------------------------------------------------------------
 * a3: the image pool -- 4096-d feature rows resident in HBM.
 * materialize: rows[p] = round(tanh(latent[p] . proj^T)) computed in fp64, the
 *   frozen extractor of reference images.py:48-71 (FixedExtractor.extract).
 * gather: out[i] = rows[row_ids[i]] as fp32 for i < *count_dev (bit-exact);
 *   reference images.py:96-101 (ImageFeatureStore.raw_features).
 * ---------------------------------------------------------------------- */
int dicm_pool_materialize(const float* latents, const double* proj, int64_t rows, int d_raw,
                          int latent_dim, void* pool, int pool_dtype, dicm_stream_t stream);
int dicm_pool_gather(const void* pool, int pool_dtype, int d_raw, const int32_t* row_ids,
                     const int32_t* count_dev, int64_t n_max, float* out, dicm_stream_t stream);

/* ------------------------------------------------------------------------
 * a4/a5: the image MLP d_raw -> 256 -> 64 -> 12 (reference model.py:108-120,
 * image_net_apply) and its reverse path (autograd.py:201-204, 222-225;
 * distributed: ServerNode.local_model_gradient runtime.py:169-201).
 * Rows are pool rows rows[0..*count_dev); weights are [out, in] row-major.
 * fwd writes the pre-activations act0 [n,256], act1 [n,64] and the
 * embeddings emb [n,12].  bwd consumes demb [n,12] and writes the gradients
 * of all img/ parameters (overwriting).  The input gradient of layer 0 is not
 * formed (the features are frozen; the reference computes and drops it).
 * ---------------------------------------------------------------------- */
typedef struct {
  const float *w0, *b0, *a0, *w1, *b1, *a1, *w2, *b2;
} dicm_imgmlp_params_t;
typedef struct {
  float *w0, *b0, *a0, *w1, *b1, *a1, *w2, *b2;
} dicm_imgmlp_grads_t;

size_t dicm_imgmlp_workspace(int64_t rows_max, int d_raw, int precision);
int dicm_imgmlp_fwd(const void* pool, int pool_dtype, int d_raw, const int32_t* rows,
                    const int32_t* count_dev, int64_t rows_max, const dicm_imgmlp_params_t* p,
                    float* act0, float* act1, float* emb, int precision, void* workspace,
                    size_t workspace_bytes, dicm_stream_t stream);
int dicm_imgmlp_bwd(const void* pool, int pool_dtype, int d_raw, const int32_t* rows,
                    const int32_t* count_dev, int64_t rows_max, const dicm_imgmlp_params_t* p,
                    const float* act0, const float* act1, const float* demb,
                    const dicm_imgmlp_grads_t* g, int precision, void* workspace,
                    size_t workspace_bytes, dicm_stream_t stream);

/* ------------------------------------------------------------------------
 * a6-a10: per-sample gather / pooling, forward and backward, fused.
 * Forward (reference model.py:358-396): writes every part of the head input
 *   x = hstack(field vectors, ad-image embedding, pooled behaviors):
 *   one-hot field rows (rows(table, ids), autograd.py:262-272), multi-hot
 *   sums (segment_sum, autograd.py:275-287), the ad-image embedding
 *   (rows(E, inverse), model.py:373-376) and the aggregator: sum pooling
 *   (model.py:219-220) or attentive pooling with the ad-image query
 *   (model.py:206-215, 225-226) and the complementary ID query
 *   (multi-query, model.py:227-229, 381-383).
 * Backward: the same graph reversed (segment_softmax bwd autograd.py:334-337,
 *   col_scale bwd 348-350); embedding and ID-row gradients are summed into
 *   the deduplicated row buffers (np.add.at, autograd.py:267-271) WITHOUT
 *   float atomics: every unique key sums its references (grouped by
 *   dicm_ref_transpose) in ascending reference order (groups of up to 16) or
 *   exactly in 64-bit fixed point (larger groups: independent of the order),
 *   so a step is bit-reproducible like the reference's (runtime.py:16-21);
 *   attention-parameter gradients are written as per-block partial sums.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t kind;                 /* 0 sum, 1 attn, 2 multiquery-attn, 3 max (segment_max, autograd.py:289-319),
                                   4 concat (scatter_concat, autograd.py:370-385: width - pool_col = 12 b_max) */
  int32_t normalize;            /* softmax over scores (model.py:211-214) */
  int32_t use_ad_image;
  int32_t use_behavior_images;
  int32_t n_fields;
  int32_t field_multi[8];
  int32_t field_col[8];         /* column of each field vector in the head input */
  int32_t ad_col;               /* column of the ad-image embedding (or -1) */
  int32_t pool_col;             /* column of the aggregator output (or -1) */
  int32_t width;                /* head input width */
  int32_t n_query;              /* multiquery: number of ID query fields (1 or 2) */
  int32_t query_col[2];         /* their columns in the head input */
  int32_t query_field[2];       /* their field indices */
} dicm_layout_t;

typedef struct {
  int32_t batch;
  int64_t refs;                 /* R = behavior rows */
  const int32_t* field_ids[8];  /* one-hot: [B]; multi-hot: flat [R_f] */
  const int32_t* field_off[8];  /* multi-hot CSR offsets [B+1]; NULL for one-hot */
  const float* tables[8];       /* id_emb/<field> [V_f, 12] */
  const int32_t* field_inv[8];  /* per reference: row in the deduplicated ID-row list */
  const int32_t* ad_local;      /* [B] inverse of the ad images into emb */
  const int32_t* beh_local;     /* [R] inverse of the behavior images into emb */
  const int32_t* beh_off;       /* [B+1] */
  const float* emb;             /* [U,12] image embeddings */
  /* backward only: the ordered per-key sums (see above) */
  const int32_t* img_order;     /* image references [ad (B, if used) | behaviors (R, if used)] grouped by
                                   unique image, ascending within a group (dicm_ref_transpose of the inverse) */
  const int32_t* img_start;     /* [U+1] group starts in img_order */
  const int32_t* id_order;      /* ID references (fields in schema order) grouped by unique key */
  const int32_t* id_start;      /* [K+1] */
  int64_t field_ref_begin[8];   /* first position of each field's references in the ID reference list */
  const int32_t* beh_seg;       /* [R] sample of each behavior reference (dicm_csr_segments) */
  const int32_t* field_seg[8];  /* multi-hot fields: [R_f] sample of each reference */
  const int32_t* n_img_keys;    /* device: U */
  const int32_t* n_id_keys;     /* device: K */
  int64_t img_cap, id_cap;      /* capacities of d_emb / d_rows (>= U, K) */
  float* ref_grad;              /* attn / max / concat: [R, 12] scratch, gradient per behavior reference */
  float* q_grad;                /* attn: [B, 36] scratch, query gradients (ad image 12 | ID query fields 24) */
  int32_t* hot;                 /* [4 + 2 (img_cap + id_cap)] scratch: work lists of keys with many references */
  void* hot_acc;                /* dicm_hot_acc_bytes() scratch, zeroed once at allocation (the kernels leave
                                   it ready for the next step): per-key accumulators that spread a key with
                                   thousands of references (Zipf keys) over every SM; NULL = one block per key */
} dicm_batch_view_t;

/* Bytes of the batch view's hot_acc scratch (both key lists). */
size_t dicm_hot_acc_bytes(void);

/* Transpose of a dedup inverse (inv[p] = key of reference p, keys < key_cap):
 * order[] = 0..n-1 grouped by key (any order inside a group), start[k] = first
 * slot of key k, start[k] = n for every k past the last key.  A counting sort
 * (integer atomics, exclusive scan, cursor fill); stream-ordered; ws of
 * dicm_ref_transpose_workspace bytes.  With the order-independent exact group
 * sums of dicm_sample_bwd it replaces np.add.at (autograd.py:267-271)
 * deterministically. */
size_t dicm_ref_transpose_workspace(int64_t n, int64_t key_cap);
int dicm_ref_transpose(const int32_t* inv, int64_t n, int64_t key_cap, void* ws, size_t ws_bytes,
                       int32_t* order, int32_t* start /* [key_cap + 1] */, dicm_stream_t stream);
/* Rank-invariant counter-based table init for tables too large for the
 * reference's host init (model.py:316-319 draws 0.05 N(0,1) per row): row r,
 * column c = scale * normal(hash(key, r*d + c)); this rank's rows
 * r = local*world + rank, rows >= vocab zero. */
int dicm_table_init(float* out, int64_t n_local, int d, int world, int rank, int64_t vocab, uint64_t key,
                    float scale, dicm_stream_t stream);
/* seg[i] = b for off[b] <= i < off[b+1]: the sample of every CSR reference
 * (the reference's Batch.beh_seg / multihot segment arrays, model.py:144-150) */
int dicm_csr_segments(const int32_t* off, int batch, int32_t* seg, dicm_stream_t stream);

typedef struct {
  const float *w0, *b0, *a0, *w1, *b1; /* attn/<ch>/0/{w,b,a}, attn/<ch>/1/{w,b} */
} dicm_attn_params_t;

/* number of float partial slots one block writes (attention grads, both channels) */
int64_t dicm_attn_partial_size(const dicm_layout_t* layout);
int dicm_sample_blocks(int batch);
int dicm_sample_fwd(const dicm_layout_t* layout, const dicm_batch_view_t* bv,
                    const dicm_attn_params_t* attn /* [2]: img, id */, float* head_in,
                    float* scores /* [2, R] */, float* stats /* [2, B, 2] */,
                    dicm_stream_t stream);
/* dicm_sample_fwd in two parts that may run on different streams: the ID-field
 * columns of the head input (needs only the compact ID rows) and the image
 * columns (ad image, pooled behaviors; needs the embeddings and, for
 * multiquery-attn, the ID rows of the query fields). */
int dicm_fields_fwd(const dicm_layout_t* layout, const dicm_batch_view_t* bv, float* head_in,
                    dicm_stream_t stream);
int dicm_images_fwd(const dicm_layout_t* layout, const dicm_batch_view_t* bv,
                    const dicm_attn_params_t* attn, float* head_in, float* scores, float* stats,
                    dicm_stream_t stream);
/* Stream-ordered on `stream`.  Writes every row d_emb[0..U) and
 * d_rows[0..K) (no zeroing needed); the scratch buffers of the batch view are
 * overwritten.  d_rows = NULL leaves the ID rows to dicm_id_row_grads, which
 * reads only d_head_in and the ID half of the batch view's scratch, so it may
 * run on another stream concurrently with this call (once the head has
 * written d_head_in). */
int dicm_sample_bwd(const dicm_layout_t* layout, const dicm_batch_view_t* bv,
                    const dicm_attn_params_t* attn, const float* head_in, const float* d_head_in,
                    const float* scores, const float* stats, float* d_emb /* [U,12] */,
                    float* d_rows /* [K,12] */, float* attn_partials,
                    dicm_stream_t stream);

/* The ID-row half of dicm_sample_bwd: d_rows[0..K), each unique (field, row)
 * key the ordered sum of its references' gradients (np.add.at into the
 * table gradient, autograd.py:267-271, model.py:407-408). */
int dicm_id_row_grads(const dicm_layout_t* layout, const dicm_batch_view_t* bv, const float* d_head_in,
                      float* d_rows /* [K,12] */, dicm_stream_t stream);

/* ------------------------------------------------------------------------
 * a11-a12: head MLP width -> 128 -> 64 -> 1 and BCE (reference model.py:397-401,
 * autograd.py:230-246, training.py:39-42), forward and backward fused per
 * sample tile.  d_head_in = dLoss/dx; weight gradients of the mlp/ group are
 * written as per-block partials in sorted-name layout (mlp/0/a, mlp/0/b,
 * mlp/0/w, mlp/1/a, mlp/1/b, mlp/1/w, mlp/2/b, mlp/2/w).
 * ---------------------------------------------------------------------- */
typedef struct {
  const float *w0, *b0, *a0, *w1, *b1, *a1, *w2, *b2;
} dicm_head_params_t;

int64_t dicm_head_partial_size(int width);
int dicm_head_blocks(int batch);
int dicm_head_fwd_bwd(const float* head_in, int batch, int width, const float* labels,
                      float inv_denominator, const dicm_head_params_t* p, float* logits,
                      float* d_head_in, float* partials, float* loss_partials,
                      dicm_stream_t stream);

/* forward only (inference, reference KvPredictor.predict / predict_logits,
 * inference.py:72-81, training.py:109-118): logits[b] for b < batch */
int dicm_head_fwd(const float* head_in, int batch, int width, const dicm_head_params_t* p, float* logits,
                  dicm_stream_t stream);

/* ------------------------------------------------------------------------
 * Two-tower pre-rank scoring (reference PrerankModel, model.py:420-531;
 * replaces tower_reps + logits_graph, model.py:508-526): per sample, each
 * tower maps its input (12-wide blocks of the head input, in the reference's
 * hstack order) through PReLU(x W0^T + b0) W1^T + b1, the score is the
 * row-wise inner product of the two representations (autograd.py:388-398),
 * then BCE as in the head.  d_head_in = dLoss/dx for the head-input layout
 * (columns outside both towers are zero).  Tower weight gradients go to one
 * partial row per block at the offsets given (the fused dense buffer's sorted
 * order), reduced by dicm_reduce_partials.
 * ---------------------------------------------------------------------- */
#define DICM_TOWER_MAX_PARTS 10
#define DICM_TOWER_MAX_HIDDEN 128
#define DICM_TOWER_MAX_REP 64
typedef struct {
  const float *w0, *b0, *a0; /* [hidden][n_in], [hidden], [hidden] */
  const float *w1, *b1;      /* [rep][hidden], [rep] */
  int32_t n_parts;           /* input blocks, each 12 wide: n_in = 12 * n_parts */
  int32_t part_col[DICM_TOWER_MAX_PARTS]; /* head-input column of each block */
  int64_t g_w0, g_b0, g_a0, g_w1, g_b1;   /* gradient offsets inside one partial row */
} dicm_tower_t;

int dicm_towers_blocks(int batch);
/* towers[0] = user tower, towers[1] = ad tower; part_stride = partial row length */
int dicm_towers_fwd_bwd(const float* head_in, int batch, int width, const dicm_tower_t* towers, int hidden,
                        int rep, const float* labels, float inv_denominator, float* logits, float* d_head_in,
                        float* partials, int64_t part_stride, float* loss_partials, dicm_stream_t stream);
/* forward only (reference forward_prerank, model.py:529-535): logits[b] = score */
int dicm_towers_fwd(const float* head_in, int batch, int width, const dicm_tower_t* towers, int hidden, int rep,
                    float* logits, dicm_stream_t stream);

/* Wide head input (> 128 columns: the concat aggregator, reference
 * scatter_concat, autograd.py:370-385): layer 0 runs as fp32 GEMMs, the rest
 * of the head as in dicm_head_fwd_bwd.  Gradients of the whole mlp/ group are
 * written (not accumulated) straight into ``grads`` -- the fused buffer's
 * mlp/ range in sorted order (a0, b0, w0, a1, b1, w1, b2, w2), the same layout
 * as one head partial row -- and loss_partials feed dicm_loss_finalize. */
#define DICM_HEAD_MAX_WIDE 16384
size_t dicm_head_wide_workspace(int batch, int width);
int dicm_head_wide_fwd_bwd(const float* head_in, int batch, int width, const float* labels,
                           float inv_denominator, const dicm_head_params_t* p, float* logits,
                           float* d_head_in, float* grads, float* loss_partials, void* workspace,
                           size_t workspace_bytes, dicm_stream_t stream);
int dicm_head_wide_fwd(const float* head_in, int batch, int width, const dicm_head_params_t* p,
                       float* logits, void* workspace, size_t workspace_bytes, dicm_stream_t stream);

/* zero a device buffer on the stream (a memset node, no kernel) */
int dicm_zero_async(void* ptr, size_t bytes, dicm_stream_t stream);

/* partials [nblk, n] -> out[n] (deterministic, fixed order; += if accumulate) */
int dicm_reduce_partials(const float* partials, int nblk, int64_t n, float* out, int accumulate,
                         dicm_stream_t stream);
/* loss = sum(loss_partials) * scale; latches a non-finite loss into status */
int dicm_loss_finalize(const float* loss_partials, int nblk, float scale, float* loss_out,
                       int32_t* status, dicm_stream_t stream);
/* latches non-finite values of x[0..n) into status[DICM_ST_NONFINITE] |= bit */
int dicm_check_finite(const float* x, int64_t n, const int32_t* count_dev, int row_width,
                      int bit, int32_t* status, dicm_stream_t stream);

/* ------------------------------------------------------------------------
 * a14: optimizer (reference optim.py).
 * dense: bias-corrected Adam per parameter span (optim.py:44-63); an all-zero
 *   gradient leaves the span and its state untouched, each span keeps its own
 *   step count t[span]; nothing moves if status flags a non-finite value.
 * rows: per-row Adam on the deduplicated rows (optim.py:83-104); keys are
 *   global keys of dicm_dedup over tables laid out at `base`.
 * ---------------------------------------------------------------------- */
typedef struct {
  int64_t offset;
  int64_t size;
} dicm_span_t;

size_t dicm_adam_dense_workspace(int nspans);
int dicm_adam_dense(float* param, const float* grad, float* m, float* v, int32_t* t,
                    const dicm_span_t* spans, int nspans, float lr, float beta1, float beta2,
                    float eps, void* workspace, size_t workspace_bytes, int32_t* status,
                    dicm_stream_t stream);

typedef struct {
  float* table;
  float* m;
  float* v;
  int32_t* t;
  int64_t base;
  int64_t vocab;
} dicm_table_state_t;

int dicm_adam_rows(const dicm_table_state_t* tabs, int ntab, const int32_t* uniq_keys,
                   const int32_t* count_dev, int64_t max_rows, const float* grads, float lr,
                   float beta1, float beta2, float eps, int32_t* status, dicm_stream_t stream);

/* ------------------------------------------------------------------------
 * a16: AMS exchange helpers for the multi-GPU step (reference
 * Cluster.run_iteration runtime.py:370-470, shard_of runtime.py:60-68).
 * Keys are owned by rank = key % world; the owner's local row is key / world.
 * bucket: stable partition of sorted keys[0..*count_dev) by owner ->
 *   send_keys (owner-local ids), send_counts[world], perm[i] = slot of key i,
 *   perm_inv[slot] = i (optional, NULL to skip: the gather form of perm, used
 *   to push per-key rows to the owners with dicm_p2p_gather_scatter12).
 * permute rows: out[perm[i]] = in[i] (scatter) or out[i] = in[perm[i]] (gather)
 *   for 12-float rows.
 * ---------------------------------------------------------------------- */
int dicm_bucket_by_owner(const int32_t* keys, const int32_t* count_dev, int64_t n_max, int world,
                         int32_t* send_keys, int32_t* send_counts, int32_t* perm, int32_t* perm_inv,
                         void* workspace, size_t workspace_bytes, dicm_stream_t stream);
size_t dicm_bucket_workspace(int64_t n_max, int world);
int dicm_permute_rows12(const float* in, const int32_t* perm, const int32_t* count_dev,
                        int64_t n_max, int scatter, float* out, dicm_stream_t stream);
/* out[i] = row (key_i - base_f) of the table whose key range holds key_i
 * (the compact ID rows of a batch; the owner's answer to an ID-row pull,
 * reference ServerNode.handle_id_pull runtime.py:155-163) */
int dicm_gather_rows_by_key(const dicm_table_state_t* tabs, int ntab, const int32_t* keys,
                            const int32_t* count_dev, int64_t n_max, float* out, dicm_stream_t stream);
/* owner-side reduction of pushed gradient rows: out[u] = sum over sources in
 * ascending order of the row each source pushed for unique key u (reference
 * ServerNode.local_model_gradient runtime.py:177-185, apply_id_updates
 * 208-219).  recv rows are grouped by source (segment offsets seg_dev[nsrc+1]
 * on the device), inv maps each received row to its unique key; idx_ws holds
 * nsrc * ucap int32.  Deterministic: no floating-point atomics. */
int dicm_owner_reduce_rows12(const float* recv, const int32_t* inv, const int64_t* seg_dev, int nsrc,
                             int64_t n_recv_max, const int32_t* count_dev, int64_t ucap, int32_t* idx_ws,
                             float* out, dicm_stream_t stream);

/* ------------------------------------------------------------------------
 * a16 over NVLink peer memory: the all-to-all-v exchanges of the AMS step
 * (reference Cluster._route of EmbedRequest / EmbedResponse / IdParamPull /
 * IdParamResponse / EmbedGradPush / IdParamPush, runtime.py:337-343,
 * 387-422) written directly into the peers' receive
 * buffers by copy kernels, with every count staying on the device (no host
 * round trip per iteration).
 * Each rank allocates one exchange region with dicm_p2p_alloc (same size and
 * layout on every rank), shares it with dicm_ipc_handle / dicm_ipc_open, and
 * fills dicm_peers_t.region[r] with rank r's region as mapped locally.
 * barrier: every rank stores `epoch` (increasing) into slot [rank] of the
 *   uint32 flag array at `flags_off` of every region (release, system scope)
 *   and waits until its own slots all reach `epoch`; a peer that never
 *   arrives latches status[DICM_ST_P2P_TIMEOUT] after ~10 s instead of hanging.
 *   epoch 0 = the next value of a counter kept in slot 63 of the local flag
 *   array (advanced on the device, so captured CUDA graphs replay correctly).
 * counts: writes this rank's per-destination counts send_counts[world][2]
 *   (column 0 images, 1 ID rows) into row [rank] of the [world][world][2]
 *   int32 count matrix at cmat_off of every region.
 * plan: from the local count matrix: the receive segments seg_img / seg_id
 *   [world+1] (int64, by source), cnt_dev = {n_recv_img, n_recv_id,
 *   n_send_img, n_send_id} and the placement table plan[2][4][world+1].
 * scatter: dir 0 (requester -> owners): rows [send_off[d], +cnt[d]) of src go
 *   to region[d] + dst_off at the position this rank's segment has there;
 *   dir 1 (owner -> requesters): the rows of source s's segment (in receive
 *   order) go back to region[s] + dst_off where s expects them.  row_bytes is
 *   4 (keys) or 48 (12-float rows).
 * ---------------------------------------------------------------------- */
#define DICM_MAX_PEERS 8
#define DICM_ST_P2P_TIMEOUT 4 /* != 0: a peer missed a barrier */
typedef struct {
  int32_t world, rank;
  void* region[DICM_MAX_PEERS];
} dicm_peers_t;

int dicm_p2p_alloc(size_t bytes, void** out);
int dicm_p2p_free(void* ptr);
int dicm_ipc_handle(const void* ptr, void* handle /* 64 bytes */);
int dicm_ipc_open(const void* handle, void** out);
int dicm_ipc_close(void* ptr);
int dicm_p2p_barrier(const dicm_peers_t* peers, int64_t flags_off, uint32_t epoch, int32_t* status,
                     dicm_stream_t stream);
int dicm_p2p_counts(const dicm_peers_t* peers, const int32_t* send_counts /* [2][world]: image, ID */,
                    int64_t cmat_off, dicm_stream_t stream);
int dicm_p2p_plan(const dicm_peers_t* peers, int64_t cmat_off, int64_t* seg_img, int64_t* seg_id,
                  int32_t* cnt_dev, int64_t* plan, dicm_stream_t stream);
int dicm_p2p_scatter(const dicm_peers_t* peers, const int64_t* plan, int kind /* 0 img, 1 id */,
                     int dir, const void* src, int row_bytes, int64_t dst_off, dicm_stream_t stream);
/* dicm_permute_rows12(rows, idx) fused into dicm_p2p_scatter for 12-float
 * rows: row j of each peer's segment is rows[idx[s0 + j]], gathered locally
 * and stored into the peer's buffer over NVLink in one pass (the owner's
 * embeddings back to the requesters, reference runtime.py:387-422). */
int dicm_p2p_gather_scatter12(const dicm_peers_t* peers, const int64_t* plan, int kind, int dir, const float* rows,
                              const int32_t* idx, int64_t dst_off, dicm_stream_t stream);
/* Sum of src[0..n) over every rank, into dst on every rank, over peer
 * memory: stage into this rank's region (stage_off, float4-padded), barrier,
 * each rank reduces 1/world of the elements in rank order and writes the sums
 * into every rank's region (res_off), barrier, copy out.  The same order on
 * every rank: bit-identical replicas (the dense all-reduce of runtime.py's
 * WorkerSync/ServerSync phases 4-5, runtime.py:424-463). */
int dicm_p2p_allreduce(const dicm_peers_t* peers, const float* src, int64_t n, int64_t stage_off,
                       int64_t res_off, int64_t flags_off, int32_t* status, float* dst, dicm_stream_t stream);
/* dedup of keys[0..*n_dev) (n_dev on the device, n_max its bound) over
 * [0, vocab): the owner-side dedup across sources (runtime.py:143-150) */
int dicm_dedup_devn(const int32_t* keys, const int32_t* n_dev, int64_t n_max, int64_t vocab, void* workspace,
                    size_t workspace_bytes, int32_t* uniq_out, int32_t* inv_out, int32_t* count_dev,
                    int32_t tag, int32_t* status, dicm_stream_t stream);

/* ------------------------------------------------------------------------
 * Host input pipeline (reference data.py:293-311 read_samples + encode_batch
 * model.py:158-198): JSONL sample records parsed natively on `nthreads`
 * threads (0 = all cores) into columns.  Keys are the JSON field names; a
 * list key keeps the most recent b_max entries of each record.  parse
 * returns a handle (NULL on a malformed record: *bad_line = its 1-based line
 * and dicm_last_error() says why); export copies column `key` out: int32
 * values (+ CSR offsets [n+1] for list keys), or float32 labels for "label".
 * Host-only: needs no GPU.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t n_keys;
  const char* keys[16];
  int32_t key_is_list[16];
  int32_t b_max;
} dicm_jsonl_spec_t;
void* dicm_jsonl_parse(const char* buf, int64_t len, const dicm_jsonl_spec_t* spec, int nthreads,
                       int64_t* n_records, int64_t* bad_line);
int64_t dicm_jsonl_list_total(void* handle, int key);
int dicm_jsonl_export(void* handle, int key, int32_t* values, int32_t* offsets, float* labels);
void dicm_jsonl_free(void* handle);
/* Host-side packing of a batch's columns into the pinned upload buffer on
 * several threads (replaces the per-column copies behind the reference's
 * encode_batch arrays, model.py:158-198): segment i = bytes[i] bytes from
 * srcs[i] to (char*)dst + dst_off[i]. */
int dicm_host_pack(void* dst, const void* const* srcs, const int64_t* bytes, const int64_t* dst_off, int n,
                   int nthreads);

/* ------------------------------------------------------------------------
 * Timing probe (instrumentation, no reference counterpart): while enabled,
 * the library records a CUDA event pair on the launching stream around each
 * of its dominant kernels; dicm_probe_read returns the elapsed ms of the
 * recorded launches of one kernel (waits on their end events).  Enabling
 * clears earlier records.
 * ---------------------------------------------------------------------- */
enum {
  DICM_PROBE_IMG_FWD_L0 = 0,  /* layer-0 forward GEMM (gather + tcgen05) */
  DICM_PROBE_IMG_FWD_L12 = 1, /* layers 1-2 forward */
  DICM_PROBE_IMG_BWD_L12 = 2, /* layers 2-1 backward (dE -> da0) */
  DICM_PROBE_IMG_BWD_DW1 = 3, /* dW1 */
  DICM_PROBE_IMG_BWD_DW0 = 4, /* dW0 = da0^T X (gather + tcgen05) */
  DICM_PROBE_SAMPLE_FWD = 5,  /* per-sample gather / pooling forward */
  DICM_PROBE_SAMPLE_BWD = 6   /* per-sample pooling backward */
};
int dicm_probe_enable(int on);
int dicm_probe_read(int kernel, float* ms, int max, int* n);

#ifdef __cplusplus
}
#endif
#endif /* DICM_B200_H */
