/*
 * csvd_b200 -- C ABI of the B200-native CSV-Decode output-layer hot path.
 *
 * The reference (`csvd`, /root/reference/pkg/src/csvd) is a pure-Python
 * package with no FFI; its hot-path entry points are Python functions.  This
 * header is the drop-in boundary underneath a Python mirror of that API
 * (paper_2511_21702_b200/engine.py binds it with ctypes; INTEGRATION.md shows
 * the binding a `csvd` maintainer would add).  Each entry point names the
 * reference interface it replaces.
 *
 * Conventions: plain pointers and sizes, no torch types.  Host pointers are
 * host memory unless the name says `_dev`.  `stream` is a cudaStream_t passed
 * as void* (NULL = the context's own stream).  All calls return 0 on success
 * or a negative CSVD_E* code; csvd_strerror() describes the last error of the
 * context.  One context per (table, index, device); a context is not thread
 * safe (the reference's step is single-threaded too: SPEC.md:345).
 */
#ifndef CSVD_B200_H
#define CSVD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes -> Python: CONFIG -> ConfigError, DIM/VALUE -> ValueError,
 * CUDA/STATE -> RuntimeError  (decode.py:63-64,104-115; bounds.py:53-55,67-76) */
#define CSVD_OK 0
#define CSVD_ECONFIG (-1)      /* bad DecodeConfig / unsupported option        */
#define CSVD_EDIM (-2)         /* dimension mismatch                           */
#define CSVD_EVALUE (-3)       /* non-finite bounds / bad epsilon              */
#define CSVD_ECUDA (-4)        /* CUDA runtime failure                         */
#define CSVD_ESTATE (-5)       /* device state machine inconsistency           */
#define CSVD_ENOMEM (-6)

/* weight storage */
#define CSVD_W_F32 0
#define CSVD_W_BF16 1          /* uint16 bf16 bit patterns                      */

/* index modes: cluster_index.py:47 MODES */
#define CSVD_MODE_EUCLIDEAN 0
#define CSVD_MODE_SPHERICAL 1
#define CSVD_MODE_BIAS_AUGMENTED 2

/* certificate kinds: certify.py:50 */
#define CSVD_KIND_NONE (-1)
#define CSVD_KIND_TOPK_EXACT 0
#define CSVD_KIND_SOFTMAX_EPS 1
#define CSVD_KIND_TOPP_MASS 2

/* targets (decode.py:59 TARGET_KINDS) */
#define CSVD_TARGET_TOPK 0
#define CSVD_TARGET_SOFTMAX 1
#define CSVD_TARGET_TOPP 2

/* fallback levels (decode.py:67-81) and fallback_used codes */
#define CSVD_FB_NONE (-1)
#define CSVD_FB_PARTIAL_EXPAND 0
#define CSVD_FB_RELAX_EPS 1
#define CSVD_FB_FULL_VOCAB 2

/* step variants */
#define CSVD_VARIANT_INCREMENTAL 0   /* decode.decode_step              decode.py:312-343 */
#define CSVD_VARIANT_BATCHSELECT 1   /* decode.decode_step_batchselect  decode.py:362-382 */

#define CSVD_MAX_LEVELS 8

/* EmbeddingTable (tensor_io.py:69-94), ORIGINAL token order, host memory. */
typedef struct {
    int64_t vocab_size;       /* V */
    int64_t hidden_dim;       /* d */
    int32_t w_dtype;          /* CSVD_W_F32 | CSVD_W_BF16 */
    const void *weights;      /* [V, d] row-major */
    const double *bias;       /* [V]  float64 (any finite values; added to the f64 dot exactly as
                                 tensor_io.EmbeddingTable holds them) */
} csvd_table_desc;

/* ClusterIndex stacked arrays (cluster_index.py:96-124), host memory. */
typedef struct {
    int32_t n_clusters;       /* C */
    int32_t mode;             /* CSVD_MODE_* */
    const int64_t *perm;      /* [V] permuted position -> original token id */
    const int64_t *starts;    /* [C] */
    const int64_t *sizes;     /* [C] */
    const double *centroids;  /* [C, bd], bd = d (+1 for bias_augmented) */
    const double *radii;      /* [C] */
    const double *max_biases; /* [C] */
    const double *log_sizes;  /* [C] numpy np.log(sizes) (certify.py:119) */
    /* spherical only (may be NULL otherwise) */
    const double *centroid_norms, *angulars, *max_norms, *min_norms;
} csvd_index_desc;

/* DecodeConfig (decode.py:84-115) flattened. */
typedef struct {
    int32_t k;
    int32_t n_targets;
    int32_t targets[3];               /* CSVD_TARGET_*, in cfg.targets order */
    int32_t n_levels;                 /* cfg.fallback (FullVocab appended by the engine) */
    int32_t level_kind[CSVD_MAX_LEVELS];
    double level_param[CSVD_MAX_LEVELS]; /* delta_c (PartialExpand) or factor (RelaxEps) */
    double epsilon;
    int64_t k_max;                    /* resolved budget (cfg.resolved_k_max or override) */
    int32_t variant;                  /* CSVD_VARIANT_* */
    int32_t slack_f32;                /* cfg.slack_mode == "f32" (bounds.py:58-64) */
    int64_t first_wave_tokens;        /* speculative wave policy; 0 = default */
    int32_t shard_lo, shard_hi;       /* csvd_shard_open: opening positions [lo, hi); hi 0 = the
                                         batch-select prefix (decode.py:346-359) */
} csvd_config;

/* Per-shard aggregate of one csvd_shard_open call (sharded_decode_step,
 * shard_sim.py:134-208): everything a rank contributes to the merge, plus the
 * global-order facts every rank computes identically.  Layout of the double
 * buffer returned by csvd_shard_open / csvd_shard_dense: */
#define CSVD_SH_LSE 0        /* log-sum-exp of this shard's logits in the range      */
#define CSVD_SH_MIN 1        /* min / max of them (+inf / -inf when none)             */
#define CSVD_SH_MAX 2
#define CSVD_SH_NTOK 3       /* tokens of this shard in the range                     */
#define CSVD_SH_NLIST 4      /* entries in the top-k list (min(k, NTOK))              */
#define CSVD_SH_P_LO 5       /* resolved range [p_lo, p_hi) in opening positions      */
#define CSVD_SH_P_HI 6
#define CSVD_SH_P_SEL 7      /* batch-select prefix                                   */
#define CSVD_SH_CUM_LO 8     /* tokens before p_lo / p_hi in the global opening order */
#define CSVD_SH_CUM_HI 9
#define CSVD_SH_U_NEXT 10    /* bound at position p_hi (max unopened), -inf if p_hi == C */
#define CSVD_SH_LRH_NEXT 11  /* log R-hat after opening [0, p_hi)                     */
#define CSVD_SH_QNORM 12
#define CSVD_SH_SLACK 13
#define CSVD_SH_TOPK 16      /* then the shard's top-k logits (descending)            */

/* result flags: a tested prefix had |rho - eps| < 1e-12 eps (softmax target)
 * or |delta - eps/(1-eps)| < 1e-12 of it (top-p target): that decision is a
 * tie at the ulp level (the device's exp/log and numpy's may disagree). */
#define CSVD_FLAG_TIE_AMBIGUOUS 1

/* CertStatus + StepMetrics scalars (certify.py:48-53, decode.py:118-130). */
typedef struct {
    int32_t kind;             /* CSVD_KIND_* */
    int32_t fallback;         /* CSVD_FB_* */
    int64_t sub_size;         /* |S| */
    int32_t clusters_opened;
    int32_t heap_pops;
    double epsilon_achieved;
    double u_max;
    double topk_min;
    double rho;
    double xi;                /* NaN when undefined */
    double query_norm;
    double slack;
    int32_t error;            /* 0, or CSVD_EVALUE for non-finite bounds */
    int32_t waves;            /* device wave-loop iterations (diagnostic) */
    int32_t flags;            /* CSVD_FLAG_* */
    int32_t reserved;
} csvd_result;

typedef struct csvd_ctx csvd_ctx;

/* Upload a (table, index) pair: permutes W into cluster order on the device,
 * f64 centroids, f64 bias.  Replaces the per-step `_check_table_index`
 * (decode.py:142-144): the caller verifies the fingerprint once here. */
int csvd_create(csvd_ctx **out, int device, const csvd_table_desc *table,
                const csvd_index_desc *index);
int csvd_destroy(csvd_ctx *ctx);
const char *csvd_strerror(csvd_ctx *ctx);

/* Shard context for vocabulary-sharded decoding (shard_sim.py:84-208 made
 * real): every cluster's centroid / bound data is replicated (bounds and the
 * opening order are computed identically on every rank), but only the W rows
 * of clusters with owned[c] != 0 are uploaded and ever read. */
int csvd_create_shard(csvd_ctx **out, int device, const csvd_table_desc *table,
                      const csvd_index_desc *index, const uint8_t *owned);

/* Open the owned clusters among opening positions [cfg->shard_lo, hi) (hi =
 * cfg->shard_hi, or the batch-select prefix when 0) from HOST h: bounds and the
 * global order on the device, this shard's rows, its aggregate (CSVD_SH_*,
 * `summary` holds CSVD_SH_TOPK + k doubles), and its tokens in the range in
 * opening order: global opening position, token id, logit (n_out entries). */
int csvd_shard_open(csvd_ctx *ctx, const double *h, const csvd_config *cfg, double *summary,
                    int64_t *positions, int64_t *ids, double *logits, int64_t cap, int64_t *n_out);

/* Full-vocabulary fallback on this shard (decode.py:239-262): logits of the
 * owned tokens (ids ascending) and the shard's top-k list in `summary`. */
int csvd_shard_dense(csvd_ctx *ctx, const double *h, int32_t k, double *summary, int64_t *ids,
                     double *logits, int64_t cap, int64_t *n_out);

/* Batched decode: B independent decode_step calls (decode.py:312-343) in one
 * graph replay.  Each query runs the step kernel on its own slice of the GPU
 * (a cooperative grid of ~148/B CTAs; all B run concurrently, sharing the
 * centroid and W reads through L2).  H: [B, d] host doubles; res[B];
 * ids / logits: B rows of `cap` entries (query b's |S| entries at row b). */
int csvd_step_batch_host(csvd_ctx *ctx, int32_t B, const double *H, const csvd_config *cfg,
                         csvd_result *res, int64_t *ids, double *logits, int64_t cap);
/* Device-resident variant (H_dev: [B, d] device doubles), asynchronous. */
int csvd_step_batch_device(csvd_ctx *ctx, int32_t B, const double *H_dev, const csvd_config *cfg,
                           void *stream);
/* Lanes currently built and the CTAs each lane's step runs on. */
int csvd_batch_lanes(csvd_ctx *ctx, int32_t *lanes, int32_t *grid_per_lane);

/* Workspace capacity for k (top-k list length); grows on demand. */
int csvd_reserve_k(csvd_ctx *ctx, int32_t k);

/* One certified step, end to end from HOST buffers (replaces
 * csvd.decode_step / decode_step_batchselect, decode.py:312-382):
 * H2D of h, graph replay, D2H of the result.  ids/logits receive |S| entries
 * (capacity `cap` >= V is always sufficient), in the reference's order:
 * opening order, or 0..V-1 for the full-vocabulary fallback. */
int csvd_step_host(csvd_ctx *ctx, const double *h, const csvd_config *cfg,
                   csvd_result *res, int64_t *ids, double *logits, int64_t cap);

/* Device-resident variant: h_dev is a device pointer to d doubles (the
 * bias-augmented [h, 1] is formed on the device), nothing is copied back; read
 * results with csvd_outputs().  Asynchronous on `stream`.  For head-eligible
 * configs the step kernel reads h_dev in place (16-byte aligned pointers; the
 * graph's kernel node is re-pointed on the host when h_dev changes), so the
 * buffer must hold h until the step has run in stream order, as for any
 * kernel input; otherwise h is first copied into the context's own buffer. */
int csvd_step_device(csvd_ctx *ctx, const double *h_dev, const csvd_config *cfg,
                     void *stream);
int csvd_outputs(csvd_ctx *ctx, int64_t **ids_dev, double **logits_dev,
                 csvd_result **res_dev);

/* csvd.cluster_bounds (bounds.py:178-184): U[C], query norm, slack. */
int csvd_bounds_host(csvd_ctx *ctx, const double *h, int32_t slack_f32, double *values,
                     double *query_norm, double *slack);

/* Full-vocabulary logits (oracle.dense_logits, oracle.py:33-41; decode.py:239-262):
 * logits[V] in original token order. */
int csvd_dense_host(csvd_ctx *ctx, const double *h, double *logits);

/* Device-resident dense GEMV timing hook: same kernel as the full_vocab
 * fallback, logits stay on the device. */
int csvd_dense_device(csvd_ctx *ctx, const double *h_dev, void *stream);

/* Introspection for tests / bench. */
int csvd_info(csvd_ctx *ctx, int64_t *V, int64_t *d, int32_t *C, int32_t *bd,
              int32_t *w_plan_regular, int32_t *b_plan_regular, int32_t *grid_ctas);

/* The context's own CUDA stream (cudaStream_t as void*): callers that time
 * or order work around csvd_*_device calls record events on it. */
int csvd_stream(csvd_ctx *ctx, void **stream);

/* Launch the step's kernels directly instead of replaying the CUDA graph
 * (identical results; for per-kernel profiling, since profilers cannot see
 * into conditional graph nodes).  The host then syncs once per wave. */
int csvd_set_direct(csvd_ctx *ctx, int32_t direct);

/* Benchmark utility: stream-read a 384 MiB buffer on `stream` so the next step
 * starts with an L2 holding none of its inputs (and no dirty lines). */
int csvd_l2_flush(csvd_ctx *ctx, void *stream);

/* Kernel launch counter (number of kernels launched by the last step call,
 * counting graph kernel nodes executed; diagnostic for bench gpu_launches). */
int csvd_last_launches(csvd_ctx *ctx, int32_t *n);

#ifdef __cplusplus
}
#endif
#endif
