/*
 * pfc_gpu.h — C ABI of the B200-native Partial-FC hot path (libpfc_gpu.so).
 *
 * Drop-in for the reference's distributed step
 *   StepResult pfc::distributed_partial_step(std::vector<CenterShard>& shards,
 *                                            const FeatureBatch& batch,
 *                                            const StepConfig& cfg,
 *                                            const SeededRng& iteration_rng)
 *   (/root/reference/proj/include/pfc/shardsim.hpp:166-168)
 * and of the pieces a caller touches around it:
 *   ShardLayout / buffer_capacity         (proj/include/pfc/sampler.hpp:16-33, 50-57)
 *   init_center_shards                    (proj/include/pfc/shardsim.hpp:56-82)
 *   CenterShard weights / momentum        (proj/include/pfc/types.hpp:29-47)
 *   StepConfig / MarginConfig             (shardsim.hpp:117-127, margin.hpp:17-37)
 *   StepResult.{loss, d_features, trace, buffers} (shardsim.hpp:129-135)
 *   error taxonomy                        (proj/include/pfc/error.hpp:9-42)
 *
 * Plain C types only (no torch / CUDA types): a context owns one GPU (one rank) and the
 * class-sharded centre matrix W and its momentum for the reference shards
 * [rank*K/world, (rank+1)*K/world).  Every entry point returns a pfc_status; on failure
 * pfc_gpu_last_error() holds the reference's message text for the matching pfc::*Error.
 * The C++ adapter include/pfc/gpu_step.hpp rethrows these as the reference exception types.
 */
#ifndef PFC_GPU_H_
#define PFC_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PFC_OK = 0,
  PFC_ERR_SHAPE = 1,      /* pfc::ShapeError */
  PFC_ERR_CONTRACT = 2,   /* pfc::ContractError */
  PFC_ERR_CAPACITY = 3,   /* pfc::CapacityError */
  PFC_ERR_CONFIG = 4,     /* pfc::ConfigError */
  PFC_ERR_NUMERICAL = 5,  /* pfc::NumericalError */
  PFC_ERR_CUDA = 6,       /* CUDA runtime / driver failure (no reference counterpart) */
  PFC_ERR_NCCL = 7,       /* NCCL failure (no reference counterpart) */
  PFC_ERR_IO = 8          /* pfc::DataError (checkpoint streams, io.hpp) */
} pfc_status;

typedef enum { /* MarginKind, margin.hpp:11 */
  PFC_MARGIN_PLAIN = 0,
  PFC_MARGIN_ADDITIVE_COSINE = 1, /* CosFace-style */
  PFC_MARGIN_ADDITIVE_ANGULAR = 2, /* ArcFace-style */
  PFC_MARGIN_COMBINED = 3          /* extension, not a reference MarginKind: the combined margin
                                      s (cos(m1 theta + m2) - m3) on the positive, s cos elsewhere
                                      (m2 = margin_m; m1 = margin_m1 in (0, 2], m3 = margin_m3 in
                                      [0, 1); theta = acos of the cosine clamped like ArcFace).
                                      (1, m, 0) is ArcFace and (1, 0, m) CosFace up to the clamp */
} pfc_margin_kind;

typedef enum {
  PFC_PRECISION_BF16 = 0, /* tcgen05 kind::f16 GEMMs, fp32 accumulate, fp32 master W / momentum;
                             needs dim % 4 == 0 and dim <= 1024 (pfc_gpu_create: PFC_ERR_CONFIG) */
  PFC_PRECISION_FP32 = 1, /* fp32 validation mode: SIMT fp32 GEMMs, fp64 softmax / gradient stage */
  PFC_PRECISION_TF32 = 2  /* tcgen05 kind::tf32 GEMMs on fp32 operands (10-bit mantissa inputs, fp32
                             accumulate, fp32 E), fp32 master W / momentum: the tensor-core mode for
                             a tighter value contract than bf16; same dim limits as bf16 */
} pfc_precision;

typedef struct {
  int64_t num_classes;     /* C  (ShardLayout::num_classes) */
  int64_t dim;             /* D  (embedding dimension) */
  int64_t num_shards;      /* K  (ShardLayout::num_shards; the reference's shard count) */
  int64_t max_batch;       /* largest global batch B the context will see (<= 2^20) */
  double r;                /* StepConfig::r */
  int32_t margin_kind;     /* pfc_margin_kind */
  double margin_scale;     /* MarginConfig::scale */
  double margin_m;         /* MarginConfig::margin */
  int32_t has_filter;      /* StepConfig::filter_threshold engaged */
  double filter_threshold;
  double momentum;         /* StepConfig::momentum */
  double weight_decay;     /* StepConfig::weight_decay */
  int32_t precision;       /* pfc_precision */
  int32_t device;          /* CUDA device ordinal of this rank */
  int32_t rank;            /* this process's rank, 0 <= rank < world_size */
  int32_t world_size;      /* GPUs (ranks); must divide num_shards */
  const uint8_t* nccl_id;  /* 128-byte ncclUniqueId from pfc_gpu_nccl_unique_id (world_size > 1),
                              or a loopback id from pfc_gpu_loopback_id */
  int32_t flags;           /* PFC_FLAG_* */
  double margin_m1;        /* PFC_MARGIN_COMBINED only (ignored otherwise): angular factor m1 */
  double margin_m3;        /* PFC_MARGIN_COMBINED only (ignored otherwise): cosine margin m3 */
} pfc_gpu_desc;

#define PFC_FLAG_FORCE_SEQUENTIAL_SAMPLER 1 /* test hook: always use the exact sequential FY */
#define PFC_FLAG_NO_GRAPH 2                  /* do not capture the step in a CUDA graph */
#define PFC_FLAG_EXACT_SOFTMAX 4             /* per-row max softmax offsets on every step (the
                                                default above margin_scale 64; below it a fixed
                                                offset, rerun per row if a row underflows) */
#define PFC_FLAG_DEBUG_LOGITS 8              /* test hook: keep the last step's logits
                                                (pfc_gpu_debug_logits) */
#define PFC_FLAG_NO_PDL 32                   /* launch the step's kernels without programmatic
                                                dependent launch (A/B timing) */
#define PFC_FLAG_FORCE_COLLECTIVES 128     /* test hook: world_size 1 still runs every collective
                                                of the N > 1 path, through a 1-rank group
                                                (nccl_id: a real ncclUniqueId, or a loopback
                                                id): real NCCL calls on a one-GPU box */
#define PFC_FLAG_WIDE_SAMPLER_CHUNKS 64      /* test hook: 1024-word label-bitmap chunks (the
                                                sampler's multi-word rank path, used by default
                                                only past 16.7M classes) */
#define PFC_FLAG_GUARD 16                    /* test hook: every device buffer of the context
                                                sits between two 4 KB guard regions filled with
                                                a pattern; pfc_gpu_check_guards reports any
                                                guard byte a kernel overwrote */

typedef struct {
  uint64_t seed;       /* iteration_rng.seed()      (rng.hpp:44) */
  uint64_t stream_id;  /* iteration_rng.stream_id() (rng.hpp:45) */
  double lr;           /* StepConfig::lr */
  int64_t step_index;  /* StepConfig::step_index (error context only) */
} pfc_gpu_step_args;

typedef struct {
  double loss;               /* StepResult::loss */
  uint64_t allgather_bytes;  /* StepResult::trace, reference closed form (shardsim.hpp:192-193) */
  uint64_t reduce_scalar_bytes;
  uint64_t reduce_grad_bytes;
  uint64_t reduce_ops;
  int64_t capacity;          /* per-shard buffer size (buffer_capacity) */
  int32_t rejection_shards;  /* shards that needed the exact sequential sampler this step */
  int32_t reserved;
  /* bytes this rank handed to NCCL collectives in the step (buffer sizes of the all-gathers,
   * all-reduces and reduce-scatters; 0 with one rank): what the GPU path actually moves, next to
   * the reference's closed-form trace above (costmodel.hpp:37-69) */
  uint64_t nccl_bytes;
  /* the same collectives under the ring model of the reference's cost model (costmodel.hpp:37-69,
   * "totals across workers, per step"): (R-1) S per all-gather / reduce-scatter and 2 (R-1) S per
   * all-reduce of S bytes in total, summed over the collectives the step issued (every rank
   * reports the same total; 0 with one rank) */
  uint64_t wire_bytes;
} pfc_gpu_step_out;

/* ---- lifecycle ------------------------------------------------------------------------ */
int pfc_gpu_create(const pfc_gpu_desc* desc, void** ctx_out);
int pfc_gpu_destroy(void* ctx);
/* Message of the last failure on ctx (or of the last failed create on this thread if NULL). */
const char* pfc_gpu_last_error(const void* ctx);
int pfc_gpu_nccl_unique_id(uint8_t out[128]);
/* Test hook: an id that makes world_size contexts created in ONE process (one host thread each,
 * any device, e.g. all on one GPU) ranks of a loopback communicator instead of NCCL.  The
 * collectives are host-synchronised (CUDA events, no kernel waits on another rank), summed in
 * ascending rank order, and never captured in a graph.  Every rank must call pfc_gpu_create
 * with the same id concurrently. */
int pfc_gpu_loopback_id(uint8_t out[128]);
const char* pfc_gpu_version(void);

/* ---- per-step configuration ------------------------------------------------------------ */
/* The StepConfig fields a context holds between steps (r, margin, filter, momentum, weight
 * decay; StepConfig, shardsim.hpp:117-127).  The reference takes a StepConfig per call: a caller
 * whose config changes between steps sets the new one here before the step (validated like
 * pfc_gpu_create: MarginConfig::validate's ConfigError texts, r in (0, 1]).  A new r changes the
 * buffer capacity (the column buffers grow when needed); the captured step graphs are rebuilt. */
typedef struct {
  double r;
  int32_t margin_kind;
  double margin_scale;
  double margin_m;
  int32_t has_filter;
  double filter_threshold;
  double momentum;
  double weight_decay;
  double margin_m1;  /* PFC_MARGIN_COMBINED only */
  double margin_m3;
} pfc_gpu_step_config;
int pfc_gpu_set_step_config(void* ctx, const pfc_gpu_step_config* cfg);

/* ---- shape queries (ShardLayout / buffer_capacity) ------------------------------------ */
int64_t pfc_gpu_capacity(const void* ctx);
int pfc_gpu_local_shards(const void* ctx, int64_t* first_shard, int64_t* num_local_shards);
int pfc_gpu_shard_range(const void* ctx, int64_t shard, int64_t* class_begin, int64_t* class_end);

/* ---- centre state (CenterShard weights / momentum, reference layout D x owned fp64) ----- */
int pfc_gpu_set_shard(void* ctx, int64_t shard, const double* weights_d_by_owned,
                      const double* momentum_d_by_owned /* NULL -> zeros */);
int pfc_gpu_get_shard(void* ctx, int64_t shard, double* weights_d_by_owned,
                      double* momentum_d_by_owned /* may be NULL */);
/* init_center_shards on the device: per-class stream ("center-init", class), Box-Muller in
 * fp64, unit-normalised, momentum = 0 (shardsim.hpp:56-82). */
int pfc_gpu_init_shards(void* ctx, uint64_t seed);
/* device pointers to the rank-local fp32 row-major [local classes x D] W and momentum */
int pfc_gpu_device_state(void* ctx, float** weights, float** momentum, int64_t* rows);

/* ---- the step --------------------------------------------------------------------------- */
/* Drop-in (host buffers): batch is the already-gathered global batch like FeatureBatch:
 * X is D x B row-major fp64, labels[B]; d_features_out receives the full D x B gradient
 * summed over all shards (StepResult::d_features).  Synchronous. */
int pfc_gpu_step(void* ctx, const double* features_d_by_b, const int64_t* labels, int64_t batch,
                 const pfc_gpu_step_args* args, double* d_features_d_by_b,
                 pfc_gpu_step_out* out);
/* Device path: this rank's slice of the global batch (rank-major order), device pointers:
 * x_local [b_local x D] fp32 row-major, labels_local [b_local] int64; dx_local [b_local x D]
 * fp32 receives this rank's rows of the summed gradient (NCCL reduce-scatter when
 * world_size > 1).  Enqueued on the context stream; with out != NULL it synchronises and
 * validates, with out == NULL it returns immediately (call pfc_gpu_sync to validate). */
int pfc_gpu_step_device(void* ctx, const float* x_local, const int64_t* labels_local,
                        int64_t b_local, const pfc_gpu_step_args* args, float* dx_local,
                        pfc_gpu_step_out* out);
int pfc_gpu_sync(void* ctx, pfc_gpu_step_out* out);
/* The last step's SampleBuffer of a local shard: cap class ids (positives ascending, then
 * negatives in Fisher-Yates order) and num_positives (sampler.hpp:38-46). */
int pfc_gpu_get_buffers(void* ctx, int64_t shard, int64_t* class_indices, int64_t* num_positives);
/* The context's CUDA stream (cudaStream_t) for callers that enqueue around the step. */
void* pfc_gpu_stream(void* ctx);

/* ---- diagnostics (StepConfig::with_diagnostics, shardsim.hpp:401-410) -------------------- */
typedef struct {
  double apcs;              /* metrics.hpp:56-79 */
  double amncs;             /* metrics.hpp:91-146 */
  double amncs_conflicted;  /* valid when has_conflicted */
  double amncs_hard;        /* valid when has_split */
  int32_t has_conflicted;   /* AmncsResult::conflicted.has_value() */
  int32_t has_split;        /* the conflict ground truth was given */
  int32_t reserved[2];
} pfc_gpu_diag_out;
/* apcs / amncs of a (global, already gathered) batch against the CURRENT shards, i.e. what the
 * reference step reports with with_diagnostics (computed there on the pre-update shards: call
 * this before pfc_gpu_step).  X is D x B fp64 row-major, labels[B] (host).  class_identity[C]
 * and sample_identity[B] (host, both or neither) give ConflictInfo (types.hpp:80-86).  Every
 * rank calls it; the maxima are merged over ranks.  amncs is exact (fp64 re-evaluation of the
 * bf16 GEMM's near-maximal classes).  Errors carry the reference's text. */
int pfc_gpu_diagnostics(void* ctx, const double* features_d_by_b, const int64_t* labels,
                        int64_t batch, const int64_t* class_identity,
                        const int64_t* sample_identity, pfc_gpu_diag_out* out);

/* mics (metrics.hpp:150-164): per class, the maximum cosine to any other class centre, for the
 * current shards; out[C] (class order).  Exact (fp64 re-evaluation of the bf16 screening GEMM's
 * near-maximal pairs).  O(C^2 D): a final-state diagnostic.  Single-rank contexts only. */
int pfc_gpu_mics(void* ctx, double* out);

/* ---- checkpoints (trainer.hpp:235-338 shard section; io.hpp:18-91 encoding) --------------- */
/* Write this rank's shard section in the reference's checkpoint encoding: int64 count, then per
 * local shard int64 shard_id, class_begin, class_end and weights, momentum as put_matrix
 * (int64 rows = D, int64 cols = owned, D x owned fp64 row-major).  append != 0 appends (after
 * a caller-written header, as save_checkpoint's sections follow one another). */
int pfc_gpu_write_shards(void* ctx, const char* path, int append);
/* Read a shard section starting at byte `offset` of `path` (written by the reference's
 * save_checkpoint or by pfc_gpu_write_shards) into the device state; shards of other ranks are
 * skipped; *end_offset (may be NULL) receives the offset after the section.  Matrices larger
 * than the reference reader's 2^32-element cap (io.hpp:78) are accepted. */
int pfc_gpu_read_shards(void* ctx, const char* path, int64_t offset, int64_t* end_offset);

/* ---- device-resident FeatureBatch ------------------------------------------------------- */
/* pfc_gpu_step with the FeatureBatch in DEVICE memory: features D x B fp64 row-major and
 * labels[B] int64; d_features_dev (D x B fp64, device; NULL = leave it in the context) receives
 * the full summed gradient.  Same kernels and results as pfc_gpu_step on the same values; the
 * label / capacity errors come from the device sampler's checks.  Synchronous. */
int pfc_gpu_step_features(void* ctx, const double* features_d_by_b_dev, const int64_t* labels_dev,
                          int64_t batch, const pfc_gpu_step_args* args, double* d_features_d_by_b_dev,
                          pfc_gpu_step_out* out);

/* ---- trainer integration (trainer.hpp:362-581) --------------------------
 * The caller of the step with its backbone on the device: the dataset points (SyntheticDataset,
 * datasynth.hpp:47-75) are uploaded once, the backbone (trainer.hpp:51-126: hidden =
 * tanh(w1 x + b1), output = w2 hidden + b2, fp64, products summed like matmul, matrix.hpp:86-105)
 * runs on the device, and the step's features and d_features never leave it: per step the host
 * sends the batch's point ids and reads the status.  Single-rank contexts; the context must
 * outlive the trainer.  The loop (split, shuffle, schedule, checkpoints, final metrics) is
 * pfc::gpu::train in include/pfc/gpu_trainer.hpp. */
/* points: input_dim x num_points fp64 row-major (host); observed_labels[num_points].  The
 * backbone is Backbone::init(input_dim, hidden_dim, embed_dim, seed) (trainer.hpp:65-77), bit
 * for bit; embed_dim must equal the context's dim. */
int pfc_gpu_trainer_create(void* ctx, const double* points, int64_t input_dim, int64_t num_points,
                           const int64_t* observed_labels, int64_t hidden_dim, int64_t embed_dim,
                           uint64_t seed, void** trainer_out);
int pfc_gpu_trainer_destroy(void* trainer);
/* backbone parameters in the reference layouts (host fp64): w1 hidden x input, b1 hidden,
 * w2 embed x hidden, b2 embed (checkpoints, trainer.hpp:264-267) */
int pfc_gpu_trainer_get_backbone(void* trainer, double* w1, double* b1, double* w2, double* b2);
int pfc_gpu_trainer_set_backbone(void* trainer, const double* w1, const double* b1,
                                 const double* w2, const double* b2);
/* Backbone::forward of the batch point_ids[batch] (host ids); the features stay on the device */
int pfc_gpu_trainer_forward(void* trainer, const int64_t* point_ids, int64_t batch);
/* apcs / amncs of the forward batch against the current shards (with_diagnostics; call between
 * forward and step, as the reference reports them for the pre-update shards) */
int pfc_gpu_trainer_diagnostics(void* trainer, const int64_t* class_identity,
                                const int64_t* sample_identity, pfc_gpu_diag_out* out);
/* distributed_partial_step on the forward batch; d_features stay on the device */
int pfc_gpu_trainer_step(void* trainer, const pfc_gpu_step_args* args, pfc_gpu_step_out* out);
/* Backbone::apply_gradient(inputs, act, d_features, lr) (trainer.hpp:99-125) with the cached
 * activations and the step's d_features; a non-finite gradient product raises the reference's
 * "matmul: non-finite entry" NumericalError before w1 / w2 change (the SGD rows run only after
 * the products' finiteness flags are read) */
int pfc_gpu_trainer_apply_gradient(void* trainer, double lr);
/* forward-only embeddings of point_ids[n] into emb (embed x n fp64, host), chunked by max_batch
 * (evaluation: nearest-centre accuracy, verification); discards the cached activations */
int pfc_gpu_trainer_embed(void* trainer, const int64_t* point_ids, int64_t n, double* emb);

/* Evaluation of the trained model on the device (trainer.hpp:519-577), fp64 in the reference's
 * operation order (separate multiply / add, d ascending), on the points' normalised embeddings
 * (l2_normalize_columns of Backbone::forward) and the context's current centres:
 *   nearest_center: best_class[n] = the first class with the largest cosine to the point's
 *                   embedding over all C unit centres (the training-accuracy scan, 532-545);
 *   pair_cosines:   cos_out[n (n-1) / 2] = the cosines of every pair i < j in (i, j)
 *                   lexicographic order (the verification score loop, 553-561).
 * Single-rank contexts (all classes local); embed_dim <= 512 for nearest_center. */
int pfc_gpu_trainer_nearest_center(void* trainer, const int64_t* point_ids, int64_t n,
                                   int64_t* best_class);
int pfc_gpu_trainer_pair_cosines(void* trainer, const int64_t* point_ids, int64_t n,
                                 double* cos_out);

/* ---- bench / test helpers --------------------------------------------------------------- */
/* PFC_FLAG_GUARD contexts: synchronises the device, compares every guard region with its
 * pattern; *corrupted = the number of changed regions (PFC_ERR_CUDA naming them if any). */
int pfc_gpu_check_guards(void* ctx, int64_t* corrupted);
/* Synthetic inputs of the bench convention on the device:
 * labels[b] = SeededRng(seed, make_stream("bench-labels", step)).next_below(C) and
 * X[b][d] = SeededRng(seed, make_stream("bench-x", step)).next_normal() (b-major, d inner). */
int pfc_gpu_bench_inputs(void* ctx, uint64_t seed, uint64_t step, int64_t batch, float* x_dev,
                         int64_t* labels_dev);
/* Kernel timing of the last step (ms, CUDA events around each phase); n <= 16 entries. */
int pfc_gpu_phase_times(void* ctx, float* ms, const char** names, int n);
int pfc_gpu_set_phase_timing(void* ctx, int enabled);
/* Test hook (PFC_FLAG_DEBUG_LOGITS): the last step's logits z of this rank, B x local columns
 * fp32 row-major (columns: local shards in order, cap each): s cos (margin on the positive),
 * -inf where the filter masked the column (shardsim.hpp:258-281). */
int pfc_gpu_debug_logits(void* ctx, float* out_b_by_cols);
/* Number of kernels (ours) launched by one step at the current batch shape. */
int64_t pfc_gpu_launches_per_step(void* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PFC_GPU_H_ */
