/*
 * cmlb.h -- C ABI of the B200 operator-representation inference path.
 *
 * The reference ("mlower", pure Python) runs a KernelPlan through a Python
 * interpreter loop (pkg/src/mlower/runtime.py:198-212) that dispatches numpy
 * kernels (pkg/src/mlower/kernels.py:47-287).  This library replaces that
 * executor's compute: each entry point below executes one fused operator
 * representation on the GPU.  Plain pointers and sizes only; no torch types.
 * Device pointers are CUDA device memory; `stream` is a cudaStream_t (NULL =
 * legacy default stream).  All entry points are thread-safe; programs are
 * immutable after creation and may be run concurrently on different streams.
 *
 * Status codes map 1:1 onto the reference error classes
 * (pkg/src/mlower/errors.py:10-93); see paper_2301_13441_b200/errors.py.
 */
#ifndef CMLB_H_
#define CMLB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CMLB_ABI_VERSION 3

enum cmlb_status {
  CMLB_OK = 0,
  CMLB_E_VALIDATION = 1,   /* ValidationError        errors.py:22-25 */
  CMLB_E_SHAPE = 2,        /* ShapeMismatch          errors.py:36-38 */
  CMLB_E_INDEX = 3,        /* IndexOutOfBounds       errors.py:56-58 */
  CMLB_E_OVERFLOW = 4,     /* AccumulatorOverflowRisk errors.py:60-62 */
  CMLB_E_UNRESOLVED = 5,   /* UnresolvedKernel       errors.py:72-74 */
  CMLB_E_INPUT = 6,        /* InputMismatch          errors.py:80-82 */
  CMLB_E_DEVICE = 7        /* CUDA failure (no reference analogue) */
};

/* Output element type: the reference output dtype after dispatch promotion
 * (dtypes.py:112-118); BOOL is one byte holding 0/1 (dtypes.py:51-59). */
enum cmlb_out_dtype {
  CMLB_OUT_BOOL = 0, CMLB_OUT_INT8 = 1, CMLB_OUT_INT16 = 2, CMLB_OUT_INT32 = 3, CMLB_OUT_F32 = 4
};

/* Thread-local message for the last non-zero status on this thread. */
const char* cmlb_last_error(void);
int cmlb_abi_version(void);
/* Number of kernel launches issued by this process so far (all entry points). */
int64_t cmlb_launch_count(void);

/* ------------------------------------------------------------------------ *
 * Forest: the tree operator representation plus the ensemble tail.
 *
 * Replaces, per tree, the chain  matmul|sparse_dense_matmul(W1) -> greater(W2)
 * -> [cast] -> matmul(W3) -> argmax -> gather_rows(leaf_table)
 * (convert.py:192-204, runtime.py:160-187) and the ensemble tail
 * stack -> [cast] -> reduce_mean|reduce_sum -> [mul lr -> add base]
 * -> argmax|sigmoid-threshold -> gather_rows(classes) (convert.py:287-311,
 * 211-222), in ONE kernel.  Trees are given in the reference's canonical
 * numbering: internal nodes in level order, leaves in in-order
 * (convert.py:110-135).  A child reference c >= 0 is an internal node of the
 * same tree, c < 0 is leaf (-1 - c).
 * ------------------------------------------------------------------------ */

enum cmlb_aggregation {
  CMLB_AGG_NONE = 0,   /* single tree: output = leaf payload (convert_tree) */
  CMLB_AGG_MEAN = 1,   /* random forests: float64 mean over trees (kernels.py:180-184) */
  CMLB_AGG_SUM = 2     /* gradient boosting: float64 sum, *lr, +base (kernels.py:185-190) */
};

enum cmlb_tail {
  CMLB_TAIL_VALUES = 0,   /* write the aggregated float32 values (N x C) */
  CMLB_TAIL_ARGMAX = 1,   /* first-max over C, then class label (convert.py:211-214) */
  CMLB_TAIL_SIGMOID = 2   /* float64 sigmoid -> float32 > 0.5 -> label (convert.py:217-222) */
};

/* Fused preprocessing ("prologue"): model input column f is computed from a
 * raw input column as the reference scaler / scikit-learn one-hot encoder
 * would (float32, pinned rounding: convert.py:255-284), so a pipeline
 * scaler -> one-hot -> model runs as ONE kernel reading the raw rows.  Used
 * by the forest, linear and SVM programs (optional) and by the standalone
 * column program below. */
enum cmlb_col_op {
  CMLB_COL_COPY = 0,      /* x                                                  */
  CMLB_COL_SUB_DIV = 1,   /* (x - a) / b       StandardScaler, RobustScaler     */
  CMLB_COL_DIV = 2,       /* x / a             MaxAbsScaler                     */
  CMLB_COL_MUL_ADD = 3,   /* x * a + b, two roundings   MinMaxScaler            */
  CMLB_COL_GREATER = 4,   /* x > a ? 1 : 0     Binarizer                        */
  CMLB_COL_EQUAL = 5      /* x == a ? 1 : 0    OneHotEncoder indicator column   */
};

typedef struct cmlb_column_op {
  int32_t src;            /* raw input column */
  int32_t op;             /* cmlb_col_op */
  float a;
  float b;
} cmlb_column_op;

enum cmlb_forest_variant {
  CMLB_FOREST_AUTO = 0,        /* pick by (depth, trees, features) from the measured table */
  CMLB_FOREST_PERFECT = 1,     /* perfect-padded trees staged in shared memory */
  CMLB_FOREST_GENERAL = 2,     /* arbitrary depth, canonical nodes read through L1 */
  CMLB_FOREST_RANKED = 3,      /* perfect trees, rank-quantized thresholds: one word per node */
  CMLB_FOREST_MMA = 4,         /* the GEMM form on tcgen05 kind::i8: bits x path matrix in TMEM */
  CMLB_FOREST_SKEW = 5         /* ranked walk, 32-tree groups skewed across the smem banks; only
                                * for forests whose float64 sums are certified order-free (ABI 3) */
};

typedef struct cmlb_forest_desc {
  int32_t n_trees;
  int32_t n_features;
  int32_t n_outputs;            /* C: payload width per leaf */
  const int64_t* node_offset;   /* [n_trees + 1] into feature/threshold/left/right */
  const int64_t* leaf_offset;   /* [n_trees + 1] into payload rows */
  const int32_t* feature;       /* internal nodes, level order */
  const float* threshold;
  const int32_t* left;
  const int32_t* right;
  const float* payload;         /* [total leaves][n_outputs], in-order leaf rows */
  int32_t aggregation;          /* cmlb_aggregation */
  int32_t tail;                 /* cmlb_tail */
  float learning_rate;
  float base_score;
  const double* classes;        /* class labels (tail ARGMAX / SIGMOID) */
  int32_t n_classes;
  int32_t out_dtype;            /* cmlb_out_dtype */
  int32_t dense_selector;       /* 1: replicate dense W1 (0*inf = NaN) semantics */
  int32_t variant;              /* cmlb_forest_variant */
  const cmlb_column_op* prologue; /* optional [n_features]: feature f = op(x[src]) (ABI 2) */
  int32_t n_inputs;             /* raw input columns when prologue != NULL */
  int32_t n_trees_total;        /* ABI 3: trees of the WHOLE ensemble when this program is one
                                 * tree shard (MEAN divides by it); 0 = n_trees */
} cmlb_forest_desc;

typedef struct cmlb_forest cmlb_forest;

/* Build device tables on `device` (host arrays are copied; caller keeps ownership). */
int cmlb_forest_create(const cmlb_forest_desc* desc, int device, cmlb_forest** out);
/* x: device float32 [n_rows][ldx] row-major; y: device output [n_rows][k] of out_dtype
 * (k = C for VALUES, 1 otherwise); leaf_out: optional device int32 [n_rows][n_trees]
 * in-order leaf index per tree (reference argmax slots). */
int cmlb_forest_run(const cmlb_forest* f, const float* x, int64_t n_rows, int64_t ldx,
                    void* y, int32_t* leaf_out, void* stream);
/* Tree-sharded partial: float64 raw sums over this program's trees in the
 * reference's pairwise order restricted to the shard (no tail), [n_rows][C]. */
int cmlb_forest_partial(const cmlb_forest* f, const float* x, int64_t n_rows, int64_t ldx,
                        double* partial, void* stream);
/* Tree-shard combine + tail: partials = device float64 [n_shards][n_rows][1],
 * each the raw sum of one contiguous tree range; merges = host int32 pairs
 * (a, b) applied in order as p[a] += p[b] (the shard nodes of numpy's pairwise
 * recursion, leaving the sum in p[0]); then the reference tail
 * (kernels.py:180-190, convert.py:297-311) with this program's tail
 * parameters and n_trees_total.  Scalar ensembles only (C == 1): numpy sums a
 * (N, T, C >= 2) stack tree after tree, which no shard cut reproduces, so
 * those are sharded by rows (CMLB_E_UNRESOLVED otherwise).  n_shards == 1,
 * n_merges == 0 finishes an already-reduced partial. */
int cmlb_forest_finish(const cmlb_forest* f, const double* partials, int32_t n_shards, const int32_t* merges,
                       int32_t n_merges, int64_t n_rows, void* y, void* stream);
/* One step of the cross-GPU pairwise tree reduce (reference kernels.py:185-190,
 * numpy pairwise_sum): dst[i] = dst[i] + src[i] in float64 for the n_rows
 * scalar partials, on this program's device.  The caller received src from the
 * peer that owns the right-hand shard node (NCCL point-to-point over NVLink). */
int cmlb_forest_merge(const cmlb_forest* f, double* dst, const double* src, int64_t n_rows, void* stream);
/* Introspection: chosen variant, padded depth, trees per shared-memory chunk. */
int cmlb_forest_info(const cmlb_forest* f, int32_t* variant, int32_t* depth, int32_t* chunk_trees,
                     int32_t* rows_per_cta);
void cmlb_forest_destroy(cmlb_forest* f);

/* ------------------------------------------------------------------------ *
 * Linear models: matmul(X, coef^T) -> add(intercept) -> tail
 * (convert.py:230-252).  Logits are float64 ascending-k dot products rounded
 * once to float32 (kernels.py:95-100), then float32 + b.
 * ------------------------------------------------------------------------ */

enum cmlb_linear_tail {
  CMLB_LIN_VALUES = 0,      /* regressors: (N, C) float32 */
  CMLB_LIN_ARGMAX = 1,      /* multi-class: first-max over C (softmax removed by RE) */
  CMLB_LIN_SOFTMAX_ARGMAX = 2, /* multi-class with softmax kept (passes without RE) */
  CMLB_LIN_SIGMOID = 3,     /* binary logistic: sigmoid -> f32 > 0.5 */
  CMLB_LIN_SIGN = 4         /* binary margin: z > 0 */
};

typedef struct cmlb_linear_desc {
  int32_t n_features;
  int32_t n_outputs;        /* C = rows of coef */
  const float* coef;        /* [C][n_features] */
  const float* intercept;   /* [C] */
  int32_t tail;             /* cmlb_linear_tail */
  const double* classes;
  int32_t n_classes;
  int32_t out_dtype;
  int32_t sparse_coef;      /* 1: CSR weight semantics (skip zero weights, kernels.py:115-123) */
  const cmlb_column_op* prologue; /* optional [n_features] (ABI 2) */
  int32_t n_inputs;
} cmlb_linear_desc;

typedef struct cmlb_linear cmlb_linear;
int cmlb_linear_create(const cmlb_linear_desc* desc, int device, cmlb_linear** out);
int cmlb_linear_run(const cmlb_linear* m, const float* x, int64_t n_rows, int64_t ldx,
                    void* y, void* stream);
void cmlb_linear_destroy(cmlb_linear* m);

/* ------------------------------------------------------------------------ *
 * Preprocessing operators (convert.py:255-284): float32 elementwise with the
 * reference's rounding sequence (no FMA contraction), Normalizer row norms in
 * float64 (kernels.py:245-261).
 * ------------------------------------------------------------------------ */

enum cmlb_scaler_kind {
  CMLB_SCALER_BINARIZER = 0, CMLB_SCALER_NORMALIZER_L1 = 1, CMLB_SCALER_NORMALIZER_L2 = 2,
  CMLB_SCALER_NORMALIZER_MAX = 3, CMLB_SCALER_MINMAX = 4, CMLB_SCALER_SUB_DIV = 5,
  CMLB_SCALER_DIV = 6
};

typedef struct cmlb_scaler_desc {
  int32_t kind;             /* cmlb_scaler_kind */
  int32_t n_features;
  float threshold;          /* binarizer */
  const float* a;           /* minmax: scale; sub_div: center/mean; div: scale */
  const float* b;           /* minmax: min;   sub_div: scale */
} cmlb_scaler_desc;

typedef struct cmlb_scaler cmlb_scaler;
int cmlb_scaler_create(const cmlb_scaler_desc* desc, int device, cmlb_scaler** out);
/* y: device float32 [n_rows][n_features] (may alias x when ldx == n_features). */
int cmlb_scaler_run(const cmlb_scaler* s, const float* x, int64_t n_rows, int64_t ldx,
                    float* y, void* stream);
void cmlb_scaler_destroy(cmlb_scaler* s);

/* ------------------------------------------------------------------------ *
 * Kernel SVMs (SVC / NuSVC / SVR / NuSVR).  Not in the reference:
 * the semantics are libsvm's dense svm_predict_values as shipped in
 * scikit-learn (see oracle/svm_oracle.c).  The Gram contraction X . SV^T runs
 * on tcgen05 tensor cores as split-TF32 (3 products per K step, ~fp32
 * accurate) with the kernel function and the one-vs-one decision sums fused
 * into the TMEM epilogue (float64 accumulators); rows whose decision is within
 * the epilogue's error bound of a vote flip are recomputed exactly in float64
 * in libsvm's operation order by a second kernel.
 * ------------------------------------------------------------------------ */

enum cmlb_svm_kernel { CMLB_SVM_LINEAR = 0, CMLB_SVM_POLY = 1, CMLB_SVM_RBF = 2, CMLB_SVM_SIGMOID = 3 };

typedef struct cmlb_svm_desc {
  int32_t n_features;
  int32_t n_sv;
  int32_t kernel;              /* cmlb_svm_kernel */
  int32_t degree;
  double gamma;
  double coef0;
  const float* support_vectors; /* [n_sv][n_features], grouped by class for svc */
  const float* dual_coef;      /* [n_classes - 1][n_sv] (svc) or [1][n_sv] (svr) */
  const float* intercept;      /* [n_classes (n_classes - 1) / 2] (svc) or [1] (svr) */
  const int32_t* n_support;    /* [n_classes] (svc); NULL for svr */
  int32_t n_classes;           /* >= 2 for svc, 0 for svr */
  const double* classes;       /* svc labels */
  int32_t out_dtype;           /* svc: label dtype; svr: CMLB_OUT_F32 */
  const cmlb_column_op* prologue; /* optional [n_features] */
  int32_t n_inputs;
} cmlb_svm_desc;

typedef struct cmlb_svm cmlb_svm;
int cmlb_svm_create(const cmlb_svm_desc* desc, int device, cmlb_svm** out);
/* y: [n_rows][1] labels (svc) or float32 values (svr).  decision: optional
 * device float64 [n_rows][max(1, pairs)] libsvm decision values (sum - rho).
 * exact_rows: optional device int32, receives how many rows took the float64
 * path.  Scratch is stream-ordered (cudaMallocAsync), so runs on different
 * streams do not share state. */
int cmlb_svm_run(const cmlb_svm* m, const float* x, int64_t n_rows, int64_t ldx, void* y, double* decision,
                 int32_t* exact_rows, void* stream);
void cmlb_svm_destroy(cmlb_svm* m);

/* ------------------------------------------------------------------------ *
 * Column transform: OneHotEncoder / ColumnTransformer / elementwise scalers
 * as one gather-transform kernel (y[:, f] = op_f(x[:, src_f])), plus the
 * OneHotEncoder(handle_unknown='error') membership check: `checks` lists raw
 * columns whose value must be one of its sorted category list.
 * ------------------------------------------------------------------------ */

typedef struct cmlb_columns_desc {
  int32_t n_inputs;
  int32_t n_outputs;
  const cmlb_column_op* ops;     /* [n_outputs] */
  int32_t n_checks;
  const int32_t* check_col;      /* [n_checks] raw column */
  const int64_t* check_offset;   /* [n_checks + 1] into check_values */
  const float* check_values;     /* ascending categories per checked column */
} cmlb_columns_desc;

typedef struct cmlb_columns cmlb_columns;
int cmlb_columns_create(const cmlb_columns_desc* desc, int device, cmlb_columns** out);
/* y: device float32 [n_rows][n_outputs] (NULL: check only).  bad_row:
 * optional device int64 the caller initialises to -1; it is lowered to the
 * first row holding an unknown category (min-combined, so several check
 * stages may share one slot) and the caller raises, as
 * OneHotEncoder.transform does. */
int cmlb_columns_run(const cmlb_columns* c, const float* x, int64_t n_rows, int64_t ldx, float* y,
                     int64_t* bad_row, void* stream);
void cmlb_columns_destroy(cmlb_columns* c);

/* ------------------------------------------------------------------------ *
 * Diagnostics (tests and measurement tools only; not on the predict path).
 * ------------------------------------------------------------------------ */

/* The numpy pairwise-sum replay codes the forest kernels use for C == 1
 * ensembles (tests/test_native_abi.py checks them against numpy). */
int cmlb_debug_pairwise_schedule(int64_t n, uint32_t* codes);
/* 1 when the forest's float64 sums over trees are certified exact in any
 * order (the SKEW variant's precondition), 0 when not, <0 on a bad
 * descriptor.  Host only. */
int cmlb_debug_sums_order_free(const cmlb_forest_desc* desc);
/* Rows the most recent certified linear run (class tails) sent to the float64
 * recompute, when the process runs with CMLB_LINEAR_QSTAT set (that run then
 * synchronizes its stream); -1 otherwise. */
int64_t cmlb_debug_linear_queued(void);
/* SVM fast path only, on every row, with the epilogue's per-row error bound
 * written to err (device float32 [n_rows]); CMLB_SVM_PROBE switches pipeline
 * roles off (tools/svm_pipe_probe.py). */
int cmlb_svm_debug_fast(const cmlb_svm* m, const float* x, int64_t n_rows, int64_t ldx, void* y, double* decision,
                        float* err, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CMLB_H_ */
