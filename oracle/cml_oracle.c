/*
 * cml_oracle.c -- multi-threaded C restatement of the reference's tree-ensemble
 * semantics, for full-size parity checks and the CPU baseline.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): nothing in the product
 * package links or calls this.  It shares no code with libcmlb.so: it walks
 * the ORIGINAL node arrays (sklearn/JSON node ids, reference
 * pkg/src/mlower/oracle.py:52-56 pointer chasing), gathers per-tree leaf rows
 * into a buffer, and reduces them exactly like numpy reduces the reference's
 * C-contiguous (N, T, C) float64 stack over axis 1
 * (pkg/src/mlower/kernels.py:180-190):
 *   C >= 2 : out = ((0.0 + v0) + v1) + ...           (strided reduce)
 *   C == 1 : out = 0.0 + pairwise_sum(v0..vT-1)      (contiguous reduce;
 *            numpy's pairwise_sum: < 8 sequential, <= 128 eight accumulators,
 *            else split at n/2 rounded down to a multiple of 8)
 * then float32 rounding, float32 * lr + base (gbdt), float64 sigmoid rounded
 * to float32 (kernels.py:234-235), first-max argmax (kernels.py:197-203).
 * Checked against oracle/semantics.py (numpy, pinned to reference golden
 * vectors) in tests/test_c_oracle.py.
 *
 * Build: make -C oracle   (gcc -O2 -fPIC -shared -pthread, no -ffast-math)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const int64_t* offsets;  /* [T+1] node offsets */
  const uint8_t* is_leaf;
  const int32_t* feature;
  const float* threshold;
  const int32_t* left;     /* node ids local to the tree */
  const int32_t* right;
  const float* value;      /* [nodes][C] */
  const int32_t* leaf_pos; /* [nodes] in-order leaf position, -1 for internal */
  int32_t T, C, F;
  const float* x;
  int64_t n, ldx;
  int32_t agg;             /* 1 mean, 2 sum */
  int32_t tail;            /* 0 values, 1 argmax, 2 sigmoid */
  float lr, base;
  const double* classes;
  int32_t dense_selector;
  double* out;             /* [n][k] */
  int32_t* leaves;         /* nullable [n][T] */
  int64_t lo, hi;
} job_t;

static double pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

static double ref_sigmoid(double x) {
  double e = exp(-fabs(x));
  return x >= 0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
}

static void* work(void* arg) {
  job_t* j = (job_t*)arg;
  const int T = j->T, C = j->C, F = j->F;
  double* buf = (double*)malloc(sizeof(double) * (size_t)T * C);
  double* col = (double*)malloc(sizeof(double) * (size_t)T);
  float* row = (float*)malloc(sizeof(float) * (size_t)F);
  float* mean = (float*)malloc(sizeof(float) * (size_t)C);
  for (int64_t r = j->lo; r < j->hi; ++r) {
    memcpy(row, j->x + r * j->ldx, sizeof(float) * F);
    if (j->dense_selector) { /* 0*inf contamination of the dense selector */
      int bad = 0;
      for (int f = 0; f < F; ++f) bad += !isfinite(row[f]);
      if (bad)
        for (int f = 0; f < F; ++f)
          if (bad >= 2 || isfinite(row[f])) row[f] = NAN;
    }
    for (int t = 0; t < T; ++t) {
      const int64_t base = j->offsets[t];
      int64_t nd = 0;
      while (!j->is_leaf[base + nd]) {
        const int64_t g = base + nd;
        nd = row[j->feature[g]] > j->threshold[g] ? j->right[g] : j->left[g];
      }
      for (int c = 0; c < C; ++c) buf[(size_t)t * C + c] = (double)j->value[(base + nd) * C + c];
      if (j->leaves) j->leaves[r * T + t] = j->leaf_pos[base + nd];
    }
    double* o = j->out + r * (j->tail == 0 ? C : 1);
    if (j->agg == 1) { /* mean over trees */
      for (int c = 0; c < C; ++c) {
        double s;
        if (C == 1) {
          for (int t = 0; t < T; ++t) col[t] = buf[t];
          s = 0.0 + pairwise(col, T);
        } else {
          s = 0.0;
          for (int t = 0; t < T; ++t) s += buf[(size_t)t * C + c];
        }
        mean[c] = (float)(s / (double)T);
      }
      if (j->tail == 1) {
        int best = 0;
        float bv = mean[0];
        if (!isnan(bv))
          for (int c = 1; c < C; ++c) {
            if (isnan(mean[c])) { best = c; break; }
            if (mean[c] > bv) { bv = mean[c]; best = c; }
          }
        o[0] = j->classes[best];
      } else {
        for (int c = 0; c < C; ++c) o[c] = (double)mean[c];
      }
    } else { /* gradient boosting */
      for (int t = 0; t < T; ++t) col[t] = buf[t];
      float s = (float)(0.0 + pairwise(col, T));
      volatile float prod = s * j->lr; /* two float32 roundings, no FMA */
      float raw = prod + j->base;
      if (j->tail == 2) {
        float p = (float)ref_sigmoid((double)raw);
        o[0] = j->classes[p > 0.5f ? 1 : 0];
      } else {
        o[0] = (double)raw;
      }
    }
  }
  free(buf); free(col); free(row); free(mean);
  return NULL;
}

int oracle_forest(const int64_t* offsets, const uint8_t* is_leaf, const int32_t* feature,
                  const float* threshold, const int32_t* left, const int32_t* right,
                  const float* value, const int32_t* leaf_pos, int32_t T, int32_t C, int32_t F,
                  const float* x, int64_t n, int64_t ldx, int32_t agg, int32_t tail, float lr,
                  float base, const double* classes, int32_t dense_selector, double* out,
                  int32_t* leaves, int32_t nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 1024) nthreads = 1024;
  pthread_t th[1024];
  job_t jobs[1024];
  int64_t step = (n + nthreads - 1) / nthreads;
  int used = 0;
  for (int i = 0; i < nthreads; ++i) {
    int64_t lo = i * step, hi = lo + step < n ? lo + step : n;
    if (lo >= hi) break;
    job_t j = {offsets, is_leaf, feature, threshold, left, right, value, leaf_pos, T, C, F, x, n, ldx,
               agg, tail, lr, base, classes, dense_selector, out, leaves, lo, hi};
    jobs[i] = j;
    if (pthread_create(&th[i], NULL, work, &jobs[i]) != 0) return -1;
    ++used;
  }
  for (int i = 0; i < used; ++i) pthread_join(th[i], NULL);
  return 0;
}
