/*
 * svm_oracle.c -- C restatement of libsvm's dense prediction as shipped in
 * scikit-learn 1.9 (sklearn/svm/src/libsvm/svm.cpp, svm_predict_values with
 * _DENSE_REP), for SVC / NuSVC / SVR / NuSVR.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Kernel SVMs are not in
 * the reference: scikit-learn is the only oracle, so this file is
 * pinned to golden vectors produced by scikit-learn itself
 * (tools/make_golden_ext.py -> tests/golden/ext_*.npz; tests/test_ext_oracle.py).
 *
 * Arithmetic, all float64, in the order libsvm performs it (established by
 * bit-comparing candidate orders against sklearn's decision_function):
 *   every kernel dot product goes through the host BLAS ddot (sklearn's
 *   svm.cpp passes BlasFunctions); scipy's OpenBLAS 0.3.x dispatches the
 *   SkylakeX kernel on AVX-512 hosts (this container and the B200 box):
 *   FMA into 4 x 8 lanes over n & ~31, fold each 512-bit accumulator to 256
 *   (lo + hi), continue over (n & -16) with 4 x 4 lanes, combine
 *   ((a0 + a1) + a2) + a3, then (l0 + l2) + (l1 + l3), then a sequential FMA
 *   tail over the last n % 16 elements  (ddot_skx below)
 *   rbf     : d_k = x_k - s_k; exp(-gamma * ddot(d, d))
 *   linear  : ddot(x, s)
 *   poly    : powi(gamma*dot + coef0, degree) by binary powering
 *   sigmoid : tanh(gamma*dot + coef0)
 *   pair (i<j): sum = 0; += coef[j-1][k] * K_k over class i's SVs (ascending),
 *             then += coef[i][k] * K_k over class j's; sum -= rho_p where
 *             rho_p = -intercept_p; vote i if sum > 0 else j; first max wins.
 * Build: make -C oracle  (-ffp-contract=off: every fma here is explicit)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
  int32_t kernel;          /* 0 linear, 1 poly, 2 rbf, 3 sigmoid */
  double gamma, coef0;
  int32_t degree;
  const float* sv;         /* [n_sv][F] */
  int32_t n_sv, F;
  const float* coef;       /* [n_coef_rows][n_sv] */
  const float* intercept;  /* [n_pairs] */
  const int32_t* n_support;/* [C] (svc) */
  int32_t C;               /* classes (svc), 0 for svr */
  const float* x;
  int64_t n, ldx;
  double* dec;             /* [n][max(1, n_pairs)] */
  int32_t* vote_class;     /* [n] class index (svc), nullable */
  int64_t lo, hi;
} svm_job_t;

static double powi(double base, int times) {
  double tmp = base, ret = 1.0;
  for (int t = times; t > 0; t /= 2) {
    if (t % 2 == 1) ret *= tmp;
    tmp = tmp * tmp;
  }
  return ret;
}

/* OpenBLAS SkylakeX ddot (kernel/x86_64/ddot.c + ddot_microk_skylakex-2.c order). */
static double ddot_skx(const double* x, const double* y, int n) {
  const int n1 = n & -16, n32 = n1 & ~31;
  double a8[4][8] = {{0}}, a4[4][4];
  int i = 0;
  for (; i < n32; i += 32)
    for (int a = 0; a < 4; ++a)
      for (int l = 0; l < 8; ++l) a8[a][l] = fma(x[i + 8 * a + l], y[i + 8 * a + l], a8[a][l]);
  for (int a = 0; a < 4; ++a)
    for (int l = 0; l < 4; ++l) a4[a][l] = a8[a][l] + a8[a][l + 4];
  for (; i < n1; i += 16)
    for (int a = 0; a < 4; ++a)
      for (int l = 0; l < 4; ++l) a4[a][l] = fma(x[i + 4 * a + l], y[i + 4 * a + l], a4[a][l]);
  double s[4];
  for (int l = 0; l < 4; ++l) s[l] = ((a4[0][l] + a4[1][l]) + a4[2][l]) + a4[3][l];
  double dot = n1 ? (s[0] + s[2]) + (s[1] + s[3]) : 0.0;
  for (i = n1; i < n; ++i) dot = fma(y[i], x[i], dot);
  return dot;
}

static double kvalue(const svm_job_t* j, const float* x, const float* s, double* xd, double* sd) {
  for (int k = 0; k < j->F; ++k) sd[k] = (double)s[k];
  if (j->kernel == 2) {
    for (int k = 0; k < j->F; ++k) sd[k] = (double)x[k] - sd[k];
    return exp(-j->gamma * ddot_skx(sd, sd, j->F));
  }
  for (int k = 0; k < j->F; ++k) xd[k] = (double)x[k];
  const double dot = ddot_skx(xd, sd, j->F);
  if (j->kernel == 0) return dot;
  if (j->kernel == 1) return powi(j->gamma * dot + j->coef0, j->degree);
  return tanh(j->gamma * dot + j->coef0);
}

static void* svm_worker(void* arg) {
  const svm_job_t* j = (const svm_job_t*)arg;
  double* kv = (double*)malloc(sizeof(double) * (size_t)(j->n_sv > 0 ? j->n_sv : 1));
  double* xd = (double*)malloc(sizeof(double) * (size_t)j->F);
  double* sd = (double*)malloc(sizeof(double) * (size_t)j->F);
  const int C = j->C;
  int32_t* start = (int32_t*)malloc(sizeof(int32_t) * (size_t)(C + 1));
  int32_t* vote = (int32_t*)malloc(sizeof(int32_t) * (size_t)(C > 0 ? C : 1));
  if (C > 0) {
    start[0] = 0;
    for (int c = 0; c < C; ++c) start[c + 1] = start[c] + j->n_support[c];
  }
  const int npairs = C > 0 ? C * (C - 1) / 2 : 1;
  for (int64_t r = j->lo; r < j->hi; ++r) {
    const float* x = j->x + r * j->ldx;
    for (int k = 0; k < j->n_sv; ++k) kv[k] = kvalue(j, x, j->sv + (size_t)k * j->F, xd, sd);
    double* dec = j->dec + r * npairs;
    if (C == 0) {  /* svr: one-class regression sum */
      double sum = 0.0;
      for (int k = 0; k < j->n_sv; ++k) sum += (double)j->coef[k] * kv[k];
      sum -= -(double)j->intercept[0];
      dec[0] = sum;
      continue;
    }
    for (int c = 0; c < C; ++c) vote[c] = 0;
    int p = 0;
    for (int a = 0; a < C; ++a) {
      for (int b = a + 1; b < C; ++b) {
        double sum = 0.0;
        const float* c1 = j->coef + (size_t)(b - 1) * j->n_sv;
        const float* c2 = j->coef + (size_t)a * j->n_sv;
        for (int k = start[a]; k < start[a + 1]; ++k) sum += (double)c1[k] * kv[k];
        for (int k = start[b]; k < start[b + 1]; ++k) sum += (double)c2[k] * kv[k];
        sum -= -(double)j->intercept[p];
        dec[p] = sum;
        if (sum > 0) ++vote[a]; else ++vote[b];
        ++p;
      }
    }
    int best = 0;
    for (int c = 1; c < C; ++c)
      if (vote[c] > vote[best]) best = c;
    if (j->vote_class) j->vote_class[r] = best;
  }
  free(kv);
  free(xd);
  free(sd);
  free(start);
  free(vote);
  return NULL;
}

/* Returns 0 on success.  threads <= 0: one per row chunk up to 64. */
int oracle_svm(int32_t kernel, double gamma, double coef0, int32_t degree, const float* sv, int32_t n_sv,
               int32_t F, const float* coef, const float* intercept, const int32_t* n_support, int32_t C,
               const float* x, int64_t n, int64_t ldx, double* dec, int32_t* vote_class, int32_t threads) {
  if (threads <= 0) threads = 1;
  if (threads > 256) threads = 256;
  if (n < threads) threads = n > 0 ? (int32_t)n : 1;
  svm_job_t jobs[256];
  pthread_t tid[256];
  for (int t = 0; t < threads; ++t) {
    svm_job_t* j = &jobs[t];
    j->kernel = kernel; j->gamma = gamma; j->coef0 = coef0; j->degree = degree;
    j->sv = sv; j->n_sv = n_sv; j->F = F; j->coef = coef; j->intercept = intercept;
    j->n_support = n_support; j->C = C; j->x = x; j->n = n; j->ldx = ldx; j->dec = dec;
    j->vote_class = vote_class;
    j->lo = n * t / threads;
    j->hi = n * (t + 1) / threads;
    if (pthread_create(&tid[t], NULL, svm_worker, j) != 0) return 1;
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  return 0;
}
