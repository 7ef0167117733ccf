#include <cstdio>
// Kernel SVM operator (SVC / NuSVC / SVR / NuSVR) on sm_100a.
//
// Semantics (not in the reference): libsvm's dense
// svm_predict_values as shipped in scikit-learn -- see oracle/svm_oracle.c,
// which is pinned bit-exactly to scikit-learn.  Per row x:
//   K_j = k(x, sv_j)                         (rbf / poly / sigmoid / linear)
//   dec_p = sum_{j in class a} coef[b-1][j] K_j + sum_{j in class b} coef[a][j] K_j - rho_p
//   for each class pair p = (a < b); vote a iff dec_p > 0; label = first max.
//
// Two kernels:
//
//  * svm_tc_kernel -- the Gram contraction G = X . SV^T (the only O(F) work
//    per (row, SV)) on tcgen05 tensor cores, M = 128 rows x N = 256 support
//    vectors per TMEM accumulator, K = 32 features per pipeline stage.
//    TF32 keeps 10 mantissa bits, so each operand is split exactly,
//    v = big + small (big = v with the low 13 mantissa bits cleared), and
//    G += Xb.Sb + Xs.Sb + Xb.Ss: three tf32 MMAs per K step give ~fp32
//    accuracy ("3xTF32").  SV splits are prepared once on the host in the
//    UMMA core-matrix layout and streamed by TMA bulk copies; row tiles are
//    split on the fly by eight producer warps.  Warp roles: 0-7 A producers
//    (load + split X, two threads per row), 8 B producer (cp.async.bulk),
//    9 MMA issuer (one thread) + TMEM owner, 10-17 epilogue.  TMEM holds two 128 x 256 f32
//    accumulators so the epilogue of SV tile t overlaps the MMAs of t+1.
//    Epilogue (thread = row = TMEM lane): kernel function of the Gram entry,
//    float64 per-class decision sums, a running error bound E for the row;
//    after the last tile: votes -> label.  A row whose decision values are
//    within 4E of zero (a vote could flip) -- or any non-finite value -- is
//    queued for the exact path instead of written.
//
//  * svm_exact_kernel -- persistent; recomputes queued rows in float64 in
//    libsvm's exact operation order (OpenBLAS SkylakeX ddot order for every
//    kernel dot product, sequential decision sums), 32 rows per CTA batch.
//    Residual: CUDA's double exp/tanh may differ from glibc's by an ulp,
//    which moves a decision by ~1e-16 relative.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"

namespace cmlb {
namespace svm {

using namespace sm100;

constexpr int BM = 128;                       // rows per tile = TMEM lanes
constexpr int BN = 256;                       // support vectors per tile = MMA N
constexpr int BK = 32;                        // features per stage (128 B of fp32)
constexpr int STAGES = 2;
constexpr int A_BYTES = BM * BK * 4;          // 16 KB per split half
constexpr int B_BYTES = BN * BK * 4;          // 32 KB per split half
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int A_THREADS = 2 * BM;             // 8 warps: two threads per row, one half of each K chunk
constexpr int B_WARP = A_THREADS / 32;        // TMA producer
constexpr int MMA_WARP = B_WARP + 1;          // MMA issuer + TMEM owner
constexpr int EPI_WARP0 = MMA_WARP + 1;
constexpr int EPI_THREADS = 256;              // 8 warps: 2 per TMEM lane group, one column half each
constexpr int THREADS = EPI_WARP0 * 32 + EPI_THREADS;
constexpr int MAXC = 16;                      // classes handled by the fused epilogue
constexpr int XR = 8;                         // rows per exact-path batch (3 CTAs per SM)
constexpr int XCH = 256;                      // support vectors per exact-path chunk

struct Args {
  const float* x;
  int64_t n_rows, ldx;
  int F, KB, n_tiles, n_sv;
  const uint8_t* bsplit;   // [n_tiles][KB][big | small][BN x BK core-matrix layout]
  const float* ns;         // [n_tiles * BN] |sv|^2 (float64 rounded once)
  const float* w;          // [n_tiles * BN][CPS] coefficient of SV j toward class o (0 for its own class)
  const float* wmax;       // [n_tiles * BN] max_o |w|
  const float* qerr;       // [n_tiles * BN] RBF bound term wmax_j * gamma * 1.075e-6 * |sv_j|^2
  const int32_t* cls;      // [n_tiles * BN] class of SV j, -1 padding
  const double* sv;        // [n_sv][F] float64 copy (exact path)
  const float* coef;       // [rows][n_sv] libsvm sv_coef (exact path)
  const float* intercept;  // [pairs]
  const double* classes;
  int C, CP, pairs, kernel, degree, is_svr, out_dt, vec_x;
  float gamma, coef0;
  double gamma64, coef064;
  void* y;
  double* dec_out;
  float* err_out;          // debug: per-row error bound E (nullable)
  int no_exact;            // debug: write every row from the fast path
  int prob_tol;            // opt-in (CMLB_SVM_TOL=hoeffding): probabilistic vote tolerance, NOT a guarantee
  int probe;               // debug: bit 0 skip X loads, bit 1 skip B copies, bit 2 skip epilogue math
  const cmlb_column_op* pro;  // fused preprocessing (nullable)
  int32_t* queue;          // [n_rows] rows the fast path could not certify
  int32_t* queue_len;
  const double* ns64;      // [n_sv] |sv|^2 in float64 (certifying tier)
  int32_t* queue2;         // rows the float64 certifying tier could not decide -> libsvm-order exact path
  int32_t* queue2_len;
  // pair tier: rows whose only uncertain pair is p (and whose decision values
  // are not wanted) -- the certifying tier then needs the SVs of p's two
  // classes only.  Unsorted entries from the fast path, then bucketed by pair.
  int32_t* pq_row;         // [n_rows]
  int32_t* pq_pair;        // [n_rows]
  unsigned long long* pq_sign;  // [n_rows] bit q: dec_q > 0 (the fast path's certain signs)
  unsigned long long* pq_unc;   // [n_rows] bit q: pair q uncertain in the fast path
  int32_t* pq_len;
  int32_t* pcount;         // [pairs] entries per pair
  int32_t* pcur;           // [pairs] scatter cursors
  int32_t* ps_row;         // [n_rows] bucketed by pair
  unsigned long long* ps_sign;
  unsigned long long* ps_unc;
  // full certifying tier, SV-split: row blocks below cap_blocks are cut into
  // units of CB_SPAN SVs on separate CTAs (one CTA walking all SVs of a block
  // is latency-bound: 12 ms for a 64-row block of config 4b); partial decision
  // sums meet in cacc ([3][cap_blocks * 64][pairs]: sum w K, sum |w| errK,
  // sum |w K|) and svm_certify_finish_kernel decides
  double* cacc;
  int32_t* cflag;          // [cap_blocks * 64] non-finite feature
  int cap_blocks;
  double* pacc;            // pair tier: [3][pq_cap] partial sums per bucketed entry
  int32_t* pflag;          // [pq_cap] non-finite feature
  int pq_cap;              // pair-tier capacity (rows past it take the full tier)
};

__host__ __device__ inline int pair_index(int a, int b, int C) {  // a < b
  return a * (2 * C - a - 1) / 2 + (b - a - 1);
}

// ---------------------------------------------------------------------------
// fast path
// ---------------------------------------------------------------------------

// Kernel value of a Gram entry and its error bound.  de bounds the Gram
// entry's error: the dropped small*small products are each below
// 2^-20 |x_k s_k| (a tf32 "big" half keeps 11 significant bits), so they sum
// to <= 2^-20 |x| |s| <= 2^-21 (|x|^2 + |s|^2) (Cauchy-Schwarz); the tf32
// rounding of the small halves contributes the same order again, and the
// caller's 4x safety factor on the accumulated bound covers both plus the
// f32 accumulation.  Measured errors are 100-1000x below this bound
// (tools/svm_error_probe.py, profiles/r1_svm_error_probe.jsonl).
__device__ __forceinline__ float kvalue_fast(const Args& a, float g, float nx, float nsj, float& err) {
  const float de = 4.76837158203125e-07f * (nx + nsj);  // 2^-21
  if (a.kernel == CMLB_SVM_RBF) {
    // d2 = nx + ns - 2g: error 2 de (Gram) + one f32 rounding of ~(nx + ns);
    // ex2.approx: ~2 ulp; the f32 argument product: 1 ulp of ~3
    const float d2 = fmaxf(fmaf(-2.0f, g, nx + nsj), 0.0f);
    float k;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(k) : "f"(-a.gamma * 1.4426950408889634f * d2));
    err = k * (a.gamma * (2.0f * de + 1.2e-7f * (nx + nsj)) + 6.0e-7f);
    return k;
  }
  if (a.kernel == CMLB_SVM_LINEAR) {
    err = de + 1.2e-7f * fabsf(g);
    return g;
  }
  const float u = fmaf(a.gamma, g, a.coef0);
  if (a.kernel == CMLB_SVM_POLY) {
    float k = 1.0f, du = 1.0f;  // u^deg and u^(deg-1)
    for (int i = 0; i < a.degree; ++i) {
      if (i + 1 < a.degree) du *= u;
      k *= u;
    }
    err = (float)a.degree * (fabsf(du) * (a.gamma * de + 1.2e-7f * fabsf(u)) + 2.4e-7f * fabsf(k)) + 1e-30f;
    return k;
  }
  const float k = tanhf(u);
  err = (1.0f - k * k) * (a.gamma * de + 1.2e-7f * fabsf(u)) + 4.0e-7f;
  return k;
}

template <int CP>
__device__ __forceinline__ void flush(const Args& a, int cur, const double (&acc)[CP], double* dec) {
  if (cur < 0) return;
  if (a.is_svr) {
    dec[0] += acc[0];
    return;
  }
#pragma unroll
  for (int o = 0; o < CP; ++o) {
    if (o < a.C && o != cur) {
      const int p = o < cur ? pair_index(o, cur, a.C) : pair_index(cur, o, a.C);
      dec[p] += acc[o];
    }
  }
}

// SVR: every value within tol of v rounds to the same float32 (rounding is
// monotone), so the reference's float32 output equals ours.
__device__ __forceinline__ bool f32_round_certain(double v, double tol) {
  const double lo = __dsub_rd(v, tol), hi = __dadd_ru(v, tol);
  return isfinite(lo) && isfinite(hi) && __double2float_rn(lo) == __double2float_rn(hi);
}

// Vote-robust class: with `unc` marking the pairs whose sign is not certain,
// class w is libsvm's answer for EVERY resolution of those pairs when its
// certain votes beat every other class's certain-plus-uncertain votes
// (strictly for lower-indexed classes, which win ties).  Returns w, or -1.
__device__ __forceinline__ int robust_vote(const int* vmin, const int* unc, int C) {
  int w = 0;
  for (int c = 1; c < C; ++c)
    if (vmin[c] > vmin[w]) w = c;
  for (int c = 0; c < C; ++c) {
    if (c == w) continue;
    const int hi = vmin[c] + unc[c];
    if (c < w ? !(vmin[w] > hi) : !(vmin[w] >= hi)) return -1;
  }
  return w;
}

template <int CP>
__global__ void __launch_bounds__(THREADS, 1) svm_tc_kernel(const Args a) {
  constexpr int CPS = (CP + 3) & ~3;  // w row stride (16-byte aligned rows)
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  const int KB = a.KB, NT = a.n_tiles;
  const int total = NT * KB;

  // epilogue tables (after the stages)
  float* w_s = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);   // [BN][CPS]
  float* ns_s = w_s + BN * CPS;
  float* wm_s = ns_s + BN;
  int32_t* cls_s = reinterpret_cast<int32_t*>(wm_s + BN);
  float* q_s = reinterpret_cast<float*>(cls_s + BN);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full_bar[s], A_THREADS + 1);
      bar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      bar_init(&tfull_bar[b], 1);
      bar_init(&tempty_bar[b], EPI_THREADS);
    }
    bar_fence_init();
  }
  if (warp == MMA_WARP) tmem_alloc(&tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (tid < A_THREADS) {
    // ---- A producers: thread r owns row r of the tile --------------------
    // The row's next 32 features are loaded into registers BEFORE waiting for
    // their stage to drain, so the L2 latency overlaps the MMAs in flight.
    constexpr int CH = BK / 8;               // float4 chunks per thread per stage
    const int r = tid & (BM - 1), c0 = (tid / BM) * CH;
    const int64_t row = row0 + r;
    const bool valid = row < a.n_rows;
    const float* src = a.x + (valid ? row : 0) * a.ldx;
    float4 v[CH];
    auto load_k = [&](int kb) {
      const int k0 = kb * BK;
#pragma unroll
      for (int cc = 0; cc < CH; ++cc) {
        const int c = c0 + cc;
        const int k = k0 + 4 * c;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid && !(a.probe & 1)) {
          if (a.pro) {
            if (k < a.F) q.x = load_col(a.pro, src, k);
            if (k + 1 < a.F) q.y = load_col(a.pro, src, k + 1);
            if (k + 2 < a.F) q.z = load_col(a.pro, src, k + 2);
            if (k + 3 < a.F) q.w = load_col(a.pro, src, k + 3);
          } else if (a.vec_x && k + 3 < a.F) {
            q = __ldg(reinterpret_cast<const float4*>(src + k));
          } else {
            if (k < a.F) q.x = __ldg(src + k);
            if (k + 1 < a.F) q.y = __ldg(src + k + 1);
            if (k + 2 < a.F) q.z = __ldg(src + k + 2);
            if (k + 3 < a.F) q.w = __ldg(src + k + 3);
          }
        }
        v[cc] = q;
      }
    };
    load_k(0);
    for (int it = 0; it < total; ++it) {
      const int s = it % STAGES;
      bar_wait(&empty_bar[s], ((it / STAGES) & 1) ^ 1);
      uint8_t* abig = smem + s * STAGE_BYTES;
      uint8_t* asmall = abig + A_BYTES;
#pragma unroll
      for (int cc = 0; cc < CH; ++cc) {
        const int c = c0 + cc;
        float4 hi, lo;
        hi.x = __uint_as_float(__float_as_uint(v[cc].x) & 0xFFFFE000u); lo.x = v[cc].x - hi.x;
        hi.y = __uint_as_float(__float_as_uint(v[cc].y) & 0xFFFFE000u); lo.y = v[cc].y - hi.y;
        hi.z = __uint_as_float(__float_as_uint(v[cc].z) & 0xFFFFE000u); lo.z = v[cc].z - hi.z;
        hi.w = __uint_as_float(__float_as_uint(v[cc].w) & 0xFFFFE000u); lo.w = v[cc].w - hi.w;
        *reinterpret_cast<float4*>(abig + c * (BM * 16) + r * 16) = hi;
        *reinterpret_cast<float4*>(asmall + c * (BM * 16) + r * 16) = lo;
      }
      fence_async_smem();
      bar_arrive(&full_bar[s]);
      if (it + 1 < total) load_k((it + 1) % KB);
    }
  } else if (warp == B_WARP) {
    // ---- B producer: one bulk copy of the pre-split SV stage -------------
    if (lane == 0) {
      for (int it = 0; it < total; ++it) {
        const int s = it % STAGES;
        bar_wait(&empty_bar[s], ((it / STAGES) & 1) ^ 1);
        uint8_t* dst = smem + s * STAGE_BYTES + 2 * A_BYTES;
        const uint8_t* src = a.bsplit + (size_t)it * (2 * B_BYTES);
        if (a.probe & 2) {
          bar_arrive(&full_bar[s]);
        } else {
          bar_arrive_tx(&full_bar[s], 2 * B_BYTES);
          bulk_load(dst, src, B_BYTES, &full_bar[s]);
          bulk_load(dst + B_BYTES, src + B_BYTES, B_BYTES, &full_bar[s]);
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ---- MMA issuer ------------------------------------------------------
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(BM, BN);
      const uint32_t sbase = smem_addr(smem);
      for (int t = 0; t < NT; ++t) {
        const int b = t & 1;
        bar_wait(&tempty_bar[b], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * BN);
        for (int kb = 0; kb < KB; ++kb) {
          const int it = t * KB + kb, s = it % STAGES;
          bar_wait(&full_bar[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t abig = sbase + s * STAGE_BYTES, asmall = abig + A_BYTES;
          const uint32_t bbig = abig + 2 * A_BYTES, bsmall = bbig + B_BYTES;
#pragma unroll
          for (int k8 = 0; k8 < BK / 8; ++k8) {
            const uint32_t ao = (uint32_t)k8 * 2 * (BM * 16), bo = (uint32_t)k8 * 2 * (BN * 16);
            const uint64_t ab = desc_kmajor(abig + ao, BM * 16, 128), as = desc_kmajor(asmall + ao, BM * 16, 128);
            const uint64_t bb = desc_kmajor(bbig + bo, BN * 16, 128), bs = desc_kmajor(bsmall + bo, BN * 16, 128);
            mma_tf32(d, ab, bb, idesc, (kb | k8) != 0);
            mma_tf32(d, as, bb, idesc, 1u);
            mma_tf32(d, ab, bs, idesc, 1u);
          }
          mma_commit(&empty_bar[s]);  // stage s free once these MMAs retire
        }
        mma_commit(&tfull_bar[b]);    // accumulator b complete
      }
    }
  } else {
    // ---- epilogue: thread = row = TMEM lane; two warps per lane group ---
    const int e = warp - EPI_WARP0;          // 0..7
    const int eg = warp & 3;                 // TMEM lane group this warp may access
    const int half = e >> 2;                 // which 128 columns of each tile
    const int r = eg * 32 + lane;
    const int et = tid - EPI_WARP0 * 32;     // 0..255 (cooperative table loads)
    const int64_t row = row0 + r;
    const bool valid = row < a.n_rows;
    float nx = 0.0f;
    if (valid) {
      const float* src = a.x + row * a.ldx;
      double s = 0.0;
      for (int k = 0; k < a.F; ++k) {
        const double v = (double)load_col(a.pro, src, k);
        s = fma(v, v, s);
      }
      nx = (float)s;
    }
    double acc[CP];
    float pacc[CP];
#pragma unroll
    for (int o = 0; o < CP; ++o) acc[o] = 0.0, pacc[o] = 0.0f;
    double dec[MAXC * (MAXC - 1) / 2];
    for (int p = 0; p < a.pairs; ++p) dec[p] = 0.0;
    float err_sum = 0.0f, err_sq = 0.0f;
    // per-class share of the bound: pair (i, k) only sums SVs of classes i and k
    // (libsvm one-vs-one), so its tolerance is 4 (errc[i] + errc[k]), not 4 E
    float errc[MAXC], err_flushed = 0.0f;
    for (int c = 0; c < MAXC; ++c) errc[c] = 0.0f;
    int cur = -1;
    const bool rbf = a.kernel == CMLB_SVM_RBF;
    const float neg_gl2 = -a.gamma * 1.4426950408889634f;
    const float alpha = a.gamma * 1.075e-6f * nx + 1.077e-6f;
    // fp32 partial sums over <= 8 columns, folded into the fp64 class sums:
    // each adds at most 2^-21 sum|w K| of error, charged to the bound below
    auto fold = [&]() {
#pragma unroll
      for (int o = 0; o < CP; ++o) {
        acc[o] += (double)pacc[o];
        pacc[o] = 0.0f;
      }
    };
    for (int t = 0; t < NT; ++t) {
      const int b = t & 1;
      // this tile's SV tables -> shared memory (previous tile's readers are done)
      named_bar_sync(1, EPI_THREADS);
      {
        const int j0 = t * BN;
        for (int i = et; i < BN * CPS; i += EPI_THREADS) w_s[i] = __ldg(a.w + (size_t)j0 * CPS + i);
        for (int i = et; i < BN; i += EPI_THREADS) {
          ns_s[i] = __ldg(a.ns + j0 + i);
          wm_s[i] = __ldg(a.wmax + j0 + i);
          cls_s[i] = __ldg(a.cls + j0 + i);
          q_s[i] = __ldg(a.qerr + j0 + i);
        }
      }
      named_bar_sync(1, EPI_THREADS);
      bar_wait(&tfull_bar[b], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(eg * 32) << 16) + (uint32_t)(b * BN);
      for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += 32) {
        uint32_t g[32];
        tmem_ld32(taddr + (uint32_t)c0, g);
        if (a.probe & 4) continue;
#pragma unroll
        for (int grp = 0; grp < 4; ++grp) {
          const int jg = c0 + grp * 8;
          if (rbf && cls_s[jg] == cur && cls_s[jg + 7] == cur) {
            // common case: 8 SVs of the current class, RBF -- branch-free.
            // b_j = K_j * (wmax_j * alpha + q_j) is the per-SV bound of
            // kvalue_fast (Gram error, d2 rounding, ex2, fp32 partials)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int j = jg + jj;
              const float d2 = fmaxf(fmaf(-2.0f, __uint_as_float(g[grp * 8 + jj]), nx + ns_s[j]), 0.0f);
              float k;
              asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(k) : "f"(neg_gl2 * d2));
              const float bj = k * fmaf(wm_s[j], alpha, q_s[j]);
              err_sum += bj;
              err_sq = fmaf(bj, bj, err_sq);
              const float* wj = w_s + j * CPS;
#pragma unroll
              for (int o = 0; o < CP; ++o) pacc[o] = fmaf(wj[o], k, pacc[o]);
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int j = jg + jj;
              const int c = cls_s[j];
              if (c != cur) {  // uniform: classes are contiguous
                fold();
                flush<CP>(a, cur, acc, dec);
                if (cur >= 0) errc[cur] += err_sum - err_flushed;
                err_flushed = err_sum;
#pragma unroll
                for (int o = 0; o < CP; ++o) acc[o] = 0.0;
                cur = c;
              }
              float ek;
              const float k = kvalue_fast(a, __uint_as_float(g[grp * 8 + jj]), nx, ns_s[j], ek);
              const float we = wm_s[j] * (ek + 4.76837158203125e-07f * fabsf(k));
              err_sum += we;
              err_sq = fmaf(we, we, err_sq);
              const float* wj = w_s + j * CPS;
#pragma unroll
              for (int o = 0; o < CP; ++o) pacc[o] = fmaf(wj[o], k, pacc[o]);
            }
          }
          fold();
        }
      }
      tc_fence_before();
      bar_arrive(&tempty_bar[b]);
    }
    flush<CP>(a, cur, acc, dec);
    if (cur >= 0) errc[cur] += err_sum - err_flushed;
    // combine the two column halves of each row: half 1 hands its sums over
    float* xch = reinterpret_cast<float*>(smem);  // the stages are idle now
    double* xd = reinterpret_cast<double*>(xch);
    named_bar_sync(1, EPI_THREADS);               // every epilogue thread is past its last tile
    const int nc = a.is_svr ? 0 : a.C;
    const int stride = a.pairs + 1 + nc;
    if (half == 1) {
      for (int p = 0; p < a.pairs; ++p) xd[r * stride + p] = dec[p];
      xd[r * stride + a.pairs] = (double)err_sum;
      for (int c = 0; c < nc; ++c) xd[r * stride + a.pairs + 1 + c] = (double)errc[c];
      xch[2 * BM * stride + r] = err_sq;
    }
    named_bar_sync(1, EPI_THREADS);
    if (half == 1) return;
    for (int p = 0; p < a.pairs; ++p) dec[p] += xd[r * stride + p];
    err_sum += (float)xd[r * stride + a.pairs];
    for (int c = 0; c < nc; ++c) errc[c] += (float)xd[r * stride + a.pairs + 1 + c];
    err_sq += xch[2 * BM * stride + r];
    if (valid) {
      // b_j = per-SV error bound and E = sum b_j: the deterministic bound
      // with every per-SV error aligned.  The vote threshold is tol = 4 E,
      // so a row the fast path decides is provably decided like the float64
      // path; every other row is recomputed exactly.  (Opt-in only,
      // CMLB_SVM_TOL=hoeffding: tol = min(4 E, 8 sigma) with sigma^2 = sum
      // b_j^2, a Hoeffding argument that assumes independent zero-mean
      // per-SV errors -- not a guarantee, since the tf32 split residual of
      // x repeats across all SVs.  Measured errors stay below 0.2 sigma,
      // tools/svm_error_probe.py.)
      const float bound = a.prob_tol ? fminf(err_sum, 2.0f * sqrtf(err_sq)) : err_sum;
      const float tol = 4.0f * bound + 1e-30f;
      if (a.err_out) a.err_out[row] = bound;
      bool exact = !(tol < 3.0e38f);
      if (a.is_svr) {
        const double v = dec[0] + (double)a.intercept[0];
        exact = exact || !f32_round_certain(v, (double)tol);
        if (a.no_exact) exact = false;
        if (!exact) {
          store_out(a.y, row, a.out_dt, (double)(float)v);
          if (a.dec_out) a.dec_out[row] = v;
        }
      } else {
        // certain votes (vote) and uncertain pairs per class (unc): a pair is
        // uncertain when |dec| is inside its tolerance
        int vote[MAXC], unc[MAXC];
        for (int c = 0; c < a.C; ++c) vote[c] = unc[c] = 0;
        bool any_unc = false, nonfin = false;
        int n_unc = 0;
        unsigned long long signs = 0ull, uncmask = 0ull;
        int p = 0;
        for (int i = 0; i < a.C; ++i) {
          for (int j = i + 1; j < a.C; ++j, ++p) {
            const double v = dec[p] + (double)a.intercept[p];
            dec[p] = v;
            const float tol_p = a.prob_tol ? tol : 4.0f * (errc[i] + errc[j]) + 1e-30f;
            nonfin = nonfin || !isfinite(v);
            if (p < 64 && v > 0) signs |= 1ull << p;
            if (!(fabs(v) > (double)tol_p)) {
              any_unc = true;
              ++unc[i];
              ++unc[j];
              ++n_unc;
              if (p < 64) uncmask |= 1ull << p;
            } else if (v > 0) {
              ++vote[i];
            } else {
              ++vote[j];
            }
          }
        }
        // uncertain pairs need the exact path only when they could change the
        // class (or when the decision values themselves are wanted)
        int best = -1;
        if (!exact && !nonfin && (!any_unc || !a.dec_out)) best = robust_vote(vote, unc, a.C);
        exact = best < 0;
        if (a.no_exact && exact) {  // debug probe: vote with the fast-path signs as they are
          for (int c = 0; c < a.C; ++c) vote[c] = 0;
          p = 0;
          for (int i = 0; i < a.C; ++i)
            for (int j = i + 1; j < a.C; ++j, ++p) {
              if (dec[p] > 0) ++vote[i]; else ++vote[j];
            }
          best = 0;
          for (int c = 1; c < a.C; ++c)
            if (vote[c] > vote[best]) best = c;
          exact = false;
        }
        if (!exact) {
          store_out(a.y, row, a.out_dt, a.classes[best]);
          if (a.dec_out)
            for (int q = 0; q < a.pairs; ++q) a.dec_out[row * a.pairs + q] = dec[q];
        } else if (a.pq_row && n_unc >= 1 && !nonfin && !a.dec_out && !(tol >= 3.0e38f)) {
          // the pair tier resolves the uncertain pair between the strongest
          // contenders from its two classes' SVs; what stays uncertain after
          // that goes on to the full certifying tier
          int p_best = -1, s_best = -1;
          p = 0;
          for (int i = 0; i < a.C; ++i)
            for (int j = i + 1; j < a.C; ++j, ++p)
              if ((uncmask >> p) & 1ull) {
                const int sc = min(vote[i] + unc[i], vote[j] + unc[j]);
                if (sc > s_best) { s_best = sc; p_best = p; }
              }
          const int q = atomicAdd(a.pq_len, 1);
          if (q < a.pq_cap) {
            a.pq_row[q] = (int32_t)row;
            a.pq_pair[q] = p_best;
            a.pq_sign[q] = signs;
            a.pq_unc[q] = uncmask;
            atomicAdd(a.pcount + p_best, 1);
            exact = false;
          }
        }
      }
      if (exact) a.queue[atomicAdd(a.queue_len, 1)] = (int32_t)row;
    }
    return;
  }
  // producers and the MMA warp: TMEM is released once the epilogue has
  // drained the last accumulator (its final tempty arrival)
  if (warp == MMA_WARP) {
    if (NT >= 1) bar_wait(&tempty_bar[(NT - 1) & 1], ((NT - 1) >> 1) & 1);
    tc_fence_after();
    tmem_free(tmem, 512);
  }
}

// ---------------------------------------------------------------------------
// exact path: libsvm order in float64
// ---------------------------------------------------------------------------

// OpenBLAS SkylakeX ddot order (oracle/svm_oracle.c: ddot_skx) for one
// (row, SV) pair; xs = the row's features in shared memory (float64, one
// padded row), s = the SV in float64.  RBF: the vectors are d = x - s
// (ddot(d, d)); otherwise ddot(x, s).
__device__ double exact_dot(const double* xs, const double* s, int F, bool rbf) {
  const int n1 = F & -16, n32 = n1 & ~31;
  auto term = [&](int k, double acc) {
    const double xv = xs[k], sv = __ldg(s + k);
    if (rbf) {
      const double d = __dsub_rn(xv, sv);
      return fma(d, d, acc);
    }
    return fma(xv, sv, acc);
  };
  auto term2 = [&](double xv, double sv, double acc) {
    if (rbf) {
      const double d = __dsub_rn(xv, sv);
      return fma(d, d, acc);
    }
    return fma(xv, sv, acc);
  };
  // stream k in order: element k feeds lane k % 32 of the 4 x 8 AVX-512
  // accumulators (32 independent FMA chains), then lane k % 16 of the
  // 4 x 4 AVX2 ones; x (padded shared-memory row) and the SV are read two
  // doubles at a time when F is even
  double a8[32];
#pragma unroll
  for (int u = 0; u < 32; ++u) a8[u] = 0.0;
  int k = 0;
  if ((F & 1) == 0) {
    for (; k < n32; k += 32) {
#pragma unroll
      for (int u = 0; u < 32; u += 2) {
        const double2 xv = *reinterpret_cast<const double2*>(xs + k + u);
        const double2 sv = __ldg(reinterpret_cast<const double2*>(s + k + u));
        a8[u] = term2(xv.x, sv.x, a8[u]);
        a8[u + 1] = term2(xv.y, sv.y, a8[u + 1]);
      }
    }
  } else {
    for (; k < n32; k += 32) {
#pragma unroll
      for (int u = 0; u < 32; ++u) a8[u] = term(k + u, a8[u]);
    }
  }
  double a4[16];
#pragma unroll
  for (int aa = 0; aa < 4; ++aa)
#pragma unroll
    for (int l = 0; l < 4; ++l) a4[aa * 4 + l] = __dadd_rn(a8[aa * 8 + l], a8[aa * 8 + l + 4]);
  for (; k < n1; k += 16) {
#pragma unroll
    for (int u = 0; u < 16; ++u) a4[u] = term(k + u, a4[u]);
  }
  double sl[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) sl[l] = __dadd_rn(__dadd_rn(__dadd_rn(a4[l], a4[4 + l]), a4[8 + l]), a4[12 + l]);
  double dot = n1 ? __dadd_rn(__dadd_rn(sl[0], sl[2]), __dadd_rn(sl[1], sl[3])) : 0.0;
  for (int i = n1; i < F; ++i) dot = term(i, dot);
  return dot;
}

__device__ double exact_k(const Args& a, const double* xs, const double* s) {
  if (a.kernel == CMLB_SVM_RBF) return exp(__dmul_rn(-a.gamma64, exact_dot(xs, s, a.F, true)));
  const double dot = exact_dot(xs, s, a.F, false);
  if (a.kernel == CMLB_SVM_LINEAR) return dot;
  const double u = __dadd_rn(__dmul_rn(a.gamma64, dot), a.coef064);
  if (a.kernel == CMLB_SVM_SIGMOID) return tanh(u);
  double tmp = u, ret = 1.0;  // libsvm powi
  for (int t = a.degree; t > 0; t /= 2) {
    if (t % 2 == 1) ret = __dmul_rn(ret, tmp);
    tmp = __dmul_rn(tmp, tmp);
  }
  return ret;
}

constexpr int XTHREADS = 256;

// ---------------------------------------------------------------------------
// certifying tier: float64 Gram for the rows the fast path queued
// ---------------------------------------------------------------------------
//
// The fast path's bound covers the split residuals and kernel-function
// roundings, but the fp32 accumulation inside the tensor core is modeled, not
// proved, and a worst-case fp32 bound would flag most rows.  The rows it
// queues are therefore decided here with float64 arithmetic whose error is
// bounded RIGOROUSLY against libsvm's own float64 computation:
//   G = x.s as a sequential float64 FMA chain (|err| <= gamma_F sum|x_k s_k|
//   <= gamma_F sqrt(nx ns)), d2 = nx + ns - 2G, K = kernel(d2 or G), then the
//   decision sums in libsvm's order (class-i block, class-k block, - rho).
//   libsvm computes the same decision with its own float64 roundings; both
//   differ from the exact value by at most the standard gamma_n bounds, so
//   |dec_ours - dec_libsvm| <= tol2 = sum|w_j| errK_j + 2 gamma_{n+2} (sum|w_j K_j| + |rho|)
//   and a pair with |dec_ours| > tol2 votes exactly as libsvm does.
// Rows with any pair inside tol2 (or a non-finite feature) go on to the
// libsvm-order exact kernel.  Tile: 64 rows x 64 SVs per CTA step, 4 x 4
// outputs per thread, K staged in 32-feature float64 chunks (double-buffered);
// decision sums per (row, pair) task in ascending SV order (deterministic).
constexpr int CB_ROWS = 64, CB_SV = 64, CB_K = 16, CB_THREADS = 256;
constexpr int CB_KS = CB_K + 4, CB_SS = CB_SV + 1;              // padded strides: KS = 20 doubles puts the DMMA
                                                                  // fragment loads of a half warp in 16 distinct bank pairs
constexpr int CB_TPT = 12;                                        // (row, pair) tasks per thread: pairs <= 48
constexpr int CB_MAXP = CB_TPT * CB_THREADS / CB_ROWS;
constexpr size_t CB_SMEM = (size_t)2 * (CB_ROWS + CB_SV) * CB_KS * 8 + (size_t)2 * CB_ROWS * CB_SS * 8 + CB_ROWS * 8;
constexpr int CB_SPAN = 4 * CB_SV;                               // SVs per split unit
constexpr int CB_CAP_BLOCKS = 256;                               // split row blocks (16,384 rows)

__device__ __forceinline__ double gamma_n(int n) {
  const double nu = n * 1.1102230246251565e-16;  // n * 2^-53
  return nu / (1.0 - nu);
}

// PAIR: the pair tier -- blocks of 64 rows that share their one uncertain pair
// p = (ca, cb); only the SVs of classes ca and cb enter the Gram, only pair p's
// decision is formed, and the other pairs' signs come from the fast path.
template <bool PAIR>
__global__ void __launch_bounds__(CB_THREADS, 2) svm_certify_kernel(const Args a, const int* n_sv_start) {
  extern __shared__ __align__(16) uint8_t csm[];
  double* xc = reinterpret_cast<double*>(csm);                  // [2][CB_ROWS][CB_KS]
  double* sc = xc + 2 * CB_ROWS * CB_KS;                          // [2][CB_SV][CB_KS]
  double* ks = sc + 2 * CB_SV * CB_KS;                            // [CB_ROWS][CB_SS] kernel values
  double* eks = ks + CB_ROWS * CB_SS;                              // [CB_ROWS][CB_SS] |K_ours - K_libsvm| bounds
  double* nxs = eks + CB_ROWS * CB_SS;                             // [CB_ROWS] |x|^2
  __shared__ int32_t rows[CB_ROWS];
  __shared__ int undecided[CB_ROWS];                 // non-finite feature: the exact kernel decides
  __shared__ unsigned long long uncm[CB_ROWS];       // bit p: pair p inside its bound
  __shared__ int pblk[65], poff[65], punits[65];     // PAIR: per-pair unit / entry prefix sums, units per block
  const int tid = threadIdx.x;
  const int F = a.F, C = a.C;
  const int npairs = a.is_svr ? 1 : a.pairs;
  const int ntasks = PAIR ? CB_ROWS : CB_ROWS * npairs;
  int nblocks, sblocks = 0, nsplit = 1;
  if constexpr (PAIR) {
    if (tid == 0) {
      // units: (row block of a pair's bucket, group of CB_SPAN / CB_SV SV tiles
      // of the pair's two classes)
      int usum = 0, esum0 = 0, qa = 0, qr = 0;
      for (int q = 0; q < a.pairs; ++q) {
        const int qb = qa + 1 + qr;  // pair q = (qa, qb)
        const int ta = (n_sv_start[qa + 1] - n_sv_start[qa] + CB_SV - 1) / CB_SV;
        const int tb = (n_sv_start[qb + 1] - n_sv_start[qb] + CB_SV - 1) / CB_SV;
        punits[q] = max(1, (ta + tb + CB_SPAN / CB_SV - 1) / (CB_SPAN / CB_SV));
        pblk[q] = usum;
        poff[q] = esum0;
        const int c = a.pcount[q];
        usum += (c + CB_ROWS - 1) / CB_ROWS * punits[q];
        esum0 += c;
        if (++qr == C - 1 - qa) { ++qa; qr = 0; }
      }
      pblk[a.pairs] = usum;
      poff[a.pairs] = esum0;
    }
    __syncthreads();
    nblocks = pblk[a.pairs];
  } else {
    const int nrb = (*a.queue_len + CB_ROWS - 1) / CB_ROWS;
    sblocks = a.cacc ? min(nrb, a.cap_blocks) : 0;
    nsplit = (a.n_sv + CB_SPAN - 1) / CB_SPAN;
    nblocks = sblocks * nsplit + (nrb - sblocks);  // split units, then whole blocks
  }
  // The Gram on the FP64 tensor pipe: mma.sync m8n8k4 f64 (DMMA, 256 FMAs per
  // instruction; measured at the DFMA rate, 64 FMAs/clk/SM, with 1/8 of the
  // issue slots and operand traffic).  Warp tile 32 rows x 16 SVs = 4 x 2 MMA
  // tiles; 8 warps cover the 64 x 64 CTA tile.  Fragments (PTX m8n8k4 .f64):
  // a = A[g][t], b = B[t][g], c = C[g][2t + {0,1}] with g = lane / 4, t = lane % 4.
  const int warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int rw0 = 32 * (warp >> 2), sw0 = 16 * (warp & 3);
  // the DMMA accumulation order and internal roundings are the hardware's:
  // charge 2 roundings per term (covers round-toward-zero adds too)
  const double gF = gamma_n(2 * F + 6);
  constexpr double U = 1.1102230246251565e-16;
  for (int blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    int nb, bp = 0;  // rows in this block; PAIR: their shared pair
    int rb = 0, jlo = 0, jhi = a.n_sv;  // general: row block and SV range of this unit
    bool split = false;
    int pfirst = 0, pgroup = 0;  // PAIR: first sorted entry of the block, SV tile group of the unit
    if constexpr (PAIR) {
      while (blk >= pblk[bp + 1]) ++bp;
      const int ub = blk - pblk[bp];
      pgroup = ub % punits[bp];
      const int first = (ub / punits[bp]) * CB_ROWS;
      pfirst = poff[bp] + first;
      nb = min(CB_ROWS, a.pcount[bp] - first);
      if (tid < CB_ROWS) rows[tid] = tid < nb ? a.ps_row[pfirst + tid] : -1;
      split = true;
    } else {
      if (blk < sblocks * nsplit) {
        rb = blk / nsplit;
        jlo = (blk % nsplit) * CB_SPAN;
        jhi = min(a.n_sv, jlo + CB_SPAN);
        split = true;
      } else {
        rb = sblocks + (blk - sblocks * nsplit);
      }
      const int b0 = rb * CB_ROWS;
      nb = min(CB_ROWS, *a.queue_len - b0);
      if (tid < CB_ROWS) rows[tid] = tid < nb ? a.queue[b0 + tid] : -1;
    }
    // SV segments: every SV, or (PAIR) the SVs of the block pair's two classes
    int pca = 0, pcb = 0;
    if constexpr (PAIR) {
      int rem = bp;
      while (rem >= C - 1 - pca) { rem -= C - 1 - pca; ++pca; }
      pcb = pca + 1 + rem;
    }
    int seg_lo[2] = {jlo, 0}, seg_hi[2] = {jhi, 0};
    if constexpr (PAIR) {  // this unit's tiles of the concatenated class-ca, class-cb SV lists
      const int sa = n_sv_start[pca], ea = n_sv_start[pca + 1], sb = n_sv_start[pcb], eb = n_sv_start[pcb + 1];
      const int ta = (ea - sa + CB_SV - 1) / CB_SV, tb = (eb - sb + CB_SV - 1) / CB_SV;
      const int t0 = pgroup * (CB_SPAN / CB_SV), t1 = min(t0 + CB_SPAN / CB_SV, ta + tb);
      seg_lo[0] = sa + CB_SV * min(t0, ta);
      seg_hi[0] = min(ea, sa + CB_SV * min(t1, ta));
      seg_lo[1] = sb + CB_SV * (max(t0, ta) - ta);
      seg_hi[1] = t1 > ta ? min(eb, sb + CB_SV * (t1 - ta)) : seg_lo[1];
    }
    __syncthreads();
    if (tid < CB_ROWS) {  // |x|^2 in float64 and the non-finite check
      double sacc = 0.0;
      int nf = 0;
      if (rows[tid] >= 0) {
        const float* src = a.x + (int64_t)rows[tid] * a.ldx;
        for (int k = 0; k < F; ++k) {
          const double v = (double)load_col(a.pro, src, k);
          nf |= !isfinite(v);
          sacc = fma(v, v, sacc);
        }
      }
      nxs[tid] = sacc;
      undecided[tid] = nf;
      uncm[tid] = 0ull;
    }
    double dsum[CB_TPT], esum[CB_TPT];
    float asum[CB_TPT];  // sum |w K|, rounded up (an upper bound is all the certificate needs)
#pragma unroll
    for (int q = 0; q < CB_TPT; ++q) dsum[q] = esum[q] = 0.0, asum[q] = 0.0f;
    __syncthreads();
    const int nkc = (F + CB_K - 1) / CB_K;
    for (int sg = 0; sg < 2; ++sg)
    for (int j0 = seg_lo[sg]; j0 < seg_hi[sg]; j0 += CB_SV) {
      const int nj = min(CB_SV, seg_hi[sg] - j0);
      double g[4][2][2];  // [row block][SV block][c0, c1]
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) g[i][j][0] = g[i][j][1] = 0.0;
      // chunk kc: SVs by cp.async (float64 already), x by a register prefetch
      // of the next chunk (float32 -> float64 on the way into shared memory)
      float xpre[CB_ROWS * CB_K / CB_THREADS];
      auto load_x = [&](int kc) {
        const int k0 = kc * CB_K;
#pragma unroll
        for (int u = 0; u < CB_ROWS * CB_K / CB_THREADS; ++u) {
          const int i = tid + u * CB_THREADS, r = i / CB_K, k = i % CB_K;
          xpre[u] = (rows[r] >= 0 && k0 + k < F) ? load_col(a.pro, a.x + (int64_t)rows[r] * a.ldx, k0 + k) : 0.0f;
        }
      };
      auto store_x = [&](int buf) {
        double* xb = xc + buf * CB_ROWS * CB_KS;
#pragma unroll
        for (int u = 0; u < CB_ROWS * CB_K / CB_THREADS; ++u) {
          const int i = tid + u * CB_THREADS, r = i / CB_K, k = i % CB_K;
          xb[r * CB_KS + k] = (double)xpre[u];
        }
      };
      auto stage_s = [&](int kc, int buf) {
        const int k0 = kc * CB_K;
        double* sb = sc + buf * CB_SV * CB_KS;
        for (int i = tid; i < CB_SV * CB_K / 2; i += CB_THREADS) {  // 16-byte pieces
          const int jj = i / (CB_K / 2), kp = i % (CB_K / 2);
          if (F & 1) {  // odd F: rows are not 16-byte aligned, plain loads
            for (int h = 0; h < 2; ++h) {
              const int k = k0 + 2 * kp + h;
              sb[jj * CB_KS + 2 * kp + h] = (jj < nj && k < F) ? __ldg(a.sv + (size_t)(j0 + jj) * F + k) : 0.0;
            }
            continue;
          }
          // bytes present: 16 or 0 (F even: pieces never straddle the row end)
          const int nbytes = (jj < nj && k0 + 2 * kp < F) ? 16 : 0;
          const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sb + jj * CB_KS + 2 * kp);
          const double* src = nbytes ? a.sv + (size_t)(j0 + jj) * F + k0 + 2 * kp : a.sv;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(nbytes) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      };
      load_x(0);
      store_x(0);
      stage_s(0, 0);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      for (int kc = 0; kc < nkc; ++kc) {
        const bool more = kc + 1 < nkc;
        if (more) {
          load_x(kc + 1);
          stage_s(kc + 1, (kc + 1) & 1);
        }
        const double* xb = xc + (kc & 1) * CB_ROWS * CB_KS;
        const double* sb = sc + (kc & 1) * CB_SV * CB_KS;
#pragma unroll
        for (int k = 0; k < CB_K; k += 4) {
          double af[4], bf[2];
#pragma unroll
          for (int i = 0; i < 4; ++i) af[i] = xb[(rw0 + 8 * i + gq) * CB_KS + k + tq];
#pragma unroll
          for (int j = 0; j < 2; ++j) bf[j] = sb[(sw0 + 8 * j + gq) * CB_KS + k + tq];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                           : "+d"(g[i][j][0]), "+d"(g[i][j][1]) : "d"(af[i]), "d"(bf[j]));
        }
        if (more) store_x((kc + 1) & 1);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
      }
      // kernel values of this tile and their error bounds against libsvm's
#pragma unroll
      for (int e = 0; e < 16; ++e) {
          const int i = e >> 2, j = (e >> 1) & 1, h = e & 1;
          const int r = rw0 + 8 * i + gq, jj = sw0 + 8 * j + 2 * tq + h;
          double kv = 0.0, ek = 0.0;
          if (jj < nj) {
            const double G = g[i][j][h], nx = nxs[r], ns = __ldg(a.ns64 + j0 + jj);
            // G: ours and libsvm's float64 dot products each within gamma_{F+3} sum|x s| <= gamma (nx + ns) / 2
            const double eg = gF * (nx + ns);
            if (a.kernel == CMLB_SVM_RBF) {
              // d2 = nx + ns - 2G here, sum (x - s)^2 in libsvm: both within (2 gF + 6u)(nx + ns) of exact
              const double d2 = fmax(nx + ns - 2.0 * G, 0.0);
              kv = exp(-a.gamma64 * d2);
              const double gd = fabs(a.gamma64) * (4.0 * gF + 12.0 * U) * (nx + ns);
              // + the roundings of exp (<= 1 ulp each side) and of its argument gamma * d2
              ek = kv * (gd * (1.0 + 2.0 * gd) + 8.0 * U + 4.0 * U * fabs(a.gamma64) * d2) + 1e-300;
            } else if (a.kernel == CMLB_SVM_LINEAR) {
              kv = G;
              ek = 2.0 * eg + 4.0 * U * fabs(G);
            } else {
              const double u = a.gamma64 * G + a.coef064;
              const double eu = fabs(a.gamma64) * 2.0 * eg + 4.0 * U * (fabs(a.gamma64 * G) + fabs(a.coef064));
              if (a.kernel == CMLB_SVM_SIGMOID) {
                kv = tanh(u);
                ek = 2.0 * eu + 8.0 * U;
              } else {
                double t = u, ret = 1.0;
                for (int e = a.degree; e > 0; e /= 2) {
                  if (e % 2 == 1) ret *= t;
                  t *= t;
                }
                kv = ret;
                double m = 1.0;  // (|u| + eu)^(deg - 1)
                for (int e = 1; e < a.degree; ++e) m *= fabs(u) + eu;
                ek = 2.0 * a.degree * m * eu * (1.0 + eu) + 8.0 * a.degree * U * fabs(kv) + 1e-300;
              }
            }
          }
          ks[r * CB_SS + jj] = kv;
          eks[r * CB_SS + jj] = ek;
      }
      __syncthreads();
      // decision sums per (row, pair) task, ascending SV order (libsvm's)
#pragma unroll
      for (int q = 0; q < CB_TPT; ++q) {
        const int task = tid + q * CB_THREADS;
        if (task >= ntasks) break;
        const int r = task % CB_ROWS, p = PAIR ? bp : task / CB_ROWS;
        auto add = [&](const float* coefrow, int lo, int hi) {
          for (int j = max(lo, j0); j < min(hi, j0 + nj); ++j) {
            const double w = (double)__ldg(coefrow + j);
            const double kv = ks[r * CB_SS + (j - j0)];
            dsum[q] = __dadd_rn(dsum[q], __dmul_rn(w, kv));
            asum[q] = __fadd_ru(asum[q], __double2float_ru(fabs(w * kv)));
            esum[q] += fabs(w) * eks[r * CB_SS + (j - j0)];
          }
        };
        if (a.is_svr) {
          add(a.coef, 0, a.n_sv);
        } else {
          int ca = 0, rem = p;
          while (rem >= C - 1 - ca) { rem -= C - 1 - ca; ++ca; }
          const int cb = ca + 1 + rem;
          add(a.coef + (size_t)(cb - 1) * a.n_sv, n_sv_start[ca], n_sv_start[ca + 1]);
          add(a.coef + (size_t)ca * a.n_sv, n_sv_start[cb], n_sv_start[cb + 1]);
        }
      }
      __syncthreads();  // ks / eks reused by the next tile
    }
    if constexpr (PAIR) {  // partial sums of this unit's SVs -> the sorted entry's accumulators
      if (tid < nb) {
        const size_t i = (size_t)pfirst + tid, np = (size_t)a.pq_cap;
        atomicAdd(a.pacc + i, dsum[0]);
        atomicAdd(a.pacc + np + i, esum[0]);
        atomicAdd(a.pacc + 2 * np + i, (double)asum[0]);
        if (undecided[tid]) a.pflag[i] = 1;
      }
      __syncthreads();
      continue;
    }
    if (split) {  // partial sums of this unit's SVs -> the block's accumulators
      const size_t nacc = (size_t)a.cap_blocks * CB_ROWS * npairs;
#pragma unroll
      for (int q = 0; q < CB_TPT; ++q) {
        const int task = tid + q * CB_THREADS;
        if (task >= ntasks) break;
        const int r = task % CB_ROWS, p = task / CB_ROWS;
        if (r >= nb) continue;
        const size_t i = ((size_t)rb * CB_ROWS + r) * npairs + p;
        atomicAdd(a.cacc + i, dsum[q]);
        atomicAdd(a.cacc + nacc + i, esum[q]);
        atomicAdd(a.cacc + 2 * nacc + i, (double)asum[q]);
      }
      if (tid < nb && undecided[tid]) a.cflag[rb * CB_ROWS + tid] = 1;
      __syncthreads();
      continue;
    }
    // certify: a row is decided when every pair clears its bound
    double* decs = xc;  // [CB_ROWS][npairs <= 48]: 24.6 KB over the free staging buffers (xc + sc, 34.8 KB)
#pragma unroll
    for (int q = 0; q < CB_TPT; ++q) {
      const int task = tid + q * CB_THREADS;
      if (task >= ntasks) break;
      const int r = task % CB_ROWS, p = task / CB_ROWS;
      const double rho = (double)a.intercept[p];
      const double dec = __dsub_rn(dsum[q], -rho);
      const double tol2 = esum[q] + 2.0 * gamma_n(a.n_sv + 2) * (asum[q] + fabs(rho)) + 1e-300;
      if (a.is_svr) {
        if (!f32_round_certain(dec, tol2)) atomicOr(&undecided[r], 1);
      } else if (!(fabs(dec) > tol2)) {
        atomicOr(&uncm[r], 1ull << p);
      }
      decs[r * npairs + p] = dec;
    }
    __syncthreads();
    if (tid < nb) {
      const int64_t row = rows[tid];
      const double* d = decs + tid * npairs;
      int best = -1;
      bool exact = undecided[tid] != 0;
      if (!exact && !a.is_svr && uncm[tid]) {
        // uncertain pairs matter only if they could change the class
        exact = a.dec_out != nullptr;
        if (!exact) {
          int vmin[MAXC], unc[MAXC];
          for (int c = 0; c < C; ++c) vmin[c] = unc[c] = 0;
          int p = 0;
          for (int i = 0; i < C; ++i)
            for (int j = i + 1; j < C; ++j, ++p) {
              if (!isfinite(d[p])) exact = true;
              if ((uncm[tid] >> p) & 1ull) { ++unc[i]; ++unc[j]; }
              else if (d[p] > 0) ++vmin[i];
              else ++vmin[j];
            }
          if (!exact) best = robust_vote(vmin, unc, C);
          exact = best < 0;
        }
      }
      if (exact) {
        a.queue2[atomicAdd(a.queue2_len, 1)] = (int32_t)row;
      } else if (best >= 0) {
        store_out(a.y, row, a.out_dt, a.classes[best]);
      } else if (a.is_svr) {
        store_out(a.y, row, a.out_dt, (double)(float)d[0]);
        if (a.dec_out) a.dec_out[row] = d[0];
      } else {
        int vote[MAXC];
        for (int c = 0; c < C; ++c) vote[c] = 0;
        int p = 0;
        for (int i = 0; i < C; ++i)
          for (int j = i + 1; j < C; ++j, ++p) {
            if (d[p] > 0) ++vote[i]; else ++vote[j];
          }
        int best = 0;
        for (int c = 1; c < C; ++c)
          if (vote[c] > vote[best]) best = c;
        store_out(a.y, row, a.out_dt, a.classes[best]);
        if (a.dec_out)
          for (int q = 0; q < npairs; ++q) a.dec_out[row * npairs + q] = d[q];
      }
    }
    __syncthreads();
  }
}

// Decisions of the SV-split row blocks of the full certifying tier (see
// Args::cacc): the same certificate as the in-CTA finalize, with the summation
// bound widened for the split (partial sums per unit, then <= n_sv / CB_SPAN
// float64 atomic additions in any order: gamma_{n_sv + 64}).
__global__ void __launch_bounds__(128) svm_certify_finish_kernel(const Args a) {
  const int nq = *a.queue_len;
  const int n = min(nq, a.cap_blocks * CB_ROWS);
  const int npairs = a.is_svr ? 1 : a.pairs;
  const int C = a.C;
  const size_t nacc = (size_t)a.cap_blocks * CB_ROWS * npairs;
  const double gs = 2.0 * gamma_n(a.n_sv + 64);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int64_t row = a.queue[i];
    bool exact = a.cflag[i] != 0;
    double d[CB_MAXP];
    unsigned long long uncm = 0ull;
    for (int p = 0; p < npairs; ++p) {
      const size_t k = (size_t)i * npairs + p;
      const double rho = (double)a.intercept[p];
      const double dec = __dsub_rn(a.cacc[k], -rho);
      const double tol2 = a.cacc[nacc + k] * (1.0 + 1e-9) + gs * (a.cacc[2 * nacc + k] * (1.0 + 1e-12) + fabs(rho)) +
                          1e-300;
      d[p] = dec;
      if (a.is_svr) {
        if (!f32_round_certain(dec, tol2)) exact = true;
      } else if (!(fabs(dec) > tol2)) {
        uncm |= 1ull << p;
      }
    }
    int best = -1;
    if (!exact && !a.is_svr && uncm) {
      exact = a.dec_out != nullptr;
      if (!exact) {
        int vmin[MAXC], unc[MAXC];
        for (int c = 0; c < C; ++c) vmin[c] = unc[c] = 0;
        int p = 0;
        for (int ci = 0; ci < C; ++ci)
          for (int cj = ci + 1; cj < C; ++cj, ++p) {
            if (!isfinite(d[p])) exact = true;
            if ((uncm >> p) & 1ull) { ++unc[ci]; ++unc[cj]; }
            else if (d[p] > 0) ++vmin[ci];
            else ++vmin[cj];
          }
        if (!exact) best = robust_vote(vmin, unc, C);
        exact = best < 0;
      }
    }
    if (exact) {
      a.queue2[atomicAdd(a.queue2_len, 1)] = (int32_t)row;
    } else if (best >= 0) {
      store_out(a.y, row, a.out_dt, a.classes[best]);
    } else if (a.is_svr) {
      store_out(a.y, row, a.out_dt, (double)(float)d[0]);
      if (a.dec_out) a.dec_out[row] = d[0];
    } else {
      int vote[MAXC];
      for (int c = 0; c < C; ++c) vote[c] = 0;
      int p = 0;
      for (int ci = 0; ci < C; ++ci)
        for (int cj = ci + 1; cj < C; ++cj, ++p) {
          if (d[p] > 0) ++vote[ci]; else ++vote[cj];
        }
      int bc = 0;
      for (int c = 1; c < C; ++c)
        if (vote[c] > vote[bc]) bc = c;
      store_out(a.y, row, a.out_dt, a.classes[bc]);
      if (a.dec_out)
        for (int q = 0; q < npairs; ++q) a.dec_out[row * npairs + q] = d[q];
    }
  }
}

// Pair tier decisions: the entry's pair resolved from the summed units, the
// other pairs' signs from the fast path; rows still open go to the full tier.
__global__ void __launch_bounds__(128) svm_pair_finish_kernel(const Args a, const int* n_sv_start) {
  __shared__ int off[65];
  const int C = a.C;
  if (threadIdx.x == 0) {
    int e = 0;
    for (int q = 0; q < a.pairs; ++q) {
      off[q] = e;
      e += a.pcount[q];
    }
    off[a.pairs] = e;
  }
  __syncthreads();
  const int n = min(*a.pq_len, a.pq_cap);
  const size_t np = (size_t)a.pq_cap;
  const double gs = 2.0 * gamma_n(a.n_sv + 64);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int bp = 0;
    while (i >= off[bp + 1]) ++bp;
    const int64_t row = a.ps_row[i];
    const double rho = (double)a.intercept[bp];
    const double dec = __dsub_rn(a.pacc[i], -rho);
    const double tol2 = a.pacc[np + i] * (1.0 + 1e-9) + gs * (a.pacc[2 * np + i] * (1.0 + 1e-12) + fabs(rho)) + 1e-300;
    if (a.pflag[i] || !(fabs(dec) > tol2)) {
      a.queue2[atomicAdd(a.queue2_len, 1)] = (int32_t)row;
      continue;
    }
    unsigned long long sg = a.ps_sign[i] & ~(1ull << bp);
    if (dec > 0) sg |= 1ull << bp;
    const unsigned long long un = a.ps_unc[i] & ~(1ull << bp);
    int vote[MAXC], unc[MAXC];
    for (int c = 0; c < C; ++c) vote[c] = unc[c] = 0;
    int q = 0;
    for (int ci = 0; ci < C; ++ci)
      for (int cj = ci + 1; cj < C; ++cj, ++q) {
        if ((un >> q) & 1ull) { ++unc[ci]; ++unc[cj]; }
        else if ((sg >> q) & 1ull) ++vote[ci];
        else ++vote[cj];
      }
    const int best = robust_vote(vote, unc, C);
    if (best >= 0) store_out(a.y, row, a.out_dt, a.classes[best]);
    else a.queue[atomicAdd(a.queue_len, 1)] = (int32_t)row;  // the full certifying tier decides
  }
}

// Pair tier: bucket the fast path's one-uncertain-pair rows by that pair
// (counting sort: per-pair offsets from the counts, cursors by atomics; the
// order inside a bucket does not matter -- every row is decided on its own).
__global__ void __launch_bounds__(256) svm_pair_scatter_kernel(const Args a) {
  __shared__ int off[64];
  if (threadIdx.x == 0) {
    int e = 0;
    for (int q = 0; q < a.pairs; ++q) {
      off[q] = e;
      e += a.pcount[q];
    }
  }
  __syncthreads();
  const int n = min(*a.pq_len, a.pq_cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int q = a.pq_pair[i];
    const int dst = off[q] + atomicAdd(a.pcur + q, 1);
    a.ps_row[dst] = a.pq_row[i];
    a.ps_sign[dst] = a.pq_sign[i];
    a.ps_unc[dst] = a.pq_unc[i];
  }
}

__global__ void __launch_bounds__(XTHREADS) svm_exact_kernel(const Args a, const int* n_sv_start) {
  extern __shared__ __align__(16) uint8_t xsm[];
  const int xstr = a.F + 2;                                           // padded row stride (doubles)
  double* xs = reinterpret_cast<double*>(xsm);                       // [XR][xstr] row-major
  double* kv = xs + (size_t)xstr * XR;                                // [XCH][XR]
  double* decs = kv + XCH * XR;                                      // [XR][pairs]
  __shared__ int32_t rows[XR];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nq = *a.queue_len;
  const int npairs = a.is_svr ? 1 : a.pairs;
  const int ntasks = XR * npairs;
  const int TPT = (ntasks + XTHREADS - 1) / XTHREADS;  // (row, pair) tasks per thread, <= 4
  for (int b0 = blockIdx.x * XR; b0 < nq; b0 += gridDim.x * XR) {
    const int nb = min(XR, nq - b0);
    if (tid < XR) rows[tid] = tid < nb ? a.queue[b0 + tid] : -1;
    __syncthreads();
    for (int i = tid; i < a.F * XR; i += XTHREADS) {
      const int r = i / a.F, k = i - r * a.F;
      xs[(size_t)r * xstr + k] = rows[r] >= 0 ? (double)load_col(a.pro, a.x + (int64_t)rows[r] * a.ldx, k) : 0.0;
    }
    double sum[4];
    for (int q = 0; q < 4; ++q) sum[q] = 0.0;
    __syncthreads();
    for (int j0 = 0; j0 < a.n_sv; j0 += XCH) {
      const int nj = min(XCH, a.n_sv - j0);
      // K values of this chunk: each warp takes 32 / XR SVs at a time;
      // lane % XR = row
      constexpr int SPW = 32 / XR;
      for (int jj = SPW * warp + lane / XR; jj < nj; jj += SPW * (XTHREADS / 32))
        kv[jj * XR + (lane % XR)] = exact_k(a, xs + (size_t)(lane % XR) * xstr, a.sv + (size_t)(j0 + jj) * a.F);
      __syncthreads();
      // sequential decision sums in libsvm order, one (row, pair) per slot
      for (int q = 0; q < TPT; ++q) {
        const int task = tid + q * XTHREADS;
        if (task >= ntasks) break;
        const int r = task % XR, p = task / XR;
        double s = sum[q];
        if (a.is_svr) {
          for (int jj = 0; jj < nj; ++jj)
            s = __dadd_rn(s, __dmul_rn((double)__ldg(a.coef + j0 + jj), kv[jj * XR + r]));
        } else {
          // pair p -> (ca, cb)
          int ca = 0, rem = p;
          while (rem >= a.C - 1 - ca) { rem -= a.C - 1 - ca; ++ca; }
          const int cb = ca + 1 + rem;
          const int lo_a = n_sv_start[ca], hi_a = n_sv_start[ca + 1];
          const int lo_b = n_sv_start[cb], hi_b = n_sv_start[cb + 1];
          const float* c1 = a.coef + (size_t)(cb - 1) * a.n_sv;
          const float* c2 = a.coef + (size_t)ca * a.n_sv;
#pragma unroll 8
          for (int j = max(lo_a, j0); j < min(hi_a, j0 + nj); ++j)
            s = __dadd_rn(s, __dmul_rn((double)__ldg(c1 + j), kv[(j - j0) * XR + r]));
#pragma unroll 8
          for (int j = max(lo_b, j0); j < min(hi_b, j0 + nj); ++j)
            s = __dadd_rn(s, __dmul_rn((double)__ldg(c2 + j), kv[(j - j0) * XR + r]));
        }
        sum[q] = s;
      }
      __syncthreads();
    }
    for (int q = 0; q < TPT; ++q) {
      const int task = tid + q * XTHREADS;
      if (task < ntasks) {
        const int r = task % XR, p = task / XR;
        decs[r * npairs + p] = __dsub_rn(sum[q], -(double)a.intercept[p]);
      }
    }
    __syncthreads();
    if (tid < nb) {
      const int64_t row = rows[tid];
      const double* d = decs + tid * npairs;
      if (a.is_svr) {
        store_out(a.y, row, a.out_dt, (double)(float)d[0]);
        if (a.dec_out) a.dec_out[row] = d[0];
      } else {
        int vote[MAXC];
        for (int c = 0; c < a.C; ++c) vote[c] = 0;
        int p = 0;
        for (int i = 0; i < a.C; ++i)
          for (int j = i + 1; j < a.C; ++j, ++p) {
            if (d[p] > 0) ++vote[i]; else ++vote[j];
          }
        int best = 0;
        for (int c = 1; c < a.C; ++c)
          if (vote[c] > vote[best]) best = c;
        store_out(a.y, row, a.out_dt, a.classes[best]);
        if (a.dec_out)
          for (int q = 0; q < npairs; ++q) a.dec_out[row * npairs + q] = d[q];
      }
    }
    __syncthreads();
  }
}

}  // namespace svm

// ---------------------------------------------------------------------------
// host program
// ---------------------------------------------------------------------------

struct cmlb_svm_impl {
  int device;
  int n_inputs;
  svm::Args a;
  int CP;
  std::vector<void*> bufs;
  int32_t* sv_start;   // device [C + 1]
  size_t tc_smem, x_smem;
};

}  // namespace cmlb

struct cmlb_svm : cmlb::cmlb_svm_impl {};

namespace cmlb {

template <typename T>
static int upload(cmlb_svm* m, const std::vector<T>& h, const T** out) {
  void* d = nullptr;
  const size_t bytes = std::max<size_t>(h.size() * sizeof(T), 16);
  CMLB_CUDA(cudaMalloc(&d, bytes));
  m->bufs.push_back(d);
  if (!h.empty()) CMLB_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  *out = static_cast<const T*>(d);
  return CMLB_OK;
}

static void destroy_svm(cmlb_svm* m) {
  if (!m) return;
  DeviceGuard g(m->device);
  for (void* p : m->bufs) cudaFree(p);
  delete m;
}

static int make_svm(const cmlb_svm_desc* d, int device, cmlb_svm** out) {
  using namespace svm;
  if (!d || !out) return fail(CMLB_E_VALIDATION, "null svm descriptor");
  const int F = d->n_features, NSV = d->n_sv;
  if (F <= 0 || NSV <= 0) return fail(CMLB_E_VALIDATION, "svm needs n_features > 0 and n_sv > 0");
  if (d->kernel < CMLB_SVM_LINEAR || d->kernel > CMLB_SVM_SIGMOID) return fail(CMLB_E_VALIDATION, "unknown svm kernel");
  const bool svr = d->n_classes == 0;
  const int C = svr ? 1 : d->n_classes;
  if (!svr && (C < 2 || C > MAXC)) return fail(CMLB_E_UNRESOLVED, "svc supports 2..16 classes");
  if (!svr && !d->n_support) return fail(CMLB_E_VALIDATION, "svc needs n_support");
  if (!out_dtype_ok(d->out_dtype)) return fail(CMLB_E_VALIDATION, "bad out_dtype");
  const int pairs = svr ? 1 : C * (C - 1) / 2;
  // accumulators per row: the smallest instantiated width >= C
  const int CP = C <= 2 ? 2 : C <= 3 ? 3 : C <= 4 ? 4 : C <= 6 ? 6 : C <= 8 ? 8 : C <= 10 ? 10 : C <= 12 ? 12 : 16;
  const int CPS = (CP + 3) & ~3;
  const int KB = (F + BK - 1) / BK, NT = (NSV + BN - 1) / BN, NP = NT * BN;

  cmlb_svm* m = new (std::nothrow) cmlb_svm();
  if (!m) return fail(CMLB_E_DEVICE, "out of host memory");
  m->device = device;
  DeviceGuard g(device);
  int st = CMLB_OK;

  std::vector<int32_t> start(C + 1, 0);
  std::vector<int32_t> cls(NP, -1);
  if (svr) {
    start[1] = NSV;
  } else {
    for (int c = 0; c < C; ++c) start[c + 1] = start[c] + d->n_support[c];
    if (start[C] != NSV) {
      destroy_svm(m);
      return fail(CMLB_E_VALIDATION, "n_support does not sum to n_sv");
    }
  }
  for (int c = 0; c < C; ++c)
    for (int j = start[c]; j < start[c + 1]; ++j) cls[j] = c;
  // per-SV coefficient toward each other class (libsvm: SV of class c in
  // pair (c, o) uses coef[o-1] if c < o, else coef[o])
  std::vector<float> w((size_t)NP * CPS, 0.0f), wmax(NP, 0.0f), ns(NP, 0.0f), qerr(NP, 0.0f);
  std::vector<double> ns64(std::max(NSV, 1), 0.0);
  for (int j = 0; j < NSV; ++j) {
    const int c = cls[j];
    for (int o = 0; o < C; ++o) {
      float v;
      if (svr) v = d->dual_coef[j];
      else if (o == c) continue;
      else v = d->dual_coef[(size_t)(c < o ? o - 1 : o) * NSV + j];
      w[(size_t)j * CPS + o] = v;
      wmax[j] = std::max(wmax[j], std::fabs(v));
    }
    double s = 0.0;
    for (int k = 0; k < F; ++k) {
      const double v = d->support_vectors[(size_t)j * F + k];
      s += v * v;
    }
    ns[j] = (float)s;
    ns64[j] = s;
    qerr[j] = (float)((double)wmax[j] * d->gamma * 1.075e-6 * s * (1.0 + 1e-6));
  }
  // SV splits in the UMMA core-matrix layout: [tile][kb][big|small][c][row][4]
  std::vector<uint8_t> bsplit((size_t)NT * KB * 2 * B_BYTES, 0);
  for (int t = 0; t < NT; ++t)
    for (int kb = 0; kb < KB; ++kb) {
      uint8_t* base = bsplit.data() + ((size_t)t * KB + kb) * 2 * B_BYTES;
      for (int r = 0; r < BN; ++r) {
        const int j = t * BN + r;
        if (j >= NSV) continue;
        for (int e = 0; e < BK; ++e) {
          const int k = kb * BK + e;
          if (k >= F) continue;
          const float v = d->support_vectors[(size_t)j * F + k];
          uint32_t u;
          std::memcpy(&u, &v, 4);
          u &= 0xFFFFE000u;
          float hi;
          std::memcpy(&hi, &u, 4);
          const float lo = v - hi;
          const size_t off = (size_t)(e / 4) * (BN * 16) + (size_t)r * 16 + (size_t)(e % 4) * 4;
          std::memcpy(base + off, &hi, 4);
          std::memcpy(base + B_BYTES + off, &lo, 4);
        }
      }
    }
  std::vector<double> svv(d->support_vectors, d->support_vectors + (size_t)NSV * F);
  std::vector<float> coef(d->dual_coef, d->dual_coef + (size_t)(svr ? 1 : C - 1) * NSV);
  std::vector<float> ic(d->intercept, d->intercept + pairs);
  std::vector<double> classes(svr ? 1 : C, 0.0);
  if (!svr)
    for (int c = 0; c < C; ++c) classes[c] = d->classes[c];

  Args& a = m->a;
  std::memset(&a, 0, sizeof(a));
  const uint8_t* bs = nullptr;
  const int32_t* ss = nullptr;
  if ((st = upload(m, bsplit, &bs)) || (st = upload(m, ns, &a.ns)) || (st = upload(m, w, &a.w)) ||
      (st = upload(m, wmax, &a.wmax)) || (st = upload(m, qerr, &a.qerr)) || (st = upload(m, cls, &a.cls)) || (st = upload(m, svv, &a.sv)) ||
      (st = upload(m, coef, &a.coef)) || (st = upload(m, ic, &a.intercept)) ||
      (st = upload(m, classes, &a.classes)) || (st = upload(m, start, &ss)) || (st = upload(m, ns64, &a.ns64))) {
    destroy_svm(m);
    return st;
  }
  a.bsplit = bs;
  m->sv_start = const_cast<int32_t*>(ss);
  a.F = F; a.KB = KB; a.n_tiles = NT; a.n_sv = NSV;
  a.C = C; a.CP = CP; a.pairs = pairs; a.kernel = d->kernel; a.degree = d->degree; a.is_svr = svr;
  a.out_dt = d->out_dtype;
  a.gamma = (float)d->gamma; a.coef0 = (float)d->coef0; a.gamma64 = d->gamma; a.coef064 = d->coef0;
  m->CP = CP;
  m->n_inputs = F;
  if (d->prologue) {
    if (d->n_inputs <= 0) {
      destroy_svm(m);
      return fail(CMLB_E_VALIDATION, "prologue needs n_inputs > 0");
    }
    std::vector<cmlb_column_op> pro(d->prologue, d->prologue + F);
    for (const auto& o : pro)
      if (o.src < 0 || o.src >= d->n_inputs || o.op < CMLB_COL_COPY || o.op > CMLB_COL_EQUAL) {
        destroy_svm(m);
        return fail(CMLB_E_VALIDATION, "bad prologue column op");
      }
    if ((st = upload(m, pro, &a.pro))) {
      destroy_svm(m);
      return st;
    }
    m->n_inputs = d->n_inputs;
  }
  m->tc_smem = (size_t)STAGES * STAGE_BYTES + (size_t)BN * CPS * 4 + BN * 4 * 4;
  m->x_smem = (size_t)(F + 2) * XR * 8 + (size_t)XCH * XR * 8 + (size_t)XR * pairs * 8;
  if (m->x_smem > 227 * 1024) {
    destroy_svm(m);
    return fail(CMLB_E_UNRESOLVED, "svm exact path: features x classes exceed shared memory");
  }
  *out = m;
  return CMLB_OK;
}

template <int CP>
static int launch_tc(const svm::Args& a, int64_t n, size_t smem, cudaStream_t s) {
  auto fn = svm::svm_tc_kernel<CP>;
  CMLB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fn<<<(unsigned)ceil_div(n, svm::BM), svm::THREADS, smem, s>>>(a);
  CMLB_CUDA(cudaGetLastError());
  note_launch();
  return CMLB_OK;
}

static int launch_any(int CP, const svm::Args& a, int64_t n, size_t smem, cudaStream_t s) {
  switch (CP) {
    case 2: return launch_tc<2>(a, n, smem, s);
    case 3: return launch_tc<3>(a, n, smem, s);
    case 4: return launch_tc<4>(a, n, smem, s);
    case 6: return launch_tc<6>(a, n, smem, s);
    case 8: return launch_tc<8>(a, n, smem, s);
    case 10: return launch_tc<10>(a, n, smem, s);
    case 12: return launch_tc<12>(a, n, smem, s);
    default: return launch_tc<16>(a, n, smem, s);
  }
}

}  // namespace cmlb

extern "C" {

int cmlb_svm_create(const cmlb_svm_desc* desc, int device, cmlb_svm** out) {
  try {
    return cmlb::make_svm(desc, device, out);
  } catch (const std::exception& e) {
    return cmlb::fail(CMLB_E_DEVICE, e.what());
  }
}

int cmlb_svm_run(const cmlb_svm* m, const float* x, int64_t n_rows, int64_t ldx, void* y, double* decision,
                 int32_t* exact_rows, void* stream) {
  using namespace cmlb;
  if (!m) return fail(CMLB_E_VALIDATION, "null svm");
  if (n_rows < 0 || ldx < m->n_inputs) return fail(CMLB_E_INPUT, "bad svm input shape");
  if (n_rows > INT32_MAX) return fail(CMLB_E_INPUT, "svm batch exceeds 2^31 rows");
  if (n_rows == 0) return CMLB_OK;
  DeviceGuard g(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  svm::Args a = m->a;
  a.x = x; a.n_rows = n_rows; a.ldx = ldx; a.y = y; a.dec_out = decision;
  a.vec_x = ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (ldx & 3) == 0) ? 1 : 0;
  static const int prob_tol = [] {
    const char* e = std::getenv("CMLB_SVM_TOL");
    return e && std::string(e) == "hoeffding" ? 1 : 0;
  }();
  a.prob_tol = prob_tol;
  keep_pool(m->device);
  // scratch: counters (queue lengths, 64 pair counts, 64 pair cursors), the
  // two row queues, and the pair tier's entries (unsorted + bucketed)
  const bool certify = (a.is_svr ? 1 : a.pairs) <= svm::CB_MAXP && !a.no_exact;
  static const bool no_pair_tier = std::getenv("CMLB_SVM_NO_PAIR_TIER") != nullptr;  // measurement knob
  const bool pair_tier = certify && !a.is_svr && !decision && a.pairs <= 64 && !no_pair_tier;
  const size_t nhead = 256;  // int32 slots
  const int npairs_c = a.is_svr ? 1 : a.pairs;
  const int cap_blocks = certify ? (int)std::min<int64_t>(svm::CB_CAP_BLOCKS, ceil_div(n_rows, svm::CB_ROWS)) : 0;
  const size_t nacc = (size_t)cap_blocks * svm::CB_ROWS * npairs_c;
  const size_t acc_bytes = nacc * 3 * sizeof(double) + (size_t)cap_blocks * svm::CB_ROWS * sizeof(int32_t);
  // pair tier: [pacc 3 x n doubles][pflag n int32] zeroed with the head
  // pair-tier capacity: 1/8 of the batch (>= 64K rows); config 4b queues 0.15%
  const int64_t pq_cap = pair_tier ? std::min<int64_t>(n_rows, std::max<int64_t>(65536, n_rows / 8)) : 0;
  const size_t pacc_bytes = pair_tier ? (size_t)pq_cap * 3 * sizeof(double) + ((size_t)pq_cap * 4 + 7) / 8 * 8 : 0;
  const size_t zero_bytes = acc_bytes + pacc_bytes;
  const size_t bytes = zero_bytes + (nhead + 2 * (size_t)n_rows) * sizeof(int32_t) +
                       (pair_tier ? (size_t)pq_cap * (3 * sizeof(int32_t) + 4 * sizeof(unsigned long long)) : 0);
  void* scratch = nullptr;
  CMLB_CUDA(cudaMallocAsync(&scratch, bytes, s));
  // [cacc doubles][cflag int32][head int32 ...]
  a.cacc = cap_blocks ? static_cast<double*>(scratch) : nullptr;
  a.cflag = reinterpret_cast<int32_t*>(static_cast<double*>(scratch) + nacc * 3);
  a.cap_blocks = cap_blocks;
  a.pacc = reinterpret_cast<double*>(static_cast<uint8_t*>(scratch) + acc_bytes);  // 8-aligned: acc_bytes % 8 == 0
  a.pflag = reinterpret_cast<int32_t*>(a.pacc + 3 * (size_t)pq_cap);
  a.pq_cap = (int)pq_cap;
  int32_t* head = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(scratch) + zero_bytes);
  a.queue_len = head;
  a.queue2_len = head + 1;
  a.pq_len = head + 2;
  a.pcount = head + 64;
  a.pcur = head + 128;
  a.queue = head + nhead;
  a.queue2 = a.queue + n_rows;
  if (pair_tier) {
    unsigned long long* sg = reinterpret_cast<unsigned long long*>(a.queue2 + n_rows);  // 8-aligned: nhead + 2n int32
    a.pq_sign = sg;
    a.ps_sign = sg + pq_cap;
    a.pq_unc = sg + 2 * pq_cap;
    a.ps_unc = sg + 3 * pq_cap;
    a.pq_row = reinterpret_cast<int32_t*>(sg + 4 * pq_cap);
    a.pq_pair = a.pq_row + pq_cap;
    a.ps_row = a.pq_pair + pq_cap;
  } else {
    a.pq_row = nullptr;
  }
  int st = CMLB_OK;
  if (cudaMemsetAsync(scratch, 0, zero_bytes + nhead * sizeof(int32_t), s) != cudaSuccess) st = fail(CMLB_E_DEVICE, "memset");
  if (!st) {
    st = launch_any(m->CP, a, n_rows, m->tc_smem, s);
  }
  if (!st) {
    cudaError_t e = cudaFuncSetAttribute(svm::svm_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)m->x_smem);
    if (e != cudaSuccess) st = cuda_fail(e, "svm_exact smem");
  }
  // certifying tier (float64 Gram, rigorous bound against libsvm) for the
  // queued rows; what it cannot decide goes on to the libsvm-order exact path
  svm::Args ax = a;
  if (!st && certify) {
    const int grid = std::max(1, std::min<int>(2 * num_sms(m->device), (int)ceil_div(n_rows, svm::CB_ROWS)));
    if (pair_tier) {
      svm::svm_pair_scatter_kernel<<<std::max(1, std::min<int>(2 * num_sms(m->device), (int)ceil_div(n_rows, 256))),
                                     256, 0, s>>>(a);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) st = cuda_fail(e, "svm_pair_scatter_kernel");
      else note_launch();
      if (!st) e = cudaFuncSetAttribute(svm::svm_certify_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)svm::CB_SMEM);
      if (!st && e != cudaSuccess) st = cuda_fail(e, "svm_certify smem");
      if (!st) {
        svm::svm_certify_kernel<true><<<8 * num_sms(m->device), svm::CB_THREADS, svm::CB_SMEM, s>>>(a, m->sv_start);
        e = cudaGetLastError();
        if (e != cudaSuccess) st = cuda_fail(e, "svm_certify_kernel<pair>");
        else note_launch();
      }
      if (!st) {
        svm::svm_pair_finish_kernel<<<std::max(1, std::min<int>(num_sms(m->device), (int)ceil_div(n_rows, 128))), 128, 0,
                                      s>>>(a, m->sv_start);
        e = cudaGetLastError();
        if (e != cudaSuccess) st = cuda_fail(e, "svm_pair_finish_kernel");
        else note_launch();
      }
    }
    cudaError_t e = cudaFuncSetAttribute(svm::svm_certify_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)svm::CB_SMEM);
    if (!st && e != cudaSuccess) st = cuda_fail(e, "svm_certify smem");
    if (!st) {
      // split units: up to cap_blocks x ceil(n_sv / CB_SPAN) CTAs of work
      const int ugrid = std::max(grid, (int)std::min<int64_t>(8 * num_sms(m->device),
                                                               (int64_t)cap_blocks * ceil_div(a.n_sv, svm::CB_SPAN)));
      svm::svm_certify_kernel<false><<<ugrid, svm::CB_THREADS, svm::CB_SMEM, s>>>(a, m->sv_start);
      e = cudaGetLastError();
      if (e != cudaSuccess) st = cuda_fail(e, "svm_certify_kernel");
      else note_launch();
    }
    if (!st && cap_blocks) {
      svm::svm_certify_finish_kernel<<<std::max(1, std::min<int>(num_sms(m->device), (int)ceil_div((int64_t)cap_blocks * svm::CB_ROWS, 128))),
                                       128, 0, s>>>(a);
      e = cudaGetLastError();
      if (e != cudaSuccess) st = cuda_fail(e, "svm_certify_finish_kernel");
      else note_launch();
    }
    ax.queue = a.queue2;
    ax.queue_len = a.queue2_len;
  }
  if (!st) {
    const int grid = std::max(1, std::min<int>(3 * num_sms(m->device), (int)ceil_div(n_rows, svm::XR)));
    svm::svm_exact_kernel<<<grid, svm::XTHREADS, m->x_smem, s>>>(ax, m->sv_start);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = cuda_fail(e, "svm_exact_kernel");
    else note_launch();
  }
  static const char* dump_unc = std::getenv("CMLB_SVM_DUMP_UNC");  // measurement knob: fast-path uncertain-pair masks
  if (!st && pair_tier && dump_unc) {
    int32_t nq = 0;
    cudaMemcpyAsync(&nq, a.pq_len, sizeof(nq), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    nq = std::min(nq, a.pq_cap);
    std::vector<unsigned long long> h((size_t)nq);
    if (nq) cudaMemcpy(h.data(), a.pq_unc, (size_t)nq * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    int32_t ql[3] = {0, 0, 0};
    cudaMemcpy(ql, a.queue_len, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "svm queues: rows %lld pair-tier %d full-certify %d exact %d\n", (long long)n_rows, ql[2], ql[0], ql[1]);
    if (FILE* fh = std::fopen(dump_unc, "wb")) {
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), fh);
      std::fclose(fh);
    }
  }
  if (!st && exact_rows) {
    cudaError_t e = cudaMemcpyAsync(exact_rows, ax.queue_len, sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) st = cuda_fail(e, "exact_rows");
  }
  cudaFreeAsync(scratch, s);
  return st;
}

void cmlb_svm_destroy(cmlb_svm* m) { cmlb::destroy_svm(m); }

/* Diagnostics (tests/tools only): fast path for every row, with the
 * epilogue's per-row error bound E written to err (device float32 [n]). */
int cmlb_svm_debug_fast(const cmlb_svm* m, const float* x, int64_t n_rows, int64_t ldx, void* y, double* decision,
                        float* err, void* stream) {
  using namespace cmlb;
  if (!m || n_rows <= 0) return fail(CMLB_E_VALIDATION, "debug_fast: bad arguments");
  DeviceGuard g(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  svm::Args a = m->a;
  a.x = x; a.n_rows = n_rows; a.ldx = ldx; a.y = y; a.dec_out = decision; a.err_out = err; a.no_exact = 1;
  if (const char* pe = std::getenv("CMLB_SVM_PROBE")) a.probe = std::atoi(pe);
  a.vec_x = ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (ldx & 3) == 0) ? 1 : 0;
  void* scratch = nullptr;
  CMLB_CUDA(cudaMallocAsync(&scratch, (size_t)(n_rows + 4) * sizeof(int32_t), s));
  a.queue_len = static_cast<int32_t*>(scratch);
  a.queue = a.queue_len + 4;
  CMLB_CUDA(cudaMemsetAsync(a.queue_len, 0, sizeof(int32_t), s));
  int st;
  st = launch_any(m->CP, a, n_rows, m->tc_smem, s);
  cudaFreeAsync(scratch, s);
  return st;
}

}  // extern "C"
