// Preprocessing operator representations (pkg/src/mlower/convert.py:255-284).
//
// float32 elementwise with the reference's exact rounding sequence:
//   Binarizer   greater -> cast f32          (x > t ? 1 : 0; NaN -> 0)
//   MinMax      mul(scale) -> add(min)       two roundings, never an FMA
//   Robust/Std  sub(center) -> div(scale)    IEEE division
//   MaxAbs      div(scale)
//   Normalizer  row_norm (float64, numpy pairwise over the row, zero -> 1.0,
//               rounded to float32; kernels.py:245-261) -> div
// __fmul_rn/__fadd_rn/__fsub_rn/__fdiv_rn pin the rounding regardless of
// compiler contraction flags.

#include <algorithm>
#include <cstdint>
#include <memory>

#include "common.cuh"

namespace cmlb {

struct ScalerArgs {
  const float* x;
  int64_t n_rows, ldx;
  float* y;
  const float* a;
  const float* b;
  float thr;
  int F, kind;
};

__device__ __forceinline__ float scale1(const ScalerArgs& s, float v, int f) {
  switch (s.kind) {
    case CMLB_SCALER_BINARIZER: return v > s.thr ? 1.0f : 0.0f;
    case CMLB_SCALER_MINMAX: return __fadd_rn(__fmul_rn(v, __ldg(s.a + f)), __ldg(s.b + f));
    case CMLB_SCALER_SUB_DIV: return __fdiv_rn(__fsub_rn(v, __ldg(s.a + f)), __ldg(s.b + f));
    default: return __fdiv_rn(v, __ldg(s.a + f));  // DIV
  }
}

// Contiguous (ldx == F, F % 4 == 0, 16-byte aligned) fast path: float4 streams.
__global__ void scaler_ew_vec_kernel(const ScalerArgs s) {
  const int64_t total4 = s.n_rows * s.F / 4;
  const float4* x4 = reinterpret_cast<const float4*>(s.x);
  float4* y4 = reinterpret_cast<float4*>(s.y);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)((i * 4) % s.F);
    const float4 v = __ldg(x4 + i);
    float4 o;
    o.x = scale1(s, v.x, f);
    o.y = scale1(s, v.y, f + 1);
    o.z = scale1(s, v.z, f + 2);
    o.w = scale1(s, v.w, f + 3);
    __stcs(y4 + i, o);
  }
}

__global__ void scaler_ew_kernel(const ScalerArgs s) {
  const int64_t total = s.n_rows * s.F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / s.F;
    const int f = (int)(i - r * s.F);
    const float v = __ldg(s.x + r * s.ldx + f);
    float o;
    switch (s.kind) {
      case CMLB_SCALER_BINARIZER: o = v > s.thr ? 1.0f : 0.0f; break;
      case CMLB_SCALER_MINMAX: o = __fadd_rn(__fmul_rn(v, __ldg(s.a + f)), __ldg(s.b + f)); break;
      case CMLB_SCALER_SUB_DIV: o = __fdiv_rn(__fsub_rn(v, __ldg(s.a + f)), __ldg(s.b + f)); break;
      default: o = __fdiv_rn(v, __ldg(s.a + f)); break;  // DIV
    }
    s.y[i] = o;
  }
}

// numpy pairwise_sum over one row (|x| for l1, x*x for l2), any length.
__device__ double row_pairwise(const float* row, int lo, int n, bool square) {
  auto term = [&](int i) -> double {
    const double v = (double)row[lo + i];
    return square ? v * v : fabs(v);
  };
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += term(i);
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = term(j);
    const int m = n - n % 8;
    for (int i = 8; i < m; i += 8)
      for (int j = 0; j < 8; ++j) r[j] += term(i + j);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (int i = m; i < n; ++i) res += term(i);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return row_pairwise(row, lo, n2, square) + row_pairwise(row, lo + n2, n - n2, square);
}

__global__ void scaler_norm_kernel(const ScalerArgs s) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < s.n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const float* row = s.x + r * s.ldx;
    double n;
    if (s.kind == CMLB_SCALER_NORMALIZER_MAX) {
      n = fabs((double)row[0]);
      bool nan = n != n;
      for (int f = 1; f < s.F; ++f) {
        const double v = fabs((double)row[f]);
        nan |= v != v;
        n = v > n ? v : n;
      }
      if (nan) n = __longlong_as_double(0x7ff8000000000000LL);  // np.max propagates NaN
    } else {
      n = 0.0 + row_pairwise(row, 0, s.F, s.kind == CMLB_SCALER_NORMALIZER_L2);
      if (s.kind == CMLB_SCALER_NORMALIZER_L2) n = sqrt(n);
    }
    if (n == 0.0) n = 1.0;
    const float nf = __double2float_rn(n);
    for (int f = 0; f < s.F; ++f) s.y[r * s.F + f] = __fdiv_rn(row[f], nf);
  }
}

}  // namespace cmlb

struct cmlb_scaler {
  int device = 0, kind = 0, F = 0;
  float thr = 0.f;
  float* a = nullptr;
  float* b = nullptr;
  ~cmlb_scaler() { cudaFree(a); cudaFree(b); }
};

extern "C" {

int cmlb_scaler_create(const cmlb_scaler_desc* d, int device, cmlb_scaler** out) {
  using namespace cmlb;
  if (!out || !d) return fail(CMLB_E_VALIDATION, "null scaler descriptor/handle");
  *out = nullptr;
  if (d->n_features < 1 || d->kind < CMLB_SCALER_BINARIZER || d->kind > CMLB_SCALER_DIV)
    return fail(CMLB_E_VALIDATION, "bad scaler descriptor");
  DeviceGuard guard(device);
  std::unique_ptr<cmlb_scaler> s(new cmlb_scaler());
  s->device = device; s->kind = d->kind; s->F = d->n_features; s->thr = d->threshold;
  const size_t bytes = (size_t)s->F * sizeof(float);
  const bool needs_a = d->kind >= CMLB_SCALER_MINMAX;
  const bool needs_b = d->kind == CMLB_SCALER_MINMAX || d->kind == CMLB_SCALER_SUB_DIV;
  if (needs_a) {
    if (!d->a) return fail(CMLB_E_VALIDATION, "scaler vector missing");
    CMLB_CUDA(cudaMalloc(&s->a, bytes));
    CMLB_CUDA(cudaMemcpy(s->a, d->a, bytes, cudaMemcpyHostToDevice));
  }
  if (needs_b) {
    if (!d->b) return fail(CMLB_E_VALIDATION, "scaler vector missing");
    CMLB_CUDA(cudaMalloc(&s->b, bytes));
    CMLB_CUDA(cudaMemcpy(s->b, d->b, bytes, cudaMemcpyHostToDevice));
  }
  *out = s.release();
  return CMLB_OK;
}

int cmlb_scaler_run(const cmlb_scaler* s, const float* x, int64_t n_rows, int64_t ldx, float* y,
                    void* stream) {
  using namespace cmlb;
  if (!s) return fail(CMLB_E_VALIDATION, "null scaler");
  if (n_rows < 0 || ldx < s->F) return fail(CMLB_E_INPUT, "bad input extents");
  if (n_rows == 0) return CMLB_OK;
  DeviceGuard guard(s->device);
  ScalerArgs a{};
  a.x = x; a.n_rows = n_rows; a.ldx = ldx; a.y = y; a.a = s->a; a.b = s->b; a.thr = s->thr;
  a.F = s->F; a.kind = s->kind;
  const int sms = num_sms(s->device);
  const bool norm = s->kind >= CMLB_SCALER_NORMALIZER_L1 && s->kind <= CMLB_SCALER_NORMALIZER_MAX;
  const int64_t work = norm ? n_rows : n_rows * s->F;
  const int64_t grid = std::min<int64_t>(ceil_div(work, 256), (int64_t)sms * 16);
  const bool vec = !norm && s->F % 4 == 0 && ldx == s->F && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(y) & 15) == 0;
  if (norm) scaler_norm_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
  else if (vec) scaler_ew_vec_kernel<<<(unsigned)std::min<int64_t>(ceil_div(work / 4, 256), (int64_t)sms * 16), 256, 0,
                                       (cudaStream_t)stream>>>(a);
  else scaler_ew_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
  note_launch();
  CMLB_CUDA(cudaGetLastError());
  return CMLB_OK;
}

void cmlb_scaler_destroy(cmlb_scaler* s) { delete s; }

}  // extern "C"
