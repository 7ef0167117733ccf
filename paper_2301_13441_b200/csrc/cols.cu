// Column transform: OneHotEncoder / ColumnTransformer / elementwise scalers as
// one gather-transform kernel, y[:, f] = op_f(x[:, src_f]) (cmlb.h
// cmlb_column_op), and OneHotEncoder(handle_unknown='error')'s membership
// check (scikit-learn _encoders.py _transform: a value outside categories_
// raises).  Not in the reference (exporter/export.py:245-246 rejects
// Pipeline / OneHotEncoder); the scaler ops keep the reference float32
// rounding (convert.py:255-284).
//
// Used standalone when a pipeline ends in a transformer or feeds a stage
// that cannot take a prologue; otherwise the same ops run fused inside the
// consumer's row load (forest / linear / SVM) and only the check runs here.

#include <algorithm>
#include <memory>
#include <vector>

#include "common.cuh"

namespace cmlb {

struct ColsArgs {
  const float* x;
  int64_t n_rows, ldx;
  float* y;
  const cmlb_column_op* ops;
  int n_out;
  // membership checks
  int n_checks;
  const int32_t* check_col;
  const int64_t* check_off;
  const float* check_val;
  unsigned long long* bad;  // atomicMin target (row index), sentinel = ~0
};

// One thread per 4 consecutive outputs of a row (y row-major): coalesced
// float4 stores when rows are 16-byte multiples; the raw row is gathered
// through L1 (consecutive threads share a row).
__global__ void columns_kernel(const ColsArgs a) {
  const int groups = (a.n_out + 3) / 4;
  const int64_t total = a.n_rows * groups;
  const bool vec = (a.n_out & 3) == 0 && (reinterpret_cast<uintptr_t>(a.y) & 15) == 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / groups;
    const int f0 = (int)(i - r * groups) * 4;
    const float* row = a.x + r * a.ldx;
    float* out = a.y + r * a.n_out + f0;
    if (vec) {
      float4 v;
      v.x = load_col(a.ops, row, f0);
      v.y = load_col(a.ops, row, f0 + 1);
      v.z = load_col(a.ops, row, f0 + 2);
      v.w = load_col(a.ops, row, f0 + 3);
      __stcs(reinterpret_cast<float4*>(out), v);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (f0 + q < a.n_out) out[q] = load_col(a.ops, row, f0 + q);
    }
  }
}

__global__ void columns_check_kernel(const ColsArgs a) {
  const int64_t total = a.n_rows * a.n_checks;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / a.n_checks;
    const int c = (int)(i - r * a.n_checks);
    const float v = __ldg(a.x + r * a.ldx + __ldg(a.check_col + c));
    int64_t lo = __ldg(a.check_off + c), hi = __ldg(a.check_off + c + 1);
    bool found = false;
    while (lo < hi) {  // lower_bound
      const int64_t mid = (lo + hi) >> 1;
      const float u = __ldg(a.check_val + mid);
      if (u < v) lo = mid + 1;
      else hi = mid;
    }
    if (lo < __ldg(a.check_off + c + 1)) found = __ldg(a.check_val + lo) == v;
    if (!found) atomicMin(a.bad, (unsigned long long)r);
  }
}

// Folds this stage's first offending row into *out (initialised to -1 by the
// caller): several check stages may share one slot, and a clean stage must not
// erase an earlier stage's hit.
__global__ void columns_bad_finish(const unsigned long long* bad, int64_t* out) {
  if (*bad == ~0ull) return;
  const int64_t r = (int64_t)*bad;
  if (*out < 0 || r < *out) *out = r;
}

}  // namespace cmlb

struct cmlb_columns {
  int device = 0, n_in = 0, n_out = 0, n_checks = 0;
  cmlb_column_op* ops = nullptr;
  int32_t* check_col = nullptr;
  int64_t* check_off = nullptr;
  float* check_val = nullptr;
  ~cmlb_columns() { cudaFree(ops); cudaFree(check_col); cudaFree(check_off); cudaFree(check_val); }
};

namespace cmlb {
template <typename T>
static int dev_copy(T** dst, const T* src, size_t n) {
  CMLB_CUDA(cudaMalloc((void**)dst, std::max<size_t>(n, 1) * sizeof(T)));
  if (n) CMLB_CUDA(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return CMLB_OK;
}
}  // namespace cmlb

extern "C" {

int cmlb_columns_create(const cmlb_columns_desc* d, int device, cmlb_columns** out) {
  using namespace cmlb;
  if (!d || !out) return fail(CMLB_E_VALIDATION, "null columns descriptor");
  *out = nullptr;
  if (d->n_inputs < 1 || d->n_outputs < 0 || d->n_checks < 0) return fail(CMLB_E_VALIDATION, "bad column counts");
  for (int f = 0; f < d->n_outputs; ++f) {
    const cmlb_column_op& o = d->ops[f];
    if (o.src < 0 || o.src >= d->n_inputs || o.op < CMLB_COL_COPY || o.op > CMLB_COL_EQUAL)
      return fail(CMLB_E_VALIDATION, "bad column op");
  }
  for (int c = 0; c < d->n_checks; ++c) {
    if (d->check_col[c] < 0 || d->check_col[c] >= d->n_inputs) return fail(CMLB_E_VALIDATION, "bad check column");
    for (int64_t i = d->check_offset[c] + 1; i < d->check_offset[c + 1]; ++i)
      if (!(d->check_values[i - 1] < d->check_values[i])) return fail(CMLB_E_VALIDATION, "categories must ascend");
  }
  DeviceGuard guard(device);
  std::unique_ptr<cmlb_columns> m(new cmlb_columns());
  m->device = device; m->n_in = d->n_inputs; m->n_out = d->n_outputs; m->n_checks = d->n_checks;
  int st;
  if ((st = dev_copy(&m->ops, d->ops, (size_t)d->n_outputs))) return st;
  if (d->n_checks > 0) {
    const int64_t nv = d->check_offset[d->n_checks];
    if ((st = dev_copy(&m->check_col, d->check_col, (size_t)d->n_checks)) ||
        (st = dev_copy(&m->check_off, d->check_offset, (size_t)d->n_checks + 1)) ||
        (st = dev_copy(&m->check_val, d->check_values, (size_t)nv)))
      return st;
  }
  *out = m.release();
  return CMLB_OK;
}

int cmlb_columns_run(const cmlb_columns* m, const float* x, int64_t n_rows, int64_t ldx, float* y,
                     int64_t* bad_row, void* stream) {
  using namespace cmlb;
  if (!m) return fail(CMLB_E_VALIDATION, "null columns program");
  if (n_rows < 0 || ldx < m->n_in) return fail(CMLB_E_INPUT, "bad input extents");
  DeviceGuard guard(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ColsArgs a{};
  a.x = x; a.n_rows = n_rows; a.ldx = ldx; a.y = y; a.ops = m->ops; a.n_out = m->n_out;
  a.n_checks = m->n_checks; a.check_col = m->check_col; a.check_off = m->check_off; a.check_val = m->check_val;
  const int sms = num_sms(m->device);
  if (y && n_rows > 0 && m->n_out > 0) {
    const int64_t work = n_rows * ((m->n_out + 3) / 4);
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(work, 256), (int64_t)sms * 16);
    columns_kernel<<<grid, 256, 0, s>>>(a);
    CMLB_CUDA(cudaGetLastError());
    note_launch();
  }
  if (bad_row) {
    keep_pool(m->device);
    void* scratch = nullptr;
    CMLB_CUDA(cudaMallocAsync(&scratch, sizeof(unsigned long long), s));
    a.bad = static_cast<unsigned long long*>(scratch);
    CMLB_CUDA(cudaMemsetAsync(a.bad, 0xFF, sizeof(unsigned long long), s));
    if (m->n_checks > 0 && n_rows > 0) {
      const int64_t work = n_rows * m->n_checks;
      const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(work, 256), (int64_t)sms * 16);
      columns_check_kernel<<<grid, 256, 0, s>>>(a);
      CMLB_CUDA(cudaGetLastError());
      note_launch();
    }
    columns_bad_finish<<<1, 1, 0, s>>>(a.bad, bad_row);
    CMLB_CUDA(cudaGetLastError());
    note_launch();
    CMLB_CUDA(cudaFreeAsync(scratch, s));
  }
  return CMLB_OK;
}

void cmlb_columns_destroy(cmlb_columns* m) {
  if (!m) return;
  cmlb::DeviceGuard guard(m->device);
  delete m;
}

}  // extern "C"
