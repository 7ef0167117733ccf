// Shared plumbing for the cmlb C ABI: status/error reporting, launch
// accounting, and the bit-exact scalar helpers every epilogue uses.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <string>

#include "cmlb.h"

namespace cmlb {

// ---- status / last error (thread-local, cmlb_last_error) -------------------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void note_launch(int n = 1);

#define CMLB_CUDA(call)                                   \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return ::cmlb::cuda_fail(_e, #call); \
  } while (0)

// Device-side guard used by every run entry point.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ---- bit-exact scalar semantics --------------------------------------------

// numpy.argmax over float32: first maximum; the first NaN wins outright
// (np.argmax treats NaN as maximal), reference kernels.py:197-203.
template <int CT>
__device__ __forceinline__ int first_max(const float (&v)[CT], int c) {
  int best = 0;
  float bv = v[0];
  if (bv != bv) return 0;
#pragma unroll
  for (int i = 1; i < CT; ++i) {
    if (i < c) {
      float x = v[i];
      if (x != x) return i;
      if (x > bv) { bv = x; best = i; }
    }
  }
  return best;
}

// Reference sigmoid (kernels.py:234-235): float64, branch on sign, then the
// caller rounds to float32.  NaN takes the second branch and stays NaN.
__device__ __forceinline__ double ref_sigmoid(double x) {
  double e = exp(-fabs(x));
  return x >= 0.0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
}

// Store one output element in the reference output dtype.
__device__ __forceinline__ void store_out(void* y, int64_t i, int dt, double v) {
  switch (dt) {
    case CMLB_OUT_BOOL: static_cast<uint8_t*>(y)[i] = (uint8_t)(int)v; break;
    case CMLB_OUT_INT8: static_cast<int8_t*>(y)[i] = (int8_t)(int)v; break;
    case CMLB_OUT_INT16: static_cast<int16_t*>(y)[i] = (int16_t)(int)v; break;
    case CMLB_OUT_INT32: static_cast<int32_t*>(y)[i] = (int32_t)v; break;
    default: static_cast<float*>(y)[i] = (float)v; break;
  }
}

// Fused preprocessing: model feature f = op(x[src]) with the reference
// scalers' float32 rounding (convert.py:255-284) and OneHotEncoder's
// indicator (cmlb.h: cmlb_column_op).  A null prologue reads x[f].
__device__ __forceinline__ float col_apply(int op, float v, float a, float b) {
  switch (op) {
    case CMLB_COL_COPY: return v;
    case CMLB_COL_SUB_DIV: return __fdiv_rn(__fsub_rn(v, a), b);
    case CMLB_COL_DIV: return __fdiv_rn(v, a);
    case CMLB_COL_MUL_ADD: return __fadd_rn(__fmul_rn(v, a), b);
    case CMLB_COL_GREATER: return v > a ? 1.0f : 0.0f;
    default: return v == a ? 1.0f : 0.0f;  // CMLB_COL_EQUAL
  }
}
__device__ __forceinline__ float load_col(const cmlb_column_op* pro, const float* row, int f) {
  if (pro == nullptr) return __ldg(row + f);
  const int4 w = __ldg(reinterpret_cast<const int4*>(pro) + f);
  return col_apply(w.y, __ldg(row + w.x), __int_as_float(w.z), __int_as_float(w.w));
}

inline int out_dtype_ok(int dt) { return dt >= CMLB_OUT_BOOL && dt <= CMLB_OUT_F32; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int num_sms(int device);
void keep_pool(int device);

}  // namespace cmlb
