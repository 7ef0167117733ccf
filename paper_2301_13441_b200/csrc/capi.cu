// Error plumbing and process-wide counters behind include/cmlb.h.
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace cmlb {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof(buf), "CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
  g_last_error = buf;
  return CMLB_E_DEVICE;
}

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default
// pool; keep freed blocks cached there instead of returning them to the
// driver at every synchronisation (the default threshold of 0 turns each
// run's scratch into a fresh mapping).
void keep_pool(int device) {
  static std::mutex mu;
  static std::unordered_map<int, bool> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[device] = true;
}

int num_sms(int device) {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) n = 148;
  cache[device] = n;
  return n;
}

}  // namespace cmlb

extern "C" {

const char* cmlb_last_error(void) { return cmlb::g_last_error.c_str(); }
int cmlb_abi_version(void) { return CMLB_ABI_VERSION; }
int64_t cmlb_launch_count(void) { return cmlb::g_launches.load(); }

}  // extern "C"
