// Library-level entry points: version, error string, device info.
#include <stdarg.h>

#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace rsr {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return RSR_ECUDA;
  }
  return RSR_OK;
}

int ensure_dynamic_smem(const void* fn, size_t bytes) {
  // cudaFuncSetAttribute costs microseconds per call and the per-iteration
  // launches of the Stage-1 loop repeat it: remember what each (device, kernel)
  // already allows
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  int dev = 0;
  RSR_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = granted[{dev, fn}];
  if (bytes <= have) return RSR_OK;
  RSR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  have = bytes;
  return RSR_OK;
}

}  // namespace rsr

extern "C" int rsr_version(void) { return 1; }

extern "C" const char* rsr_last_error(void) { return rsr::g_err; }

extern "C" int rsr_thermo_kpad(int n_components, int n_states) {
  if (n_components < 1 || n_states < 2) return -1;
  return rsr::thermo_kpad(n_components, n_states);
}

extern "C" int rsr_device_info(int* sm_count_host, int* cc_major_host, int* cc_minor_host) {
  int dev = 0;
  RSR_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp p;
  RSR_CUDA(cudaGetDeviceProperties(&p, dev));
  if (sm_count_host) *sm_count_host = p.multiProcessorCount;
  if (cc_major_host) *cc_major_host = p.major;
  if (cc_minor_host) *cc_minor_host = p.minor;
  return RSR_OK;
}
