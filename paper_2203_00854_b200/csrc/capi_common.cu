#include <cstdlib>
// Library-level C-ABI entry points and the error-string plumbing shared by all
// kernels (include/evo.h).  Errors are per host thread.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace evo {

static thread_local char g_err[512] = "no error";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
  return EVO_ERR_CUDA;
}

}  // namespace evo

extern "C" const char* evo_version(void) { return "evo-b200 0.1.0 (sm_100a)"; }

namespace evo {
bool pdl_enabled() {
  static const bool on = [] { const char* e = getenv("EVO_NO_PDL"); return !(e && e[0] == '1'); }();
  return on;
}
}  // namespace evo

extern "C" const char* evo_last_error_string(void) { return evo::g_err; }

extern "C" int evo_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return evo::cuda_status(e, "cudaGetDevice");
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) return evo::cuda_status(e, "cudaGetDeviceProperties");
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return EVO_OK;
}
