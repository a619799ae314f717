// Error state and device checks for the C ABI (include/sparse24_b200.h).
// Errors are recorded per calling thread; kernels never abort the process.
#include <cstdarg>
#include <cstdio>

#include "s24_common.cuh"

static thread_local char g_err[512] = "no error";

int s24_set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int s24_check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return s24_set_error(S24_ERR_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
  return S24_OK;
}

extern "C" const char* s24_last_error_string(void) { return g_err; }

extern "C" int s24_abi_version(void) { return S24_ABI_VERSION; }

extern "C" int s24_device_check(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return s24_set_error(S24_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return s24_set_error(S24_ERR_UNSUPPORTED, "kernels are built for sm_100a, device is sm_%d%d", major, minor);
  return S24_OK;
}
