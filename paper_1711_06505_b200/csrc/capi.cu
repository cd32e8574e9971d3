// Error plumbing and small C-ABI utilities.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace {
thread_local char g_err[1024] = "";
}

namespace dicm {

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return DICM_OK;
  return fail(DICM_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

int last_launch(const char* where) { return check_cuda(cudaGetLastError(), where); }

}  // namespace dicm

extern "C" {

const char* dicm_last_error(void) { return g_err; }

int dicm_version(void) { return 1; }

int dicm_device_arch(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return -1;
  return p.major * 10 + p.minor;
}

}  // extern "C"
