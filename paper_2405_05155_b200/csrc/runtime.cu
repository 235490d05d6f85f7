// runtime.cu — library identity and error reporting for the sphb C ABI.
#include <stdio.h>

#include "common.cuh"

static thread_local char g_last_error[256] = "";

const char* sphb_set_cuda_error(cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e),
           cudaGetErrorString(e));
  return g_last_error;
}

extern "C" const char* sphb_version(void) { return "sphb 0.1 (sm_100a)"; }

extern "C" const char* sphb_last_cuda_error(void) { return g_last_error; }

extern "C" int sphb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}
