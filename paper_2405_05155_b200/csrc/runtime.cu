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

// FP64 pipe probe: 8 independent DFMA chains per thread; flops = 2 * 8 * iters
// per thread.  Used by bench.py to measure the FP64 roofline denominator live
// (MEASURED_PEAKS.json carries no FP64 figure).
__global__ void k_fp64_probe(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

extern "C" int sphb_fp64_probe(double* out, int32_t blocks, int32_t threads, int32_t iters,
                               void* stream) {
  if (blocks <= 0 || threads <= 0 || iters <= 0) return SPHB_ERR_ARG;
  k_fp64_probe<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, iters, 0.999999, 1e-7);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

// Small device -> host reads without the copy engines: one warp stores the
// words straight into mapped pinned host memory.  A cudaMemcpy of a few
// bytes would queue behind any bulk transfer in flight on the same copy
// engine (e.g. a 512 MiB read_state), stalling the host for its duration.
__global__ void k_mirror_words(const uint32_t* __restrict__ src, volatile uint32_t* dst,
                               int64_t words) {
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
  __threadfence_system();
}

extern "C" int sphb_mirror_to_host(const void* src, void* host_dst, int64_t bytes, void* stream) {
  if (!src || !host_dst || bytes <= 0 || bytes % 4 || bytes > 4096) return SPHB_ERR_ARG;
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, host_dst, 0) != cudaSuccess || !dptr) {
    cudaGetLastError();                       // not mapped pinned memory: caller falls back
    return SPHB_ERR_ARG;
  }
  k_mirror_words<<<1, 32, 0, (cudaStream_t)stream>>>((const uint32_t*)src, (uint32_t*)dptr,
                                                     bytes / 4);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
