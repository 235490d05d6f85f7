// Microbenchmark (vector f64 red is not available on sm_100a): throughput of FP64 reductions to global memory in the
// pattern a pair-symmetric WC stage would issue (lane i of a warp adds 4
// doubles into row i + off_k, rows consecutive across the warp).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_f64 red_f64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_red(long n, const int* off, int slots, double4* acc, int vec) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 1e-3 * (double)(i & 1023);
  for (int k = 0; k < slots; ++k) {
    long j = i + off[k];
    if (j >= n) j -= n;
    if (j < 0) j += n;
    double* p = reinterpret_cast<double*>(acc + j);
    if (vec) {   // one component per lane-quarter: 4 rows' x, then y, ... (same count)
      atomicAdd(p + (k & 3), v); atomicAdd(p + ((k + 1) & 3), v);
      atomicAdd(p + ((k + 2) & 3), v); atomicAdd(p + ((k + 3) & 3), v);
    } else {
      atomicAdd(p, v); atomicAdd(p + 1, v); atomicAdd(p + 2, v); atomicAdd(p + 3, v);
    }
  }
}

__global__ void k_store(long n, const int* off, int slots, double4* acc) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 1e-3 * (double)(i & 1023);
  for (int k = 0; k < slots; ++k) {
    long j = i + off[k];
    if (j >= n) j -= n;
    if (j < 0) j += n;
    acc[j] = make_double4(v, v, v, v);
  }
}

int main() {
  const long n = 256L * 256 * 256;
  const int slots = 16;
  int hoff[slots];
  // half stencil of a 3D lattice (x fastest, 256 x 256 layers)
  int c = 0;
  for (int dz = 0; dz <= 2 && c < slots; ++dz)
    for (int dy = -2; dy <= 2 && c < slots; ++dy)
      for (int dx = -2; dx <= 2 && c < slots; ++dx) {
        long o = dx + 256L * dy + 65536L * dz;
        if (o > 0 && dx * dx + dy * dy + dz * dz <= 4) hoff[c++] = (int)o;
      }
  int* off;
  double4* acc;
  cudaMalloc(&off, sizeof(hoff));
  cudaMemcpy(off, hoff, sizeof(hoff), cudaMemcpyHostToDevice);
  cudaMalloc(&acc, n * sizeof(double4));
  cudaMemset(acc, 0, n * sizeof(double4));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode == 2)
        k_store<<<(n + 255) / 256, 256>>>(n, off, c, acc);
      else
        k_red<<<(n + 255) / 256, 256>>>(n, off, c, acc, mode);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2)
        printf("%s slots=%d: %.3f ms, %.1f G f64-adds/s\n",
               mode == 0 ? "atomicAdd x4" : (mode == 1 ? "atomicAdd x4 rotated" : "store (no atomics)"), c,
               ms, n * (double)c * 4 / (ms * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
