// common.cuh — shared device helpers for the sphb kernels (sm_100a).
//
// Kernel profiles restate kernels.py:41-59; cell geometry restates
// neighbors.py:38-53 and the stencil walk of _search (neighbors.py:87-167).
// Every operation that decides neighbour MEMBERSHIP uses explicit
// round-to-nearest intrinsics (__dsub_rn/__dmul_rn/__dadd_rn) so the result
// is bit-identical to the reference's un-contracted numba arithmetic no
// matter how the translation unit is compiled.
#pragma once

#include <cuda_pipeline.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sphb.h"

namespace sphb {

constexpr double kEpsSV = 1e-4;    // correction.py:24
constexpr double kEpsDet = 1e-6;   // correction.py:25
constexpr double kEtaLinearized = 15.0;  // eulerian.py:30

// ---------------------------------------------------------------- profiles
// Same association order as the numba source (left to right).
__device__ __forceinline__ double profile(int code, double q) {
  if (code == SPHB_CODE_WENDLAND) {
    double t = 1.0 - 0.5 * q;
    return t * t * t * t * (2.0 * q + 1.0);
  }
  double q2 = q * q;
  return (1.0 - 0.5 * q2 + q2 * q2 / 6.0) * exp(-q2);
}

__device__ __forceinline__ double profile_deriv(int code, double q) {
  if (code == SPHB_CODE_WENDLAND) {
    double t = 1.0 - 0.5 * q;
    return -5.0 * q * t * t * t;
  }
  double q2 = q * q;
  return q * (-3.0 + (5.0 / 3.0) * q2 - q2 * q2 / 3.0) * exp(-q2);
}

// ---------------------------------------------------------------- helpers
// numpy float remainder (npy_divmod): fmod, then shift into the sign of b.
__device__ __forceinline__ double np_remainder(double a, double b) {
  // already inside (0, b): fmod(a, b) == a exactly (the common case for
  // wrapped coordinates); skips the multi-instruction fmod sequence
  if (a > 0.0 && a < b) return a;
  double mod = fmod(a, b);
  if (mod != 0.0) {
    if ((b < 0.0) != (mod < 0.0)) mod += b;
  } else {
    mod = copysign(0.0, b);
  }
  return mod;
}

// Python-semantics integer modulo (numba `c % n` on int64).
__device__ __forceinline__ int64_t py_mod(int64_t c, int64_t n) {
  int64_t r = c % n;
  return r < 0 ? r + n : r;
}

// Cell coordinate of one wrapped coordinate (neighbors.py:38-53).
__device__ __forceinline__ int64_t cell_coord(const sphb_grid& g, int a, double w) {
  int64_t c = (int64_t)floor(__dmul_rn(w, g.inv_cell[a]));
  if (g.periodic) {
    c = py_mod(c, g.ncell[a]);
  } else {
    if (c < 0) c = 0;
    else if (c >= g.ncell[a]) c = g.ncell[a] - 1;
  }
  return c;
}

// Exact pair displacement on wrapped coordinates with the reference's
// minimum-image branch (neighbors.py:152-157 of _search).
__device__ __forceinline__ double min_image(double dx, double box, int periodic) {
  if (periodic) {
    double half = 0.5 * box;  // exact
    if (dx > half) dx = __dsub_rn(dx, box);
    else if (dx < -half) dx = __dadd_rn(dx, box);
  }
  return dx;
}

// Walk the 3^D stencil of sorted particle s in the reference's order
// (offset index k with axis 0 fastest; ascending index inside a cell) and
// call f(t, dx, r2) for every candidate t with 0 < r2 <= cut2.
template <int D, class F>
__device__ __forceinline__ void for_each_neighbor(const sphb_grid& g, int64_t n,
                                                  const double* __restrict__ ws,
                                                  const int32_t* __restrict__ cs,
                                                  const int32_t* __restrict__ ce,
                                                  int32_t s, F&& f) {
  double wi[D];
  int64_t ci[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    wi[a] = ws[(int64_t)a * n + s];
    ci[a] = cell_coord(g, a, wi[a]);
  }
  constexpr int noff = D == 1 ? 3 : (D == 2 ? 9 : 27);
  for (int k = 0; k < noff; ++k) {
    int rem = k;
    int64_t flat = 0;
    bool ok = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      int off = rem % 3 - 1;
      rem /= 3;
      int64_t c = ci[a] + off;
      if (g.periodic) {
        c = py_mod(c, g.ncell[a]);
      } else if (c < 0 || c >= g.ncell[a]) {
        ok = false;
      }
      flat += c * g.strides[a];
    }
    if (!ok) continue;
    const int32_t t0 = cs[flat];
    const int32_t t1 = ce[flat];
    for (int32_t t = t0; t < t1; ++t) {
      if (t == s) continue;
      double dx[D];
      double r2 = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        dx[a] = min_image(__dsub_rn(wi[a], ws[(int64_t)a * n + t]), g.box[a], g.periodic);
        r2 = __dadd_rn(r2, __dmul_rn(dx[a], dx[a]));
      }
      if (r2 <= g.cut2 && r2 > 0.0) f(t, dx, r2);
    }
  }
}

// Dynamic shared memory above this needs cudaFuncAttributeMaxDynamicSharedMemorySize:
// the 48 KB default covers static + dynamic, so leave room for the kernels'
// static arrays (at most 5 KB here).
constexpr size_t kDynSmemDefault = 43 * 1024;
// Launches above the default raise cudaFuncAttributeMaxDynamicSharedMemorySize
// to this fixed bound (never to the launch's own size): the attribute is per
// function, so a per-call value set by one host thread could be lowered by
// another between its set and its launch (thread-simulated slab ranks).
constexpr int kDynSmemMax = 200 * 1024;

// Debug builds (make debug: -DSPHB_DEBUG_BOUNDS) check every pass-list index
// before it addresses a record: out-of-range indices raise
// SPHB_EFLAG_BAD_INDEX in the kernel's error word and are clamped to 0.
#ifdef SPHB_DEBUG_BOUNDS
#define SPHB_CHECK_INDEX(j, n, err)                                       \
  do {                                                                    \
    if ((uint64_t)(j) >= (uint64_t)(n)) {                                 \
      atomicOr((err), SPHB_EFLAG_BAD_INDEX);                              \
      (j) = 0;                                                            \
    }                                                                     \
  } while (0)
#else
#define SPHB_CHECK_INDEX(j, n, err) \
  do {                              \
  } while (0)
#endif

// 256-bit read-only gather (sm_100: LDG.E.ENL2.256).  A plain double4 load
// compiles to two LDG.128; one request per 32-byte record halves the L1
// requests of the neighbour gathers.  Only for data not written by the
// running kernel.
__device__ __forceinline__ double4 ldg4(const double4* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p));
  return v;
}

// 1/sqrt(x) and 1/x for normal positive doubles: MUFU seed (~2^-23) and
// one third-order correction (error ~eps^3, below double rounding), i.e. the
// accuracy of two Newton steps with a shorter dependent chain; no
// special-value handling, so no slow-path call.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);         // 1 - x y^2
  // y (1 + e/2 + 3 e^2 / 8)
  return fma(y * e, fma(0.375, e, 0.5), y);
}

__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);               // 1 - x y
  return fma(y, fma(e, e, e), y);                  // y (1 + e + e^2)
}

// ----------------------------------------------------------- reductions
// Copy a block's ELL columns nbr[k * n + base + r] (k < width, r < RB) into
// shared memory s_nbr[k * RB + r] and wait: the pass list then costs one
// DRAM round trip per block instead of one per loop iteration.  When every
// column slice is 16-byte aligned (n, base and the row count multiples of 4)
// one thread issues a TMA bulk copy per column (cp.async.bulk, completion on
// an mbarrier); otherwise every thread copies 4-byte words with LDGSTS.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int RB>
__device__ __forceinline__ void stage_pass_list(const int32_t* __restrict__ nbr, int64_t n,
                                                int64_t base, int64_t lim, int width,
                                                int32_t* s_nbr) {
  const int64_t rows = lim - base < RB ? lim - base : RB;
  const bool bulk = ((n | base | rows) & 3) == 0 && rows > 0;
  if (bulk) {
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = smem_u32(&bar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bytes = (uint32_t)(rows * sizeof(int32_t));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   ::"r"(b), "r"(bytes * (uint32_t)width) : "memory");
      for (int k = 0; k < width; ++k)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_u32(s_nbr + k * RB)), "l"(nbr + (int64_t)k * n + base), "r"(bytes), "r"(b)
            : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
          " selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done) : "r"(b) : "memory");
    return;
  }
  for (int e = threadIdx.x; e < width * RB; e += blockDim.x) {
    const int k = e / RB, r = e % RB;
    if (base + r < lim)
      __pipeline_memcpy_async(s_nbr + e, nbr + (int64_t)k * n + base + r, sizeof(int32_t));
  }
  __pipeline_commit();
  __pipeline_wait_prior(0);
  __syncthreads();
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their int64 bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            (unsigned long long)__double_as_longlong(v));
}

template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = v > w ? v : w;
  }
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace sphb

// ---------------------------------------------------------------- host side
const char* sphb_set_cuda_error(cudaError_t e);

#define SPHB_CUDA_CHECK(expr)                      \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) {                       \
      sphb_set_cuda_error(_e);                     \
      return SPHB_ERR_CUDA;                        \
    }                                              \
  } while (0)

#define SPHB_LAUNCH_CHECK() SPHB_CUDA_CHECK(cudaGetLastError())

static inline unsigned int sphb_blocks(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned int)(b < 1 ? 1 : b);
}

static inline size_t sphb_align(size_t x) { return (x + 255) & ~(size_t)255; }
