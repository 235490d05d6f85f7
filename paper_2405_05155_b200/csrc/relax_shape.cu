// relax_shape.cu — shape-bounded particle relaxation.
//
// relax() for a shape (relaxation.py:132-210 with box=None) adds two pieces
// to the periodic step of relax_engine.cu:
//   * the analytic wall confinement (relaxation.py:92-117, 162-168): a
//     particle at depth s < cutoff below the surface gets
//     acc -= (2 p0 / rho0) w2(s) n, where w2 is the planar kernel integral
//     tabulated on the host (np.interp with right = 0 restated here) and n
//     the unit SDF gradient by central differences (geometry.py:137-147);
//   * the surface projection after the capped update (relaxation.py:120-129,
//     196-198): up to three Newton steps x -= sd(x) grad(x) for particles
//     that left the shape.
// Signed distances follow geometry.py:16-126 term by term.  Compiled with
// --fmad=false so every expression rounds as numpy does.
#include <algorithm>

#include "common.cuh"

using namespace sphb;

namespace {

template <int D>
__device__ __forceinline__ double norm_d(const double* v) {
  double s = v[0] * v[0];
#pragma unroll
  for (int a = 1; a < D; ++a) s = s + v[a] * v[a];
  return sqrt(s);
}

// geometry.py:37-39 (circle), 60-69 (rectangle), 107-126 (half disk)
template <int D>
__device__ double sdf(const sphb_shape& s, const double* x) {
  if (s.kind == 1) {
    double p[D];
#pragma unroll
    for (int a = 0; a < D; ++a) p[a] = x[a] - s.center[a];
    return norm_d<D>(p) - s.radius;
  }
  if (s.kind == 2) {
    double q[D], qp[D];
    double qmax = -INFINITY;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double c = 0.5 * (s.lo[a] + s.hi[a]);
      const double half = 0.5 * (s.hi[a] - s.lo[a]);
      q[a] = fabs(x[a] - c) - half;
      qp[a] = q[a] > 0.0 ? q[a] : 0.0;
      qmax = q[a] > qmax ? q[a] : qmax;
    }
    return norm_d<D>(qp) + (qmax < 0.0 ? qmax : 0.0);
  }
  // half disk
  double p[D], t[D];
#pragma unroll
  for (int a = 0; a < D; ++a) p[a] = x[a] - s.center[a];
  double h = p[0] * s.normal[0];
#pragma unroll
  for (int a = 1; a < D; ++a) h = h + p[a] * s.normal[a];
#pragma unroll
  for (int a = 0; a < D; ++a) t[a] = p[a] - h * s.normal[a];
  const double tn = norm_d<D>(t);
  if (h <= 0.0) {
    const double d_disk = norm_d<D>(p) - s.radius;
    return d_disk > h ? d_disk : h;
  }
  const double tc = tn < s.radius ? tn : s.radius;
  double m = tn - tc;
  m = m > 0.0 ? m : 0.0;
  return sqrt(m * m + h * h);
}

// geometry.py:137-147 (eps = 1e-7)
template <int D>
__device__ void sdf_grad(const sphb_shape& s, const double* x, double* g) {
  const double eps = 1e-7;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double xp[D], xm[D];
#pragma unroll
    for (int b = 0; b < D; ++b) xp[b] = xm[b] = x[b];
    xp[a] = x[a] + eps;
    xm[a] = x[a] - eps;
    g[a] = (sdf<D>(s, xp) - sdf<D>(s, xm)) / (2.0 * eps);
  }
  double n = norm_d<D>(g);
  if (n == 0.0) n = 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) g[a] = g[a] / n;
}

// np.interp(x, xp, fp, right=0.0) (left = fp[0])
__device__ double interp_right0(double x, const double* __restrict__ xp,
                                const double* __restrict__ fp, int n) {
  if (x != x) return x;
  if (x < xp[0]) return fp[0];
  if (x > xp[n - 1]) return 0.0;
  if (x == xp[n - 1]) return fp[n - 1];
  int lo = 0, hi = n - 1;   // xp[lo] <= x < xp[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (xp[mid] <= x) lo = mid;
    else hi = mid;
  }
  if (xp[lo] == x) return fp[lo];
  const double slope = (fp[lo + 1] - fp[lo]) / (xp[lo + 1] - xp[lo]);
  return slope * (x - xp[lo]) + fp[lo];
}

template <int D>
__global__ void k_shape_sdf(sphb_shape s, int64_t n, const double* __restrict__ x,
                            double* __restrict__ sd, double* __restrict__ grad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[D];
#pragma unroll
  for (int a = 0; a < D; ++a) p[a] = x[i * D + a];
  if (sd) sd[i] = sdf<D>(s, p);
  if (grad) {
    double g[D];
    sdf_grad<D>(s, p, g);
#pragma unroll
    for (int a = 0; a < D; ++a) grad[i * D + a] = g[a];
  }
}

// relaxation.py:162-170: confinement near the surface, then |a| summed
// into sums[2] over every particle (the residual's numerator).
template <int D>
__global__ void __launch_bounds__(128)
k_relax_confine(sphb_shape s, int64_t n, const double* __restrict__ pos, double cutoff,
                const double* __restrict__ s_grid, const double* __restrict__ w2, int32_t n_s,
                double coef, double* __restrict__ acc, double* __restrict__ sums) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double norm = 0.0;
  if (i < n) {
    double p[D], a_[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      p[a] = pos[i * D + a];
      a_[a] = acc[i * D + a];
    }
    const double depth = -sdf<D>(s, p);
    if (depth < cutoff) {
      double g[D];
      sdf_grad<D>(s, p, g);
      const double cw = coef * interp_right0(depth, s_grid, w2, n_s);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        a_[a] = a_[a] - cw * g[a];
        acc[i * D + a] = a_[a];
      }
    }
    norm = norm_d<D>(a_);
  }
  norm = warp_sum(norm);
  if ((threadIdx.x & 31) == 0 && norm != 0.0) atomicAdd(sums + 2, norm);
}

// relaxation.py:188-198 + _project_to_surface (:120-129)
template <int D>
__global__ void k_relax_update_shape(sphb_shape s, int64_t n, const double* __restrict__ acc,
                                     double dt2, double cap, double surf_tol,
                                     double* __restrict__ pos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double dx[D], p[D];
#pragma unroll
  for (int a = 0; a < D; ++a) dx[a] = acc[i * D + a] * dt2;
  const double nrm = norm_d<D>(dx);
  if (nrm > cap) {
    const double f = cap / nrm;
#pragma unroll
    for (int a = 0; a < D; ++a) dx[a] = dx[a] * f;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) p[a] = pos[i * D + a] + dx[a];
  bool outside = sdf<D>(s, p) > surf_tol;
  for (int it = 0; it < 3 && outside; ++it) {
    const double sd = sdf<D>(s, p);
    double g[D];
    sdf_grad<D>(s, p, g);
#pragma unroll
    for (int a = 0; a < D; ++a) p[a] = p[a] - sd * g[a];
    outside = sdf<D>(s, p) > 1e-12;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) pos[i * D + a] = p[a];
}

__device__ void atomic_min_d(double* addr, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *a;
  while (v < __longlong_as_double((long long)old)) {
    const unsigned long long prev = atomicCAS(a, old, (unsigned long long)__double_as_longlong(v));
    if (prev == old) break;
    old = prev;
  }
}

__device__ void atomic_max_d(double* addr, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *a;
  while (v > __longlong_as_double((long long)old)) {
    const unsigned long long prev = atomicCAS(a, old, (unsigned long long)__double_as_longlong(v));
    if (prev == old) break;
    old = prev;
  }
}

__global__ void k_init_bounds(int32_t dim, double* out) {
  const int a = threadIdx.x;
  if (a < dim) {
    out[a] = INFINITY;
    out[dim + a] = -INFINITY;
  }
}

template <int D>
__global__ void __launch_bounds__(256)
k_bounds(int64_t n, const double* __restrict__ pos, double* __restrict__ out) {
  double lo[D], hi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lo[a] = INFINITY;
    hi[a] = -INFINITY;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double v = pos[i * D + a];
      lo[a] = v < lo[a] ? v : lo[a];
      hi[a] = v > hi[a] ? v : hi[a];
    }
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      const double l = __shfl_xor_sync(0xffffffffu, lo[a], o);
      const double h = __shfl_xor_sync(0xffffffffu, hi[a], o);
      lo[a] = l < lo[a] ? l : lo[a];
      hi[a] = h > hi[a] ? h : hi[a];
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      atomic_min_d(out + a, lo[a]);
      atomic_max_d(out + D + a, hi[a]);
    }
  }
}

bool shape_ok(const sphb_shape* s) {
  return s && s->kind >= 1 && s->kind <= 3 && s->dim >= 1 && s->dim <= 3;
}

}  // namespace

#define SPHB_SHAPE_D(dim, kern, grid, T, ...)                                   \
  switch (dim) {                                                                 \
    case 1: kern<1><<<grid, T, 0, st>>>(__VA_ARGS__); break;                     \
    case 2: kern<2><<<grid, T, 0, st>>>(__VA_ARGS__); break;                     \
    case 3: kern<3><<<grid, T, 0, st>>>(__VA_ARGS__); break;                     \
    default: return SPHB_ERR_ARG;                                                \
  }

extern "C" int sphb_shape_sdf(const sphb_shape* s, int64_t n, const double* x, double* sd,
                              double* grad, void* stream) {
  if (!shape_ok(s) || n < 0 || (n > 0 && !x)) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_SHAPE_D(s->dim, k_shape_sdf, sphb_blocks(n, 128), 128, *s, n, x, sd, grad);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_relax_confine(const sphb_shape* s, int64_t n, const double* pos,
                                  double cutoff, const double* s_grid, const double* w2,
                                  int32_t n_s, double coef, double* acc, double* sums,
                                  void* stream) {
  if (!shape_ok(s) || n < 0 || n_s < 2 || !s_grid || !w2 || !sums) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_CUDA_CHECK(cudaMemsetAsync(sums + 2, 0, sizeof(double), st));
  if (n == 0) return SPHB_OK;
  SPHB_SHAPE_D(s->dim, k_relax_confine, sphb_blocks(n, 128), 128, *s, n, pos, cutoff, s_grid,
               w2, n_s, coef, acc, sums);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_relax_update_shape(const sphb_shape* s, int64_t n, const double* acc,
                                       double dt2, double cap, double surf_tol, double* pos,
                                       void* stream) {
  if (!shape_ok(s) || n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_SHAPE_D(s->dim, k_relax_update_shape, sphb_blocks(n, 128), 128, *s, n, acc, dt2, cap,
               surf_tol, pos);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_bounds(int64_t n, int32_t dim, const double* pos, double* out,
                           void* stream) {
  if (n < 0 || dim < 1 || dim > 3 || !out) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  k_init_bounds<<<1, 32, 0, st>>>(dim, out);
  if (n > 0) {
    const unsigned grid = (unsigned)std::min<int64_t>(sphb_blocks(n, 256), 4 * 148);
    SPHB_SHAPE_D(dim, k_bounds, grid, 256, n, pos, out);
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
