// relax_engine.cu — one pseudo-time step of periodic particle relaxation.
//
// relax() (relaxation.py:157-195) rebuilds the neighbour list every step and
// then streams it once through _pressure_accel (:66-80).  Here the list is
// never materialised: after binning (sphb_bin) each thread walks its cell
// stencil in the reference's order and accumulates the constant-pressure
// acceleration directly, with r = sqrt(r2), e = dx / r, q = r / h and the
// coefficient evaluated in the reference's association order.  This unit is
// compiled with --fmad=false so the per-row sums equal the reference's
// CSR-order sums bit for bit (Wendland; LG differs only through exp()).
#include "common.cuh"

using namespace sphb;

namespace {

template <int D>
__global__ void __launch_bounds__(128)
k_relax_accel(sphb_grid g, int64_t n, const double* __restrict__ ws,
              const int32_t* __restrict__ perm, const int32_t* __restrict__ cs,
              const int32_t* __restrict__ ce, const double* __restrict__ vols, sphb_kernel k,
              double p0, double rho0, double* __restrict__ acc, double* __restrict__ sums) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double norm = 0.0, isolated = 0.0;
  if (s < n) {
    const double scale = k.alpha / k.h;
    double a_[D];
#pragma unroll
    for (int a = 0; a < D; ++a) a_[a] = 0.0;
    int32_t count = 0;
    for_each_neighbor<D>(g, n, ws, cs, ce, (int32_t)s, [&](int32_t t, const double* dx, double r2) {
      ++count;
      const double r = sqrt(r2);
      const double q = r / k.h;
      if (q > k.kappa) return;
      const double coeff = -2.0 * p0 * vols[perm[t]] * scale * profile_deriv(k.code, q) / rho0;
#pragma unroll
      for (int a = 0; a < D; ++a) a_[a] += coeff * (dx[a] / r);
    });
    const int64_t i = perm[s];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[i * D + a] = a_[a];
    double s2 = a_[0] * a_[0];
#pragma unroll
    for (int a = 1; a < D; ++a) s2 += a_[a] * a_[a];
    norm = sqrt(s2);
    isolated = count == 0 ? 1.0 : 0.0;
  }
  norm = warp_sum(norm);
  isolated = warp_sum(isolated);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(sums, norm);
    if (isolated != 0.0) atomicAdd(sums + 1, isolated);
  }
}

template <int D>
__global__ void k_relax_update(int64_t n, const double* __restrict__ acc, double dt2, double cap,
                               double b0, double b1, double b2, double* __restrict__ pos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double box[3] = {b0, b1, b2};
  double dx[D];
#pragma unroll
  for (int a = 0; a < D; ++a) dx[a] = acc[i * D + a] * dt2;
  double s2 = dx[0] * dx[0];
#pragma unroll
  for (int a = 1; a < D; ++a) s2 += dx[a] * dx[a];
  const double nrm = sqrt(s2);
  if (nrm > cap) {
    const double f = cap / nrm;
#pragma unroll
    for (int a = 0; a < D; ++a) dx[a] *= f;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) pos[i * D + a] = np_remainder(pos[i * D + a] + dx[a], box[a]);
}

}  // namespace

extern "C" int sphb_relax_accel(const sphb_grid* g, int64_t n, const double* ws,
                                const int32_t* perm, const int32_t* cs, const int32_t* ce,
                                const double* vols, const sphb_kernel* k, double p0, double rho0,
                                double* acc, double* sums, void* stream) {
  if (!g || !k || n < 0 || g->dim != k->dim) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_CUDA_CHECK(cudaMemsetAsync(sums, 0, 2 * sizeof(double), st));
  if (n == 0) return SPHB_OK;
  const int T = 128;
  switch (g->dim) {
    case 1: k_relax_accel<1><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, perm, cs, ce, vols, *k, p0, rho0, acc, sums); break;
    case 2: k_relax_accel<2><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, perm, cs, ce, vols, *k, p0, rho0, acc, sums); break;
    case 3: k_relax_accel<3><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, perm, cs, ce, vols, *k, p0, rho0, acc, sums); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_relax_update(int64_t n, int32_t dim, const double* acc, double dt2, double cap,
                                 const double* box3, double* pos, void* stream) {
  if (n < 0 || !box3) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 256;
  switch (dim) {
    case 1: k_relax_update<1><<<sphb_blocks(n, T), T, 0, st>>>(n, acc, dt2, cap, box3[0], box3[1], box3[2], pos); break;
    case 2: k_relax_update<2><<<sphb_blocks(n, T), T, 0, st>>>(n, acc, dt2, cap, box3[0], box3[1], box3[2], pos); break;
    case 3: k_relax_update<3><<<sphb_blocks(n, T), T, 0, st>>>(n, acc, dt2, cap, box3[0], box3[1], box3[2], pos); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
