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

// Warp-per-particle variant for small sets (C1: 10k particles would fill
// half the SMs with one warp each).  The 32 lanes take consecutive
// candidates of the stencil walk (same order as for_each_neighbor: stencil
// offsets with axis 0 fastest, ascending index inside a cell) and evaluate
// the expensive per-pair terms in parallel; the terms are then added into
// the row sum strictly in candidate order (ballot + shuffles), so the sums
// round exactly as the thread-per-particle kernel and the reference's CSR
// loop do.
template <int D>
__global__ void __launch_bounds__(512)
k_relax_accel_warp(sphb_grid g, int64_t n, const double* __restrict__ ws,
                   const int32_t* __restrict__ perm, const int32_t* __restrict__ cs,
                   const int32_t* __restrict__ ce, const double* __restrict__ vols,
                   sphb_kernel k, double p0, double rho0, double* __restrict__ acc,
                   double* __restrict__ sums) {
  constexpr int noff = D == 1 ? 3 : (D == 2 ? 9 : 27);
  const int lane = threadIdx.x & 31;
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double norm = 0.0, isolated = 0.0;
  if (s < n) {
    double wi[D];
    int64_t ci[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      wi[a] = ws[(int64_t)a * n + s];
      ci[a] = cell_coord(g, a, wi[a]);
    }
    const double scale = k.alpha / k.h;
    double a_[D];
#pragma unroll
    for (int a = 0; a < D; ++a) a_[a] = 0.0;
    int32_t count = 0;
    // stencil cells, 32 at a time (one per lane), in the reference's order
    for (int kb = 0; kb < noff; kb += 32) {
      const int kc = kb + lane;
      int32_t t0 = 0, len = 0;
      if (kc < noff) {
        int rem = kc;
        int64_t flat = 0;
        bool ok = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const int off = rem % 3 - 1;
          rem /= 3;
          int64_t c = ci[a] + off;               // off in {-1, 0, 1}: wrap without a division
          if (g.periodic) c = c < 0 ? c + g.ncell[a] : (c >= g.ncell[a] ? c - g.ncell[a] : c);
          else if (c < 0 || c >= g.ncell[a]) ok = false;
          flat += c * g.strides[a];
        }
        if (ok) {
          t0 = cs[flat];
          len = ce[flat] - t0;
        }
      }
      // exclusive prefix of the cell lengths over the lanes
      int32_t start = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, start, o);
        if (lane >= o) start += v;
      }
      const int32_t total = __shfl_sync(0xffffffffu, start, 31);
      start -= len;
      const int ncell_here = noff - kb < 32 ? noff - kb : 32;
      for (int32_t cb = 0; cb < total; cb += 32) {
        const int32_t c = cb + lane;
        // candidate c lives in the last cell whose start <= c
        int32_t t = -1;
        for (int q = 0; q < ncell_here; ++q) {
          const int32_t sq = __shfl_sync(0xffffffffu, start, q);
          const int32_t lq = __shfl_sync(0xffffffffu, len, q);
          const int32_t tq = __shfl_sync(0xffffffffu, t0, q);
          if (c >= sq && c < sq + lq) t = tq + (c - sq);
        }
        double term[D];
        bool valid = false, in_cut = false;
        if (t >= 0 && t != s) {
          double dx[D];
          double r2 = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            dx[a] = min_image(__dsub_rn(wi[a], ws[(int64_t)a * n + t]), g.box[a], g.periodic);
            r2 = __dadd_rn(r2, __dmul_rn(dx[a], dx[a]));
          }
          if (r2 <= g.cut2 && r2 > 0.0) {
            in_cut = true;
            const double r = sqrt(r2);
            const double q = r / k.h;
            if (!(q > k.kappa)) {
              valid = true;
              const double coeff =
                  -2.0 * p0 * vols[perm[t]] * scale * profile_deriv(k.code, q) / rho0;
#pragma unroll
              for (int a = 0; a < D; ++a) term[a] = coeff * (dx[a] / r);
            }
          }
        }
        count += __popc(__ballot_sync(0xffffffffu, in_cut));
        unsigned m = __ballot_sync(0xffffffffu, valid);
        while (m) {                      // candidate order = lane order (the reference's sum)
          const int src = __ffs(m) - 1;
          m &= m - 1;
#pragma unroll
          for (int a = 0; a < D; ++a) a_[a] += __shfl_sync(0xffffffffu, term[a], src);
        }
      }
    }
    if (lane == 0) {
      const int64_t i = perm[s];
#pragma unroll
      for (int a = 0; a < D; ++a) acc[i * D + a] = a_[a];
      double s2 = a_[0] * a_[0];
#pragma unroll
      for (int a = 1; a < D; ++a) s2 += a_[a] * a_[a];
      norm = sqrt(s2);
      isolated = count == 0 ? 1.0 : 0.0;
    }
  }
  // one particle per warp: the per-particle values sit in lane 0 of each warp
  __shared__ double red[2][16];
  if (lane == 0) {
    red[0][threadIdx.x >> 5] = norm;
    red[1][threadIdx.x >> 5] = isolated;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    atomicAdd(sums, a);
    if (b != 0.0) atomicAdd(sums + 1, b);
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

// sets up to this size run warp-per-particle (the GPU has 148 SMs x 64 warps)
constexpr int64_t kWarpPerParticleMax = 1 << 17;

}  // namespace

extern "C" int sphb_relax_accel(const sphb_grid* g, int64_t n, const double* ws,
                                const int32_t* perm, const int32_t* cs, const int32_t* ce,
                                const double* vols, const sphb_kernel* k, double p0, double rho0,
                                double* acc, double* sums, void* stream) {
  if (!g || !k || n < 0 || g->dim != k->dim) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_CUDA_CHECK(cudaMemsetAsync(sums, 0, 2 * sizeof(double), st));
  if (n == 0) return SPHB_OK;
  if (n <= kWarpPerParticleMax) {   // small sets: one warp per particle
    const int TW = 512;
    const unsigned grid = (unsigned)((n * 32 + TW - 1) / TW);
    switch (g->dim) {
      case 1: k_relax_accel_warp<1><<<grid, TW, 0, st>>>(*g, n, ws, perm, cs, ce, vols, *k, p0, rho0, acc, sums); break;
      case 2: k_relax_accel_warp<2><<<grid, TW, 0, st>>>(*g, n, ws, perm, cs, ce, vols, *k, p0, rho0, acc, sums); break;
      case 3: k_relax_accel_warp<3><<<grid, TW, 0, st>>>(*g, n, ws, perm, cs, ce, vols, *k, p0, rho0, acc, sums); break;
      default: return SPHB_ERR_ARG;
    }
    SPHB_LAUNCH_CHECK();
    return SPHB_OK;
  }
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
