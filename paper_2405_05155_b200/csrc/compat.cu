// compat.cu — operator passes over a device CSR in the reference's order.
//
// These are the drop-in operators behind the reference's Python functions
// (sph_unity_sum, relax_accelerations, moment_matrices, correction_matrices,
// pair_gradients, the WC flux and the two TL-SPH loops).  One thread owns
// one CSR row and walks it in order, and this translation unit is compiled
// with --fmad=false, so each row's arithmetic is performed in the same order
// and with the same roundings as the reference's numba loop.  The engines
// (wc_engine.cu, tl_engine.cu) are the fused, FMA-enabled hot path; these
// kernels back the generic API and the parity tests.
#include "common.cuh"

using namespace sphb;

namespace {

__global__ void k_unity_sums(int64_t n, const int64_t* __restrict__ starts,
                             const int32_t* __restrict__ idx, const double* __restrict__ r,
                             const double* __restrict__ vols, sphb_kernel k,
                             double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // approx.py:41-52
  double acc = k.alpha * profile(k.code, 0.0) * vols[i];
  for (int64_t p = starts[i]; p < starts[i + 1]; ++p) {
    double q = r[p] / k.h;
    if (q <= k.kappa) acc += k.alpha * profile(k.code, q) * vols[idx[p]];
  }
  out[i] = acc;
}

template <int D>
__global__ void k_pressure_accel(int64_t n, const int64_t* __restrict__ starts,
                                 const int32_t* __restrict__ idx, const double* __restrict__ r,
                                 const double* __restrict__ e, const double* __restrict__ vols,
                                 sphb_kernel k, double p0, double rho0,
                                 double* __restrict__ acc) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // relaxation.py:66-80
  const double scale = k.alpha / k.h;
  double a_[D];
#pragma unroll
  for (int a = 0; a < D; ++a) a_[a] = 0.0;
  for (int64_t p = starts[i]; p < starts[i + 1]; ++p) {
    double q = r[p] / k.h;
    if (q > k.kappa) continue;
    double coeff = -2.0 * p0 * vols[idx[p]] * scale * profile_deriv(k.code, q) / rho0;
#pragma unroll
    for (int a = 0; a < D; ++a) a_[a] += coeff * e[p * D + a];
  }
#pragma unroll
  for (int a = 0; a < D; ++a) acc[i * D + a] = a_[a];
}

template <int D>
__global__ void k_moment_matrices(int64_t n, const int64_t* __restrict__ starts,
                                  const int32_t* __restrict__ idx, const double* __restrict__ r,
                                  const double* __restrict__ e, const double* __restrict__ vols,
                                  sphb_kernel k, double* __restrict__ m) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // correction.py:35-52
  const double scale = k.alpha / k.h;
  double mm[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) mm[a][b] = 0.0;
  for (int64_t p = starts[i]; p < starts[i + 1]; ++p) {
    int32_t j = idx[p];
    double q = r[p] / k.h;
    if (q > k.kappa) continue;
    double dw = scale * profile_deriv(k.code, q);
    double w = dw * vols[j] * r[p];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) mm[a][b] += w * e[p * D + a] * e[p * D + b];
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) m[(i * D + a) * D + b] = mm[a][b];
}

// ---------------------------------------------------------------- SVD
// One-sided (Hestenes) Jacobi SVD of a DxD matrix: A V = U S.
template <int D>
__device__ void jacobi_svd(const double (&A)[D][D], double (&U)[D][D], double (&S)[D],
                           double (&V)[D][D]) {
  double W[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      W[a][b] = A[a][b];
      V[a][b] = a == b ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rotated = false;
    for (int pcol = 0; pcol < D - 1; ++pcol) {
      for (int qcol = pcol + 1; qcol < D; ++qcol) {
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          al += W[a][pcol] * W[a][pcol];
          be += W[a][qcol] * W[a][qcol];
          ga += W[a][pcol] * W[a][qcol];
        }
        if (ga == 0.0 || fabs(ga) <= 1e-17 * sqrt(al * be)) continue;
        rotated = true;
        double zeta = (be - al) / (2.0 * ga);
        double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = c * t;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double wp = W[a][pcol], wq = W[a][qcol];
          W[a][pcol] = c * wp - s * wq;
          W[a][qcol] = s * wp + c * wq;
          double vp = V[a][pcol], vq = V[a][qcol];
          V[a][pcol] = c * vp - s * vq;
          V[a][qcol] = s * vp + c * vq;
        }
      }
    }
    if (!rotated) break;
  }
#pragma unroll
  for (int b = 0; b < D; ++b) {
    double nrm = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) nrm += W[a][b] * W[a][b];
    nrm = sqrt(nrm);
    S[b] = nrm;
#pragma unroll
    for (int a = 0; a < D; ++a) U[a][b] = nrm > 0.0 ? W[a][b] / nrm : (a == b ? 1.0 : 0.0);
  }
}

template <int D>
__device__ double det_small(const double (&A)[D][D]) {
  if constexpr (D == 1) {
    return A[0][0];
  } else if constexpr (D == 2) {
    return A[0][0] * A[1][1] - A[0][1] * A[1][0];
  } else {
    return A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) -
           A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
           A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
  }
}

template <int D>
__global__ void k_correction(int64_t n, const double* __restrict__ m, double* __restrict__ b,
                             double* __restrict__ det_neg, int8_t* __restrict__ reg) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // correction.py:64-81
  double A[D][D], NA[D][D], U[D][D], V[D][D], S[D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      A[a][c] = m[(i * D + a) * D + c];
      NA[a][c] = -A[a][c];
    }
  jacobi_svd<D>(A, U, S, V);
  double smax = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) smax = S[a] > smax ? S[a] : smax;
  const double floor_ = kEpsSV * fmax(smax, 1e-300);
  bool clamped = false;
  double inv_s[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (S[a] < floor_) clamped = true;
    inv_s[a] = 1.0 / fmax(S[a], floor_);
  }
  const double dn = det_small<D>(NA);
  double theta = dn / kEpsDet;
  theta = theta < 0.0 ? 0.0 : (theta > 1.0 ? 1.0 : theta);
  // minv = V diag(1/s) U^T ; B = theta (-minv) + (1 - theta) I
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double mv = 0.0;
#pragma unroll
      for (int q = 0; q < D; ++q) mv += V[a][q] * inv_s[q] * U[c][q];
      b[(i * D + a) * D + c] = theta * (-mv) + (1.0 - theta) * (a == c ? 1.0 : 0.0);
    }
  det_neg[i] = dn;
  reg[i] = (clamped || theta < 1.0) ? 1 : 0;
}

template <int D>
__global__ void k_pair_gradients(int64_t n, const int64_t* __restrict__ starts,
                                 const int32_t* __restrict__ idx, const double* __restrict__ r,
                                 const double* __restrict__ e, sphb_kernel k,
                                 const double* __restrict__ b, double* __restrict__ gw) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // correction.py:89-112
  const double scale = k.alpha / k.h;
  for (int64_t p = starts[i]; p < starts[i + 1]; ++p) {
    int32_t j = idx[p];
    double q = r[p] / k.h;
    if (q > k.kappa) {
#pragma unroll
      for (int a = 0; a < D; ++a) gw[p * D + a] = 0.0;
      continue;
    }
    double dw = scale * profile_deriv(k.code, q);
    if (b) {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c)
          acc += 0.5 * (b[((int64_t)i * D + a) * D + c] + b[((int64_t)j * D + a) * D + c]) *
                 e[p * D + c];
        gw[p * D + a] = dw * acc;
      }
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) gw[p * D + a] = dw * e[p * D + a];
    }
  }
}

template <int D>
__global__ void k_rhs_wc(int64_t n_int, const int64_t* __restrict__ starts,
                         const int32_t* __restrict__ idx, const double* __restrict__ e,
                         const double* __restrict__ gwv, const double* __restrict__ viscv,
                         const double* __restrict__ rho, const double* __restrict__ v,
                         const double* __restrict__ p, double c_art, double mu,
                         const int8_t* __restrict__ wall_tag, double* __restrict__ drho,
                         double* __restrict__ dmom, double* __restrict__ wf) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_int) return;
  // eulerian.py:224-266
  const double rho_i = rho[i];
  const double p_i = p[i];
  double vi[D], dm[D], wfi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    vi[a] = v[i * D + a];
    dm[a] = dmom[i * D + a];
    wfi[a] = 0.0;
  }
  double dr = 0.0;
  for (int64_t q = starts[i]; q < starts[i + 1]; ++q) {
    const int32_t j = idx[q];
    double ul = 0.0, ur = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      ul += vi[a] * (-e[q * D + a]);
      ur += v[(int64_t)j * D + a] * (-e[q * D + a]);
    }
    const double du = ul - ur;
    double beta = kEtaLinearized * du / c_art;
    if (beta < 0.0) beta = 0.0;
    else if (beta > 1.0) beta = 1.0;
    const double rbar = 0.5 * (rho_i + rho[j]);
    const double u_star = 0.5 * (ul + ur) + 0.5 * beta * beta * (p_i - p[j]) / (rbar * c_art);
    const double p_star = 0.5 * (p_i + p[j]) + 0.5 * beta * rbar * c_art * du;
    const double ubar = 0.5 * (ul + ur);
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double vs = u_star * (-e[q * D + a]) + 0.5 * (vi[a] + v[(int64_t)j * D + a]) -
                  ubar * (-e[q * D + a]);
      s += vs * gwv[q * D + a];
    }
    dr += -2.0 * rbar * s;
    const bool tagged = wall_tag && wall_tag[j] != 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double vja = v[(int64_t)j * D + a];
      double vs = u_star * (-e[q * D + a]) + 0.5 * (vi[a] + vja) - ubar * (-e[q * D + a]);
      double fm = -2.0 * (rbar * vs * s + p_star * gwv[q * D + a]) + mu * viscv[q] * (vi[a] - vja);
      dm[a] += fm;
      if (tagged) wfi[a] -= fm;
    }
  }
  drho[i] = dr;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    dmom[i * D + a] = dm[a];
    if (wf) wf[i * D + a] = wfi[a];
  }
}

template <int D>
__global__ void k_tl_acc(int64_t n, const int64_t* __restrict__ starts,
                         const int32_t* __restrict__ idx, const double* __restrict__ g0,
                         const double* __restrict__ q, double rho0, double* __restrict__ acc) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // tlsph.py:88-102
  double out[D];
#pragma unroll
  for (int a = 0; a < D; ++a) out[a] = 0.0;
  for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
    const int64_t j = idx[k];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double t = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b)
        t += (q[(i * D + a) * D + b] + q[(j * D + a) * D + b]) * g0[k * D + b];
      out[a] += t / rho0;
    }
  }
#pragma unroll
  for (int a = 0; a < D; ++a) acc[i * D + a] = out[a];
}

template <int D>
__global__ void k_tl_dF(int64_t n, const int64_t* __restrict__ starts,
                        const int32_t* __restrict__ idx, const double* __restrict__ g0,
                        const double* __restrict__ v, const double* __restrict__ b0,
                        double* __restrict__ dF) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // tlsph.py:105-123
  double m[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) m[a][b] = 0.0;
  for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
    const int64_t j = idx[k];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double dv = v[j * D + a] - v[i * D + a];
#pragma unroll
      for (int b = 0; b < D; ++b) m[a][b] += dv * g0[k * D + b];
    }
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) t += m[a][c] * b0[(i * D + c) * D + b];
      dF[(i * D + a) * D + b] = t;
    }
}

// Moment matrices straight from the engine's ELL list (sorted order), with
// exact geometry (r = sqrt(r2), e = dx / r) so each row's sum equals the
// CSR-based _moment_matrices row bit for bit without materialising r and e.
template <int D>
__global__ void k_ell_moments(sphb_grid g, int64_t n, const double* __restrict__ ws,
                              const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                              const double* __restrict__ vols, sphb_kernel k,
                              double* __restrict__ m) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double scale = k.alpha / k.h;
  double wi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) wi[a] = ws[(int64_t)a * n + s];
  double mm[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) mm[a][b] = 0.0;
  const int32_t c = cnt[s];
  for (int32_t kk = 0; kk < c; ++kk) {
    const int64_t t = nbr[(int64_t)kk * n + s];
    double dx[D];
    double r2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      dx[a] = min_image(wi[a] - ws[(int64_t)a * n + t], g.box[a], g.periodic);
      r2 += dx[a] * dx[a];
    }
    const double r = sqrt(r2);
    double e[D];
#pragma unroll
    for (int a = 0; a < D; ++a) e[a] = dx[a] / r;
    const double q = r / k.h;
    const double dw = scale * profile_deriv(k.code, q);
    const double w = dw * vols[t] * r;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) mm[a][b] += w * e[a] * e[b];
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) m[(s * D + a) * D + b] = mm[a][b];
}

// Per-pair geometry of the WC flux, exactly as the reference precomputes it
// in EulerianSolver.__init__ (eulerian.py:506-513 via _pair_gradients,
// correction.py:89-112): e_ij, gwv_ij = dW 0.5 (B_i + B_j) e_ij V_j and
// viscv_ij = 2 dW / r V_j, for every slot of the ELL pass list, stored as
// planes geo[(c * width + k) * n + s] (c < D: e, D..2D-1: gwv, 2D: viscv) so
// the stage kernel streams them coalesced.  B is the full (unsymmetrised)
// sorted correction matrix; no FMA contraction (this translation unit).
template <int D>
__global__ void k_wc_geometry(sphb_grid g, int64_t n, const double* __restrict__ ws,
                              const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                              int32_t width, const double* __restrict__ b,
                              const double* __restrict__ vol, sphb_kernel k,
                              double* __restrict__ geo) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double scale = k.alpha / k.h;
  double wi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) wi[a] = ws[(int64_t)a * n + s];
  const int32_t m = cnt[s];
  for (int32_t kk = 0; kk < m; ++kk) {
    const int64_t t = nbr[(int64_t)kk * n + s];
    double dx[D];
    double r2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      dx[a] = min_image(wi[a] - ws[(int64_t)a * n + t], g.box[a], g.periodic);
      r2 += dx[a] * dx[a];
    }
    const double r = sqrt(r2);
    double e[D];
#pragma unroll
    for (int a = 0; a < D; ++a) e[a] = dx[a] / r;
    const double q = r / k.h;
    const double dw = scale * profile_deriv(k.code, q);
    const double vj = vol[t];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c)
        acc += 0.5 * (b[(s * D + a) * D + c] + b[(t * D + a) * D + c]) * e[c];
      geo[((int64_t)a * width + kk) * n + s] = e[a];
      geo[((int64_t)(D + a) * width + kk) * n + s] = dw * acc * vj;
    }
    geo[((int64_t)(2 * D) * width + kk) * n + s] = 2.0 * dw / r * vj;
  }
}

// Reference-configuration gradients of SolidSystem (tlsph.py:145-146:
// g0 = pair_gradients(nlist0, kernel, None) * V0, correction.py:110-111) per
// slot of the ELL pass list, as planes g0[(c * width + k) * n + s];
// reference arithmetic (no FMA in this unit).
template <int D>
__global__ void k_tl_geometry(sphb_grid g, int64_t n, const double* __restrict__ ws,
                              const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                              int32_t width, sphb_kernel k, double vol0,
                              double* __restrict__ g0) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double scale = k.alpha / k.h;
  double wi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) wi[a] = ws[(int64_t)a * n + s];
  const int32_t m = cnt[s];
  for (int32_t kk = 0; kk < m; ++kk) {
    const int64_t t = nbr[(int64_t)kk * n + s];
    double dx[D];
    double r2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      dx[a] = min_image(wi[a] - ws[(int64_t)a * n + t], g.box[a], g.periodic);
      r2 += dx[a] * dx[a];
    }
    const double r = sqrt(r2);
    const double dw = scale * profile_deriv(k.code, r / k.h);
#pragma unroll
    for (int a = 0; a < D; ++a) g0[((int64_t)a * width + kk) * n + s] = dw * (dx[a] / r) * vol0;
  }
}

// _weak_gradient (approx.py:61-71): 2 sum_j 0.5 (f_i + f_j) V_j gw_ij, CSR rows.
template <int D>
__global__ void k_weak_gradient(int64_t n, const int64_t* __restrict__ starts,
                                const int32_t* __restrict__ idx, const double* __restrict__ f,
                                const double* __restrict__ vols, const double* __restrict__ gw,
                                double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double o[D];
#pragma unroll
  for (int a = 0; a < D; ++a) o[a] = 0.0;
  for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
    const int32_t j = idx[k];
    const double fbar_v = 0.5 * (f[i] + f[j]) * vols[j];
#pragma unroll
    for (int a = 0; a < D; ++a) o[a] += 2.0 * fbar_v * gw[k * D + a];
  }
#pragma unroll
  for (int a = 0; a < D; ++a) out[i * D + a] = o[a];
}

}  // namespace

#define SPHB_DISPATCH_D(dim, KERNEL, GRID, ...)                                   \
  do {                                                                            \
    switch (dim) {                                                                \
      case 1: KERNEL<1><<<GRID, T, 0, st>>>(__VA_ARGS__); break;                  \
      case 2: KERNEL<2><<<GRID, T, 0, st>>>(__VA_ARGS__); break;                  \
      case 3: KERNEL<3><<<GRID, T, 0, st>>>(__VA_ARGS__); break;                  \
      default: return SPHB_ERR_ARG;                                               \
    }                                                                             \
  } while (0)

extern "C" int sphb_weak_gradient(int64_t n, int32_t dim, const int64_t* starts,
                                  const int32_t* idx, const double* f, const double* vols,
                                  const double* gw, double* out, void* stream) {
  if (n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(dim, k_weak_gradient, sphb_blocks(n, T), n, starts, idx, f, vols, gw, out);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_unity_sums(int64_t n, const int64_t* starts, const int32_t* idx,
                               const double* r, const double* vols, const sphb_kernel* k,
                               double* out, void* stream) {
  if (n < 0 || !k) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  k_unity_sums<<<sphb_blocks(n, T), T, 0, st>>>(n, starts, idx, r, vols, *k, out);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_pressure_accel(int64_t n, int32_t dim, const int64_t* starts,
                                   const int32_t* idx, const double* r, const double* e,
                                   const double* vols, const sphb_kernel* k, double p0,
                                   double rho0, double* acc, void* stream) {
  if (n < 0 || !k) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(dim, k_pressure_accel, sphb_blocks(n, T), n, starts, idx, r, e, vols, *k, p0,
                  rho0, acc);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_moment_matrices(int64_t n, int32_t dim, const int64_t* starts,
                                    const int32_t* idx, const double* r, const double* e,
                                    const double* vols, const sphb_kernel* k, double* m,
                                    void* stream) {
  if (n < 0 || !k) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(dim, k_moment_matrices, sphb_blocks(n, T), n, starts, idx, r, e, vols, *k, m);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_correction_from_moments(int64_t n, int32_t dim, const double* m, double* b,
                                            double* det_neg_m, int8_t* reg, void* stream) {
  if (n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(dim, k_correction, sphb_blocks(n, T), n, m, b, det_neg_m, reg);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_pair_gradients(int64_t n, int32_t dim, const int64_t* starts,
                                   const int32_t* idx, const double* r, const double* e,
                                   const sphb_kernel* k, const double* b, double* gw,
                                   void* stream) {
  if (n < 0 || !k) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(dim, k_pair_gradients, sphb_blocks(n, T), n, starts, idx, r, e, *k, b, gw);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_rhs_wc_csr(int64_t n_int, int32_t dim, const int64_t* starts,
                               const int32_t* idx, const double* e, const double* gwv,
                               const double* viscv, const double* rho, const double* v,
                               const double* p, double c_art, double mu,
                               const int8_t* wall_tag, double* drho, double* dmom,
                               double* wall_force_partial, void* stream) {
  if (n_int < 0) return SPHB_ERR_ARG;
  if (n_int == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(dim, k_rhs_wc, sphb_blocks(n_int, T), n_int, starts, idx, e, gwv, viscv, rho,
                  v, p, c_art, mu, wall_tag, drho, dmom, wall_force_partial);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_tl_accelerations_csr(int64_t n, int32_t dim, const int64_t* starts,
                                         const int32_t* idx, const double* g0, const double* q,
                                         double rho0, double* acc, void* stream) {
  if (n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(dim, k_tl_acc, sphb_blocks(n, T), n, starts, idx, g0, q, rho0, acc);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_tl_deformation_rates_csr(int64_t n, int32_t dim, const int64_t* starts,
                                             const int32_t* idx, const double* g0,
                                             const double* v, const double* b0, double* dF,
                                             void* stream) {
  if (n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(dim, k_tl_dF, sphb_blocks(n, T), n, starts, idx, g0, v, b0, dF);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_ell_moments(const sphb_grid* g, int64_t n, const double* ws,
                                const int32_t* nbr, const int32_t* cnt, const double* vols,
                                const sphb_kernel* k, double* m, void* stream) {
  if (!g || !k || n < 0 || g->dim != k->dim) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(g->dim, k_ell_moments, sphb_blocks(n, T), *g, n, ws, nbr, cnt, vols, *k, m);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_wc_geometry(const sphb_grid* g, int64_t n, const double* ws,
                                const int32_t* nbr, const int32_t* cnt, int32_t width,
                                const double* b, const double* vol, const sphb_kernel* k,
                                double* geo, void* stream) {
  if (!g || !k || n < 0 || width < 0) return SPHB_ERR_ARG;
  if (n == 0 || width == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(g->dim, k_wc_geometry, sphb_blocks(n, T), *g, n, ws, nbr, cnt, width, b, vol,
                  *k, geo);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_tl_geometry(const sphb_grid* g, int64_t n, const double* ws,
                                const int32_t* nbr, const int32_t* cnt, int32_t width,
                                const sphb_kernel* k, double vol0, double* g0, void* stream) {
  if (!g || !k || n < 0 || width < 0) return SPHB_ERR_ARG;
  if (n == 0 || width == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  SPHB_DISPATCH_D(g->dim, k_tl_geometry, sphb_blocks(n, T), *g, n, ws, nbr, cnt, width, *k,
                  vol0, g0);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
