// wc_engine.cu — fused weakly-compressible Eulerian stage kernels.
//
// One launch per midpoint stage of EulerianSolver._substep
// (eulerian.py:610-643).  Each thread owns one particle (cell-sorted order),
// walks its ELL row (the reference CSR row minus the pairs the passes skip)
// and, per pair, recomputes what the reference precomputes and streams:
//   r, e_ij                         (neighbors.py:161-165)
//   grad'W_ij V_j = dW 0.5(B_i+B_j) e_ij V_j   (correction.py:102-108,
//                                    eulerian.py:506-507)
//   viscv = 2 dW / r V_j             (eulerian.py:509-513)
// then evaluates the limited linearised Riemann flux (eulerian.py:145-157,
// 224-266), accumulates d(rho)/dt and d(mom)/dt in registers, and applies the
// stage update (eulerian.py:619-629) in the epilogue.  Stage 2 also folds
// max(c + |v|) into a device scalar so the next dt (compute_dt,
// eulerian.py:553-560) never leaves the GPU.
//
// Particle data (sorted SoA-of-vectors, one 32-byte record per particle):
//   X[i]  = {x0, x1, x2, vol}   (static; 2D: {x0, x1, vol, 0})
//   B[i]  = 2 x double4 {b00, b01, b02, b11 | b12, b22, -, -} (symmetrised)
//           2D: {b00, b01, b11, -}; 1D: {b00, ...}
//   S[i]  = {v0, v1, v2, rho}   (primitive state; 2D: {v0, v1, rho, 0})
//   M[i]  = {m0, m1, m2, 0}     (momentum per unit volume)
#include "common.cuh"

using namespace sphb;

namespace {

constexpr int kThreads = 128;

template <int D>
struct Sym;  // symmetric DxD matrix in packed storage
template <>
struct Sym<1> {
  double a00;
  __device__ __forceinline__ void load(const double4* B, int64_t i) { a00 = B[2 * i].x; }
  __device__ __forceinline__ void add(const Sym& o, Sym& r) const { r.a00 = a00 + o.a00; }
  __device__ __forceinline__ void mv(const double (&e)[1], double (&out)[1]) const {
    out[0] = a00 * e[0];
  }
};
template <>
struct Sym<2> {
  double a00, a01, a11;
  __device__ __forceinline__ void load(const double4* B, int64_t i) {
    double4 t = B[2 * i];
    a00 = t.x; a01 = t.y; a11 = t.z;
  }
  __device__ __forceinline__ void add(const Sym& o, Sym& r) const {
    r.a00 = a00 + o.a00; r.a01 = a01 + o.a01; r.a11 = a11 + o.a11;
  }
  __device__ __forceinline__ void mv(const double (&e)[2], double (&out)[2]) const {
    out[0] = fma(a00, e[0], a01 * e[1]);
    out[1] = fma(a01, e[0], a11 * e[1]);
  }
};
template <>
struct Sym<3> {
  double a00, a01, a02, a11, a12, a22;
  __device__ __forceinline__ void load(const double4* B, int64_t i) {
    double4 t = B[2 * i];
    double4 u = B[2 * i + 1];
    a00 = t.x; a01 = t.y; a02 = t.z; a11 = t.w; a12 = u.x; a22 = u.y;
  }
  __device__ __forceinline__ void add(const Sym& o, Sym& r) const {
    r.a00 = a00 + o.a00; r.a01 = a01 + o.a01; r.a02 = a02 + o.a02;
    r.a11 = a11 + o.a11; r.a12 = a12 + o.a12; r.a22 = a22 + o.a22;
  }
  __device__ __forceinline__ void mv(const double (&e)[3], double (&out)[3]) const {
    out[0] = fma(a00, e[0], fma(a01, e[1], a02 * e[2]));
    out[1] = fma(a01, e[0], fma(a11, e[1], a12 * e[2]));
    out[2] = fma(a02, e[0], fma(a12, e[1], a22 * e[2]));
  }
};

template <int D>
__device__ __forceinline__ void unpack_x(const double4& t, double (&x)[D], double& vol) {
  const double c[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int a = 0; a < D; ++a) x[a] = c[a];
  vol = c[D];
}

template <int D>
__device__ __forceinline__ void unpack_s(const double4& t, double (&v)[D], double& rho) {
  const double c[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int a = 0; a < D; ++a) v[a] = c[a];
  rho = c[D];
}

template <int D>
__device__ __forceinline__ double4 pack_s(const double (&v)[D], double rho) {
  double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = v[a];
  c[D] = rho;
  return make_double4(c[0], c[1], c[2], c[3]);
}

template <int D>
__device__ __forceinline__ double norm_exact(const double (&v)[D]) {
  // np.linalg.norm over a row: sqrt(((v0*v0) + v1*v1) + v2*v2)
  double s = __dmul_rn(v[0], v[0]);
#pragma unroll
  for (int a = 1; a < D; ++a) s = __dadd_rn(s, __dmul_rn(v[a], v[a]));
  return __dsqrt_rn(s);
}

template <int D>
__global__ void __launch_bounds__(kThreads)
k_wc_stage(const sphb_wc_params P, const int stage, const double4* __restrict__ X,
           const double4* __restrict__ B, const int32_t* __restrict__ nbr,
           const int32_t* __restrict__ cnt, const double4* __restrict__ S_in,
           const double4* Sn, const double4* Mn, double4* S_out, double4* M_out,
           double* __restrict__ scalars, int32_t* __restrict__ err) {
  const int64_t n = P.n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double speed = 0.0;
  int32_t flags = 0;
  if (i < n) {
    const double c = P.c_art;
    const double c2 = c * c;
    const double eta_c = kEtaLinearized / c;
    const double inv_h = 1.0 / P.h;
    const double scale = P.alpha / P.h;
    const double half_cinv = 0.5 / c;

    double xi[D], vol_i, vi[D], rho_i;
    unpack_x<D>(X[i], xi, vol_i);
    unpack_s<D>(S_in[i], vi, rho_i);
    Sym<D> Bi;
    Bi.load(B, i);
    const double p_i = c2 * (rho_i - P.rho0);

    double dr = 0.0;
    double dm[D];
#pragma unroll
    for (int a = 0; a < D; ++a) dm[a] = 0.0;

    const int32_t m = cnt[i];
    const int32_t* __restrict__ row = nbr + i;
    for (int32_t k = 0; k < m; ++k) {
      const int64_t j = row[(int64_t)k * n];
      double xj[D], vol_j, vj[D], rho_j;
      unpack_x<D>(X[j], xj, vol_j);
      unpack_s<D>(S_in[j], vj, rho_j);
      Sym<D> Bj;
      Bj.load(B, j);
      if (P.uniform_vol) vol_j = P.vol_const;

      // geometry
      double dx[D];
      double r2 = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double d = xi[a] - xj[a];
        if (P.periodic) {
          const double bx = P.box[a];
          if (d > 0.5 * bx) d -= bx;
          else if (d < -0.5 * bx) d += bx;
        }
        dx[a] = d;
        r2 = fma(d, d, r2);
      }
      const double inv_r = rsqrt(r2);
      const double r = r2 * inv_r;
      const double q = r * inv_h;
      const double t = fma(-0.5, q, 1.0);
      const double dW = scale * (-5.0 * q) * (t * t * t);  // (alpha/h) dP/dq
      double e[D];
#pragma unroll
      for (int a = 0; a < D; ++a) e[a] = dx[a] * inv_r;
      Sym<D> Bs;
      Bi.add(Bj, Bs);
      double g[D];
      Bs.mv(e, g);
      const double gs = 0.5 * dW * vol_j;  // 0.5 (B_i + B_j) e dW V_j
#pragma unroll
      for (int a = 0; a < D; ++a) g[a] *= gs;
      const double viscv = 2.0 * dW * inv_r * vol_j;

      // limited linearised Riemann problem along n = -e
      double ul = 0.0, ur = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        ul = fma(-vi[a], e[a], ul);
        ur = fma(-vj[a], e[a], ur);
      }
      const double du = ul - ur;
      double beta = du * eta_c;
      beta = beta < 0.0 ? 0.0 : (beta > 1.0 ? 1.0 : beta);
      const double rbar = 0.5 * (rho_i + rho_j);
      const double p_j = c2 * (rho_j - P.rho0);
      const double ubar = 0.5 * (ul + ur);
      double ustar_m_ubar = 0.0;
      if (beta > 0.0) ustar_m_ubar = (beta * beta) * (p_i - p_j) * half_cinv / rbar;
      const double p_star = fma(0.5 * beta * rbar * c, du, 0.5 * (p_i + p_j));
      (void)ubar;
      double vs[D];
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        vs[a] = fma(-ustar_m_ubar, e[a], 0.5 * (vi[a] + vj[a]));
        s = fma(vs[a], g[a], s);
      }
      dr = fma(-2.0 * rbar, s, dr);
      const double rs = rbar * s;
      const double mv = P.mu * viscv;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double fm = -2.0 * fma(rs, vs[a], p_star * g[a]);
        dm[a] = fma(mv, vi[a] - vj[a], dm[a] + fm);
      }
    }

    // ---------------------------------------------------------- epilogue
    if (stage == 0) {  // rhs only: S_out = {dmom, drho} (EulerianSolver.rhs)
      S_out[i] = pack_s<D>(dm, dr);
      if (!isfinite(dr)) flags |= SPHB_EFLAG_NONFINITE_FLUX;
#pragma unroll
      for (int a = 0; a < D; ++a)
        if (!isfinite(dm[a])) flags |= SPHB_EFLAG_NONFINITE_FLUX;
      if (flags) atomicOr(err, flags);
      return;
    }
    const double dt = scalars[0];
    const double cdt = stage == 1 ? 0.5 * dt : dt;
    double mom_n[D], rho_n;
    {
      const double4 mn = Mn[i];
      const double cm[4] = {mn.x, mn.y, mn.z, mn.w};
#pragma unroll
      for (int a = 0; a < D; ++a) mom_n[a] = cm[a];
      double vtmp[D];
      unpack_s<D>(Sn[i], vtmp, rho_n);
    }
    bool finite = isfinite(dr);
#pragma unroll
    for (int a = 0; a < D; ++a) finite = finite && isfinite(dm[a]);
    if (!finite) flags |= SPHB_EFLAG_NONFINITE_FLUX;
    const double rho_new = fma(cdt, dr, rho_n);
    double mom_new[D], v_new[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      mom_new[a] = fma(cdt, dm[a], mom_n[a]);
      v_new[a] = __ddiv_rn(mom_new[a], rho_new);
    }
    if (!(rho_new > 0.0)) flags |= SPHB_EFLAG_NONPOS_DENSITY;
    S_out[i] = pack_s<D>(v_new, rho_new);
    if (stage == 2) {
      double mc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int a = 0; a < D; ++a) mc[a] = mom_new[a];
      M_out[i] = make_double4(mc[0], mc[1], mc[2], mc[3]);
      speed = __dadd_rn(c, norm_exact<D>(v_new));
    }
  }
  if (stage == 2) {
    __shared__ double red[kThreads / 32];
    double w = warp_max(speed);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = red[0];
#pragma unroll
      for (int q = 1; q < kThreads / 32; ++q) b = b > red[q] ? b : red[q];
      atomic_max_nonneg(scalars + 2, b);
    }
  }
  if (flags) atomicOr(err, flags);
}

template <int D>
__global__ void __launch_bounds__(256)
k_speed_max(int64_t n, double c, const double4* __restrict__ S, double* __restrict__ scalars) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double sp = 0.0;
  if (i < n) {
    double v[D], rho;
    unpack_s<D>(S[i], v, rho);
    sp = __dadd_rn(c, norm_exact<D>(v));
  }
  __shared__ double red[8];
  double w = warp_max(sp);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = red[0];
    for (int q = 1; q < 8; ++q) b = b > red[q] ? b : red[q];
    atomic_max_nonneg(scalars + 2, b);
  }
}


// --------------------------------------------------------- state transfer
// U (caller order, AoS rho (n), mom (n, d)) -> sorted records S = {v, rho},
// M = {mom}; v = mom / rho as FluidState.velocity (eulerian.py:461-462).
template <int D>
__global__ void k_wc_pack(int64_t n, const int32_t* __restrict__ perm,
                          const double* __restrict__ rho, const double* __restrict__ mom,
                          double4* __restrict__ S, double4* __restrict__ M) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t i = perm[s];
  const double r = rho[i];
  double v[D], m[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    m[a] = mom[i * D + a];
    v[a] = __ddiv_rn(m[a], r);
  }
  S[s] = pack_s<D>(v, r);
  double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = m[a];
  M[s] = make_double4(c[0], c[1], c[2], c[3]);
}

template <int D>
__global__ void k_wc_unpack(int64_t n, const int32_t* __restrict__ perm,
                            const double4* __restrict__ S, const double4* __restrict__ M,
                            double* __restrict__ rho, double* __restrict__ mom) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t i = perm[s];
  double v[D], r;
  unpack_s<D>(S[s], v, r);
  rho[i] = r;
  const double4 mm = M[s];
  const double c[4] = {mm.x, mm.y, mm.z, mm.w};
#pragma unroll
  for (int a = 0; a < D; ++a) mom[i * D + a] = c[a];
}

}  // namespace

// dt = dt_override or cfl_h / (c_add + smax)  (eulerian.py:553-560,
// tlsph.py:178-180); t += dt; the speed accumulator is reset for the step.
__global__ void k_set_dt(double cfl_h, double c_add, double dt_override, double* scalars,
                         int32_t* err) {
  double dt = dt_override;
  if (!(dt > 0.0)) {
    const double denom = c_add + scalars[2];
    if (!(denom > 0.0) || !isfinite(denom)) {
      atomicOr(err, SPHB_EFLAG_NONFINITE_STATE);
      dt = 0.0;
    } else {
      dt = cfl_h / denom;
    }
  }
  scalars[0] = dt;
  scalars[1] += dt;
  scalars[2] = 0.0;
}

extern "C" int sphb_wc_stage(const sphb_wc_params* p, int32_t stage, const double* x,
                             const double* b, const int32_t* nbr, const int32_t* cnt,
                             const double* s_in, const double* s_n, const double* m_n,
                             double* s_out, double* m_out, double* scalars, int32_t* err,
                             void* stream) {
  if (!p || p->n < 0 || stage < 0 || stage > 2) return SPHB_ERR_ARG;
  if (p->n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = sphb_blocks(p->n, kThreads);
  const double4* X = (const double4*)x;
  const double4* B = (const double4*)b;
  const double4* Sin = (const double4*)s_in;
  const double4* Sn = (const double4*)s_n;
  const double4* Mn = (const double4*)m_n;
  double4* Sout = (double4*)s_out;
  double4* Mout = (double4*)m_out;
  switch (p->dim) {
    case 1: k_wc_stage<1><<<grid, kThreads, 0, st>>>(*p, stage, X, B, nbr, cnt, Sin, Sn, Mn, Sout, Mout, scalars, err); break;
    case 2: k_wc_stage<2><<<grid, kThreads, 0, st>>>(*p, stage, X, B, nbr, cnt, Sin, Sn, Mn, Sout, Mout, scalars, err); break;
    case 3: k_wc_stage<3><<<grid, kThreads, 0, st>>>(*p, stage, X, B, nbr, cnt, Sin, Sn, Mn, Sout, Mout, scalars, err); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_wc_speed_max(const sphb_wc_params* p, const double* s, double* scalars,
                                 void* stream) {
  if (!p || p->n < 0) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_CUDA_CHECK(cudaMemsetAsync(scalars + 2, 0, sizeof(double), st));
  if (p->n == 0) return SPHB_OK;
  const double4* S = (const double4*)s;
  const unsigned grid = sphb_blocks(p->n, 256);
  switch (p->dim) {
    case 1: k_speed_max<1><<<grid, 256, 0, st>>>(p->n, p->c_art, S, scalars); break;
    case 2: k_speed_max<2><<<grid, 256, 0, st>>>(p->n, p->c_art, S, scalars); break;
    case 3: k_speed_max<3><<<grid, 256, 0, st>>>(p->n, p->c_art, S, scalars); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_set_dt(double cfl_h, double c_add, double dt_override, double* scalars,
                           int32_t* err, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  k_set_dt<<<1, 1, 0, st>>>(cfl_h, c_add, dt_override, scalars, err);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_wc_pack_state(int64_t n, int32_t dim, const int32_t* perm, const double* rho,
                                  const double* mom, double* s, double* m, void* stream) {
  if (n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = sphb_blocks(n, 256);
  switch (dim) {
    case 1: k_wc_pack<1><<<grid, 256, 0, st>>>(n, perm, rho, mom, (double4*)s, (double4*)m); break;
    case 2: k_wc_pack<2><<<grid, 256, 0, st>>>(n, perm, rho, mom, (double4*)s, (double4*)m); break;
    case 3: k_wc_pack<3><<<grid, 256, 0, st>>>(n, perm, rho, mom, (double4*)s, (double4*)m); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_wc_unpack_state(int64_t n, int32_t dim, const int32_t* perm, const double* s,
                                    const double* m, double* rho, double* mom, void* stream) {
  if (n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = sphb_blocks(n, 256);
  switch (dim) {
    case 1: k_wc_unpack<1><<<grid, 256, 0, st>>>(n, perm, (const double4*)s, (const double4*)m, rho, mom); break;
    case 2: k_wc_unpack<2><<<grid, 256, 0, st>>>(n, perm, (const double4*)s, (const double4*)m, rho, mom); break;
    case 3: k_wc_unpack<3><<<grid, 256, 0, st>>>(n, perm, (const double4*)s, (const double4*)m, rho, mom); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
