// tl_common.cuh — record layouts and per-row helpers of the TL-SPH passes,
// shared by the general pass-list kernels (tl_engine.cu) and the lattice
// kernels (tl_lattice.cu).
#pragma once

#include "common.cuh"

namespace sphb {
namespace tl {

// 3x3 records are three row planes M[r * ms + i] (ms = plane stride), so a
// warp's access to one row covers consecutive 32-byte records
template <int D>
__device__ __forceinline__ void load_mat(const double4* __restrict__ M, int64_t ms, int64_t i,
                                         double (&a)[D][D]) {
  if constexpr (D == 3) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double4 t = M[r * ms + i];
      a[r][0] = t.x; a[r][1] = t.y; a[r][2] = t.z;
    }
  } else if constexpr (D == 2) {
    double4 t = M[i];
    a[0][0] = t.x; a[0][1] = t.y; a[1][0] = t.z; a[1][1] = t.w;
  } else {
    a[0][0] = M[i].x;
  }
}

// 3D deformation gradient F: 9 doubles in three planes of n records,
// {F00, F01, F02, F10} {F11, F12, F20, F21} {F22} (72 bytes per particle
// instead of 96 for padded rows); 2D / 1D: the single-record layout.
template <int D>
__device__ __forceinline__ void load_f(const double4* __restrict__ F, int64_t n, int64_t i,
                                       double (&a)[D][D]) {
  if constexpr (D == 3) {
    const double4 p = F[i], q = F[n + i];
    const double r = reinterpret_cast<const double*>(F + 2 * n)[i];
    a[0][0] = p.x; a[0][1] = p.y; a[0][2] = p.z;
    a[1][0] = p.w; a[1][1] = q.x; a[1][2] = q.y;
    a[2][0] = q.z; a[2][1] = q.w; a[2][2] = r;
  } else {
    load_mat<D>(F, n, i, a);
  }
}

template <int D>
__device__ __forceinline__ void store_f(double4* __restrict__ F, int64_t n, int64_t i,
                                        const double (&a)[D][D]);

// 3D correction matrix B0 (symmetric, correction.py:64-81): planes
// {b00, b01, b02, b11} and {b12, b22} (48 bytes per particle).
template <int D>
__device__ __forceinline__ void load_b0(const double4* __restrict__ B, int64_t n, int64_t i,
                                        double (&a)[D][D]) {
  if constexpr (D == 3) {
    const double4 p = B[i];
    const double2 q = reinterpret_cast<const double2*>(B + n)[i];
    a[0][0] = p.x; a[0][1] = p.y; a[0][2] = p.z;
    a[1][0] = p.y; a[1][1] = p.w; a[1][2] = q.x;
    a[2][0] = p.z; a[2][1] = q.x; a[2][2] = q.y;
  } else {
    load_mat<D>(B, n, i, a);
  }
}

template <int D>
__device__ __forceinline__ void store_mat(double4* __restrict__ M, int64_t ms, int64_t i,
                                          const double (&a)[D][D]) {
  if constexpr (D == 3) {
#pragma unroll
    for (int r = 0; r < 3; ++r) M[r * ms + i] = make_double4(a[r][0], a[r][1], a[r][2], 0.0);
  } else if constexpr (D == 2) {
    M[i] = make_double4(a[0][0], a[0][1], a[1][0], a[1][1]);
  } else {
    M[i] = make_double4(a[0][0], 0.0, 0.0, 0.0);
  }
}

template <int D>
__device__ __forceinline__ void store_f(double4* __restrict__ F, int64_t n, int64_t i,
                                        const double (&a)[D][D]) {
  if constexpr (D == 3) {
    F[i] = make_double4(a[0][0], a[0][1], a[0][2], a[1][0]);
    F[n + i] = make_double4(a[1][1], a[1][2], a[2][0], a[2][1]);
    reinterpret_cast<double*>(F + 2 * n)[i] = a[2][2];
  } else {
    store_mat<D>(F, n, i, a);
  }
}

// Q record with the particle's reference coordinates in the padding (3D:
// COLUMNS {q_0c, q_1c, q_2c, X0_c} in three planes of stride qs); pass B
// then reads Q_j and X0_j with three 256-bit gathers instead of four, each
// over consecutive records (plane layout: 8 instead of 24 lines per warp
// request), and the lattice pass B (tl_lattice.cu) reads only the columns
// c with g0_c != 0 (o_c != 0: 2.08 of 3 on average at 1.6h).  2D/1D records
// have no padding and no planes.
template <int D>
__device__ __forceinline__ void store_q(double4* __restrict__ Q, int64_t qs, int64_t i,
                                        const double (&a)[D][D], const double (&w)[D]) {
  if constexpr (D == 3) {
#pragma unroll
    for (int c = 0; c < 3; ++c) Q[c * qs + i] = make_double4(a[0][c], a[1][c], a[2][c], w[c]);
  } else {
    store_mat<D>(Q, qs, i, a);
  }
}

// Dense 3D Q records (sphb_tl_params.q_dense): column c = double2 plane
// {q_0c, q_1c} at ((double2*)Q)[c n + i] + double plane q_2c at Q[6n + c n + i]
__device__ __forceinline__ void store_q_dense(double4* __restrict__ Q, int64_t n, int64_t i,
                                              const double (&a)[3][3]) {
  double2* q2 = reinterpret_cast<double2*>(Q);
  double* q1 = reinterpret_cast<double*>(Q) + 6 * n;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    q2[c * n + i] = make_double2(a[0][c], a[1][c]);
    q1[c * n + i] = a[2][c];
  }
}

// column c of a dense record, read-only path (16 + 8 bytes)
__device__ __forceinline__ void gather_qcol_dense(const double4* __restrict__ Q, int64_t n, int c,
                                                  int64_t j, double& q0, double& q1,
                                                  double& q2) {
  const double2 t = __ldg(reinterpret_cast<const double2*>(Q) + c * n + j);
  q0 = t.x;
  q1 = t.y;
  q2 = __ldg(reinterpret_cast<const double*>(Q) + 6 * n + c * n + j);
}

__device__ __forceinline__ void load_q_dense(const double4* __restrict__ Q, int64_t n, int64_t i,
                                             double (&a)[3][3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double2 t = reinterpret_cast<const double2*>(Q)[c * n + i];
    a[0][c] = t.x;
    a[1][c] = t.y;
    a[2][c] = reinterpret_cast<const double*>(Q)[6 * n + c * n + i];
  }
}

template <int D>
__device__ __forceinline__ void load_q(const double4* __restrict__ Q, int64_t qs, int64_t i,
                                       double (&a)[D][D]) {
  if constexpr (D == 3) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double4 t = Q[c * qs + i];
      a[0][c] = t.x; a[1][c] = t.y; a[2][c] = t.z;
    }
  } else {
    load_mat<D>(Q, qs, i, a);
  }
}

template <int D>
__device__ __forceinline__ void load_vec(const double4* __restrict__ V, int64_t i, double (&v)[D]) {
  double4 t = V[i];
  const double c[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int a = 0; a < D; ++a) v[a] = c[a];
}

template <int D>
__device__ __forceinline__ void store_vec(double4* __restrict__ V, int64_t i, const double (&v)[D]) {
  double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = v[a];
  V[i] = make_double4(c[0], c[1], c[2], c[3]);
}

// neighbour gathers of data the kernel does not write: 256-bit .nc loads
template <int D>
__device__ __forceinline__ void load_vec_nc(const double4* __restrict__ V, int64_t i,
                                            double (&v)[D]) {
  const double4 t = ldg4(V + i);
  const double c[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int a = 0; a < D; ++a) v[a] = c[a];
}

template <int D>
__device__ __forceinline__ void load_mat_nc(const double4* __restrict__ M, int64_t i,
                                            double (&a)[D][D]) {
  static_assert(D < 3, "3D gathers read the Q planes directly");
  if constexpr (D == 2) {
    const double4 t = ldg4(M + i);
    a[0][0] = t.x; a[0][1] = t.y; a[1][0] = t.z; a[1][1] = t.w;
  } else {
    a[0][0] = ldg4(M + i).x;
  }
}

template <int D>
__device__ __forceinline__ void load_x0(const double4* __restrict__ X0, int64_t i, double (&w)[D],
                                        bool& fixed) {
  const double4 t = ldg4(X0 + i);
  const double c[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int a = 0; a < D; ++a) w[a] = c[a];
  fixed = c[3] != 0.0;
}

// g0 = (alpha/h) dP(q) e V0 from the reference-configuration displacement:
// dW V0 / r = (alpha/h) (-5 q t^3) V0 / r = c5v t^3 with c5v = -5 alpha V0 / h^2
// (q / r = 1 / h), t = 1 - r / (2h).
template <int D>
__device__ __forceinline__ void ref_gradient(const double (&dx)[D], double c5v,
                                             double mhalf_inv_h, double (&g)[D]) {
  double r2 = dx[0] * dx[0];
#pragma unroll
  for (int a = 1; a < D; ++a) r2 = fma(dx[a], dx[a], r2);
  const double inv_r = rsqrt_nr(r2);
  const double t = fma(mhalf_inv_h, r2 * inv_r, 1.0);
  const double f = c5v * ((t * t) * t);
#pragma unroll
  for (int a = 0; a < D; ++a) g[a] = f * dx[a];
}

template <int D>
__device__ __forceinline__ double det_mat(const double (&A)[D][D]) {
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

// Q = (F S) B0^T with the St. Venant-Kirchhoff PK2 (tlsph.py:54-65, 160-167)
template <int D>
__device__ __forceinline__ void svk_q(const double (&F)[D][D], const double (&B0)[D][D], double lam,
                                      double g2, double (&Q)[D][D]) {
  double E[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) s = fma(F[b][a], F[b][c], s);
      E[a][c] = 0.5 * (s - (a == c ? 1.0 : 0.0));
    }
  double tr = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) tr += E[a][a];
  double S[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) S[a][c] = g2 * E[a][c] + (a == c ? lam * tr : 0.0);
  double P[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) s = fma(F[a][b], S[b][c], s);
      P[a][c] = s;
    }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) s = fma(P[a][b], B0[c][b], s);
      Q[a][c] = s;
    }
}

// FP32 companion of Q (FP32 mode): float4 column planes {q_0c, q_1c, q_2c, 0}
// (3D) or one float4 {q00, q01, q10, q11} (2D).
template <int D>
__device__ __forceinline__ void store_q32(float* Q32, int64_t qs, int64_t i,
                                          const double (&a)[D][D]) {
  float4* q = reinterpret_cast<float4*>(Q32);
  if constexpr (D == 3) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      q[c * qs + i] = make_float4((float)a[0][c], (float)a[1][c], (float)a[2][c], 0.f);
  } else if constexpr (D == 2) {
    q[i] = make_float4((float)a[0][0], (float)a[0][1], (float)a[1][0], (float)a[1][1]);
  } else {
    q[i] = make_float4((float)a[0][0], 0.f, 0.f, 0.f);
  }
}

template <int D>
__device__ __forceinline__ void load_q32(const float* Q32, int64_t qs, int64_t i,
                                         double (&a)[D][D]) {
  const float4* q = reinterpret_cast<const float4*>(Q32);
  if constexpr (D == 3) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float4 t = __ldg(q + c * qs + i);
      a[0][c] = t.x; a[1][c] = t.y; a[2][c] = t.z;
    }
  } else if constexpr (D == 2) {
    const float4 t = __ldg(q + i);
    a[0][0] = t.x; a[0][1] = t.y; a[1][0] = t.z; a[1][1] = t.w;
  } else {
    a[0][0] = __ldg(q + i).x;
  }
}

// Compressible Neo-Hookean PK2 stress S = G (I - C^-1) + lam ln(J) C^-1,
// C = F^T F, J = det F (BASELINE configs 3-4; not in the
// reference), then Q = (F S) B0^T as for SVK.
template <int D>
__device__ __forceinline__ void neo_hookean_q(const double (&F)[D][D], const double (&B0)[D][D],
                                              double lam, double g, double (&Q)[D][D]) {
  double Cm[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) s = fma(F[b][a], F[b][c], s);
      Cm[a][c] = s;
    }
  double Ci[D][D];                  // C^-1 by the adjugate (C is symmetric positive definite)
  double detC;
  if constexpr (D == 1) {
    detC = Cm[0][0];
    Ci[0][0] = 1.0 / detC;
  } else if constexpr (D == 2) {
    detC = Cm[0][0] * Cm[1][1] - Cm[0][1] * Cm[1][0];
    const double inv = 1.0 / detC;
    Ci[0][0] = Cm[1][1] * inv; Ci[1][1] = Cm[0][0] * inv;
    Ci[0][1] = -Cm[0][1] * inv; Ci[1][0] = -Cm[1][0] * inv;
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int a1 = (a + 1) % 3, a2 = (a + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
        Ci[c][a] = Cm[a1][c1] * Cm[a2][c2] - Cm[a1][c2] * Cm[a2][c1];   // cofactor^T
      }
    detC = Cm[0][0] * Ci[0][0] + Cm[0][1] * Ci[1][0] + Cm[0][2] * Ci[2][0];
    const double inv = 1.0 / detC;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) Ci[a][c] *= inv;
  }
  const double lnJ = 0.5 * log(detC);
  double S[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) S[a][c] = g * ((a == c ? 1.0 : 0.0) - Ci[a][c]) + lam * lnJ * Ci[a][c];
  double Pm[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) s = fma(F[a][b], S[b][c], s);
      Pm[a][c] = s;
    }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) s = fma(Pm[a][b], B0[c][b], s);
      Q[a][c] = s;
    }
}

// Q = P B0^T of the material law in P.law
template <int D>
__device__ __forceinline__ void stress_q(const sphb_tl_params& P, const double (&F)[D][D],
                                         const double (&B0)[D][D], double (&Q)[D][D]) {
  if (P.law == 1)
    neo_hookean_q<D>(F, B0, P.lam, P.g, Q);
  else
    svk_q<D>(F, B0, P.lam, 2.0 * P.g, Q);
}

// Pass A after the pair loop (tlsph.py:191-199, 54-65, 160-167): F_i += dt
// (m B0_i), det F > 0, Q_i = (F S) B0^T with X0_i in the row padding (+ the
// fused halo push), x_i += dt v_half_i.  m = sum_j (v_half_j - v_half_i) (x) g0_ij.
// UB0 (3D lattice interior rows with a uniform B0): B0 from bu (the
// {b00, b01, b02, b11, b12, b22} of sphb_tl_lattice.b0) instead of the record
template <int D, bool UB0 = false>
__device__ __forceinline__ void tl_a_finish(const sphb_tl_params& P, int64_t i,
                                            const double (&m)[D][D], const double (&wi)[D],
                                            const double (&vhi)[D], double dt,
                                            const double4* __restrict__ B0,
                                            double4* __restrict__ F, double4* __restrict__ Q,
                                            double4* __restrict__ XC, int32_t* __restrict__ err,
                                            const double* bu = nullptr) {
  const int64_t n = P.n;
  double B[D][D], Fi[D][D];
  if constexpr (UB0 && D == 3) {
    B[0][0] = bu[0]; B[0][1] = bu[1]; B[0][2] = bu[2];
    B[1][0] = bu[1]; B[1][1] = bu[3]; B[1][2] = bu[4];
    B[2][0] = bu[2]; B[2][1] = bu[4]; B[2][2] = bu[5];
  } else {
    load_b0<D>(B0, n, i, B);
  }
  load_f<D>(F, n, i, Fi);
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) s = fma(m[a][c], B[c][b], s);
      Fi[a][b] = fma(dt, s, Fi[a][b]);
    }
  const double J = det_mat<D>(Fi);
  if (!(J > 0.0)) atomicOr(err, SPHB_EFLAG_DET_NONPOS);
  double Qi[D][D];
  stress_q<D>(P, Fi, B, Qi);
  store_f<D>(F, n, i, Fi);
  const int64_t qs = P.q_stride ? P.q_stride : n;
  if (P.q32) {
    store_q32<D>(P.q32, qs, i, Qi);
  } else if constexpr (D == 3) {
    if (P.q_dense)
      store_q_dense(Q, P.n, i, Qi);
    else
      store_q<D>(Q, qs, i, Qi, wi);
  } else {
    store_q<D>(Q, qs, i, Qi, wi);
  }
  {   // fused halo push of the boundary layers' Q records
    bool pushed = false;
    if (P.push_q_prev && i >= P.push_lo0 && i < P.push_lo1) {
      store_q<D>(reinterpret_cast<double4*>(P.push_q_prev), qs, P.push_prev_at + (i - P.push_lo0),
                 Qi, wi);
      pushed = true;
    }
    if (P.push_q_next && i >= P.push_hi0 && i < P.push_hi1) {
      store_q<D>(reinterpret_cast<double4*>(P.push_q_next), qs, P.push_next_at + (i - P.push_hi0),
                 Qi, wi);
      pushed = true;
    }
    if (pushed) __threadfence_system();
  }
  double xc[D];
  load_vec<D>(XC, i, xc);
#pragma unroll
  for (int a = 0; a < D; ++a) xc[a] = fma(dt, vhi[a], xc[a]);
  store_vec<D>(XC, i, xc);
}

// Pass B after the pair loop (tlsph.py:164-171, 88-102, 200-202): a_i =
// (acc + Q_i gsum) / rho0 (0 when clamped; with_qi = false: acc / rho0) into A {a, fixed} (+ push), the
// second kick v = v_half + dt/2 a when update_v (+ push); returns |v_i|.
// acc = sum_j Q_j g0_ij, gsum = sum_j g0_ij.
template <int D>
__device__ __forceinline__ double tl_b_finish(const sphb_tl_params& P, int64_t i, bool fixed_i,
                                              double (&acc)[D], const double (&gsum)[D],
                                              const double4* __restrict__ Q,
                                              const double4* __restrict__ Vh,
                                              double4* __restrict__ A, double4* __restrict__ V,
                                              const double* __restrict__ scalars, int update_v,
                                              bool with_qi) {
  const int64_t n = P.n;
  const int64_t qs = P.q_stride ? P.q_stride : n;
  const double inv_rho0 = 1.0 / P.rho0;
  if (with_qi) {
    double Qi[D][D];                // loaded after the loop: 18 registers free in it
    if (P.q32) {
      load_q32<D>(P.q32, qs, i, Qi);
    } else if constexpr (D == 3) {
      if (P.q_dense)
        load_q_dense(Q, n, i, Qi);
      else
        load_q<D>(Q, qs, i, Qi);
    } else {
      load_q<D>(Q, qs, i, Qi);
    }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) acc[a] = fma(Qi[a][b], gsum[b], acc[a]);
  }
#pragma unroll
  for (int a = 0; a < D; ++a) acc[a] = fixed_i ? 0.0 : acc[a] * inv_rho0;
  {   // acceleration record {a0, a1, a2, fixed}: the clamp flag rides in .w
    double c4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < D; ++a) c4[a] = acc[a];
    c4[3] = fixed_i ? 1.0 : 0.0;
    const double4 a4 = make_double4(c4[0], c4[1], c4[2], c4[3]);
    A[i] = a4;
    if (P.push_a_prev && i >= P.push_lo0 && i < P.push_lo1)
      reinterpret_cast<double4*>(P.push_a_prev)[P.push_prev_at + (i - P.push_lo0)] = a4;
    if (P.push_a_next && i >= P.push_hi0 && i < P.push_hi1)
      reinterpret_cast<double4*>(P.push_a_next)[P.push_next_at + (i - P.push_hi0)] = a4;
  }
  double v[D];
  if (update_v) {
    const double hdt = 0.5 * scalars[0];
    load_vec<D>(Vh, i, v);
#pragma unroll
    for (int a = 0; a < D; ++a) v[a] = fixed_i ? 0.0 : fma(hdt, acc[a], v[a]);
    store_vec<D>(V, i, v);
    if (P.push_v_prev && i >= P.push_lo0 && i < P.push_lo1)
      store_vec<D>(reinterpret_cast<double4*>(P.push_v_prev), P.push_prev_at + (i - P.push_lo0), v);
    if (P.push_v_next && i >= P.push_hi0 && i < P.push_hi1)
      store_vec<D>(reinterpret_cast<double4*>(P.push_v_next), P.push_next_at + (i - P.push_hi0), v);
  } else {
    load_vec<D>(V, i, v);
  }
  if ((P.push_a_prev || P.push_a_next) &&
      ((i >= P.push_lo0 && i < P.push_lo1) || (i >= P.push_hi0 && i < P.push_hi1)))
    __threadfence_system();
  double s2 = __dmul_rn(v[0], v[0]);
#pragma unroll
  for (int a = 1; a < D; ++a) s2 = __dadd_rn(s2, __dmul_rn(v[a], v[a]));
  return __dsqrt_rn(s2);
}

// max |v| of the block's rows folded into scalars[2] (all threads call)
template <int NT>
__device__ __forceinline__ void tl_block_speed_max(double speed, double* scalars) {
  __shared__ double red[NT / 32];
  double w = warp_max(speed);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = red[0];
#pragma unroll
    for (int q = 1; q < NT / 32; ++q) b = b > red[q] ? b : red[q];
    atomic_max_nonneg(scalars + 2, b);
  }
}

}  // namespace tl
}  // namespace sphb
