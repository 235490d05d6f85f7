// wc_common.cuh — record packing helpers shared by the WC stage kernels.
#pragma once

#include "common.cuh"

namespace sphb {
namespace wc {

// Symmetrised correction matrix, two planes so consecutive particles'
// records are contiguous: plane 0 = double4 {b00, b01, b02, b11} (2D: {b00,
// b01, b11, 0}; 1D: {b00, ..}) at B[0 .. 4n), plane 1 = double2 {b12, b22}
// at B[4n .. 6n) (3D only).
template <int D>
struct Sym;
template <>
struct Sym<1> {
  double a00;
  __device__ __forceinline__ void load(const double* B, int64_t, int64_t i) {
    a00 = ldg4(reinterpret_cast<const double4*>(B) + i).x;
  }
  __device__ __forceinline__ void add(const Sym& o, Sym& r) const { r.a00 = a00 + o.a00; }
  __device__ __forceinline__ void mv(const double (&e)[1], double (&out)[1]) const {
    out[0] = a00 * e[0];
  }
};
template <>
struct Sym<2> {
  double a00, a01, a11;
  __device__ __forceinline__ void load(const double* B, int64_t, int64_t i) {
    const double4 t = ldg4(reinterpret_cast<const double4*>(B) + i);
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
  __device__ __forceinline__ void load(const double* B, int64_t n, int64_t i) {
    const double4 t = ldg4(reinterpret_cast<const double4*>(B) + i);
    const double2 u = reinterpret_cast<const double2*>(B + 4 * n)[i];
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
struct NSym { static constexpr int value = D == 3 ? 6 : (D == 2 ? 3 : 1); };

}  // namespace wc
}  // namespace sphb
