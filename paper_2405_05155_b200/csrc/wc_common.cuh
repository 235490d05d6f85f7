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
  __device__ __forceinline__ double at(int r, int c) const {
    return r != c ? a01 : (r == 0 ? a00 : a11);
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
  __device__ __forceinline__ double at(int r, int c) const {
    const int k = r < c ? r * 3 + c : c * 3 + r;
    return k == 0 ? a00 : k == 1 ? a01 : k == 2 ? a02 : k == 4 ? a11 : k == 5 ? a12 : a22;
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
// Stage epilogue shared by the WC stage kernels (eulerian.py:548-550,
// 619-629): error flags, the stage update into S_out / M_out (stage 0: the
// rhs record {dmom, drho}), the fused halo push, and for stage 2 the
// block-reduced max(c + |v|) folded into scalars[2].  Every thread of the
// block must call it (block reduction); `write` selects the rows it owns.
// wc_row_update: the per-row part (flags into `flags`, returns c + |v| of
// stage 2, else 0); wc_block_finish: the block part (speed reduction, error
// word).  wc_epilogue = both, for one row per thread.
template <int D>
__device__ __forceinline__ double wc_row_update(const sphb_wc_params& P, int stage, int64_t i,
                                                double c, double dr, const double (&dm)[D],
                                                const double4* Sn, const double4* Mn,
                                                double4* S_out, double4* M_out,
                                                const double* scalars, int32_t& flags) {
  double speed = 0.0;
  {
    bool finite = isfinite(dr);
#pragma unroll
    for (int a = 0; a < D; ++a) finite = finite && isfinite(dm[a]);
    if (!finite) flags |= SPHB_EFLAG_NONFINITE_FLUX;
    if (stage == 0) {  // rhs only: S_out = {dmom, drho} (EulerianSolver.rhs)
      S_out[i] = pack_s<D>(dm, dr);
    } else {
      const double dt = scalars[0];
      const double cdt = stage == 1 ? 0.5 * dt : dt;
      const double4 mn = Mn[i];
      const double cm[4] = {mn.x, mn.y, mn.z, mn.w};
      double vtmp[D], rho_n;
      unpack_s<D>(Sn[i], vtmp, rho_n);
      const double rho_new = fma(cdt, dr, rho_n);   // eulerian.py:619-627
      double mom_new[D], v_new[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        mom_new[a] = fma(cdt, dm[a], cm[a]);
        v_new[a] = __ddiv_rn(mom_new[a], rho_new);
      }
      if (!(rho_new > 0.0)) flags |= SPHB_EFLAG_NONPOS_DENSITY;
      const double4 s_new = pack_s<D>(v_new, rho_new);
      S_out[i] = s_new;
      // fused halo push: boundary layers go straight into the neighbour
      // ranks' halo rows (peer memory) from this epilogue
      bool pushed = false;
      if (P.push_prev && i >= P.push_lo0 && i < P.push_lo1) {
        reinterpret_cast<double4*>(P.push_prev)[P.push_prev_at + (i - P.push_lo0)] = s_new;
        pushed = true;
      }
      if (P.push_next && i >= P.push_hi0 && i < P.push_hi1) {
        reinterpret_cast<double4*>(P.push_next)[P.push_next_at + (i - P.push_hi0)] = s_new;
        pushed = true;
      }
      if (pushed) __threadfence_system();
      if (stage == 2) {
        double mc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < D; ++a) mc[a] = mom_new[a];
        M_out[i] = make_double4(mc[0], mc[1], mc[2], mc[3]);
        speed = __dadd_rn(c, norm_exact<D>(v_new));
      }
    }
  }
  return speed;
}

template <int NT>
__device__ __forceinline__ void wc_block_finish(int stage, double speed, int32_t flags,
                                                double* scalars, int32_t* err) {
  if (stage == 2) {
    __shared__ double red[NT / 32];
    const double w = warp_max(speed);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = red[0];
#pragma unroll
      for (int q = 1; q < NT / 32; ++q) b = b > red[q] ? b : red[q];
      atomic_max_nonneg(scalars + 2, b);
    }
  }
  if (flags) atomicOr(err, flags);
}

template <int D, int NT>
__device__ __forceinline__ void wc_epilogue(const sphb_wc_params& P, int stage, bool write,
                                            int64_t i, double c, double dr,
                                            const double (&dm)[D], const double4* Sn,
                                            const double4* Mn, double4* S_out, double4* M_out,
                                            double* scalars, int32_t* err) {
  int32_t flags = 0;
  const double speed =
      write ? wc_row_update<D>(P, stage, i, c, dr, dm, Sn, Mn, S_out, M_out, scalars, flags)
            : 0.0;
  wc_block_finish<NT>(stage, speed, flags, scalars, err);
}

}  // namespace wc
}  // namespace sphb
