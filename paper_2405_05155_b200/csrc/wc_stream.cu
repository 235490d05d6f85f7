// wc_stream.cu — WC stage kernel over streamed per-pair geometry.
//
// Particles never move in the Eulerian solver, so the pair geometry that the
// reference precomputes once (eulerian.py:506-513: e_ij, gwv_ij, viscv_ij)
// is static.  sphb_wc_geometry stores it per slot of the ELL pass list as
// coalesced planes; this kernel then streams it (7 doubles per directed pair
// in 3D, contiguous across a warp) and gathers only the neighbour's state
// record S_j = {v_j, rho_j} (one 256-bit request).  Compared with
// recomputing the geometry from X_j and B_j (wc_engine.cu) it trades FP64
// work and three scattered requests per pair for sequential HBM bytes, which
// makes the pass bandwidth-bound instead of latency-bound.
//
// The flux is evaluated with the reference's expressions in the reference's
// order (eulerian.py:236-265) in a translation unit compiled without FMA
// contraction, so per-row sums reproduce _rhs_wc's roundings.
#include "wc_common.cuh"

using namespace sphb;
using namespace sphb::wc;

namespace {

constexpr int kThreads = 128;

template <int D>
__global__ void __launch_bounds__(kThreads)
k_wc_stage_geo(const sphb_wc_params P, const int stage, const int32_t* __restrict__ nbr,
               const int32_t* __restrict__ cnt, const double* __restrict__ geo,
               const double4* __restrict__ S_in, const double4* Sn, const double4* Mn,
               double4* S_out, double4* M_out, double* __restrict__ scalars,
               int32_t* __restrict__ err) {
  const int64_t n = P.n;
  const int64_t W = P.width;
  const int64_t i = P.row0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < P.row0 + P.nrows && (P.interior == nullptr || P.interior[i]);
  const double c_art = P.c_art;
  double speed = 0.0;
  int32_t flags = 0;
  if (active) {
    const double c2 = c_art * c_art;
    double vi[D], rho_i;
    unpack_s<D>(S_in[i], vi, rho_i);
    const double p_i = c2 * (rho_i - P.rho0);
    double dr = 0.0;
    double dm[D];
#pragma unroll
    for (int a = 0; a < D; ++a) dm[a] = 0.0;
    const int32_t m = cnt[i];
    for (int32_t k = 0; k < m; ++k) {
      const int64_t slot = (int64_t)k * n + i;
      const int64_t j = nbr[slot];
      double vj[D], rho_j;
      unpack_s<D>(ldg4(S_in + j), vj, rho_j);
      double e[D], gwv[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        e[a] = __ldg(geo + (a * W) * n + slot);
        gwv[a] = __ldg(geo + ((D + a) * W) * n + slot);
      }
      const double viscv = __ldg(geo + (2 * D * W) * n + slot);
      const double p_j = c2 * (rho_j - P.rho0);
      // eulerian.py:236-265, term for term
      double u_l = 0.0, u_r = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        u_l += vi[a] * (-e[a]);
        u_r += vj[a] * (-e[a]);
      }
      const double du = u_l - u_r;
      double beta = kEtaLinearized * du / c_art;
      if (beta < 0.0) beta = 0.0;
      else if (beta > 1.0) beta = 1.0;
      const double rbar = 0.5 * (rho_i + rho_j);
      const double u_star = 0.5 * (u_l + u_r) + 0.5 * beta * beta * (p_i - p_j) / (rbar * c_art);
      const double p_star = 0.5 * (p_i + p_j) + 0.5 * beta * rbar * c_art * du;
      const double ubar = 0.5 * (u_l + u_r);
      double vs[D];
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        vs[a] = u_star * (-e[a]) + 0.5 * (vi[a] + vj[a]) - ubar * (-e[a]);
        s += vs[a] * gwv[a];
      }
      dr += -2.0 * rbar * s;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double fm = -2.0 * (rbar * vs[a] * s + p_star * gwv[a]) + P.mu * viscv * (vi[a] - vj[a]);
        dm[a] += fm;
      }
    }

    bool finite = isfinite(dr);
#pragma unroll
    for (int a = 0; a < D; ++a) finite = finite && isfinite(dm[a]);
    if (!finite) flags |= SPHB_EFLAG_NONFINITE_FLUX;
    if (stage == 0) {
      S_out[i] = pack_s<D>(dm, dr);
    } else {
      // eulerian.py:619-627: U = U^n + (c dt) R
      const double dt = scalars[0];
      const double cdt = stage == 1 ? 0.5 * dt : dt;
      const double4 mn = Mn[i];
      const double cm[4] = {mn.x, mn.y, mn.z, mn.w};
      double vtmp[D], rho_n;
      unpack_s<D>(Sn[i], vtmp, rho_n);
      const double rho_new = rho_n + cdt * dr;
      double mom_new[D], v_new[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        mom_new[a] = cm[a] + cdt * dm[a];
        v_new[a] = mom_new[a] / rho_new;
      }
      if (!(rho_new > 0.0)) flags |= SPHB_EFLAG_NONPOS_DENSITY;
      S_out[i] = pack_s<D>(v_new, rho_new);
      if (stage == 2) {
        double mc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < D; ++a) mc[a] = mom_new[a];
        M_out[i] = make_double4(mc[0], mc[1], mc[2], mc[3]);
        speed = c_art + norm_exact<D>(v_new);
      }
    }
  }
  if (stage == 2) {
    __shared__ double red[kThreads / 32];
    const double w = warp_max(speed);
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

}  // namespace

extern "C" int sphb_wc_stage_geo(const sphb_wc_params* p, int32_t stage, const int32_t* nbr,
                                 const int32_t* cnt, const double* geo, const double* s_in,
                                 const double* s_n, const double* m_n, double* s_out,
                                 double* m_out, double* scalars, int32_t* err, void* stream) {
  if (!p || p->n < 0 || stage < 0 || stage > 2 || p->row0 < 0 || p->nrows < 0 ||
      p->row0 + p->nrows > p->n || p->wall_tag || p->push_prev || p->push_next)
    return SPHB_ERR_ARG;
  if (p->nrows == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = sphb_blocks(p->nrows, kThreads);
  const double4* Sin = (const double4*)s_in;
  const double4* Sn = (const double4*)s_n;
  const double4* Mn = (const double4*)m_n;
  double4* Sout = (double4*)s_out;
  double4* Mout = (double4*)m_out;
  switch (p->dim) {
    case 1: k_wc_stage_geo<1><<<grid, kThreads, 0, st>>>(*p, stage, nbr, cnt, geo, Sin, Sn, Mn, Sout, Mout, scalars, err); break;
    case 2: k_wc_stage_geo<2><<<grid, kThreads, 0, st>>>(*p, stage, nbr, cnt, geo, Sin, Sn, Mn, Sout, Mout, scalars, err); break;
    case 3: k_wc_stage_geo<3><<<grid, kThreads, 0, st>>>(*p, stage, nbr, cnt, geo, Sin, Sn, Mn, Sout, Mout, scalars, err); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
