// hllc.cu — compressible (ideal-gas) Eulerian path: limited HLLC flux with
// the energy equation.
//
// Restates EulerianSolver's ideal-gas branch: eos_eval (eulerian.py:67-85),
// _hllc_scalar (:90-142), the fan sampling of _rhs_hllc (:269-338), the
// midpoint update of rho, mom and E (:619-636) and apply_boundaries for the
// ideal-gas kinds incl. the time-dependent double-Mach-reflection top
// (:371-447, dmr_shock_x :366-368).  The pair geometry (e_ij, gwv_ij) is
// streamed from sphb_wc_geometry, and this unit is compiled without FMA
// contraction so each row repeats the reference's roundings.
//
// Records (cell-sorted): S {v, rho} and M {mom, 0} as in the WC engine, plus
// Q {E, p, c, 0} (total energy per volume, pressure, sound speed).
#include "wc_common.cuh"

using namespace sphb;
using namespace sphb::wc;

namespace {

constexpr int kThreads = 128;

struct Star {
  double u_star, p_star, rho_sl, rho_sr, e_sl, e_sr, s_l, s_r, s_star;
};

// _hllc_scalar (eulerian.py:90-142), eta = ETA_HLLC = 1
__device__ __forceinline__ Star hllc_scalar(double rho_l, double u_l, double p_l, double c_l,
                                            double e_l, double rho_r, double u_r, double p_r,
                                            double c_r, double e_r) {
  const double eta = 1.0;
  double s_l = u_l - c_l;
  double s_r = u_r + c_r;
  double den = rho_r * (s_r - u_r) + rho_l * (u_l - s_l);
  double s_star = (rho_r * u_r * (s_r - u_r) + rho_l * u_l * (u_l - s_l) + p_l - p_r) / den;
  if (!(s_l < s_star && s_star < s_r)) {
    s_l = fmin(u_l - c_l, u_r - c_r);
    s_r = fmax(u_l + c_l, u_r + c_r);
    den = rho_r * (s_r - u_r) + rho_l * (u_l - s_l);
    s_star = (rho_r * u_r * (s_r - u_r) + rho_l * u_l * (u_l - s_l) + p_l - p_r) / den;
  }
  const double cbar = 0.5 * (c_l + c_r);
  const double du = u_l - u_r;
  double beta = eta * du / cbar;
  if (beta < 0.0) beta = 0.0;
  else if (beta > 1.0) beta = 1.0;
  const double w_l = rho_l * (u_l - s_l);
  const double w_r = rho_r * (s_r - u_r);
  const double ws = w_l + w_r;
  Star st;
  st.u_star = (w_l * u_l + w_r * u_r) / ws + (p_l - p_r) * beta * beta / ws;
  st.p_star = 0.5 * (p_l + p_r) + 0.5 * beta * (w_r * (st.u_star - u_r) + w_l * (u_l - st.u_star));
  const double den_l = s_l - s_star;
  const double den_r = s_r - s_star;
  st.rho_sl = rho_l * (s_l - u_l) / den_l;
  st.rho_sr = rho_r * (s_r - u_r) / den_r;
  st.e_sl = ((s_l - u_l) * e_l - p_l * u_l + st.p_star * s_star) / den_l;
  st.e_sr = ((s_r - u_r) * e_r - p_r * u_r + st.p_star * s_star) / den_r;
  st.s_l = s_l;
  st.s_r = s_r;
  st.s_star = s_star;
  return st;
}

// eos_eval ideal gas (eulerian.py:78-85) on one particle: p, c, e >= 0 flag
template <int D>
__device__ __forceinline__ bool ideal_gas(double rho, const double (&mom)[D], double etot,
                                          double gamma, double& p, double& c) {
  double m2 = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) m2 += mom[a] * mom[a];
  const double v2 = m2 / (rho * rho);
  const double e = etot / rho - 0.5 * v2;
  p = rho * (gamma - 1.0) * e;
  c = sqrt(gamma * p / rho);
  return e >= 0.0 && rho > 0.0;
}

template <int D>
__global__ void __launch_bounds__(kThreads)
k_hllc_stage(const sphb_wc_params P, const int stage, const int32_t* __restrict__ nbr,
             const int32_t* __restrict__ cnt, const double* __restrict__ geo,
             const double4* __restrict__ S_in, const double4* __restrict__ Q_in,
             const double4* Sn, const double4* Mn, const double4* Qn, double4* S_out,
             double4* M_out, double4* Q_out, double* __restrict__ scalars,
             int32_t* __restrict__ err) {
  const int64_t n = P.n;
  const int64_t W = P.width;
  const int64_t i = P.row0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < P.row0 + P.nrows && (P.interior == nullptr || P.interior[i]);
  double speed = 0.0;
  int32_t flags = 0;
  if (active) {
    double vi[D], rho_i;
    unpack_s<D>(S_in[i], vi, rho_i);
    const double4 qi = Q_in[i];
    const double E_i = qi.x, p_i = qi.y, c_i = qi.z;
    double dr = 0.0, de = 0.0;
    double dm[D], wf[D];
#pragma unroll
    for (int a = 0; a < D; ++a) dm[a] = wf[a] = 0.0;
    const bool track = P.wall_tag != nullptr && stage != 1;
    const int32_t m = cnt[i];
    for (int32_t k = 0; k < m; ++k) {
      const int64_t slot = (int64_t)k * n + i;
      const int64_t j = nbr[slot];
      double vj[D], rho_j;
      unpack_s<D>(ldg4(S_in + j), vj, rho_j);
      const double4 qj = ldg4(Q_in + j);
      double e[D], gwv[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        e[a] = __ldg(geo + (a * W) * n + slot);
        gwv[a] = __ldg(geo + ((D + a) * W) * n + slot);
      }
      double u_l = 0.0, u_r = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        u_l += vi[a] * (-e[a]);
        u_r += vj[a] * (-e[a]);
      }
      const Star o = hllc_scalar(rho_i, u_l, p_i, c_i, E_i, rho_j, u_r, qj.y, qj.z, qj.x);
      // eulerian.py:289-311: sample the wave fan at the interface
      double rho_s, e_s, p_use;
      int side;  // 0 star, 1 left state, 2 right state
      if (o.s_l > 0.0) {
        rho_s = rho_i; e_s = E_i; p_use = p_i; side = 1;
      } else if (o.s_r < 0.0) {
        rho_s = rho_j; e_s = qj.x; p_use = qj.y; side = 2;
      } else if (o.s_star >= 0.0) {
        rho_s = o.rho_sl; e_s = o.e_sl; p_use = o.p_star; side = 0;
      } else {
        rho_s = o.rho_sr; e_s = o.e_sr; p_use = o.p_star; side = 0;
      }
      const double ubar = 0.5 * (u_l + u_r);
      double vs[D];
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        vs[a] = side == 0 ? (o.u_star - ubar) * (-e[a]) + 0.5 * (vi[a] + vj[a])
                          : (side == 1 ? vi[a] : vj[a]);
        s += vs[a] * gwv[a];
      }
      dr += -2.0 * rho_s * s;
      de += -2.0 * (e_s + p_use) * s;
      const bool tagged = track && P.wall_tag[j] != 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double fm = -2.0 * (rho_s * vs[a] * s + p_use * gwv[a]);
        dm[a] += fm;
        if (tagged) wf[a] -= fm;              // eulerian.py:333-335
      }
    }
    if (track) {
#pragma unroll
      for (int a = 0; a < D; ++a)
        if (wf[a] != 0.0) atomicAdd(P.wall_force + a, wf[a]);
    }
    bool finite = isfinite(dr) && isfinite(de);
#pragma unroll
    for (int a = 0; a < D; ++a) finite = finite && isfinite(dm[a]);
    if (!finite) flags |= SPHB_EFLAG_NONFINITE_FLUX;
    if (stage == 0) {
      S_out[i] = pack_s<D>(dm, dr);
      Q_out[i] = make_double4(de, 0.0, 0.0, 0.0);
    } else {
      const double dt = scalars[0];
      const double cdt = stage == 1 ? 0.5 * dt : dt;
      const double4 mn = Mn[i];
      const double cm[4] = {mn.x, mn.y, mn.z, mn.w};
      double vtmp[D], rho_n;
      unpack_s<D>(Sn[i], vtmp, rho_n);
      const double E_n = Qn[i].x;
      const double rho_new = rho_n + cdt * dr;
      const double E_new = E_n + cdt * de;
      double mom_new[D], v_new[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        mom_new[a] = cm[a] + cdt * dm[a];
        v_new[a] = mom_new[a] / rho_new;
      }
      double p_new, c_new;
      if (!(rho_new > 0.0)) flags |= SPHB_EFLAG_NONPOS_DENSITY;
      if (!ideal_gas<D>(rho_new, mom_new, E_new, P.gamma, p_new, c_new))
        flags |= SPHB_EFLAG_NONFINITE_STATE;
      S_out[i] = pack_s<D>(v_new, rho_new);
      Q_out[i] = make_double4(E_new, p_new, c_new, 0.0);
      double mc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int a = 0; a < D; ++a) mc[a] = mom_new[a];
      if (M_out) M_out[i] = make_double4(mc[0], mc[1], mc[2], mc[3]);
      if (stage == 2) speed = c_new + norm_exact<D>(v_new);
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

// Conserved (rho, mom, E) in caller order -> S, M, Q records + max(c + |v|)
// over interior rows (eos_eval + compute_dt, eulerian.py:78-85, 553-560).
template <int D>
__global__ void k_hllc_pack(int64_t n, const int32_t* __restrict__ perm,
                            const int8_t* __restrict__ interior, double gamma,
                            const double* __restrict__ rho, const double* __restrict__ mom,
                            const double* __restrict__ etot, double4* __restrict__ S,
                            double4* __restrict__ M, double4* __restrict__ Q,
                            double* __restrict__ scalars, int32_t* __restrict__ err) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double speed = 0.0;
  if (s < n) {
    const int64_t i = perm[s];
    const double r = rho[i];
    double m[D], v[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      m[a] = mom[i * D + a];
      v[a] = m[a] / r;
    }
    double p, c;
    if (!ideal_gas<D>(r, m, etot[i], gamma, p, c)) atomicOr(err, SPHB_EFLAG_NONFINITE_STATE);
    S[s] = pack_s<D>(v, r);
    double mc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < D; ++a) mc[a] = m[a];
    M[s] = make_double4(mc[0], mc[1], mc[2], mc[3]);
    Q[s] = make_double4(etot[i], p, c, 0.0);
    if (interior == nullptr || interior[s]) speed = c + norm_exact<D>(v);
  }
  __shared__ double red[32];
  const double w = warp_max(speed);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = red[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) b = b > red[q] ? b : red[q];
    atomic_max_nonneg(scalars + 2, b);
  }
}

template <int D>
__global__ void k_hllc_unpack(int64_t n, const int32_t* __restrict__ perm,
                              const double4* __restrict__ S, const double4* __restrict__ M,
                              const double4* __restrict__ Q, double* __restrict__ rho,
                              double* __restrict__ mom, double* __restrict__ etot) {
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
  etot[i] = Q[s].x;
}

// apply_boundaries, ideal gas (eulerian.py:371-447).  fixed / dmr_post /
// dmr_pre hold conserved (rho, mom, E).  t_shift selects the stage time:
// t = scalars[1] - scalars[0] + t_shift * scalars[0] (step start + shift dt).
template <int D>
__global__ void k_hllc_ghosts(int64_t ng, const int32_t* __restrict__ gs,
                              const int32_t* __restrict__ ss, const int8_t* __restrict__ kind,
                              const double* __restrict__ normal,
                              const double* __restrict__ wall_v,
                              const double* __restrict__ fixed, const double* __restrict__ blend,
                              const double* __restrict__ dmr_x, double dmr_x0, double dmr_tan,
                              const double* __restrict__ dmr_post,
                              const double* __restrict__ dmr_pre, double gamma, double t_shift,
                              const double* __restrict__ scalars, double4* S, double4* M,
                              double4* Q, int32_t* __restrict__ err) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t src = ss[g];
  double vs[D], rho_s;
  unpack_s<D>(S[src], vs, rho_s);
  const double E_s = Q[src].x;
  double rho = rho_s, E = E_s, mom[D];
  const int k = kind[g];
  if (k == 0) {                                  // G_COPY
    const double4 ms = M[src];
    const double c[4] = {ms.x, ms.y, ms.z, ms.w};
#pragma unroll
    for (int a = 0; a < D; ++a) mom[a] = c[a];
  } else if (k == 1 || k == 5) {                 // G_MIRROR / G_BLEND_MIRROR
    double dot = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) dot += vs[a] * normal[g * D + a];
    double vg[D], vs2 = 0.0, vg2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      vg[a] = k == 1 ? vs[a] - 2.0 * dot * normal[g * D + a]
                     : vs[a] - 2.0 * blend[g] * (dot * normal[g * D + a]);
      mom[a] = rho_s * vg[a];
      vs2 += vs[a] * vs[a];
      vg2 += vg[a] * vg[a];
    }
    if (k == 5) E = E_s - 0.5 * rho_s * (vs2 - vg2);
  } else if (k == 2) {                           // G_WALL
#pragma unroll
    for (int a = 0; a < D; ++a) mom[a] = rho_s * wall_v[g * D + a];
  } else if (k == 3) {                           // G_FIXED
    rho = fixed[g * (D + 2)];
#pragma unroll
    for (int a = 0; a < D; ++a) mom[a] = fixed[g * (D + 2) + 1 + a];
    E = fixed[g * (D + 2) + 1 + D];
  } else {                                       // G_DMR_TOP
    const double t = scalars[1] - scalars[0] + t_shift * scalars[0];
    const double xs = dmr_x0 + (1.0 + 20.0 * t) / dmr_tan;   // host math.tan(radians(60))
    const double* st = dmr_x[g] < xs ? dmr_post : dmr_pre;
    rho = st[0];
#pragma unroll
    for (int a = 0; a < D; ++a) mom[a] = st[1 + a];
    E = st[1 + D];
  }
  double v[D];
#pragma unroll
  for (int a = 0; a < D; ++a) v[a] = mom[a] / rho;
  double p, c;
  if (!ideal_gas<D>(rho, mom, E, gamma, p, c)) atomicOr(err, SPHB_EFLAG_NONFINITE_STATE);
  const int64_t dst = gs[g];
  S[dst] = pack_s<D>(v, rho);
  double mc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 0; a < D; ++a) mc[a] = mom[a];
  M[dst] = make_double4(mc[0], mc[1], mc[2], mc[3]);
  Q[dst] = make_double4(E, p, c, 0.0);
}

}  // namespace

#define HLLC_D(FN, GRID, ...)                                                      \
  do {                                                                             \
    switch (dim) {                                                                 \
      case 1: FN<1><<<GRID, kThreads, 0, st>>>(__VA_ARGS__); break;                \
      case 2: FN<2><<<GRID, kThreads, 0, st>>>(__VA_ARGS__); break;                \
      case 3: FN<3><<<GRID, kThreads, 0, st>>>(__VA_ARGS__); break;                \
      default: return SPHB_ERR_ARG;                                                \
    }                                                                              \
  } while (0)

extern "C" int sphb_hllc_stage(const sphb_wc_params* p, int32_t stage, const int32_t* nbr,
                               const int32_t* cnt, const double* geo, const double* s_in,
                               const double* q_in, const double* s_n, const double* m_n,
                               const double* q_n, double* s_out, double* m_out, double* q_out,
                               double* scalars, int32_t* err, void* stream) {
  if (!p || p->n < 0 || stage < 0 || stage > 2 || !(p->gamma > 1.0) ||
      (p->wall_tag && !p->wall_force))
    return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->wall_tag && stage != 1)
    SPHB_CUDA_CHECK(cudaMemsetAsync(p->wall_force, 0, sizeof(double) * p->dim, st));
  if (p->nrows <= 0) return SPHB_OK;
  const int dim = p->dim;
  HLLC_D(k_hllc_stage, sphb_blocks(p->nrows, kThreads), *p, stage, nbr, cnt, geo,
         (const double4*)s_in, (const double4*)q_in, (const double4*)s_n, (const double4*)m_n,
         (const double4*)q_n, (double4*)s_out, (double4*)m_out, (double4*)q_out, scalars, err);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_hllc_pack_state(int64_t n, int32_t dim, const int32_t* perm,
                                    const int8_t* interior, double gamma, const double* rho,
                                    const double* mom, const double* etot, double* s, double* m,
                                    double* q, double* scalars, int32_t* err, void* stream) {
  if (n < 0) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_CUDA_CHECK(cudaMemsetAsync(scalars + 2, 0, sizeof(double), st));
  if (n == 0) return SPHB_OK;
  HLLC_D(k_hllc_pack, sphb_blocks(n, kThreads), n, perm, interior, gamma, rho, mom, etot,
         (double4*)s, (double4*)m, (double4*)q, scalars, err);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_hllc_unpack_state(int64_t n, int32_t dim, const int32_t* perm,
                                      const double* s, const double* m, const double* q,
                                      double* rho, double* mom, double* etot, void* stream) {
  if (n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  HLLC_D(k_hllc_unpack, sphb_blocks(n, kThreads), n, perm, (const double4*)s,
         (const double4*)m, (const double4*)q, rho, mom, etot);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_hllc_ghosts(int32_t dim, int64_t ng, const int32_t* ghost_sorted,
                                const int32_t* src_sorted, const int8_t* kind,
                                const double* normal, const double* wall_v, const double* fixed,
                                const double* blend, const double* dmr_x, double dmr_x0,
                                double dmr_tan, const double* dmr_post, const double* dmr_pre,
                                double gamma,
                                double t_shift, const double* scalars, double* s, double* m,
                                double* q, int32_t* err, void* stream) {
  if (ng < 0) return SPHB_ERR_ARG;
  if (ng == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  HLLC_D(k_hllc_ghosts, sphb_blocks(ng, kThreads), ng, ghost_sorted, src_sorted, kind, normal,
         wall_v, fixed, blend, dmr_x, dmr_x0, dmr_tan, dmr_post, dmr_pre, gamma, t_shift, scalars,
         (double4*)s, (double4*)m, (double4*)q, err);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
