// wc_tiled.cu — shared-memory tiled weakly-compressible stage kernel.
//
// Same per-pair mathematics as k_wc_stage (wc_engine.cu; eulerian.py:224-266
// with the geometry of :506-513 recomputed), restructured for the B200 memory
// system.  Profiling the one-thread-per-particle kernel showed it bound by
// L1 LSU wavefronts: every neighbour record is a scattered 32-byte request,
// 4 per pair.  Here a CTA owns a tile of 256/G consecutive (cell-sorted)
// particles; it first copies the union of the tile's neighbours — a few
// contiguous runs of sorted indices, precomputed by sphb_tile_plan — into
// shared memory as SoA with coalesced loads, then G threads cooperate on
// each particle (each walks every G-th entry of the row; partial sums are
// combined with warp shuffles) reading neighbour data from shared memory
// through the uint16 local neighbour table.  Uniform particle volumes.
#include <cuda_pipeline.h>

#include "wc_common.cuh"

using namespace sphb;
using namespace sphb::wc;

namespace {

// Shared-memory record of one staged particle, 16-byte chunks:
//   X  {x0, x1, x2, vol}            chunks 0-1
//   B0 {b00, b01, b02, b11}         chunks 2-3
//   B1 {b12, b22}                   chunk 4     (3D only)
//   S  {v0, v1, v2, rho}            chunks 5-6  (2D/1D: 4-5)
// A 112-byte stride (7 chunks) puts consecutive records on 8 distinct
// 4-bank groups, so random per-lane 16-byte reads spread over all banks.
template <int D>
struct Rec {
  static constexpr int kChunks = D == 3 ? 7 : 6;
  static constexpr int kDoubles = 2 * kChunks;
  static constexpr int kX = 0, kB0 = 4, kB1 = 8;
  static constexpr int kS = D == 3 ? 10 : 8;
};

template <int D, int G>
__global__ void __launch_bounds__(256, 2)
k_wc_stage_tiled(const sphb_wc_params P, const int stage, const double4* __restrict__ X,
                 const double* __restrict__ B, const int32_t* __restrict__ cnt,
                 const uint16_t* __restrict__ lnbr, const int32_t* __restrict__ runs,
                 const int32_t* __restrict__ meta, const int32_t rmax, const int32_t umax,
                 const double4* __restrict__ S_in, const double4* Sn, const double4* Mn,
                 double4* S_out, double4* M_out, double* __restrict__ scalars,
                 int32_t* __restrict__ err) {
  extern __shared__ __align__(16) double smem[];
  using RC = Rec<D>;
  constexpr int NB = NSym<D>::value;
  constexpr int PT = 256 / G;  // particles per tile
  const int64_t n = P.n;
  const int64_t tile = blockIdx.x;
  const int32_t* M4 = meta + tile * 4;
  const int nrun = M4[0];
  const int self = M4[2];
  const int32_t* R = runs + tile * (int64_t)rmax * 3;

  // ---- stage the union: cp.async (LDGSTS) 16-byte chunks, field-major per
  // run so consecutive threads copy consecutive chunks of one array
  for (int r = 0; r < nrun; ++r) {
    const int32_t start = R[r * 3], len = R[r * 3 + 1], lbase = R[r * 3 + 2];
    const char* srcs[4] = {reinterpret_cast<const char*>(X + start),
                           reinterpret_cast<const char*>(B) + (size_t)start * 32,
                           reinterpret_cast<const char*>(B + 4 * n) + (size_t)start * 16,
                           reinterpret_cast<const char*>(S_in + start)};
    const int nch[4] = {2, 2, D == 3 ? 1 : 0, 2};
    const int off[4] = {RC::kX, RC::kB0, RC::kB1, RC::kS};
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      if (nch[f] == 0) continue;
      const int total = len * nch[f];
      for (int c = threadIdx.x; c < total; c += blockDim.x) {
        const int rec = c / nch[f], ch = c - rec * nch[f];
        double* dst = smem + (size_t)(lbase + rec) * RC::kDoubles + off[f] + 2 * ch;
        __pipeline_memcpy_async(dst, srcs[f] + (size_t)c * 16, 16);
      }
    }
  }
  __pipeline_commit();
  __pipeline_wait_prior(0);
  __syncthreads();

  const int p = threadIdx.x / G;
  const int gl = threadIdx.x % G;
  const int64_t i = tile * PT + p;
  const bool active = i >= P.row0 && i < P.row0 + P.nrows;
  const int li = self + p;
  const double c = P.c_art;
  const double c2 = c * c;
  const double eta_c = kEtaLinearized / c;
  const double inv_h = 1.0 / P.h;
  const double scale = P.alpha / P.h;
  const double half_cinv = 0.5 / c;
  const double vol_j = P.vol_const;

  double dr = 0.0;
  double dm[D];
#pragma unroll
  for (int a = 0; a < D; ++a) dm[a] = 0.0;
  if (active) {
    double xi[D], vi[D], bi[NB];
    const double* ri = smem + (size_t)li * RC::kDoubles;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      xi[a] = ri[RC::kX + a];
      vi[a] = ri[RC::kS + a];
    }
#pragma unroll
    for (int a = 0; a < NB; ++a) bi[a] = ri[RC::kB0 + a];
    const double rho_i = ri[RC::kS + D];
    const double p_i = c2 * (rho_i - P.rho0);
    const int32_t m = cnt[i];
    for (int32_t k = gl; k < m; k += G) {
      const int lj = lnbr[(int64_t)k * n + i];
      const double* rj = smem + (size_t)lj * RC::kDoubles;
      const double2 xj01 = *reinterpret_cast<const double2*>(rj + RC::kX);
      const double2 xj23 = *reinterpret_cast<const double2*>(rj + RC::kX + 2);
      const double2 bj01 = *reinterpret_cast<const double2*>(rj + RC::kB0);
      const double2 bj23 = *reinterpret_cast<const double2*>(rj + RC::kB0 + 2);
      const double2 bj45 = *reinterpret_cast<const double2*>(rj + RC::kB1);
      const double2 sj01 = *reinterpret_cast<const double2*>(rj + RC::kS);
      const double2 sj23 = *reinterpret_cast<const double2*>(rj + RC::kS + 2);
      const double xjc[4] = {xj01.x, xj01.y, xj23.x, xj23.y};
      const double bjc[6] = {bj01.x, bj01.y, bj23.x, bj23.y, bj45.x, bj45.y};
      const double sjc[4] = {sj01.x, sj01.y, sj23.x, sj23.y};
      // geometry (neighbors.py:152-165, correction.py:102-108)
      double dx[D];
      double r2 = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double d = xi[a] - xjc[a];
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
      const double dW = scale * (-5.0 * q) * (t * t * t);
      double e[D];
#pragma unroll
      for (int a = 0; a < D; ++a) e[a] = dx[a] * inv_r;
      double bs[NB];
#pragma unroll
      for (int a = 0; a < NB; ++a) bs[a] = bi[a] + bjc[a];
      double g[D];
      if constexpr (D == 3) {
        g[0] = fma(bs[0], e[0], fma(bs[1], e[1], bs[2] * e[2]));
        g[1] = fma(bs[1], e[0], fma(bs[3], e[1], bs[4] * e[2]));
        g[2] = fma(bs[2], e[0], fma(bs[4], e[1], bs[5] * e[2]));
      } else if constexpr (D == 2) {
        g[0] = fma(bs[0], e[0], bs[1] * e[1]);
        g[1] = fma(bs[1], e[0], bs[2] * e[1]);
      } else {
        g[0] = bs[0] * e[0];
      }
      const double gs = 0.5 * dW * vol_j;
#pragma unroll
      for (int a = 0; a < D; ++a) g[a] *= gs;
      const double viscv = 2.0 * dW * inv_r * vol_j;

      // limited linearised Riemann problem (eulerian.py:145-157, 236-264)
      double vj[D];
#pragma unroll
      for (int a = 0; a < D; ++a) vj[a] = sjc[a];
      const double rho_j = sjc[D];
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
      double ustar_m_ubar = 0.0;
      if (beta > 0.0) ustar_m_ubar = (beta * beta) * (p_i - p_j) * half_cinv / rbar;
      const double p_star = fma(0.5 * beta * rbar * c, du, 0.5 * (p_i + p_j));
      double vs[D];
      double sdot = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        vs[a] = fma(-ustar_m_ubar, e[a], 0.5 * (vi[a] + vj[a]));
        sdot = fma(vs[a], g[a], sdot);
      }
      dr = fma(-2.0 * rbar, sdot, dr);
      const double rs = rbar * sdot;
      const double mv = P.mu * viscv;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double fm = -2.0 * fma(rs, vs[a], p_star * g[a]);
        dm[a] = fma(mv, vi[a] - vj[a], dm[a] + fm);
      }
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    dr += __shfl_xor_sync(0xffffffffu, dr, o);
#pragma unroll
    for (int a = 0; a < D; ++a) dm[a] += __shfl_xor_sync(0xffffffffu, dm[a], o);
  }

  // ---- epilogue (eulerian.py:619-633, 553-560): one lane per particle
  double speed = 0.0;
  int32_t flags = 0;
  if (active && gl == 0) {
    bool fin = isfinite(dr);
#pragma unroll
    for (int a = 0; a < D; ++a) fin = fin && isfinite(dm[a]);
    if (!fin) flags |= SPHB_EFLAG_NONFINITE_FLUX;
    if (stage == 0) {
      S_out[i] = pack_s<D>(dm, dr);
    } else {
      const double dt = scalars[0];
      const double cdt = stage == 1 ? 0.5 * dt : dt;
      const double4 mn = Mn[i];
      const double cm[4] = {mn.x, mn.y, mn.z, mn.w};
      double vtmp[D], rho_n;
      unpack_s<D>(Sn[i], vtmp, rho_n);
      const double rho_new = fma(cdt, dr, rho_n);
      double mom_new[D], v_new[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        mom_new[a] = fma(cdt, dm[a], cm[a]);
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
  }
  if (stage == 2) {
    __shared__ double red[8];
    const double w = warp_max(speed);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = red[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) b = b > red[q] ? b : red[q];
      atomic_max_nonneg(scalars + 2, b);
    }
  }
  if (flags) atomicOr(err, flags);
}

template <int D, int G>
int launch_tiled(const sphb_wc_params* p, int32_t stage, const double* x, const double* b,
                 const int32_t* cnt, const uint16_t* lnbr, const int32_t* runs,
                 const int32_t* meta, int32_t rmax, int32_t umax, const double* s_in,
                 const double* s_n, const double* m_n, double* s_out, double* m_out,
                 double* scalars, int32_t* err, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)Rec<D>::kDoubles * (size_t)umax;
  auto kern = k_wc_stage_tiled<D, G>;
  static size_t configured = 0;
  if (smem > configured) {
    SPHB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
    configured = smem;
  }
  const int64_t ntiles = (p->n + (256 / G) - 1) / (256 / G);
  kern<<<(unsigned)ntiles, 256, smem, st>>>(*p, stage, (const double4*)x, b, cnt,
                                            lnbr, runs, meta, rmax, umax, (const double4*)s_in,
                                            (const double4*)s_n, (const double4*)m_n,
                                            (double4*)s_out, (double4*)m_out, scalars, err);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

}  // namespace

extern "C" int sphb_wc_stage_tiled(const sphb_wc_params* p, int32_t stage, int32_t group,
                                   const double* x, const double* b, const int32_t* cnt,
                                   const uint16_t* lnbr, const int32_t* runs, const int32_t* meta,
                                   int32_t rmax, int32_t umax, const double* s_in,
                                   const double* s_n, const double* m_n, double* s_out,
                                   double* m_out, double* scalars, int32_t* err, void* stream) {
  if (!p || p->n <= 0 || stage < 0 || stage > 2 || umax <= 0 || p->wall_tag || p->push_prev ||
      p->push_next)
    return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
#define SPHB_TILED(D, G)                                                                   \
  return launch_tiled<D, G>(p, stage, x, b, cnt, lnbr, runs, meta, rmax, umax, s_in, s_n, \
                            m_n, s_out, m_out, scalars, err, st)
  switch (p->dim * 16 + group) {
    case 16 + 1: SPHB_TILED(1, 1);
    case 16 + 2: SPHB_TILED(1, 2);
    case 32 + 1: SPHB_TILED(2, 1);
    case 32 + 2: SPHB_TILED(2, 2);
    case 32 + 4: SPHB_TILED(2, 4);
    case 32 + 8: SPHB_TILED(2, 8);
    case 48 + 1: SPHB_TILED(3, 1);
    case 48 + 2: SPHB_TILED(3, 2);
    case 48 + 4: SPHB_TILED(3, 4);
    case 48 + 8: SPHB_TILED(3, 8);
    default: return SPHB_ERR_ARG;
  }
#undef SPHB_TILED
}
