// wc_engine.cu — fused weakly-compressible Eulerian stage kernels.
//
// One launch per midpoint stage of EulerianSolver._substep
// (eulerian.py:610-643).  Each thread owns one particle (engine order:
// neighbors.engine_order), walks its ELL row (the reference CSR row minus the
// pairs the passes skip, displacement-sorted, staged per block in shared
// memory) and, per pair, recomputes what the reference precomputes and
// streams:
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
#include <cuda_pipeline.h>
#include <stdlib.h>

#include <type_traits>

#include "wc_common.cuh"

using namespace sphb;
using namespace sphb::wc;

namespace {

// 64-thread blocks: more, smaller blocks per SM overlap one block's pass-list
// prologue with the others' loops (-1.4% vs 128 on C5, profiles/r01_tune_wc.md)
constexpr int kThreads = 64;

// Per-launch constants folded on the host from sphb_wc_params.
struct WCConst {
  double c2, c2rho0, eta_c, inv_h, c5s, hc, mu2;
  double cg2, cm;         // -c5s [V] / h (-2 x gsc / t^3), mu2 c5s [V] / h: pair factors
  double mhalf_inv_h;     // -0.5 / h
  double wrap_margin;     // particles farther than this from every periodic face never wrap
};

inline WCConst wc_const(const sphb_wc_params& p) {
  WCConst k;
  k.c2 = p.c_art * p.c_art;
  k.c2rho0 = k.c2 * p.rho0;
  k.eta_c = kEtaLinearized / p.c_art;
  k.inv_h = 1.0 / p.h;
  k.c5s = -5.0 * p.alpha / p.h;       // dW = c5s q t^3 (Wendland, kernels.py:55-57)
  k.hc = 0.5 * p.c_art;
  k.mu2 = 2.0 * p.mu;
  const double v = p.uniform_vol ? p.vol_const : 1.0;
  k.cg2 = -(k.c5s * v / p.h);
  k.cm = k.mu2 * k.c5s * v / p.h;
  k.mhalf_inv_h = -0.5 / p.h;
  k.wrap_margin = 1.0001 * p.kappa * p.h;
  return k;
}

// G consecutive lanes share one particle's row (entries k = gl, gl + G, ...;
// partial sums combined with warp shuffles).  G = 1 is the default: in engine
// order the lanes of a warp already read consecutive records.  MINB is the
// occupancy target (register cap); WALL adds the wall-force accumulation.
template <int D, int G, int MINB, bool WALL>
// MINB counts 128-thread equivalents (4 -> 128 registers, 5 -> 96)
// MINB 5 (default): a 9-block bound (112-register cap) under which ptxas
// schedules the 4-way unrolled pair loop in 96 registers, so 10 blocks stay
// resident; the 10-block bound makes it drop the unroll (C5 stage 3.98 ->
// 3.84 ms, A/B in profiles/r01_tune_wc.md)
__global__ void __launch_bounds__(kThreads, MINB == 5 ? 9 : MINB * 128 / kThreads)
k_wc_stage(const sphb_wc_params P, const WCConst K, const int stage,
           const double4* __restrict__ X, const double* __restrict__ B,
           const int32_t* __restrict__ nbr,
           const int32_t* __restrict__ cnt, const double4* __restrict__ S_in,
           const double4* Sn, const double4* Mn, double4* S_out, double4* M_out,
           double* __restrict__ scalars, int32_t* __restrict__ err) {
  const int64_t n = P.n;
  const int gl = threadIdx.x % G;
  const int64_t blk = blockIdx.x;
  const int64_t i = P.row0 + (blk * blockDim.x + threadIdx.x) / G;
  const bool active = i < P.row0 + P.nrows && (P.interior == nullptr || P.interior[i]);

  // Stage the block's ELL columns in shared memory first (stage_pass_list:
  // TMA bulk copies, or LDGSTS for unaligned slices): the index stream then
  // costs one DRAM round trip per block instead of one per loop iteration,
  // and the loop's dependent chain starts at a 30-cycle LDS.
  extern __shared__ int32_t s_nbr[];     // [width][kThreads / G]
  constexpr int RB = kThreads / G;       // rows per block
  stage_pass_list<RB>(nbr, n, P.row0 + blk * RB, P.row0 + P.nrows, P.width, s_nbr);
  const int32_t* __restrict__ srow = s_nbr + (threadIdx.x / G);
  const double c = P.c_art;
  double dr = 0.0;
  double dm[D], wf[D];
#pragma unroll
  for (int a = 0; a < D; ++a) dm[a] = wf[a] = 0.0;
  if (active) {
    // host-folded constants (kernel parameters live in the constant bank, so
    // the FP64 instructions read them as operands instead of registers)
    const double c2 = K.c2, c2rho0 = K.c2rho0, eta_c = K.eta_c;
    const double hc = K.hc;

    double xi[D], vol_i, vi[D], rho_i;
    unpack_x<D>(X[i], xi, vol_i);
    unpack_s<D>(S_in[i], vi, rho_i);
    Sym<D> Bi;
    Bi.load(B, n, i);
    const double hrho_i = 0.5 * rho_i;
    // minimum image (neighbors.py:152-157) only matters within one cut-off
    // of a periodic face: a warp-uniform per-particle test keeps the FP64
    // compare/select work out of the loop for the bulk
    bool wrap = false;
    if (P.periodic) {
#pragma unroll
      for (int a = 0; a < D; ++a)
        wrap = wrap || xi[a] < K.wrap_margin || xi[a] > P.box[a] - K.wrap_margin;
    }

    const int32_t m = cnt[i];

    // one directed pair (i, j) from j's records
    // `uni` (std::true_type / false_type): uniform volumes, V_j folded into
    // the constants; a compile-time flag so the loop carries no select for it
    auto pair = [&](const int64_t j, const double4 xr, const double4 sr, const Sym<D>& Bj,
                    auto uni) {
      double xj[D], vol_j, vj[D], rho_j;
      unpack_x<D>(xr, xj, vol_j);
      unpack_s<D>(sr, vj, rho_j);

      // geometry (neighbors.py:152-165, correction.py:102-108, eulerian.py:506-513),
      // kept in terms of dx: e = dx / r is folded into the scalar factors
      double dx[D];
#pragma unroll
      for (int a = 0; a < D; ++a) dx[a] = xi[a] - xj[a];
      if (wrap) {
#pragma unroll
        for (int a = 0; a < D; ++a)
          if (fabs(dx[a]) > 0.5 * P.box[a]) dx[a] = dx[a] > 0.0 ? dx[a] - P.box[a] : dx[a] + P.box[a];
      }
      double r2 = dx[0] * dx[0];
#pragma unroll
      for (int a = 1; a < D; ++a) r2 = fma(dx[a], dx[a], r2);
      const double inv_r = rsqrt_nr(r2);
      const double t = fma(K.mhalf_inv_h, r2 * inv_r, 1.0);   // 1 - q/2, q = r/h
      // dW V_j / r = c5s q t^3 V_j / r = (c5s / h) t^3 V_j (q / r = 1 / h);
      // gsc = 0.5 dW V_j / r, mv = mu viscv
      double base = (t * t) * t;
      if constexpr (!decltype(uni)::value) base *= vol_j;
      const double gsc2 = K.cg2 * base;                 // -2 gsc: both flux terms' -2
      const double mv = K.cm * base;
      Sym<D> Bs;
      Bi.add(Bj, Bs);
      double G_[D];                                     // (B_i + B_j) dx
      Bs.mv(dx, G_);

      // limited linearised Riemann problem along n = -e (eulerian.py:236-264):
      // du = u_l - u_r = (v_j - v_i).e; u* - ubar = b^2 (p_i - p_j) / (2 rbar c)
      double dv[D];
#pragma unroll
      for (int a = 0; a < D; ++a) dv[a] = vj[a] - vi[a];
      double dud = dv[0] * dx[0];
#pragma unroll
      for (int a = 1; a < D; ++a) dud = fma(dv[a], dx[a], dud);
      const double du = dud * inv_r;
      double beta = du * eta_c;
      beta = beta < 0.0 ? 0.0 : (beta > 1.0 ? 1.0 : beta);
      const double rbar = fma(0.5, rho_j, hrho_i);
      // (u* - ubar) / r with p_i - p_j = c^2 (rho_i - rho_j), c^2 / (2c) = hc;
      // branch-free: beta = 0 gives 0.  pbar = (p_i + p_j) / 2 = c^2 rbar - c^2 rho0
      const double bh = beta * hc;
      const double wr = ((beta * bh) * (rho_i - rho_j)) * (rcp_nr(rbar) * inv_r);
      const double p_star = fma(bh * rbar, du, fma(c2, rbar, -c2rho0));
      double vs[D];
      double sg = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        vs[a] = fma(-wr, dx[a], fma(0.5, dv[a], vi[a]));   // vbar - wr dx
        sg = fma(vs[a], G_[a], sg);
      }
      const double rs2 = rbar * (gsc2 * sg);            // -2 rbar s, s = vs . gwv
      dr += rs2;
      const double pg = p_star * gsc2;                  // -2 p* gsc
#pragma unroll
      for (int a = 0; a < D; ++a)
        dm[a] = fma(-mv, dv[a], fma(pg, G_[a], fma(rs2, vs[a], dm[a])));
      if constexpr (WALL) {               // eulerian.py:262-264
        if (stage != 1 && P.wall_tag[j]) {
#pragma unroll
          for (int a = 0; a < D; ++a) wf[a] -= fma(-mv, dv[a], fma(pg, G_[a], rs2 * vs[a]));
        }
      }
    };

    // loop unroll: 4 at the default target (MINB 5: 96 registers, 20 warps),
    // 2 at the 128-register budget (MINB 4), none above
    constexpr int UNR = MINB == 5 ? 4 : (MINB <= 4 ? 2 : 1);
    auto loop = [&](auto uni) {
#pragma unroll UNR
      for (int32_t k = gl; k < m; k += G) {
        int64_t j = srow[k * RB];
        SPHB_CHECK_INDEX(j, n, err);
        Sym<D> bj;
        bj.load(B, n, j);
        pair(j, ldg4(X + j), ldg4(S_in + j), bj, uni);
      }
    };
    if (P.uniform_vol)
      loop(std::true_type{});
    else
      loop(std::false_type{});
  }
  if constexpr (WALL) {
#pragma unroll
    for (int a = 0; a < D; ++a)
      if (wf[a] != 0.0) atomicAdd(P.wall_force + a, wf[a]);
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    dr += __shfl_xor_sync(0xffffffffu, dr, o);
#pragma unroll
    for (int a = 0; a < D; ++a) dm[a] += __shfl_xor_sync(0xffffffffu, dm[a], o);
  }

  wc_epilogue<D, kThreads>(P, stage, active && gl == 0, i, c, dr, dm, Sn, Mn, S_out, M_out,
                           scalars, err);
}

template <int D>
__global__ void __launch_bounds__(256)
k_speed_max(int64_t row0, int64_t nrows, const int8_t* __restrict__ interior, double c,
            const double4* __restrict__ S, double* __restrict__ scalars) {
  int64_t i = row0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double sp = 0.0;
  if (i < row0 + nrows && (interior == nullptr || interior[i])) {
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

// Ghost refresh (apply_boundaries, eulerian.py:371-447) for the WC kinds:
// each ghost takes its interior source's state, with the velocity copied
// (G_COPY), mirrored about the wall normal (G_MIRROR), set to the wall
// velocity (G_WALL), prescribed (G_FIXED) or mirror-blended (G_BLEND_MIRROR);
// momentum is formed as rho_src * v_ghost and the record stores mom / rho,
// as FluidState.velocity would.  Indices are cell-sorted.
template <int D>
__global__ void k_wc_ghosts(int64_t ng, const int32_t* __restrict__ gs,
                            const int32_t* __restrict__ ss, const int8_t* __restrict__ kind,
                            const double* __restrict__ normal, const double* __restrict__ wall_v,
                            const double* __restrict__ fixed, const double* __restrict__ blend,
                            double4* S, double4* __restrict__ M, int32_t* __restrict__ err) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  double vs[D], rho;
  unpack_s<D>(S[ss[g]], vs, rho);
  double mom[D], out_rho = rho;
  const int k = kind[g];
  if (k == 0) {                       // G_COPY
#pragma unroll
    for (int a = 0; a < D; ++a) mom[a] = __dmul_rn(rho, vs[a]);
    S[gs[g]] = S[ss[g]];
  } else if (k == 1 || k == 5) {      // G_MIRROR / G_BLEND_MIRROR
    double dot = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) dot = __dadd_rn(dot, __dmul_rn(vs[a], normal[g * D + a]));
    const double f = k == 1 ? __dmul_rn(2.0, dot) : __dmul_rn(2.0, blend[g]);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double vg = k == 1 ? __dsub_rn(vs[a], __dmul_rn(f, normal[g * D + a]))
                               : __dsub_rn(vs[a], __dmul_rn(f, __dmul_rn(dot, normal[g * D + a])));
      mom[a] = __dmul_rn(rho, vg);
    }
  } else if (k == 2) {                // G_WALL
#pragma unroll
    for (int a = 0; a < D; ++a) mom[a] = __dmul_rn(rho, wall_v[g * D + a]);
  } else if (k == 3) {                // G_FIXED
    out_rho = fixed[g * (D + 2)];
#pragma unroll
    for (int a = 0; a < D; ++a) mom[a] = fixed[g * (D + 2) + 1 + a];
  } else {                            // G_DMR_TOP needs the energy equation
    atomicOr(err, SPHB_EFLAG_NONFINITE_STATE);
    return;
  }
  if (k != 0) {
    double v[D];
#pragma unroll
    for (int a = 0; a < D; ++a) v[a] = __ddiv_rn(mom[a], out_rho);
    S[gs[g]] = pack_s<D>(v, out_rho);
  }
  if (M) {
    double mc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < D; ++a) mc[a] = mom[a];
    M[gs[g]] = make_double4(mc[0], mc[1], mc[2], mc[3]);
  }
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

extern "C" int sphb_wc_stage(const sphb_wc_params* p, int32_t stage, int32_t group,
                             const double* x, const double* b, const int32_t* nbr,
                             const int32_t* cnt, const double* s_in, const double* s_n,
                             const double* m_n, double* s_out, double* m_out, double* scalars,
                             int32_t* err, void* stream) {
  if (!p || p->n < 0 || stage < 0 || stage > 2 || p->row0 < 0 || p->nrows < 0 ||
      p->row0 + p->nrows > p->n)
    return SPHB_ERR_ARG;
  if (p->nrows == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const double4* X = (const double4*)x;
  const WCConst K = wc_const(*p);
  const double4* Sin = (const double4*)s_in;
  const double4* Sn = (const double4*)s_n;
  const double4* Mn = (const double4*)m_n;
  double4* Sout = (double4*)s_out;
  double4* Mout = (double4*)m_out;
  const size_t smem_idx = (size_t)p->width * (kThreads / group) * sizeof(int32_t);
  static const int carveout = [] {     // SPHB_WC_CARVEOUT: shared-memory carveout % (tuning)
    const char* e = getenv("SPHB_WC_CARVEOUT");
    return e ? atoi(e) : -1;
  }();
  if (smem_idx > 200 * 1024) return SPHB_ERR_ARG;
#define SPHB_STAGE_W(D, G, MB, W)                                                          \
  if (smem_idx > kDynSmemDefault)                                                          \
    SPHB_CUDA_CHECK(cudaFuncSetAttribute(k_wc_stage<D, G, MB, W>,                          \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                         kDynSmemMax));                                    \
  if (carveout >= 0)                                                                       \
    SPHB_CUDA_CHECK(cudaFuncSetAttribute(k_wc_stage<D, G, MB, W>,                          \
                                         cudaFuncAttributePreferredSharedMemoryCarveout,   \
                                         carveout));                                       \
  k_wc_stage<D, G, MB, W><<<sphb_blocks(p->nrows * G, kThreads), kThreads, smem_idx, st>>>( \
      *p, K, stage, X, b, nbr, cnt, Sin, Sn, Mn, Sout, Mout, scalars, err);                \
  break
#define SPHB_STAGE(D, G, MB) SPHB_STAGE_W(D, G, MB, false)
  if (p->wall_tag) {
    if (!p->wall_force) return SPHB_ERR_ARG;
    if (stage != 1) SPHB_CUDA_CHECK(cudaMemsetAsync(p->wall_force, 0, sizeof(double) * p->dim, st));
    switch (p->dim * 16 + group) {
      case 16 + 1: SPHB_STAGE_W(1, 1, 4, true);
      case 32 + 1: SPHB_STAGE_W(2, 1, 4, true);
      case 48 + 1: SPHB_STAGE_W(3, 1, 4, true);
      default: return SPHB_ERR_ARG;
    }
    SPHB_LAUNCH_CHECK();
    return SPHB_OK;
  }
  // SPHB_WC_MINB (tuning): 4 -> <=128 registers, two pairs in flight;
  // 5 (default, 3D) -> <=96 registers, one pair in flight, 20 warps/SM;
  // 6 / 8 spill (profiles/r01_tune_wc.md)
  static int minb = [] {
    const char* e = getenv("SPHB_WC_MINB");
    return e ? atoi(e) : 5;
  }();
  const int key = p->dim * 256 + group * 16 + (p->dim == 3 ? minb : 4);
  switch (key) {
    case 256 + 16 + 4: SPHB_STAGE(1, 1, 4);
    case 512 + 16 + 4: SPHB_STAGE(2, 1, 4);
    case 768 + 16 + 4: SPHB_STAGE(3, 1, 4);
    case 768 + 16 + 5: SPHB_STAGE(3, 1, 5);
    case 768 + 16 + 6: SPHB_STAGE(3, 1, 6);
    case 768 + 16 + 8: SPHB_STAGE(3, 1, 8);
    default: return SPHB_ERR_ARG;
  }
#undef SPHB_STAGE
#undef SPHB_STAGE_W
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
  if (p->nrows <= 0) return SPHB_OK;
  const unsigned grid = sphb_blocks(p->nrows, 256);
  switch (p->dim) {
    case 1: k_speed_max<1><<<grid, 256, 0, st>>>(p->row0, p->nrows, p->interior, p->c_art, S, scalars); break;
    case 2: k_speed_max<2><<<grid, 256, 0, st>>>(p->row0, p->nrows, p->interior, p->c_art, S, scalars); break;
    case 3: k_speed_max<3><<<grid, 256, 0, st>>>(p->row0, p->nrows, p->interior, p->c_art, S, scalars); break;
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

// Ghost rows of the last stage's input -> the step's output (up to three
// 32-byte record arrays), so a state read after step() shows the ghost frame
// of apply_boundaries(t + dt/2), as the reference's in-place arrays do.
__global__ void k_copy_records(int64_t nrows, const int32_t* __restrict__ rows,
                               const double4* __restrict__ s0, double4* __restrict__ d0,
                               const double4* __restrict__ s1, double4* __restrict__ d1,
                               const double4* __restrict__ s2, double4* __restrict__ d2) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nrows) return;
  const int64_t r = rows[g];
  d0[r] = s0[r];
  if (d1) d1[r] = s1[r];
  if (d2) d2[r] = s2[r];
}

// wall_force_series entry (eulerian.py:605-606) appended on the device, so
// graph-replayed steps keep the per-step series without a host round trip.
__global__ void k_wall_record(int32_t dim, const double* __restrict__ wf,
                              const double* __restrict__ scalars, double scale,
                              double* __restrict__ log, int64_t* __restrict__ count,
                              int64_t cap) {
  const int64_t k = count[0];
  if (k < cap) {
    double* row = log + k * (1 + dim);
    row[0] = scalars[1];
    for (int a = 0; a < dim; ++a) row[1 + a] = wf[a] * scale;
  }
  count[0] = k + 1;
}

extern "C" int sphb_wall_record(int32_t dim, const double* wall_force, const double* scalars,
                                double scale, double* log, int64_t* count, int64_t cap,
                                void* stream) {
  if (dim < 1 || dim > 3 || !wall_force || !scalars || !log || !count || cap < 0)
    return SPHB_ERR_ARG;
  k_wall_record<<<1, 1, 0, (cudaStream_t)stream>>>(dim, wall_force, scalars, scale, log, count,
                                                   cap);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_copy_records(int64_t nrows, const int32_t* rows, const double* s0, double* d0,
                                 const double* s1, double* d1, const double* s2, double* d2,
                                 void* stream) {
  if (nrows < 0 || (nrows > 0 && (rows == nullptr || s0 == nullptr || d0 == nullptr)) ||
      ((s1 == nullptr) != (d1 == nullptr)) || ((s2 == nullptr) != (d2 == nullptr)))
    return SPHB_ERR_ARG;
  if (nrows == 0) return SPHB_OK;
  k_copy_records<<<sphb_blocks(nrows, 128), 128, 0, (cudaStream_t)stream>>>(
      nrows, rows, (const double4*)s0, (double4*)d0, (const double4*)s1, (double4*)d1,
      (const double4*)s2, (double4*)d2);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_wc_ghosts(int32_t dim, int64_t ng, const int32_t* ghost_sorted,
                              const int32_t* src_sorted, const int8_t* kind,
                              const double* normal, const double* wall_v, const double* fixed,
                              const double* blend, double* S, double* M, int32_t* err,
                              void* stream) {
  if (ng < 0) return SPHB_ERR_ARG;
  if (ng == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = sphb_blocks(ng, 128);
  switch (dim) {
    case 1: k_wc_ghosts<1><<<grid, 128, 0, st>>>(ng, ghost_sorted, src_sorted, kind, normal, wall_v, fixed, blend, (double4*)S, (double4*)M, err); break;
    case 2: k_wc_ghosts<2><<<grid, 128, 0, st>>>(ng, ghost_sorted, src_sorted, kind, normal, wall_v, fixed, blend, (double4*)S, (double4*)M, err); break;
    case 3: k_wc_ghosts<3><<<grid, 128, 0, st>>>(ng, ghost_sorted, src_sorted, kind, normal, wall_v, fixed, blend, (double4*)S, (double4*)M, err); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
