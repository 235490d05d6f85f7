// tl_engine.cu — fused total-Lagrangian SPH passes (kick-drift-kick).
//
// SolidSystem.step (tlsph.py:182-206) is two grid-wide dependencies (the dF
// pass needs every neighbour's half-kicked velocity, the momentum pass needs
// every neighbour's new stress), so it is two launches:
//
//   pass A  (tlsph.py:191-199, :105-123, :54-65, :160-167)
//     v_half_j = fixed_j ? 0 : v_j + dt/2 a_j       recomputed per neighbour
//     dF_i = [sum_j (v_half_j - v_half_i) (x) g0_ij] B0_i
//     F_i += dt dF_i ; det F_i > 0 ; x_i += dt v_half_i
//     epilogue: S = lam tr(E) I + 2 G E, E = (F^T F - I)/2 ; Q_i = (F S) B0^T
//   pass B  (tlsph.py:164-171, :88-102, :200-202, :178-180)
//     a_i = sum_j (Q_i + Q_j) g0_ij / rho0 ; a[fixed] = 0
//     v_i = v_half_i + dt/2 a_i ; v[fixed] = 0 ; fold max |v_i|
//
// g0_ij = (alpha/h) dP(q) e_ij V0 (tlsph.py:145-146) is recomputed from the
// reference configuration instead of being streamed from a per-pair array.
//
// Records (cell-sorted order):
//   X0[i]  double4 {w0, w1, w2, fixed}  (w = X0 - min(X0), as the CSR's r/e)
//   V, A, Vh, XC  double4 vectors
//   B0, F, Q      3x3: 3 x double4 rows {a0, a1, a2, 0}; 2D: 1 x double4
//                 {a00, a01, a10, a11}; 1D: {a00, 0, 0, 0}
#include <stdlib.h>

#include "tl_common.cuh"

using namespace sphb;
using namespace sphb::tl;

namespace {

constexpr int kThreads = 128;
constexpr int64_t kStageMinRows = 32768;   // stage pass lists from this many rows up

// widest pass list still staged in shared memory (SPHB_TL_STAGE_MAXW, tuning)
inline int tl_stage_max_width() {
  static const int w = [] {
    const char* e = getenv("SPHB_TL_STAGE_MAXW");
    return e ? atoi(e) : 1 << 20;
  }();
  return w;
}

// GEO: read g0_ij from the streamed per-slot planes g0[(c * width + k) * n + i]
// (sphb_tl_geometry) instead of recomputing it from X0_j; the clamp flag of
// j then comes from A_j.w (pass B keeps it there).
// First kick of the KDK step for every local row (owned + halo):
// vh = v + dt/2 a, 0 for clamped particles (tlsph.py:186-189); pass A then
// gathers one half-step velocity record per pair instead of v_j and a_j.
template <int D>
__global__ void k_tl_kick(int64_t n, const double4* __restrict__ V, const double4* __restrict__ A,
                          double4* __restrict__ Vh, const double* __restrict__ scalars,
                          float4* __restrict__ Vh32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double hdt = 0.5 * scalars[0];
  double v[D], a_[D], vh[D];
  load_vec<D>(V, i, v);
  const double4 a4 = A[i];          // {a0, a1, a2, fixed}: the clamp flag rides in .w
  const double c4[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
  for (int a = 0; a < D; ++a) a_[a] = c4[a];
  const bool fixed = a4.w != 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) vh[a] = fixed ? 0.0 : fma(hdt, a_[a], v[a]);
  {   // the clamp flag rides in Vh.w too (table-mode lattice pass B reads it)
    double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < D; ++a) c[a] = vh[a];
    c[3] = a4.w;
    Vh[i] = make_double4(c[0], c[1], c[2], c[3]);
  }
  if (Vh32) {                       // FP32 mode: the gathered companion
    float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < D; ++a) c[a] = (float)vh[a];
    Vh32[i] = make_float4(c[0], c[1], c[2], c[3]);
  }
}

// UNR: pairs in flight per thread; 3D default 2 (two Vh_j + X0_j gather
// pairs outstanding: -12% on C4, profiles/r01_tune_tl.md)
template <int D, bool GEO, bool STAGED, int MINB = 1, int UNR = (D == 3 ? 2 : 1)>
__global__ void __launch_bounds__(kThreads, MINB)
k_tl_pass_a(const sphb_tl_params P, const double4* __restrict__ X0, const double4* __restrict__ B0,
            const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
            const double* __restrict__ g0,
            const double4* __restrict__ Vh,
            double4* __restrict__ XC, double4* __restrict__ F, double4* __restrict__ Q,
            const double* __restrict__ scalars, int32_t* __restrict__ err) {
  const int64_t n = P.n;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  extern __shared__ int32_t s_nbr[];
  // small sets (C3: 41 blocks) gain nothing from staging and pay its round trip
  if constexpr (STAGED)
    stage_pass_list<kThreads>(nbr, n, P.row0 + (int64_t)blockIdx.x * kThreads,
                              P.row0 + P.nrows, P.width, s_nbr);
  if (t >= P.nrows) return;
  const int64_t i = P.row0 + t;
  const double dt = scalars[0];
  const double hdt = 0.5 * dt;
  const double inv_h = 1.0 / P.h;
  const double scale_v0 = P.alpha / P.h * P.vol0;
  const double c5v = -5.0 * scale_v0 * inv_h, mhalf_inv_h = -0.5 * inv_h;

  double wi[D], vhi[D];
  bool fixed_i;
  load_x0<D>(X0, i, wi, fixed_i);
  load_vec<D>(Vh, i, vhi);            // k_tl_kick: v + dt/2 a, 0 when clamped

  double m[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) m[a][b] = 0.0;

  const int32_t cn = cnt[i];
  const int32_t* __restrict__ srow = s_nbr + threadIdx.x;
  const int32_t* __restrict__ grow = nbr + i;
#pragma unroll UNR
  for (int32_t k = 0; k < cn; ++k) {
    int64_t j = STAGED ? srow[k * kThreads] : grow[(int64_t)k * n];
    SPHB_CHECK_INDEX(j, n, err);
    double vhj[D], g[D];
    load_vec_nc<D>(Vh, j, vhj);
    if constexpr (GEO) {
      const int64_t slot = (int64_t)k * n + i;
#pragma unroll
      for (int a = 0; a < D; ++a) g[a] = __ldg(g0 + ((int64_t)a * P.width) * n + slot);
    } else {
      double wj[D];
      bool fixed_j;
      load_x0<D>(X0, j, wj, fixed_j);
      double dx[D];
#pragma unroll
      for (int a = 0; a < D; ++a) dx[a] = wi[a] - wj[a];
      ref_gradient<D>(dx, c5v, mhalf_inv_h, g);
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double dv = vhj[a] - vhi[a];
#pragma unroll
      for (int b = 0; b < D; ++b) m[a][b] = fma(dv, g[b], m[a][b]);
    }
  }

  tl_a_finish<D>(P, i, m, wi, vhi, dt, B0, F, Q, XC, err);
}

template <int D, bool GEO, bool STAGED, int MINB = 1, int UNR = 1>
__global__ void __launch_bounds__(kThreads, MINB)
k_tl_pass_b(const sphb_tl_params P, const double4* __restrict__ X0,
            const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
            const double* __restrict__ g0,
            const double4* __restrict__ Q, const double4* __restrict__ Vh,
            double4* __restrict__ A, double4* __restrict__ V, double* __restrict__ scalars,
            int update_v, int32_t* __restrict__ err) {
  const int64_t n = P.n;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  extern __shared__ int32_t s_nbr[];
  if constexpr (STAGED)
    stage_pass_list<kThreads>(nbr, n, P.row0 + (int64_t)blockIdx.x * kThreads,
                              P.row0 + P.nrows, P.width, s_nbr);
  double speed = 0.0;
  if (t < P.nrows) {
    const int64_t i = P.row0 + t;
    const double inv_h = 1.0 / P.h;
    const double scale_v0 = P.alpha / P.h * P.vol0;
    const double c5v = -5.0 * scale_v0 * inv_h, mhalf_inv_h = -0.5 * inv_h;
    double wi[D];
    bool fixed_i;
    load_x0<D>(X0, i, wi, fixed_i);
    const int64_t qs = P.q_stride ? P.q_stride : n;
    double gsum[D], acc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) { gsum[a] = 0.0; acc[a] = 0.0; }
    const int32_t cn = cnt[i];
    const int32_t* __restrict__ srow = s_nbr + threadIdx.x;
    const int32_t* __restrict__ grow = nbr + i;
#pragma unroll UNR
    for (int32_t k = 0; k < cn; ++k) {
      int64_t j = STAGED ? srow[k * kThreads] : grow[(int64_t)k * n];
      SPHB_CHECK_INDEX(j, n, err);
      double Qj[D][D], wj[D];
      if constexpr (D == 3) {      // Q columns carry X0_j in their padding (store_q)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double4 t4 = ldg4(Q + c * qs + j);
          Qj[0][c] = t4.x; Qj[1][c] = t4.y; Qj[2][c] = t4.z;
          wj[c] = t4.w;
        }
      } else {
        load_mat_nc<D>(Q, j, Qj);
        if constexpr (!GEO) {
          bool fixed_j;
          load_x0<D>(X0, j, wj, fixed_j);
        }
      }
      double g[D];
      if constexpr (GEO) {
        const int64_t slot = (int64_t)k * n + i;
#pragma unroll
        for (int a = 0; a < D; ++a) g[a] = __ldg(g0 + ((int64_t)a * P.width) * n + slot);
      } else {
        double dx[D];
#pragma unroll
        for (int a = 0; a < D; ++a) dx[a] = wi[a] - wj[a];
        ref_gradient<D>(dx, c5v, mhalf_inv_h, g);
      }
      // sum_j (Q_i + Q_j) g = Q_i sum_j g + sum_j Q_j g
#pragma unroll
      for (int b = 0; b < D; ++b) gsum[b] += g[b];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) acc[a] = fma(Qj[a][b], g[b], acc[a]);
    }
    speed = tl_b_finish<D>(P, i, fixed_i, acc, gsum, Q, Vh, A, V, scalars, update_v, true);
  }
  tl_block_speed_max<kThreads>(speed, scalars);
}

template <int D>
__global__ void k_tl_stress(const sphb_tl_params P, const double4* __restrict__ F,
                            const double4* __restrict__ B0, const double4* __restrict__ X0,
                            double4* __restrict__ Q) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  double Fi[D][D], B[D][D], Qi[D][D], w[D];
  bool fixed;
  load_f<D>(F, P.n, i, Fi);
  load_b0<D>(B0, P.n, i, B);
  load_x0<D>(X0, i, w, fixed);
  stress_q<D>(P, Fi, B, Qi);
  if constexpr (D == 3) {
    if (P.q_dense)
      store_q_dense(Q, P.n, i, Qi);
    else
      store_q<D>(Q, P.q_stride ? P.q_stride : P.n, i, Qi, w);
  } else {
    store_q<D>(Q, P.q_stride ? P.q_stride : P.n, i, Qi, w);
  }
  if (P.q32) store_q32<D>(P.q32, P.q_stride ? P.q_stride : P.n, i, Qi);
}

template <int D>
__global__ void k_tl_speed(int64_t row0, int64_t nrows, const double4* __restrict__ V,
                           double* __restrict__ scalars) {
  const int64_t i = row0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double speed = 0.0;
  if (i < row0 + nrows) {
    double v[D];
    load_vec<D>(V, i, v);
    double s2 = __dmul_rn(v[0], v[0]);
#pragma unroll
    for (int a = 1; a < D; ++a) s2 = __dadd_rn(s2, __dmul_rn(v[a], v[a]));
    speed = __dsqrt_rn(s2);
  }
  __shared__ double red[8];
  double w = warp_max(speed);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = red[0];
    for (int q = 1; q < 8; ++q) b = b > red[q] ? b : red[q];
    atomic_max_nonneg(scalars + 2, b);
  }
}

}  // namespace

#define TL_DISPATCH(KERNEL, GRID, TH, ...)                                 \
  do {                                                                     \
    switch (p->dim) {                                                      \
      case 1: KERNEL<1><<<GRID, TH, 0, st>>>(__VA_ARGS__); break;          \
      case 2: KERNEL<2><<<GRID, TH, 0, st>>>(__VA_ARGS__); break;          \
      case 3: KERNEL<3><<<GRID, TH, 0, st>>>(__VA_ARGS__); break;          \
      default: return SPHB_ERR_ARG;                                        \
    }                                                                      \
  } while (0)

// SPHB_TL_CARVEOUT (tuning): preferred shared-memory carveout, % of the
// unified L1 / shared array; default -1 = the driver's choice (a fixed 40%
// gains 1.6% at 1.6h but starves the 2h pass-list staging, r01_tune_tl.md)
inline int tl_carveout() {
  static const int c = [] {
    const char* e = getenv("SPHB_TL_CARVEOUT");
    return e ? atoi(e) : -1;
  }();
  return c;
}

// dynamic shared memory: the block's pass-list columns (stage_pass_list)
#define TL_LAUNCH(KERNEL, GRID, TH, SMEM, ...)                                                   \
  do {                                                                                         \
    if ((SMEM) > kDynSmemDefault)                                                              \
      SPHB_CUDA_CHECK(cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           kDynSmemMax));                                      \
    if (tl_carveout() >= 0)                                                                    \
      SPHB_CUDA_CHECK(cudaFuncSetAttribute(KERNEL,                                             \
                                           cudaFuncAttributePreferredSharedMemoryCarveout,     \
                                           tl_carveout()));                                    \
    KERNEL<<<GRID, TH, SMEM, st>>>(__VA_ARGS__);                                               \
  } while (0)

#define TL_DISPATCH_GEO(KERNEL, GEOPTR, GRID, TH, ...)                                     \
  do {                                                                                     \
    const bool geo_ = (GEOPTR) != nullptr;                                                 \
    const bool stg_ = p->nrows >= kStageMinRows && p->width <= tl_stage_max_width();       \
    const size_t smem_ = stg_ ? (size_t)p->width * kThreads * sizeof(int32_t) : 0;        \
    if (smem_ > 200 * 1024) return SPHB_ERR_ARG;                                           \
    switch (p->dim * 4 + (geo_ ? 2 : 0) + (stg_ ? 1 : 0)) {                                \
      case 4: TL_LAUNCH((KERNEL<1, false, false>), GRID, TH, smem_, __VA_ARGS__); break;   \
      case 5: TL_LAUNCH((KERNEL<1, false, true>), GRID, TH, smem_, __VA_ARGS__); break;    \
      case 6: TL_LAUNCH((KERNEL<1, true, false>), GRID, TH, smem_, __VA_ARGS__); break;    \
      case 7: TL_LAUNCH((KERNEL<1, true, true>), GRID, TH, smem_, __VA_ARGS__); break;     \
      case 8: TL_LAUNCH((KERNEL<2, false, false>), GRID, TH, smem_, __VA_ARGS__); break;   \
      case 9: TL_LAUNCH((KERNEL<2, false, true>), GRID, TH, smem_, __VA_ARGS__); break;    \
      case 10: TL_LAUNCH((KERNEL<2, true, false>), GRID, TH, smem_, __VA_ARGS__); break;   \
      case 11: TL_LAUNCH((KERNEL<2, true, true>), GRID, TH, smem_, __VA_ARGS__); break;    \
      case 12: TL_LAUNCH((KERNEL<3, false, false>), GRID, TH, smem_, __VA_ARGS__); break;  \
      case 13: TL_LAUNCH((KERNEL<3, false, true>), GRID, TH, smem_, __VA_ARGS__); break;   \
      case 14: TL_LAUNCH((KERNEL<3, true, false>), GRID, TH, smem_, __VA_ARGS__); break;   \
      case 15: TL_LAUNCH((KERNEL<3, true, true>), GRID, TH, smem_, __VA_ARGS__); break;    \
      default: return SPHB_ERR_ARG;                                                        \
    }                                                                                      \
  } while (0)

extern "C" int sphb_tl_pass_a(const sphb_tl_params* p, const double* x0, const double* b0,
                              const int32_t* nbr, const int32_t* cnt, const double* g0,
                              const double* v, const double* a, double* vh, double* xc,
                              double* f, double* q, const double* scalars, int32_t* err,
                              void* stream) {
  if (!p || p->n < 0) return SPHB_ERR_ARG;
  if (p->n == 0 || p->nrows <= 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  TL_DISPATCH(k_tl_kick, sphb_blocks(p->n, 256), 256, p->n, (const double4*)v, (const double4*)a, (double4*)vh, scalars, (float4*)p->vh32);
  TL_DISPATCH_GEO(k_tl_pass_a, g0, sphb_blocks(p->nrows, kThreads), kThreads, *p,
                    (const double4*)x0, (const double4*)b0, nbr, cnt, g0, (const double4*)vh,
                    (double4*)xc, (double4*)f, (double4*)q, scalars, err);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_tl_pass_b(const sphb_tl_params* p, const double* x0, const int32_t* nbr,
                              const int32_t* cnt, const double* g0, const double* q,
                              const double* vh, double* a, double* v, double* scalars,
                              int32_t update_v, int32_t* err, void* stream) {
  if (!p || p->n < 0) return SPHB_ERR_ARG;
  if (p->n == 0 || p->nrows <= 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  TL_DISPATCH_GEO(k_tl_pass_b, g0, sphb_blocks(p->nrows, kThreads), kThreads, *p,
                    (const double4*)x0, nbr, cnt, g0, (const double4*)q, (const double4*)vh,
                    (double4*)a, (double4*)v, scalars, (int)update_v, err);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_tl_kick(const sphb_tl_params* p, const double* v, const double* a,
                            double* vh, const double* scalars, void* stream) {
  if (!p || p->n < 0 || !v || !a || !vh || !scalars) return SPHB_ERR_ARG;
  if (p->n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  TL_DISPATCH(k_tl_kick, sphb_blocks(p->n, 256), 256, p->n, (const double4*)v, (const double4*)a,
              (double4*)vh, scalars, (float4*)p->vh32);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_tl_stress(const sphb_tl_params* p, const double* f, const double* b0,
                              const double* x0, double* q, void* stream) {
  if (!p || p->n < 0 || !x0) return SPHB_ERR_ARG;
  if (p->n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  TL_DISPATCH(k_tl_stress, sphb_blocks(p->n, 128), 128, *p, (const double4*)f, (const double4*)b0,
              (const double4*)x0, (double4*)q);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_tl_speed_max(const sphb_tl_params* p, const double* v, double* scalars,
                                 void* stream) {
  if (!p || p->n < 0) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_CUDA_CHECK(cudaMemsetAsync(scalars + 2, 0, sizeof(double), st));
  if (p->n == 0) return SPHB_OK;
  if (p->nrows <= 0) return SPHB_OK;
  TL_DISPATCH(k_tl_speed, sphb_blocks(p->nrows, 256), 256, p->row0, p->nrows, (const double4*)v,
              scalars);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
