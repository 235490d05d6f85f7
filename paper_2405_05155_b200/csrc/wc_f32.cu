// wc_f32.cu — optional FP32 mode of the WC stage kernel.
//
// North star: FP64 to match the oracle, "with an optional FP32 mode whose
// error is reported separately".  Pair geometry and the limited linearised
// Riemann flux (eulerian.py:145-157, 224-266; geometry :506-513) are
// evaluated in FP32 from FP32 neighbour records, which halves the gathered
// bytes; the per-particle sums are accumulated and the stage update applied
// in FP64 on the FP64 conserved state, so round-off does not accumulate in
// the state across steps.  Records (cell-sorted):
//   X32 float4 {x0, x1, x2, 0}          static
//   B32 float4 {b00,b01,b02,b11} plane + float2 {b12,b22} plane   static
//   S32 float4 {v0, v1, v2, rho - rho0} written by every stage epilogue
// (density is carried as its deviation so p = c^2 (rho - rho0) keeps FP32
// relative precision).
#include "wc_common.cuh"

using namespace sphb;
using namespace sphb::wc;

namespace {

constexpr int kThreads = 64;

__device__ __forceinline__ float4 ldg4f(const float4* p) { return __ldg(p); }

// 3D: 16 blocks of 64 per SM (64 registers, 32 warps) and 1/rbar from the
// fast approximate divide: 3.54 -> 2.99 ms per C5 stage (r01_tune_wc.md)
template <int D>
__global__ void __launch_bounds__(kThreads, D == 3 ? 16 : 1)
k_wc_stage_f32(const sphb_wc_params P, const int stage, const float4* __restrict__ X,
               const float* __restrict__ B, const int32_t* __restrict__ nbr,
               const int32_t* __restrict__ cnt, const float4* __restrict__ S32_in,
               const double4* Sn, const double4* Mn, float4* __restrict__ S32_out,
               double4* S_out, double4* M_out, double* __restrict__ scalars,
               int32_t* __restrict__ err) {
  const int64_t n = P.n;
  const int64_t i = P.row0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < P.row0 + P.nrows && (P.interior == nullptr || P.interior[i]);
  extern __shared__ int32_t s_nbr[];
  stage_pass_list<kThreads>(nbr, n, P.row0 + (int64_t)blockIdx.x * kThreads, P.row0 + P.nrows,
                            P.width, s_nbr);
  const double c_art = P.c_art;
  double speed = 0.0;
  int32_t flags = 0;
  if (active) {
    const float c = (float)c_art;
    const float c2 = c * c;
    const float eta_c = (float)(kEtaLinearized / c_art);
    const float inv_h = (float)(1.0 / P.h);
    const float scale = (float)(P.alpha / P.h);
    const float half_cinv = 0.5f / c;
    const float vol = (float)P.vol_const;
    const float mu = (float)P.mu;
    float box[3] = {(float)P.box[0], (float)P.box[1], (float)P.box[2]};
    const float4 xr = X[i];
    const float xi[3] = {xr.x, xr.y, xr.z};
    const float4 sr = S32_in[i];
    const float vi[3] = {sr.x, sr.y, sr.z};
    const float drho_i = D == 3 ? sr.w : (D == 2 ? sr.z : sr.y);
    const float4 bi4 = reinterpret_cast<const float4*>(B)[i];
    const float2 bi2 = reinterpret_cast<const float2*>(B + 4 * n)[i];
    const float bi[6] = {bi4.x, bi4.y, bi4.z, bi4.w, bi2.x, bi2.y};
    const float p_i = c2 * drho_i;
    double dr = 0.0;
    double dm[D];
#pragma unroll
    for (int a = 0; a < D; ++a) dm[a] = 0.0;
    // pair factors in t^3 form (q / r = 1 / h): gsc = 0.5 dW V / r, mv = mu viscv
    const float mhalf_inv_h = -0.5f * inv_h;
    const float cg = 0.5f * scale * -5.0f * inv_h * vol;
    const float cm = 2.0f * mu * scale * -5.0f * inv_h * vol;
    const float rho0f = (float)P.rho0;
    float hvi[3];
#pragma unroll
    for (int a = 0; a < D; ++a) hvi[a] = 0.5f * vi[a];
    const int32_t m = cnt[i];
    for (int32_t k = 0; k < m; ++k) {
      const int64_t j = s_nbr[k * kThreads + threadIdx.x];
      const float4 xj4 = ldg4f(X + j);
      const float4 sj4 = ldg4f(S32_in + j);
      const float4 bj4 = ldg4f(reinterpret_cast<const float4*>(B) + j);
      const float xj[3] = {xj4.x, xj4.y, xj4.z};
      const float vj[3] = {sj4.x, sj4.y, sj4.z};
      const float drho_j = D == 3 ? sj4.w : (D == 2 ? sj4.z : sj4.y);
      float bs[6];
      bs[0] = bi[0] + bj4.x; bs[1] = bi[1] + bj4.y; bs[2] = bi[2] + bj4.z; bs[3] = bi[3] + bj4.w;
      if (D == 3) {
        const float2 bj2 = __ldg(reinterpret_cast<const float2*>(B + 4 * n) + j);
        bs[4] = bi[4] + bj2.x; bs[5] = bi[5] + bj2.y;
      } else {
        bs[4] = bs[5] = 0.f;
      }
      float dx[3] = {0.f, 0.f, 0.f};
      float r2 = 0.f;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        float d = xi[a] - xj[a];
        if (P.periodic) {
          if (d > 0.5f * box[a]) d -= box[a];
          else if (d < -0.5f * box[a]) d += box[a];
        }
        dx[a] = d;
        r2 = fmaf(d, d, r2);
      }
      const float inv_r = rsqrtf(r2);
      const float t = fmaf(mhalf_inv_h, r2 * inv_r, 1.0f);
      const float t3 = (t * t) * t;
      const float gsc = cg * t3, mv = cm * t3;
      float G_[3];                                  // (B_i + B_j) dx
      if (D == 3) {
        G_[0] = fmaf(bs[0], dx[0], fmaf(bs[1], dx[1], bs[2] * dx[2]));
        G_[1] = fmaf(bs[1], dx[0], fmaf(bs[3], dx[1], bs[4] * dx[2]));
        G_[2] = fmaf(bs[2], dx[0], fmaf(bs[4], dx[1], bs[5] * dx[2]));
      } else if (D == 2) {
        G_[0] = fmaf(bs[0], dx[0], bs[1] * dx[1]);
        G_[1] = fmaf(bs[1], dx[0], bs[2] * dx[1]);
        G_[2] = 0.f;
      } else {
        G_[0] = bs[0] * dx[0];
        G_[1] = G_[2] = 0.f;
      }
      float dv[3] = {0.f, 0.f, 0.f};
      float dud = 0.f;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        dv[a] = vj[a] - vi[a];
        dud = fmaf(dv[a], dx[a], dud);
      }
      const float du = dud * inv_r;                 // u_l - u_r
      const float beta = fminf(fmaxf(du * eta_c, 0.f), 1.f);
      const float rbar = rho0f + 0.5f * (drho_i + drho_j);
      const float p_j = c2 * drho_j;
      // (u* - ubar) / r, branch-free (beta = 0 gives 0)
      const float wr = (beta * beta) * (p_i - p_j) * half_cinv * __fdividef(1.0f, rbar) * inv_r;
      const float p_star = fmaf(0.5f * beta * rbar * c, du, 0.5f * (p_i + p_j));
      float vs[3];
      float sg = 0.f;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        vs[a] = fmaf(-wr, dx[a], fmaf(0.5f, vj[a], hvi[a]));
        sg = fmaf(vs[a], G_[a], sg);
      }
      const float rs2 = -2.0f * rbar * gsc * sg;
      const float pg = -2.0f * p_star * gsc;
      dr += (double)rs2;
#pragma unroll
      for (int a = 0; a < D; ++a)
        dm[a] += (double)fmaf(-mv, dv[a], fmaf(pg, G_[a], rs2 * vs[a]));
    }
    bool finite = isfinite(dr);
#pragma unroll
    for (int a = 0; a < D; ++a) finite = finite && isfinite(dm[a]);
    if (!finite) flags |= SPHB_EFLAG_NONFINITE_FLUX;
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
      float s32[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int a = 0; a < D; ++a) s32[a] = (float)v_new[a];
      s32[D] = (float)(rho_new - P.rho0);
      S32_out[i] = make_float4(s32[0], s32[1], s32[2], s32[3]);
      if (stage == 2) {
        S_out[i] = pack_s<D>(v_new, rho_new);
        double mc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < D; ++a) mc[a] = mom_new[a];
        M_out[i] = make_double4(mc[0], mc[1], mc[2], mc[3]);
        speed = __dadd_rn(c_art, norm_exact<D>(v_new));
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

// FP64 state -> FP32 neighbour record {v, rho - rho0}
template <int D>
__global__ void k_s_to_f32(int64_t n, double rho0, const double4* __restrict__ S,
                           float4* __restrict__ S32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v[D], rho;
  unpack_s<D>(S[i], v, rho);
  float s32[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int a = 0; a < D; ++a) s32[a] = (float)v[a];
  s32[D] = (float)(rho - rho0);
  S32[i] = make_float4(s32[0], s32[1], s32[2], s32[3]);
}

}  // namespace

extern "C" int sphb_wc_stage_f32(const sphb_wc_params* p, int32_t stage, const float* x32,
                                 const float* b32, const int32_t* nbr, const int32_t* cnt,
                                 const float* s32_in, const double* s_n, const double* m_n,
                                 float* s32_out, double* s_out, double* m_out, double* scalars,
                                 int32_t* err, void* stream) {
  if (!p || p->n < 0 || stage < 0 || stage > 2 || p->row0 < 0 || p->nrows < 0 ||
      p->row0 + p->nrows > p->n || !p->uniform_vol || p->wall_tag || p->push_prev || p->push_next)
    return SPHB_ERR_ARG;
  if (p->nrows == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = sphb_blocks(p->nrows, kThreads);
  const size_t smem = (size_t)p->width * kThreads * sizeof(int32_t);
  if (smem > 200 * 1024) return SPHB_ERR_ARG;
#define SPHB_F32(D)                                                                         \
  if (smem > kDynSmemDefault)                                                               \
    SPHB_CUDA_CHECK(cudaFuncSetAttribute(k_wc_stage_f32<D>,                                 \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                         kDynSmemMax));                                     \
  k_wc_stage_f32<D><<<grid, kThreads, smem, st>>>(                                          \
      *p, stage, (const float4*)x32, b32, nbr, cnt, (const float4*)s32_in,                  \
      (const double4*)s_n, (const double4*)m_n, (float4*)s32_out, (double4*)s_out,          \
      (double4*)m_out, scalars, err)
  switch (p->dim) {
    case 1: SPHB_F32(1); break;
    case 2: SPHB_F32(2); break;
    case 3: SPHB_F32(3); break;
    default: return SPHB_ERR_ARG;
  }
#undef SPHB_F32
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_wc_state_to_f32(int64_t n, int32_t dim, double rho0, const double* s,
                                    float* s32, void* stream) {
  if (n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = sphb_blocks(n, 256);
  switch (dim) {
    case 1: k_s_to_f32<1><<<grid, 256, 0, st>>>(n, rho0, (const double4*)s, (float4*)s32); break;
    case 2: k_s_to_f32<2><<<grid, 256, 0, st>>>(n, rho0, (const double4*)s, (float4*)s32); break;
    case 3: k_s_to_f32<3><<<grid, 256, 0, st>>>(n, rho0, (const double4*)s, (float4*)s32); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
