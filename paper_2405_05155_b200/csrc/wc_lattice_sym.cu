// wc_lattice_sym.cu — pair-symmetric WC stage on a complete 3D lattice
// (the C5 config; slab ranks whose owned rows are whole lattice planes).
//
// Same stage as k_wc_lattice (wc_lattice.cu; reference _rhs_wc,
// eulerian.py:224-266, and the midpoint update, eulerian.py:610-643).  With
// uniform volumes the pair term of _rhs_wc is exactly antisymmetric:
// swapping i and j flips e_ij, so u_l, u_r -> -u_r, -u_l, du, beta, rbar,
// p* and the star velocity vs are unchanged, and s = vs . gwv, the density
// term -2 rbar s and the momentum term -2 (rbar vs s + p* gwv) +
// mu viscv (v_i - v_j) all change sign.  So each unordered pair is
// evaluated ONCE, from the endpoint whose offset lies in the forward half
// stencil H (o_z > 0, or o_z = 0 and o_y > 0, or o_z = o_y = 0 and o_x > 0),
// and credited +c to i and -c to j.  That halves the FP64 pair arithmetic,
// which bounds this kernel (profiles/r02_ncu_c5_256.md).
//
// Work decomposition (deterministic, no atomics on the fields):
//   * a CTA owns an x-segment of a block of Y lattice rows (y) and marches
//     through a chunk of planes (z).  Warp w < Y holds row w; its 32 lanes
//     hold 32 consecutive x, of which lanes [HL, 32 - HR) are owned (the
//     others are x-halo lanes: every pair of an owned particle then lies
//     inside the warp's window);
//   * a slot's partner j = i + o sits in lane t + o_x of row w + o_y, plane
//     z + o_z.  Its -c reaches lane t + o_x by a warp shuffle; slots are
//     ordered by (o_z, o_y) group, each group summed in registers and then
//     routed: same row and plane -> the owner's accumulator; same row,
//     planes z+1 / z+2 -> two pending accumulators carried along the march;
//     other rows -> a shared-memory buffer read after the plane's barrier
//     (double-buffered on plane parity: one barrier per plane);
//   * pairs that cross the block's y edges are evaluated by extra halo
//     warps (rows -1, -2 / Y, Y+1) that compute only the slots landing in
//     owned rows, and pairs that cross the chunk's z start by two warm-up
//     planes, so every owned particle receives each of its pairs exactly
//     once (the CTA that owns the other endpoint evaluates it again for
//     its own side).
// Summation order differs from k_wc_lattice (own slots in canonical order,
// then the received groups); the fields agree to rounding.
#include <stdlib.h>

#include <type_traits>
#include <utility>

#include "wc_common.cuh"

using namespace sphb;
using namespace sphb::wc;

namespace {

constexpr int isqrt_s(int v) {
  int r = 0;
  while ((r + 1) * (r + 1) <= v) ++r;
  return r;
}

// Canonical full stencil (same order as wc_lattice.cu: z slowest, x fastest)
// and its forward half, in canonical order, i.e. grouped by (o_z, o_y).
struct HalfList {
  int nfull;
  int n;                      // |H|
  int full[SPHB_LATTICE_MAXW / 2];
  int o[SPHB_LATTICE_MAXW / 2][3];
  int grp[SPHB_LATTICE_MAXW / 2];       // group id (consecutive)
  int last[SPHB_LATTICE_MAXW / 2];      // 1: last slot of its group
  int ng;                     // groups
  int gdz[16], gdy[16];
  int gbuf[16];               // shared-memory buffer index (-1: register)
  int nbuf;                   // groups with o_y != 0
  int hl, hr;                 // x-halo lanes left / right
  int nhb, nht;               // halo rows below / above
  int maxdz;
};

template <int R2>
constexpr HalfList make_half() {
  HalfList H{};
  const int R = isqrt_s(R2);
  int kf = 0;
  for (int z = -R; z <= R; ++z)
    for (int y = -R; y <= R; ++y)
      for (int x = -R; x <= R; ++x) {
        const int q = x * x + y * y + z * z;
        if (q == 0 || q > R2) continue;
        const bool fwd = z > 0 || (z == 0 && (y > 0 || (y == 0 && x > 0)));
        if (fwd) {
          H.full[H.n] = kf;
          H.o[H.n][0] = x;
          H.o[H.n][1] = y;
          H.o[H.n][2] = z;
          ++H.n;
        }
        ++kf;
      }
  H.nfull = kf;
  H.ng = 0;
  H.nbuf = 0;
  for (int h = 0; h < H.n; ++h) {
    const bool newg = h == 0 || H.o[h][2] != H.o[h - 1][2] || H.o[h][1] != H.o[h - 1][1];
    if (newg) {
      H.gdz[H.ng] = H.o[h][2];
      H.gdy[H.ng] = H.o[h][1];
      H.gbuf[H.ng] = H.o[h][1] != 0 ? H.nbuf++ : -1;
      ++H.ng;
    }
    H.grp[h] = H.ng - 1;
  }
  for (int h = 0; h < H.n; ++h) H.last[h] = h + 1 == H.n || H.grp[h + 1] != H.grp[h];
  H.hl = H.hr = H.nhb = H.nht = H.maxdz = 0;
  for (int h = 0; h < H.n; ++h) {
    const int ox = H.o[h][0], oy = H.o[h][1], oz = H.o[h][2];
    if (ox > H.hl) H.hl = ox;
    if (-ox > H.hr) H.hr = -ox;
    if (oy > H.nhb) H.nhb = oy;
    if (-oy > H.nht) H.nht = -oy;
    if (oz > H.maxdz) H.maxdz = oz;
  }
  return H;
}

template <int R2>
constexpr HalfList kHalf = make_half<R2>();

template <int R2>
struct HalfStencil {
  static constexpr HalfList H = kHalf<R2>;
  static constexpr int R = isqrt_s(R2);
  static constexpr int NH = H.n;
  static constexpr int NBUF = H.nbuf;
  static constexpr int HL = H.hl, HR = H.hr;
  static constexpr int NHB = H.nhb, NHT = H.nht;
  static constexpr int OWN = 32 - HL - HR;     // owned lanes per warp
  static constexpr int MAXDZ = H.maxdz;
};

template <class F, int... Is>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int K, class F>
__device__ __forceinline__ void sfor(F&& f) {
  sfor_impl(f, std::make_integer_sequence<int, K>{});
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

struct LatConstS {
  double c2, c2rho0, eta_c, hc;
};

__device__ __forceinline__ int wrap_mod(int v, int n) {
  v %= n;
  return v < 0 ? v + n : v;
}

// Shift a value from lane t - s to lane t (s > 0: up, s < 0: down); lanes
// whose source falls outside the warp get their own value (never used: they
// are x-halo lanes).
template <int S>
__device__ __forceinline__ double lane_shift(double v) {
  if constexpr (S > 0) return __shfl_up_sync(0xffffffffu, v, S);
  else if constexpr (S < 0) return __shfl_down_sync(0xffffffffu, v, -S);
  else return v;
}

struct Acc4 {
  double r, m0, m1, m2;
  __device__ __forceinline__ void zero() { r = m0 = m1 = m2 = 0.0; }
  __device__ __forceinline__ void add(const Acc4& o) {
    r += o.r; m0 += o.m0; m1 += o.m1; m2 += o.m2;
  }
};

// The pair term c(i, j) of _rhs_wc at full-stencil slot K (compile-time
// offset O) with the per-slot table geometry of sphb_lattice (same
// arithmetic as k_wc_lattice's pair body, c returned instead of summed).
template <int K, int OX, int OY, int OZ>
__device__ __forceinline__ void pair_c(const LatConstS& KC, const sphb_lattice& L,
                                       const double (&vi)[3], double rho_i, double hrho_i,
                                       const Sym<3>& Bi, const double4 sj, const Sym<3>& Bj,
                                       Acc4& c) {
  constexpr int o[3] = {OX, OY, OZ};
  const double vj[3] = {sj.x, sj.y, sj.z};
  const double rho_j = sj.w;
  Sym<3> Bs;
  Bi.add(Bj, Bs);
  double dx[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) dx[q] = o[q] == 0 ? 0.0 : L.dx[K][q];
  const double inv_r = L.inv_r[K];
  double G_[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    double acc = 0.0;
    bool first = true;
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (o[q] != 0) {
        acc = first ? Bs.at(r, q) * dx[q] : fma(Bs.at(r, q), dx[q], acc);
        first = false;
      }
    G_[r] = acc;
  }
  double dv[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) dv[q] = vj[q] - vi[q];
  double dud = 0.0;
#pragma unroll
  for (int q = 0; q < 3; ++q)
    if (o[q] != 0) dud = fma(dv[q], dx[q], dud);
  const double du = dud * inv_r;                   // u_l - u_r (eulerian.py:236-243)
  double beta = du * KC.eta_c;
  beta = beta < 0.0 ? 0.0 : (beta > 1.0 ? 1.0 : beta);
  const double rbar = fma(0.5, rho_j, hrho_i);
  const double bh = beta * KC.hc;
  const double wr = ((beta * bh) * (rho_i - rho_j)) * (rcp_nr(rbar) * inv_r);
  const double p_star = fma(bh * rbar, du, fma(KC.c2, rbar, -KC.c2rho0));
  double vs[3];
  double sg = 0.0;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double vb = fma(0.5, dv[q], vi[q]);
    vs[q] = o[q] == 0 ? vb : fma(-wr, dx[q], vb);
    sg = fma(vs[q], G_[q], sg);
  }
  const double rs2 = rbar * (L.g2[K] * sg);        // -2 rbar s
  const double pg = p_star * L.g2[K];               // -2 p* gsc
  c.r = rs2;
  c.m0 = fma(-L.mv[K], dv[0], fma(pg, G_[0], rs2 * vs[0]));
  c.m1 = fma(-L.mv[K], dv[1], fma(pg, G_[1], rs2 * vs[1]));
  c.m2 = fma(-L.mv[K], dv[2], fma(pg, G_[2], rs2 * vs[2]));
}

// Work items: (x segment, y block, z chunk), x fastest.
struct SymGrid {
  int nxs, nyb, nzc;
  int yb;              // owned rows per block (<= Y)
  int zc;              // planes per chunk
  int z0, z1;          // owned planes [z0, z1)
  int probe;           // timing probe only (SPHB_SYM_PROBE=1): gathers read row i
};

template <int R2, int Y>
struct SymCfg {
  using HS = HalfStencil<R2>;
  static constexpr int NW = Y + HS::NHB + HS::NHT;   // warps per CTA
  static constexpr int NT = NW * 32;
  // double4 buffers: [parity][buffer][target row][lane]
  static constexpr size_t SMEM = (size_t)2 * HS::NBUF * Y * 32 * sizeof(double4);
};

template <int R2, int Y, int MINB>
__global__ void __launch_bounds__(SymCfg<R2, Y>::NT, MINB)
k_wc_lattice_sym(const sphb_wc_params P, const LatConstS KC, const sphb_lattice L,
                 const SymGrid G, const int stage, const double* __restrict__ B,
                 const double4* __restrict__ S_in, const double4* Sn, const double4* Mn,
                 double4* S_out, double4* M_out, double* __restrict__ scalars,
                 int32_t* __restrict__ err) {
  using HS = HalfStencil<R2>;
#define H kHalf<R2>
  constexpr int R = HS::R;
  extern __shared__ double4 sbuf[];
  auto buf = [&](int par, int b, int row, int lane) -> double4& {
    return sbuf[((par * HS::NBUF + b) * Y + row) * 32 + lane];
  };

  const int n0 = L.n[0], n1 = L.n[1], n2 = L.n[2];
  const int64_t n = P.n;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;

  int item = blockIdx.x;
  const int xseg = item % G.nxs;
  item /= G.nxs;
  const int yblk = item % G.nyb;
  const int zchk = item / G.nyb;
  const int yb0 = yblk * G.yb;
  const int yb = min(G.yb, n1 - yb0);                 // owned rows of this block
  const int zc0 = G.z0 + zchk * G.zc;
  const int zc1 = min(zc0 + G.zc, G.z1);

  // local row of this warp: [0, Y) owned rows, then the halo rows
  // -1 .. -NHB and yb .. yb + NHT - 1
  int lr;
  bool owned_warp;
  if (warp < Y) {
    lr = warp;
    owned_warp = true;
  } else if (warp < Y + HS::NHB) {
    lr = -(warp - Y + 1);
    owned_warp = false;
  } else {
    lr = yb + (warp - Y - HS::NHB);
    owned_warp = false;
  }
  const bool active = !owned_warp || lr < yb;         // idle warps only sync
  const int y = wrap_mod(yb0 + lr, n1);

  // lanes: x = xs0 - HL + lane; owned lanes [HL, HL + OWN) inside the row
  const int xoff = xseg * HS::OWN + lane - HS::HL;
  const bool own_lane = lane >= HS::HL && lane < HS::HL + HS::OWN && xoff < n0;
  const int x = wrap_mod(xoff, n0);
  int xs[2 * R + 1], ys[2 * R + 1];
#pragma unroll
  for (int s = -R; s <= R; ++s) {
    xs[s + R] = wrap_mod(x + s, n0);
    ys[s + R] = n0 * wrap_mod(y + s, n1);
  }
  const int plane = n0 * n1;
  const double c = P.c_art;

  Acc4 P1, P2;
  P1.zero();
  P2.zero();
  double speed = 0.0;
  int32_t flags = 0;
  int par = 0;

  for (int zz = zc0 - HS::MAXDZ; zz < zc1; ++zz) {
    const int z = wrap_mod(zz, n2);
    int zs[HS::MAXDZ + 1];
#pragma unroll
    for (int s = 0; s <= HS::MAXDZ; ++s) zs[s] = plane * wrap_mod(z + s, n2);
    const int64_t i = (int64_t)xs[R] + ys[R] + zs[0];

    // prefetch: the epilogue's own-state records two planes ahead and the
    // records first gathered two planes ahead (slot (0, 0, 2) of the next
    // plane) into L2; the epilogue's records of the next plane into L1.
    // All warps of the CTA reach the epilogue together after the barrier,
    // so its DRAM latency would otherwise be exposed once per plane.
    if (active && zz + 1 < zc1) {
      const int64_t i1 = (int64_t)xs[R] + ys[R] + plane * wrap_mod(z + 1, n2);
      const int64_t i2 = (int64_t)xs[R] + ys[R] + plane * wrap_mod(z + 2, n2);
      const int64_t i3 = (int64_t)xs[R] + ys[R] + plane * wrap_mod(z + 3, n2);
      if (stage > 0) {
        prefetch_l1(Sn + i1);
        prefetch_l2(Sn + i2);
        if (stage == 2) {
          prefetch_l1(Mn + i1);
          prefetch_l2(Mn + i2);
        }
      }
      prefetch_l2(S_in + i3);
      prefetch_l2(reinterpret_cast<const double4*>(B) + i3);
      prefetch_l2(reinterpret_cast<const double2*>(B + 4 * n) + i3);
    }
    Acc4 own = P1;
    P1 = P2;
    P2.zero();
    if (active) {
      double vi[3], rho_i;
      unpack_s<3>(S_in[i], vi, rho_i);
      Sym<3> Bi;
      Bi.load(B, n, i);
      const double hrho_i = 0.5 * rho_i;
      Acc4 gs;
      gs.zero();
      if (owned_warp) {
        sfor<HS::NH>([&](auto hc) {
          constexpr int h = decltype(hc)::value;
          constexpr int K = H.full[h];
          constexpr int OX = H.o[h][0], OY = H.o[h][1], OZ = H.o[h][2];
          constexpr int g = H.grp[h];
          int64_t j = (int64_t)xs[OX + R] + ys[OY + R] + zs[OZ];
          j = G.probe ? i : j;
          Sym<3> Bj;
          Bj.load(B, n, j);
          Acc4 cc;
          pair_c<K, OX, OY, OZ>(KC, L, vi, rho_i, hrho_i, Bi, ldg4(S_in + j), Bj, cc);
          own.add(cc);
          gs.r -= lane_shift<OX>(cc.r);
          gs.m0 -= lane_shift<OX>(cc.m0);
          gs.m1 -= lane_shift<OX>(cc.m1);
          gs.m2 -= lane_shift<OX>(cc.m2);
          if constexpr (H.last[h]) {
            constexpr int dz = H.gdz[g], dy = H.gdy[g], b = H.gbuf[g];
            if constexpr (dy == 0) {
              if constexpr (dz == 0) own.add(gs);
              else if constexpr (dz == 1) P1.add(gs);
              else P2.add(gs);
            } else {
              const int tr = lr + dy;
              if (tr >= 0 && tr < yb)
                buf(par, b, tr, lane) = make_double4(gs.r, gs.m0, gs.m1, gs.m2);
            }
            gs.zero();
          }
        });
      } else {
        // halo row: only the slots whose partner row lies in [0, yb)
        sfor<HS::NH>([&](auto hc) {
          constexpr int h = decltype(hc)::value;
          constexpr int OY = H.o[h][1];
          if constexpr (OY != 0) {
            constexpr int K = H.full[h];
            constexpr int OX = H.o[h][0], OZ = H.o[h][2];
            constexpr int g = H.grp[h];
            const int tr = lr + OY;
            if (tr >= 0 && tr < yb) {
              const int64_t j = (int64_t)xs[OX + R] + ys[OY + R] + zs[OZ];
              Sym<3> Bj;
              Bj.load(B, n, j);
              Acc4 cc;
              pair_c<K, OX, OY, OZ>(KC, L, vi, rho_i, hrho_i, Bi, ldg4(S_in + j), Bj, cc);
              gs.r -= lane_shift<OX>(cc.r);
              gs.m0 -= lane_shift<OX>(cc.m0);
              gs.m1 -= lane_shift<OX>(cc.m1);
              gs.m2 -= lane_shift<OX>(cc.m2);
              if constexpr (H.last[h]) {
                constexpr int b = H.gbuf[g];
                buf(par, b, tr, lane) = make_double4(gs.r, gs.m0, gs.m1, gs.m2);
                gs.zero();
              }
            }
          }
        });
      }
    }
    __syncthreads();
    if (owned_warp && lr < yb) {
      // received groups (other rows), fixed order
      sfor<H.ng>([&](auto gc) {
        constexpr int g = decltype(gc)::value;
        constexpr int dz = H.gdz[g], dy = H.gdy[g], b = H.gbuf[g];
        if constexpr (dy != 0) {
          const double4 v = buf(par, b, lr, lane);
          Acc4 a{v.x, v.y, v.z, v.w};
          if constexpr (dz == 0) own.add(a);
          else if constexpr (dz == 1) P1.add(a);
          else P2.add(a);
        }
      });
      if (own_lane && zz >= zc0) {
        const double dm[3] = {own.m0, own.m1, own.m2};
        wc_update<3>(P, stage, i, c, own.r, dm, Sn, Mn, S_out, M_out, scalars, speed, flags);
      }
    }
    par ^= 1;
  }
  if (stage == 2) wc_speed_fold<SymCfg<R2, Y>::NT>(speed, scalars);
  if (flags) atomicOr(err, flags);
#undef H
}

}  // namespace

// Launch the pair-symmetric kernel when the set qualifies: 3D, (r2 = 4 or
// 6), every lattice axis at least as long as the warp window / block plus
// its halo, and [row0, row0 + nrows) whole planes.  Returns SPHB_ERR_ARG
// (nothing launched) otherwise; sphb_wc_stage_lattice then runs
// k_wc_lattice.
extern "C" int sphb_wc_stage_lattice_sym(const sphb_wc_params* p, const sphb_lattice* L,
                                         int32_t stage, const double* b, const double* s_in,
                                         const double* s_n, const double* m_n, double* s_out,
                                         double* m_out, double* scalars, int32_t* err,
                                         void* stream) {
  if (!p || !L || p->dim != 3 || (L->r2 != 4 && L->r2 != 6) || stage < 0 || stage > 2 ||
      p->interior || p->wall_tag || !p->uniform_vol || p->n <= 0 || p->n >= ((int64_t)1 << 31))
    return SPHB_ERR_ARG;
  const int n0 = L->n[0], n1 = L->n[1], n2 = L->n[2];
  if ((int64_t)n0 * n1 * n2 != p->n) return SPHB_ERR_ARG;
  const int64_t plane = (int64_t)n0 * n1;
  if (p->row0 % plane || p->nrows % plane || p->row0 + p->nrows > p->n) return SPHB_ERR_ARG;
  if (p->nrows == 0) return SPHB_OK;
  static const int y_env = [] {
    const char* e = getenv("SPHB_SYM_Y");
    return e ? atoi(e) : 0;
  }();
  const bool r4 = L->r2 == 4;
  const int Y = r4 && y_env == 4 ? 4 : 8;
  const int hl = r4 ? HalfStencil<4>::HL : HalfStencil<6>::HL;
  const int hr = r4 ? HalfStencil<4>::HR : HalfStencil<6>::HR;
  const int nhb = r4 ? HalfStencil<4>::NHB : HalfStencil<6>::NHB;
  const int nht = r4 ? HalfStencil<4>::NHT : HalfStencil<6>::NHT;
  const int own = 32 - hl - hr;
  // the warp window (32 x) and the block rows with their halo rows must
  // not alias periodic images; the march needs distinct z + 0..2 planes
  if (n0 < 32 || n1 < 1 + nhb + nht + 1 || n2 < 5) return SPHB_ERR_ARG;
  static const int zc_env = [] {
    const char* e = getenv("SPHB_SYM_ZC");
    return e ? atoi(e) : 0;
  }();
  static const int probe_env = [] {
    const char* e = getenv("SPHB_SYM_PROBE");
    return e ? atoi(e) : 0;
  }();
  SymGrid G;
  G.probe = probe_env;
  G.yb = n1 - nhb - nht >= Y ? Y : n1 - nhb - nht;
  G.nxs = (n0 + own - 1) / own;
  G.nyb = (n1 + G.yb - 1) / G.yb;
  G.z0 = (int)(p->row0 / plane);
  G.z1 = (int)((p->row0 + p->nrows) / plane);
  const int nz = G.z1 - G.z0;
  int zc = zc_env > 0 ? zc_env : 32;
  if (zc > nz) zc = nz;
  G.zc = zc;
  G.nzc = (nz + zc - 1) / zc;
  const int64_t items = (int64_t)G.nxs * G.nyb * G.nzc;
  if (items >= ((int64_t)1 << 31)) return SPHB_ERR_ARG;
  LatConstS K;
  K.c2 = p->c_art * p->c_art;
  K.c2rho0 = K.c2 * p->rho0;
  K.eta_c = kEtaLinearized / p->c_art;
  K.hc = 0.5 * p->c_art;
  cudaStream_t st = (cudaStream_t)stream;
  const double4* Sin = (const double4*)s_in;
  const double4* Sn = (const double4*)s_n;
  const double4* Mn = (const double4*)m_n;
  double4* Sout = (double4*)s_out;
  double4* Mout = (double4*)m_out;
#define SPHB_SYM(R2, YY, MB)                                                                \
  {                                                                                         \
    using C = SymCfg<R2, YY>;                                                               \
    static const bool attr_ok = [] {                                                        \
      return cudaFuncSetAttribute(k_wc_lattice_sym<R2, YY, MB>,                             \
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                                  (int)C::SMEM) == cudaSuccess;                             \
    }();                                                                                    \
    if (!attr_ok) return SPHB_ERR_CUDA;                                                     \
    k_wc_lattice_sym<R2, YY, MB><<<(unsigned)items, C::NT, C::SMEM, st>>>(                  \
        *p, K, *L, G, stage, b, Sin, Sn, Mn, Sout, Mout, scalars, err);                     \
  }
  if (r4 && Y == 4) SPHB_SYM(4, 4, 2)
  else if (r4) SPHB_SYM(4, 8, 1)
  else SPHB_SYM(6, 8, 1)
#undef SPHB_SYM
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
