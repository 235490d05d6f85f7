// tile_plan.cu — shared-memory staging plans for static particle sets.
//
// The fluid (eulerian.py) and solid (tlsph.py) particles never move, so the
// neighbourhood of every block of particles is known at set-up.  A tile is P
// consecutive particles in cell-sorted order; because cells are sorted with
// axis 0 fastest, the union of its neighbours is a handful of contiguous
// sorted-index runs (one per neighbouring cell row, split at a periodic
// wrap).  The plan stores those runs per tile and rewrites the ELL pass list
// as uint16 indices into the staged union, so a pass kernel can copy the
// union into shared memory with coalesced loads and then gather per pair
// from shared memory instead of issuing one scattered L1 request per
// neighbour record.
#include <cub/cub.cuh>

#include "common.cuh"

using namespace sphb;

namespace {

constexpr int kRawRuns = 96;

__global__ void k_cell_counts(int64_t ntot, const int32_t* __restrict__ cs,
                              const int32_t* __restrict__ ce, int32_t* __restrict__ cnt) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ntot) cnt[c] = ce[c] - cs[c];
  if (c == ntot) cnt[c] = 0;
}

template <int D>
__device__ __forceinline__ void cell_of(const sphb_grid& g, int64_t n, const double* ws, int64_t s,
                                        int64_t (&c)[3]) {
  c[0] = c[1] = c[2] = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = cell_coord(g, a, ws[(int64_t)a * n + s]);
}

// One thread per tile: runs of the neighbour union + local bases.
template <int D>
__global__ void k_tile_runs(sphb_grid g, int64_t n, const double* __restrict__ ws, int32_t P,
                            int32_t rmax, const int32_t* __restrict__ cell_lo,
                            int32_t* __restrict__ runs, int32_t* __restrict__ meta,
                            int32_t* __restrict__ max_u) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ntiles = (n + P - 1) / P;
  if (t >= ntiles) return;
  const int64_t s0 = t * P;
  const int64_t s1 = (s0 + P < n ? s0 + P : n) - 1;
  int64_t c0[3], c1[3];
  cell_of<D>(g, n, ws, s0, c0);
  cell_of<D>(g, n, ws, s1, c1);
  const int64_t nx = g.ncell[0];
  const int64_t ny = D > 1 ? g.ncell[1] : 1;
  const int64_t nz = D > 2 ? g.ncell[2] : 1;
  const int64_t row0 = c0[1] + ny * c0[2];
  const int64_t row1 = c1[1] + ny * c1[2];
  int32_t rs[kRawRuns], re[kRawRuns];
  int nraw = 0;
  bool ok = (row1 - row0) <= 3;
  for (int64_t row = row0; ok && row <= row1; ++row) {
    const int64_t cy = row % ny, cz = row / ny;
    const int64_t xa = row == row0 ? c0[0] : 0;
    const int64_t xb = row == row1 ? c1[0] : nx - 1;
    const int ny_off = D > 1 ? 3 : 1, nz_off = D > 2 ? 3 : 1;
    for (int oz = 0; oz < nz_off && ok; ++oz) {
      for (int oy = 0; oy < ny_off && ok; ++oy) {
        int64_t y = cy + (D > 1 ? oy - 1 : 0);
        int64_t z = cz + (D > 2 ? oz - 1 : 0);
        if (g.periodic) {
          y = py_mod(y, ny);
          z = py_mod(z, nz);
        } else if (y < 0 || y >= ny || z < 0 || z >= nz) {
          continue;
        }
        const int64_t base = nx * (y + ny * z);
        int64_t lo = xa - 1, hi = xb + 1;  // inclusive cell range along x
        int64_t segs[2][2];
        int nseg = 0;
        if (hi - lo + 1 >= nx) {
          segs[nseg][0] = 0; segs[nseg][1] = nx - 1; ++nseg;
        } else if (g.periodic) {
          if (lo < 0) {
            segs[nseg][0] = 0; segs[nseg][1] = hi; ++nseg;
            segs[nseg][0] = lo + nx; segs[nseg][1] = nx - 1; ++nseg;
          } else if (hi >= nx) {
            segs[nseg][0] = lo; segs[nseg][1] = nx - 1; ++nseg;
            segs[nseg][0] = 0; segs[nseg][1] = hi - nx; ++nseg;
          } else {
            segs[nseg][0] = lo; segs[nseg][1] = hi; ++nseg;
          }
        } else {
          segs[nseg][0] = lo < 0 ? 0 : lo;
          segs[nseg][1] = hi >= nx ? nx - 1 : hi;
          ++nseg;
        }
        for (int q = 0; q < nseg; ++q) {
          const int32_t a = cell_lo[base + segs[q][0]];
          const int32_t b = cell_lo[base + segs[q][1] + 1];
          if (b <= a) continue;
          if (nraw >= kRawRuns) { ok = false; break; }
          rs[nraw] = a; re[nraw] = b; ++nraw;
        }
      }
    }
  }
  // sort by start (insertion sort; nraw is small) and merge overlaps
  for (int a = 1; a < nraw; ++a) {
    int32_t xs = rs[a], xe = re[a];
    int b = a - 1;
    while (b >= 0 && rs[b] > xs) { rs[b + 1] = rs[b]; re[b + 1] = re[b]; --b; }
    rs[b + 1] = xs; re[b + 1] = xe;
  }
  int nrun = 0;
  int32_t* R = runs + t * (int64_t)rmax * 3;
  int32_t usize = 0;
  for (int a = 0; a < nraw && ok; ++a) {
    if (nrun > 0 && rs[a] <= R[(nrun - 1) * 3 + 0] + R[(nrun - 1) * 3 + 1]) {
      int32_t end = R[(nrun - 1) * 3 + 0] + R[(nrun - 1) * 3 + 1];
      if (re[a] > end) {
        usize += re[a] - end;
        R[(nrun - 1) * 3 + 1] = re[a] - R[(nrun - 1) * 3 + 0];
      }
      continue;
    }
    if (nrun >= rmax) { ok = false; break; }
    R[nrun * 3 + 0] = rs[a];
    R[nrun * 3 + 1] = re[a] - rs[a];
    R[nrun * 3 + 2] = usize;
    usize += re[a] - rs[a];
    ++nrun;
  }
  // local bases are assigned in merged order; recompute them (merging may
  // have extended a run after its base was set, which does not move later
  // bases because later runs are appended after the extension)
  int32_t acc = 0;
  for (int a = 0; a < nrun; ++a) { R[a * 3 + 2] = acc; acc += R[a * 3 + 1]; }
  usize = acc;
  // local index of the tile's first particle
  int32_t self = -1;
  for (int a = 0; a < nrun; ++a)
    if (s0 >= R[a * 3] && s0 < R[a * 3] + R[a * 3 + 1]) self = R[a * 3 + 2] + (int32_t)(s0 - R[a * 3]);
  if (self < 0) ok = false;
  int32_t* M = meta + t * 4;
  M[0] = ok ? nrun : 0;
  M[1] = ok ? usize : 0;
  M[2] = self;
  M[3] = ok ? 1 : 0;
  if (ok) atomicMax(max_u, usize);
  else atomicMax(max_u, 0x40000000);  // plan unusable: caller falls back
}

// Rewrite every ELL entry as an index into its tile's staged union.
__global__ void k_tile_local(int64_t n, int32_t P, int32_t rmax, const int32_t* __restrict__ nbr,
                             const int32_t* __restrict__ cnt, const int32_t* __restrict__ runs,
                             const int32_t* __restrict__ meta, uint16_t* __restrict__ lnbr,
                             int32_t* __restrict__ err) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t t = s / P;
  const int32_t* R = runs + t * (int64_t)rmax * 3;
  const int32_t nrun = meta[t * 4];
  const int32_t c = cnt[s];
  for (int32_t k = 0; k < c; ++k) {
    const int32_t j = nbr[(int64_t)k * n + s];
    int32_t l = -1;
    for (int a = 0; a < nrun; ++a) {
      if (j >= R[a * 3] && j < R[a * 3] + R[a * 3 + 1]) {
        l = R[a * 3 + 2] + (j - R[a * 3]);
        break;
      }
    }
    if (l < 0 || l > 0xffff) {
      atomicOr(err, 1);
      l = 0;
    }
    lnbr[(int64_t)k * n + s] = (uint16_t)l;
  }
}

}  // namespace

extern "C" size_t sphb_tile_plan_workspace_bytes(const sphb_grid* g) {
  if (!g) return 0;
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int32_t*)nullptr, (int32_t*)nullptr,
                                (int)(g->ntot + 1));
  return sphb_align(sizeof(int32_t) * (size_t)(g->ntot + 1)) +
         sphb_align(sizeof(int32_t) * (size_t)(g->ntot + 1)) + sphb_align(cub_bytes);
}

extern "C" int sphb_tile_plan(const sphb_grid* g, int64_t n, const double* ws, const int32_t* cs,
                              const int32_t* ce, int32_t P, int32_t rmax, int32_t* runs,
                              int32_t* meta, int32_t* max_u, void* workspace,
                              size_t workspace_bytes, void* stream) {
  if (!g || n <= 0 || P <= 0 || rmax <= 0 || g->ntot + 1 > 0x7fffffffLL) return SPHB_ERR_ARG;
  if (workspace_bytes < sphb_tile_plan_workspace_bytes(g)) return SPHB_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  int32_t* counts = (int32_t*)w;
  int32_t* cell_lo = (int32_t*)(w + sphb_align(sizeof(int32_t) * (size_t)(g->ntot + 1)));
  char* cub_tmp = w + 2 * sphb_align(sizeof(int32_t) * (size_t)(g->ntot + 1));
  size_t cub_bytes = workspace_bytes - 2 * sphb_align(sizeof(int32_t) * (size_t)(g->ntot + 1));
  k_cell_counts<<<sphb_blocks(g->ntot + 1, 256), 256, 0, st>>>(g->ntot, cs, ce, counts);
  SPHB_LAUNCH_CHECK();
  SPHB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, counts, cell_lo,
                                                (int)(g->ntot + 1), st));
  SPHB_CUDA_CHECK(cudaMemsetAsync(max_u, 0, sizeof(int32_t), st));
  const int64_t ntiles = (n + P - 1) / P;
  switch (g->dim) {
    case 1: k_tile_runs<1><<<sphb_blocks(ntiles, 128), 128, 0, st>>>(*g, n, ws, P, rmax, cell_lo, runs, meta, max_u); break;
    case 2: k_tile_runs<2><<<sphb_blocks(ntiles, 128), 128, 0, st>>>(*g, n, ws, P, rmax, cell_lo, runs, meta, max_u); break;
    case 3: k_tile_runs<3><<<sphb_blocks(ntiles, 128), 128, 0, st>>>(*g, n, ws, P, rmax, cell_lo, runs, meta, max_u); break;
    default: return SPHB_ERR_ARG;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_tile_local_nbr(int64_t n, int32_t P, int32_t rmax, const int32_t* nbr,
                                   const int32_t* cnt, const int32_t* runs, const int32_t* meta,
                                   uint16_t* lnbr, int32_t* err, void* stream) {
  if (n <= 0 || P <= 0) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  k_tile_local<<<sphb_blocks(n, 128), 128, 0, st>>>(n, P, rmax, nbr, cnt, runs, meta, lnbr, err);
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
