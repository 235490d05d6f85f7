// neighbors.cu — cell binning, CSR export and engine pass lists.
//
// Replaces the reference's cell-linked list (neighbors.py:171-210 with
// _cell_index :38-53 and _search :56-168).  The reference builds head/next
// chains with a reversed counting sort so chains run in ascending index; the
// B200 design replaces that with a stable LSD radix sort of (cell key,
// index) pairs — identical cell contents in identical order — plus
// cell_start/cell_end tables, so every row is enumerated in exactly the
// reference's order and the CSR written here is byte-identical to the
// reference's.
#include <cub/cub.cuh>

#include "common.cuh"

using namespace sphb;

// --------------------------------------------------------------- binning
template <int D>
__global__ void k_wrap_key(sphb_grid g, const double* __restrict__ pos, int64_t n,
                           double* __restrict__ wrapped_aos, uint32_t* __restrict__ key,
                           int32_t* __restrict__ val) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t flat = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double p = pos[i * D + a];
    double w = g.periodic ? np_remainder(p, g.box[a]) : __dsub_rn(p, g.lo[a]);
    wrapped_aos[i * D + a] = w;
    flat += cell_coord(g, a, w) * g.sstrides[a];   // storage key
  }
  key[i] = (uint32_t)flat;
  val[i] = (int32_t)i;
}

template <int D>
__global__ void k_gather_sorted(int64_t n, const double* __restrict__ wrapped_aos,
                                const int32_t* __restrict__ perm, double* __restrict__ ws) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  int64_t i = perm[s];
#pragma unroll
  for (int a = 0; a < D; ++a) ws[(int64_t)a * n + s] = wrapped_aos[i * D + a];
}

// storage key -> reference flat key (identity when slow_axis == dim - 1)
__device__ __forceinline__ int64_t ref_key(const sphb_grid& g, uint32_t skey) {
  if (g.slow_axis == g.dim - 1) return skey;
  int64_t ref = 0;
  for (int a = 0; a < g.dim; ++a) ref += ((int64_t)skey / g.sstrides[a] % g.ncell[a]) * g.strides[a];
  return ref;
}

__global__ void k_cell_ranges(sphb_grid g, int64_t n, const uint32_t* __restrict__ key,
                              int32_t* __restrict__ cs, int32_t* __restrict__ ce) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  uint32_t k = key[s];
  if (s == 0 || key[s - 1] != k) cs[ref_key(g, k)] = (int32_t)s;
  if (s == n - 1 || key[s + 1] != k) ce[ref_key(g, k)] = (int32_t)(s + 1);
}

// Small sets (C1, the relaxation loop: 10k particles rebinned every update):
// the whole binning in ONE block — wrap + key, cell counts in shared memory,
// exclusive scan, scatter, per-cell sort by original index (= the stable
// radix sort's order), cell tables, gather — instead of ~8 launches.
constexpr int kSmallBinThreads = 1024;
constexpr int64_t kSmallBinMaxN = 16384;
constexpr int64_t kSmallBinMaxCells = 8192;

template <int D>
__global__ void __launch_bounds__(kSmallBinThreads)
k_bin_small(sphb_grid g, int64_t n, const double* __restrict__ wrapped,
            const uint32_t* __restrict__ keys, int32_t* __restrict__ perm, int32_t* __restrict__ cs,
            int32_t* __restrict__ ce, double* __restrict__ ws) {
  constexpr int KPT = (int)(kSmallBinMaxN / kSmallBinThreads);   // particles per thread
  extern __shared__ int32_t sm[];
  const int ntot = (int)g.ntot;
  int32_t* count = sm;                  // [ntot]
  int32_t* fill = sm + ntot;            // [ntot]
  int32_t* sperm = sm + 2 * ntot;       // [n]
  const int tid = threadIdx.x;
  for (int c = tid; c < ntot; c += blockDim.x) count[c] = 0;
  __syncthreads();
  // keys and wrapped coordinates come from k_wrap_key (all SMs)
  uint32_t key[KPT];
#pragma unroll
  for (int q = 0; q < KPT; ++q) {
    const int64_t i = tid + (int64_t)q * kSmallBinThreads;
    key[q] = i < n ? keys[i] : 0u;
  }
#pragma unroll
  for (int q = 0; q < KPT; ++q) {
    const int64_t i = tid + (int64_t)q * kSmallBinThreads;
    if (i < n) atomicAdd(count + key[q], 1);
  }
  __syncthreads();
  // exclusive scan: each thread a contiguous chunk, chunk totals scanned by warp 0
  __shared__ int32_t part[kSmallBinThreads];
  const int chunk = (ntot + blockDim.x - 1) / blockDim.x;
  const int c0 = min(tid * chunk, ntot), c1 = min(c0 + chunk, ntot);
  int32_t tot = 0;
  for (int c = c0; c < c1; ++c) tot += count[c];
  part[tid] = tot;
  __syncthreads();
  if (tid < 32) {
    int32_t run = 0;
    for (int b = 0; b < (int)blockDim.x; b += 32) {
      int32_t v = part[b + tid];
      const int32_t mine = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (tid >= o) v += u;
      }
      part[b + tid] = v - mine + run;          // exclusive
      run += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  int32_t off = part[tid];
  for (int c = c0; c < c1; ++c) {
    const int32_t k = count[c];
    fill[c] = off;
    // every cell's range, empty ones as [off, off) (no memset of the
    // tables needed before this kernel)
    const int64_t r = g.slow_axis == g.dim - 1 ? c : ref_key(g, (uint32_t)c);
    cs[r] = off;
    ce[r] = off + k;
    off += k;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < KPT; ++q) {
    const int64_t i = tid + (int64_t)q * kSmallBinThreads;
    if (i < n) sperm[atomicAdd(fill + key[q], 1)] = (int32_t)i;
  }
  __syncthreads();
  // ascending original index inside each cell (cells hold a handful of particles)
  for (int c = c0; c < c1; ++c) {
    const int32_t e = fill[c], b = e - count[c];
    for (int32_t s = b + 1; s < e; ++s) {
      const int32_t v = sperm[s];
      int32_t t = s;
      while (t > b && sperm[t - 1] > v) {
        sperm[t] = sperm[t - 1];
        --t;
      }
      sperm[t] = v;
    }
  }
  __syncthreads();
  // gathers issued four rows at a time before their stores (fewer
  // dependent L2 round trips per thread)
  constexpr int QB = 4;
#pragma unroll
  for (int q0 = 0; q0 < KPT; q0 += QB) {
    if (tid + (int64_t)q0 * kSmallBinThreads >= n) break;
    int32_t src[QB];
    double wv[QB][D];
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      const int64_t s = tid + (int64_t)(q0 + q) * kSmallBinThreads;
      src[q] = s < n ? sperm[s] : 0;
    }
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      const int64_t s = tid + (int64_t)(q0 + q) * kSmallBinThreads;
#pragma unroll
      for (int a = 0; a < D; ++a) wv[q][a] = s < n ? wrapped[(int64_t)src[q] * D + a] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      const int64_t s = tid + (int64_t)(q0 + q) * kSmallBinThreads;
      if (s < n) {
        perm[s] = src[q];
#pragma unroll
        for (int a = 0; a < D; ++a) ws[(int64_t)a * n + s] = wv[q][a];
      }
    }
  }
}

static bool grid_ok(const sphb_grid* g) {
  if (!g || g->dim < 1 || g->dim > 3) return false;
  if (g->slow_axis < 0 || g->slow_axis >= g->dim) return false;
  if (g->ntot < 1 || g->ntot > 0x7fffffffLL) return false;
  return true;
}

struct BinLayout {
  size_t keys_in, keys_out, vals_in, wrapped, cub, total;
};

static BinLayout bin_layout(int64_t n, int dim) {
  BinLayout L;
  size_t off = 0;
  L.keys_in = off;  off += sphb_align(sizeof(uint32_t) * (size_t)n);
  L.keys_out = off; off += sphb_align(sizeof(uint32_t) * (size_t)n);
  L.vals_in = off;  off += sphb_align(sizeof(int32_t) * (size_t)n);
  L.wrapped = off;  off += sphb_align(sizeof(double) * (size_t)n * dim);
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs<uint32_t, int32_t>(nullptr, cub_bytes, (uint32_t*)nullptr,
                                                     (uint32_t*)nullptr, (int32_t*)nullptr,
                                                     (int32_t*)nullptr, (int)n, 0, 32);
  L.cub = off;      off += sphb_align(cub_bytes);
  L.total = off;
  return L;
}

static int end_bit_for(int64_t ntot) {
  int b = 1;
  while (b < 32 && ((int64_t)1 << b) < ntot) ++b;
  return b;
}

extern "C" size_t sphb_bin_workspace_bytes(int64_t n, const sphb_grid* g) {
  if (!grid_ok(g) || n < 0) return 0;
  return bin_layout(n > 0 ? n : 1, g->dim).total;
}

extern "C" int sphb_bin(const sphb_grid* g, const double* pos, int64_t n, double* ws,
                        int32_t* perm, int32_t* cs, int32_t* ce, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (!grid_ok(g) || n < 0 || n > 0x7fffffffLL) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const bool small = n > 0 && n <= kSmallBinMaxN && g->ntot <= kSmallBinMaxCells;
  if (!small) {   // the single-block path writes every cell's range itself
    SPHB_CUDA_CHECK(cudaMemsetAsync(cs, 0, sizeof(int32_t) * (size_t)g->ntot, st));
    SPHB_CUDA_CHECK(cudaMemsetAsync(ce, 0, sizeof(int32_t) * (size_t)g->ntot, st));
  }
  if (n == 0) return SPHB_OK;
  BinLayout L = bin_layout(n, g->dim);
  if (workspace_bytes < L.total) return SPHB_ERR_WORKSPACE;
  char* w = (char*)workspace;
  uint32_t* keys_in = (uint32_t*)(w + L.keys_in);
  uint32_t* keys_out = (uint32_t*)(w + L.keys_out);
  int32_t* vals_in = (int32_t*)(w + L.vals_in);
  double* wrapped = (double*)(w + L.wrapped);
  if (small) {
    const size_t smem = sizeof(int32_t) * (2 * (size_t)g->ntot + (size_t)n);
    if (smem > kDynSmemDefault) {
      // one fixed bound for every call: the attribute is per function, so a
      // per-call value could be lowered by another host thread between this
      // thread's set and launch (slab ranks of different sizes)
      const int bound = (int)(sizeof(int32_t) * (2 * kSmallBinMaxCells + kSmallBinMaxN));
      SPHB_CUDA_CHECK(cudaFuncSetAttribute(k_bin_small<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bound));
      SPHB_CUDA_CHECK(cudaFuncSetAttribute(k_bin_small<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bound));
      SPHB_CUDA_CHECK(cudaFuncSetAttribute(k_bin_small<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bound));
    }
    const int T = 256;
    switch (g->dim) {
      case 1: k_wrap_key<1><<<sphb_blocks(n, T), T, 0, st>>>(*g, pos, n, wrapped, keys_in, vals_in); break;
      case 2: k_wrap_key<2><<<sphb_blocks(n, T), T, 0, st>>>(*g, pos, n, wrapped, keys_in, vals_in); break;
      default: k_wrap_key<3><<<sphb_blocks(n, T), T, 0, st>>>(*g, pos, n, wrapped, keys_in, vals_in); break;
    }
    switch (g->dim) {
      case 1: k_bin_small<1><<<1, kSmallBinThreads, smem, st>>>(*g, n, wrapped, keys_in, perm, cs, ce, ws); break;
      case 2: k_bin_small<2><<<1, kSmallBinThreads, smem, st>>>(*g, n, wrapped, keys_in, perm, cs, ce, ws); break;
      default: k_bin_small<3><<<1, kSmallBinThreads, smem, st>>>(*g, n, wrapped, keys_in, perm, cs, ce, ws); break;
    }
    SPHB_LAUNCH_CHECK();
    return SPHB_OK;
  }
  const int T = 256;
  switch (g->dim) {
    case 1: k_wrap_key<1><<<sphb_blocks(n, T), T, 0, st>>>(*g, pos, n, wrapped, keys_in, vals_in); break;
    case 2: k_wrap_key<2><<<sphb_blocks(n, T), T, 0, st>>>(*g, pos, n, wrapped, keys_in, vals_in); break;
    default: k_wrap_key<3><<<sphb_blocks(n, T), T, 0, st>>>(*g, pos, n, wrapped, keys_in, vals_in); break;
  }
  SPHB_LAUNCH_CHECK();
  size_t cub_bytes = workspace_bytes - L.cub;
  SPHB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(w + L.cub, cub_bytes, keys_in, keys_out, vals_in,
                                                  perm, (int)n, 0, end_bit_for(g->ntot), st));
  k_cell_ranges<<<sphb_blocks(n, T), T, 0, st>>>(*g, n, keys_out, cs, ce);
  SPHB_LAUNCH_CHECK();
  switch (g->dim) {
    case 1: k_gather_sorted<1><<<sphb_blocks(n, T), T, 0, st>>>(n, wrapped, perm, ws); break;
    case 2: k_gather_sorted<2><<<sphb_blocks(n, T), T, 0, st>>>(n, wrapped, perm, ws); break;
    default: k_gather_sorted<3><<<sphb_blocks(n, T), T, 0, st>>>(n, wrapped, perm, ws); break;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

// ------------------------------------------------------------------- CSR
template <int D>
__global__ void k_csr_count(sphb_grid g, int64_t n, const double* __restrict__ ws,
                            const int32_t* __restrict__ perm, const int32_t* __restrict__ cs,
                            const int32_t* __restrict__ ce, int64_t* __restrict__ counts_orig) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  int64_t c = 0;
  for_each_neighbor<D>(g, n, ws, cs, ce, (int32_t)s,
                       [&](int32_t, const double*, double) { ++c; });
  counts_orig[perm[s]] = c;
}

extern "C" size_t sphb_csr_workspace_bytes(int64_t n) {
  size_t cub_bytes = 0;
  int64_t nn = n > 0 ? n : 1;
  cub::DeviceScan::InclusiveSum(nullptr, cub_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)nn);
  return sphb_align(sizeof(int64_t) * (size_t)nn) + sphb_align(cub_bytes);
}

extern "C" int sphb_csr_starts(const sphb_grid* g, int64_t n, const double* ws,
                               const int32_t* perm, const int32_t* cs, const int32_t* ce,
                               int64_t* starts, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (!grid_ok(g) || n < 0) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_CUDA_CHECK(cudaMemsetAsync(starts, 0, sizeof(int64_t), st));
  if (n == 0) return SPHB_OK;
  if (workspace_bytes < sphb_csr_workspace_bytes(n)) return SPHB_ERR_WORKSPACE;
  int64_t* counts = (int64_t*)workspace;
  char* cub_tmp = (char*)workspace + sphb_align(sizeof(int64_t) * (size_t)n);
  size_t cub_bytes = workspace_bytes - sphb_align(sizeof(int64_t) * (size_t)n);
  const int T = 128;
  switch (g->dim) {
    case 1: k_csr_count<1><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, perm, cs, ce, counts); break;
    case 2: k_csr_count<2><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, perm, cs, ce, counts); break;
    default: k_csr_count<3><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, perm, cs, ce, counts); break;
  }
  SPHB_LAUNCH_CHECK();
  SPHB_CUDA_CHECK(cub::DeviceScan::InclusiveSum(cub_tmp, cub_bytes, counts, starts + 1, (int)n, st));
  return SPHB_OK;
}

template <int D>
__global__ void k_csr_fill(sphb_grid g, int64_t n, const double* __restrict__ ws,
                           const int32_t* __restrict__ perm, const int32_t* __restrict__ cs,
                           const int32_t* __restrict__ ce, const int64_t* __restrict__ starts,
                           int32_t* __restrict__ idx, double* __restrict__ r,
                           double* __restrict__ e) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  int64_t w = starts[perm[s]];
  for_each_neighbor<D>(g, n, ws, cs, ce, (int32_t)s, [&](int32_t t, const double* dx, double r2) {
    double dist = __dsqrt_rn(r2);
    idx[w] = perm[t];
    r[w] = dist;
#pragma unroll
    for (int a = 0; a < D; ++a) e[w * D + a] = __ddiv_rn(dx[a], dist);
    ++w;
  });
}

extern "C" int sphb_csr_fill(const sphb_grid* g, int64_t n, const double* ws, const int32_t* perm,
                             const int32_t* cs, const int32_t* ce, const int64_t* starts,
                             int32_t* idx, double* r, double* e, void* stream) {
  if (!grid_ok(g) || n < 0) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  switch (g->dim) {
    case 1: k_csr_fill<1><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, perm, cs, ce, starts, idx, r, e); break;
    case 2: k_csr_fill<2><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, perm, cs, ce, starts, idx, r, e); break;
    default: k_csr_fill<3><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, perm, cs, ce, starts, idx, r, e); break;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

// ------------------------------------------------------------------- ELL
// Pair kept iff the passes would not skip it: q = r/h <= kappa with r and q
// rounded exactly like correction.py:99-101 (r = sqrt(r2), q = r / h).
__device__ __forceinline__ bool pass_keeps(double r2, double h, double kappa) {
  return !(__ddiv_rn(__dsqrt_rn(r2), h) > kappa);
}

template <int D>
__global__ void k_ell_count(sphb_grid g, int64_t n, const double* __restrict__ ws,
                            const int32_t* __restrict__ cs, const int32_t* __restrict__ ce,
                            double h, double kappa, int32_t* __restrict__ cnt,
                            int32_t* __restrict__ max_cnt) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t c = 0;
  if (s < n) {
    for_each_neighbor<D>(g, n, ws, cs, ce, (int32_t)s, [&](int32_t, const double*, double r2) {
      if (pass_keeps(r2, h, kappa)) ++c;
    });
    cnt[s] = c;
  }
  int32_t m = warp_max(c);
  if ((threadIdx.x & 31) == 0) atomicMax(max_cnt, m);
}

extern "C" int sphb_ell_count(const sphb_grid* g, int64_t n, const double* ws, const int32_t* cs,
                              const int32_t* ce, double h, double kappa, int32_t* cnt,
                              int32_t* max_cnt, void* stream) {
  if (!grid_ok(g) || n < 0) return SPHB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SPHB_CUDA_CHECK(cudaMemsetAsync(max_cnt, 0, sizeof(int32_t), st));
  if (n == 0) return SPHB_OK;
  const int T = 128;
  switch (g->dim) {
    case 1: k_ell_count<1><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, cs, ce, h, kappa, cnt, max_cnt); break;
    case 2: k_ell_count<2><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, cs, ce, h, kappa, cnt, max_cnt); break;
    default: k_ell_count<3><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, cs, ce, h, kappa, cnt, max_cnt); break;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

template <int D>
__global__ void k_ell_fill(sphb_grid g, int64_t n, const double* __restrict__ ws,
                           const int32_t* __restrict__ cs, const int32_t* __restrict__ ce,
                           double h, double kappa, int32_t width, int32_t* __restrict__ nbr) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  int32_t k = 0;
  for_each_neighbor<D>(g, n, ws, cs, ce, (int32_t)s, [&](int32_t t, const double*, double r2) {
    if (pass_keeps(r2, h, kappa)) {
      if (k < width) nbr[(int64_t)k * n + s] = t;
      ++k;
    }
  });
  // pad the row with itself: padded slots are never read (cnt bounds loops)
  for (; k < width; ++k) nbr[(int64_t)k * n + s] = (int32_t)s;
}

// Engine-order row sort: entries of each ELL row ordered by their quantised
// displacement (slow axis first, axis 0 fastest), ties by index.  On a
// lattice stored in lattice order every row then lists the same offsets in
// the same order, so at step k the lanes of a warp read consecutive records
// (coalesced gathers) instead of one cache line each.
constexpr int kSortMax = 192;

template <int D>
__global__ void k_ell_sort_rows(sphb_grid g, int64_t n, const double* __restrict__ ws,
                                int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                                double inv_f, int32_t* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int m = cnt[i];
  if (m > kSortMax) {
    atomicOr(err, 1);
    return;
  }
  uint64_t key[kSortMax];
  double wi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) wi[a] = ws[(int64_t)a * n + i];
  for (int k = 0; k < m; ++k) {
    const int32_t j = nbr[(int64_t)k * n + i];
    uint64_t q = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const double dx = min_image(ws[(int64_t)a * n + j] - wi[a], g.box[a], g.periodic);
      long long c = llrint(dx * inv_f) + 512;
      c = c < 0 ? 0 : (c > 1023 ? 1023 : c);
      q = (q << 10) | (uint64_t)c;
    }
    const uint64_t v = (q << 32) | (uint32_t)j;
    int p = k;
    while (p > 0 && key[p - 1] > v) {
      key[p] = key[p - 1];
      --p;
    }
    key[p] = v;
  }
  for (int k = 0; k < m; ++k) nbr[(int64_t)k * n + i] = (int32_t)(key[k] & 0xffffffffu);
}

extern "C" int sphb_ell_sort_rows(const sphb_grid* g, int64_t n, const double* ws, int32_t* nbr,
                                  const int32_t* cnt, double spacing, int32_t* err,
                                  void* stream) {
  if (!grid_ok(g) || n < 0 || !(spacing > 0.0) || !err) return SPHB_ERR_ARG;
  if (n == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 64;
  const double inv_f = 1.0 / spacing;
  switch (g->dim) {
    case 1: k_ell_sort_rows<1><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, nbr, cnt, inv_f, err); break;
    case 2: k_ell_sort_rows<2><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, nbr, cnt, inv_f, err); break;
    default: k_ell_sort_rows<3><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, nbr, cnt, inv_f, err); break;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}

extern "C" int sphb_ell_fill(const sphb_grid* g, int64_t n, const double* ws, const int32_t* cs,
                             const int32_t* ce, double h, double kappa, int32_t width,
                             int32_t* nbr, void* stream) {
  if (!grid_ok(g) || n < 0 || width < 0) return SPHB_ERR_ARG;
  if (n == 0 || width == 0) return SPHB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int T = 128;
  switch (g->dim) {
    case 1: k_ell_fill<1><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, cs, ce, h, kappa, width, nbr); break;
    case 2: k_ell_fill<2><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, cs, ce, h, kappa, width, nbr); break;
    default: k_ell_fill<3><<<sphb_blocks(n, T), T, 0, st>>>(*g, n, ws, cs, ce, h, kappa, width, nbr); break;
  }
  SPHB_LAUNCH_CHECK();
  return SPHB_OK;
}
