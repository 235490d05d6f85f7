/*
 * sphb.h — C ABI of the B200-native truncated-Wendland SPH hot path.
 *
 * Every entry point works on DEVICE pointers that the caller owns (allocated
 * by the host runtime — PyTorch in this repo), runs asynchronously on the
 * caller's CUDA stream (passed as `void*`, a cudaStream_t) and returns an
 * sphb_status.  No entry point allocates device memory: scratch space comes
 * from a caller-provided workspace whose size a *_workspace_bytes() query
 * returns.  Numerical failures (non-positive density, non-finite flux,
 * inverted deformation gradient) are reported through a device-resident
 * int32 error word that the host reads when it synchronises, mirroring the
 * exceptions raised by the reference's Python wrappers.
 *
 * Reference ("the reference" = pkg/src/sph_trunc of arXiv 2405.05155's
 * package).  The reference has no FFI: its inner operator boundary is the
 * flat signature of each @njit loop.  Each function below names the loop (or
 * the numpy glue) it replaces, file:line.
 *
 * Layout conventions
 *   - "orig"   arrays are in the caller's particle order, row-major AoS
 *              exactly like the reference numpy arrays ((n, d) doubles).
 *   - "sorted" arrays are in cell-sorted order (stable radix sort by cell
 *              key, so ascending original index inside a cell), SoA:
 *              component a of particle s lives at [a * n + s].
 *   - CSR neighbour lists are the reference's NeighborList
 *              (neighbors.py:18-35): starts (n+1) int64, idx (m) int32,
 *              r (m) f64, e (m, d) f64, rows in orig order, each row in the
 *              reference's enumeration order (3^d stencil, axis 0 fastest,
 *              then ascending index inside a cell).
 *   - ELL neighbour tables are the engine's pass lists: nbr[k * n + s]
 *              (sorted indices, column-major so a warp's loads coalesce),
 *              cnt[s] entries per row, same order as the CSR row.
 */
#ifndef SPHB_H
#define SPHB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPHB_OK = 0,
  SPHB_ERR_ARG = -1,      /* invalid argument (maps to ValueError)            */
  SPHB_ERR_CUDA = -2,     /* CUDA runtime error; see sphb_last_cuda_error()  */
  SPHB_ERR_WORKSPACE = -3,/* workspace smaller than *_workspace_bytes()      */
  SPHB_ERR_OVERFLOW = -4  /* table too small (ELL width, cell count)         */
} sphb_status;

/* device error-word bits (solver checks; see eulerian.py:548-550,631-633,
 * tlsph.py:196-199) */
#define SPHB_EFLAG_NONFINITE_FLUX   1
#define SPHB_EFLAG_NONPOS_DENSITY   2
#define SPHB_EFLAG_DET_NONPOS       4
#define SPHB_EFLAG_NONFINITE_STATE  8
#define SPHB_EFLAG_BAD_INDEX        16   /* debug builds: pass-list index out of range */

/* Kernel families: the reference's integer codes (kernels.py:26-27). */
#define SPHB_CODE_WENDLAND 0
#define SPHB_CODE_LAGUERRE_GAUSS 1

/* Uniform cell grid of the cell-linked list.  Filled on the host exactly as
 * build_neighbors() does (neighbors.py:183-203) so that cell membership and
 * therefore the candidate set and its order are identical. */
typedef struct sphb_grid {
  int32_t dim;         /* 1..3                                              */
  int32_t periodic;    /* 1: minimum image in box (neighbors.py:189)        */
  int64_t ncell[3];    /* cells per axis, >= 1                              */
  int64_t strides[3];  /* flat-key strides, axis 0 fastest (:394-396)       */
  int64_t ntot;        /* prod(ncell)                                       */
  double inv_cell[3];  /* ncell/box (periodic) or 1/cutoff (open)           */
  double box[3];       /* periodic lengths (1.0 on open axes, :383)         */
  double lo[3];        /* open-domain shift pos.min(axis=0) (:384)          */
  double cutoff;
  double cut2;         /* cutoff * cutoff (neighbors.py:266 of _search)     */
  /* Storage order: particles are sorted by a cell key whose slowest axis is
   * `slow_axis` (strides `sstrides`); with slow_axis = dim-1 it is the
   * reference flat key.  Only the storage order changes (slab layers along
   * slow_axis become contiguous); cell tables stay indexed by the reference
   * key and rows are enumerated in the reference order either way. */
  int64_t sstrides[3];
  int32_t slow_axis;
  int32_t reserved;
} sphb_grid;

/* Kernel parameters (KernelSpec, kernels.py:62-80). */
typedef struct sphb_kernel {
  int32_t code;        /* SPHB_CODE_*                                       */
  int32_t dim;
  double h;
  double alpha;
  double kappa;
} sphb_kernel;

/* Signed-distance shape (geometry.py:16-134): kind 1 circle/ball
 * (center, radius), 2 axis-aligned rectangle/box (lo, hi), 3 half disk
 * (center, radius, normal = outward unit normal of the flat face). */
typedef struct sphb_shape {
  int32_t kind;
  int32_t dim;
  double center[3];
  double radius;
  double lo[3];
  double hi[3];
  double normal[3];
} sphb_shape;

const char* sphb_version(void);
const char* sphb_last_cuda_error(void);
int sphb_device_count(void);
/* FP64 DFMA throughput probe (2*8*iters flops per thread) for the roofline. */
int sphb_fp64_probe(double* out, int32_t blocks, int32_t threads, int32_t iters, void* stream);

/* ---------------------------------------------------------------- binning */

/* Workspace for sphb_bin (cub radix-sort temp + key/value scratch). */
size_t sphb_bin_workspace_bytes(int64_t n, const sphb_grid* g);

/* Wrap/shift coordinates, cell keys, stable radix sort by key, cell tables.
 * Replaces build_neighbors' coordinate set-up + _cell_index
 * (neighbors.py:183-208, :38-53) and the head/next counting lists of _search
 * (:63-74).  Outputs: wrapped coordinates in sorted SoA order, perm[s] =
 * original index of sorted particle s, cell_start/cell_end[ntot]. */
int sphb_bin(const sphb_grid* g, const double* pos_orig, int64_t n,
             double* wrapped_sorted, int32_t* perm, int32_t* cell_start,
             int32_t* cell_end, void* workspace, size_t workspace_bytes,
             void* stream);

/* --------------------------------------------------- CSR (drop-in list) */

/* Per-row neighbour counts (pass 1 of _search, neighbors.py:87-119), written
 * in ORIGINAL order into starts[1..n], then scanned so starts becomes the CSR
 * offsets (neighbors.py:121-123).  starts has n+1 entries; starts[n] = m. */
size_t sphb_csr_workspace_bytes(int64_t n);
int sphb_csr_starts(const sphb_grid* g, int64_t n, const double* wrapped_sorted,
                    const int32_t* perm, const int32_t* cell_start,
                    const int32_t* cell_end, int64_t* starts, void* workspace,
                    size_t workspace_bytes, void* stream);

/* Fill idx/r/e (pass 2 of _search, neighbors.py:129-167). */
int sphb_csr_fill(const sphb_grid* g, int64_t n, const double* wrapped_sorted,
                  const int32_t* perm, const int32_t* cell_start,
                  const int32_t* cell_end, const int64_t* starts, int32_t* idx,
                  double* r, double* e, void* stream);

/* --------------------------------------------------- ELL (engine lists) */

/* Engine pass list: same enumeration, but pairs the passes would skip
 * (q = r/h > kappa, correction.py:99-101, approx.py:48-49,
 * relaxation.py:74-76) are dropped at build time.  cnt[s] per sorted row.
 * *max_cnt_dev receives max(cnt) (device int32). */
int sphb_ell_count(const sphb_grid* g, int64_t n, const double* wrapped_sorted,
                   const int32_t* cell_start, const int32_t* cell_end,
                   double h, double kappa, int32_t* cnt, int32_t* max_cnt_dev,
                   void* stream);
int sphb_ell_fill(const sphb_grid* g, int64_t n, const double* wrapped_sorted,
                  const int32_t* cell_start, const int32_t* cell_end,
                  double h, double kappa, int32_t width, int32_t* nbr,
                  void* stream);

/* Engine-order row sort (no reference counterpart; a layout choice): each
 * row's entries reordered by displacement quantised at `spacing` (slow axis
 * first), ties by index, so lattice rows list their offsets in one order and
 * warp gathers coalesce.  Rows longer than 192 set *err = 1. */
int sphb_ell_sort_rows(const sphb_grid* g, int64_t n, const double* ws, int32_t* nbr,
                       const int32_t* cnt, double spacing, int32_t* err, void* stream);

/* Moment matrices M_i (correction.py:35-52) straight from the ELL list,
 * sorted order, exact geometry; bit-identical rows to sphb_moment_matrices
 * on the CSR without materialising r and e. */
int sphb_ell_moments(const sphb_grid* g, int64_t n, const double* wrapped_sorted,
                     const int32_t* nbr, const int32_t* cnt, const double* vols_sorted,
                     const sphb_kernel* k, double* m_sorted, void* stream);

/* ---------------------------------------------- CSR operator passes
 * Bit-faithful restatements of the reference @njit loops (compiled without
 * FMA contraction, same summation order) over a device CSR. */

/* _unity_sums (approx.py:41-52): out[i] = a P(0) V_i + sum_{q<=kappa} a P(q) V_j */
int sphb_unity_sums(int64_t n, const int64_t* starts, const int32_t* idx,
                    const double* r, const double* vols, const sphb_kernel* k,
                    double* out, void* stream);

/* _pressure_accel (relaxation.py:66-80) */
int sphb_pressure_accel(int64_t n, int32_t dim, const int64_t* starts,
                        const int32_t* idx, const double* r, const double* e,
                        const double* vols, const sphb_kernel* k, double p0,
                        double rho0, double* acc, void* stream);

/* _moment_matrices (correction.py:35-52): m (n, d, d) */
int sphb_moment_matrices(int64_t n, int32_t dim, const int64_t* starts,
                         const int32_t* idx, const double* r, const double* e,
                         const double* vols, const sphb_kernel* k, double* m,
                         void* stream);

/* correction_matrices' numpy/LAPACK block (correction.py:64-81): SVD of M,
 * clamp s < EPS_SV s_max, pseudo-inverse, theta = clip(det(-M)/EPS_DET,0,1),
 * B = theta(-M+) + (1-theta) I.  Outputs B (n,d,d), det(-M) (n) and the
 * per-particle regularized flag (int8).  One-sided Jacobi SVD on device. */
int sphb_correction_from_moments(int64_t n, int32_t dim, const double* m,
                                 double* b, double* det_neg_m, int8_t* reg,
                                 void* stream);

/* _pair_gradients (correction.py:89-112): gw (m, d); b may be NULL */
int sphb_pair_gradients(int64_t n, int32_t dim, const int64_t* starts,
                        const int32_t* idx, const double* r, const double* e,
                        const sphb_kernel* k, const double* b, double* gw,
                        void* stream);

/* _weak_gradient (approx.py:61-86): out_i = sum_j 2 (0.5 (f_i + f_j) V_j) gw_ij
 * over CSR rows with the pair gradients of sphb_pair_gradients. */
int sphb_weak_gradient(int64_t n, int32_t dim, const int64_t* starts, const int32_t* idx,
                       const double* f, const double* vols, const double* gw, double* out,
                       void* stream);

/* _rhs_wc (eulerian.py:224-266) over precomputed gwv/viscv (CSR, orig). */
int sphb_rhs_wc_csr(int64_t n_int, int32_t dim, const int64_t* starts,
                    const int32_t* idx, const double* e, const double* gwv,
                    const double* viscv, const double* rho, const double* v,
                    const double* p, double c_art, double mu,
                    const int8_t* wall_tag, double* drho, double* dmom,
                    double* wall_force_partial, void* stream);

/* _accelerations (tlsph.py:88-102) and _deformation_rates (:105-123). */
int sphb_tl_accelerations_csr(int64_t n, int32_t dim, const int64_t* starts,
                              const int32_t* idx, const double* g0,
                              const double* q, double rho0, double* acc,
                              void* stream);
int sphb_tl_deformation_rates_csr(int64_t n, int32_t dim, const int64_t* starts,
                                  const int32_t* idx, const double* g0,
                                  const double* v, const double* b0,
                                  double* dF, void* stream);

/* ---------------------------------------------------------- WC engine
 * EulerianSolver (eulerian.py:465-662), weakly-compressible branch, fused:
 * one kernel per midpoint stage evaluates EOS + limited linearised Riemann
 * flux (_linearized_scalar :145-157, _rhs_wc :224-266) with the pair
 * geometry (r, e, corrected gradient, viscous weight; :506-513) recomputed
 * from sorted coordinates, then applies the stage update (:619-629) and,
 * in stage 2, folds max(c + |v|) for the next dt (compute_dt :553-560).
 *
 * Packed per-particle records, cell-sorted order (4 doubles = 32 B each):
 *   X  [n][4] = {x0, x1, x2, vol}      (2D {x0, x1, vol, 0}; 1D {x0, vol,..})
 *   B  two planes, 6n doubles: [n][4] {b00,b01,b02,b11} then [n][2]
 *               {b12,b22} — the symmetrised correction matrix, laid out so
 *               consecutive particles' records are contiguous
 *               (2D: plane 0 {b00,b01,b11,0}; 1D: {b00,0,0,0})
 *   S  [n][4] = {v0, v1, v2, rho}      primitive state (2D {v0, v1, rho, 0})
 *   M  [n][4] = {m0, m1, m2, 0}        momentum per unit volume
 * Device scalar block (double[4]): [0] dt, [1] t, [2] max-speed accumulator
 * (atomicMax on the bit pattern), [3] spare.  err: int32 SPHB_EFLAG_* word.
 */
typedef struct sphb_wc_params {
  int32_t dim;
  int32_t periodic;
  int32_t uniform_vol;   /* 1: vol_const used instead of X[.][dim]          */
  int32_t width;         /* ELL width                                       */
  int64_t n;             /* particles in the arrays (owned + halo)          */
  int64_t row0, nrows;   /* rows updated: [row0, row0 + nrows) (slab ranks)  */
  double box[3];
  double h, alpha, kappa; /* Wendland family only (code 0)                  */
  double c_art, rho0, mu, cfl;
  double vol_const;
  int32_t reserved0;
  int32_t reserved;
  const int8_t* interior; /* NULL, or 1 for rows to update (ghosts: 0), sorted */
  double gamma;          /* ideal-gas ratio of specific heats (HLLC path)   */
  /* wall-force diagnostic (eulerian.py:225-264, 515-519, 605-606): NULL, or
   * per sorted row 1 for particles whose pair forces count; stages 0 and 2
   * zero wall_force[dim] and accumulate -sum of the momentum flux over pairs
   * (i interior, j tagged).  sphb_wc_stage and sphb_hllc_stage only. */
  const int8_t* wall_tag;
  double* wall_force;
  /* Fused halo push (slab ranks, sphb_wc_stage stages 1-2): rows
   * [push_lo0, push_lo1) of the output records are also stored into the
   * previous rank's buffer at record push_prev_at + (i - push_lo0), rows
   * [push_hi0, push_hi1) into the next rank's at push_next_at + (i - push_hi0)
   * (peer memory over NVLink), followed by a system-scope fence; the caller
   * orders the peer's next stage after this one (a one-word collective).
   * NULL pointers: no push. */
  double* push_prev;
  double* push_next;
  int64_t push_lo0, push_lo1, push_prev_at;
  int64_t push_hi0, push_hi1, push_next_at;
} sphb_wc_params;

/* Lattice fast path of the WC stage (csrc/wc_lattice.cu): for particle sets
 * that are a complete lattice in engine order (axis 0 fastest; periodic, or
 * a slab rank whose owned rows never wrap).  Offsets o with 0 < |o|^2 <= r2
 * (lattice units) in canonical order (axis 2 slowest, axis 0 fastest);
 * supported (dim, r2): (2, 4), (2, 6), (3, 4), (3, 6) — the 1.6h / 2h
 * stencils at h = 1.3 dp.  Geometry per canonical slot k (uniform volume V
 * folded in): dx = x_i - x_j, inv_r = 1/|dx|, g2 = -2 x 0.5 dW V / r,
 * mv = mu viscv = 2 mu dW V / r (eulerian.py:506-513). */
#define SPHB_LATTICE_MAXW 80
typedef struct sphb_lattice {
  int32_t width;         /* slots per row = sphb_lattice_width(dim, r2)     */
  int32_t r2;
  int32_t n[3];          /* lattice extents, 1 for unused axes              */
  int32_t uniform_b;     /* 1: every record's B equals b0 (checked by
                          * sphb_wc_uniform_b_check); the stage then serves
                          * (B_i + B_j) gg_k from a per-slot table          */
  double dx[SPHB_LATTICE_MAXW][3];
  double inv_r[SPHB_LATTICE_MAXW];
  double g2[SPHB_LATTICE_MAXW];
  double mv[SPHB_LATTICE_MAXW];
  double b0[6];          /* {b00, b01, b02, b11, b12, b22} (2D: {b00, b01, b11}) */
} sphb_lattice;
/* Slots of the (dim, r2) stencil (0: unsupported) and their offsets
 * (off[3 k + axis]). */
int sphb_lattice_width(int32_t dim, int32_t r2);
int sphb_lattice_offsets(int32_t dim, int32_t r2, int32_t* off);
/* Proof of the specialisation for rows [row0, row0 + nrows): counts rows
 * (into *bad, device, accumulated) whose pass-list row (nbr, cnt: the ELL
 * list in engine order) is not exactly {i + o_k} or whose exact minimum-
 * image displacement (neighbors.py:152-157, from X records) differs from
 * L->dx by more than tol on any axis. */
int sphb_wc_lattice_check(const sphb_wc_params* p, const sphb_lattice* L, const double* X,
                          const int32_t* nbr, const int32_t* cnt, double tol,
                          unsigned long long* bad, void* stream);
/* 1 when L->uniform_b and b0 = beta I to 1e-12 of max|b0| (cubic / square
 * lattices): sphb_wc_stage_lattice then runs its isotropic uniform-B form
 * ((B_i + B_j) gg_k = lam_k ee_k, the star-state algebra folded onto ee_k);
 * 0 otherwise; SPHB_ERR_ARG on a bad table. */
int sphb_wc_lattice_isotropic_b(int32_t dim, const sphb_lattice* L);
/* Counts into *bad (device, accumulated) the records i in [0, p->n) whose
 * symmetrised B (the two-plane layout of sphb_wc_stage) differs from b0
 * (device, 6 doubles in the order of sphb_lattice.b0) by more than
 * tol * max|b0| in any entry: zero means the uniform-B form is exact to
 * that tolerance. */
int sphb_wc_uniform_b_check(const sphb_wc_params* p, const double* B, const double* b0,
                            double tol, unsigned long long* bad, void* stream);
/* The stage of sphb_wc_stage on a checked lattice (uniform volumes; no
 * ghosts, no wall tags): same stage / record / scalar / error contract. */
int sphb_wc_stage_lattice(const sphb_wc_params* p, const sphb_lattice* L, int32_t stage,
                          const double* B, const double* S_in, const double* S_n,
                          const double* M_n, double* S_out, double* M_out, double* scalars,
                          int32_t* err, void* stream);

/* The optional FP32 mode of sphb_wc_stage_f32 on a checked lattice: FP32
 * records (B32 planes, S32 {v, rho - rho0}) and table geometry, FP32 pair
 * math, FP64 accumulation and FP64 stage update (S_out/M_out in stage 2;
 * S32_out written by stages 1 and 2; stage 0 writes the rhs record). */
int sphb_wc_stage_lattice_f32(const sphb_wc_params* p, const sphb_lattice* L, int32_t stage,
                              const float* B32, const float* S32_in, const double* S_n,
                              const double* M_n, float* S32_out, double* S_out, double* M_out,
                              double* scalars, int32_t* err, void* stream);

/* `group` (1, 2, 4, 8) consecutive threads share one particle's row.
 * stage 0: rhs only — S_out = {dmom, drho} records (EulerianSolver.rhs).
 * stage 1: S_in = S_n, writes S_out = U^1 primitive record (M_out unused).
 * stage 2: S_in = U^1 records, own U^n from S_n/M_n, writes U^{n+1} into
 *          S_out/M_out (may alias S_n/M_n) and folds max(c+|v|). */
int sphb_wc_stage(const sphb_wc_params* p, int32_t stage, int32_t group, const double* X,
                  const double* B, const int32_t* nbr, const int32_t* cnt,
                  const double* S_in, const double* S_n, const double* M_n,
                  double* S_out, double* M_out, double* scalars, int32_t* err,
                  void* stream);
/* Static per-pair geometry of the WC flux (eulerian.py:506-513): for every
 * ELL slot, e_ij, gwv_ij = dW 0.5 (B_i + B_j) e_ij V_j and viscv_ij =
 * 2 dW / r V_j as planes geo[(c * width + k) * n + s], c = 0..2D (B: full
 * sorted (n, d, d) matrices; vol: sorted).  Reference arithmetic, no FMA. */
int sphb_wc_geometry(const sphb_grid* g, int64_t n, const double* wrapped_sorted,
                     const int32_t* nbr, const int32_t* cnt, int32_t width,
                     const double* B_full, const double* vol_sorted, const sphb_kernel* k,
                     double* geo, void* stream);
/* Stage kernel streaming that geometry and gathering only S_j (same
 * contract as sphb_wc_stage; p->width = ELL width). */
int sphb_wc_stage_geo(const sphb_wc_params* p, int32_t stage, const int32_t* nbr,
                      const int32_t* cnt, const double* geo, const double* S_in,
                      const double* S_n, const double* M_n, double* S_out, double* M_out,
                      double* scalars, int32_t* err, void* stream);

/* Optional FP32 mode (north star): FP32 pair geometry + flux from FP32
 * neighbour records X32 float4 {x, 0}, B32 planes float4 + float2, S32
 * float4 {v, rho - rho0}; FP64 accumulation and stage update on the FP64
 * state.  Stage 1 writes S32_out only; stage 2 writes S32_out, S_out, M_out.
 * Uniform volumes. */
int sphb_wc_stage_f32(const sphb_wc_params* p, int32_t stage, const float* X32,
                      const float* B32, const int32_t* nbr, const int32_t* cnt,
                      const float* S32_in, const double* S_n, const double* M_n,
                      float* S32_out, double* S_out, double* M_out, double* scalars,
                      int32_t* err, void* stream);
int sphb_wc_state_to_f32(int64_t n, int32_t dim, double rho0, const double* S, float* S32,
                         void* stream);

/* Ghost refresh (apply_boundaries, eulerian.py:371-447), WC kinds 0,1,2,3,5
 * (copy, mirror, wall, fixed, blend-mirror): ghost record S[ghost_sorted[g]]
 * from its source S[src_sorted[g]].  normal/wall_v (ng, d), fixed (ng, d+2)
 * conserved {rho, mom, E}, blend (ng) (may be NULL without kind 5). */
/* Append (t = scalars[1], scale * wall_force[0..dim)) as row count[0] of
 * log [cap][1 + dim] and increment count[0] (rows past cap are counted but
 * not written): EulerianSolver.step's wall_force_series entry
 * (eulerian.py:605-606) recorded on the device. */
int sphb_wall_record(int32_t dim, const double* wall_force, const double* scalars,
                     double scale, double* log, int64_t* count, int64_t cap, void* stream);

/* ---- shape-bounded relaxation (relaxation.py:92-198) */
/* sd[i] = signed distance of x[i] (NULL: skipped); grad[i] = unit outward
 * gradient by central differences, eps 1e-7 (geometry.py:129-147). */
int sphb_shape_sdf(const sphb_shape* s, int64_t n, const double* x, double* sd, double* grad,
                   void* stream);
/* Wall confinement (relaxation.py:162-168): for depth = -sd(pos) < cutoff,
 * acc -= coef * interp(depth; s_grid, w2, right = 0) * grad; then
 * sums[2] = sum_i |acc_i| (zeroed first).  pos/acc in caller order. */
int sphb_relax_confine(const sphb_shape* s, int64_t n, const double* pos, double cutoff,
                       const double* s_grid, const double* w2, int32_t n_s, double coef,
                       double* acc, double* sums, void* stream);
/* dx = acc dt2 capped at `cap`; pos += dx; particles with sd > surf_tol are
 * projected back (<= 3 steps x -= sd grad while sd > 1e-12),
 * relaxation.py:188-198 and _project_to_surface (:120-129). */
int sphb_relax_update_shape(const sphb_shape* s, int64_t n, const double* acc, double dt2,
                            double cap, double surf_tol, double* pos, void* stream);
/* out[0:dim] = per-axis min, out[dim:2 dim] = per-axis max of pos (n, dim):
 * the open-domain shift and extent of build_neighbors (neighbors.py:194-197). */
int sphb_bounds(int64_t n, int32_t dim, const double* pos, double* out, void* stream);

/* Copy 32-byte records at the given rows: d_k[rows[g]] = s_k[rows[g]] for
 * each non-null pair (pair 0 required).  Used after the last stage to carry
 * the ghost rows of apply_boundaries(t + dt/2) into the step's output, the
 * state the reference's in-place arrays hold after EulerianSolver.step
 * (eulerian.py:610-643). */
int sphb_copy_records(int64_t nrows, const int32_t* rows, const double* s0, double* d0,
                      const double* s1, double* d1, const double* s2, double* d2,
                      void* stream);

int sphb_wc_ghosts(int32_t dim, int64_t ng, const int32_t* ghost_sorted,
                   const int32_t* src_sorted, const int8_t* kind, const double* normal,
                   const double* wall_v, const double* fixed, const double* blend,
                   double* S, double* M, int32_t* err, void* stream);

/* Compressible path: limited HLLC flux + energy
 * equation (eulerian.py:90-142, 269-338) over streamed geometry, ideal-gas
 * EOS (:67-85).  Extra record Q [n][4] = {E, p, c, 0}.  Stage 0 writes
 * {dmom, drho} to S_out and {dE, ...} to Q_out. */
int sphb_hllc_stage(const sphb_wc_params* p, int32_t stage, const int32_t* nbr,
                    const int32_t* cnt, const double* geo, const double* S_in,
                    const double* Q_in, const double* S_n, const double* M_n,
                    const double* Q_n, double* S_out, double* M_out, double* Q_out,
                    double* scalars, int32_t* err, void* stream);
int sphb_hllc_pack_state(int64_t n, int32_t dim, const int32_t* perm, const int8_t* interior,
                         double gamma, const double* rho, const double* mom,
                         const double* etot, double* S, double* M, double* Q,
                         double* scalars, int32_t* err, void* stream);
int sphb_hllc_unpack_state(int64_t n, int32_t dim, const int32_t* perm, const double* S,
                           const double* M, const double* Q, double* rho, double* mom,
                           double* etot, void* stream);
/* Ghost refresh incl. the DMR top (kind 4; state post/pre by ghost x vs the
 * shock foot x0 + (1 + 20 t)/tan60 at t = step start + t_shift dt). */
int sphb_hllc_ghosts(int32_t dim, int64_t ng, const int32_t* ghost_sorted,
                     const int32_t* src_sorted, const int8_t* kind, const double* normal,
                     const double* wall_v, const double* fixed, const double* blend,
                     const double* dmr_x, double dmr_x0, double dmr_tan,
                     const double* dmr_post, const double* dmr_pre, double gamma,
                     double t_shift, const double* scalars, double* S, double* M, double* Q,
                     int32_t* err, void* stream);

/* max(c + |v|) of a state into scalars[2] (initial dt / compute_dt()). */
int sphb_wc_speed_max(const sphb_wc_params* p, const double* S, double* scalars,
                      void* stream);

/* Caller-order (rho (n), mom (n, d)) <-> sorted S/M records, with
 * v = mom / rho (FluidState.velocity, eulerian.py:461-462). */
int sphb_wc_pack_state(int64_t n, int32_t dim, const int32_t* perm, const double* rho,
                       const double* mom, double* S, double* M, void* stream);
int sphb_wc_unpack_state(int64_t n, int32_t dim, const int32_t* perm, const double* S,
                         const double* M, double* rho, double* mom, void* stream);

/* dt for the next step: dt = dt_override if > 0, else
 * cfl_h / (c_add + scalars[2]); then scalars[1] += dt, scalars[2] = 0.
 * WC: c_add = 0 (the speed already includes c; eulerian.py:556-560);
 * TL: c_add = c_s (tlsph.py:178-180). */
/* Copy `bytes` (a multiple of 4, at most 4096) from device memory into
 * pinned host memory with a kernel writing through the host mapping, not a
 * copy engine: small host reads (dt, error word) then never queue behind a
 * bulk transfer in flight.  SPHB_ERR_ARG if host_dst is not mapped pinned
 * memory. */
int sphb_mirror_to_host(const void* src, void* host_dst, int64_t bytes, void* stream);
int sphb_set_dt(double cfl_h, double c_add, double dt_override, double* scalars,
                int32_t* err, void* stream);

/* ---------------------------------------------------------- TL engine
 * SolidSystem.step (tlsph.py:182-206), fused into two passes over the ELL
 * list of the reference configuration X0:
 *   pass A: v_half = v + dt/2 acc (fixed -> 0) for i and every neighbour j,
 *           x += dt v_half, dF = [sum (v_j - v_i) (x) g0_ij] B0_i
 *           (_deformation_rates :105-123), F += dt dF, det F > 0 check, and
 *           the epilogue Q = (F S) B0^T with S the SVK PK2 (:54-65,160-167).
 *   pass B: acc = sum (Q_i + Q_j) g0_ij / rho0 (_accelerations :88-102),
 *           acc[fixed] = 0, v = v_half + dt/2 acc, v[fixed] = 0, and
 *           max |v| for the next stable_dt (:178-180).
 * g0_ij = (alpha/h) dP(q) e_ij V0 is recomputed from X0 (:145-146).
 * Records (sorted order): X0 [n][4] (x0,x1,x2,fixed-flag as double),
 * V/A/XC [n][4] vectors, B0/F/Q [n][12] (row-major 3x3 padded; 2D uses the
 * leading 2x2 block with stride 2... see tl_engine.cu). */
typedef struct sphb_tl_params {
  int32_t dim;
  int32_t width;
  int64_t n;
  int64_t row0, nrows;     /* rows updated (slab ranks); stress: all n */
  double h, alpha, kappa;  /* Wendland family */
  double vol0, rho0;
  double lam, g;           /* Lame parameters (tlsph.py:27-35) */
  /* Fused halo push (slab ranks): pass A also stores the Q records of rows
   * [push_lo0, push_lo1) into the previous rank's Q buffer at particle
   * push_prev_at + (i - push_lo0) and rows [push_hi0, push_hi1) into the
   * next rank's at push_next_at + (i - push_hi0); pass B does the same with
   * A (and V when it updates v).  Peer memory, system-scope fence; NULL: off. */
  double* push_q_prev;
  double* push_q_next;
  double* push_a_prev;
  double* push_a_next;
  double* push_v_prev;
  double* push_v_next;
  int64_t push_lo0, push_lo1, push_prev_at;
  int64_t push_hi0, push_hi1, push_next_at;
  /* 3D Q records are three column planes Q[c * q_stride + i] (one 32-byte
   * {q_0c, q_1c, q_2c, X0_c} per plane and particle), so a warp's gather of
   * one row touches consecutive records; q_stride >= n, 0 means n.  Slab
   * ranks use one common stride so pushes address peer buffers with it. */
  int64_t q_stride;
  /* Optional FP32 mode (lattice passes only): FP32 companions of the
   * gathered records — vh32 (float4 per particle, written by the kick) and
   * q32 (three float4 column planes of stride q_stride, {q_0c, q_1c, q_2c,
   * 0}, written instead of Q by pass A / sphb_tl_stress and read by pass B);
   * arithmetic and state stay FP64.  NULL: FP64 records. */
  float* vh32;
  float* q32;
  /* Material law of the PK2 stress: 0 = St. Venant-Kirchhoff (tlsph.py:54-65),
   * 1 = compressible Neo-Hookean S = G (I - C^-1) + lam ln(J) C^-1 (BASELINE
   * configs 3-4; not in the reference). */
  int32_t law;
  /* 1: dense 3D Q records (the lattice table mode, one GPU; set with
   * sphb_tl_lattice.table): column c is a double2 plane {q_0c, q_1c} at
   * ((double2*)Q)[c * n + i] and a double plane q_2c at Q[6 n + c * n + i]
   * (72 bytes, no X0 padding), so pass B gathers 24 instead of 32 bytes per
   * column.  Pass A, sphb_tl_stress and the lattice pass B honour it. */
  int32_t q_dense;
} sphb_tl_params;

/* Pass A first writes Vh = v + dt/2 a (0 for clamped rows) for all n rows
 * (the KDK first kick), then per owned row gathers Vh_j for dF.  g0:
 * optional per-slot reference gradients (sphb_tl_geometry); NULL ->
 * recompute g0_ij from X0 per pair.  Pass B keeps the clamp flag in A.w
 * (A record {a0, a1, a2, fixed}). */
int sphb_tl_pass_a(const sphb_tl_params* p, const double* X0, const double* B0,
                   const int32_t* nbr, const int32_t* cnt, const double* g0,
                   const double* V, const double* A, double* Vh, double* XC, double* F,
                   double* Q, const double* scalars, int32_t* err, void* stream);
int sphb_tl_pass_b(const sphb_tl_params* p, const double* X0, const int32_t* nbr,
                   const int32_t* cnt, const double* g0, const double* Q, const double* Vh,
                   double* A, double* V, double* scalars, int32_t update_v, int32_t* err,
                   void* stream);
/* Static reference gradients g0_ij = dW e_ij V0 (tlsph.py:145-146) per ELL
 * slot, planes g0[(c * width + k) * n + s]; reference arithmetic. */
int sphb_tl_geometry(const sphb_grid* g, int64_t n, const double* wrapped_sorted,
                     const int32_t* nbr, const int32_t* cnt, int32_t width,
                     const sphb_kernel* k, double vol0, double* g0, void* stream);
/* Q = (F S(F)) B0^T for every particle (first accelerations() call).  In
 * 3D each Q row carries the reference coordinate X0_r in its padding (as
 * pass A writes it), which pass B reads instead of gathering X0_j. */
int sphb_tl_stress(const sphb_tl_params* p, const double* F, const double* B0,
                   const double* X0, double* Q, void* stream);
/* The first kick alone, Vh = v + dt/2 a (0 when clamped) for all n rows. */
int sphb_tl_kick(const sphb_tl_params* p, const double* V, const double* A, double* Vh,
                 const double* scalars, void* stream);

/* Lattice fast path of the TL passes (csrc/tl_lattice.cu) for a reference
 * configuration that is a complete box lattice in engine order (axis 0
 * fastest) with separable coordinates: rows of the interior sub-box
 * [R, n_a - R) (R = isqrt(r2)) all hold the canonical offsets 0 < |o|^2 <=
 * r2 (order: axis 2 slowest), so j = i + o_k is computed, the exact
 * displacement's axis-q component is the row's difference to its neighbour
 * along axis q alone (computed once per row), and g0 = f(r2) dx with f =
 * c5v t^3 (tlsph.py:145-146) is a first-order expansion about r2k[k].
 * Shell rows run the general passes with a row list.  Supported (dim, r2):
 * (2, 3), (2, 5), (3, 3), (3, 5) — 1.6h / 2h at h = 1.15 dp.
 * table = 1: per-slot table geometry instead — dx[k] (antisymmetric,
 * dx[W-1-k] = -dx[k]) and g[k] = g0 of dx[k] (tlsph.py:145-146), so the
 * interior passes read no X0 records, and sum_k g[k] = 0 exactly removes
 * the Q_i sum_j g0_ij term (and pass B's Q_i read); the check then bounds
 * every interior pair's exact displacement to within tol (absolute) of
 * dx[k] instead of the separability / r2 tests. */
#define SPHB_TL_LATTICE_MAXW 56
typedef struct sphb_tl_lattice {
  int32_t width;         /* slots per interior row                          */
  int32_t r2;
  int32_t n[3];          /* lattice extents, 1 for unused axes              */
  int32_t table;         /* 1: table geometry (dx, g); 0: exact separable   */
  int64_t n_interior;    /* prod(n_a - 2R) over the dim axes                */
  /* the remaining (shell) rows, run in the same launches (blocks before the
   * interior ones) with the general per-pair geometry and the pass list */
  const int32_t* shell;
  int64_t n_shell;
  /* optional compact pass list of the shell rows: shell_nbr[k * n_shell + s]
   * = nbr[k * n + shell[s]], shell_cnt[s] = cnt[shell[s]] (NULL: read the
   * full list (nbr, cnt)) */
  const int32_t* shell_nbr;
  const int32_t* shell_cnt;
  double r2k[SPHB_TL_LATTICE_MAXW];
  double f[SPHB_TL_LATTICE_MAXW], df[SPHB_TL_LATTICE_MAXW];
  double dx[SPHB_TL_LATTICE_MAXW][3];   /* table geometry (table = 1)       */
  double g[SPHB_TL_LATTICE_MAXW][3];
  /* 1 (3D table mode): every interior row's B0 record equals b0 (checked by
   * sphb_tl_uniform_b0_check), so pass A takes B0 of its interior rows from
   * b0 {b00, b01, b02, b11, b12, b22} instead of reading the records */
  int32_t uniform_b0;
  int32_t reserved_b0;
  double b0[6];
} sphb_tl_lattice;
int sphb_tl_lattice_width(int32_t dim, int32_t r2);
/* Interior rows whose pass-list row is not exactly the canonical set, whose
 * exact displacements (X0 records) are not separable per axis (bitwise), or
 * whose pair r2 is off r2k by more than tol (relative): counted into *bad. */
int sphb_tl_lattice_check(const sphb_tl_params* p, const sphb_tl_lattice* L, const double* X0,
                          const int32_t* nbr, const int32_t* cnt, double tol,
                          unsigned long long* bad, void* stream);
/* Counts into *bad (device, accumulated) the interior rows whose B0 record
 * (3D two-plane layout) differs from b0 (device, 6 doubles) by more than
 * tol * max|b0| in any entry (3D only). */
int sphb_tl_uniform_b0_check(const sphb_tl_params* p, const sphb_tl_lattice* L,
                             const double* B0, const double* b0, double tol,
                             unsigned long long* bad, void* stream);
/* Passes A / B (no kick) over the interior rows (lattice) and the shell
 * rows (general, pass list) in one launch each; same records and contract
 * as sphb_tl_pass_a / sphb_tl_pass_b. */
int sphb_tl_pass_a_lattice(const sphb_tl_params* p, const sphb_tl_lattice* L, const double* X0,
                           const double* B0, const int32_t* nbr, const int32_t* cnt,
                           const double* Vh, double* XC, double* F, double* Q,
                           const double* scalars, int32_t* err, void* stream);
int sphb_tl_pass_b_lattice(const sphb_tl_params* p, const sphb_tl_lattice* L, const double* X0,
                           const int32_t* nbr, const int32_t* cnt, const double* Q,
                           const double* Vh, double* A, double* V, double* scalars,
                           int32_t update_v, int32_t* err, void* stream);

/* max |v| into scalars[2] (stable_dt). */
int sphb_tl_speed_max(const sphb_tl_params* p, const double* V, double* scalars,
                      void* stream);

/* --------------------------------------------------- relaxation engine
 * One pseudo-time step of relax() on a periodic box (relaxation.py:157-195)
 * without a materialised neighbour list: the accel kernel walks the cell
 * stencil of the binned positions in the reference order and sums the
 * constant-pressure acceleration (_pressure_accel :66-80) directly, writing
 * acc in ORIGINAL order, plus sum |a| and the isolated count (:170, :159);
 * the update kernel applies dx = a dt2 with the 0.25 dp cap and the periodic
 * wrap (:188-195).  sums: double[2] = {sum|a|, n_isolated}. */
int sphb_relax_accel(const sphb_grid* g, int64_t n, const double* wrapped_sorted,
                     const int32_t* perm, const int32_t* cell_start,
                     const int32_t* cell_end, const double* vols_orig,
                     const sphb_kernel* k, double p0, double rho0,
                     double* acc_orig, double* sums, void* stream);
int sphb_relax_update(int64_t n, int32_t dim, const double* acc_orig, double dt2,
                      double cap, const double* box3, double* pos_orig,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPHB_H */
