/*
 * sph_oracle.c — CPU ORACLE (test infrastructure only; never the product).
 *
 * Plain-C restatement of the reference's @njit loops (pkg/src/sph_trunc of
 * arXiv 2405.05155), used by tests/ to check the CUDA path and by bench.py's
 * cpu_baseline / --impl reference leg.  Each function cites the loop it
 * restates.  Compiled with -ffp-contract=off and no fast-math so every
 * expression rounds exactly like the reference's (numba does not contract to
 * FMA and evaluates left to right); rows are independent, so the OpenMP
 * row-parallel loops give the same bits as the serial reference.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load this.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ETA_LINEARIZED 15.0 /* eulerian.py:30 */

/* kernels.py:41-59 */
static inline double profile(int code, double q) {
  if (code == 0) {
    double t = 1.0 - 0.5 * q;
    return t * t * t * t * (2.0 * q + 1.0);
  }
  double q2 = q * q;
  return (1.0 - 0.5 * q2 + q2 * q2 / 6.0) * exp(-q2);
}

static inline double profile_deriv(int code, double q) {
  if (code == 0) {
    double t = 1.0 - 0.5 * q;
    return -5.0 * q * t * t * t;
  }
  double q2 = q * q;
  return q * (-3.0 + (5.0 / 3.0) * q2 - q2 * q2 / 3.0) * exp(-q2);
}

static inline int64_t pymod(int64_t a, int64_t b) {
  int64_t r = a % b;
  return r < 0 ? r + b : r;
}

/* ---------------------------------------------------------------------
 * Cell-linked-list search: _cell_index (neighbors.py:38-53) and _search
 * (neighbors.py:56-168), split as count / fill so the caller can size the
 * CSR.  `cells` (n*d) and the head/next chains are built once by
 * orc_bin() and reused by both passes.
 * ------------------------------------------------------------------- */
typedef struct {
  int64_t n, d, periodic, ntot;
  int64_t ncell[3], strides[3];
  double box[3], cut2;
  const double* wrapped;
  int64_t* cells;
  int64_t* head;
  int64_t* nxt;
} orc_bins;

void* orc_bin(const double* wrapped, int64_t n, int64_t d, const double* inv_cell,
              const int64_t* ncell, const int64_t* strides, const double* box, int64_t periodic,
              double cutoff) {
  orc_bins* b = (orc_bins*)calloc(1, sizeof(orc_bins));
  b->n = n;
  b->d = d;
  b->periodic = periodic;
  b->ntot = 1;
  for (int64_t a = 0; a < d; ++a) {
    b->ncell[a] = ncell[a];
    b->strides[a] = strides[a];
    b->box[a] = box[a];
    b->ntot *= ncell[a];
  }
  b->cut2 = cutoff * cutoff;
  b->wrapped = wrapped;
  b->cells = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n * d + 1));
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t a = 0; a < d; ++a) {
      int64_t c = (int64_t)floor(wrapped[i * d + a] * inv_cell[a]);
      if (periodic) {
        c = pymod(c, ncell[a]);
      } else {
        if (c < 0) c = 0;
        else if (c >= ncell[a]) c = ncell[a] - 1;
      }
      b->cells[i * d + a] = c;
    }
  }
  b->head = (int64_t*)malloc(sizeof(int64_t) * (size_t)b->ntot);
  b->nxt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t f = 0; f < b->ntot; ++f) b->head[f] = -1;
  for (int64_t i = n - 1; i >= 0; --i) { /* reversed: chains ascend */
    int64_t f = 0;
    for (int64_t a = 0; a < d; ++a) f += b->cells[i * d + a] * strides[a];
    b->nxt[i] = b->head[f];
    b->head[f] = i;
  }
  return b;
}

void orc_bin_free(void* p) {
  orc_bins* b = (orc_bins*)p;
  if (!b) return;
  free(b->cells);
  free(b->head);
  free(b->nxt);
  free(b);
}

/* walk row i; mode 0 counts, mode 1 fills idx/r/e from slot w */
static int64_t orc_row(const orc_bins* b, int64_t i, int mode, int64_t w, int32_t* idx,
                       double* rr, double* ee) {
  const int64_t d = b->d;
  int64_t noff = 1;
  for (int64_t a = 0; a < d; ++a) noff *= 3;
  int64_t count = 0;
  for (int64_t k = 0; k < noff; ++k) {
    int64_t rem = k, f = 0;
    int ok = 1;
    for (int64_t a = 0; a < d; ++a) {
      int64_t off = rem % 3 - 1;
      rem /= 3;
      int64_t c = b->cells[i * d + a] + off;
      if (b->periodic) {
        c = pymod(c, b->ncell[a]);
      } else if (c < 0 || c >= b->ncell[a]) {
        ok = 0;
        break;
      }
      f += c * b->strides[a];
    }
    if (!ok) continue;
    for (int64_t j = b->head[f]; j >= 0; j = b->nxt[j]) {
      if (j == i) continue;
      double r2 = 0.0, dxv[3];
      for (int64_t a = 0; a < d; ++a) {
        double dx = b->wrapped[i * d + a] - b->wrapped[j * d + a];
        if (b->periodic) {
          if (dx > 0.5 * b->box[a]) dx -= b->box[a];
          else if (dx < -0.5 * b->box[a]) dx += b->box[a];
        }
        dxv[a] = dx;
        r2 += dx * dx;
      }
      if (r2 <= b->cut2 && r2 > 0.0) {
        if (mode == 1) {
          double dist = sqrt(r2);
          idx[w] = (int32_t)j;
          rr[w] = dist;
          for (int64_t a = 0; a < d; ++a) ee[w * d + a] = dxv[a] / dist;
          ++w;
        }
        ++count;
      }
    }
  }
  return count;
}

/* pass 1 (neighbors.py:87-123): starts[0..n] */
void orc_count(const void* p, int64_t* starts) {
  const orc_bins* b = (const orc_bins*)p;
  starts[0] = 0;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < b->n; ++i) starts[i + 1] = orc_row(b, i, 0, 0, NULL, NULL, NULL);
  for (int64_t i = 0; i < b->n; ++i) starts[i + 1] += starts[i];
}

/* pass 2 (neighbors.py:129-167) */
void orc_fill(const void* p, const int64_t* starts, int32_t* idx, double* r, double* e) {
  const orc_bins* b = (const orc_bins*)p;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < b->n; ++i) orc_row(b, i, 1, starts[i], idx, r, e);
}

/* _unity_sums (approx.py:41-52) */
void orc_unity_sums(int64_t n, const int64_t* starts, const int32_t* idx, const double* r,
                    const double* vols, int64_t code, double h, double alpha, double kappa,
                    double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double acc = alpha * profile((int)code, 0.0) * vols[i];
    for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
      double q = r[k] / h;
      if (q <= kappa) acc += alpha * profile((int)code, q) * vols[idx[k]];
    }
    out[i] = acc;
  }
}

/* _pressure_accel (relaxation.py:66-80) */
void orc_pressure_accel(int64_t n, int64_t d, const int64_t* starts, const int32_t* idx,
                        const double* r, const double* e, const double* vols, int64_t code,
                        double h, double alpha, double kappa, double p0, double rho0,
                        double* acc) {
  const double scale = alpha / h;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t a = 0; a < d; ++a) acc[i * d + a] = 0.0;
    for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
      double q = r[k] / h;
      if (q > kappa) continue;
      double coeff = -2.0 * p0 * vols[idx[k]] * scale * profile_deriv((int)code, q) / rho0;
      for (int64_t a = 0; a < d; ++a) acc[i * d + a] += coeff * e[k * d + a];
    }
  }
}

/* _moment_matrices (correction.py:35-52) */
void orc_moment_matrices(int64_t n, int64_t d, const int64_t* starts, const int32_t* idx,
                         const double* r, const double* e, const double* vols, int64_t code,
                         double h, double alpha, double kappa, double* m) {
  const double scale = alpha / h;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double* mi = m + i * d * d;
    for (int64_t a = 0; a < d * d; ++a) mi[a] = 0.0;
    for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
      int32_t j = idx[k];
      double q = r[k] / h;
      if (q > kappa) continue;
      double dw = scale * profile_deriv((int)code, q);
      double w = dw * vols[j] * r[k];
      for (int64_t a = 0; a < d; ++a)
        for (int64_t c = 0; c < d; ++c) mi[a * d + c] += w * e[k * d + a] * e[k * d + c];
    }
  }
}

/* _pair_gradients (correction.py:89-112); b == NULL -> uncorrected */
void orc_pair_gradients(int64_t n, int64_t d, const int64_t* starts, const int32_t* idx,
                        const double* r, const double* e, int64_t code, double h, double alpha,
                        double kappa, const double* b, double* gw) {
  const double scale = alpha / h;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
      int64_t j = idx[k];
      for (int64_t a = 0; a < d; ++a) gw[k * d + a] = 0.0;
      double q = r[k] / h;
      if (q > kappa) continue;
      double dw = scale * profile_deriv((int)code, q);
      for (int64_t a = 0; a < d; ++a) {
        if (b) {
          double acc = 0.0;
          for (int64_t c = 0; c < d; ++c)
            acc += 0.5 * (b[(i * d + a) * d + c] + b[(j * d + a) * d + c]) * e[k * d + c];
          gw[k * d + a] = dw * acc;
        } else {
          gw[k * d + a] = dw * e[k * d + a];
        }
      }
    }
  }
}

/* _rhs_wc (eulerian.py:224-266); wall force omitted (no tags on the path) */
void orc_rhs_wc(int64_t n_int, int64_t d, const int64_t* starts, const int32_t* idx,
                const double* e, const double* gwv, const double* viscv, const double* rho,
                const double* v, const double* p, double c_art, double mu, double* drho,
                double* dmom, const int8_t* wall_tag, double* wf_rows) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n_int; ++i) {
    const double rho_i = rho[i], p_i = p[i];
    double dr = 0.0;
    if (wf_rows)
      for (int64_t a = 0; a < d; ++a) wf_rows[i * d + a] = 0.0;
    for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
      const int64_t j = idx[k];
      double u_l = 0.0, u_r = 0.0;
      for (int64_t a = 0; a < d; ++a) {
        u_l += v[i * d + a] * (-e[k * d + a]);
        u_r += v[j * d + a] * (-e[k * d + a]);
      }
      double du = u_l - u_r;
      double beta = ETA_LINEARIZED * du / c_art;
      if (beta < 0.0) beta = 0.0;
      else if (beta > 1.0) beta = 1.0;
      double rbar = 0.5 * (rho_i + rho[j]);
      double u_star = 0.5 * (u_l + u_r) + 0.5 * beta * beta * (p_i - p[j]) / (rbar * c_art);
      double p_star = 0.5 * (p_i + p[j]) + 0.5 * beta * rbar * c_art * du;
      double ubar = 0.5 * (u_l + u_r);
      double s = 0.0;
      for (int64_t a = 0; a < d; ++a) {
        double vs = u_star * (-e[k * d + a]) + 0.5 * (v[i * d + a] + v[j * d + a]) -
                    ubar * (-e[k * d + a]);
        s += vs * gwv[k * d + a];
      }
      dr += -2.0 * rbar * s;
      for (int64_t a = 0; a < d; ++a) {
        double vs = u_star * (-e[k * d + a]) + 0.5 * (v[i * d + a] + v[j * d + a]) -
                    ubar * (-e[k * d + a]);
        double fm = -2.0 * (rbar * vs * s + p_star * gwv[k * d + a]) +
                    mu * viscv[k] * (v[i * d + a] - v[j * d + a]);
        dmom[i * d + a] += fm;
        /* eulerian.py:263-264, per row; summed over rows by the caller */
        if (wall_tag && wall_tag[j]) wf_rows[i * d + a] -= fm;
      }
    }
    drho[i] = dr;
  }
}

/* _hllc_scalar (eulerian.py:90-142); out[10] as the reference tuple */
static void orc_hllc_scalar(double rho_l, double u_l, double p_l, double c_l, double e_l,
                            double rho_r, double u_r, double p_r, double c_r, double e_r,
                            double eta, double* out) {
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
  double cbar = 0.5 * (c_l + c_r);
  double du = u_l - u_r;
  double beta = eta * du / cbar;
  if (beta < 0.0) beta = 0.0;
  else if (beta > 1.0) beta = 1.0;
  double w_l = rho_l * (u_l - s_l);
  double w_r = rho_r * (s_r - u_r);
  double ws = w_l + w_r;
  double u_star = (w_l * u_l + w_r * u_r) / ws + (p_l - p_r) * beta * beta / ws;
  double p_star = 0.5 * (p_l + p_r) + 0.5 * beta * (w_r * (u_star - u_r) + w_l * (u_l - u_star));
  double den_l = s_l - s_star;
  double den_r = s_r - s_star;
  out[0] = u_star;
  out[1] = p_star;
  out[2] = rho_l * (s_l - u_l) / den_l;
  out[3] = rho_r * (s_r - u_r) / den_r;
  out[4] = ((s_l - u_l) * e_l - p_l * u_l + p_star * s_star) / den_l;
  out[5] = ((s_r - u_r) * e_r - p_r * u_r + p_star * s_star) / den_r;
  out[6] = s_l;
  out[7] = s_r;
  out[8] = s_star;
  out[9] = beta;
}

/* _rhs_hllc (eulerian.py:269-338); wall force omitted */
void orc_rhs_hllc(int64_t n_int, int64_t d, const int64_t* starts, const int32_t* idx,
                  const double* e, const double* gwv, const double* rho, const double* v,
                  const double* p, const double* c, const double* etot, double* drho,
                  double* dmom, double* detot) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n_int; ++i) {
    double dr = 0.0, de = 0.0;
    for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
      const int64_t j = idx[k];
      double u_l = 0.0, u_r = 0.0, out[10];
      for (int64_t a = 0; a < d; ++a) {
        u_l += v[i * d + a] * (-e[k * d + a]);
        u_r += v[j * d + a] * (-e[k * d + a]);
      }
      orc_hllc_scalar(rho[i], u_l, p[i], c[i], etot[i], rho[j], u_r, p[j], c[j], etot[j], 1.0,
                      out);
      const double s_l = out[6], s_r = out[7];
      double rho_s, e_s, p_use;
      int star;
      if (s_l > 0.0) {
        rho_s = rho[i]; e_s = etot[i]; p_use = p[i]; star = 0;
      } else if (s_r < 0.0) {
        rho_s = rho[j]; e_s = etot[j]; p_use = p[j]; star = 0;
      } else if (out[8] >= 0.0) {
        rho_s = out[2]; e_s = out[4]; p_use = out[1]; star = 1;
      } else {
        rho_s = out[3]; e_s = out[5]; p_use = out[1]; star = 1;
      }
      const double u_star = out[0];
      const double ubar = 0.5 * (u_l + u_r);
      double s = 0.0, vs[3];
      for (int64_t a = 0; a < d; ++a) {
        if (star) vs[a] = (u_star - ubar) * (-e[k * d + a]) + 0.5 * (v[i * d + a] + v[j * d + a]);
        else if (s_l > 0.0) vs[a] = v[i * d + a];
        else vs[a] = v[j * d + a];
        s += vs[a] * gwv[k * d + a];
      }
      dr += -2.0 * rho_s * s;
      de += -2.0 * (e_s + p_use) * s;
      for (int64_t a = 0; a < d; ++a)
        dmom[i * d + a] += -2.0 * (rho_s * vs[a] * s + p_use * gwv[k * d + a]);
    }
    drho[i] = dr;
    detot[i] = de;
  }
}

/* _weak_gradient (approx.py:61-71) */
void orc_weak_gradient(int64_t n, int64_t d, const int64_t* starts, const int32_t* idx,
                       const double* f, const double* vols, const double* gw, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t a = 0; a < d; ++a) out[i * d + a] = 0.0;
    for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
      const int64_t j = idx[k];
      const double fbar_v = 0.5 * (f[i] + f[j]) * vols[j];
      for (int64_t a = 0; a < d; ++a) out[i * d + a] += 2.0 * fbar_v * gw[k * d + a];
    }
  }
}

/* _accelerations (tlsph.py:88-102) */
void orc_tl_accelerations(int64_t n, int64_t d, const int64_t* starts, const int32_t* idx,
                          const double* g0, const double* q, double rho0, double* acc) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t a = 0; a < d; ++a) acc[i * d + a] = 0.0;
    for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
      int64_t j = idx[k];
      for (int64_t a = 0; a < d; ++a) {
        double t = 0.0;
        for (int64_t b = 0; b < d; ++b)
          t += (q[(i * d + a) * d + b] + q[(j * d + a) * d + b]) * g0[k * d + b];
        acc[i * d + a] += t / rho0;
      }
    }
  }
}

/* _deformation_rates (tlsph.py:105-123) */
void orc_tl_deformation_rates(int64_t n, int64_t d, const int64_t* starts, const int32_t* idx,
                              const double* g0, const double* v, const double* b0, double* dF) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t k = starts[i]; k < starts[i + 1]; ++k) {
      int64_t j = idx[k];
      for (int64_t a = 0; a < d; ++a) {
        double dv = v[j * d + a] - v[i * d + a];
        for (int64_t b = 0; b < d; ++b) m[a * d + b] += dv * g0[k * d + b];
      }
    }
    for (int64_t a = 0; a < d; ++a)
      for (int64_t b = 0; b < d; ++b) {
        double t = 0.0;
        for (int64_t c = 0; c < d; ++c) t += m[a * d + c] * b0[(i * d + c) * d + b];
        dF[(i * d + a) * d + b] = t;
      }
  }
}

int orc_max_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
