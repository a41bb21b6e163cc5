/*
 * oracle.c -- plain, slow, fp64 CPU definition of the SPH hot path of arXiv 2505.14538.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The CUDA product path
 * never links, calls or reads anything under oracle/, and this file shares no code,
 * header, table or constant generator with it.
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of SPEC.md,
 * "Rk" = reading k of DESIGN.md §3 (copied from SURVEY.md §8(c) c.2), "Eq. k" = the
 * paper's equation number.
 *
 * Every sum is evaluated in fp64 over neighbours in ASCENDING j (R24), with no FMA
 * contraction (built with -ffp-contract=off), so the brute-force and cell-list
 * neighbour enumerations give bit-identical sums (Pin-17).
 *
 * Positions are uint32 fixed point on a 2^-32 L grid (R25): x_a = X_a * L_a / 2^32.  The
 * minimum-image separation is the int32 difference of two coordinates, scaled.
 *
 * Parity status per function: all pinned by tests/test_oracle_*.py
 * except where a header comment below says "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_NOT_CONVERGED 5
#define ORC_ERR_MISSING 9 /* a neighbour's input of an earlier stage was not computed */

static const double PI = 3.14159265358979323846;

/* ---------------------------------------------------------------- parameters ---- */
typedef struct {
  double gamma_k;     /* H = gamma_k h; = 2 for M4 (R1)                  */
  double eta;         /* target n h^3 = eta^3 (R1)                 */
  double h_tol;       /* relative closure threshold, P:90 ("10^-4")             */
  int32_t h_max_iter; /* Newton cap (R7)                                        */
  double gamma_eos;   /* 5/3                                             */
  double beta;        /* Eq. 10 (3)                                      */
  double alpha_v_max; /* Eq. 13 (2)                                      */
  double ell;         /* Eq. 12 decay length 0.05                        */
  double alpha_c_min, alpha_c_max, beta_c; /* Eqs. 21, 23, 24           */
  double c_cfl;       /* S:261 (R22)                                            */
  int32_t fh_mode;    /* R8: 0 -> f = 1/Omega, 1 -> f = Omega (Eq. 8 literal)   */
} orc_params;

/* --------------------------------------------------------------- the kernel ---- */
/* Cubic spline M4 (R1): W(r,h) = w(r/h)/(pi h^3), support 2h.        */
double orc_w(double q) {
  if (q < 1.0) return 1.0 - 1.5 * q * q + 0.75 * q * q * q;
  if (q < 2.0) { double t = 2.0 - q; return 0.25 * t * t * t; }
  return 0.0;
}
/* dw/dq */
double orc_dw(double q) {
  if (q < 1.0) return -3.0 * q + 2.25 * q * q;
  if (q < 2.0) { double t = 2.0 - q; return -0.75 * t * t; }
  return 0.0;
}
/* d2w/dq2 (used only for a tolerance scale of the parity tests) */
double orc_ddw(double q) {
  if (q < 1.0) return -3.0 + 4.5 * q;
  if (q < 2.0) return 1.5 * (2.0 - q);
  return 0.0;
}
/* W, dW/dr and dW/dh.  dW/dh = -(3 W + r dW/dr)/h is Eq. 6's summand with n_d = 3
 * and "grad_i W" read as the scalar dW/dr (R6). */
void orc_kernel(double r, double h, double* W, double* dWdr, double* dWdh) {
  double q = r / h;
  double h3 = h * h * h;
  *W = orc_w(q) / (PI * h3);
  *dWdr = orc_dw(q) / (PI * h3 * h);
  *dWdh = -(3.0 * (*W) + r * (*dWdr)) / h;
}

/* ------------------------------------------------------------- geometry ------- */
typedef struct {
  int64_t n;
  double box[3];
  const uint32_t* X; /* [n][3] */
  int use_cells;
  double cell_side[3];
  int32_t ncell[3];
  int64_t* cell_start; /* [ncells+1] */
  int64_t* cell_idx;   /* particle indices sorted by cell, ascending within a cell */
} orc_geom;

static inline double sep(const orc_geom* g, int64_t i, int64_t j, int a) {
  int32_t d = (int32_t)(g->X[3 * i + a] - g->X[3 * j + a]); /* minimum image, R25 */
  return (double)d * (g->box[a] * (1.0 / 4294967296.0));
}
/* r_ij = r_i - r_j (R4) and |r_ij|^2 evaluated as (dx*dx + dy*dy) + dz*dz. */
static inline double sep2(const orc_geom* g, int64_t i, int64_t j, double d[3]) {
  d[0] = sep(g, i, j, 0);
  d[1] = sep(g, i, j, 1);
  d[2] = sep(g, i, j, 2);
  return d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

static int cell_of(const orc_geom* g, int64_t i, int a) {
  int c = (int)(((double)g->X[3 * i + a] / 4294967296.0) * g->ncell[a]);
  if (c >= g->ncell[a]) c = g->ncell[a] - 1;
  return c;
}

orc_geom* orc_geom_create(int64_t n, const double* box, const uint32_t* X, int use_cells, double min_side) {
  orc_geom* g = (orc_geom*)calloc(1, sizeof(orc_geom));
  g->n = n;
  memcpy(g->box, box, sizeof(double) * 3);
  g->X = X;
  g->use_cells = use_cells;
  if (use_cells) {
    int64_t nc = 1;
    for (int a = 0; a < 3; ++a) {
      int c = (int)floor(box[a] / min_side);
      if (c < 1) c = 1;
      if (c > 1024) c = 1024;
      g->ncell[a] = c;
      g->cell_side[a] = box[a] / c;
      nc *= c;
    }
    g->cell_start = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    g->cell_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t* key = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
      key[i] = ((int64_t)cell_of(g, i, 0) * g->ncell[1] + cell_of(g, i, 1)) * g->ncell[2] + cell_of(g, i, 2);
      g->cell_start[key[i] + 1]++;
    }
    for (int64_t c = 0; c < nc; ++c) g->cell_start[c + 1] += g->cell_start[c];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
    memcpy(fill, g->cell_start, sizeof(int64_t) * (size_t)nc);
    for (int64_t i = 0; i < n; ++i) g->cell_idx[fill[key[i]]++] = i; /* ascending i in a cell */
    free(fill);
    free(key);
  }
  return g;
}

void orc_geom_destroy(orc_geom* g) {
  if (!g) return;
  free(g->cell_start);
  free(g->cell_idx);
  free(g);
}

/* All j (including i itself) with |r_ij|^2 < R^2, ascending j.  Returns the count,
 * or -1 if cap is exceeded.  Brute force is the definition; the cell list is an
 * acceleration structure pinned against it (Pin-17). */
int64_t orc_neighbours(const orc_geom* g, int64_t i, double R, int64_t* out, int64_t cap) {
  double R2 = R * R, d[3];
  int64_t cnt = 0;
  if (!g->use_cells) {
    for (int64_t j = 0; j < g->n; ++j) {
      if (sep2(g, i, j, d) < R2) {
        if (cnt >= cap) return -1;
        out[cnt++] = j;
      }
    }
    return cnt;
  }
  int lo[3], hi[3], ci[3];
  for (int a = 0; a < 3; ++a) {
    int k = (int)ceil(R / g->cell_side[a]);
    ci[a] = cell_of(g, i, a);
    if (2 * k + 1 >= g->ncell[a]) { lo[a] = 0; hi[a] = g->ncell[a] - 1; ci[a] = 0; }
    else { lo[a] = -k; hi[a] = k; }
  }
  for (int dx = lo[0]; dx <= hi[0]; ++dx)
    for (int dy = lo[1]; dy <= hi[1]; ++dy)
      for (int dz = lo[2]; dz <= hi[2]; ++dz) {
        int cx = ((ci[0] + dx) % g->ncell[0] + g->ncell[0]) % g->ncell[0];
        int cy = ((ci[1] + dy) % g->ncell[1] + g->ncell[1]) % g->ncell[1];
        int cz = ((ci[2] + dz) % g->ncell[2] + g->ncell[2]) % g->ncell[2];
        int64_t c = ((int64_t)cx * g->ncell[1] + cy) * g->ncell[2] + cz;
        for (int64_t s = g->cell_start[c]; s < g->cell_start[c + 1]; ++s) {
          int64_t j = g->cell_idx[s];
          if (sep2(g, i, j, d) < R2) {
            if (cnt >= cap) return -1;
            out[cnt++] = j;
          }
        }
      }
  qsort(out, (size_t)cnt, sizeof(int64_t), cmp_i64);
  return cnt;
}

/* neighbour-buffer capacity per thread (a -1 return from orc_neighbours means it was
 * exceeded and is reported as ORC_ERR_ARG) */
static int64_t orc_cap(const orc_geom* g) {
  int64_t c = g->n > 0 ? g->n : 1;
  return c < (1 << 20) ? c : (1 << 20);
}

/* ------------------------------------------------------------ density loop ---- */
/* Density sums at smoothing length h for particle i (c.1 step 2, R2, R5):
 *   rho   = sum_j m_j W_ij                    Eq. 2  (self included)
 *   nhat  = sum_j W_ij                        Eq. 5  (self included)
 *   dn/dh = -sum_j (3 W_ij + r_ij dW/dr)/h    Eq. 6  (self included, R6)
 *   drho/dh = sum_j m_j dW_ij/dh              Eq. 6 pattern
 *   div v = -(1/rho) sum_{j!=i} m_j v_ij . grad_i W_ij      Eq. 3, difference form (R5)
 *   curl v = (1/rho) sum_{j!=i} m_j v_ij x grad_i W_ij      Eq. 4, difference form (R5)
 *   N_i   = #{j != i : r_ij < H_i}  (R2); coincident j != i (r = 0) skipped and counted
 * out[0..8] = rho, drho_dh, nhat, dn_dh, div, curl_x, curl_y, curl_z, (unused)   */
typedef struct {
  double rho, drho_dh, nhat, dn_dh, div, curl[3];
  double sdv; /* (1/rho) sum_{j!=i} m_j |dW/dr| |v_ij|: bounds every term of div and curl (a tolerance scale) */
  double sdt; /* the same with |dW/dr| -> q |d2W/dr dq|: sensitivity to the rounding of q (support edge) */
  int64_t count, coincident;
} dens_sums;

static int density_at(const orc_geom* g, const orc_params* p, int64_t i, double h, const double* v,
                      const double* m, int64_t* buf, int64_t cap, dens_sums* s) {
  double H = p->gamma_k * h, d[3];
  int64_t nn = orc_neighbours(g, i, H, buf, cap);
  if (nn < 0) return ORC_ERR_ARG;
  memset(s, 0, sizeof(*s));
  double divs = 0.0, cs[3] = {0, 0, 0};
  for (int64_t k = 0; k < nn; ++k) {
    int64_t j = buf[k];
    double r2 = sep2(g, i, j, d);
    double r = sqrt(r2);
    if (j != i && r2 == 0.0) { s->coincident++; continue; }
    double W, dWdr, dWdh;
    orc_kernel(r, h, &W, &dWdr, &dWdh);
    s->nhat += W;
    s->dn_dh += dWdh;
    s->rho += m[j] * W;
    s->drho_dh += m[j] * dWdh;
    if (j == i) continue;
    s->count++;
    double gw[3] = {dWdr * d[0] / r, dWdr * d[1] / r, dWdr * d[2] / r}; /* grad_i W_ij (R4) */
    double vij[3] = {v[3 * i] - v[3 * j], v[3 * i + 1] - v[3 * j + 1], v[3 * i + 2] - v[3 * j + 2]};
    divs += m[j] * (vij[0] * gw[0] + vij[1] * gw[1] + vij[2] * gw[2]);
    s->sdv += m[j] * fabs(dWdr) * sqrt(vij[0] * vij[0] + vij[1] * vij[1] + vij[2] * vij[2]);
    /* a relative error e of q moves dW/dr by e q |w''(q)|/(pi h^4): w' ~ (2 - q)^2 makes a pair near
     * the support edge carry a large relative error in any finite precision */
    s->sdt += m[j] * (r / h) * fabs(orc_ddw(r / h)) / (PI * h * h * h * h) *
              sqrt(vij[0] * vij[0] + vij[1] * vij[1] + vij[2] * vij[2]);
    cs[0] += m[j] * (vij[1] * gw[2] - vij[2] * gw[1]);
    cs[1] += m[j] * (vij[2] * gw[0] - vij[0] * gw[2]);
    cs[2] += m[j] * (vij[0] * gw[1] - vij[1] * gw[0]);
  }
  s->div = -divs / s->rho;
  s->sdv /= s->rho;
  s->sdt /= s->rho;
  for (int a = 0; a < 3; ++a) s->curl[a] = cs[a] / s->rho;
  return ORC_OK;
}

/* Density loop + Newton-Raphson h iteration ("ghost"; c.1 step 3; R7).
 *   g(h) = nhat(h) h^3 - eta^3;  converged when |g| <= h_tol eta^3
 *   g'(h) = 3 h^2 nhat + h^3 dnhat/dh
 *   h <- h - g/g', clamped to [h/2, 2h]; the bracket [lo, hi] is maintained from the
 *   sign of g (g is non-decreasing in h); a step leaving the bracket bisects it.
 *   h_max_iter Newton updates without convergence -> ORC_ERR_NOT_CONVERGED.
 *   h_max_iter == 0 -> density at the given h, no iteration ("fixed-h" mode).
 * For each i in idx[0..nidx): in h[i] (initial guess) -> out h[i]; out dens[i*8..]:
 *   rho, drho_dh, nhat, dn_dh, div, curl_x, curl_y, curl_z; count[i]; iters[i]; and, if
 *   scale_dv is not NULL, scale_dv[i] = (1/rho) sum_{j!=i} m_j |dW/dr| |v_ij| (the tolerance
 *   scale of div and curl: no term of either sum exceeds it in magnitude), and scale_dv_tail[i] the
 *   same sum with |dW/dr| replaced by q |d2W/dr dq| (the terms' sensitivity to the rounding of q).
 * Returns ORC_OK, or ORC_ERR_NOT_CONVERGED (state still written, flagged iters = -1). */
int orc_density(const orc_geom* g, const orc_params* p, const int64_t* idx, int64_t nidx, double* h,
                const double* v, const double* m, double* dens, int64_t* count, int32_t* iters,
                int64_t* coincident_total, double* scale_dv, double* scale_dv_tail) {
  int status = ORC_OK;
  int64_t coinc = 0;
  const double eta3 = p->eta * p->eta * p->eta;
#pragma omp parallel reduction(+ : coinc)
  {
    int64_t cap = orc_cap(g);
    int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
#pragma omp for schedule(dynamic, 64)
    for (int64_t t = 0; t < nidx; ++t) {
      int64_t i = idx[t];
      double hh = h[i], lo = 0.0, hi = INFINITY;
      dens_sums s;
      int it = 0, ok = 0;
      for (;;) {
        if (density_at(g, p, i, hh, v, m, buf, cap, &s) != ORC_OK) break;
        if (p->h_max_iter == 0) { ok = 1; break; }
        double g_ = s.nhat * hh * hh * hh - eta3;
        if (fabs(g_) <= p->h_tol * eta3) { ok = 1; break; }
        if (it >= p->h_max_iter) break;
        double gp = 3.0 * hh * hh * s.nhat + hh * hh * hh * s.dn_dh;
        if (g_ > 0.0) hi = hh; else lo = hh;
        double hn = (gp > 0.0) ? hh - g_ / gp : (g_ < 0.0 ? 2.0 * hh : 0.5 * hh);
        if (hn < 0.5 * hh) hn = 0.5 * hh;
        if (hn > 2.0 * hh) hn = 2.0 * hh;
        if (hn <= lo || hn >= hi) hn = 0.5 * (lo + hi);
        hh = hn;
        ++it;
      }
      h[i] = hh;
      double* o = dens + 8 * i;
      o[0] = s.rho; o[1] = s.drho_dh; o[2] = s.nhat; o[3] = s.dn_dh; o[4] = s.div;
      o[5] = s.curl[0]; o[6] = s.curl[1]; o[7] = s.curl[2];
      count[i] = s.count;
      if (scale_dv) scale_dv[i] = s.sdv;
      if (scale_dv_tail) scale_dv_tail[i] = s.sdt;
      iters[i] = ok ? it : -1;
      coinc += s.coincident;
      if (!ok) {
#pragma omp atomic write
        status = ORC_ERR_NOT_CONVERGED;
      }
    }
    free(buf);
  }
  if (coincident_total) *coincident_total = coinc;
  return status;
}

/* -------------------------------------------------------- density finalize ---- */
/* Elementwise (c.1 step 4): Omega = 1 + h/(3 rho) drho/dh (Eq. 8 with n_a = 3);
 * f = 1/Omega (fh_mode 0, R8) or Omega (fh_mode 1, literal Eq. 8);
 * P = (gamma-1) rho u, c_s = sqrt(gamma P/rho) (ideal gas);
 * B = |div v| / (|div v| + |curl v| + 1e-4 c_s/h), 0 if the denominator is 0 (R14).
 * out fin[i*4..] = f, P, c_s, B */
void orc_finalize(const orc_params* p, const int64_t* idx, int64_t nidx, const double* h, const double* u,
                  const double* dens, double* fin) {
  for (int64_t t = 0; t < nidx; ++t) {
    int64_t i = idx[t];
    const double* d = dens + 8 * i;
    double rho = d[0];
    double Omega = 1.0 + h[i] / (3.0 * rho) * d[1];
    double f = p->fh_mode ? Omega : 1.0 / Omega;
    double P = (p->gamma_eos - 1.0) * rho * u[i];
    double c = sqrt(p->gamma_eos * P / rho);
    double adiv = fabs(d[4]);
    double acurl = sqrt(d[5] * d[5] + d[6] * d[6] + d[7] * d[7]);
    double den = adiv + acurl + 1e-4 * c / h[i];
    double B = den > 0.0 ? adiv / den : 0.0;
    fin[4 * i] = f; fin[4 * i + 1] = P; fin[4 * i + 2] = c; fin[4 * i + 3] = B;
  }
}

/* ----------------------------------------------------------- gradient loop ---- */
/* c.1 step 5, over j != i with r_ij < H_i (R2):
 *   mu_ij = min(0, v_ij . r_ij/|r_ij|)                      Eq. 11 (R4)
 *   v_sig,i = max(2 c_i, max_j (c_i + c_j - beta mu_ij))    Eq. 10 (R15)
 *   lap u_i = 2 sum_j (m_j/rho_j)(u_i - u_j) dW/dr(r_ij, h_i)/|r_ij|   Brookshaw (R16)
 * `valid` marks particles whose density-stage outputs exist (sampled runs).
 * out grad[i*2..] = v_sig, lap_u; scale_lap[i] (if not NULL) = 2 sum_j (m_j/rho_j)|u_i - u_j||dW/dr|/r,
 * the sum of the magnitudes of lap u's terms (a tolerance scale); scale_lap_tail[i] the same with
 * |dW/dr| replaced by q |d2W/dr dq| (sensitivity to the rounding of q near the support edge) */
int orc_gradient(const orc_geom* g, const orc_params* p, const int64_t* idx, int64_t nidx, const double* h,
                 const double* v, const double* m, const double* u, const double* rho, const double* c,
                 const uint8_t* valid, double* grad, double* scale_lap, double* scale_lap_tail) {
  int status = ORC_OK;
#pragma omp parallel
  {
    int64_t cap = orc_cap(g);
    int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
#pragma omp for schedule(dynamic, 64)
    for (int64_t t = 0; t < nidx; ++t) {
      int64_t i = idx[t];
      double H = p->gamma_k * h[i], d[3];
      int64_t nn = orc_neighbours(g, i, H, buf, cap);
      double vsig = 2.0 * c[i], lap = 0.0, slap = 0.0, stail = 0.0;
      for (int64_t k = 0; k < nn; ++k) {
        int64_t j = buf[k];
        if (j == i) continue;
        double r2 = sep2(g, i, j, d);
        if (r2 == 0.0) continue;
        if (valid && !valid[j]) {
#pragma omp atomic write
          status = ORC_ERR_MISSING;
          continue;
        }
        double r = sqrt(r2);
        double vr = (v[3 * i] - v[3 * j]) * d[0] + (v[3 * i + 1] - v[3 * j + 1]) * d[1] +
                    (v[3 * i + 2] - v[3 * j + 2]) * d[2];
        double mu = vr < 0.0 ? vr / r : 0.0;
        double vs = c[i] + c[j] - p->beta * mu;
        if (vs > vsig) vsig = vs;
        double W, dWdr, dWdh;
        orc_kernel(r, h[i], &W, &dWdr, &dWdh);
        lap += m[j] / rho[j] * (u[i] - u[j]) * dWdr / r;
        slap += m[j] / rho[j] * fabs(u[i] - u[j]) * fabs(dWdr) / r;
        stail += m[j] / rho[j] * fabs(u[i] - u[j]) * (r / h[i]) * fabs(orc_ddw(r / h[i])) /
                 (PI * h[i] * h[i] * h[i] * h[i] * r);
      }
      grad[2 * i] = vsig;
      grad[2 * i + 1] = 2.0 * lap;
      if (scale_lap) scale_lap[i] = 2.0 * slap;
      if (scale_lap_tail) scale_lap_tail[i] = 2.0 * stail;
    }
    free(buf);
  }
  return status;
}

/* ---------------------------------------------------------- gradient ghost ---- */
/* Elementwise switch evolution, c.1 step 6:
 *   Ddot = (div - div_prev)/dt (Eq. 15; 0 on the first step, R19)
 *   S = H^2 max(0, -Ddot)                                   Eq. 14
 *   alpha_loc = alpha_v_max S/(v_sig^2 + S)                 Eq. 13 without the trailing dt (R18)
 *   alpha_v <- alpha_loc if alpha_v < alpha_loc, else alpha_loc + (alpha_v - alpha_loc) exp(-ell c dt/H)  (R17)
 *   dalpha_c/dt = beta_c H lap_u/sqrt(u) - (alpha_c - alpha_c_min) v_sig/H  (Eq. 21 read as R20;
 *                 source term 0 if u <= 0)
 *   alpha_c <- clamp(alpha_c + dt dalpha_c/dt, alpha_c_min, max(alpha_c_min, alpha_c_max (1 - alpha_v/alpha_v_max)))
 *                 (Eqs. 23-24 read as R21, with the alpha_v just updated)
 *   div_prev <- div
 * state[i*3..] = alpha_v, alpha_c, div_prev (in/out) */
void orc_gradient_ghost(const orc_params* p, const int64_t* idx, int64_t nidx, double dt, int first_step,
                        const double* h, const double* u, const double* c, const double* div, const double* grad,
                        double* state) {
  for (int64_t t = 0; t < nidx; ++t) {
    int64_t i = idx[t];
    double H = p->gamma_k * h[i];
    double av = state[3 * i], ac = state[3 * i + 1], dprev = state[3 * i + 2];
    double vsig = grad[2 * i], lap = grad[2 * i + 1];
    double Ddot = first_step ? 0.0 : (div[i] - dprev) / dt;
    double S = H * H * (-Ddot > 0.0 ? -Ddot : 0.0);
    double aloc = (vsig * vsig + S) > 0.0 ? p->alpha_v_max * S / (vsig * vsig + S) : 0.0;
    if (av < aloc) av = aloc;
    else av = aloc + (av - aloc) * exp(-p->ell * c[i] * dt / H);
    double src = u[i] > 0.0 ? p->beta_c * H * lap / sqrt(u[i]) : 0.0;
    double dac = src - (ac - p->alpha_c_min) * vsig / H;
    ac = ac + dt * dac;
    double ceil_ = p->alpha_c_max * (1.0 - av / p->alpha_v_max);
    if (ceil_ < p->alpha_c_min) ceil_ = p->alpha_c_min;
    if (ac > ceil_) ac = ceil_;
    if (ac < p->alpha_c_min) ac = p->alpha_c_min;
    state[3 * i] = av;
    state[3 * i + 1] = ac;
    state[3 * i + 2] = div[i];
  }
}

/* -------------------------------------------------------------- force loop ---- */
/* c.1 step 7 (R3, R9-R13), gather form of the pairwise sums of Eqs. 7, 17-19
 * over j != i with r_ij < max(H_i, H_j) (symmetric neighbour set, R3):
 *   G_i = f_i dW/dr(r_ij, h_i)/|r_ij| (0 if r_ij >= H_i);  G_j likewise with h_j
 *   A_i = P_i/rho_i^2;  Gbar = (G_i + G_j)/2
 *   mu_ij = min(0, v_ij . r_hat_ij) (Eq. 11);  v_sig,ij = c_i + c_j - beta mu_ij (Eq. 10)
 *   abar_ij = (alpha_v,i + alpha_v,j)/2 * (B_i + B_j)/2            Eq. 16
 *   Pi_ij = -abar_ij mu_ij v_sig,ij / ((rho_i + rho_j)/2)           Eq. 9 read as R9
 *   S_ij = A_i G_i + A_j G_j + Pi_ij Gbar
 *   a_i = -sum_j m_j S_ij r_ij                                     Eqs. 17 + 7
 *   alpha_c,ij = (P_i a_c,i + P_j a_c,j)/(P_i + P_j), or the mean if P_i + P_j = 0   Eq. 20 (R13)
 *   v_c,ij = |v_ij . r_hat_ij| + sqrt(2 |P_i - P_j|/(rho_i + rho_j))  Eq. 22 (R12)
 *   D_ij = alpha_c,ij v_c,ij (u_i - u_j)(G_i + G_j)|r_ij|/(rho_i + rho_j)   Eq. 19 (R11)
 *   du_i/dt = sum_j m_j [A_i G_i (v_ij.r_ij) + Pi_ij Gbar (v_ij.r_ij)/2 + D_ij]   Eq. 18 + R10 + Eq. 19
 *   v_sig,i = max(2 c_i, max_j v_sig,ij)                           (R15)
 * Also returns per-particle tolerance scales  sa_i = sum_j m_j |S_ij| |r_ij|  and
 * su_i = sum_j m_j (|A_i G_i v.r| + |Pi Gbar v.r|/2 + |D_ij|), and the pair count.
 * pp[i*8..] = f, P, c, B, rho, u, alpha_v, alpha_c.  out force[i*11..] = ax, ay, az, du,
 * v_sig, sa, su, count, sc, st, sv (the last three: sensitivity scales, below). */
int orc_force(const orc_geom* g, const orc_params* p, const int64_t* idx, int64_t nidx, const double* h,
              const double* v, const double* m, const double* pp, const uint8_t* valid, double h_max,
              double* force) {
  int status = ORC_OK;
#pragma omp parallel
  {
    int64_t cap = orc_cap(g);
    int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
#pragma omp for schedule(dynamic, 64)
    for (int64_t t = 0; t < nidx; ++t) {
      int64_t i = idx[t];
      double Hi = p->gamma_k * h[i];
      double R = Hi > p->gamma_k * h_max ? Hi : p->gamma_k * h_max;
      int64_t nn = orc_neighbours(g, i, R, buf, cap);
      const double* qi = pp + 8 * i;
      double fi = qi[0], Pi_ = qi[1], ci = qi[2], Bi = qi[3], rhoi = qi[4], ui = qi[5], avi = qi[6], aci = qi[7];
      double Ai = Pi_ / (rhoi * rhoi);
      double a[3] = {0, 0, 0}, du = 0.0, vsig = 2.0 * ci, sa = 0.0, su = 0.0, sc = 0.0, st = 0.0, sv = 0.0, d[3];
      int64_t cnt = 0;
      for (int64_t k = 0; k < nn; ++k) {
        int64_t j = buf[k];
        if (j == i) continue;
        double r2 = sep2(g, i, j, d);
        if (r2 == 0.0) continue;
        double Hj = p->gamma_k * h[j];
        double Hmax = Hi > Hj ? Hi : Hj;
        if (!(r2 < Hmax * Hmax)) continue;
        if (valid && !valid[j]) {
#pragma omp atomic write
          status = ORC_ERR_MISSING;
          continue;
        }
        const double* qj = pp + 8 * j;
        double fj = qj[0], Pj = qj[1], cj = qj[2], Bj = qj[3], rhoj = qj[4], uj = qj[5], avj = qj[6], acj = qj[7];
        double r = sqrt(r2);
        double W, dWi, dWj, dh;
        double Gi = 0.0, Gj = 0.0;
        if (r2 < Hi * Hi) { orc_kernel(r, h[i], &W, &dWi, &dh); Gi = fi * dWi / r; }
        if (r2 < Hj * Hj) { orc_kernel(r, h[j], &W, &dWj, &dh); Gj = fj * dWj / r; }
        double Aj = Pj / (rhoj * rhoj);
        double vr = (v[3 * i] - v[3 * j]) * d[0] + (v[3 * i + 1] - v[3 * j + 1]) * d[1] +
                    (v[3 * i + 2] - v[3 * j + 2]) * d[2];
        double mu = vr < 0.0 ? vr / r : 0.0;
        double vs = ci + cj - p->beta * mu;
        double abar = 0.5 * (avi + avj) * 0.5 * (Bi + Bj);
        double PiV = -abar * mu * vs / (0.5 * (rhoi + rhoj));
        double Gbar = 0.5 * (Gi + Gj);
        double S = Ai * Gi + Aj * Gj + PiV * Gbar;
        for (int ax = 0; ax < 3; ++ax) a[ax] -= m[j] * S * d[ax];
        double acij = (Pi_ + Pj) > 0.0 ? (Pi_ * aci + Pj * acj) / (Pi_ + Pj) : 0.5 * (aci + acj);
        double vc = fabs(vr / r) + sqrt(2.0 * fabs(Pi_ - Pj) / (rhoi + rhoj));
        double D = acij * vc * (ui - uj) * (Gi + Gj) * r / (rhoi + rhoj);
        double t1 = Ai * Gi * vr, t2 = 0.5 * PiV * Gbar * vr;
        du += m[j] * (t1 + t2 + D);
        if (vs > vsig) vsig = vs;
        sa += m[j] * fabs(S) * r;
        su += m[j] * (fabs(t1) + fabs(t2) + fabs(D));
        /* sensitivity to the rounding of v_ij . r_ij: the du terms with |v_ij . r_ij| replaced by
         * |v_ij| |r_ij| (a rigid rotation has v_ij . r_ij = 0 up to the input rounding of v, so its
         * terms are rounding-level and any finite precision resolves them only to ~eps |v||r|) */
        {
          double vn = sqrt((v[3 * i] - v[3 * j]) * (v[3 * i] - v[3 * j]) +
                           (v[3 * i + 1] - v[3 * j + 1]) * (v[3 * i + 1] - v[3 * j + 1]) +
                           (v[3 * i + 2] - v[3 * j + 2]) * (v[3 * i + 2] - v[3 * j + 2]));
          sv += m[j] * (fabs(Ai * Gi) + fabs(0.5 * PiV * Gbar)) * vn * r;
        }
        /* sensitivity of D to the pressure difference inside v_c (Eq. 22): sqrt(2|P_i-P_j|/rho)
         * has an unbounded derivative at P_i = P_j.  An error of the pressures of relative size
         * EPS_P = 1e-6 (f32 densities and the h-iteration tolerance) moves |P_i - P_j| by at most
         * EPS_P (P_i + P_j), hence v_c by at most
         *   dv = sqrt(2 (|P_i-P_j| + EPS_P (P_i+P_j))/rho_s) - sqrt(2 |P_i-P_j|/rho_s)
         * (~ sqrt(2 EPS_P (P_i+P_j)/rho_s) when P_i = P_j, EPS_P (P_i+P_j)/(rho_s v_p) once
         * |P_i - P_j| >> EPS_P (P_i + P_j)).  sc = sum_j m_j |D_ij/v_c| dv: an absolute du bound. */
        {
          const double EPS_P = 1e-6, rs = rhoi + rhoj, dP = fabs(Pi_ - Pj);
          const double dv = sqrt(2.0 * (dP + EPS_P * (Pi_ + Pj)) / rs) - sqrt(2.0 * dP / rs);
          sc += m[j] * fabs(acij * (ui - uj) * (Gi + Gj) * r / rs) * dv;
        }
        /* sensitivity to the kernel derivative near the support edge: w'(q) ~ (2-q)^2 has a
         * large relative error when q -> 2 in any finite precision.  A relative error e of q
         * moves w' by e q |w''(q)|; st = the du terms with |w'| replaced by q |w''(q)|, so the
         * du error from rounding q is <= e st. */
        {
          double qi = r / h[i], qj = r / h[j];
          double Ki = (r2 < Hi * Hi) ? fi * qi * fabs(orc_ddw(qi)) / (PI * h[i] * h[i] * h[i] * h[i] * r) : 0.0;
          double Kj = (r2 < Hj * Hj) ? fj * qj * fabs(orc_ddw(qj)) / (PI * h[j] * h[j] * h[j] * h[j] * r) : 0.0;
          st += m[j] * ((fabs(Ai) * Ki + fabs(0.5 * PiV) * 0.5 * (Ki + Kj)) * fabs(vr) +
                        fabs(acij * vc * (ui - uj)) * (Ki + Kj) * r / (rhoi + rhoj));
        }
        cnt++;
      }
      double* o = force + 11 * i;
      o[0] = a[0]; o[1] = a[1]; o[2] = a[2]; o[3] = du; o[4] = vsig; o[5] = sa; o[6] = su; o[7] = (double)cnt;
      o[8] = sc; o[9] = st; o[10] = sv;
    }
    free(buf);
  }
  return status;
}

/* ------------------------------------------------------------ CFL timestep ---- */
/* dt = C_cfl min_i 2 gamma_k h_i / v_sig,i  (R22) */
double orc_dt(const orc_params* p, const int64_t* idx, int64_t nidx, const double* h, const double* vsig) {
  double dt = INFINITY;
  for (int64_t t = 0; t < nidx; ++t) {
    int64_t i = idx[t];
    double d = p->c_cfl * 2.0 * p->gamma_k * h[i] / vsig[i];
    if (d < dt) dt = d;
  }
  return dt;
}

/* ------------------------------------------------------------ kick / drift ---- */
/* Kick: v <- v + a dt_k; u <- max(0, u + du dt_k).
 * Drift: x <- wrap(x + v dt_d) on the 2^-32 L fixed-point grid, rounding to nearest
 * (R25).  X is modified in place. */
void orc_kick_drift(int64_t n, const double* box, double dt_k, double dt_d, const double* a, const double* du,
                    double* v, double* u, uint32_t* X) {
  for (int64_t i = 0; i < n; ++i) {
    for (int ax = 0; ax < 3; ++ax) v[3 * i + ax] += a[3 * i + ax] * dt_k;
    u[i] += du[i] * dt_k;
    if (u[i] < 0.0) u[i] = 0.0;
    for (int ax = 0; ax < 3; ++ax) {
      double units = v[3 * i + ax] * dt_d / box[ax] * 4294967296.0;
      int64_t k = (int64_t)llround(units);
      X[3 * i + ax] = (uint32_t)((uint64_t)X[3 * i + ax] + (uint64_t)k);
    }
  }
}

/* ------------------------------------------------------- closure for sampling -- */
/* Mark every particle within R of a marked one (sampled parity needs the 1- and
 * 2-hop neighbourhoods of the sample to be computed upstream). */
void orc_closure(const orc_geom* g, const uint8_t* in, double R, uint8_t* out) {
  memcpy(out, in, (size_t)g->n);
#pragma omp parallel
  {
    int64_t cap = orc_cap(g);
    int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < g->n; ++i) {
      if (!in[i]) continue;
      int64_t nn = orc_neighbours(g, i, R, buf, cap);
      for (int64_t k = 0; k < nn; ++k) out[buf[k]] = 1; /* benign race: all writers store 1 */
    }
    free(buf);
  }
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
