/*
 * uc_oracle.c — CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the CPU baseline — never as the product path.
 *
 * Restated from the reference implementation (paths under
 * /root/reference/pkg/src/undercool/):
 *   orc_residual       assembly.py:110-171 (gather, Gauss-point state, scatter)
 *                      + models/free_growth.py:97-146, models/alloy.py:137-208
 *                      + stepping.py:40-50 (lagged rate)
 *   orc_field_stencil  assembly.py:193-211,271-303 + free_growth.py:223-231,
 *                      alloy.py:286-300 + anisotropy.py:31-62
 *   orc_rap            precond.py:162-206 (Galerkin P^T A P, kron'd 1D linear P)
 *   orc_sgs            precond.py:74-85,113-121 (multicolor symmetric GS)
 *   orc_resid / orc_restrict / orc_prolong_add   precond.py:208-222
 *
 * Formulation deliberately differs from the CUDA path: full tensor basis
 * tables (no sum factorisation) and an element loop whose scatter runs colour
 * class by colour class (mesh.py:236-243 parity colours, race-free under
 * OpenMP), i.e. a different summation order from both numpy's bincount and
 * the device's marching gather.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int32_t dim;
  int32_t pad;
  int64_t ne[3];
  double h[3];
} orc_grid;

typedef struct {
  int32_t model; /* 1 free growth, 2 alloy */
  int32_t normalized;
  double eps, reg, bg, beta, alpha, latent, hcell, tmelt;
  double at_reg2, kpart, coupling, dcoef, g4_coef, pull_velocity;
} orc_params;

/* ---- basis tables (mesh.py:52-61, 151-176) ---------------------------- */
typedef struct {
  int dim, nq, nloc;
  double val[27][8];
  double grad[27][8][3];
  double jxw[27];
  double pt[27][3];
} tables;

static void make_tables(const orc_grid* g, tables* t) {
  /* numpy leggauss(3) bit patterns */
  const double x[3] = {-0x1.8c97ef43f7248p-1, 0.0, 0x1.8c97ef43f7248p-1};
  const double w[3] = {0x1.1c71c71c71c73p-1, 0x1.c71c71c71c71cp-1, 0x1.1c71c71c71c73p-1};
  const int d = g->dim;
  t->dim = d;
  t->nq = d == 3 ? 27 : 9;
  t->nloc = d == 3 ? 8 : 4;
  double detj = 1.0;
  for (int a = 0; a < d; ++a) detj *= g->h[a] / 2.0;
  for (int q = 0; q < t->nq; ++q) {
    int qa[3] = {q % 3, (q / 3) % 3, q / 9};
    double wq = 1.0;
    for (int a = d - 1; a >= 0; --a) wq *= w[qa[a]];
    t->jxw[q] = wq * detj;
    for (int a = 0; a < d; ++a) t->pt[q][a] = x[qa[a]];
    for (int l = 0; l < t->nloc; ++l) {
      int ja[3] = {l & 1, (l >> 1) & 1, (l >> 2) & 1};
      double v = 1.0;
      for (int a = 0; a < d; ++a) v *= ja[a] ? (1.0 + x[qa[a]]) / 2.0 : (1.0 - x[qa[a]]) / 2.0;
      t->val[q][l] = v;
      for (int a = 0; a < d; ++a) {
        double gg = 1.0;
        for (int b = 0; b < d; ++b) {
          if (b == a)
            gg *= ja[b] ? 0.5 : -0.5;
          else
            gg *= ja[b] ? (1.0 + x[qa[b]]) / 2.0 : (1.0 - x[qa[b]]) / 2.0;
        }
        t->grad[q][l][a] = gg * (2.0 / g->h[a]);
      }
    }
  }
}

static inline void node_ids(const orc_grid* g, int64_t e, int64_t* ids, int64_t* ecoord) {
  const int64_t nnx = g->ne[0] + 1, nny = g->ne[1] + 1;
  const int64_t ex = e % g->ne[0];
  const int64_t r = e / g->ne[0];
  const int64_t ey = g->dim == 3 ? r % g->ne[1] : r;
  const int64_t ez = g->dim == 3 ? r / g->ne[1] : 0;
  ecoord[0] = ex;
  ecoord[1] = ey;
  ecoord[2] = ez;
  const int nloc = g->dim == 3 ? 8 : 4;
  for (int l = 0; l < nloc; ++l)
    ids[l] = (ex + (l & 1)) + nnx * ((ey + ((l >> 1) & 1)) + nny * (ez + ((l >> 2) & 1)));
}

static inline int64_t n_nodes(const orc_grid* g) {
  int64_t n = 1;
  for (int a = 0; a < g->dim; ++a) n *= g->ne[a] + 1;
  return n;
}
static inline int64_t n_elems(const orc_grid* g) {
  int64_t n = 1;
  for (int a = 0; a < g->dim; ++a) n *= g->ne[a];
  return n;
}

/* ---- anisotropy g and d(g^2)/dp (anisotropy.py:45-62) ----------------- */
static inline double aniso(const double* p, int d, double eps, double reg, double* dg, double* s2o) {
  const double avg = d == 3 ? 1.0 / 3.0 : 0.5;
  double p2[3] = {0, 0, 0}, s2 = 0, quart = 0;
  for (int a = 0; a < d; ++a) {
    p2[a] = p[a] * p[a];
    s2 += p2[a];
    quart += p2[a] * p2[a];
  }
  const double denom = s2 * s2 + reg;
  const double qa = quart + avg * reg;
  const double g = 1.0 - 3.0 * eps + 4.0 * eps * qa / denom;
  if (dg) {
    const double c = 32.0 * eps * g / (denom * denom);
    for (int a = 0; a < d; ++a) dg[a] = c * p[a] * (p2[a] * denom - qa * s2);
  }
  *s2o = s2;
  return g;
}

/* Gauss-point integrands of one level.  q[0] phase, q[1] second field,
 * gp/gs their gradients, rate/phio/xq as the reference's QuadState. */
static void integrands(const orc_params* P, int d, int newlvl, double theta, double dt,
                       double g4_shift, double phi, double sec, const double* gp,
                       const double* gs, double rate, double phio, double xq, double* r0,
                       double r1[2][3]) {
  const double wgt = newlvl ? theta : 1.0 - theta;
  const double sgn = newlvl ? 1.0 : -1.0;
  double dg[3], s2;
  const double g = aniso(gp, d, P->eps, P->reg, dg, &s2);
  const double g2 = g * g;
  if (P->model == 1) {
    /* phase: g^2 phi/dt*sign + w [bg/h^2 pq(1-2phi) - 5 beta/h (Tm - T) pq^2] */
    const double pq = phi * (1.0 - phi);
    r0[0] = g2 * phi * (sgn / dt) + wgt * P->bg / (P->hcell * P->hcell) * pq * (1.0 - 2.0 * phi) -
            wgt * 5.0 * P->beta / P->hcell * (P->tmelt - sec) * (pq * pq);
    const double nrm = sqrt(s2);
    for (int a = 0; a < d; ++a) {
      r1[0][a] = wgt * P->bg * g2 * gp[a] + 0.5 * wgt * nrm * dg[a];
      r1[1][a] = wgt * P->alpha * gs[a];
    }
    r0[1] = sec * (sgn / dt) - (newlvl ? P->latent * rate : 0.0);
  } else {
    const double k = P->kpart, omk = 1.0 - k;
    const double mass = 1.0 + omk * sec;
    const double one = 1.0 - phi * phi;
    const double g4 = P->g4_coef * (xq - g4_shift);
    const double src = phi - phi * phi * phi - P->coupling * one * one * (sec + g4);
    r0[0] = -wgt * src + (newlvl ? mass * g2 * (phi - phio) / dt : 0.0);
    for (int a = 0; a < d; ++a) r1[0][a] = wgt * g2 * gp[a] + 0.5 * wgt * s2 * dg[a];
    const double chi = 0.5 * (1.0 + k) - 0.5 * omk * phi;
    r0[1] = chi * sec * (sgn / dt);
    const double dq = wgt * P->dcoef * 0.5 * (1.0 - phi);
    for (int a = 0; a < d; ++a) r1[1][a] = dq * gs[a];
    if (newlvl) {
      r0[1] -= 0.5 * rate;
      double at = (1.0 / (2.0 * sqrt(2.0))) * mass * rate;
      if (P->normalized) at /= sqrt(s2 + P->at_reg2);
      for (int a = 0; a < d; ++a) r1[1][a] += at * gp[a];
    }
  }
}

/* out += assembled level (part 0 = new, 1 = old).  Returns the number of
 * non-finite integrands seen (first location in *loc: field,part,elem,qp). */
int64_t orc_residual(const orc_grid* g, const orc_params* P, double theta, double dt, int64_t step,
                     int part, const double* unew, const double* old, const double* prev,
                     double* out, int64_t* loc) {
  tables T;
  make_tables(g, &T);
  const int d = g->dim;
  const int64_t N = n_nodes(g), E = n_elems(g);
  const int newlvl = part == 0;
  const double t_new = (double)(step + 1) * dt;
  const double g4_shift = P->pull_velocity * t_new;
  const double ra = theta / dt, rb = (1.0 - theta) / dt;
  const double* st = newlvl ? unew : old;
  int64_t bad = 0;
  int64_t best = INT64_MAX;
  const int ncol = 1 << d;
  for (int col = 0; col < ncol; ++col) {
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t e = 0; e < E; ++e) {
      int64_t ids[8], ec[3];
      node_ids(g, e, ids, ec);
      const int c = (int)((ec[0] & 1) | ((ec[1] & 1) << 1) | ((ec[2] & 1) << 2));
      if (c != col) continue;
      double ph[8], se[8], rt[8], po[8];
      for (int l = 0; l < T.nloc; ++l) {
        ph[l] = st[ids[l]];
        se[l] = st[N + ids[l]];
        if (newlvl) {
          const double a = unew[ids[l]], o = old[ids[l]], p = prev[ids[l]];
          rt[l] = ra * (a - o) + rb * (o - p);
          po[l] = o;
        }
      }
      const double x0 = (double)ec[0] * g->h[0];
      double elem[2][8];
      memset(elem, 0, sizeof(elem));
      for (int q = 0; q < T.nq; ++q) {
        double phi = 0, sec = 0, rate = 0, phio = 0, gp[3] = {0, 0, 0}, gs[3] = {0, 0, 0};
        for (int l = 0; l < T.nloc; ++l) {
          phi += ph[l] * T.val[q][l];
          sec += se[l] * T.val[q][l];
          if (newlvl) {
            rate += rt[l] * T.val[q][l];
            phio += po[l] * T.val[q][l];
          }
          for (int a = 0; a < d; ++a) {
            gp[a] += ph[l] * T.grad[q][l][a];
            gs[a] += se[l] * T.grad[q][l][a];
          }
        }
        const double xq = x0 + (T.pt[q][0] + 1.0) / 2.0 * g->h[0];
        double r0[2], r1[2][3];
        integrands(P, d, newlvl, theta, dt, g4_shift, phi, sec, gp, gs, rate, phio, xq, r0, r1);
        for (int f = 0; f < 2; ++f) {
          int fin = isfinite(r0[f]);
          int which = fin ? -1 : 0;
          for (int a = 0; a < d && which < 0; ++a)
            if (!isfinite(r1[f][a])) which = 1 + a;
          if (which >= 0) {
            bad++;
            const int64_t key = (((int64_t)(f * (d + 1) + which)) << 44) | (e << 5) | q;
#pragma omp critical
            if (key < best) best = key;
          }
          for (int l = 0; l < T.nloc; ++l) {
            double s = r0[f] * T.val[q][l];
            for (int a = 0; a < d; ++a) s += r1[f][a] * T.grad[q][l][a];
            elem[f][l] += T.jxw[q] * s;
          }
        }
      }
      for (int f = 0; f < 2; ++f)
        for (int l = 0; l < T.nloc; ++l) out[f * N + ids[l]] += elem[f][l];
    }
  }
  if (bad && loc) {
    loc[0] = (best >> 44) / (d + 1);
    loc[1] = (best >> 44) % (d + 1);
    loc[2] = (best >> 5) & ((1LL << 39) - 1);
    loc[3] = best & 31;
  }
  return bad;
}

/* ---- preconditioner blocks -------------------------------------------- */
static inline int kidx(int d, int dx, int dy, int dz) {
  return (dx + 1) + 3 * (dy + 1) + (d == 3 ? 9 * (dz + 1) : 0);
}

/* stencil[N][3^d] (natural rows, offsets dx fastest) of block `blk`,
 * assembled from the frozen state `state` (assembly.py:271-303). */
void orc_field_stencil(const orc_grid* g, const orc_params* P, double theta, double dt,
                       const double* state, int blk, double* stencil) {
  tables T;
  make_tables(g, &T);
  const int d = g->dim, K = d == 3 ? 27 : 9;
  const int64_t N = n_nodes(g), E = n_elems(g);
  memset(stencil, 0, sizeof(double) * (size_t)N * K);
  const int ncol = 1 << d;
  for (int col = 0; col < ncol; ++col) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
      int64_t ids[8], ec[3];
      node_ids(g, e, ids, ec);
      const int c = (int)((ec[0] & 1) | ((ec[1] & 1) << 1) | ((ec[2] & 1) << 2));
      if (c != col) continue;
      double em[8][8];
      memset(em, 0, sizeof(em));
      for (int q = 0; q < T.nq; ++q) {
        double phi = 0, sec = 0, gp[3] = {0, 0, 0};
        for (int l = 0; l < T.nloc; ++l) {
          phi += state[ids[l]] * T.val[q][l];
          sec += state[N + ids[l]] * T.val[q][l];
          for (int a = 0; a < d; ++a) gp[a] += state[ids[l]] * T.grad[q][l][a];
        }
        double cm, cd;
        if (blk == 1 && P->model == 1) {
          cm = 1.0 / dt;
          cd = theta * P->alpha;
        } else if (blk == 1) {
          cm = (1.0 + P->kpart - (1.0 - P->kpart) * phi) / (2.0 * dt);
          cd = theta * P->dcoef * (1.0 - phi) / 2.0;
        } else {
          double s2;
          const double gg = aniso(gp, d, P->eps, P->reg, NULL, &s2);
          const double g2 = gg * gg;
          if (P->model == 1) {
            cm = g2 / dt;
            cd = theta * P->bg * g2;
          } else {
            cm = (1.0 + (1.0 - P->kpart) * sec) * g2 / dt;
            cd = theta * g2;
          }
        }
        cm *= T.jxw[q];
        cd *= T.jxw[q];
        for (int i = 0; i < T.nloc; ++i)
          for (int j = 0; j < T.nloc; ++j) {
            double gg = 0;
            for (int a = 0; a < d; ++a) gg += T.grad[q][i][a] * T.grad[q][j][a];
            em[i][j] += cm * T.val[q][i] * T.val[q][j] + cd * gg;
          }
      }
      for (int i = 0; i < T.nloc; ++i)
        for (int j = 0; j < T.nloc; ++j) {
          const int k = kidx(d, (j & 1) - (i & 1), ((j >> 1) & 1) - ((i >> 1) & 1),
                             ((j >> 2) & 1) - ((i >> 2) & 1));
          stencil[ids[i] * K + k] += em[i][j];
        }
    }
  }
}

/* Galerkin coarse stencil from a fine stencil on node grid n[] (coarse grid
 * (n-1)/2+1 per axis): A_c = P^T A P with P = kron of 1D linear interpolation. */
void orc_rap(int d, const int64_t* n, const double* fine, double* coarse) {
  const int K = d == 3 ? 27 : 9;
  int64_t nc[3] = {1, 1, 1}, nf[3] = {1, 1, 1};
  for (int a = 0; a < d; ++a) {
    nf[a] = n[a];
    nc[a] = (n[a] - 1) / 2 + 1;
  }
  const int64_t NC = nc[0] * nc[1] * nc[2];
  memset(coarse, 0, sizeof(double) * (size_t)NC * K);
  const int64_t NF = nf[0] * nf[1] * nf[2];
  /* scatter form: for each fine row i and each coupling j, distribute
   * A_ij * P_iI * P_jJ onto coarse (I, J) */
#pragma omp parallel for schedule(static)
  for (int64_t I = 0; I < NC; ++I) {
    const int64_t Ic[3] = {I % nc[0], (I / nc[0]) % nc[1], I / (nc[0] * nc[1])};
    double acc[27];
    memset(acc, 0, sizeof(acc));
    const int zr = d == 3 ? 1 : 0;
    for (int c2 = -zr; c2 <= zr; ++c2)
      for (int c1 = -1; c1 <= 1; ++c1)
        for (int c0 = -1; c0 <= 1; ++c0) {
          const int64_t i[3] = {2 * Ic[0] + c0, 2 * Ic[1] + c1, 2 * Ic[2] + c2};
          int ok = 1;
          for (int a = 0; a < 3; ++a) ok &= i[a] >= 0 && i[a] < nf[a];
          if (!ok) continue;
          const double wi = (c0 ? 0.5 : 1.0) * (c1 ? 0.5 : 1.0) * (c2 ? 0.5 : 1.0);
          const int64_t fi = i[0] + nf[0] * (i[1] + nf[1] * i[2]);
          for (int k = 0; k < K; ++k) {
            const int o[3] = {k % 3 - 1, (k / 3) % 3 - 1, d == 3 ? k / 9 - 1 : 0};
            int64_t j[3];
            int okj = 1;
            for (int a = 0; a < 3; ++a) {
              j[a] = i[a] + o[a];
              okj &= j[a] >= 0 && j[a] < nf[a];
            }
            if (!okj) continue;
            const double av = fine[fi * K + k] * wi;
            /* coarse nodes J with P_jJ != 0 */
            for (int s2 = 0; s2 < ((j[2] & 1) ? 2 : 1); ++s2)
              for (int s1 = 0; s1 < ((j[1] & 1) ? 2 : 1); ++s1)
                for (int s0 = 0; s0 < ((j[0] & 1) ? 2 : 1); ++s0) {
                  const int64_t J[3] = {(j[0] >> 1) + s0, (j[1] >> 1) + s1, (j[2] >> 1) + s2};
                  const double wj = ((j[0] & 1) ? 0.5 : 1.0) * ((j[1] & 1) ? 0.5 : 1.0) *
                                    ((j[2] & 1) ? 0.5 : 1.0);
                  acc[kidx(d, (int)(J[0] - Ic[0]), (int)(J[1] - Ic[1]), (int)(J[2] - Ic[2]))] +=
                      av * wj;
                }
          }
        }
    for (int k = 0; k < K; ++k) coarse[I * K + k] = acc[k];
  }
  (void)NF;
}

static inline double row_dot(int d, const int64_t* n, const double* A, int64_t row, const double* x) {
  const int K = d == 3 ? 27 : 9;
  const int64_t i0 = row % n[0], i1 = (row / n[0]) % n[1], i2 = d == 3 ? row / (n[0] * n[1]) : 0;
  double s = 0.0;
  for (int k = 0; k < K; ++k) {
    const int dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = d == 3 ? k / 9 - 1 : 0;
    const int64_t j0 = i0 + dx, j1 = i1 + dy, j2 = i2 + dz;
    if (j0 < 0 || j0 >= n[0] || j1 < 0 || j1 >= n[1] || (d == 3 && (j2 < 0 || j2 >= n[2])))
      continue;
    s += A[row * K + k] * x[j0 + n[0] * (j1 + n[1] * j2)];
  }
  return s;
}

/* `sweeps` symmetric multicolor Gauss-Seidel sweeps on x (in place). */
void orc_sgs(int d, const int64_t* n, const double* A, double* x, const double* b, int sweeps) {
  const int K = d == 3 ? 27 : 9;
  const int64_t N = n[0] * n[1] * (d == 3 ? n[2] : 1);
  const int ncol = 1 << d;
  for (int s = 0; s < sweeps; ++s)
    for (int pass = 0; pass < 2 * ncol; ++pass) {
      const int col = pass < ncol ? pass : 2 * ncol - 1 - pass;
#pragma omp parallel for schedule(static)
      for (int64_t r = 0; r < N; ++r) {
        const int64_t i0 = r % n[0], i1 = (r / n[0]) % n[1], i2 = d == 3 ? r / (n[0] * n[1]) : 0;
        if ((int)((i0 & 1) | ((i1 & 1) << 1) | ((i2 & 1) << 2)) != col) continue;
        const double diag = A[r * K + K / 2];
        x[r] += (b[r] - row_dot(d, n, A, r, x)) * (1.0 / diag);
      }
    }
}

void orc_resid(int d, const int64_t* n, const double* A, const double* x, const double* b, double* r) {
  const int64_t N = n[0] * n[1] * (d == 3 ? n[2] : 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) r[i] = b[i] - row_dot(d, n, A, i, x);
}

void orc_restrict(int d, const int64_t* n, const double* r, double* bc) {
  int64_t nc[3] = {1, 1, 1}, nf[3] = {1, 1, 1};
  for (int a = 0; a < d; ++a) {
    nf[a] = n[a];
    nc[a] = (n[a] - 1) / 2 + 1;
  }
  const int64_t NC = nc[0] * nc[1] * nc[2];
#pragma omp parallel for schedule(static)
  for (int64_t I = 0; I < NC; ++I) {
    const int64_t Ic[3] = {I % nc[0], (I / nc[0]) % nc[1], I / (nc[0] * nc[1])};
    double s = 0.0;
    const int zr = d == 3 ? 1 : 0;
    for (int c2 = -zr; c2 <= zr; ++c2)
      for (int c1 = -1; c1 <= 1; ++c1)
        for (int c0 = -1; c0 <= 1; ++c0) {
          const int64_t i0 = 2 * Ic[0] + c0, i1 = 2 * Ic[1] + c1, i2 = 2 * Ic[2] + c2;
          if (i0 < 0 || i0 >= nf[0] || i1 < 0 || i1 >= nf[1] || i2 < 0 || i2 >= nf[2]) continue;
          s += (c0 ? 0.5 : 1.0) * (c1 ? 0.5 : 1.0) * (c2 ? 0.5 : 1.0) * r[i0 + nf[0] * (i1 + nf[1] * i2)];
        }
    bc[I] = s;
  }
}

void orc_prolong_add(int d, const int64_t* n, const double* ec, double* x) {
  int64_t nc[3] = {1, 1, 1}, nf[3] = {1, 1, 1};
  for (int a = 0; a < d; ++a) {
    nf[a] = n[a];
    nc[a] = (n[a] - 1) / 2 + 1;
  }
  const int64_t NF = nf[0] * nf[1] * nf[2];
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < NF; ++i) {
    const int64_t f[3] = {i % nf[0], (i / nf[0]) % nf[1], i / (nf[0] * nf[1])};
    double s = 0.0;
    for (int s2 = 0; s2 < ((f[2] & 1) ? 2 : 1); ++s2)
      for (int s1 = 0; s1 < ((f[1] & 1) ? 2 : 1); ++s1)
        for (int s0 = 0; s0 < ((f[0] & 1) ? 2 : 1); ++s0) {
          const double w = ((f[0] & 1) ? 0.5 : 1.0) * ((f[1] & 1) ? 0.5 : 1.0) * ((f[2] & 1) ? 0.5 : 1.0);
          s += w * ec[((f[0] >> 1) + s0) + nc[0] * (((f[1] >> 1) + s1) + nc[1] * ((f[2] >> 1) + s2))];
        }
    x[i] += s;
  }
}

int orc_num_threads(void) {
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
