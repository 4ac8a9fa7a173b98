/*
 * oracle/lax.c — CPU ORACLE, Lax shock tube with one small cell and dual time stepping
 * (arXiv 2211.00705).  TEST INFRASTRUCTURE ONLY: see oracle/lax.h.
 *
 * Plain, slow, fp64, written in the paper's order: exact Riemann fluxes, the explicit
 * finite-volume update on every cell outside the block (P:753 on a fixed mesh), and Algorithm 2
 * (tab: algorithms) on the block {k-1, k, k+1} with dtau_i = theta_i dt,
 * theta_k = alpha, the residual of P:1128-1131 and the stopping rule of P:1132.
 * Readings L1-L7 are listed in DESIGN.md §3.
 */
#include "lax.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- exact Riemann solver, gamma-law gas ---------------- */

/* f_K(p) and its derivative: shock branch (p > p_K) from the Rankine-Hugoniot conditions,
 * rarefaction branch (p <= p_K) from the isentrope and the Riemann invariant. */
static void lax_fk(double g, double p, double rk, double pk, double ck, double* f, double* df) {
  if (p > pk) {
    const double A = 2.0 / ((g + 1.0) * rk), B = (g - 1.0) / (g + 1.0) * pk;
    const double q = sqrt(A / (B + p));
    *f = (p - pk) * q;
    *df = q * (1.0 - (p - pk) / (2.0 * (B + p)));
  } else {
    const double e = (g - 1.0) / (2.0 * g);
    *f = 2.0 * ck / (g - 1.0) * (pow(p / pk, e) - 1.0);
    *df = 1.0 / (rk * ck) * pow(p / pk, -(g + 1.0) / (2.0 * g));
  }
}

int eiso_lax_riemann(double g, const double wl[3], const double wr[3], double xi, double prim[3],
                     double* p_star, double* u_star, int32_t* iters) {
  const double rl = wl[0], ul = wl[1], pl = wl[2], rr = wr[0], ur = wr[1], pr = wr[2];
  if (!(rl > 0.0) || !(rr > 0.0) || !(pl > 0.0) || !(pr > 0.0)) return 3;
  const double cl = sqrt(g * pl / rl), cr = sqrt(g * pr / rr);
  if (2.0 / (g - 1.0) * (cl + cr) <= ur - ul) return 3;  /* vacuum generated */
  /* Newton on f(p) = f_L(p) + f_R(p) + (u_R - u_L) from the primitive-variable estimate (L4) */
  double p = 0.5 * (pl + pr) - 0.125 * (ur - ul) * (rl + rr) * (cl + cr);
  if (p < 1e-8 * fmin(pl, pr)) p = 1e-8 * fmin(pl, pr);
  int it = 0, ok = 0;
  for (it = 1; it <= 100; ++it) {
    double fL, dfL, fR, dfR;
    lax_fk(g, p, rl, pl, cl, &fL, &dfL);
    lax_fk(g, p, rr, pr, cr, &fR, &dfR);
    double pn = p - (fL + fR + ur - ul) / (dfL + dfR);
    if (pn < 1e-8 * fmin(pl, pr)) pn = 1e-8 * fmin(pl, pr);
    const double change = 2.0 * fabs(pn - p) / (pn + p);
    p = pn;
    if (change <= 1e-14) { ok = 1; break; }
  }
  if (iters) *iters = it;
  if (!ok) return 5;
  double fL, dfL, fR, dfR;
  lax_fk(g, p, rl, pl, cl, &fL, &dfL);
  lax_fk(g, p, rr, pr, cr, &fR, &dfR);
  const double u = 0.5 * (ul + ur) + 0.5 * (fR - fL);
  if (p_star) *p_star = p;
  if (u_star) *u_star = u;
  /* sample the self-similar solution at x/t = xi */
  const double gm = (g - 1.0) / (g + 1.0);
  if (xi <= u) {  /* left of the contact */
    if (p > pl) {  /* left shock */
      const double sl = ul - cl * sqrt((g + 1.0) / (2.0 * g) * p / pl + (g - 1.0) / (2.0 * g));
      if (xi <= sl) { prim[0] = rl; prim[1] = ul; prim[2] = pl; }
      else { prim[0] = rl * (p / pl + gm) / (gm * p / pl + 1.0); prim[1] = u; prim[2] = p; }
    } else {  /* left rarefaction */
      const double cs = cl * pow(p / pl, (g - 1.0) / (2.0 * g));
      if (xi <= ul - cl) { prim[0] = rl; prim[1] = ul; prim[2] = pl; }
      else if (xi >= u - cs) { prim[0] = rl * pow(p / pl, 1.0 / g); prim[1] = u; prim[2] = p; }
      else {  /* inside the fan */
        const double c = 2.0 / (g + 1.0) * (cl + 0.5 * (g - 1.0) * (ul - xi));
        prim[1] = 2.0 / (g + 1.0) * (cl + 0.5 * (g - 1.0) * ul + xi);
        prim[0] = rl * pow(c / cl, 2.0 / (g - 1.0));
        prim[2] = pl * pow(c / cl, 2.0 * g / (g - 1.0));
      }
    }
  } else {  /* right of the contact */
    if (p > pr) {  /* right shock */
      const double sr = ur + cr * sqrt((g + 1.0) / (2.0 * g) * p / pr + (g - 1.0) / (2.0 * g));
      if (xi >= sr) { prim[0] = rr; prim[1] = ur; prim[2] = pr; }
      else { prim[0] = rr * (p / pr + gm) / (gm * p / pr + 1.0); prim[1] = u; prim[2] = p; }
    } else {  /* right rarefaction */
      const double cs = cr * pow(p / pr, (g - 1.0) / (2.0 * g));
      if (xi >= ur + cr) { prim[0] = rr; prim[1] = ur; prim[2] = pr; }
      else if (xi <= u + cs) { prim[0] = rr * pow(p / pr, 1.0 / g); prim[1] = u; prim[2] = p; }
      else {
        const double c = 2.0 / (g + 1.0) * (cr - 0.5 * (g - 1.0) * (ur - xi));
        prim[1] = 2.0 / (g + 1.0) * (-cr + 0.5 * (g - 1.0) * ur + xi);
        prim[0] = rr * pow(c / cr, 2.0 / (g - 1.0));
        prim[2] = pr * pow(c / cr, 2.0 * g / (g - 1.0));
      }
    }
  }
  return 0;
}

int eiso_lax_flux(double g, const double wl[3], const double wr[3], double F[3]) {
  double w[3];
  const int s = eiso_lax_riemann(g, wl, wr, 0.0, w, NULL, NULL, NULL);
  if (s) return s;
  const double E = w[2] / (g - 1.0) + 0.5 * w[0] * w[1] * w[1];
  F[0] = w[0] * w[1];
  F[1] = w[0] * w[1] * w[1] + w[2];
  F[2] = w[1] * (E + w[2]);
  return 0;
}

/* conserved (rho, rho u, E) -> primitive (rho, u, p) */
static int lax_prim(double g, const double U[3], double w[3]) {
  if (!(U[0] > 0.0)) return 3;
  w[0] = U[0];
  w[1] = U[1] / U[0];
  w[2] = (g - 1.0) * (U[2] - 0.5 * U[1] * U[1] / U[0]);
  return w[2] > 0.0 ? 0 : 3;
}

static int lax_edge_flux(double g, const double Ul[3], const double Ur[3], double F[3], int64_t* solves) {
  double wl[3], wr[3];
  int s = lax_prim(g, Ul, wl);
  if (!s) s = lax_prim(g, Ur, wr);
  if (!s) s = eiso_lax_flux(g, wl, wr, F);
  ++*solves;
  return s;
}

/* ---------------- one case to t_end ---------------- */

int eiso_lax_run(const eiso_lax_case* c, double* rho, double* mom, double* E, double* x_faces,
                 eiso_lax_stats* st) {
  eiso_lax_stats S;
  memset(&S, 0, sizeof(S));
  const int64_t N = c->n;
  if (N < 6 || (N & 1) || !(c->alpha > 0.0) || !(c->x_right > c->x_left) || !(c->gamma > 1.0) ||
      !(c->cfl > 0.0) || !(c->theta_nb > 0.0) || !rho || !mom || !E) {
    S.status = 1;
    if (st) *st = S;
    return 1;
  }
  const double g = c->gamma, hh = (c->x_right - c->x_left) / (double)N;
  const int64_t nc = N + 1, k = N / 2;  /* L1: N/2 cells left of x = 0, the small cell k, N/2 right */
  double* h = malloc(sizeof(double) * nc);
  double (*U)[3] = malloc(sizeof(double[3]) * nc);
  double (*Un)[3] = malloc(sizeof(double[3]) * nc);
  double (*F)[3] = malloc(sizeof(double[3]) * (nc + 1));  /* F[i]: flux at the left face of cell i */
  for (int64_t i = 0; i < nc; ++i) {
    h[i] = i == k ? c->alpha * hh : hh;
    const int left = i < k;  /* the small cell lies in x > 0 */
    const double r = left ? c->rho_l : c->rho_r, u = left ? c->u_l : c->u_r, p = left ? c->p_l : c->p_r;
    U[i][0] = r; U[i][1] = r * u; U[i][2] = p / (g - 1.0) + 0.5 * r * u * u;
  }
  if (x_faces) {
    for (int64_t i = 0; i <= k; ++i) x_faces[i] = c->x_left + (double)i * hh;
    for (int64_t i = k + 1; i <= nc; ++i) x_faces[i] = x_faces[k] + h[k] + (double)(i - k - 1) * hh;
  }
  const int blk = c->implicit_block != 0;
  double t = 0.0;
  int status = 0;
  while (t < c->t_end && !status) {
    /* L2: dt = C_CFL h / S_max over the regular cells (with the block: every cell but k);
     * without the block the small cell's width enters (h_min) as in a plain explicit scheme */
    double smax = 0.0, hmin = INFINITY;
    for (int64_t i = 0; i < nc; ++i) {
      if (blk && i == k) continue;
      double w[3];
      if (lax_prim(g, U[i], w)) { status = 3; break; }
      const double s = fabs(w[1]) + sqrt(g * w[2] / w[0]);
      if (s > smax) smax = s;
      if (h[i] < hmin) hmin = h[i];
    }
    if (status) break;
    double dt = c->cfl * hmin / smax;
    if (t + dt > c->t_end) dt = c->t_end - t;  /* L6 */
    memcpy(Un, U, sizeof(double[3]) * nc);
    /* explicit fluxes from U^n; transmissive ends (L3): ghost = end cell */
    for (int64_t f = 0; f <= nc && !status; ++f) {
      const double* a = Un[f == 0 ? 0 : f - 1];
      const double* b = Un[f == nc ? nc - 1 : f];
      status = lax_edge_flux(g, a, b, F[f], &S.riemann_solves);
    }
    if (status) break;
    /* explicit update of every cell outside the block (fixed mesh) */
    for (int64_t i = 0; i < nc; ++i) {
      if (blk && i >= k - 1 && i <= k + 1) continue;
      for (int q = 0; q < 3; ++q) U[i][q] = Un[i][q] - dt / h[i] * (F[i + 1][q] - F[i][q]);
    }
    if (blk) {  /* Algorithm 2 on cells k-1, k, k+1 */
      const double theta[3] = {c->theta_nb, c->alpha, c->theta_nb};  /* P:1127, theta_k = alpha */
      double W[3][3], G[4][3];
      for (int j = 0; j < 3; ++j) memcpy(W[j], Un[k - 1 + j], sizeof(W[j]));
      memcpy(G[0], F[k - 1], sizeof(G[0]));  /* outer faces keep the explicit fluxes */
      memcpy(G[3], F[k + 2], sizeof(G[3]));
      int64_t l = 0;
      for (;;) {
        status = lax_edge_flux(g, W[0], W[1], G[1], &S.riemann_solves);
        if (!status) status = lax_edge_flux(g, W[1], W[2], G[2], &S.riemann_solves);
        if (status) break;
        double res[3];
        for (int j = 0; j < 3; ++j) {
          const double r = theta[j], dtau = theta[j] * dt;
          const int64_t i = k - 1 + j;
          res[j] = 0.0;
          for (int q = 0; q < 3; ++q) {
            const double target = Un[i][q] - dt / h[i] * (G[j + 1][q] - G[j][q]);
            const double wn = W[j][q] / (1.0 + r) + r / (1.0 + r) * target;
            const double rq = fabs((1.0 + r) * (wn - W[j][q]) / (dtau * fmax(fabs(W[j][q]), 1.0)));
            if (rq > res[j]) res[j] = rq;
            W[j][q] = wn;
          }
        }
        ++l;
        if (fmax(res[0], res[2]) < c->tol_nb && res[1] < c->tol_tiny) break;
        if (l >= c->dts_max_iter) { status = 7; break; }
      }
      if (status) break;
      /* Part 2: fluxes at the converged iterate, conservative update with the outer fluxes */
      status = lax_edge_flux(g, W[0], W[1], G[1], &S.riemann_solves);
      if (!status) status = lax_edge_flux(g, W[1], W[2], G[2], &S.riemann_solves);
      if (status) break;
      for (int j = 0; j < 3; ++j) {
        const int64_t i = k - 1 + j;
        for (int q = 0; q < 3; ++q) U[i][q] = Un[i][q] - dt / h[i] * (G[j + 1][q] - G[j][q]);
      }
      S.dts_iters += l;
      if (l > S.dts_max) S.dts_max = l;
    }
    t += dt;
    S.steps += 1;
  }
  for (int64_t i = 0; i < nc; ++i) { rho[i] = U[i][0]; mom[i] = U[i][1]; E[i] = U[i][2]; }
  S.t = t;
  S.status = status;
  if (st) *st = S;
  free(h); free(U); free(Un); free(F);
  return status;
}
