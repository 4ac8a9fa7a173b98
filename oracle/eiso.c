/*
 * oracle/eiso.c — plain, slow, fp64 CPU ORACLE of the explicit-implicit domain splitting
 * method of May & Thein (arXiv 2211.00705) for 1D isothermal liquid-vapour Euler flow.
 *
 * TEST INFRASTRUCTURE ONLY (see eiso.h): loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py; never by the product path.  It shares no
 * code with paper_2211_00705_b200/csrc.  Deliberate differences from the GPU path so that a
 * shared mistake is unlikely: forward-difference Newton Jacobians (GPU: analytic Eq. (14),
 * P:1505-1519), sequential Armijo back-tracking (GPU: lane-parallel candidates), outer-wave
 * functions in the printed pressure form (GPU: density form, R19), no fast paths.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (see __graft_entry__.build).
 * Every function cites the passage of /root/reference/PAPER.md ("P:n") it follows and the
 * DESIGN.md reading ("R<k>") where the paper is silent, ambiguous or garbled.
 *
 * Parity pins: tests/test_oracle_pins.py (paper values), tests/test_oracle_props.py
 * (closed forms, brute force, invariants).  Parts pinned only by invariants are marked
 * "parity unpinned" below and in DESIGN.md.
 */
#include "eiso.h"
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define VAP EISO_VAP
#define LIQ EISO_LIQ
#define SPIN EISO_SPIN

/* ------------------------------------------------------------------------------------------
 * L0 thermodynamics
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  double a_v2, a_v, a_l, a_l2, rho0, p0, tau, p_min, rho_min, rho_tilde, p_tilde;
} eos_t;

/* Maxwell equal-area residual along the EOS path liquid -> linear spinodal -> vapour
 * ("connected linearly with respect to the density ... Maxwell condition
 * holds"; reading R3).  Integral of v dp from (rho0,p0) to (rho_V0,p0):
 *   a_l^2 ln(rho_min/rho0) + s ln(rho_t/rho_min) + a_v^2 ln(rho_V0/rho_t),
 *   s = (a_v^2 rho_t - p_min)/(rho_t - rho_min). */
static double maxwell_residual(const eos_t* e, double rho_t) {
  double rho_v0 = e->p0 / e->a_v2;
  double s = (e->a_v2 * rho_t - e->p_min) / (rho_t - e->rho_min);
  return e->a_l2 * log(e->rho_min / e->rho0) + s * log(rho_t / e->rho_min) +
         e->a_v2 * log(rho_v0 / rho_t);
}

static int maxwell_rho_tilde(const eos_t* e, double* out) {
  /* plain bracket scan on a geometric grid in (rho_V0, rho_min), then bisection */
  double lo = e->p0 / e->a_v2, hi = e->rho_min;
  int K = 4000;
  double prev_x = lo * (1.0 + 1e-12), prev_f = maxwell_residual(e, prev_x);
  for (int k = 1; k <= K; ++k) {
    double x = lo * pow(hi / lo, (double)k / K) * (k == K ? (1.0 - 1e-12) : 1.0);
    double f = maxwell_residual(e, x);
    if ((prev_f < 0.0) != (f < 0.0)) {
      double a = prev_x, b = x, fa = prev_f;
      for (int it = 0; it < 300; ++it) {
        double m = 0.5 * (a + b);
        if (m <= a || m >= b) break;
        double fm = maxwell_residual(e, m);
        if ((fa < 0.0) == (fm < 0.0)) { a = m; fa = fm; } else { b = m; }
      }
      *out = 0.5 * (a + b);
      return 0;
    }
    prev_x = x; prev_f = f;
  }
  return -1;
}

static int make_eos(const eiso_eos* in, eos_t* e) {
  if (!in || !(in->a_v2 > 0) || !(in->a_l > 0) || !(in->rho0 > 0) || !(in->p0 > 0)) return EISO_E_ARG;
  e->a_v2 = in->a_v2;
  e->a_v = sqrt(in->a_v2);
  e->a_l = in->a_l;
  e->a_l2 = in->a_l * in->a_l;
  e->rho0 = in->rho0;
  e->p0 = in->p0;
  /* tau = (2 pi)^-1/2 (m/(k T0))^{3/2}, with kT0/m = a_v^2 (R22) */
  e->tau = in->tau > 0 ? in->tau : (1.0 / sqrt(2.0 * M_PI)) * pow(1.0 / in->a_v2, 1.5);
  e->p_min = in->p_min;
  /* rho_min is the liquid density at p_min (P:1121 corrected, R1) */
  e->rho_min = e->rho0 + (e->p_min - e->p0) / e->a_l2;
  if (!(e->rho_min > 0) || !(e->p_min < e->p0)) return EISO_E_ARG;
  if (in->rho_tilde > 0) e->rho_tilde = in->rho_tilde;
  else if (maxwell_rho_tilde(e, &e->rho_tilde) != 0) return EISO_E_ARG;
  e->p_tilde = e->a_v2 * e->rho_tilde; /* P:1108 at rho_tilde */
  if (!(e->rho_tilde < e->rho_min)) return EISO_E_ARG;
  return EISO_OK;
}

/* phase regions Omega_vap = (0, rho_t], Omega_spin = (rho_t, rho_min), Omega_liq = [rho_min, inf) */
static int phase_of(const eos_t* e, double rho) {
  if (rho <= e->rho_tilde) return VAP;
  if (rho >= e->rho_min) return LIQ;
  return SPIN;
}
/* vapour: ideal gas p = (kT0/m) rho; liquid: linear Tait p = p0 + K0(rho/rho0 - 1)
 * = p0 + a_l^2 (rho - rho0) (P:1121 with the typo corrected, R1). */
static double pressure(const eos_t* e, int ph, double rho) {
  return ph == VAP ? e->a_v2 * rho : e->p0 + e->a_l2 * (rho - e->rho0);
}
static double density(const eos_t* e, int ph, double p) {
  return ph == VAP ? p / e->a_v2 : e->rho0 + (p - e->p0) / e->a_l2;
}
static double sound(const eos_t* e, int ph) { return ph == VAP ? e->a_v : e->a_l; }
/* specific Gibbs energy g = int_{p0}^{p} v dp at fixed T (P:127 g = f + p/rho; normalised so
 * g_V(p0) = g_L(p0) = 0, the Maxwell/saturation condition P:1124-1125). */
static double gibbs(const eos_t* e, int ph, double p) {
  if (ph == VAP) return e->a_v2 * log(p / e->p0);
  return e->a_l2 * log(density(e, LIQ, p) / e->rho0);
}
/* classical outer-wave function f_K, written in the printed pressure form:
 * shock (p* > p_K): sqrt(-[[p]][[v]]);  rarefaction: int_{p_K}^{p*} v/a dzeta, whose exact
 * value for both affine EOS branches is a ln(rho_s/rho_K). */
static double wave_f(const eos_t* e, int ph, double rho_s, double rho_k) {
  double ps = pressure(e, ph, rho_s), pk = pressure(e, ph, rho_k);
  if (ps > pk) {
    double jp = ps - pk, jv = 1.0 / rho_s - 1.0 / rho_k;
    return sqrt(-jp * jv);
  }
  return sound(e, ph) * log(rho_s / rho_k);
}

/* ------------------------------------------------------------------------------------------
 * L1 Riemann solvers
 * ---------------------------------------------------------------------------------------- */
/* HLL flux (Toro) with Davis speed bounds (SPEC S:217 reading):
 * S_L = min(u_L - a, u_R - a), S_R = max(u_L + a, u_R + a);
 * F = F_L if S_L >= 0, F_R if S_R <= 0, else (S_R F_L - S_L F_R + S_L S_R (U_R - U_L))/(S_R - S_L). */
static void hll(const eos_t* e, int ph, double rl, double ml, double rr, double mr, double F[2]) {
  double a = sound(e, ph);
  double ul = ml / rl, ur = mr / rr;
  double FL0 = ml, FL1 = ml * ul + pressure(e, ph, rl);
  double FR0 = mr, FR1 = mr * ur + pressure(e, ph, rr);
  double SL = fmin(ul - a, ur - a), SR = fmax(ul + a, ur + a);
  if (SL >= 0.0) { F[0] = FL0; F[1] = FL1; return; }
  if (SR <= 0.0) { F[0] = FR0; F[1] = FR1; return; }
  F[0] = (SR * FL0 - SL * FR0 + SL * SR * (rr - rl)) / (SR - SL);
  F[1] = (SR * FL1 - SL * FR1 + SL * SR * (mr - ml)) / (SR - SL);
}

/* single-phase Riemann star density: root of Phi(rho*) = f(rho*;rho_L) + f(rho*;rho_R) + du
 * (P:1487 with z = 0, one phase), strictly increasing in rho*; plain bisection on log rho. */
static double single_phase_phi(const eos_t* e, int ph, double rl, double ul, double rr, double ur, double rs) {
  return wave_f(e, ph, rs, rl) + wave_f(e, ph, rs, rr) + (ur - ul);
}
static int single_phase_star(const eos_t* e, int ph, double rl, double ul, double rr, double ur, double* out) {
  double lo = fmin(rl, rr), hi = fmax(rl, rr);
  while (single_phase_phi(e, ph, rl, ul, rr, ur, lo) > 0.0) { lo *= 0.5; if (lo < 1e-300) return -1; }
  while (single_phase_phi(e, ph, rl, ul, rr, ur, hi) < 0.0) { hi *= 2.0; if (hi > 1e300) return -1; }
  for (int it = 0; it < 2000; ++it) {
    double m = sqrt(lo * hi);
    if (!(m > lo && m < hi)) break;
    if (single_phase_phi(e, ph, rl, ul, rr, ur, m) > 0.0) hi = m; else lo = m;
  }
  *out = sqrt(lo * hi);
  return 0;
}
/* Creation trigger (App. B step (i), "p* < p_min", "p* > p_tilde").
 * Because Phi is strictly increasing, p*(liquid) < p_min <=> rho* < rho_min <=> Phi(rho_min) > 0,
 * and p*(vapour) > p_tilde <=> Phi(rho_tilde) < 0 (reading R7; the oracle's bisection root is
 * checked against this in tests/test_oracle_props.py). */
static int creation_trigger(const eos_t* e, int ph, double rl, double ul, double rr, double ur) {
  if (ph == LIQ) return single_phase_phi(e, LIQ, rl, ul, rr, ur, e->rho_min) > 0.0;
  return single_phase_phi(e, VAP, rl, ul, rr, ur, e->rho_tilde) < 0.0;
}

/* Decision margins (the paper's round-off warning P:1133-1135).  A discrete decision
 * "x < threshold" is marginal when |x - threshold| is within MARGIN_ULPS times the rounding-error
 * bound of evaluating x: two correct fp64 implementations may then decide differently.  Counted
 * per member in eiso_stats.decision_margin_warnings; never changes a result. */
#define MARGIN_ULPS 16.0
static int trigger_marginal(const eos_t* e, int ph, double rl, double ul, double rr, double ur) {
  double thr = ph == LIQ ? e->rho_min : e->rho_tilde;
  double fl = wave_f(e, ph, thr, rl), fr = wave_f(e, ph, thr, rr);
  double phi = fl + fr + (ur - ul);
  return fabs(phi) <= MARGIN_ULPS * DBL_EPSILON * (fabs(fl) + fabs(fr) + fabs(ul) + fabs(ur));
}
/* width threshold h < eps h_av (tiny / merge, R4) or h > eps h_av (split) */
static int width_marginal(double h, double thr) {
  return fabs(h - thr) <= MARGIN_ULPS * DBL_EPSILON * thr;
}

/* kinetic relation z = tau p_V [[g + e_kin]] with interface-relative e_kin = z^2 v^2 / 2
 * (reading R2):  A z^2 - z + B = 0, A = tau p_V [[v^2]]/2, B = tau p_V [[g]];
 * the root continuous in A -> 0 is z = 2B / (1 + sqrt(1 - 4AB)). */
static int kinetic_z(const eos_t* e, double pV, double jg, double jv2, double* z) {
  double A = 0.5 * e->tau * pV * jv2, B = e->tau * pV * jg;
  double disc = 1.0 - 4.0 * A * B;
  if (!(disc >= 0.0)) return -1;
  *z = 2.0 * B / (1.0 + sqrt(disc));
  return 0;
}

typedef struct { double rho, u; int ph; } side_t;

/* System (13), in the orientation-general form [[x]] = x_plus - x_minus:
 * G1 = [[p]] + z^2 [[v]],  G2 = f_minus + f_plus + z [[v]] + (u_plus - u_minus),
 * unknowns (p_V*, p_L*); scaled by (p0, a_v) for the stopping test (R14). */
typedef struct { const eos_t* e; side_t m, p; } iface_ctx;
static int iface_G(const void* vc, const double x[2], double G[2]) {
  const iface_ctx* c = (const iface_ctx*)vc;
  const eos_t* e = c->e;
  double pV = x[0], pL = x[1];
  if (!(pV > 0.0)) return -1;
  double rV = density(e, VAP, pV), rL = density(e, LIQ, pL);
  if (!(rL > 0.0)) return -1;
  double gV = gibbs(e, VAP, pV), gL = gibbs(e, LIQ, pL);
  double pm, pp, rm, rp, gm, gp;
  if (c->m.ph == VAP) { pm = pV; rm = rV; gm = gV; pp = pL; rp = rL; gp = gL; }
  else { pm = pL; rm = rL; gm = gL; pp = pV; rp = rV; gp = gV; }
  double vm = 1.0 / rm, vp = 1.0 / rp;
  double jp = pp - pm, jv = vp - vm, jv2 = vp * vp - vm * vm, jg = gp - gm;
  double z;
  if (kinetic_z(e, pV, jg, jv2, &z) != 0) return -1;
  double fm = wave_f(e, c->m.ph, rm, c->m.rho), fp = wave_f(e, c->p.ph, rp, c->p.rho);
  G[0] = (jp + z * z * jv) / e->p0;
  G[1] = (fm + fp + z * jv + (c->p.u - c->m.u)) / e->a_v;
  return 0;
}

typedef int (*resid_fn)(const void*, const double*, double*);

/* Newton-Armijo (Kelley): forward-difference Jacobian, full step then halving
 * lambda up to armijo_max times until ||G(x + lambda d)||_2 <= (1 - 1e-4 lambda) ||G(x)||_2.
 * Stop (R14): |lambda d_j| <= rtol * max(|x_j|, p0) for both unknowns and ||G||_inf <= gtol. */
static int newton_armijo(resid_fn G, const void* ctx, const eos_t* e, const eiso_params* prm,
                         double x[2], int* iters) {
  double Gx[2];
  if (G(ctx, x, Gx) != 0) return -1;
  for (int it = 0; it < prm->newton_max_iter; ++it) {
    double J[2][2];
    for (int j = 0; j < 2; ++j) {
      double xs[2] = {x[0], x[1]}, Gs[2];
      double dx = 1e-7 * fmax(fabs(x[j]), 1.0);
      xs[j] = x[j] + dx;
      if (G(ctx, xs, Gs) != 0) { dx = -dx; xs[j] = x[j] + dx; if (G(ctx, xs, Gs) != 0) return -1; }
      J[0][j] = (Gs[0] - Gx[0]) / dx;
      J[1][j] = (Gs[1] - Gx[1]) / dx;
    }
    double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    if (!(fabs(det) > 0.0) || !isfinite(det)) return -1;
    double d0 = -(J[1][1] * Gx[0] - J[0][1] * Gx[1]) / det;
    double d1 = -(-J[1][0] * Gx[0] + J[0][0] * Gx[1]) / det;
    double n0 = sqrt(Gx[0] * Gx[0] + Gx[1] * Gx[1]);
    double lam = 1.0, xt[2], Gt[2];
    int ok = 0;
    for (int k = 0; k <= prm->armijo_max; ++k) {
      xt[0] = x[0] + lam * d0;
      xt[1] = x[1] + lam * d1;
      if (G(ctx, xt, Gt) == 0 && sqrt(Gt[0] * Gt[0] + Gt[1] * Gt[1]) <= (1.0 - 1e-4 * lam) * n0) { ok = 1; break; }
      lam *= 0.5;
    }
    if (!ok) {
      /* no decrease possible: accept only if already at the rounding floor */
      if (fmax(fabs(Gx[0]), fabs(Gx[1])) <= prm->newton_gtol) { *iters = it; return 0; }
      return -1;
    }
    double s0 = lam * d0, s1 = lam * d1;
    x[0] = xt[0]; x[1] = xt[1]; Gx[0] = Gt[0]; Gx[1] = Gt[1];
    if (fabs(s0) <= prm->newton_rtol * fmax(fabs(x[0]), e->p0) &&
        fabs(s1) <= prm->newton_rtol * fmax(fabs(x[1]), e->p0) &&
        fmax(fabs(Gx[0]), fabs(Gx[1])) <= prm->newton_gtol) { *iters = it + 1; return 0; }
  }
  return -1;
}

/* HLLC estimate used as the Newton start (Eq. (17)), stated for vapour left and
 * liquid right; mirrored (x -> -x, u -> -u) when the liquid is on the left.  The guess p* is
 * clamped to [0.01 p0, 4 p0] for both unknowns (reading R14b: positivity of p_V*). */
static double hllc_guess(const eos_t* e, const side_t* m, const side_t* p) {
  double rV, uV, rL, uL;
  if (m->ph == VAP) { rV = m->rho; uV = m->u; rL = p->rho; uL = p->u; }
  else { rV = p->rho; uV = -p->u; rL = m->rho; uL = -m->u; }
  double pV = pressure(e, VAP, rV), pL = pressure(e, LIQ, rL);
  double SL = uL + e->a_l, SV = uV - e->a_v;
  double w = (pL - pV + rV * uV * (SV - uV) - rL * uL * (SL - uL)) / (rV * (SV - uV) - rL * (SL - uL));
  double rLs = rL * (SL - uL) / (SL - w);
  double ps = pressure(e, LIQ, rLs);
  return fmin(fmax(ps, 0.01 * e->p0), 4.0 * e->p0);
}

/* Two-phase interface solve (Appendix A): Newton-Armijo on (13) from the HLLC start, then
 * recover star densities (EOS), z (kinetic relation), u* (wave relations), w (z = -rho(u-w)),
 * P:1521-1522, and F_PB = (-z, -z u* + p*) with vapour-side values (R17). */
static int interface_solve(const eos_t* e, const eiso_params* prm, side_t m, side_t p, eiso_iface* out) {
  memset(out, 0, sizeof(*out));
  iface_ctx c = {e, m, p};
  double g = hllc_guess(e, &m, &p);
  double x[2] = {g, g};
  int iters = 0;
  if (newton_armijo(iface_G, &c, e, prm, x, &iters) != 0) { out->status = EISO_E_NEWTON; return EISO_E_NEWTON; }
  double pV = x[0], pL = x[1];
  double rV = density(e, VAP, pV), rL = density(e, LIQ, pL);
  double gV = gibbs(e, VAP, pV), gL = gibbs(e, LIQ, pL);
  int vm = (m.ph == VAP);
  double pm = vm ? pV : pL, pp = vm ? pL : pV, rm = vm ? rV : rL, rp = vm ? rL : rV;
  double gm = vm ? gV : gL, gp = vm ? gL : gV;
  double jv2 = 1.0 / (rp * rp) - 1.0 / (rm * rm), z;
  if (kinetic_z(e, pV, gp - gm, jv2, &z) != 0) { out->status = EISO_E_NEWTON; return EISO_E_NEWTON; }
  double um = m.u - wave_f(e, m.ph, rm, m.rho); /* u*_- = u_- - f_-   (left wave) */
  double up = p.u + wave_f(e, p.ph, rp, p.rho); /* u*_+ = u_+ + f_+   (right wave) */
  double uV = vm ? um : up;
  double w = uV + z / rV; /* z = -rho_V (u_V - w) */
  out->p_minus = pm; out->p_plus = pp; out->rho_minus = rm; out->rho_plus = rp;
  out->u_minus = um; out->u_plus = up; out->z = z; out->w = w;
  out->F0 = -z;
  out->F1 = -z * uV + pV;
  out->iters = iters;
  out->status = EISO_OK;
  return EISO_OK;
}

/* Phase creation (App. B; four-wave structure P:249, Fig. 2(b)) reduced to the
 * 2x2 system of reading R18 in (p_A, p_B): A = outer (original) phase star state shared by both
 * sides, B = created middle phase; right boundary (minus = B, plus = A) carries z_r, left one
 * z_l = -z_r.  G1 = p_A - p_B + z_r^2 (v_A - v_B);
 * G2 = (u_r - u_l) + f(rho_A; rho_l) + f(rho_A; rho_r) + 2 z_r (v_A - v_B). */
typedef struct { const eos_t* e; int A, B; double rl, ul, rr, ur; } cre_ctx;
static int creation_G(const void* vc, const double x[2], double G[2]) {
  const cre_ctx* c = (const cre_ctx*)vc;
  const eos_t* e = c->e;
  double pA = x[0], pB = x[1];
  double rA = density(e, c->A, pA), rB = density(e, c->B, pB);
  if (!(rA > 0.0) || !(rB > 0.0)) return -1;
  double pV = (c->B == VAP) ? pB : pA;
  if (!(pV > 0.0)) return -1;
  double vA = 1.0 / rA, vB = 1.0 / rB;
  double jg = gibbs(e, c->A, pA) - gibbs(e, c->B, pB);
  double jv = vA - vB, jv2 = vA * vA - vB * vB, z;
  if (kinetic_z(e, pV, jg, jv2, &z) != 0) return -1;
  G[0] = (pA - pB + z * z * jv) / e->p0;
  G[1] = ((c->ur - c->ul) + wave_f(e, c->A, rA, c->rl) + wave_f(e, c->A, rA, c->rr) + 2.0 * z * jv) / e->a_v;
  return 0;
}
static int creation_solve(const eos_t* e, const eiso_params* prm, int phase_outer, double rl, double ul,
                          double rr, double ur, eiso_creation* out) {
  memset(out, 0, sizeof(*out));
  cre_ctx c = {e, phase_outer, phase_outer == LIQ ? VAP : LIQ, rl, ul, rr, ur};
  double x[2] = {e->p0, e->p0}; /* start at saturation (reading R18b) */
  int iters = 0;
  if (newton_armijo(creation_G, &c, e, prm, x, &iters) != 0) { out->status = EISO_E_CREATION; return EISO_E_CREATION; }
  double pA = x[0], pB = x[1];
  double rA = density(e, c.A, pA), rB = density(e, c.B, pB);
  double vA = 1.0 / rA, vB = 1.0 / rB;
  double pV = (c.B == VAP) ? pB : pA, zr;
  if (kinetic_z(e, pV, gibbs(e, c.A, pA) - gibbs(e, c.B, pB), vA * vA - vB * vB, &zr) != 0) {
    out->status = EISO_E_CREATION; return EISO_E_CREATION;
  }
  double zl = -zr;
  double uAl = ul - wave_f(e, c.A, rA, rl);  /* left outer wave */
  double uB = uAl + zr * (vB - vA);          /* [[u]] + z [[v]] = 0 across the left boundary */
  double wl = uB + zl * vB, wr = uB + zr * vB; /* z = -rho_B (u_B - w) */
  out->p_A = pA; out->p_B = pB; out->rho_A = rA; out->rho_B = rB; out->u_B = uB;
  out->z_l = zl; out->z_r = zr; out->w_l = wl; out->w_r = wr;
  out->Fl0 = -zl; out->Fl1 = -zl * uB + pB;
  out->Fr0 = -zr; out->Fr1 = -zr * uB + pB;
  out->iters = iters;
  if (!(wr > wl)) { out->status = EISO_E_CREATION; return EISO_E_CREATION; }
  out->status = EISO_OK;
  return EISO_OK;
}

/* ------------------------------------------------------------------------------------------
 * point-function exports (pins)
 * ---------------------------------------------------------------------------------------- */
int eiso_thresholds_of(const eiso_eos* eos, eiso_thresholds* out) {
  eos_t e;
  int s = make_eos(eos, &e);
  if (s) return s;
  out->rho_min = e.rho_min; out->rho_tilde = e.rho_tilde; out->p_tilde = e.p_tilde;
  out->tau = e.tau; out->a_v = e.a_v;
  return 0;
}
int eiso_phase(const eiso_eos* eos, double rho) { eos_t e; if (make_eos(eos, &e)) return -1; return phase_of(&e, rho); }
double eiso_pressure(const eiso_eos* eos, int ph, double rho) { eos_t e; make_eos(eos, &e); return pressure(&e, ph, rho); }
double eiso_gibbs(const eiso_eos* eos, int ph, double p) { eos_t e; make_eos(eos, &e); return gibbs(&e, ph, p); }
double eiso_wave_f(const eiso_eos* eos, int ph, double rs, double rk) { eos_t e; make_eos(eos, &e); return wave_f(&e, ph, rs, rk); }
int eiso_hll(const eiso_eos* eos, double rl, double ml, double rr, double mr, double F[2]) {
  eos_t e;
  int s = make_eos(eos, &e);
  if (s) return s;
  int pl = phase_of(&e, rl), pr = phase_of(&e, rr);
  if (pl != pr || pl == SPIN) return EISO_E_ARG;
  hll(&e, pl, rl, ml, rr, mr, F);
  return 0;
}
int eiso_single_phase_star(const eiso_eos* eos, int ph, double rl, double ul, double rr, double ur, double* rs) {
  eos_t e;
  int s = make_eos(eos, &e);
  if (s) return s;
  return single_phase_star(&e, ph, rl, ul, rr, ur, rs) ? EISO_E_NEWTON : 0;
}
int eiso_creation_trigger(const eiso_eos* eos, int ph, double rl, double ul, double rr, double ur) {
  eos_t e;
  if (make_eos(eos, &e)) return -1;
  return creation_trigger(&e, ph, rl, ul, rr, ur);
}
int eiso_interface_solve(const eiso_eos* eos, const eiso_params* prm, double rm, double um, double rp,
                         double up, eiso_iface* out) {
  eos_t e;
  int s = make_eos(eos, &e);
  if (s) return s;
  side_t m = {rm, um, phase_of(&e, rm)}, p = {rp, up, phase_of(&e, rp)};
  if (m.ph == SPIN || p.ph == SPIN || m.ph == p.ph) return EISO_E_ARG;
  return interface_solve(&e, prm, m, p, out);
}
int eiso_creation_solve(const eiso_eos* eos, const eiso_params* prm, int phase_outer, double rl, double ul,
                        double rr, double ur, eiso_creation* out) {
  eos_t e;
  int s = make_eos(eos, &e);
  if (s) return s;
  return creation_solve(&e, prm, phase_outer, rl, ul, rr, ur, out);
}

/* ------------------------------------------------------------------------------------------
 * L2/L3: moving mesh + time stepping (Alg. 1-2; §3.4; App. B)
 * ---------------------------------------------------------------------------------------- */
struct eiso_ctx {
  eos_t e;
  eiso_params prm;
  int64_t M, N, cap;
  double x_left, x_right, h_av;
  double *rho, *mom, *h, *t;
  uint8_t* tiny;
  int64_t* n;
  int32_t* status;
  eiso_stats* mstats;
  int state_set;
  int nthreads;  /* OpenMP threads: over members (M > 1) or over cells / regions (M == 1) */
  struct scratch { void* p; size_t bytes; } * scr;  /* per-thread step work space, reused */
};

/* step work space of n cells, grown on demand (the arrays of one step, carved in order) */
static void* scratch_get(struct scratch* s, size_t bytes) {
  if (s->bytes < bytes) {
    free(s->p);
    s->p = malloc(bytes);
    s->bytes = s->p ? bytes : 0;
  }
  return s->p;
}
static void* carve(char** cur, size_t bytes) {
  void* r = *cur;
  *cur += (bytes + 63) & ~(size_t)63;
  return r;
}

int eiso_create(const eiso_eos* eos, const eiso_params* prm, int64_t M, int64_t N, int64_t cap,
                double xl, double xr, eiso_ctx** out) {
  if (!out || !prm || M < 1 || N < 3 || cap < N || !(xr > xl)) return EISO_E_ARG;
  eiso_ctx* c = (eiso_ctx*)calloc(1, sizeof(eiso_ctx));
  int s = make_eos(eos, &c->e);
  if (s) { free(c); return s; }
  c->prm = *prm;
  c->M = M; c->N = N; c->cap = cap;
  c->x_left = xl; c->x_right = xr;
  c->h_av = (xr - xl) / (double)N; /* h_av = (b - a)/N, fixed (reading R9) */
  c->rho = (double*)calloc(M * cap, sizeof(double));
  c->mom = (double*)calloc(M * cap, sizeof(double));
  c->h = (double*)calloc(M * cap, sizeof(double));
  c->tiny = (uint8_t*)calloc(M * cap, 1);
  c->t = (double*)calloc(M, sizeof(double));
  c->n = (int64_t*)calloc(M, sizeof(int64_t));
  c->status = (int32_t*)calloc(M, sizeof(int32_t));
  c->mstats = (eiso_stats*)calloc(M, sizeof(eiso_stats));
  c->nthreads = 1;
  c->scr = (struct scratch*)calloc(1, sizeof(struct scratch));
  *out = c;
  return 0;
}

int eiso_set_threads(eiso_ctx* c, int nthreads) {
  if (!c || nthreads < 1) return EISO_E_ARG;
  for (int k = 0; k < c->nthreads; ++k) free(c->scr[k].p);
  free(c->scr);
  c->nthreads = nthreads;
  c->scr = (struct scratch*)calloc(nthreads, sizeof(struct scratch));
  return 0;
}

void eiso_destroy(eiso_ctx* c) {
  if (!c) return;
  free(c->rho); free(c->mom); free(c->h); free(c->tiny); free(c->t); free(c->n); free(c->status); free(c->mstats);
  for (int k = 0; k < c->nthreads; ++k) free(c->scr[k].p);
  free(c->scr);
  free(c);
}

/* tiny flag: width below eps_tiny*h_av and no same-phase neighbour to merge with (P:303,
 * P:746, Fig. 4 caption P:389; readings R4, R9) */
static void mark_tiny(eiso_ctx* c, int64_t m, int nth) {
  int64_t n = c->n[m];
  double* rho = c->rho + m * c->cap;
  double* h = c->h + m * c->cap;
  uint8_t* tiny = c->tiny + m * c->cap;
#pragma omp parallel for num_threads(nth) if (nth > 1)
  for (int64_t i = 0; i < n; ++i) {
    int ph = phase_of(&c->e, rho[i]);
    int same_l = i > 0 && phase_of(&c->e, rho[i - 1]) == ph;
    int same_r = i < n - 1 && phase_of(&c->e, rho[i + 1]) == ph;
    tiny[i] = (h[i] < c->prm.eps_tiny * c->h_av) && !same_l && !same_r;
  }
}

int eiso_set_state(eiso_ctx* c, const double* rho, const double* mom, const double* width,
                   const int64_t* n_cells, double t0) {
  if (!c || !rho || !mom) return EISO_E_ARG;
  for (int64_t m = 0; m < c->M; ++m) {
    int64_t n = n_cells ? n_cells[m] : c->N;
    if (n < 3 || n > c->cap) return EISO_E_ARG;
    c->n[m] = n;
    c->t[m] = t0;
    c->status[m] = EISO_OK;
    memset(&c->mstats[m], 0, sizeof(eiso_stats));
    for (int64_t i = 0; i < n; ++i) {
      int64_t k = m * c->cap + i;
      c->rho[k] = rho[k];
      c->mom[k] = mom[k];
      c->h[k] = width ? width[k] : c->h_av;
      if (!(rho[k] > 0)) c->status[m] = EISO_E_NONPOS_DENSITY;
      else if (phase_of(&c->e, rho[k]) == SPIN) c->status[m] = EISO_E_SPINODAL;
    }
    if (c->status[m] == EISO_OK) mark_tiny(c, m, c->nthreads);
  }
  c->state_set = 1;
  return 0;
}

/* per-edge record of step n */
typedef struct {
  double F0, F1, w;  /* flux across the edge (relative to its motion) and edge speed   */
  int kind;          /* 0 bulk (HLL), 1 phase boundary, 2 accepted creation, -1 skipped */
  double Fl0, Fl1, wl, Fr0, Fr1, wr; /* creation: left-cell side / right-cell side     */
  double rhoB, momB, hB;             /* created cell                                  */
} edge_t;

/* flux across an edge between two cells (used for U^n and for DTS iterates) */
static int edge_flux(eiso_ctx* c, double rl, double ml, double rr, double mr, double* F0, double* F1,
                     double* w, int* kind, int64_t* nsolves) {
  int pl = phase_of(&c->e, rl), pr = phase_of(&c->e, rr);
  if (pl == SPIN || pr == SPIN) return EISO_E_SPINODAL;
  if (pl == pr) {
    double F[2];
    hll(&c->e, pl, rl, ml, rr, mr, F);
    *F0 = F[0]; *F1 = F[1]; *w = 0.0; *kind = 0;
    return 0;
  }
  side_t m = {rl, ml / rl, pl}, p = {rr, mr / rr, pr};
  eiso_iface s;
  ++*nsolves;
  if (interface_solve(&c->e, &c->prm, m, p, &s) != 0) return EISO_E_NEWTON;
  *F0 = s.F0; *F1 = s.F1; *w = s.w; *kind = 1;
  return 0;
}

/* Algorithm 2 on an implicit block of cells [a, b] with the moving-cell form of
 * §3.4 and local pseudo steps dtau_i = theta_i dt: theta = alpha =
 * h_i^n / h_av on tiny cells, theta_nb on the others (R12).  The block generalises the
 * triple {k-1, k, k+1} (overlapping triples merged, reading R11).  Outer fluxes F_left =
 * F_{a-1/2}(U^n), F_right = F_{b+1/2}(U^n) are the ones the explicit step used (flux
 * bounding).  Residual (R8): res_i = max_c |(1+dtau/dt)(W^{l+1}
 * - W^l) / (dtau max(|W^l|, 1))|; stop when max res over non-tiny cells < tol_nb and over tiny
 * cells < tol_tiny.  Part 2: fluxes at U* and the conservative update.
 * Parity unpinned beyond invariants (DTS fixed point, conservation): DESIGN.md §3. */
static int dts_block(eiso_ctx* c, int64_t m, int64_t a, int64_t b, const edge_t* E, double dt,
                     double* rho_new, double* mom_new, double* h_new, int64_t* iters_out, int64_t* nsolves,
                     int64_t* margins) {
  int64_t base = m * c->cap;
  const double* rho = c->rho + base;
  const double* mom = c->mom + base;
  const double* h = c->h + base;
  const uint8_t* tiny = c->tiny + base;
  int64_t K = b - a + 1;
  double* W0 = (double*)malloc(sizeof(double) * 12 * (K + 1));
  double *W1 = W0 + (K + 1), *N0 = W1 + (K + 1), *N1 = N0 + (K + 1);
  double *dtau = N1 + (K + 1), *r = dtau + (K + 1), *hl = r + (K + 1);
  double *F0 = hl + (K + 1), *F1 = F0 + (K + 1), *w = F1 + (K + 1); /* edges a .. b+1 -> 0..K */
  int* ph0 = (int*)malloc(sizeof(int) * (K + 1));
  int st = 0;
  for (int64_t i = 0; i < K; ++i) {
    W0[i] = rho[a + i]; W1[i] = mom[a + i];
    ph0[i] = phase_of(&c->e, rho[a + i]);
    double theta = tiny[a + i] ? h[a + i] / c->h_av : c->prm.theta_nb;
    dtau[i] = theta * dt;
    r[i] = dtau[i] / dt;
  }
  F0[0] = E[a].F0; F1[0] = E[a].F1; w[0] = E[a].w;
  F0[K] = E[b + 1].F0; F1[K] = E[b + 1].F1; w[K] = E[b + 1].w;
  int64_t l;
  int done = 0;
  int prev_cont_robust = 1; /* decision margin of the previous iteration's "continue" */
  for (l = 0; l < c->prm.dts_max_iter; ++l) {
    for (int64_t j = 1; j < K; ++j) { /* (a) interior fluxes at W^l */
      int kind;
      st = edge_flux(c, W0[j - 1], W1[j - 1], W0[j], W1[j], &F0[j], &F1[j], &w[j], &kind, nsolves);
      if (st) goto out;
    }
    double res_nb = 0.0, res_t = 0.0;
    int stop_robust = 1, cont_robust = 0;
    for (int64_t i = 0; i < K; ++i) { /* (b) relaxed moving-cell update */
      hl[i] = h[a + i] + (w[i + 1] - w[i]) * dt;
      if (!(hl[i] > 0.0)) { st = EISO_E_WIDTH; goto out; }
      double q = r[i] / (1.0 + r[i]);
      N0[i] = W0[i] / (1.0 + r[i]) + q * ((h[a + i] / hl[i]) * rho[a + i] - (dt / hl[i]) * (F0[i + 1] - F0[i]));
      N1[i] = W1[i] / (1.0 + r[i]) + q * ((h[a + i] / hl[i]) * mom[a + i] - (dt / hl[i]) * (F1[i + 1] - F1[i]));
      double r0 = fabs((1.0 + r[i]) * (N0[i] - W0[i]) / (dtau[i] * fmax(fabs(W0[i]), 1.0)));
      double r1 = fabs((1.0 + r[i]) * (N1[i] - W1[i]) / (dtau[i] * fmax(fabs(W1[i]), 1.0)));
      double ri = fmax(r0, r1);
      if (tiny[a + i]) res_t = fmax(res_t, ri); else res_nb = fmax(res_nb, ri);
      /* margins: res_i against its tolerance, within the rounding-error bound of N - W */
      double tol = tiny[a + i] ? c->prm.tol_tiny : c->prm.tol_nb;
      for (int comp = 0; comp < 2; ++comp) {
        double Wc = comp ? W1[i] : W0[i], Un = comp ? mom[a + i] : rho[a + i];
        double FL = comp ? F1[i] : F0[i], FR = comp ? F1[i + 1] : F0[i + 1], rc = comp ? r1 : r0;
        double err = MARGIN_ULPS * DBL_EPSILON *
                     (fabs(Wc) + q * (fabs((h[a + i] / hl[i]) * Un) + (dt / hl[i]) * (fabs(FL) + fabs(FR)))) *
                     (1.0 + r[i]) / (dtau[i] * fmax(fabs(Wc), 1.0));
        if (!(rc < tol - err)) stop_robust = 0;
        if (rc >= tol + err) cont_robust = 1;
      }
    }
    if (res_nb < c->prm.tol_nb && res_t < c->prm.tol_tiny) {
      if (!stop_robust || !prev_cont_robust) ++*margins;
    }
    prev_cont_robust = cont_robust;
    for (int64_t i = 0; i < K; ++i) {
      W0[i] = N0[i]; W1[i] = N1[i];
      if (!(W0[i] > 0.0) || phase_of(&c->e, W0[i]) != ph0[i]) { st = EISO_E_SPINODAL; goto out; }
    }
    if (res_nb < c->prm.tol_nb && res_t < c->prm.tol_tiny) { done = 1; ++l; break; }
  }
  if (!done) { st = EISO_E_DTS_CAP; goto out; }
  *iters_out = l;
  /* Part 2: fluxes at U* and conservative moving-cell update */
  for (int64_t j = 1; j < K; ++j) {
    int kind;
    st = edge_flux(c, W0[j - 1], W1[j - 1], W0[j], W1[j], &F0[j], &F1[j], &w[j], &kind, nsolves);
    if (st) goto out;
  }
  for (int64_t i = 0; i < K; ++i) {
    double hn = h[a + i] + (w[i + 1] - w[i]) * dt;
    if (!(hn > 0.0)) { st = EISO_E_WIDTH; goto out; }
    h_new[a + i] = hn;
    rho_new[a + i] = (h[a + i] / hn) * rho[a + i] - (dt / hn) * (F0[i + 1] - F0[i]);
    mom_new[a + i] = (h[a + i] / hn) * mom[a + i] - (dt / hn) * (F1[i + 1] - F1[i]);
  }
out:
  free(W0);
  free(ph0);
  return st;
}

/* ---- Newton-like solve of the implicit system (mode NEWTON; readings N1-N5) ----
 * The fixed point of Algorithm 2's Part 1 is the implicit moving-cell system W = T(W),
 * T_i(W) = (h_i^n / h_i(W)) U_i^n - (dt / h_i(W)) (F_{i+1/2}(W) - F_{i-1/2}(W)),
 * h_i(W) = h_i^n + (w_{i+1/2}(W) - w_{i-1/2}(W)) dt, outer fluxes as in dts_block (N1).  It is
 * solved by a chord Newton iteration on R(W) = W - T(W) from W^0 = U^n with a forward-difference
 * Jacobian at W^0, eps_q = 1e-7 max(|W_q|, 1) (N2), dense Gaussian elimination with partial
 * pivoting; stop when the step satisfies max_q |dW_q| / max(|W_q|, 1) <= 1e-10, or when it no
 * longer halves after the second chord step (the rounding floor of the inner Riemann solves,
 * N3); the Jacobian is refreshed at the current iterate every 8 chord steps.  *iters_out counts
 * evaluations of T (1 + 2K for R and the Jacobian, 1 per further chord step, N4).  Part 2 is
 * Algorithm 2's. */
static int newton_T(eiso_ctx* c, int64_t m, int64_t a, int64_t K, const edge_t* E, double dt, const double* X,
                    double* T, double* F0, double* F1, double* w, int64_t* nsolves) {
  int64_t base = m * c->cap;
  const double* rho = c->rho + base;
  const double* mom = c->mom + base;
  const double* h = c->h + base;
  F0[0] = E[a].F0; F1[0] = E[a].F1; w[0] = E[a].w;
  F0[K] = E[a + K].F0; F1[K] = E[a + K].F1; w[K] = E[a + K].w;
  for (int64_t j = 1; j < K; ++j) {
    int kind;
    int st = edge_flux(c, X[2 * (j - 1)], X[2 * (j - 1) + 1], X[2 * j], X[2 * j + 1], &F0[j], &F1[j], &w[j], &kind,
                       nsolves);
    if (st) return st;
  }
  for (int64_t i = 0; i < K; ++i) {
    double hl = h[a + i] + (w[i + 1] - w[i]) * dt;
    if (!(hl > 0.0)) return EISO_E_WIDTH;
    T[2 * i] = (h[a + i] / hl) * rho[a + i] - (dt / hl) * (F0[i + 1] - F0[i]);
    T[2 * i + 1] = (h[a + i] / hl) * mom[a + i] - (dt / hl) * (F1[i + 1] - F1[i]);
  }
  return 0;
}

/* J x = b by Gaussian elimination with partial pivoting (J, b overwritten; x = b on return) */
static int dense_solve(int64_t n, double* J, double* b) {
  for (int64_t p = 0; p < n; ++p) {
    int64_t piv = p;
    for (int64_t i = p + 1; i < n; ++i)
      if (fabs(J[i * n + p]) > fabs(J[piv * n + p])) piv = i;
    if (!(fabs(J[piv * n + p]) > 0.0)) return 1;
    if (piv != p) {
      for (int64_t q = 0; q < n; ++q) { double t = J[p * n + q]; J[p * n + q] = J[piv * n + q]; J[piv * n + q] = t; }
      double t = b[p]; b[p] = b[piv]; b[piv] = t;
    }
    for (int64_t i = p + 1; i < n; ++i) {
      double f = J[i * n + p] / J[p * n + p];
      for (int64_t q = p; q < n; ++q) J[i * n + q] -= f * J[p * n + q];
      b[i] -= f * b[p];
    }
  }
  for (int64_t p = n - 1; p >= 0; --p) {
    double s = b[p];
    for (int64_t q = p + 1; q < n; ++q) s -= J[p * n + q] * b[q];
    b[p] = s / J[p * n + p];
  }
  return 0;
}

static int newton_jacobian(eiso_ctx* c, int64_t m, int64_t a, int64_t K, const edge_t* E, double dt, const double* X,
                           const double* T, double* J, double* Xp, double* Tp, double* F0, double* F1, double* w,
                           int64_t* nsolves) {
  int64_t n = 2 * K;
  for (int64_t q = 0; q < n; ++q) {
    memcpy(Xp, X, sizeof(double) * n);
    double eps = 1e-7 * fmax(fabs(X[q]), 1.0);
    Xp[q] += eps;
    int st = newton_T(c, m, a, K, E, dt, Xp, Tp, F0, F1, w, nsolves);
    if (st) return st;
    for (int64_t i = 0; i < n; ++i) J[i * n + q] = (i == q ? 1.0 : 0.0) - (Tp[i] - T[i]) / eps;
  }
  return 0;
}

static int newton_block(eiso_ctx* c, int64_t m, int64_t a, int64_t b, const edge_t* E, double dt,
                        double* rho_new, double* mom_new, double* h_new, int64_t* iters_out, int64_t* nsolves) {
  int64_t base = m * c->cap;
  const double* rho = c->rho + base;
  const double* mom = c->mom + base;
  const double* h = c->h + base;
  int64_t K = b - a + 1, n = 2 * K;
  double* X = (double*)malloc(sizeof(double) * (5 * n + 3 * (K + 1) + n * n * 2));
  double *T = X + n, *R = T + n, *Xp = R + n, *Tp = Xp + n;
  double *F0 = Tp + n, *F1 = F0 + (K + 1), *w = F1 + (K + 1);
  double *J = w + (K + 1), *LU = J + n * n;
  int* ph0 = (int*)malloc(sizeof(int) * K);
  int st = 0;
  int64_t evals = 0;
  for (int64_t i = 0; i < K; ++i) {
    X[2 * i] = rho[a + i]; X[2 * i + 1] = mom[a + i];
    ph0[i] = phase_of(&c->e, rho[a + i]);
  }
  st = newton_T(c, m, a, K, E, dt, X, T, F0, F1, w, nsolves);
  ++evals;
  if (st) goto out;
  st = newton_jacobian(c, m, a, K, E, dt, X, T, J, Xp, Tp, F0, F1, w, nsolves);
  evals += n;
  if (st) goto out;
  double prev = INFINITY;
  for (int64_t it = 1;; ++it) {
    if (it > c->prm.dts_max_iter) { st = EISO_E_DTS_CAP; goto out; }
    for (int64_t i = 0; i < n; ++i) R[i] = -(X[i] - T[i]);
    memcpy(LU, J, sizeof(double) * n * n);
    if (dense_solve(n, LU, R)) { st = EISO_E_NEWTON; goto out; }
    double step = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      X[i] += R[i];
      step = fmax(step, fabs(R[i]) / fmax(fabs(X[i]), 1.0));
    }
    for (int64_t i = 0; i < K; ++i)
      if (!(X[2 * i] > 0.0) || phase_of(&c->e, X[2 * i]) != ph0[i]) { st = EISO_E_SPINODAL; goto out; }
    if (step <= 1e-10 || (it >= 2 && step >= 0.5 * prev)) break;  /* N3 */
    prev = step;
    st = newton_T(c, m, a, K, E, dt, X, T, F0, F1, w, nsolves);
    ++evals;
    if (st) goto out;
    if (it % 8 == 0) {  /* refresh the chord Jacobian at the current iterate */
      st = newton_jacobian(c, m, a, K, E, dt, X, T, J, Xp, Tp, F0, F1, w, nsolves);
      evals += n;
      if (st) goto out;
    }
  }
  *iters_out = evals;
  /* Part 2: fluxes at U* and the conservative moving-cell update */
  st = newton_T(c, m, a, K, E, dt, X, T, F0, F1, w, nsolves);
  if (st) goto out;
  for (int64_t i = 0; i < K; ++i) {
    double hn = h[a + i] + (w[i + 1] - w[i]) * dt;
    if (!(hn > 0.0)) { st = EISO_E_WIDTH; goto out; }
    h_new[a + i] = hn;
    rho_new[a + i] = (h[a + i] / hn) * rho[a + i] - (dt / hn) * (F0[i + 1] - F0[i]);
    mom_new[a + i] = (h[a + i] / hn) * mom[a + i] - (dt / hn) * (F1[i + 1] - F1[i]);
  }
out:
  free(X);
  free(ph0);
  return st;
}

/* Explicit time-accurate local time stepping (LTS) on an implicit block [a, b]: the paper's
 * comparison method, the reduced Mueller-Stiriba scheme of the disabled passage
 * P:1068-1091, readings R29-R31.  The tiny cells of the block advance with 2^n0 sub-steps of
 * dtau = dt / 2^n0, n0 the smallest integer with dtau <= C_CFL h_T / S_max (h_T the smallest
 * tiny width at t^n, S_max the step's, R29; P:1077 footnote); the other block cells stay at U^n
 * meanwhile.  Each sub-step nu: fluxes F^nu and boundary speeds w^nu at the block's
 * interior edges next to a tiny cell from the current states, then the moving small-cell update
 * (P:1079-1081): h^{nu+1} = h^nu + (w_R - w_L) dtau, W^{nu+1} = (h^nu/h^{nu+1}) W^nu -
 * (dtau/h^{nu+1})(F_R - F_L).  The non-tiny block cells then take the large step with the time
 * averages Fbar = sum_nu (dtau/dt) F^nu and wbar = sum_nu (dtau/dt) w^nu at the edges they share
 * with tiny cells (R30) and the U^n fluxes elsewhere, which balances mass, momentum
 * and width exactly.  *iters_out = number of sub-steps ("local iterations"). */
static int lts_block(eiso_ctx* c, int64_t m, int64_t a, int64_t b, const edge_t* E, double dt, double Smax,
                     double* rho_new, double* mom_new, double* h_new, int64_t* iters_out, int64_t* nsolves) {
  int64_t base = m * c->cap;
  const double* rho = c->rho + base;
  const double* mom = c->mom + base;
  const double* h = c->h + base;
  const uint8_t* tiny = c->tiny + base;
  int64_t K = b - a + 1;
  double* W0 = (double*)malloc(sizeof(double) * 10 * (K + 1));
  double *W1 = W0 + (K + 1), *hw = W1 + (K + 1);
  double *F0 = hw + (K + 1), *F1 = F0 + (K + 1), *w = F1 + (K + 1);     /* edges a .. b+1 -> 0..K */
  double *Fb0 = w + (K + 1), *Fb1 = Fb0 + (K + 1), *wb = Fb1 + (K + 1);
  int* sub = (int*)malloc(sizeof(int) * (K + 1)); /* edge j next to a tiny cell */
  int* ph0 = (int*)malloc(sizeof(int) * (K + 1));
  int st = 0;
  double hT = INFINITY;
  for (int64_t i = 0; i < K; ++i) {
    W0[i] = rho[a + i]; W1[i] = mom[a + i]; hw[i] = h[a + i];
    ph0[i] = phase_of(&c->e, rho[a + i]);
    if (tiny[a + i] && h[a + i] < hT) hT = h[a + i];
  }
  /* R29: dtau = dt / 2^n0 <= C_CFL h_T / S_max */
  double dtau = dt;
  int n0 = 0;
  while (dtau > c->prm.cfl * hT / Smax) { dtau *= 0.5; if (++n0 > 62) { st = EISO_E_DTS_CAP; goto out; } }
  const int64_t ns = (int64_t)1 << n0;
  const double f = dtau / dt; /* 2^-n0, exact */
  /* outer edges: the explicit step's U^n fluxes (flux bounding); interior edges not next
   * to a tiny cell: U^n fluxes, constant during the sub-steps */
  F0[0] = E[a].F0; F1[0] = E[a].F1; w[0] = E[a].w;
  F0[K] = E[b + 1].F0; F1[K] = E[b + 1].F1; w[K] = E[b + 1].w;
  sub[0] = sub[K] = 0;
  for (int64_t j = 1; j < K; ++j) {
    sub[j] = tiny[a + j - 1] || tiny[a + j];
    Fb0[j] = Fb1[j] = wb[j] = 0.0;
    if (!sub[j]) {
      int kind;
      st = edge_flux(c, rho[a + j - 1], mom[a + j - 1], rho[a + j], mom[a + j], &F0[j], &F1[j], &w[j], &kind, nsolves);
      if (st) goto out;
    }
  }
  for (int64_t nu = 0; nu < ns; ++nu) {
    for (int64_t j = 1; j < K; ++j) { /* fluxes at the current sub-step states */
      if (!sub[j]) continue;
      int kind;
      st = edge_flux(c, W0[j - 1], W1[j - 1], W0[j], W1[j], &F0[j], &F1[j], &w[j], &kind, nsolves);
      if (st) goto out;
    }
    for (int64_t i = 0; i < K; ++i) { /* small-cell updates */
      if (!tiny[a + i]) continue;
      double hn = hw[i] + (w[i + 1] - w[i]) * dtau;
      if (!(hn > 0.0)) { st = EISO_E_WIDTH; goto out; }
      W0[i] = (hw[i] / hn) * W0[i] - (dtau / hn) * (F0[i + 1] - F0[i]);
      W1[i] = (hw[i] / hn) * W1[i] - (dtau / hn) * (F1[i + 1] - F1[i]);
      hw[i] = hn;
      if (!(W0[i] > 0.0) || phase_of(&c->e, W0[i]) != ph0[i]) { st = EISO_E_SPINODAL; goto out; }
    }
    for (int64_t j = 1; j < K; ++j) { /* time averages for the large cells (R30) */
      if (!sub[j]) continue;
      Fb0[j] += f * F0[j]; Fb1[j] += f * F1[j]; wb[j] += f * w[j];
    }
  }
  for (int64_t i = 0; i < K; ++i) {
    if (tiny[a + i]) { rho_new[a + i] = W0[i]; mom_new[a + i] = W1[i]; h_new[a + i] = hw[i]; continue; }
    const double FL0 = sub[i] ? Fb0[i] : F0[i], FL1 = sub[i] ? Fb1[i] : F1[i], wL = sub[i] ? wb[i] : w[i];
    const double FR0 = sub[i + 1] ? Fb0[i + 1] : F0[i + 1], FR1 = sub[i + 1] ? Fb1[i + 1] : F1[i + 1];
    const double wR = sub[i + 1] ? wb[i + 1] : w[i + 1];
    double hn = h[a + i] + (wR - wL) * dt;
    if (!(hn > 0.0)) { st = EISO_E_WIDTH; goto out; }
    h_new[a + i] = hn;
    rho_new[a + i] = (h[a + i] / hn) * rho[a + i] - (dt / hn) * (FR0 - FL0);
    mom_new[a + i] = (h[a + i] / hn) * mom[a + i] - (dt / hn) * (FR1 - FL1);
  }
  *iters_out = ns;
out:
  free(W0);
  free(sub);
  free(ph0);
  return st;
}

/* One large time step of one member: Algorithm 1 extended by the moving mesh
 * (§2.3, §3.4) and phase creation (App. B).  Order of sub-steps: DESIGN.md
 * §2. */
/* One large step of member m (Algorithm 1 with the moving mesh, App. B creation, Algorithm 2).
 * nth > 1 spreads the per-cell, per-edge and per-region loops over OpenMP threads: every cell,
 * edge and region is computed exactly as with one thread (no value depends on another thread's
 * work; S_max / h_min are exact max / min; counters are integer sums), the creation acceptance
 * (leftmost wins) and the remesh stay serial, and a failure reports the status of the first
 * failing cell / edge / region in index order -- so results are bitwise those of nth = 1. */
static int step_member(eiso_ctx* c, int64_t m, double t_end, int nth, struct scratch* scr) {
  const eos_t* e = &c->e;
  const eiso_params* P = &c->prm;
  int64_t n = c->n[m], base = m * c->cap;
  double* rho = c->rho + base;
  double* mom = c->mom + base;
  double* h = c->h + base;
  uint8_t* tiny = c->tiny + base;
  eiso_stats* S = &c->mstats[m];
  int st = 0;
  /* work arrays of the step (remesh buffers: each old cell emits at most 1 created + 2 split
   * halves), carved from the calling thread's reused work space */
  const size_t nr = 3 * (size_t)n + 2;
  char* cur = (char*)scratch_get(scr, 64 * 12 + sizeof(int) * n + n + sizeof(edge_t) * (n + 1) + 3 * sizeof(double) * n +
                                           3 * sizeof(double) * nr + sizeof(int) * nr + sizeof(int64_t) * (nr + 1));
  if (!cur) return EISO_E_CAPACITY;
  int* ph = (int*)carve(&cur, sizeof(int) * n);
  uint8_t* inreg = (uint8_t*)carve(&cur, n);
  edge_t* E = (edge_t*)carve(&cur, sizeof(edge_t) * (n + 1));
  double* rho_new = (double*)carve(&cur, sizeof(double) * n);
  double* mom_new = (double*)carve(&cur, sizeof(double) * n);
  double* h_new = (double*)carve(&cur, sizeof(double) * n);
  double* R0 = (double*)carve(&cur, sizeof(double) * nr);
  double* R1 = (double*)carve(&cur, sizeof(double) * nr);
  double* RH = (double*)carve(&cur, sizeof(double) * nr);
  int* RP = (int*)carve(&cur, sizeof(int) * nr);
  int64_t* partner = (int64_t*)carve(&cur, sizeof(int64_t) * (nr + 1));
  int64_t* blk = NULL; /* implicit blocks [blk[2k], blk[2k+1]] */
  int* bst = NULL;
  int64_t nb = 0, first = INT64_MAX;

  /* 1. phases and the CFL time step (readings R5, R6):
   *    S = max over all cells of |u| + a; h_min over non-tiny cells (all cells when EXPLICIT). */
  double Smax = 0.0, hmin = INFINITY;
#pragma omp parallel for num_threads(nth) if (nth > 1) reduction(max : Smax) reduction(min : hmin, first)
  for (int64_t i = 0; i < n; ++i) {
    ph[i] = phase_of(e, rho[i]);
    if (!(rho[i] > 0.0) || ph[i] == SPIN) { if (i < first) first = i; continue; }
    double s = fabs(mom[i] / rho[i]) + sound(e, ph[i]);
    if (s > Smax) Smax = s;
    if ((P->mode == EISO_MODE_EXPLICIT || !tiny[i]) && h[i] < hmin) hmin = h[i];
  }
  if (first < n) { st = !(rho[first] > 0.0) ? EISO_E_NONPOS_DENSITY : EISO_E_SPINODAL; goto out; }
  double dt = P->cfl * hmin / Smax;
  if (c->t[m] + dt > t_end) dt = t_end - c->t[m]; /* last step clipped (run_to) */

  /* 2. implicit regions {k-1, k, k+1} around tiny cells, overlapping ones merged
   *    (SPLIT: dual time stepping; LTS: local time stepping of the tiny cells) */
  const int split = P->mode != EISO_MODE_EXPLICIT;
  if (split && (tiny[0] || tiny[n - 1])) { st = EISO_E_UNSUPPORTED; goto out; }
#pragma omp parallel for num_threads(nth) if (nth > 1)
  for (int64_t i = 0; i < n; ++i) inreg[i] = split && (tiny[i] || (i > 0 && tiny[i - 1]) || (i < n - 1 && tiny[i + 1]));

  /* 3. edge fluxes from U^n (Alg. 1 Step 1(a)); edge e lies between cells e-1 and e; the domain
   *    ends use a transmissive ghost = copy of the end cell (reading R15).  Edges interior to an
   *    implicit block are left to Algorithm 2. */
  {
    int64_t solves = 0;
    first = INT64_MAX;
#pragma omp parallel for num_threads(nth) if (nth > 1) reduction(+ : solves) reduction(min : first)
    for (int64_t ed = 0; ed <= n; ++ed) {
      int64_t L = ed == 0 ? 0 : ed - 1, R = ed == n ? n - 1 : ed;
      if (ed > 0 && ed < n && inreg[L] && inreg[R]) { E[ed].kind = -1; continue; }
      if (edge_flux(c, rho[L], mom[L], rho[R], mom[R], &E[ed].F0, &E[ed].F1, &E[ed].w, &E[ed].kind, &solves) &&
          ed < first)
        first = ed;
    }
    S->iface_solves += solves;
    if (first != INT64_MAX) { /* the first failing edge's status */
      int64_t ed = first, L = ed == 0 ? 0 : ed - 1, R = ed == n ? n - 1 : ed, dummy = 0;
      st = edge_flux(c, rho[L], mom[L], rho[R], mom[R], &E[ed].F0, &E[ed].F1, &E[ed].w, &E[ed].kind, &dummy);
      goto out;
    }
  }

  /* 4. phase creation (App. B steps (i)-(v)) on eligible edges (reading R16): interior,
   *    same phase, both cells explicit; increasing edge order, an edge whose left neighbour
   *    edge was accepted is skipped (leftmost wins).  The trigger tests are independent per edge
   *    (kind 3 marks a triggered edge), the acceptance runs in edge order, the solves again per
   *    edge. */
  {
    int64_t marg = 0, ncre = 0;
#pragma omp parallel for num_threads(nth) if (nth > 1) reduction(+ : marg)
    for (int64_t ed = 1; ed < n; ++ed) {
      if (E[ed].kind != 0 || inreg[ed - 1] || inreg[ed]) continue;
      int phe = ph[ed];
      double ul = mom[ed - 1] / rho[ed - 1], ur = mom[ed] / rho[ed];
      if (trigger_marginal(e, phe, rho[ed - 1], ul, rho[ed], ur)) marg++;
      if (creation_trigger(e, phe, rho[ed - 1], ul, rho[ed], ur)) E[ed].kind = 3;
    }
    S->decision_margin_warnings += marg;
    for (int64_t ed = 1; ed < n; ++ed)
      if (E[ed].kind == 3) E[ed].kind = E[ed - 1].kind == 2 ? 0 : 2;
    first = INT64_MAX;
#pragma omp parallel for num_threads(nth) if (nth > 1) reduction(+ : ncre) reduction(min : first)
    for (int64_t ed = 1; ed < n; ++ed) {
      if (E[ed].kind != 2) continue;
      double ul = mom[ed - 1] / rho[ed - 1], ur = mom[ed] / rho[ed];
      eiso_creation cr;
      if (creation_solve(e, P, ph[ed], rho[ed - 1], ul, rho[ed], ur, &cr) != 0) { if (ed < first) first = ed; continue; }
      E[ed].Fl0 = cr.Fl0; E[ed].Fl1 = cr.Fl1; E[ed].wl = cr.w_l;
      E[ed].Fr0 = cr.Fr0; E[ed].Fr1 = cr.Fr1; E[ed].wr = cr.w_r;
      E[ed].rhoB = cr.rho_B;
      E[ed].momB = cr.rho_B * cr.u_B;
      E[ed].hB = (cr.w_r - cr.w_l) * dt; /* created width (w_right - w_left) dt, P:1581 / P:1608 */
      ncre++;
    }
    S->creations += ncre;
    if (first != INT64_MAX) { st = EISO_E_CREATION; goto out; }
  }

  /* 5. explicit moving-cell update of every cell outside the implicit blocks (Alg. 1 Step 1(b)
   *    in the form (12)): h^{n+1} = h^n + (w_R - w_L) dt,
   *    U^{n+1} = (h^n/h^{n+1}) U^n - (dt/h^{n+1}) (F_R - F_L). */
  first = INT64_MAX;
#pragma omp parallel for num_threads(nth) if (nth > 1) reduction(min : first)
  for (int64_t i = 0; i < n; ++i) {
    if (inreg[i]) continue;
    const edge_t* El = &E[i];
    const edge_t* Er = &E[i + 1];
    double FL0 = El->kind == 2 ? El->Fr0 : El->F0, FL1 = El->kind == 2 ? El->Fr1 : El->F1;
    double wL = El->kind == 2 ? El->wr : El->w;
    double FR0 = Er->kind == 2 ? Er->Fl0 : Er->F0, FR1 = Er->kind == 2 ? Er->Fl1 : Er->F1;
    double wR = Er->kind == 2 ? Er->wl : Er->w;
    double hn = h[i] + (wR - wL) * dt;
    if (!(hn > 0.0)) { if (i < first) first = i; continue; }
    h_new[i] = hn;
    rho_new[i] = (h[i] / hn) * rho[i] - (dt / hn) * (FR0 - FL0);
    mom_new[i] = (h[i] / hn) * mom[i] - (dt / hn) * (FR1 - FL1);
  }
  if (first != INT64_MAX) { st = EISO_E_WIDTH; goto out; }

  /* 6. Algorithm 2 on every implicit block (Alg. 1 Step 2), or local time stepping (LTS mode):
   *    the blocks are listed in cell order, solved independently, the first failure reported */
  for (int64_t i = 0; i < n;) {
    if (!inreg[i]) { ++i; continue; }
    int64_t a = i;
    while (i < n && inreg[i]) ++i;
    if (nb % 64 == 0) blk = (int64_t*)realloc(blk, sizeof(int64_t) * 2 * (nb + 64));
    blk[2 * nb] = a; blk[2 * nb + 1] = i - 1; ++nb;
  }
  if (nb) {
    bst = (int*)calloc(nb, sizeof(int));
    int64_t iters = 0, solves = 0, marg = 0;
#pragma omp parallel for num_threads(nth) if (nth > 1) schedule(dynamic, 1) reduction(+ : iters, solves, marg)
    for (int64_t k = 0; k < nb; ++k) {
      int64_t a = blk[2 * k], b = blk[2 * k + 1], it = 0;
      if (P->mode == EISO_MODE_LTS)
        bst[k] = lts_block(c, m, a, b, E, dt, Smax, rho_new, mom_new, h_new, &it, &solves);
      else if (P->mode == EISO_MODE_NEWTON)
        bst[k] = newton_block(c, m, a, b, E, dt, rho_new, mom_new, h_new, &it, &solves);
      else
        bst[k] = dts_block(c, m, a, b, E, dt, rho_new, mom_new, h_new, &it, &solves, &marg);
      iters += it;
    }
    S->iface_solves += solves;
    S->decision_margin_warnings += marg;
    for (int64_t k = 0; k < nb; ++k) {
      if (bst[k]) { st = bst[k]; goto out; }
      S->regions++;
    }
    S->dts_iters += iters;
  }

  /* 7. remesh (readings R9, R10): insert created cells -> merge cells with
   *    h < eps_tiny*h_av into their same-phase neighbour (union of merge pairs, conservative
   *    h-weighted average) -> split h > eps_split*h_av into two equal halves -> tiny flags. */
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (i > 0 && E[i].kind == 2) { R0[q] = E[i].rhoB; R1[q] = E[i].momB; RH[q] = E[i].hB; ++q; }
    R0[q] = rho_new[i]; R1[q] = mom_new[i]; RH[q] = h_new[i]; ++q;
  }
  int64_t wmarg = 0;
  first = INT64_MAX;
#pragma omp parallel for num_threads(nth) if (nth > 1) reduction(+ : wmarg)
  for (int64_t i = 0; i < n; ++i) /* width decisions of the cells whose width changed (R4) */
    if (h_new[i] != h[i] && (width_marginal(h_new[i], P->eps_tiny * c->h_av) ||
                             width_marginal(h_new[i], P->eps_split * c->h_av)))
      wmarg++;
  S->decision_margin_warnings += wmarg;
#pragma omp parallel for num_threads(nth) if (nth > 1) reduction(min : first)
  for (int64_t i = 0; i < q; ++i) {
    RP[i] = phase_of(e, R0[i]);
    if ((!(R0[i] > 0.0) || RP[i] == SPIN) && i < first) first = i;
  }
  if (first != INT64_MAX) { st = !(R0[first] > 0.0) ? EISO_E_NONPOS_DENSITY : EISO_E_SPINODAL; goto out; }
  /* merge partner: the same-phase neighbour; both -> the smaller, ties to the left */
#pragma omp parallel for num_threads(nth) if (nth > 1)
  for (int64_t i = 0; i < q; ++i) {
    partner[i] = -1;
    if (!(RH[i] < P->eps_tiny * c->h_av)) continue;
    int sl = i > 0 && RP[i - 1] == RP[i], sr = i < q - 1 && RP[i + 1] == RP[i];
    if (sl && sr) partner[i] = (RH[i + 1] < RH[i - 1]) ? i + 1 : i - 1;
    else if (sl) partner[i] = i - 1;
    else if (sr) partner[i] = i + 1;
  }
  int64_t q2 = 0;
  for (int64_t i = 0; i < q;) {
    int64_t j = i; /* group [i, j]: consecutive cells joined by merge pairs */
    while (j + 1 < q && (partner[j] == j + 1 || partner[j + 1] == j)) ++j;
    if (j == i) { R0[q2] = R0[i]; R1[q2] = R1[i]; RH[q2] = RH[i]; RP[q2] = RP[i]; }
    else {
      double hs = 0.0, s0 = 0.0, s1 = 0.0;
      for (int64_t k = i; k <= j; ++k) { hs += RH[k]; s0 += RH[k] * R0[k]; s1 += RH[k] * R1[k]; }
      double h_sum = hs;
      R0[q2] = s0 / h_sum; R1[q2] = s1 / h_sum; RH[q2] = h_sum; RP[q2] = RP[i];
      S->merges += j - i;
    }
    ++q2;
    i = j + 1;
  }
  int64_t q3 = 0;
  for (int64_t i = 0; i < q2; ++i) q3 += (RH[i] > P->eps_split * c->h_av) ? 2 : 1;
  if (q3 > c->cap) { st = EISO_E_CAPACITY; goto out; }
  for (int64_t i = q2 - 1, o = q3 - 1; i >= 0; --i) { /* split, writing from the back */
    if (RH[i] > P->eps_split * c->h_av) {
      double hh = 0.5 * RH[i];
      rho[o] = R0[i]; mom[o] = R1[i]; h[o] = hh; --o;
      rho[o] = R0[i]; mom[o] = R1[i]; h[o] = hh; --o;
      S->splits++;
    } else { rho[o] = R0[i]; mom[o] = R1[i]; h[o] = RH[i]; --o; }
  }
  S->cell_updates += n;
  c->n[m] = q3;
  mark_tiny(c, m, nth);
  c->t[m] += dt;
  S->steps++;
  if (S->steps == 1 || dt < S->dt_min) S->dt_min = dt;
  if (dt > S->dt_max) S->dt_max = dt;
out:
  free(blk); free(bst);
  return st;
}

static int thread_slot(void) {
#ifdef _OPENMP
  return omp_get_thread_num();
#else
  return 0;
#endif
}

static void accumulate(const eiso_ctx* c, eiso_stats* out) {
  memset(out, 0, sizeof(*out));
  out->t_min = INFINITY; out->t_max = -INFINITY; out->dt_min = INFINITY;
  for (int64_t m = 0; m < c->M; ++m) {
    const eiso_stats* s = &c->mstats[m];
    out->steps += s->steps; out->cell_updates += s->cell_updates; out->dts_iters += s->dts_iters;
    out->iface_solves += s->iface_solves; out->creations += s->creations; out->splits += s->splits;
    out->merges += s->merges; out->regions += s->regions;
    out->decision_margin_warnings += s->decision_margin_warnings;
    if (c->t[m] < out->t_min) out->t_min = c->t[m];
    if (c->t[m] > out->t_max) out->t_max = c->t[m];
    if (s->steps && s->dt_min < out->dt_min) out->dt_min = s->dt_min;
    if (s->dt_max > out->dt_max) out->dt_max = s->dt_max;
  }
}

int eiso_step(eiso_ctx* c, int64_t n_steps, eiso_stats* out) {
  if (!c) return EISO_E_ARG;
  if (!c->state_set) return EISO_E_ORDER;
  /* members in parallel (each member's steps in order), or one member's loops in parallel */
  const int nth = c->nthreads, inner = c->M > 1 ? 1 : nth;
#pragma omp parallel for num_threads(nth) if (nth > 1 && c->M > 1) schedule(dynamic, 1)
  for (int64_t m = 0; m < c->M; ++m)
    for (int64_t k = 0; k < n_steps && c->status[m] == EISO_OK; ++k)
      c->status[m] = step_member(c, m, INFINITY, inner, &c->scr[thread_slot()]);
  if (out) accumulate(c, out);
  return 0;
}

int eiso_run_to(eiso_ctx* c, double t_end, int64_t max_steps, eiso_stats* out) {
  if (!c) return EISO_E_ARG;
  if (!c->state_set) return EISO_E_ORDER;
  const int nth = c->nthreads, inner = c->M > 1 ? 1 : nth;
#pragma omp parallel for num_threads(nth) if (nth > 1 && c->M > 1) schedule(dynamic, 1)
  for (int64_t m = 0; m < c->M; ++m)
    for (int64_t k = 0; k < max_steps && c->status[m] == EISO_OK && c->t[m] < t_end; ++k)
      c->status[m] = step_member(c, m, t_end, inner, &c->scr[thread_slot()]);
  if (out) accumulate(c, out);
  return 0;
}

int eiso_get_state(const eiso_ctx* c, double* rho, double* mom, double* width, uint8_t* phase,
                   int64_t* n_cells, double* t) {
  if (!c) return EISO_E_ARG;
  for (int64_t m = 0; m < c->M; ++m) {
    int64_t n = c->n[m];
    for (int64_t i = 0; i < c->cap; ++i) {
      int64_t k = m * c->cap + i;
      int live = i < n;
      if (rho) rho[k] = live ? c->rho[k] : 0.0;
      if (mom) mom[k] = live ? c->mom[k] : 0.0;
      if (width) width[k] = live ? c->h[k] : 0.0;
      if (phase) phase[k] = live ? (uint8_t)phase_of(&c->e, c->rho[k]) : 255;
    }
    if (n_cells) n_cells[m] = n;
    if (t) t[m] = c->t[m];
  }
  return 0;
}

/* interface positions: x_left + widths summed left to right (plain order, no FMA) */
int eiso_interfaces(const eiso_ctx* c, eiso_interface* out, int64_t capacity, int64_t* count) {
  int64_t k = 0;
  for (int64_t m = 0; m < c->M; ++m) {
    int64_t n = c->n[m];
    const double* rho = c->rho + m * c->cap;
    const double* h = c->h + m * c->cap;
    double x = c->x_left;
    for (int64_t i = 0; i < n; ++i) {
      x = x + h[i];
      if (i + 1 < n) {
        int a = phase_of(&c->e, rho[i]), b = phase_of(&c->e, rho[i + 1]);
        if (a != b) {
          if (k < capacity && out) {
            out[k].member = m; out[k].edge = i + 1; out[k].x = x; out[k].left_phase = a; out[k].right_phase = b;
            /* the phase-boundary Riemann problem of the two adjacent cells (App. A) */
            const double* mom = c->mom + m * c->cap;
            side_t sm = {rho[i], mom[i] / rho[i], a}, sp = {rho[i + 1], mom[i + 1] / rho[i + 1], b};
            eiso_iface s;
            out[k].solve_status = 0; out[k].reserved = 0;
            out[k].w = out[k].z = out[k].p_vap = out[k].p_liq = 0.0;
            if (a == SPIN || b == SPIN || interface_solve(&c->e, &c->prm, sm, sp, &s) != 0) {
              out[k].solve_status = EISO_E_NEWTON;
            } else {
              out[k].w = s.w; out[k].z = s.z;
              out[k].p_vap = a == VAP ? s.p_minus : s.p_plus;
              out[k].p_liq = a == VAP ? s.p_plus : s.p_minus;
            }
          }
          ++k;
        }
      }
    }
  }
  *count = k;
  return k > capacity ? EISO_E_CAPACITY : 0;
}

int eiso_member_status(const eiso_ctx* c, int32_t* out) {
  for (int64_t m = 0; m < c->M; ++m) out[m] = c->status[m];
  return 0;
}

int eiso_member_stats(const eiso_ctx* c, int64_t m, eiso_stats* out) {
  if (m < 0 || m >= c->M) return EISO_E_ARG;
  *out = c->mstats[m];
  out->t_min = out->t_max = c->t[m];
  return 0;
}
