// eis_device.cuh — device-side thermodynamics and Riemann solvers (sm_100a, fp64).
//
// "P:n" = line n of /root/reference/PAPER.md; "R<k>" = DESIGN.md §3 reading.  Written
// independently of oracle/ (which uses FD Jacobians, sequential Armijo and the pressure form
// of the wave functions); this file uses the analytic Jacobian of Eq. (14),
// half-warp lane-parallel Armijo candidates and the density form of the wave functions (R19).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace eis {

enum : int { VAP = 0, LIQ = 1, SPIN = 2 };

// status codes (values of eis_status)
enum : int {
  ST_OK = 0, ST_NONPOS = 3, ST_SPINODAL = 4, ST_NEWTON = 5, ST_CREATION = 6, ST_DTS_CAP = 7,
  ST_WIDTH = 8, ST_CAPACITY = 9, ST_UNSUPPORTED = 12, ST_INTERNAL = 13
};

// Derived, immutable EOS constants (thresholds per R3).
struct Eos {
  double a_v2, a_v, a_l, a_l2, rho0, p0, tau, rho_min, rho_tilde;
  double inv_av2, inv_al2, inv_p0, inv_av, inv_rho0;
};

struct Prm {
  double cfl, eps_split, eps_tiny, theta_nb, tol_nb, tol_tiny, newton_rtol, newton_gtol, newton_stol, h_av;
  double lin_gtol;  // quadratic-regime acceptance (R14d) only below this scaled residual; 0: off
  long long dts_max_iter;
  int newton_max_iter, armijo_max, mode;
};

__device__ __forceinline__ int phase_of(const Eos& e, double rho) {
  return rho <= e.rho_tilde ? VAP : (rho >= e.rho_min ? LIQ : SPIN);
}
// vapour ideal gas, liquid linear Tait (R1)
__device__ __forceinline__ double pres(const Eos& e, int ph, double rho) {
  return ph == VAP ? e.a_v2 * rho : e.p0 + e.a_l2 * (rho - e.rho0);
}
__device__ __forceinline__ double sound(const Eos& e, int ph) { return ph == VAP ? e.a_v : e.a_l; }

// Reciprocal for the bulk passes: the hardware seed (rcp.approx.ftz.f64, ~2^-23 relative)
// and one cubic refinement r (1 + e + e^2), e = 1 - x r, relative error ~e^3 before rounding,
// so within an ulp of the correctly rounded value; 4 instructions, deterministic.  Arguments
// are positive normal numbers (densities, HLL speed spans) wherever the result is kept.
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

#ifndef EIS_FAST_RCP
#define EIS_FAST_RCP 1
#endif
// the reciprocals of the interface solver's evaluation chain: rcp_fast (within an ulp, a shorter
// dependent chain; the default since round 2, DESIGN R14e), or correctly rounded (__drcp_rn) in
// EIS_FAST_RCP=0 builds
__device__ __forceinline__ double rcp_sel(double x) {
#if EIS_FAST_RCP
  return rcp_fast(x);
#else
  return __drcp_rn(x);
#endif
}

// ln x for a positive normal x, written for latency (the default; EIS_FAST_LOG=0: log()): x = 2^k m with m in
// [1/sqrt2, sqrt2), ln m = 2 atanh(s), s = (m - 1)/(m + 1) (|s| <= 0.172), the series
// 2 s (1 + s^2/3 + ... + s^22/23) (truncation < 1e-19 relative) in Estrin form, k ln2 in two
// parts.  Within a few ulp of log(x).
__device__ __forceinline__ double log_fast(double x) {
  int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  int k = (hi >> 20) - 1023;
  hi = (hi & 0x000fffff) | 0x3ff00000;
  if (hi >= 0x3ff6a09e) { hi -= 0x00100000; ++k; }
  const double m = __hiloint2double(hi, lo), f = m - 1.0;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(2.0 + f));
  const double e1 = fma(-(2.0 + f), r, 1.0);
  const double s = f * fma(r, fma(e1, e1, e1), r);
  const double z = s * s, z2 = z * z, z4 = z2 * z2, z8 = z4 * z4;
  const double p0 = fma(z, 1.0 / 3, 1.0), p1 = fma(z, 1.0 / 7, 1.0 / 5), p2 = fma(z, 1.0 / 11, 1.0 / 9);
  const double p3 = fma(z, 1.0 / 15, 1.0 / 13), p4 = fma(z, 1.0 / 19, 1.0 / 17), p5 = fma(z, 1.0 / 23, 1.0 / 21);
  const double q0 = fma(z2, p1, p0), q1 = fma(z2, p3, p2), q2 = fma(z2, p5, p4);
  const double poly = fma(z8, q2, fma(z4, q1, q0));
  const double kd = (double)k;
  return fma(kd, 6.93147180369123816490e-01, fma(2.0 * s, poly, kd * 1.90821492927058770002e-10));
}
#ifndef EIS_FAST_LOG
#define EIS_FAST_LOG 1
#endif
__device__ __forceinline__ double log_sel(double x) {
#if EIS_FAST_LOG
  return log_fast(x);
#else
  return log(x);
#endif
}

// ln(a/b) for a/b near 1 (liquid densities, |a/b - 1| < 1e-2): 9-term series of ln(1 + x),
// truncation < 1e-19 relative; otherwise log.  Exact reciprocals use __drcp_rn (correctly rounded,
// so 1/x bit-for-bit, at half the latency of a division).
__device__ __forceinline__ double ln_ratio(double a, double b) {
  const double x = (a - b) * rcp_sel(b);
  if (fabs(x) < 1e-2) {
    return x * (1.0 + x * (-0.5 + x * (1.0 / 3 + x * (-0.25 + x * (0.2 + x * (-1.0 / 6 + x * (1.0 / 7 + x * (-0.125 + x * (1.0 / 9)))))))));
  }
  return log_sel(a * rcp_sel(b));
}

// Outer-wave function in density form (P:1496-1503 with R19): rarefaction a ln(r*/r_K),
// shock a (r* - r_K)/sqrt(r* r_K); df/dr* alongside.
__device__ __forceinline__ void wave_fd(double a, double rs, double rk, double& f, double& df) {
  if (rs > rk) {
    const double iq = rsqrt(rs * rk);
    f = a * (rs - rk) * iq;
    df = 0.5 * a * (rs + rk) * iq * rcp_sel(rs);
  } else {
    f = a * ln_ratio(rs, rk);
    df = a * rcp_sel(rs);
  }
}
__device__ __forceinline__ double wave_f(double a, double rs, double rk) {
  if (rs > rk) return a * (rs - rk) / sqrt(rs * rk);
  return a * log(rs / rk);
}

// HLL flux with Davis bounds.  Same phase, constant sound speed a.
__device__ __forceinline__ void hll(const Eos& e, int ph, double rl, double ml, double ul, double rr,
                                    double mr, double ur, double& F0, double& F1) {
  double a = sound(e, ph);
  double FL1 = ml * ul + pres(e, ph, rl);
  double FR1 = mr * ur + pres(e, ph, rr);
  double SL = fmin(ul, ur) - a, SR = fmax(ul, ur) + a;
  if (SL >= 0.0) { F0 = ml; F1 = FL1; return; }
  if (SR <= 0.0) { F0 = mr; F1 = FR1; return; }
  double inv = 1.0 / (SR - SL), SLSR = SL * SR;
  F0 = (SR * ml - SL * mr + SLSR * (rr - rl)) * inv;
  F1 = (SR * FL1 - SL * FR1 + SLSR * (mr - ml)) * inv;
}

// HLL with the cell pressures precomputed (the bulk pass shuffles them between lanes).
__device__ __forceinline__ void hll_p(double a, double rl, double ml, double ul, double pl, double rr, double mr,
                                      double ur, double pr, double& F0, double& F1) {
  const double FL1 = ml * ul + pl, FR1 = mr * ur + pr;
  const double SL = fmin(ul, ur) - a, SR = fmax(ul, ur) + a;
  if (SL >= 0.0) { F0 = ml; F1 = FL1; return; }
  if (SR <= 0.0) { F0 = mr; F1 = FR1; return; }
  const double inv = rcp_sel(SR - SL), SLSR = SL * SR;
  F0 = (SR * ml - SL * mr + SLSR * (rr - rl)) * inv;
  F1 = (SR * FL1 - SL * FR1 + SLSR * (mr - ml)) * inv;
}

// Branch-light HLL for the bulk pass: min/max as compare-selects (finite inputs), the general
// HLL formula always evaluated, the upwind cases selected afterwards.
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ void hll_fast(double a, double rl, double ml, double ul, double pl, double rr, double mr,
                                         double ur, double pr, double& F0, double& F1) {
  const double FL1 = ml * ul + pl, FR1 = mr * ur + pr;
  const double SL = dmin(ul, ur) - a, SR = dmax(ul, ur) + a;
  const double inv = rcp_fast(SR - SL), SLSR = SL * SR;
  double f0 = (SR * ml - SL * mr + SLSR * (rr - rl)) * inv;
  double f1 = (SR * FL1 - SL * FR1 + SLSR * (mr - ml)) * inv;
  f0 = SL >= 0.0 ? ml : (SR <= 0.0 ? mr : f0);
  f1 = SL >= 0.0 ? FL1 : (SR <= 0.0 ? FR1 : f1);
  F0 = f0; F1 = f1;
}

// Decision margins: a threshold decision is marginal when its test value
// lies within MARGIN_ULPS times the rounding-error bound of its own evaluation; counted in
// eis_stats.decision_margin_warnings, never used to decide anything.
constexpr double MARGIN_EPS = 16.0 * 2.220446049250313e-16;
__device__ __forceinline__ bool width_marginal(double h, double thr) { return fabs(h - thr) <= MARGIN_EPS * thr; }

// Creation trigger, reading R7: liquid edge cavitates iff Phi(rho_min) > 0, vapour edge
// nucleates iff Phi(rho_tilde) < 0, Phi(r) = f(r; r_L) + f(r; r_R) + du.  Exact pre-filters:
// ln y >= 1 - 1/y gives Phi_liq(rho_min) <= du - a(1 - rho_min^2/(r_L r_R))... (no trigger when
// du <= a_l (1 - rho_min^2/(r_L r_R)) for two rarefactions); nucleation needs du < 0.
// marg: set when the test value Phi lies within its rounding-error bound of 0 (only reached past
// the pre-filters, whose 1e-9 m/s margin is far above that bound)
__device__ __forceinline__ bool creation_trigger(const Eos& e, int ph, double rl, double ul, double rr, double ur,
                                                 bool& marg) {
  double du = ur - ul;
  if (ph == LIQ) {
    // pre-filter (exact, ln y <= y - 1): both rarefactions and du <= a_l (1 - rho_min^2/(r_L r_R)),
    // in product form with a 1e-9 m/s margin so rounding never hides a trigger
    const double x = rl * rr;
    if (rl >= e.rho_min && rr >= e.rho_min && du * x <= e.a_l * (x - e.rho_min * e.rho_min) - 1e-9 * x) return false;
  } else if (du >= 0.0) {
    return false;
  }
  const double a = ph == LIQ ? e.a_l : e.a_v, thr = ph == LIQ ? e.rho_min : e.rho_tilde;
  const double fl = wave_f(a, thr, rl), fr = wave_f(a, thr, rr), phi = fl + fr + du;
  marg = fabs(phi) <= MARGIN_EPS * (fabs(fl) + fabs(fr) + fabs(ul) + fabs(ur));
  return ph == LIQ ? phi > 0.0 : phi < 0.0;
}

// ---------------------------------------------------------------------------------------
// Nonlinear 2x2 problems: G and the analytic Jacobian.
// ---------------------------------------------------------------------------------------
// Kinetic relation z = tau p_V [[g + e_kin]], e_kin interface-relative (R2):
// A z^2 - z + B = 0 -> z = 2B/(1 + sqrt(1 - 4AB)); since 2Az - 1 = -sqrt(1 - 4AB) for this
// root, dz/dq = (dA/dq z^2 + dB/dq) / sqrt(1 - 4AB).

// Two-phase interface (App. A, system (13), orientation-general [[x]] = x+ - x-),
// unknowns x = (p_V*, p_L*).  aux = (z, f_V).
struct IfaceProb {
  double rV, uV, rL, uL;  // outer states by phase
  double du;              // u_plus - u_minus
  double sV;              // +1 if the vapour is the plus side, -1 if it is the minus side
};

__device__ __forceinline__ bool iface_eval(const Eos& e, const IfaceProb& P, double pV, double pL,
                                           double G[2], double J[4], double aux[2], double daux[4]) {
  if (!(pV > 0.0)) return false;
  const double rVs = pV * e.inv_av2;
  const double rLs = e.rho0 + (pL - e.p0) * e.inv_al2;
  if (!(rLs > 0.0)) return false;
  const double vV = e.a_v2 * rcp_sel(pV), vL = rcp_sel(rLs);
  const double gV = e.a_v2 * log_sel(pV * e.inv_p0), gL = e.a_l2 * ln_ratio(rLs, e.rho0);
  const double sV = P.sV, sL = -P.sV;
  const double jp = sV * pV + sL * pL, jv = sV * vV + sL * vL;
  const double jv2 = sV * vV * vV + sL * vL * vL, jg = sV * gV + sL * gL;
  const double tp = e.tau * pV;
  const double A = 0.5 * tp * jv2, B = tp * jg;
  const double disc = 1.0 - 4.0 * A * B;
  if (!(disc > 0.0)) return false;
  const double sq = sqrt(disc);
  const double z = 2.0 * B * rcp_sel(1.0 + sq);
  double fV, dfV, fL, dfL;
  wave_fd(e.a_v, rVs, P.rV, fV, dfV);
  wave_fd(e.a_l, rLs, P.rL, fL, dfL);
  G[0] = (jp + z * z * jv) * e.inv_p0;
  G[1] = (fV + fL + z * jv + P.du) * e.inv_av;
  aux[0] = z;
  aux[1] = fV;
  const double dvV = -vV * vV * e.inv_av2, dvL = -vL * vL * e.inv_al2;  // dv/dp
  const double dA_V = 0.5 * e.tau * jv2 + tp * sV * vV * dvV;           // d(v^2)/dp = 2 v dv/dp
  const double dA_L = tp * sL * vL * dvL;
  const double dB_V = e.tau * jg + tp * sV * vV;                         // dg/dp = v
  const double dB_L = tp * sL * vL;
  const double isq = rcp_sel(sq), z2 = z * z;
  const double zV = (dA_V * z2 + dB_V) * isq, zL = (dA_L * z2 + dB_L) * isq;
  J[0] = (sV + 2.0 * z * zV * jv + z2 * sV * dvV) * e.inv_p0;
  J[1] = (sL + 2.0 * z * zL * jv + z2 * sL * dvL) * e.inv_p0;
  J[2] = (dfV * e.inv_av2 + zV * jv + z * sV * dvV) * e.inv_av;
  J[3] = (dfL * e.inv_al2 + zL * jv + z * sL * dvL) * e.inv_av;
  daux[0] = zV; daux[1] = zL;           // d aux / d (pV, pL): z, then f(rho_V*; rho_V)
  daux[2] = dfV * e.inv_av2; daux[3] = 0.0;
  return true;
}

// Creation (App. B, reading R18): unknowns x = (p_A, p_B); A = outer phase, B = created.
// aux = (z_r, f(rho_A*; rho_l)).
struct CreateProb {
  int A;                 // outer phase (LIQ: cavitation, VAP: nucleation)
  double rl, rr, du;     // outer states' densities and u_r - u_l
};

__device__ __forceinline__ bool create_eval(const Eos& e, const CreateProb& P, double pA, double pB,
                                            double G[2], double J[4], double aux[2], double* /*daux: unused*/) {
  const bool cav = (P.A == LIQ);
  const double rA = cav ? e.rho0 + (pA - e.p0) * e.inv_al2 : pA * e.inv_av2;
  const double rB = cav ? pB * e.inv_av2 : e.rho0 + (pB - e.p0) * e.inv_al2;
  if (!(rA > 0.0) || !(rB > 0.0)) return false;
  const double pV = cav ? pB : pA;
  if (!(pV > 0.0)) return false;
  const double vA = __drcp_rn(rA), vB = __drcp_rn(rB);
  const double gA = cav ? e.a_l2 * ln_ratio(rA, e.rho0) : e.a_v2 * log(pA * e.inv_p0);
  const double gB = cav ? e.a_v2 * log(pB * e.inv_p0) : e.a_l2 * ln_ratio(rB, e.rho0);
  const double jv = vA - vB, jv2 = vA * vA - vB * vB, jg = gA - gB;  // right boundary: minus B, plus A
  const double tp = e.tau * pV;
  const double A = 0.5 * tp * jv2, B = tp * jg;
  const double disc = 1.0 - 4.0 * A * B;
  if (!(disc > 0.0)) return false;
  const double sq = sqrt(disc);
  const double z = 2.0 * B * rcp_sel(1.0 + sq);
  const double aA = cav ? e.a_l : e.a_v;
  double f1, df1, f2, df2;
  wave_fd(aA, rA, P.rl, f1, df1);
  wave_fd(aA, rA, P.rr, f2, df2);
  G[0] = (pA - pB + z * z * jv) * e.inv_p0;
  G[1] = (P.du + f1 + f2 + 2.0 * z * jv) * e.inv_av;
  aux[0] = z;
  aux[1] = f1;
  const double ia2A = cav ? e.inv_al2 : e.inv_av2, ia2B = cav ? e.inv_av2 : e.inv_al2;
  const double dvA = -vA * vA * ia2A, dvB = -vB * vB * ia2B;
  const double dA_A = (cav ? 0.0 : 0.5 * e.tau * jv2) + tp * vA * dvA;
  const double dA_B = (cav ? 0.5 * e.tau * jv2 : 0.0) - tp * vB * dvB;
  const double dB_A = (cav ? 0.0 : e.tau * jg) + tp * vA;
  const double dB_B = (cav ? e.tau * jg : 0.0) - tp * vB;
  const double isq = rcp_sel(sq), z2 = z * z;
  const double zA = (dA_A * z2 + dB_A) * isq, zB = (dA_B * z2 + dB_B) * isq;
  J[0] = (1.0 + 2.0 * z * zA * jv + z2 * dvA) * e.inv_p0;
  J[1] = (-1.0 + 2.0 * z * zB * jv - z2 * dvB) * e.inv_p0;
  J[2] = ((df1 + df2) * ia2A + 2.0 * zA * jv + 2.0 * z * dvA) * e.inv_av;
  J[3] = (2.0 * zB * jv - 2.0 * z * dvB) * e.inv_av;
  return true;
}

// ---------------------------------------------------------------------------------------
// Newton-Armijo (Kelley) executed by a group of 16 lanes (a half warp):
// every lane holds the same iterate; Armijo candidates lambda = 2^-k are evaluated in
// parallel, k = lane (+16 per round), the accepted step is the smallest k satisfying
// ||G(x + lambda d)||_2 <= (1 - 1e-4 lambda) ||G(x)||_2 (identical to sequential halving).
// Each candidate evaluation returns G, the analytic Jacobian (14) and aux, so one
// evaluation latency per iteration.  Stop (R14c): ||G(x_new)||_inf <= gtol and the accepted
// step |s_j| <= sqrt(rtol) max(|x_j|, p0) -- with quadratic convergence the new iterate is then
// within ~rtol of the root (the oracle tests the step against rtol itself, one extra iteration).
// Returns the iteration count (>= 0) or -1; aux holds the value at the returned iterate.
// ---------------------------------------------------------------------------------------
#ifdef EIS_DTS_DEBUG  // development: counts of the one-thread solver (dts_jobs)
__device__ unsigned long long g_dbg[8];  // solves, newton iterations, evaluations, armijo evals, retries, LIN exits
#define EIS_DBG(i) do { if (!HALF) atomicAdd(&g_dbg[i], 1ull); } while (0)
#else
#define EIS_DBG(i) do { } while (0)
#endif
// R14d's acceptance test and update (shared with the one-evaluation fast path iface_try_lin)
__device__ __forceinline__ bool lin_accept(const Eos& e, const Prm& p, const double G[2], double d0, double d1, double x0,
                                           double x1, bool wellc) {
  return wellc && fmax(fabs(G[0]), fabs(G[1])) <= p.lin_gtol && fabs(d0) <= p.newton_stol * fmax(fabs(x0), e.p0) &&
         fabs(d1) <= p.newton_stol * fmax(fabs(x1), e.p0);
}
__device__ __forceinline__ void lin_apply(const double da[4], double d0, double d1, double aux[2], double& x0, double& x1) {
  aux[0] += da[0] * d0 + da[1] * d1;
  aux[1] += da[2] * d0 + da[3] * d1;
  x0 += d0; x1 += d1;
}
// the Newton direction d = -J^-1 G (2x2, Cramer); false for a singular or non-finite Jacobian.
// wellc: det has not cancelled below 1e-8 of its terms (R14d's shortcut needs a well-conditioned J)
__device__ __forceinline__ bool newton_dir(const double G[2], const double J[4], double& d0, double& d1, bool& wellc) {
  const double det = J[0] * J[3] - J[1] * J[2];
  if (!(fabs(det) > 0.0) || !isfinite(det)) return false;
  wellc = fabs(det) >= 1e-8 * (fabs(J[0] * J[3]) + fabs(J[1] * J[2]));
  const double idet = rcp_sel(det);
  d0 = -(J[3] * G[0] - J[1] * G[1]) * idet;
  d1 = -(-J[2] * G[0] + J[0] * G[1]) * idet;
  return true;
}
// HALF = false: the same iteration by one thread, the Armijo candidates tried in order (the first
// accepted k is the smallest: the result is the half warp's bit for bit).
template <class Prob, bool (*EVAL)(const Eos&, const Prob&, double, double, double*, double*, double*, double*),
          bool LIN, bool HALF = true>
__device__ int newton_hw(const Eos& e, const Prm& p, const Prob& P, double& x0, double& x1, double aux[2],
                         unsigned mask, int hl, int base_lane) {
  double G[2], J[4], da[4];
  EIS_DBG(2);
  if (!EVAL(e, P, x0, x1, G, J, aux, da)) return -1;
  for (int it = 0; it < p.newton_max_iter; ++it) {
    EIS_DBG(1);
    // R14d needs a well-conditioned Jacobian (the O(|d|^2) constant grows like 1/|det|): no
    // shortcut when det has cancelled to below 1e-8 of its terms
    double d0, d1;
    bool wellc;
    if (!newton_dir(G, J, d0, d1, wellc)) return -1;
    // quadratic regime (LIN, reading R14d): a residual already <= sqrt(gtol) whose Newton step is
    // within sqrt(rtol) of the iterate puts x + d within ~|d|^2 <= rtol of the root: accept it
    // without another evaluation, the auxiliary values to first order (error O(|d|^2))
    if (LIN && lin_accept(e, p, G, d0, d1, x0, x1, wellc)) {
      lin_apply(da, d0, d1, aux, x0, x1);
      EIS_DBG(5);
      return it + 1;
    }
    const double n0 = G[0] * G[0] + G[1] * G[1];
    // the full step first, on every lane alike (no divergence, no shuffles): accepted almost always
    double y0 = x0 + d0, y1 = x1 + d1, Gy[2], Jy[4], ay[2], dy[4];
    const double c1 = 1.0 - 1e-4;
    EIS_DBG(2);
    bool ok = EVAL(e, P, y0, y1, Gy, Jy, ay, dy) && Gy[0] * Gy[0] + Gy[1] * Gy[1] <= c1 * c1 * n0;
    double s0 = d0, s1 = d1;
    if (!ok && !HALF) {  // back-tracking, lambda = 2^-k in order
      int acc = -1;
      for (int k = 1; k <= p.armijo_max && acc < 0; ++k) {
        const double lam = __longlong_as_double((long long)(1023 - k) << 52);  // 2^-k
        y0 = x0 + lam * d0; y1 = x1 + lam * d1;
        const double cl = 1.0 - 1e-4 * lam;
        EIS_DBG(3);
        if (EVAL(e, P, y0, y1, Gy, Jy, ay, dy) && Gy[0] * Gy[0] + Gy[1] * Gy[1] <= cl * cl * n0) acc = k;
      }
      if (acc < 0) return fmax(fabs(G[0]), fabs(G[1])) <= p.newton_gtol ? it : -1;  // rounding floor
      s0 = y0 - x0; s1 = y1 - x1;
    } else if (!ok) {  // lane-parallel back-tracking: lane k tries lambda = 2^-(k+1), then 2^-(k+17)
      int acc = -1;
      for (int round = 0; round * 16 + 1 <= p.armijo_max && acc < 0; ++round) {
        const int k = round * 16 + hl + 1;
        const double lam = __longlong_as_double((long long)(1023 - k) << 52);  // 2^-k
        y0 = x0 + lam * d0; y1 = x1 + lam * d1;
        const double cl = 1.0 - 1e-4 * lam;
        const bool okk = k <= p.armijo_max && EVAL(e, P, y0, y1, Gy, Jy, ay, dy) &&
                         Gy[0] * Gy[0] + Gy[1] * Gy[1] <= cl * cl * n0;
        const unsigned b = __ballot_sync(mask, okk) & mask;
        if (b) {
          const int src = __ffs(b) - 1;  // the smallest accepted k
          acc = k;
          y0 = __shfl_sync(mask, y0, src); y1 = __shfl_sync(mask, y1, src);
          Gy[0] = __shfl_sync(mask, Gy[0], src); Gy[1] = __shfl_sync(mask, Gy[1], src);
          for (int q = 0; q < 4; ++q) Jy[q] = __shfl_sync(mask, Jy[q], src);
          ay[0] = __shfl_sync(mask, ay[0], src); ay[1] = __shfl_sync(mask, ay[1], src);
          if (LIN) for (int q = 0; q < 4; ++q) dy[q] = __shfl_sync(mask, dy[q], src);
        }
      }
      if (acc < 0) return fmax(fabs(G[0]), fabs(G[1])) <= p.newton_gtol ? it : -1;  // rounding floor
      s0 = y0 - x0; s1 = y1 - x1;
    }
    x0 = y0; x1 = y1;
    G[0] = Gy[0]; G[1] = Gy[1];
    for (int q = 0; q < 4; ++q) J[q] = Jy[q];
    aux[0] = ay[0]; aux[1] = ay[1];
    if (LIN) for (int q = 0; q < 4; ++q) da[q] = dy[q];
    if (fmax(fabs(G[0]), fabs(G[1])) <= p.newton_gtol && fabs(s0) <= p.newton_stol * fmax(fabs(x0), e.p0) &&
        fabs(s1) <= p.newton_stol * fmax(fabs(x1), e.p0))
      return it + 1;
  }
  return -1;
}

#ifndef EIS_NEWTON_LIN
#define EIS_NEWTON_LIN true
#endif

// HLLC starting value (Eq. (17)), vapour left / liquid right, mirrored when the
// liquid is on the left; clamped to [0.01 p0, 4 p0] (R14b).
__device__ __forceinline__ double hllc_guess(const Eos& e, double rV, double uV, double rL, double uL) {
  double pV = e.a_v2 * rV, pL = e.p0 + e.a_l2 * (rL - e.rho0);
  double SL = uL + e.a_l, SV = uV - e.a_v;
  double w = (pL - pV + rV * uV * (SV - uV) - rL * uL * (SL - uL)) / (rV * (SV - uV) - rL * (SL - uL));
  double rLs = rL * (SL - uL) / (SL - w);
  double ps = e.p0 + e.a_l2 * (rLs - e.rho0);
  return fmin(fmax(ps, 0.01 * e.p0), 4.0 * e.p0);
}

struct IfaceSol {
  double F0, F1, w, pV, pL;
  int iters;  // -1 on failure
};

// Phase-boundary Riemann solve by a half warp (HALF) or one thread.  (rm, um) minus (left)
// state, (rp, up) plus.  Warm start: if x_init0 > 0 use (x_init0, x_init1) as the first iterate,
// else HLLC.  Outputs F_PB = (-z, -z u_V* + p_V*) (vapour side R17), w = u_V* + z v_V*.
__device__ __forceinline__ IfaceProb iface_prob(double rm, double um, double rp, double up, bool vap_minus) {
  IfaceProb P;
  if (vap_minus) { P.rV = rm; P.uV = um; P.rL = rp; P.uL = up; P.sV = -1.0; }
  else { P.rV = rp; P.uV = up; P.rL = rm; P.uL = um; P.sV = 1.0; }
  P.du = up - um;
  return P;
}
// the boundary's flux and speed from the converged star pressures and aux = (z, f_V)
__device__ __forceinline__ void iface_finish(const Eos& e, const IfaceProb& P, bool vap_minus, double x0,
                                             const double aux[2], IfaceSol& s) {
  const double z = aux[0], fV = aux[1];
  const double uVs = vap_minus ? P.uV - fV : P.uV + fV;  // wave relations
  s.w = uVs + z * e.a_v2 * rcp_sel(x0);                  // z = -rho_V* (u_V* - w)
  s.F0 = -z;
  s.F1 = -z * uVs + x0;
}

template <bool HALF>
__device__ __forceinline__ IfaceSol iface_solve_x(const Eos& e, const Prm& p, double rm, double um, double rp,
                                                  double up, bool vap_minus, double x_init0, double x_init1,
                                                  unsigned mask, int hl, int base_lane) {
  const IfaceProb P = iface_prob(rm, um, rp, up, vap_minus);
  double x0, x1, aux[2];
  if (x_init0 > 0.0) { x0 = x_init0; x1 = x_init1; }
  else {
    const double g = vap_minus ? hllc_guess(e, P.rV, P.uV, P.rL, P.uL) : hllc_guess(e, P.rV, -P.uV, P.rL, -P.uL);
    x0 = g; x1 = g;
  }
  EIS_DBG(0);
  int it = newton_hw<IfaceProb, iface_eval, EIS_NEWTON_LIN, HALF>(e, p, P, x0, x1, aux, mask, hl, base_lane);
  if (it < 0 && x_init0 > 0.0) {  // warm start failed: retry from the HLLC estimate
    EIS_DBG(4);
    const double g = vap_minus ? hllc_guess(e, P.rV, P.uV, P.rL, P.uL) : hllc_guess(e, P.rV, -P.uV, P.rL, -P.uL);
    x0 = g; x1 = g;
    it = newton_hw<IfaceProb, iface_eval, EIS_NEWTON_LIN, HALF>(e, p, P, x0, x1, aux, mask, hl, base_lane);
  }
  IfaceSol s;
  s.iters = it;
  s.pV = x0; s.pL = x1;
  if (it < 0) { s.F0 = s.F1 = s.w = 0.0; return s; }
  iface_finish(e, P, vap_minus, x0, aux, s);
  return s;
}
// The warm-started solve when its first Newton step is accepted by R14d (the usual case inside
// Algorithm 2): one evaluation, straight-line code (two of these side by side overlap).  Returns
// false when the general solver is needed; when true, s is iface_solve_x's result (the same
// expressions; compiled in another context the compiler may contract a multiply-add differently,
// so equal up to the last bits).
__device__ __forceinline__ bool iface_try_lin(const Eos& e, const Prm& p, double rm, double um, double rp, double up,
                                              bool vap_minus, double x0, double x1, IfaceSol& s) {
  if (!EIS_NEWTON_LIN || !(x0 > 0.0) || !(p.newton_max_iter > 0)) return false;
  const IfaceProb P = iface_prob(rm, um, rp, up, vap_minus);
  double G[2], J[4], aux[2], da[4];
  if (!iface_eval(e, P, x0, x1, G, J, aux, da)) return false;
  double d0, d1;
  bool wellc;
  if (!newton_dir(G, J, d0, d1, wellc)) return false;
  if (!lin_accept(e, p, G, d0, d1, x0, x1, wellc)) return false;
  lin_apply(da, d0, d1, aux, x0, x1);
  s.iters = 1;
  s.pV = x0; s.pL = x1;
  iface_finish(e, P, vap_minus, x0, aux, s);
  return true;
}
__device__ __noinline__ IfaceSol iface_solve_hw(const Eos& e, const Prm& p, double rm, double um, double rp,
                                                double up, bool vap_minus, double x_init0, double x_init1,
                                                unsigned mask, int hl, int base_lane) {
  return iface_solve_x<true>(e, p, rm, um, rp, up, vap_minus, x_init0, x_init1, mask, hl, base_lane);
}
__device__ __noinline__ IfaceSol iface_solve_t(const Eos& e, const Prm& p, double rm, double um, double rp,
                                               double up, bool vap_minus, double x_init0, double x_init1) {
  return iface_solve_x<false>(e, p, rm, um, rp, up, vap_minus, x_init0, x_init1, 0u, 0, 0);
}

struct CreateSol {
  double Fl0, Fl1, wl, Fr0, Fr1, wr, rB, mB;
  int iters;
};

// Phase creation by a half warp (App. B steps (ii)-(v), reading R18), Newton start (p0, p0).
__device__ __noinline__ CreateSol create_solve_hw(const Eos& e, const Prm& p, int phase_outer, double rl,
                                                  double ul, double rr, double ur, unsigned mask, int hl,
                                                  int base_lane) {
  CreateProb P{phase_outer, rl, rr, ur - ul};
  double x0 = e.p0, x1 = e.p0, aux[2];
  const int it = newton_hw<CreateProb, create_eval, false>(e, p, P, x0, x1, aux, mask, hl, base_lane);
  CreateSol s;
  s.iters = it;
  if (it < 0) return s;
  const bool cav = (phase_outer == LIQ);
  const double rA = cav ? e.rho0 + (x0 - e.p0) * e.inv_al2 : x0 * e.inv_av2;
  const double rB = cav ? x1 * e.inv_av2 : e.rho0 + (x1 - e.p0) * e.inv_al2;
  const double zr = aux[0];
  const double uAl = ul - aux[1];  // left outer wave
  const double vA = __drcp_rn(rA), vB = __drcp_rn(rB);
  const double uB = uAl + zr * (vB - vA);
  const double zl = -zr;
  s.wl = uB + zl * vB;
  s.wr = uB + zr * vB;
  s.Fl0 = -zl; s.Fl1 = -zl * uB + x1;
  s.Fr0 = -zr; s.Fr1 = -zr * uB + x1;
  s.rB = rB;
  s.mB = rB * uB;
  if (!(s.wr > s.wl)) s.iters = -1;
  return s;
}

}  // namespace eis
