/*
 * oracle/eiso.h — CPU ORACLE for May & Thein, "Explicit-Implicit Domain Splitting for Two
 * Phase Flows with Phase Transition" (arXiv 2211.00705).
 *
 * TEST INFRASTRUCTURE ONLY.  This header and oracle/eiso.c are a plain, slow, fp64 CPU
 * implementation of what the GPU hot path computes.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load or call it.  It shares no
 * code, header, constant or helper with the CUDA path (paper_2211_00705_b200/csrc,
 * include/eis.h); the two only meet through the seeded input arrays made by
 * paper_2211_00705_b200/workloads.py.
 *
 * Citations: "P:n" = line n of /root/reference/PAPER.md (the paper's LaTeX source);
 * "R<k>" = reading k listed in DESIGN.md §3 (taken from SURVEY.md §8(c)).
 *
 * Parity-pin status (see DESIGN.md §3 and tests/test_oracle_*.py):
 *   EOS, thresholds, HLL, interface solve, creation solve, CFL rule  -> pinned
 *   (paper-printed values P:1244, P:1263-1264, P:1277, P:1297, P:1390, P:1410, P:1422,
 *    closed forms, brute force, invariants).
 *   DTS loop (Alg. 2 stop rule, residual, pseudo steps)             -> pinned by the paper's
 *   local-iteration counts: cavitation 355 within 10 % (a wrong theta, tolerance or
 *   residual moves it further), nucleation 1,367,460 within the rounding regime of
 *   reading R28 (factor 3, every stop flagged by the decision-margin accounting).
 *   DTS iteration counts at 293 K, C4/C5 long-time dynamics           -> parity unpinned
 *   beyond the invariants (constant states, conservation, mode degeneracy, DTS fixed point).
 */
#ifndef EISO_H
#define EISO_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same numeric meaning as the product's, declared independently) */
enum {
  EISO_OK = 0, EISO_E_ARG = 1, EISO_E_ORDER = 2, EISO_E_NONPOS_DENSITY = 3,
  EISO_E_SPINODAL = 4, EISO_E_NEWTON = 5, EISO_E_CREATION = 6, EISO_E_DTS_CAP = 7,
  EISO_E_WIDTH = 8, EISO_E_CAPACITY = 9, EISO_E_UNSUPPORTED = 12
};
enum { EISO_VAP = 0, EISO_LIQ = 1, EISO_SPIN = 2 };
enum { EISO_MODE_SPLIT = 0, EISO_MODE_EXPLICIT = 1, EISO_MODE_LTS = 2, EISO_MODE_NEWTON = 3 };

typedef struct {
  double a_v2;       /* vapour  p = a_v2 * rho              */
  double a_l, rho0, p0; /* liquid p = p0 + a_l^2 (rho - rho0)         (reading R1)  */
  double tau;        /* kinetic coefficient; <= 0 -> (2 pi)^-1/2 a_v2^-3/2 (R22)   */
  double p_min;      /* minimum liquid pressure; default -9e6 Pa at 293 K (R3)      */
  double rho_tilde;  /* maximum vapour density; <= 0 -> Maxwell equal area (R3)      */
} eiso_eos;

typedef struct {
  double cfl;                 /* C_CFL                                             */
  double eps_split, eps_tiny; /* split h > eps_split*h_av; merge/tiny h < eps_tiny*h_av (R4) */
  double theta_nb;            /* theta_{k+-1}; theta_k = alpha (R12)      */
  double tol_nb, tol_tiny;    /* DTS stop: max(res_{k+-1}) < tol_nb, res_k < tol_tiny */
  int64_t dts_max_iter;       /* l_max                                             */
  double newton_rtol;         /* R14 */
  double newton_gtol;         /* R14 */
  int32_t newton_max_iter, armijo_max; /* R14; Armijo halvings (Kelley)          */
  int32_t mode;               /* EISO_MODE_SPLIT (Alg. 1-2) | EISO_MODE_EXPLICIT | EISO_MODE_LTS |
                               EISO_MODE_NEWTON (Alg. 2's implicit system by chord Newton, N1-N5) */
} eiso_params;

/* derived thresholds (R3) */
typedef struct { double rho_min, rho_tilde, p_tilde, tau, a_v; } eiso_thresholds;

/* two-phase interface Riemann solution (Appendix A) */
typedef struct {
  double p_minus, p_plus;     /* star pressures of the minus (left) / plus (right) side      */
  double rho_minus, rho_plus, u_minus, u_plus;
  double z, w;                /* mass flux z = -rho (u - w) and phase-boundary speed         */
  double F0, F1;              /* F_PB = (-z, -z u* + p*) with vapour-side star values (R17) */
  int32_t iters, status;
} eiso_iface;

/* phase creation (Appendix B, reading R18) */
typedef struct {
  double p_A, p_B;            /* outer star pressure (both sides) and created-phase pressure */
  double rho_A, rho_B, u_B;
  double z_l, z_r, w_l, w_r;
  double Fl0, Fl1, Fr0, Fr1;  /* boundary fluxes (P:1586-1588 / P:1613-1615, reading R17)    */
  int32_t iters, status;
} eiso_creation;

typedef struct {
  int64_t steps, cell_updates, dts_iters, iface_solves, creations, splits, merges, regions;
  double t_min, t_max, dt_min, dt_max;
  /* discrete decisions taken within the rounding-error bound of their own threshold test
   * (the paper's round-off warning P:1133-1135): DTS stop / continue,
   * creation trigger (R7), tiny / merge / split width thresholds (R4).  Such a decision
   * can flip between two correct fp64 implementations; the parity tests accept a differing
   * DTS count only in a member that logged one. */
  int64_t decision_margin_warnings;
} eiso_stats;

typedef struct {
  int64_t member, edge; double x; int32_t left_phase, right_phase;
  double w, z, p_vap, p_liq;  /* Riemann solution of the two adjacent cells (App. A)        */
  int32_t solve_status, reserved;
} eiso_interface;

typedef struct eiso_ctx eiso_ctx;

/* point functions (for pins) */
int  eiso_thresholds_of(const eiso_eos* eos, eiso_thresholds* out);
int  eiso_phase(const eiso_eos* eos, double rho);
double eiso_pressure(const eiso_eos* eos, int phase, double rho);
double eiso_gibbs(const eiso_eos* eos, int phase, double p);
double eiso_wave_f(const eiso_eos* eos, int phase, double rho_star, double rho_k);
int  eiso_hll(const eiso_eos* eos, double rl, double ml, double rr, double mr, double F[2]);
int  eiso_single_phase_star(const eiso_eos* eos, int phase, double rl, double ul, double rr,
                            double ur, double* rho_star);
int  eiso_creation_trigger(const eiso_eos* eos, int phase, double rl, double ul, double rr, double ur);
int  eiso_interface_solve(const eiso_eos* eos, const eiso_params* prm, double rm, double um,
                          double rp, double up, eiso_iface* out);
int  eiso_creation_solve(const eiso_eos* eos, const eiso_params* prm, int phase_outer,
                         double rl, double ul, double rr, double ur, eiso_creation* out);

/* whole-method driver (per member independent; Alg. 1-2 + §3.4 + App. B) */
int  eiso_create(const eiso_eos* eos, const eiso_params* prm, int64_t n_members, int64_t n_cells,
                 int64_t cell_capacity, double x_left, double x_right, eiso_ctx** out);
int  eiso_set_state(eiso_ctx* c, const double* rho, const double* mom, const double* width,
                    const int64_t* n_cells, double t0);
/* OpenMP threads (default 1): over members when n_members > 1, else over the cells, edges and
 * implicit regions of the one member; results are bitwise those of one thread */
int  eiso_set_threads(eiso_ctx* c, int nthreads);
int  eiso_step(eiso_ctx* c, int64_t n_steps, eiso_stats* out);
int  eiso_run_to(eiso_ctx* c, double t_end, int64_t max_steps, eiso_stats* out);
int  eiso_get_state(const eiso_ctx* c, double* rho, double* mom, double* width, uint8_t* phase,
                    int64_t* n_cells, double* t);
int  eiso_interfaces(const eiso_ctx* c, eiso_interface* out, int64_t capacity, int64_t* count);
int  eiso_member_status(const eiso_ctx* c, int32_t* out);
int  eiso_member_stats(const eiso_ctx* c, int64_t member, eiso_stats* out);
void eiso_destroy(eiso_ctx* c);

#ifdef __cplusplus
}
#endif
#endif
