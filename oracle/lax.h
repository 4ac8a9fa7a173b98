/*
 * oracle/lax.h — CPU ORACLE for the paper's first test (arXiv 2211.00705, Sec. "Stationary
 * Phase Boundary without Phase Transition"): the Lax shock tube for the full
 * 1D compressible Euler equations of an ideal gas (gamma = 1.4) on a fixed model mesh with
 * one small cell of width alpha*h, solved with dual time stepping (Algorithm 2) on the cells
 * k-1, k, k+1 and the exact Riemann solver as numerical flux.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/eiso.h): only tests/, __graft_entry__.smoke() and
 * bench.py's reference legs may load it.  It shares no code with the CUDA path.
 *
 * Readings (L1-L7) are cited where the paper is silent.
 *
 * Parity-pin status: exact Riemann solver -> pinned (Rankine-Hugoniot and isentropic /
 * Riemann-invariant relations checked independently, closed-form special cases); explicit
 * Godunov scheme -> pinned (conservation, L1 convergence to the exact solution); DTS
 * iteration averages -> pinned only to the printed trend of tab:iterations (P:1177-1189,
 * reading R23: ordering and a factor 1.5), absolute counts parity unpinned.
 */
#ifndef EISO_LAX_H
#define EISO_LAX_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double gamma;                         /* ratio of specific heats (1.4)               */
  double rho_l, u_l, p_l;               /* state for x < 0                            */
  double rho_r, u_r, p_r;               /* state for x > 0                            */
  double x_left, x_right;               /* [x_L, x_R] = [-5, 5]; h = (x_R - x_L)/N     */
  int64_t n;                            /* N: equidistant cells; the mesh has N + 1 cells (L1) */
  double alpha;                         /* small-cell width alpha*h, left face at x = 0 */
  double theta_nb;                      /* theta_{k+-1} (tab:iterations: 0.9, 0.1 or alpha)    */
  double cfl;                           /* C_CFL (0.8)                                 */
  double t_end;                         /* 1.0                                         */
  double tol_nb, tol_tiny;              /* DTS stop: max(res_{k+-1}) < tol_nb, res_k < tol_tiny */
  int64_t dts_max_iter;                 /* cap on DTS iterations per step (status 7 beyond)    */
  int32_t implicit_block;               /* 1: DTS on {k-1, k, k+1}; 0: every cell explicit     */
} eiso_lax_case;

typedef struct {
  int64_t steps;           /* large time steps taken                                     */
  int64_t dts_iters;       /* DTS iterations summed over the steps (Part 1, Alg. 2)      */
  int64_t dts_max;         /* the most DTS iterations of one step                        */
  int64_t riemann_solves;  /* exact Riemann solves                                       */
  double t;                /* time reached                                               */
  int32_t status;          /* 0 ok, 1 bad arguments, 5 Riemann Newton failure, 7 DTS cap, 3 vacuum / non-positive state */
} eiso_lax_stats;

/* Exact Riemann solver for the gamma-law gas (Toro's construction restated): star
 * pressure p* of f_L(p) + f_R(p) + u_R - u_L = 0 by Newton, u*, and the solution sampled at
 * x/t = xi: prim = (rho, u, p).  Returns 0 or a status (3 vacuum, 5 no convergence). */
int eiso_lax_riemann(double gamma, const double wl[3], const double wr[3], double xi, double prim[3],
                     double* p_star, double* u_star, int32_t* iters);

/* Godunov flux at x/t = 0: F = (rho u, rho u^2 + p, u (E + p)), E = p/(gamma-1) + rho u^2/2 */
int eiso_lax_flux(double gamma, const double wl[3], const double wr[3], double F[3]);

/* Runs one case to t_end.  rho, mom, E: host arrays of n + 1 cells (the final conserved
 * state); x_faces: n + 2 face positions (or NULL).  Returns the status (also in st). */
int eiso_lax_run(const eiso_lax_case* c, double* rho, double* mom, double* E, double* x_faces,
                 eiso_lax_stats* st);

#ifdef __cplusplus
}
#endif
#endif
