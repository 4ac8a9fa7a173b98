/*
 * include/eis.h — C ABI of libeis.so, the B200-native (sm_100a, fp64) hot path of
 * May & Thein, "Explicit-Implicit Domain Splitting for Two Phase Flows with Phase
 * Transition" (arXiv 2211.00705).  "P:n" cites line n of the paper's LaTeX source
 * (/root/reference/PAPER.md); "R<k>" cites the readings table of DESIGN.md §3.
 *
 * What a call computes: one or more LARGE TIME STEPS of the mixed explicit-implicit scheme
 * (Algorithm 1) for the 1D isothermal Euler equations with a sharp,
 * grid-aligned liquid-vapour phase boundary, per member of an ensemble of
 * independent grids:
 *   a1-a2  decode + CFL time step  dt = C h_min / S_max        (R5, R6)
 *   a3     HLL fluxes on same-phase edges
 *   a4     cavitation / nucleation trigger                      (R7)
 *   a5     phase-boundary Riemann solve with the kinetic relation (App. A; R2)
 *   a6     phase creation (four-wave solution)                  (App. B; R17, R18)
 *   a7     explicit moving-cell update
 *   a8-a9  tiny cells -> implicit blocks -> dual time stepping
 *   a10    remesh: insert, merge, split                         (R9, R10)
 *
 * Conventions
 *  - Layout: structure of arrays, member-major, fp64: rho[m*cap + i], mom[m*cap + i] (= rho u),
 *    width[m*cap + i]; only i < n_cells[m] is live (entries beyond are unspecified: a single
 *    grid moves only its live cells between host and device).  cap = eis_grid.cell_capacity.
 *  - where = EIS_HOST: pointers are host memory (copied with cudaMemcpyAsync on the context's
 *    stream, then the call synchronises).  where = EIS_DEVICE: device pointers on grid.device,
 *    accessed stream-ordered on grid.stream (no synchronisation unless stated).
 *  - Ownership: all buffers passed in are BORROWED for the duration of the call.  The context
 *    owns every device buffer it allocates; eis_destroy frees them.
 *  - Errors: every call returns an eis_status.  A call-level error (bad argument, CUDA
 *    failure) is sticky: later calls return it until eis_set_state succeeds.  Member-level
 *    numerical failures (Newton non-convergence, DTS cap, spinodal state, capacity) do NOT fail
 *    the call: that member is frozen and eis_member_status reports the code.
 *  - Threads: one host thread per context at a time.
 */
#ifndef EIS_H
#define EIS_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EIS_OK = 0,
  EIS_E_ARG = 1,             /* invalid argument                                            */
  EIS_E_ORDER = 2,           /* step/get before a successful eis_set_state                 */
  EIS_E_NONPOS_DENSITY = 3,  /* rho <= 0                                                   */
  EIS_E_SPINODAL = 4,        /* a density in (rho_tilde, rho_min)                  */
  EIS_E_NEWTON = 5,          /* interface Newton-Armijo did not converge (R14)             */
  EIS_E_CREATION = 6,        /* creation solve failed or w_r <= w_l                        */
  EIS_E_DTS_CAP = 7,         /* dual time stepping reached dts_max_iter (P:688 l_max)       */
  EIS_E_WIDTH = 8,           /* a cell width became <= 0                                   */
  EIS_E_CAPACITY = 9,        /* cell_capacity or an internal table exceeded                */
  EIS_E_CUDA = 10,           /* CUDA runtime error (message in eis_last_error)             */
  EIS_E_NCCL = 11,           /* reserved: NCCL error                                       */
  EIS_E_UNSUPPORTED = 12,    /* tiny cell at a domain end (R26)                            */
  EIS_E_INTERNAL = 13        /* internal consistency check failed (a bug: please report)   */
} eis_status;

enum { EIS_HOST = 0, EIS_DEVICE = 1 };
enum {
  EIS_MODE_SPLIT = 0,    /* Algorithms 1-2: dual time stepping on the tiny cells' neighbourhoods        */
  EIS_MODE_EXPLICIT = 1, /* global explicit, dt from all cells                                          */
  EIS_MODE_LTS = 2,      /* explicit local time stepping of the tiny cells (the paper's comparison method,
                            P:472-482; readings R29-R31); stats count its sub-steps as
                            dts_iters ("local iterations")                                               */
  EIS_MODE_NEWTON = 3    /* as SPLIT, with Algorithm 2's implicit system W = T(W) solved by a chord Newton
                            iteration (forward-difference Jacobian at U^n) instead of dual time stepping:
                            the paper's "Newton-like approach" (readings N1-N5); stats
                            count evaluations of T as dts_iters                                          */
};
enum { EIS_VAP = 0, EIS_LIQ = 1, EIS_SPIN = 2 };
enum { EIS_LAYOUT_AUTO = 0, EIS_LAYOUT_RESIDENT = 1, EIS_LAYOUT_TILED = 2 };

/* EOS record (immutable per context).  Vapour p = a_v2 rho; liquid
 * p = p0 + a_l^2 (rho - rho0) (P:1121 corrected, R1). */
typedef struct {
  double a_v2;      /* kT0/m, m^2/s^2                                                       */
  double a_l;       /* liquid sound speed sqrt(K0/rho0), m/s                               */
  double rho0, p0;  /* saturation liquid density and pressure at T0                        */
  double tau;       /* kinetic coefficient; <= 0 -> (2 pi)^-1/2 a_v2^-3/2 (R22)   */
  double p_min;     /* minimum liquid pressure; rho_min = rho0 + (p_min - p0)/a_l^2 */
  double rho_tilde; /* maximum vapour density; <= 0 -> Maxwell equal area from p_min (R3)  */
} eis_eos;

/* scheme parameters (P:1127-1135 and DESIGN.md readings) */
typedef struct {
  double cfl;                /* C_CFL                                               */
  double eps_split;          /* split cells wider than eps_split*h_av: 2            */
  double eps_tiny;           /* merge / tiny below eps_tiny*h_av (R4): 0.5                 */
  double theta_nb;           /* theta_{k+-1}: 0.9; theta_k = alpha (R12)          */
  double tol_nb, tol_tiny;   /* DTS stop: 1e-3, 1e-1                             */
  int64_t dts_max_iter;      /* l_max                                             */
  double newton_rtol;        /* R14: 1e-13                                                 */
  double newton_gtol;        /* R14: 1e-12 (scaled residual)                               */
  int32_t newton_max_iter;   /* R14: 50                                                    */
  int32_t armijo_max;        /* Armijo halvings (Kelley): 30                       */
  int32_t mode;              /* EIS_MODE_SPLIT | _EXPLICIT | _LTS | _NEWTON                */
  int32_t reserved;
} eis_params;

typedef struct {
  int64_t n_members;      /* independent grids (ensembles C3/C4; 1 for C1/C2)              */
  int64_t n_cells;        /* initial cells per member N; h_av = (x_right - x_left)/N (R9) */
  int64_t cell_capacity;  /* >= n_cells: slack for created / split cells                   */
  double x_left, x_right; /* domain                                                        */
  double h_av;            /* 0: (x_right - x_left)/n_cells; > 0: this value (a slice of a grid
                             cut over ranks keeps the whole grid's h_av bit for bit)          */
  int32_t device;         /* CUDA device ordinal                                           */
  int32_t threads;        /* CTA size per member / tile (0 = automatic)                    */
  int32_t layout;         /* EIS_LAYOUT_AUTO (tiled when cell_capacity > 2048) | _RESIDENT (each
                             member in shared memory across the steps of a call, cell_capacity
                             <= 16384) | _TILED (members streamed through HBM every step in
                             halo-overlapped tiles; halos never cross members; each member its
                             own dt, t and status; rank mode requires n_members == 1)          */
  int32_t tile_cells;     /* tiled: owned cells per tile (0 = 1400, range 40..8192); a member's
                             ceil(n_cells / tile_cells) tiles are fixed-size from the left, the
                             last one takes the remainder; a member whose live count does not
                             reach its last tile by 10 cells is frozen with EIS_E_CAPACITY    */
  int32_t nbr_left;       /* tiled rank mode: 1 if this grid is the right part of a grid cut
                             over ranks (its left halo arrives through the exchange buffer)  */
  int32_t nbr_right;      /* ... 1 if a rank continues the grid on the right                   */
  void* stream;           /* cudaStream_t (NULL = legacy default stream)                   */
} eis_grid;

typedef struct {
  int64_t member, edge;   /* edge e lies between cells e-1 and e                           */
  double x;               /* x_left + widths summed left to right (fixed order, no FMA)    */
  int32_t left_phase, right_phase;
  /* the phase-boundary Riemann problem (App. A, kinetic relation R2) of the two
   * adjacent cells' current states, solved from the HLLC estimate:           */
  double w;               /* speed of the phase boundary                                   */
  double z;               /* mass flux through it, z = -rho (u - w) (same on both sides)    */
  double p_vap, p_liq;    /* star pressures on the vapour and liquid sides                 */
  int32_t solve_status;   /* 0, or EIS_E_NEWTON if that solve did not converge             */
  int32_t reserved;
} eis_interface;

typedef struct {
  int64_t steps;          /* member steps taken (summed over members)                      */
  int64_t cell_updates;   /* live cells advanced by one large step (the bench metric unit) */
  int64_t dts_iters;      /* dual-time iterations ("local iterations")             */
  int64_t iface_solves;   /* phase-boundary Riemann solves                                 */
  int64_t creations, splits, merges, regions;
  double t_min, t_max, dt_min, dt_max;
  int64_t dts_iter_max;   /* most dual-time iterations one implicit block took in one step */
  /* discrete decisions taken within the rounding-error bound of their own threshold test
   * (the paper's round-off warning P:1133-1135): DTS stop / continue,
   * creation trigger (R7), tiny / merge / split width thresholds (R4).  Such a decision
   * may flip between two correct fp64 implementations (it never changes a result here). */
  int64_t decision_margin_warnings;
} eis_stats;

typedef struct { double rho_min, rho_tilde, p_tilde, tau, a_v; } eis_thresholds;

/* Derived thresholds (R3): host computation, no context needed. */
eis_status eis_thresholds_of(const eis_eos* eos, eis_thresholds* out);

typedef struct eis_ctx eis_ctx;

/* Create a context on grid->device: validates the records, derives the thresholds, allocates
 * n_members * cell_capacity fp64 state in device memory.  *out is NULL on error. */
eis_status eis_create(const eis_eos* eos, const eis_params* params, const eis_grid* grid, eis_ctx** out);

/* Load the state U^0 = (rho, mom) and widths (NULL: uniform h_av) of every member, the live
 * cell counts (NULL: all n_cells) and the start time t0.  Resets member status and counters,
 * clears a sticky error.  Tiny flags are derived from the state (R4, R10). */
eis_status eis_set_state(eis_ctx* ctx, const double* rho, const double* mom, const double* width,
                         const int64_t* n_cells, int32_t where, double t0);

/* Every non-frozen member takes n_steps large steps (its own dt, R25).  Stream-ordered: with
 * out == NULL nothing synchronises; with out != NULL the call synchronises and fills the
 * counters accumulated since eis_set_state. */
eis_status eis_step(eis_ctx* ctx, int64_t n_steps, eis_stats* out);

/* Every non-frozen member steps until t >= t_end (last dt clipped to t_end - t) or max_steps
 * steps were taken in this call.  Same synchronisation rule as eis_step. */
eis_status eis_run_to(eis_ctx* ctx, double t_end, int64_t max_steps, eis_stats* out);

/* Copy the state out: arrays sized n_members*cell_capacity (entries past n_cells[m] are 0;
 * phase is EIS_VAP/EIS_LIQ/EIS_SPIN per cell, 255 past the end), n_cells[n_members] and
 * t[n_members].  Any pointer may be NULL.  where = EIS_HOST synchronises. */
eis_status eis_get_state(eis_ctx* ctx, double* rho, double* mom, double* width, uint8_t* phase,
                         int64_t* n_cells, double* t, int32_t where);

/* Phase boundaries of the current state, member-major and left to right, into a host array of
 * `capacity` records, each with the Riemann solution of its two adjacent cells (one half warp
 * per boundary); *count gets the total (EIS_E_CAPACITY if it exceeds capacity; out == NULL is a
 * pure count query). */
eis_status eis_interfaces(eis_ctx* ctx, eis_interface* out, int64_t capacity, int64_t* count);

/* Per-member status codes (host array of n_members). */
eis_status eis_member_status(eis_ctx* ctx, int32_t* out);

/* Per-member counters (host array of n_members eis_stats; t_min = t_max = member time). */
eis_status eis_member_stats(eis_ctx* ctx, eis_stats* out);

/* ---- rank mode: one tiled grid cut over ranks (BASELINE configs[4] on 2-8 GPUs) ----------
 * Each rank owns a contiguous, tile-aligned slice.  Per step the caller runs
 *   eis_step_local   -> (exchange: send_left -> left rank's recv_right, send_right -> right
 *                       rank's recv_left; min-allreduce of the 2-double CFL pair)
 *   eis_step_finish(after_step = 1)
 * and after eis_set_state: exchange, then eis_step_finish(after_step = 0) (initial dt).
 * eis_step_local and eis_step_finish only enqueue work on the context's stream (no host
 * synchronisation, no allocation), so the per-step sequence, the exchange's NCCL calls included,
 * can be captured into a CUDA graph on that stream and replayed (decomp.RankGrid); steps issued
 * during a capture record no eis_set_timing events.
 * Exchange buffer: EIS_XB_DOUBLES doubles of device memory owned by the caller, borrowed for
 * the context's lifetime: records of EIS_HALO cells (rho[EIS_HALO], mom[..], h[..], count)
 * at offsets EIS_XB_SEND_LEFT, _SEND_RIGHT, _RECV_LEFT, _RECV_RIGHT, then the pair
 * (-S_max, h_min) at EIS_XB_DT.  Min-reduction of the pair gives the global CFL dt. */
#define EIS_HALO 10
#define EIS_XB_REC (3 * EIS_HALO + 1)
#define EIS_XB_SEND_LEFT 0
#define EIS_XB_SEND_RIGHT EIS_XB_REC
#define EIS_XB_RECV_LEFT (2 * EIS_XB_REC)
#define EIS_XB_RECV_RIGHT (3 * EIS_XB_REC)
#define EIS_XB_DT (4 * EIS_XB_REC)
#define EIS_XB_DOUBLES (4 * EIS_XB_REC + 2)
eis_status eis_set_exchange_buffer(eis_ctx* ctx, double* dev_xbuf);
/* Peer mode (the exchange inside the kernels, over NVLink peer memory): every
 * rank's exchange buffer holds EIS_XB_DOUBLES_PEER doubles, zero-initialised, device memory that
 * every rank's device can access (peer-mapped / symmetric memory).  `left` / `right`: the left /
 * right neighbour's buffer (NULL exactly where nbr_left / nbr_right is 0), `all[q]`: rank q's
 * buffer (host array of `world` <= EIS_XB_MAXRANKS device pointers; all[rank] is this context's
 * own).  Then the step's last CTA writes this rank's send records into the neighbours' receive
 * slots and its CFL pair into every rank's pair table (double-buffered by the parity of a
 * publication count, tagged after a system-scope fence); eis_step_finish waits for every rank's
 * tag (one warp; a peer that never publishes ends the wait after ~2 s with member status
 * EIS_E_INTERNAL), folds the pairs (min) and moves the records into the receive slots.  The
 * caller runs no collective: per step eis_step_local -> eis_step_finish(after_step = 1), and
 * after eis_set_state eis_step_finish(after_step = 0).  Every rank must issue the same sequence
 * of calls.  Returns EIS_E_ARG for inconsistent pointers or world. */
#define EIS_XB_MAXRANKS 8
#define EIS_XB_DOUBLES_PEER (EIS_XB_DOUBLES + 4 * EIS_XB_REC + 8 * EIS_XB_MAXRANKS)
eis_status eis_set_exchange_peers(eis_ctx* ctx, double* left, double* right, double* const* all, int32_t rank,
                                  int32_t world);
eis_status eis_step_local(eis_ctx* ctx, double t_end);
eis_status eis_step_finish(eis_ctx* ctx, double t_end, int32_t after_step);

/* Tiled-layout diagnostics (EIS_E_ARG for a member-resident context): the number of tiles, and
 * the tile-steps since eis_set_state that took the full step of the whole tile, or of a window
 * of at most 150 owned cells around the tile's special cells (phase boundaries, creation
 * candidates), rather than only the single-phase fast path.  Synchronises the stream. */
eis_status eis_tile_info(eis_ctx* ctx, int64_t* n_tiles, int64_t* full_tile_steps, int64_t* window_steps);

/* Window prediction (tiled layout, dual time stepping): a window's full step
 * predicts which cells of its tile the next step's streaming pass will flag as special, so that
 * the first part of the predicted windows' full step (phase-boundary solves P:1481-1562, the
 * explicit pass, the export of the implicit blocks) and Algorithm 2 on those blocks
 * run beside the streaming pass of the next step; the streaming pass compares its
 * own classification with the prediction and a window whose prediction failed takes the same
 * full step after it.  Results do not depend on the predictions.  Outputs (host pointers): the
 * window full steps since eis_set_state and how many of them were predicted; enabled = 0 when
 * the context runs without predictions (another mode, rank slices, EIS_WIN_SPEC=0).
 * Synchronises the stream.  EIS_E_ARG for a member-resident context or null pointers. */
eis_status eis_window_prediction(eis_ctx* ctx, int64_t* windows, int64_t* predicted, int32_t* enabled);

/* Window diagnostics (tiled layout, context created with the environment variable
 * EIS_WINDOW_DEBUG set): per window full step of the last step, 11 int64 each -- SM clock cycles,
 * dual-time iterations, window owned cells, phase boundaries in the window grid, start clock,
 * then 6 phase durations (load, to barrier A, to barrier B, creations, remesh, assembly; zero
 * unless the library was built with -DEIS_PHASE_CLOCK).
 * *count = windows of the last step; out may be NULL (count query). */
eis_status eis_window_diag(eis_ctx* ctx, int64_t* out, int64_t capacity, int64_t* count);

/* Kernel timing (measurement support): with timing enabled, every step launch records CUDA
 * events on the context's stream around each kernel (a few microseconds per step).
 * eis_get_timing synchronises the stream and returns the summed milliseconds since
 * eis_set_timing: ms[0] tiled fast pass, ms[1] tiled window full steps, ms[2] tiled whole-tile
 * full steps + next dt (window split: part A, dts_jobs and part B are all in ms[1]), ms[3]
 * member-resident kernel; *launches = kernels the step calls launched meanwhile. */
eis_status eis_set_timing(eis_ctx* ctx, int32_t enable);
eis_status eis_get_timing(eis_ctx* ctx, double* ms /* [4] */, int64_t* launches);

/* ---------------------------------------------------------------------------------------
 * Lax shock tube with one small cell (the paper's first test): a batch of
 * independent cases of the full 1D Euler equations of an ideal gas, each on a fixed mesh of
 * N + 1 cells -- N/2 cells of width h = (x_right - x_left)/N left of x_left + (N/2) h, the small
 * cell of width alpha*h, N/2 cells of width h -- run from the Riemann data (left state for the
 * cells left of the small cell, right state from it on) to t_end.  Every step: dt = cfl h /
 * S_max (S_max = max |u| + c over every cell but the small one when implicit_block, over all
 * cells and with h_min otherwise; the last step clipped to t_end), exact Riemann fluxes
 * on every face, transmissive ends, the explicit update (fixed mesh) outside
 * {k-1, k, k+1}, and Algorithm 2 on {k-1, k, k+1} with dtau = theta dt, theta_k =
 * alpha, the residual of P:1128-1131 and the stop rule max(res_{k+-1}) < tol_nb, res_k <
 * tol_tiny.  Readings L1-L7: DESIGN.md §3.
 *
 * One CTA per case; cases run concurrently.  cases and stats: HOST arrays of n_cases records.
 * rho, mom, E: DEVICE arrays of n_cases * stride doubles; case c's final conserved state is at
 * [c*stride, c*stride + n + 1).  Requirements: n even, 6 <= n, n + 2 <= stride, n <= 4094,
 * alpha > 0, theta_nb > 0, cfl > 0, gamma > 1 (EIS_E_ARG otherwise).  Case failures (vacuum or
 * a non-positive pressure: EIS_E_NONPOS_DENSITY; Riemann Newton: EIS_E_NEWTON; DTS cap:
 * EIS_E_DTS_CAP) are reported in stats[c].status and do not fail the call.  Runs on `stream`
 * (a cudaStream_t, NULL = legacy default) and synchronises it.  No context needed.
 * --------------------------------------------------------------------------------------- */
typedef struct {
  double gamma;                      /* ratio of specific heats (1.4)                */
  double rho_l, u_l, p_l;            /* Riemann data, left                                    */
  double rho_r, u_r, p_r;            /* Riemann data, right                                   */
  double x_left, x_right;            /* domain of the N regular cells ([-5, 5])       */
  int64_t n;                         /* N                                                     */
  double alpha, theta_nb, cfl, t_end;
  double tol_nb, tol_tiny;           /* 1e-3, 1e-1                                   */
  int64_t dts_max_iter;
  int32_t implicit_block;            /* 1: Algorithm 2 on {k-1, k, k+1}; 0: all explicit      */
  int32_t dts_loop;                  /* Algorithm 2 by 0: one warp (dts_warp, the member-resident
                                        kernels' loop); 1: one thread (dts_thread, the tiled
                                        window path's loop) -- same arithmetic, same bits      */
} eis_lax_case;

typedef struct {
  int64_t steps, dts_iters, dts_max, riemann_solves;
  double t;
  int32_t status;
  int32_t margins;                   /* DTS stop decisions within their rounding-error bound   */
} eis_lax_stats;

eis_status eis_lax_run(const eis_lax_case* cases, int64_t n_cases, int64_t stride, double* rho, double* mom,
                       double* E, eis_lax_stats* stats, void* stream);

/* Last error message of the context (static storage owned by the context). */
const char* eis_last_error(const eis_ctx* ctx);

void eis_destroy(eis_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
