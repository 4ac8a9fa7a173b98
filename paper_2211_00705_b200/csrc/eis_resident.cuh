// eis_resident.cuh — the member-resident large-step kernel (ensembles of members up to 2048
// cells under EIS_LAYOUT_AUTO: C1-C3), and step_body, the whole large step on a grid in shared
// memory, which the tiled window / whole-tile kernels (eis_tiled.cuh) reuse.
//
// One CTA owns one member (an independent 1D grid, R25) for a whole eis_step / eis_run_to
// call: the grid is loaded from HBM into shared memory once, advanced n_steps large steps of
// Algorithm 1 with the moving mesh (§3.4), phase creation (App. B) and
// dual time stepping (Alg. 2), and written back once.  HBM traffic is paid per call,
// not per step; inside a step the kernel is bound by the FP64 pipe and shared memory.
//
// Phase boundaries are kept as an ordered list across steps: phases never change during a step
// (a change is a spinodal error), so boundaries appear only through creation and move only
// through the remesh; tiny cells (R4, R10) are the cells between two consecutive boundaries, so
// implicit blocks (R11) follow from the list in O(#boundaries).
//
// Warp specialisation inside a step (the serial, latency-bound parts run beside the bulk):
//   solver warp (the last warp):
//     S1 tiny cells, implicit blocks, flags, from the boundary list                    (a8)
//     S2 explicit phase-boundary solves, warm-started from the previous step, half warps (a5)
//     -- barrier A (dt) --
//     S4 every implicit block: dual time stepping (a9), or local time stepping (mode LTS)
//        or the chord Newton solve (mode NEWTON)
//     S5 moving-cell update of the cells next to phase boundaries                       (a7)
//   bulk warps (all others; the solver joins when done), dynamic 32-wide windows:
//     P1 per edge: u = m/rho, HLL flux (a3), creation trigger (a4), S_max / h_min (a2)
//     -- barrier A (dt) --
//     P2 per cell: explicit update of cells with two HLL edges (a7)
//   -- barrier B --
//   creations (a6, rare: acceptance R16, half-warp solves, neighbour updates)
//   remesh (a10): event lists (merge pairs, splits, creations) -> per-cell shift -> scatter
#pragma once
#include "eis_device.cuh"
#include "eis_dts.cuh"

namespace eis {

constexpr int MAXIF = 16;    // phase boundaries per member
constexpr int MAXTRG = 8;    // creation triggers per member per step
constexpr int MAXBLK = 8;    // implicit blocks per member
constexpr int MAXEV = 16;    // remesh events (merge edges, split cells) per member per step
constexpr int DTS_SCRATCH = 72;

// flag byte per index i (cell i and its LEFT edge i share the byte)
enum : uint8_t {
  F_TINY = 0x04,    // cell i tiny                      (solver, S1)
  F_REG = 0x08,     // cell i in an implicit block      (solver, S1)
  F_SPEC = 0x10,    // edge i: explicit phase boundary  (solver, S1)
  F_IF = 0x20       // edge i: phase boundary           (boundary list; kernel start / remesh)
};

struct Ifc {            // phase-boundary edge (list ordered by e)
  double F0, F1, w;     // F_PB and the boundary speed
  double pV, pL;        // converged star pressures (warm start of the next solve)
  int e, interior;      // interior: inside an implicit block (solved by DTS)
};
struct Trg {            // creation trigger
  double Fl0, Fl1, wl, Fr0, Fr1, wr, rB, mB;
  int e, acc;
};
struct Grp {            // remesh output replacing cells g0..g1 (merge group, or one split cell)
  double r, m, h;
  int g0, g1, split;
};

struct MemberStats {
  long long steps, cell_updates, dts_iters, iface_solves, creations, splits, merges, regions;
  double dt_min, dt_max;
  long long dts_max;
  long long margins;  // decision_margin_warnings (eis.h): decisions within their rounding-error bound
};

struct Members {  // global (HBM) state, member-major SoA
  double *rho, *mom, *h;
  long long* n;
  double* t;
  int* status;
  MemberStats* stats;
  long long cap;
  long long* dbg;  // development (-DEIS_PHASE_CLOCK): per member summed phase clocks, else null
};

struct CtaShared {
  double part_s[32], part_h[32];
  double ws0[MAXIF], ws1[MAXIF];  // warm start by boundary ordinal (previous step)
  double dts[DTS_SCRATCH];
  Ifc ifc[MAXIF];
  Trg trg[MAXTRG];
  Grp grp[MAXEV];
  int mev[MAXEV], sev[MAXEV];
  int blkA[MAXBLK], blkB[MAXBLK];
  int dj[MAXBLK];  // window split: the DTS job of each block (-1: none)
  int tc[MAXIF];
  int nifc, wsn, ntrg, nblk, n, status, remesh, nmev, nsev, ngrp, n_new;
  int c_merges, c_splits, c_creations;
  int olo, ohi;  // tiles: owned output range after the remesh
  int pf_j, pf_k, pf_wa, pf_wb, pf_slot;  // tiles: the next window job, claimed during the current one
  int fbits;     // tiles: phase bits of the smem grid (fast-path test)
  int sv_n;      // window split: the grid's cell count and dt, saved with it between parts A and B
  double sv_dt;
  int o_cre, o_merges, o_splits;  // events owned by this grid (tiles: not the halo's)
  unsigned long long c_dts, c_solves, c_regions, c_dtsmax, c_margin;
  MemberStats st;
#ifdef EIS_PHASE_CLOCK
  long long tclk[10];  // development: clock64 at phase boundaries of the last step (thread 0)
#endif
#ifdef EIS_FINE_CLOCK
  long long fclk[8];   // development: thread 0's clock after S2, P1, barrier A, S4, barrier B, creations, remesh
#endif
#ifdef EIS_DTS_CLOCK
  long long dclk[5];   // development: DTS cycles in boundary rounds, in updates; iterations; blocks; Newton its
#endif
};
// development probes (-DEIS_PHASE_CLOCK): clock64 at step start (0), arrivals of the solver
// warp (1, 3) and of warp 0 (2, 4) at barriers A and B, step end (5), S4 start/end (6, 7).
// (Reads right after a barrier may issue before the barrier completes, so arrivals are used.)
#ifdef EIS_PHASE_CLOCK
#define EIS_TCLK(i) do { if (threadIdx.x == 0) sh.tclk[i] = clock64(); } while (0)
#define EIS_ARRIVE(i) do { if ((threadIdx.x & 31) == 0) { if (warp == SW) sh.tclk[i] = clock64(); if (warp == 0) sh.tclk[(i) + 1] = clock64(); } } while (0)
#else
#define EIS_TCLK(i) do { } while (0)
#define EIS_ARRIVE(i) do { } while (0)
#endif
#ifdef EIS_FINE_CLOCK
#define EIS_FCLK(i) do { if (threadIdx.x == 0) sh.fclk[i] = clock64(); } while (0)
#else
#define EIS_FCLK(i) do { } while (0)
#endif

__device__ __forceinline__ void set_status(CtaShared& sh, int code) { atomicCAS(&sh.status, 0, code); }

// warp reductions with compare-selects (finite values; a NaN state has already set a status)
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) { const double w = __shfl_xor_sync(0xffffffffu, v, o); v = w > v ? w : v; }
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) { const double w = __shfl_xor_sync(0xffffffffu, v, o); v = w < v ? w : v; }
  return v;
}

__device__ __forceinline__ const Ifc* find_ifc(const CtaShared& sh, int e) {
  for (int k = 0; k < sh.nifc; ++k)
    if (sh.ifc[k].e == e) return &sh.ifc[k];
  return nullptr;
}
__device__ __forceinline__ const Trg* find_trg(const CtaShared& sh, int ntrg, int e) {
  for (int k = 0; k < ntrg; ++k)
    if (sh.trg[k].e == e) return &sh.trg[k];
  return nullptr;
}
__device__ __forceinline__ bool created_at(const CtaShared& sh, int ntrg, int e) {
  const Trg* t = ntrg ? find_trg(sh, ntrg, e) : nullptr;
  return t && t->acc;
}

// tiny / region predicates straight from the shared state (R4, R10, R11); used off the hot
// path only (creation eligibility, R16)
__device__ __forceinline__ bool tiny_at(const Eos& e, const Prm& p, const double* rho, const double* h, int n, int i) {
  if (i < 0 || i >= n) return false;
  if (!(h[i] < p.eps_tiny * p.h_av)) return false;
  const int ph = phase_of(e, rho[i]);
  if (i > 0 && phase_of(e, rho[i - 1]) == ph) return false;
  if (i < n - 1 && phase_of(e, rho[i + 1]) == ph) return false;
  return true;
}
__device__ __forceinline__ bool region_at(const Eos& e, const Prm& p, const double* rho, const double* h, int n, int i) {
  return p.mode != 1 && (tiny_at(e, p, rho, h, n, i - 1) || tiny_at(e, p, rho, h, n, i) || tiny_at(e, p, rho, h, n, i + 1));
}

// moving-cell update: h^{n+1} = h + (wR - wL) dt, U^{n+1} = (h/h^{n+1}) U - (dt/h^{n+1}) dF
__device__ __forceinline__ int cell_update(double* rho, double* mom, double* h, int i, double FL0, double FL1,
                                           double wL, double FR0, double FR1, double wR, double dt, const Prm& p,
                                           int& remesh, int& marg) {
  const double hn = h[i];
  const double hn1 = __dadd_rn(hn, __dmul_rn(wR - wL, dt));  // no contraction: the oracle's roundings
  if (!(hn1 > 0.0)) return ST_WIDTH;
  if (hn1 != hn && (width_marginal(hn1, p.eps_tiny * p.h_av) || width_marginal(hn1, p.eps_split * p.h_av))) marg = 1;
  const double q = hn / hn1, c = dt / hn1;
  rho[i] = q * rho[i] - c * (FR0 - FL0);
  mom[i] = q * mom[i] - c * (FR1 - FL1);
  h[i] = hn1;
  if (hn1 < p.eps_tiny * p.h_av || hn1 > p.eps_split * p.h_av) remesh = 1;
  return 0;
}

// flux and speed of edge `ed` seen from the cell on side `right_cell` (0: the cell left of the
// edge, 1: the one right of it): accepted creation, explicit phase boundary, or the HLL arrays.
__device__ __forceinline__ void edge_view(const CtaShared& sh, const uint8_t* fl, const double* F0, const double* F1,
                                          int ed, int right_cell, double& G0, double& G1, double& w) {
  if (fl[ed] & F_SPEC) {
    const Ifc* s = find_ifc(sh, ed);
    if (s) { G0 = s->F0; G1 = s->F1; w = s->w; return; }
  }
  const int ntrg = sh.ntrg < MAXTRG ? sh.ntrg : MAXTRG;
  if (ntrg) {
    const Trg* t = find_trg(sh, ntrg, ed);
    if (t && t->acc) {
      if (right_cell) { G0 = t->Fr0; G1 = t->Fr1; w = t->wr; }
      else { G0 = t->Fl0; G1 = t->Fl1; w = t->wl; }
      return;
    }
  }
  G0 = F0[ed]; G1 = F1[ed]; w = 0.0;
}

// remesh: position shift of old cell i (cells before it: created cells, merge groups, splits)
__device__ __forceinline__ int remesh_shift(const CtaShared& sh, int ntrg, int i) {
  int s = 0;
  for (int k = 0; k < ntrg; ++k)
    if (sh.trg[k].acc && sh.trg[k].e <= i) s += 1;  // created cell inserted before cell e
  for (int k = 0; k < sh.ngrp; ++k) {
    const Grp& g = sh.grp[k];
    if (g.g1 < i) s += g.split - (g.g1 - g.g0);
  }
  return s;
}

// ------------------------------------------------------------------------------------------
// Algorithm 2 on one implicit block [a, b] by one warp (
// R11-R13).  Interior boundaries are solved by the two half warps in parallel, each warm-started
// from its previous iterate; cell updates by lanes 0..K-1; residual (R8) by warp max.
// Outer fluxes F_left, F_right are the explicit step's (flux bounding).
// ------------------------------------------------------------------------------------------
// the isothermal two-phase system for the generic loop (eis_dts.cuh): interior edges are phase
// boundaries (Appendix-A solve by the half warp, warm-started from the previous iterate) or HLL
// (P:1103); phases are those of U^n (an iterate leaving its phase is ST_SPINODAL, R27)
struct TwoPhaseDts {
  static constexpr int NV = 2;
  // past the loop's scratch (W at offset 0): star pressures of the interior boundaries (warm
  // starts) xs0, xs1 [MAXB + 1] and the iterate's velocities Wu [MAXB] (one division per cell)
  static constexpr int XS0 = dts_scratch<2>(), XS1 = XS0 + MAXB + 1, WU = XS1 + MAXB + 1;
  const Eos& e;
  const Prm& p;
  unsigned vapm, liqm;
  int solves;
  __device__ __forceinline__ int phase_n(int c) const { return (vapm >> c & 1u) ? VAP : ((liqm >> c & 1u) ? LIQ : SPIN); }
  __device__ __forceinline__ int edge(int j, double* W, double* Fe, double* we, int half, int hl, unsigned hmask) {
    const double rl = W[j - 1], ml = W[MAXB + j - 1], rr = W[j], mr = W[MAXB + j], ul = W[WU + j - 1], ur = W[WU + j];
    const int pl = phase_n(j - 1), pr = phase_n(j);  // phases of U^n
    int err = 0;
    if (pl != pr) {
      IfaceSol s = iface_solve_hw(e, p, rl, ul, rr, ur, pl == VAP, W[XS0 + j], W[XS1 + j], hmask, hl, half * 16);
      if (hl == 0) {
        if (s.iters < 0) err = ST_NEWTON;
        Fe[j] = s.F0; Fe[MAXB + 1 + j] = s.F1; we[j] = s.w; W[XS0 + j] = s.pV; W[XS1 + j] = s.pL;
        ++solves;
      }
    } else if (hl == 0) {
      hll(e, pl, rl, ml, ul, rr, mr, ur, Fe[j], Fe[MAXB + 1 + j]);
      we[j] = 0.0;
    }
    return err;
  }
  __device__ __forceinline__ int check(int lane, const double (&w)[2]) const {
    return (!(w[0] > 0.0) || phase_of(e, w[0]) != phase_n(lane)) ? ST_SPINODAL : 0;
  }
  __device__ __forceinline__ void store(double* W, int lane, const double (&w)[2]) { W[WU + lane] = w[1] / w[0]; }
};
static_assert(dts_scratch<2>() + 3 * MAXB + 2 <= DTS_SCRATCH, "dts scratch");

__device__ __noinline__ int dts_block(const Eos& e, const Prm& p, CtaShared& sh, double* rho, double* mom, double* h,
                                      const double* F0, const double* F1, const uint8_t* fl, int a, int b, double dt,
                                      long long& it_out, long long& solves, int& remesh, int& marg) {
  const int lane = threadIdx.x & 31;
  const int K = b - a + 1;
  double* sc = sh.dts;
  double* Fe = sc + 2 * MAXB;
  double* we = Fe + 2 * (MAXB + 1);
  if (lane == 0) {  // outer edges: the explicit step's fluxes and speeds
    double g0, g1, w;
    edge_view(sh, fl, F0, F1, a, 1, g0, g1, w);
    Fe[0] = g0; Fe[MAXB + 1] = g1; we[0] = w;
    edge_view(sh, fl, F0, F1, b + 1, 0, g0, g1, w);
    Fe[K] = g0; Fe[MAXB + 1 + K] = g1; we[K] = w;
  }
  if (lane >= 1 && lane < K) {  // warm start of interior boundaries from the last step
    const Ifc* s = find_ifc(sh, a + lane);
    sc[TwoPhaseDts::XS0 + lane] = s ? s->pV : -1.0;
    sc[TwoPhaseDts::XS1 + lane] = s ? s->pL : -1.0;
  }
  DtsCell<2> c{};
  int ph0 = SPIN;
  if (lane < K) {
    c.un[0] = rho[a + lane]; c.un[1] = mom[a + lane]; c.hn = h[a + lane];
    const bool tin = fl[a + lane] & F_TINY;
    ph0 = phase_of(e, c.un[0]);
    c.theta = tin ? c.hn / p.h_av : p.theta_nb;  // theta_k = alpha = h_k^n / h_av (R12)
    c.tol = tin ? p.tol_tiny : p.tol_nb;
  }
  TwoPhaseDts S{e, p, __ballot_sync(0xffffffffu, lane < K && ph0 == VAP), __ballot_sync(0xffffffffu, lane < K && ph0 == LIQ), 0};
  double u1[2] = {0.0, 0.0}, hn1 = 0.0;
  const int err = dts_warp(S, sc, K, dt, p.dts_max_iter, c, u1, hn1, it_out, marg);
  solves += S.solves;
  bool wm = false;  // width decision margin of this lane's cell
  if (!err && lane < K) {
    wm = hn1 != c.hn && (width_marginal(hn1, p.eps_tiny * p.h_av) || width_marginal(hn1, p.eps_split * p.h_av));
    rho[a + lane] = u1[0]; mom[a + lane] = u1[1]; h[a + lane] = hn1;
    if (hn1 < p.eps_tiny * p.h_av || hn1 > p.eps_split * p.h_av) remesh = 1;
  }
  marg += __popc(__ballot_sync(0xffffffffu, wm));
  if (lane >= 1 && lane < K && !err) {  // keep the converged boundary states for the next step
    Ifc* s = const_cast<Ifc*>(find_ifc(sh, a + lane));
    if (s) { s->pV = sc[TwoPhaseDts::XS0 + lane]; s->pL = sc[TwoPhaseDts::XS1 + lane]; }
  }
  __syncwarp();
  return err;
}

// The same system for the per-thread loop (dts_thread): one lane owns a whole block; the
// boundary solver runs on that lane (iface_solve_t, the half warp's iteration in one thread).
template <int KMAX>
struct TwoPhaseDtsT {
  static constexpr int NV = 2;
  const Eos& e;
  const Prm& p;
  unsigned vapm, liqm;  // phases of U^n by cell
  int solves;
  double xs0[KMAX + 1], xs1[KMAX + 1];  // star pressures of the interior boundaries (warm starts)
  double Wu[KMAX];                      // velocities of the iterate
  __device__ __forceinline__ int phase_n(int c) const { return (vapm >> c & 1u) ? VAP : ((liqm >> c & 1u) ? LIQ : SPIN); }
  __device__ __forceinline__ int edge(int j, const double (&Wl)[2], const double (&Wr)[2], double (&F)[2], double& w) {
    const int pl = phase_n(j - 1), pr = phase_n(j);
    if (pl != pr) {
      IfaceSol s = iface_solve_t(e, p, Wl[0], Wu[j - 1], Wr[0], Wu[j], pl == VAP, xs0[j], xs1[j]);
      F[0] = s.F0; F[1] = s.F1; w = s.w; xs0[j] = s.pV; xs1[j] = s.pL;
      ++solves;
      return s.iters < 0 ? ST_NEWTON : 0;
    }
    hll(e, pl, Wl[0], Wl[1], Wu[j - 1], Wr[0], Wr[1], Wu[j], F[0], F[1]);
    w = 0.0;
    return 0;
  }
  __device__ __forceinline__ int check(int i, const double (&w)[2]) const {
    return (!(w[0] > 0.0) || phase_of(e, w[0]) != phase_n(i)) ? ST_SPINODAL : 0;
  }
  __device__ __forceinline__ void store(int i, const double (&w)[2]) { Wu[i] = w[1] / w[0]; }
  __device__ __forceinline__ void put(int j, const IfaceSol& s, double (&F)[2], double& w) {
    F[0] = s.F0; F[1] = s.F1; w = s.w; xs0[j] = s.pV; xs1[j] = s.pL;
    ++solves;
  }
  // all interior edges; the usual 3-cell block around a tiny cell of the other phase has two
  // warm-started boundary solves, tried first as one-evaluation R14d steps side by side (the two
  // evaluations overlap); any that is not accepted takes the general solver (same bits)
  __device__ __forceinline__ int edges(int K, const double (&W)[KMAX][2], double (&Fe)[KMAX + 1][2], double (&we)[KMAX + 1]) {
    if (KMAX == 3 && K == 3 && phase_n(0) != phase_n(1) && phase_n(1) != phase_n(2) && xs0[1] > 0.0 && xs0[2] > 0.0) {
      IfaceSol s1, s2;
      const bool ok1 = iface_try_lin(e, p, W[0][0], Wu[0], W[1][0], Wu[1], phase_n(0) == VAP, xs0[1], xs1[1], s1);
      const bool ok2 = iface_try_lin(e, p, W[1][0], Wu[1], W[2][0], Wu[2], phase_n(1) == VAP, xs0[2], xs1[2], s2);
      int err = 0;
      if (ok1) put(1, s1, Fe[1], we[1]);
      else err = max(err, edge(1, W[0], W[1], Fe[1], we[1]));
      if (ok2) put(2, s2, Fe[2], we[2]);
      else err = max(err, edge(2, W[1], W[2], Fe[2], we[2]));
      return err;
    }
    int err = 0;
#pragma unroll
    for (int j = 1; j < KMAX; ++j)
      if (j < K) err = max(err, edge(j, W[j - 1], W[j], Fe[j], we[j]));
    return err;
  }
};

// one DTS job by this thread: U^n, h^n, outer edges and warm starts from the record, results
// (U^{n+1}, h^{n+1}, converged boundary states, counts, status) back into it
template <int KMAX>
__device__ __forceinline__ void run_dts_job(const Eos& e, const Prm& p, DtsJob& J) {
  const int K = J.K;
  DtsCell<2> c[KMAX];
  double Fe[KMAX + 1][2], we[KMAX + 1], u1[KMAX][2], h1[KMAX];
  TwoPhaseDtsT<KMAX> S{e, p, 0u, 0u, 0};
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    c[i].un[0] = c[i].un[1] = 0.0; c[i].hn = 1.0; c[i].theta = 1.0; c[i].tol = 1.0;
    if (i < K) {
      c[i].un[0] = J.un[i][0]; c[i].un[1] = J.un[i][1]; c[i].hn = J.hn[i];
      const bool tin = (J.tiny >> i) & 1;
      c[i].theta = tin ? c[i].hn / p.h_av : p.theta_nb;  // theta_k = alpha = h_k^n / h_av (R12)
      c[i].tol = tin ? p.tol_tiny : p.tol_nb;
      const int ph = phase_of(e, c[i].un[0]);
      S.vapm |= (ph == VAP ? 1u : 0u) << i;
      S.liqm |= (ph == LIQ ? 1u : 0u) << i;
    }
  }
#pragma unroll
  for (int j = 0; j <= KMAX; ++j) {
    we[j] = 0.0; Fe[j][0] = Fe[j][1] = 0.0;
    S.xs0[j] = (j >= 1 && j < K) ? J.xs[j][0] : -1.0;
    S.xs1[j] = (j >= 1 && j < K) ? J.xs[j][1] : -1.0;
    if (j == 0) { Fe[0][0] = J.Fo[0][0]; Fe[0][1] = J.Fo[0][1]; we[0] = J.wo[0]; }
    if (j == K) { Fe[j][0] = J.Fo[1][0]; Fe[j][1] = J.Fo[1][1]; we[j] = J.wo[1]; }
  }
  long long it = 0;
  int marg = 0;
  const int err = dts_thread<TwoPhaseDtsT<KMAX>, KMAX>(S, K, J.dt, p.dts_max_iter, c, Fe, we, u1, h1, it, marg);
  J.it = it; J.solves = S.solves; J.status = err; J.marg = marg;
  if (err) return;
#pragma unroll
  for (int i = 0; i < KMAX; ++i)
    if (i < K) { J.un[i][0] = u1[i][0]; J.un[i][1] = u1[i][1]; J.hn[i] = h1[i]; }
#pragma unroll
  for (int j = 1; j < KMAX; ++j)
    if (j < K) { J.xs[j][0] = S.xs0[j]; J.xs[j][1] = S.xs1[j]; }
}

// ------------------------------------------------------------------------------------------
// Mode NEWTON (readings N1-N5): Algorithm 2's implicit system W = T(W) on the
// block [a, b] by a chord Newton iteration, one warp.  Lane i < K owns cell i: its state X_i,
// T_i(X), U_i^n and its row of the block-tridiagonal Jacobian of R = X - T (2x2 blocks L_i, D_i,
// U_i), built by forward differences: perturbing one unknown of cell j changes only edges j and
// j+1, which the two half warps re-solve in one round (warm-started from the base solution);
// lanes j-1, j, j+1 then form their column entries.  The linear solve is a block Thomas sweep
// across the lanes (2x2 inverses, shuffles).  Same blocks, outer fluxes and Part 2 as dts_block.
// ------------------------------------------------------------------------------------------
struct NtRow {  // lane i's row of the block-tridiagonal Jacobian
  double L[4], D[4], U[4];  // row-major 2x2
};

__device__ __forceinline__ void nt_set_col(double (&B)[4], int c, double v0, double v1) {
  if (c == 0) { B[0] = v0; B[2] = v1; } else { B[1] = v0; B[3] = v1; }
}

// T_i from the edge values left (g0l, g1l, wl) and right (g0r, g1r, wr) of cell i
__device__ __forceinline__ bool nt_T(double rn0, double rn1, double hn, double dt, double g0l, double g1l, double wl,
                                     double g0r, double g1r, double wr, double& t0, double& t1) {
  const double hl = __dadd_rn(hn, __dmul_rn(wr - wl, dt));
  if (!(hl > 0.0)) return false;
  t0 = (hn / hl) * rn0 - (dt / hl) * (g0r - g0l);
  t1 = (hn / hl) * rn1 - (dt / hl) * (g1r - g1l);
  return true;
}

// flux of the edge between cells (rl, ml) and (rr, mr) of phases pl, pr (of U^n) by a half warp;
// returns false if the boundary solve failed.  x0/x1: warm start in, root out (interface edges).
__device__ __forceinline__ bool nt_edge(const Eos& e, const Prm& p, double rl, double ml, double rr, double mr, int pl,
                                        int pr, double& x0, double& x1, unsigned hmask, int hl, int half, double& F0,
                                        double& F1, double& w, long long& solves) {
  if (pl != pr) {
    IfaceSol s = iface_solve_hw(e, p, rl, ml / rl, rr, mr / rr, pl == VAP, x0, x1, hmask, hl, half * 16);
    F0 = s.F0; F1 = s.F1; w = s.w; x0 = s.pV; x1 = s.pL;
    if (hl == 0) ++solves;
    return s.iters >= 0;
  }
  hll(e, pl, rl, ml, ml / rl, rr, mr, mr / rr, F0, F1);
  w = 0.0;
  return true;
}

__device__ __noinline__ int newton_block(const Eos& e, const Prm& p, CtaShared& sh, double* rho, double* mom, double* h,
                                         const double* F0, const double* F1, const uint8_t* fl, int a, int b, double dt,
                                         long long& it_out, long long& solves, int& remesh) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  const int K = b - a + 1;
  double* sc = sh.dts;
  double* W0 = sc;               // [MAXB] the current iterate X (broadcast for the edge solves)
  double* W1 = sc + MAXB;
  double* Fe0 = sc + 2 * MAXB;   // [MAXB+1] edge values at X (edges 0 and K: the outer fluxes)
  double* Fe1 = Fe0 + MAXB + 1;
  double* we = Fe1 + MAXB + 1;
  double* xs0 = we + MAXB + 1;   // warm starts of the interface edges
  double* xs1 = xs0 + MAXB + 1;
  if (lane == 0) {
    double g0, g1, w;
    edge_view(sh, fl, F0, F1, a, 1, g0, g1, w);
    Fe0[0] = g0; Fe1[0] = g1; we[0] = w;
    edge_view(sh, fl, F0, F1, b + 1, 0, g0, g1, w);
    Fe0[K] = g0; Fe1[K] = g1; we[K] = w;
  }
  if (lane >= 1 && lane < K) {
    const Ifc* s = find_ifc(sh, a + lane);
    xs0[lane] = s ? s->pV : -1.0;
    xs1[lane] = s ? s->pL : -1.0;
  }
  double rn0 = 1.0, rn1 = 0.0, hn = 1.0, X0 = 1.0, X1 = 0.0, T0 = 0.0, T1 = 0.0;
  int ph0 = 0;
  if (lane < K) {
    rn0 = rho[a + lane]; rn1 = mom[a + lane]; hn = h[a + lane];
    ph0 = phase_of(e, rn0);
    X0 = rn0; X1 = rn1;
    W0[lane] = X0; W1[lane] = X1;
  }
  __syncwarp();
  int err = 0;
  long long evals = 0;
  // edges 1..K-1 at X (two per round), then T_i on lanes i < K
  auto eval_T = [&]() {
    for (int j0 = 1; j0 < K; j0 += 2) {
      const int j = j0 + half;
      if (j < K) {
        double x0 = xs0[j], x1 = xs1[j], g0, g1, w;
        const bool ok = nt_edge(e, p, W0[j - 1], W1[j - 1], W0[j], W1[j], phase_of(e, rho[a + j - 1]),
                                phase_of(e, rho[a + j]), x0, x1, hmask, hl, half, g0, g1, w, solves);
        if (hl == 0) {
          if (!ok) err = ST_NEWTON;
          Fe0[j] = g0; Fe1[j] = g1; we[j] = w; xs0[j] = x0; xs1[j] = x1;
        }
      }
      __syncwarp();
    }
    err = __reduce_max_sync(FULL, err);
    if (!err && lane < K && !nt_T(rn0, rn1, hn, dt, Fe0[lane], Fe1[lane], we[lane], Fe0[lane + 1], Fe1[lane + 1],
                                  we[lane + 1], T0, T1))
      err = ST_WIDTH;
    err = __reduce_max_sync(FULL, err);
    ++evals;
  };
  NtRow J;
  for (int q = 0; q < 4; ++q) { J.L[q] = 0.0; J.D[q] = 0.0; J.U[q] = 0.0; }
  // forward-difference Jacobian of R = X - T at X (N2): one round per unknown (j, c)
  auto jacobian = [&]() {
    for (int j = 0; j < K && !err; ++j) {
      for (int c = 0; c < 2 && !err; ++c) {
        const double xq = __shfl_sync(FULL, c == 0 ? X0 : X1, j);
        const double eps = 1e-7 * fmax(fabs(xq), 1.0);
        const double pj0 = W0[j] + (c == 0 ? eps : 0.0), pj1 = W1[j] + (c == 1 ? eps : 0.0);
        // half 0: edge j (cells j-1 | j'), half 1: edge j+1 (cells j' | j+1)
        const int ed = j + half;
        double g0 = 0.0, g1 = 0.0, w = 0.0;
        bool ok = true;
        if (ed >= 1 && ed < K) {
          double x0 = xs0[ed], x1 = xs1[ed];
          const double rl = half ? pj0 : W0[j - 1], ml = half ? pj1 : W1[j - 1];
          const double rr = half ? W0[j + 1] : pj0, mr = half ? W1[j + 1] : pj1;
          ok = nt_edge(e, p, rl, ml, rr, mr, phase_of(e, rho[a + ed - 1]), phase_of(e, rho[a + ed]), x0, x1, hmask, hl,
                       half, g0, g1, w, solves);
        }
        err = __reduce_max_sync(FULL, ok ? 0 : ST_NEWTON);
        if (err) break;
        // perturbed edge j from lane 0 (half 0), edge j+1 from lane 16 (half 1); outer edges fixed
        double pl0 = __shfl_sync(FULL, g0, 0), pl1 = __shfl_sync(FULL, g1, 0), plw = __shfl_sync(FULL, w, 0);
        double pr0 = __shfl_sync(FULL, g0, 16), pr1 = __shfl_sync(FULL, g1, 16), prw = __shfl_sync(FULL, w, 16);
        if (j == 0) { pl0 = Fe0[0]; pl1 = Fe1[0]; plw = we[0]; }
        if (j == K - 1) { pr0 = Fe0[K]; pr1 = Fe1[K]; prw = we[K]; }
        double t0, t1;
        bool okT = true;
        if (lane == j - 1) {  // row j-1: edges j-1 (base), j (perturbed) -> U block
          okT = nt_T(rn0, rn1, hn, dt, Fe0[lane], Fe1[lane], we[lane], pl0, pl1, plw, t0, t1);
          nt_set_col(J.U, c, -(t0 - T0) / eps, -(t1 - T1) / eps);
        } else if (lane == j) {  // row j: both perturbed edges -> D block
          okT = nt_T(rn0, rn1, hn, dt, pl0, pl1, plw, pr0, pr1, prw, t0, t1);
          nt_set_col(J.D, c, (c == 0 ? 1.0 : 0.0) - (t0 - T0) / eps, (c == 1 ? 1.0 : 0.0) - (t1 - T1) / eps);
        } else if (lane == j + 1 && lane < K) {  // row j+1: edges j+1 (perturbed), j+2 (base) -> L block
          okT = nt_T(rn0, rn1, hn, dt, pr0, pr1, prw, Fe0[lane + 1], Fe1[lane + 1], we[lane + 1], t0, t1);
          nt_set_col(J.L, c, -(t0 - T0) / eps, -(t1 - T1) / eps);
        }
        err = __reduce_max_sync(FULL, okT ? 0 : ST_WIDTH);
      }
    }
    evals += 2 * K;
  };
  eval_T();
  if (!err) jacobian();
  double prev = INFINITY;
  for (long long it = 1; !err; ++it) {
    if (it > p.dts_max_iter) { err = ST_DTS_CAP; break; }
    // block Thomas on J d = -(X - T): forward sweep (lane i receives lane i-1's D'^-1 U and D'^-1 r')
    double Dp[4] = {J.D[0], J.D[1], J.D[2], J.D[3]};
    double r0 = -(X0 - T0), r1 = -(X1 - T1);
    double M[4] = {0.0, 0.0, 0.0, 0.0}, y0 = 0.0, y1 = 0.0;
    bool sing = false;
    for (int i = 0; i < K; ++i) {
      if (lane == i) {  // finish row i: D'_i^-1 U_i and D'_i^-1 r'_i
        const double det = Dp[0] * Dp[3] - Dp[1] * Dp[2];
        if (!(fabs(det) > 0.0) || !isfinite(det)) sing = true;
        const double id = 1.0 / det;
        const double I0 = Dp[3] * id, I1 = -Dp[1] * id, I2 = -Dp[2] * id, I3 = Dp[0] * id;
        M[0] = I0 * J.U[0] + I1 * J.U[2]; M[1] = I0 * J.U[1] + I1 * J.U[3];
        M[2] = I2 * J.U[0] + I3 * J.U[2]; M[3] = I2 * J.U[1] + I3 * J.U[3];
        y0 = I0 * r0 + I1 * r1; y1 = I2 * r0 + I3 * r1;
      }
      if (i + 1 < K) {
        const double m0 = __shfl_sync(FULL, M[0], i), m1 = __shfl_sync(FULL, M[1], i);
        const double m2 = __shfl_sync(FULL, M[2], i), m3 = __shfl_sync(FULL, M[3], i);
        const double q0 = __shfl_sync(FULL, y0, i), q1 = __shfl_sync(FULL, y1, i);
        if (lane == i + 1) {  // D'_{i+1} = D - L M, r' = r - L y
          Dp[0] -= J.L[0] * m0 + J.L[1] * m2; Dp[1] -= J.L[0] * m1 + J.L[1] * m3;
          Dp[2] -= J.L[2] * m0 + J.L[3] * m2; Dp[3] -= J.L[2] * m1 + J.L[3] * m3;
          r0 -= J.L[0] * q0 + J.L[1] * q1; r1 -= J.L[2] * q0 + J.L[3] * q1;
        }
      }
    }
    if (__any_sync(FULL, sing)) { err = ST_NEWTON; break; }
    double d0 = y0, d1 = y1;  // back substitution: d_i = y_i - M_i d_{i+1}
    for (int i = K - 2; i >= 0; --i) {
      const double n0 = __shfl_sync(FULL, d0, i + 1), n1 = __shfl_sync(FULL, d1, i + 1);
      if (lane == i) { d0 = y0 - (M[0] * n0 + M[1] * n1); d1 = y1 - (M[2] * n0 + M[3] * n1); }
    }
    double step = 0.0;
    bool bad = false;
    if (lane < K) {
      X0 += d0; X1 += d1;
      step = fmax(fabs(d0) / fmax(fabs(X0), 1.0), fabs(d1) / fmax(fabs(X1), 1.0));
      W0[lane] = X0; W1[lane] = X1;
      bad = !(X0 > 0.0) || phase_of(e, X0) != ph0;
    }
    step = warp_max(step);
    __syncwarp();
    if (__any_sync(FULL, bad)) { err = ST_SPINODAL; break; }
    if (step <= 1e-10 || (it >= 2 && step >= 0.5 * prev)) break;  // N3
    prev = step;
    eval_T();
    if (err) break;
    if (it % 8 == 0) jacobian();
  }
  if (!err) {  // Part 2: fluxes at U* = X and the conservative update
    eval_T();
    --evals;  // Part 2's edge fluxes are not an iteration (as the oracle counts)
  }
  if (!err && lane < K) {
    const double hn1 = __dadd_rn(hn, __dmul_rn(we[lane + 1] - we[lane], dt));
    if (!(hn1 > 0.0)) err = ST_WIDTH;
    else {
      rho[a + lane] = (hn / hn1) * rn0 - (dt / hn1) * (Fe0[lane + 1] - Fe0[lane]);
      mom[a + lane] = (hn / hn1) * rn1 - (dt / hn1) * (Fe1[lane + 1] - Fe1[lane]);
      h[a + lane] = hn1;
      if (hn1 < p.eps_tiny * p.h_av || hn1 > p.eps_split * p.h_av) remesh = 1;
    }
  }
  if (lane >= 1 && lane < K && !err) {  // keep the converged boundary states for the next step
    Ifc* s = const_cast<Ifc*>(find_ifc(sh, a + lane));
    if (s) { s->pV = xs0[lane]; s->pL = xs1[lane]; }
  }
  err = __reduce_max_sync(FULL, err);
  __syncwarp();
  it_out = evals;
  return err;
}

// ------------------------------------------------------------------------------------------
// Explicit local time stepping (mode LTS, the paper's comparison method, the
// disabled passage P:1068-1091, readings R29-R31) on one implicit block [a, b] by one warp: the
// tiny cells advance with 2^n0 sub-steps of dtau = dt / 2^n0 (dtau <= C_CFL h_T / S_max, R29),
// the other block cells stay at U^n meanwhile; fluxes at the edges next to a tiny cell from the
// current sub-step states (the two half warps solve two boundaries at a time, warm-started from
// the previous sub-step), moving small-cell update, time averages of the fluxes
// and boundary speeds for the large cells (R30), which then take the large step.  The same
// order of operations and accumulation as the oracle's lts_block.
// ------------------------------------------------------------------------------------------
__device__ __noinline__ int lts_block(const Eos& e, const Prm& p, CtaShared& sh, double* rho, double* mom, double* h,
                                      const double* F0, const double* F1, const uint8_t* fl, int a, int b, double dt,
                                      double smax, long long& it_out, long long& solves, int& remesh) {
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  const int K = b - a + 1;
  double* sc = sh.dts;
  double* W0 = sc;               // [MAXB] sub-step states (tiny cells) / U^n (others)
  double* W1 = sc + MAXB;        // [MAXB]
  double* Fe0 = sc + 2 * MAXB;   // [MAXB+1] current edge fluxes
  double* Fe1 = Fe0 + MAXB + 1;
  double* we = Fe1 + MAXB + 1;
  double* xs0 = we + MAXB + 1;   // warm starts of the boundary solves
  double* xs1 = xs0 + MAXB + 1;
  double fb0 = 0.0, fb1 = 0.0, wbar = 0.0;  // lane j: averages at edge j (R30)
  if (lane == 0) {
    double g0, g1, w;
    edge_view(sh, fl, F0, F1, a, 1, g0, g1, w);
    Fe0[0] = g0; Fe1[0] = g1; we[0] = w;
    edge_view(sh, fl, F0, F1, b + 1, 0, g0, g1, w);
    Fe0[K] = g0; Fe1[K] = g1; we[K] = w;
  }
  if (lane >= 1 && lane < K) {
    const Ifc* s = find_ifc(sh, a + lane);
    xs0[lane] = s ? s->pV : -1.0;
    xs1[lane] = s ? s->pL : -1.0;
  }
  double rn0 = 0, rn1 = 0, hn = 0, w0 = 0, w1 = 0, hw = 0;
  bool tin = false;
  int ph0 = 0;
  if (lane < K) {
    const uint8_t f = fl[a + lane];
    rn0 = rho[a + lane]; rn1 = mom[a + lane]; hn = h[a + lane];
    tin = f & F_TINY;
    ph0 = phase_of(e, rn0);
    w0 = rn0; w1 = rn1; hw = hn;
    W0[lane] = w0; W1[lane] = w1;
  }
  // R29: dtau = dt / 2^n0 <= C_CFL h_T / S_max
  const double hT = warp_min(lane < K && tin ? hn : INFINITY);
  double dtau = dt;
  int n0 = 0;
  while (dtau > p.cfl * hT / smax && n0 <= 62) { dtau *= 0.5; ++n0; }
  if (n0 > 62) { it_out = 0; return ST_DTS_CAP; }
  const long long ns = 1ll << n0;
  const double f = dtau / dt;
  // edge j (1 <= j < K) is sub-stepped iff next to a tiny cell; the others keep the U^n flux
  const unsigned tmask = __ballot_sync(0xffffffffu, lane < K && tin);
  auto sub_edge = [&](int j) { return j >= 1 && j < K && (((tmask >> (j - 1)) & 1u) || ((tmask >> j) & 1u)); };
  __syncwarp();
  int err = 0;
  for (int j0 = 1; j0 < K; j0 += 2) {  // constant interior fluxes (U^n) of edges not next to a tiny cell
    const int j = j0 + half;
    if (j < K && !sub_edge(j)) {
      const double rl = rho[a + j - 1], ml = mom[a + j - 1], rr = rho[a + j], mr = mom[a + j];
      const int pl = phase_of(e, rl), pr = phase_of(e, rr);
      if (pl != pr) {
        IfaceSol s = iface_solve_hw(e, p, rl, ml / rl, rr, mr / rr, pl == VAP, xs0[j], xs1[j], hmask, hl, half * 16);
        if (hl == 0) {
          if (s.iters < 0) err = ST_NEWTON;
          Fe0[j] = s.F0; Fe1[j] = s.F1; we[j] = s.w;
          ++solves;
        }
      } else if (hl == 0) {
        hll(e, pl, rl, ml, ml / rl, rr, mr, mr / rr, Fe0[j], Fe1[j]);
        we[j] = 0.0;
      }
    }
  }
  err = __reduce_max_sync(0xffffffffu, err);
  __syncwarp();
  long long nu = 0;
  for (; nu < ns && !err; ++nu) {
    for (int j0 = 1; j0 < K; j0 += 2) {  // fluxes at the current sub-step states
      const int j = j0 + half;
      if (j < K && sub_edge(j)) {
        const double rl = W0[j - 1], ml = W1[j - 1], rr = W0[j], mr = W1[j];
        const int pl = phase_of(e, rho[a + j - 1]), pr = phase_of(e, rho[a + j]);  // phases of U^n
        if (pl != pr) {
          IfaceSol s = iface_solve_hw(e, p, rl, ml / rl, rr, mr / rr, pl == VAP, xs0[j], xs1[j], hmask, hl, half * 16);
          if (hl == 0) {
            if (s.iters < 0) err = ST_NEWTON;
            Fe0[j] = s.F0; Fe1[j] = s.F1; we[j] = s.w; xs0[j] = s.pV; xs1[j] = s.pL;
            ++solves;
          }
        } else if (hl == 0) {
          hll(e, pl, rl, ml, ml / rl, rr, mr, mr / rr, Fe0[j], Fe1[j]);
          we[j] = 0.0;
        }
      }
    }
    err = __reduce_max_sync(0xffffffffu, err);
    __syncwarp();
    if (err) break;
    int bad = 0;
    if (lane < K && tin) {  // small-cell update
      const double hn1 = __dadd_rn(hw, __dmul_rn(we[lane + 1] - we[lane], dtau));
      if (!(hn1 > 0.0)) bad = ST_WIDTH;
      w0 = (hw / hn1) * w0 - (dtau / hn1) * (Fe0[lane + 1] - Fe0[lane]);
      w1 = (hw / hn1) * w1 - (dtau / hn1) * (Fe1[lane + 1] - Fe1[lane]);
      hw = hn1;
      if (!(w0 > 0.0) || phase_of(e, w0) != ph0) bad = bad ? bad : ST_SPINODAL;
    }
    if (sub_edge(lane)) { fb0 += f * Fe0[lane]; fb1 += f * Fe1[lane]; wbar += f * we[lane]; }  // R30
    bad = __reduce_max_sync(0xffffffffu, bad);
    __syncwarp();
    if (lane < K && tin) { W0[lane] = w0; W1[lane] = w1; }
    __syncwarp();
    if (bad) { err = bad; break; }
  }
  // large step of the non-tiny block cells with the averaged fluxes at their sub-stepped edges
  if (sub_edge(lane)) { Fe0[lane] = fb0; Fe1[lane] = fb1; we[lane] = wbar; }
  __syncwarp();
  if (!err && lane < K) {
    if (tin) {
      rho[a + lane] = w0; mom[a + lane] = w1; h[a + lane] = hw;
      if (hw < p.eps_tiny * p.h_av || hw > p.eps_split * p.h_av) remesh = 1;
    } else {
      const double hn1 = __dadd_rn(hn, __dmul_rn(we[lane + 1] - we[lane], dt));
      if (!(hn1 > 0.0)) err = ST_WIDTH;
      else {
        rho[a + lane] = (hn / hn1) * rn0 - (dt / hn1) * (Fe0[lane + 1] - Fe0[lane]);
        mom[a + lane] = (hn / hn1) * rn1 - (dt / hn1) * (Fe1[lane + 1] - Fe1[lane]);
        h[a + lane] = hn1;
        if (hn1 < p.eps_tiny * p.h_av || hn1 > p.eps_split * p.h_av) remesh = 1;
      }
    }
  }
  if (lane >= 1 && lane < K && !err) {  // keep the last boundary states for the next step
    Ifc* s = const_cast<Ifc*>(find_ifc(sh, a + lane));
    if (s) { s->pV = xs0[lane]; s->pL = xs1[lane]; }
  }
  err = __reduce_max_sync(0xffffffffu, err);
  __syncwarp();
  it_out = nu;
  return err;
}

// ------------------------------------------------------------------------------------------
// Boundary list from a full scan (kernel start only): ordered ballot by the solver warp.
// ------------------------------------------------------------------------------------------
__device__ void build_boundary_list(const Eos& e, CtaShared& sh, const double* rho, uint8_t* fl, int n) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  int nif = 0;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int i = c0 + lane;
    const bool isif = i >= 1 && i < n && phase_of(e, rho[i - 1]) != phase_of(e, rho[i]);
    const unsigned mi = __ballot_sync(0xffffffffu, isif);
    if (isif) {
      const int k = nif + __popc(mi & lt_mask);
      if (k < MAXIF) { sh.ifc[k].e = i; fl[i] |= F_IF; }
      else set_status(sh, ST_CAPACITY);
    }
    nif += __popc(mi);
  }
  if (lane == 0) sh.nifc = nif < MAXIF ? nif : MAXIF;
  __syncwarp();
}

// ------------------------------------------------------------------------------------------
// One large step of one grid held in shared memory (the whole method, a1-a11), shared by the
// member-resident kernel (ensembles) and the tiled kernel (the single huge grid).  Z restricts
// error reporting, creation triggers and DTS blocks to the exactly-computed zone of a tile
// and records which output cells a tile owns after the remesh.  Returns dt, or -1 when the
// member stopped on an error.  All threads of the CTA call it.
// ------------------------------------------------------------------------------------------
struct Zone {
  int zlo, zhi;          // cells [zlo, zhi) are computed exactly (tiles: owned cells +- 2)
  int own_lo, own_hi;    // owned cells [own_lo, own_hi); owned edges (own_lo, own_hi]
  double dt_given;       // > 0: this dt (tiles: the global CFL step); else the grid's own CFL dt
  double s_given;        // > 0: the S_max of that step (tiles, LTS mode); else the grid's own
  bool left_real, right_real;  // the smem grid ends are domain ends (transmissive, R15)
  DtsJob* djobs = nullptr;     // window split (step_body<1>): blocks are exported as DTS jobs
  int* djn = nullptr;          //   job counter
  int djcap = 0;               //   job capacity
};
struct Arr {
  double *rho, *mom, *h, *F0, *F1, *X;
  uint8_t* fl;
  int n, C;
};

__device__ __forceinline__ void zone_status(CtaShared& sh, const Zone& Z, int i, int code) {
  if (i >= Z.zlo && i < Z.zhi) set_status(sh, code);
}
__device__ __forceinline__ void zone_status_e(CtaShared& sh, const Zone& Z, int ed, int code) {
  if ((ed - 1 >= Z.zlo && ed - 1 < Z.zhi) || (ed >= Z.zlo && ed < Z.zhi)) set_status(sh, code);
}

// ------------------------------------------------------------------------------------------
// Bulk pass P1 (own register allocation: the loop invariants stay in registers).
// window w: 32 CPL cells, CPL per lane, c_j = 31 CPL w - CPL + CPL l + j (lane 0 is the left
// halo; transmissive ghosts at the ends, R15); lane l >= 1 owns its CPL cells, the LEFT edge of
// its first cell and its internal edges: HLL flux (a3), creation trigger (a4), S_max / h_min
// partials (a2).  One reciprocal per cell (u = m/rho); the left neighbour's state arrives by
// shuffle.  Interior windows skip the ghost clamps.  Flagged cells are re-checked in full (rare).
// (EIS_P1_CPL: cells per lane, 2; 4 measured 5 % slower on C3 in round 2.)
// ------------------------------------------------------------------------------------------
#ifndef EIS_P1_CPL
#define EIS_P1_CPL 2
#endif
template <int CPL>
__device__ __forceinline__ void bulk_p1_t(const Eos& e_ref, const Prm& p_ref, CtaShared& sh, const Zone& Z,
                                          const double* __restrict__ rho, const double* __restrict__ mom,
                                          const double* __restrict__ h, double* __restrict__ F0, double* __restrict__ F1,
                                          const uint8_t* __restrict__ fl, int n, int warp, int nbulk, double* parts) {
  const Eos e = e_ref;  // constants into registers once (not a generic load per use)
  const double rho_tilde = e.rho_tilde, rho_min = e.rho_min, a_v2 = e.a_v2, a_l2 = e.a_l2, p0 = e.p0, rho0 = e.rho0;
  const double a_v = e.a_v, a_l = e.a_l, rmin2 = e.rho_min * e.rho_min, inv_rt = 1.0 / e.rho_tilde;
  const double eps_h = p_ref.eps_tiny * p_ref.h_av;
  const bool explicit_mode = p_ref.mode == 1;
  const int lane = threadIdx.x & 31;
  constexpr int WW = 31 * CPL;  // owned cells (and left edges) per window
  double s_part = 0.0, h_part = INFINITY;
  bool bad = false;      // a non-positive or spinodal density somewhere (reported below, rare)
  bool special = false;  // a trigger candidate or a phase change (handled below, rare)
  const int nwp = (n + WW) / WW;  // edges 0..n
  for (int w = warp; w < nwp; w += nbulk) {
    const int cb = WW * w - CPL + CPL * lane;  // this lane's first cell
    const bool interior_win = w > 0 && WW * w + WW < n;  // every cell of the window and its right neighbour exist
    double r[CPL], m[CPL], u[CPL], q[CPL], a[CPL];
    unsigned ph[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      int i = cb + j;
      if (!interior_win) i = i < 0 ? 0 : (i >= n ? n - 1 : i);
      r[j] = rho[i]; m[j] = mom[i];
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      u[j] = m[j] * rcp_fast(r[j]);
      const bool v = r[j] <= rho_tilde, l = r[j] >= rho_min;
      ph[j] = v ? 1u : (l ? 2u : 0u);
      q[j] = v ? a_v2 * r[j] : p0 + a_l2 * (r[j] - rho0);
      a[j] = v ? a_v : a_l;
    }
    const double rl = __shfl_up_sync(0xffffffffu, r[CPL - 1], 1), ml = __shfl_up_sync(0xffffffffu, m[CPL - 1], 1);
    const double ul = __shfl_up_sync(0xffffffffu, u[CPL - 1], 1), pl = __shfl_up_sync(0xffffffffu, q[CPL - 1], 1);
    const unsigned phl = __shfl_up_sync(0xffffffffu, ph[CPL - 1], 1);
    unsigned phr = __shfl_down_sync(0xffffffffu, ph[0], 1);
    if (lane == 31) {
      const int ir = cb + CPL;
      const double rr = rho[ir < n ? ir : n - 1];
      phr = rr <= rho_tilde ? 1u : (rr >= rho_min ? 2u : 0u);
    }
    if (lane >= 1) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) {  // cell c_j: S_max, h_min partials
        const int c = cb + j;
        if (c < n) {
          bad |= !(r[j] > 0.0) || ph[j] == 0u;
          const double su = fabs(u[j]) + a[j];
          s_part = su > s_part ? su : s_part;  // S over all cells (R5)
          const double hc = h[c];
          const bool same_l = j == 0 ? (c > 0 && phl == ph[0]) : ph[j - 1] == ph[j];
          const bool same_r = c + 1 < n && (j == CPL - 1 ? phr : ph[j + 1]) == ph[j];
          const bool tiny = hc < eps_h && !same_l && !same_r;
          const double hh = (explicit_mode || !tiny) ? hc : INFINITY;
          h_part = hh < h_part ? hh : h_part;  // h_min over non-tiny cells (R6)
        }
      }
      // creation pre-filters (R7), exact bounds with a 1e-9 m/s margin: liquid, both waves
      // rarefactions and ln y <= y - 1; vapour, both shocks and sqrt(rt r) <= rt, so
      // Phi(rt) >= du + a_v (2 - (r_L + r_R)/rt)
#pragma unroll
      for (int j = 0; j < CPL; ++j) {  // edge c_j between cells c_j - 1 and c_j
        const int c = cb + j;
        const double rL = j == 0 ? rl : r[j - 1], mL = j == 0 ? ml : m[j - 1];
        const double uL = j == 0 ? ul : u[j - 1], pL = j == 0 ? pl : q[j - 1];
        const unsigned phL = j == 0 ? phl : ph[j - 1];
        if (c <= n && phL == ph[j] && ph[j] != 0u) {
          double f0, f1;
          hll_fast(a[j], rL, mL, uL, pL, r[j], m[j], u[j], q[j], f0, f1);
          F0[c] = f0; F1[c] = f1;
          const double du = u[j] - uL, x = rL * r[j];
          const bool cand = ph[j] == 2u ? !(du * x <= a_l * (x - rmin2) - 1e-9 * x)
                                        : (du < -a_v * (2.0 - (rL + r[j]) * inv_rt) + 1e-9);
          special |= cand && c > 0 && c < n;
        } else if (c > 0 && c < n && phL != ph[j]) {
          special |= !(fl[c] & F_IF);  // a phase change must be a listed boundary
        }
      }
    }
  }
  parts[0] = s_part;
  parts[1] = h_part;
  if (__any_sync(0xffffffffu, bad || special)) {  // rare: redo this warp's cells and edges in full
    for (int w = warp; w < nwp; w += nbulk) {
      for (int qq = 0; qq < CPL; ++qq) {
        const int cj = WW * w - CPL + CPL * lane + qq;
        if (lane < 1 || cj >= n) continue;
        const double rc = rho[cj];
        const int pc = phase_of(e, rc);
        if (!(rc > 0.0)) zone_status(sh, Z, cj, ST_NONPOS);
        else if (pc == SPIN) zone_status(sh, Z, cj, ST_SPINODAL);
        if (cj < 1) continue;
        const double rL = rho[cj - 1];
        const int pL = phase_of(e, rL);
        if (pL == pc && pc != SPIN) {
          const double uc = mom[cj] / rc, uL = mom[cj - 1] / rL;
          bool marg = false;
          if (cj - 1 >= Z.zlo && cj < Z.zhi && !region_at(e, p_ref, rho, h, n, cj - 1) &&
              !region_at(e, p_ref, rho, h, n, cj) && creation_trigger(e, pc, rL, uL, rc, uc, marg)) {  // R16
            const int k = atomicAdd(&sh.ntrg, 1);
            if (k < MAXTRG) { sh.trg[k].e = cj; sh.trg[k].acc = 0; } else set_status(sh, ST_CAPACITY);
          }
          if (marg && Z.own_lo < cj && cj <= Z.own_hi) atomicAdd(&sh.c_margin, 1ull);  // owned edge
        } else if (pL != pc && !(fl[cj] & F_IF)) {
          zone_status_e(sh, Z, cj, ST_INTERNAL);  // a phase boundary missing from the list
        }
      }
    }
  }
}
__device__ __noinline__ void bulk_p1(const Eos& e_ref, const Prm& p_ref, CtaShared& sh, const Zone& Z,
                                     const double* __restrict__ rho, const double* __restrict__ mom,
                                     const double* __restrict__ h, double* __restrict__ F0, double* __restrict__ F1,
                                     const uint8_t* __restrict__ fl, int n, int warp, int nbulk, double* parts) {
  bulk_p1_t<EIS_P1_CPL>(e_ref, p_ref, sh, Z, rho, mom, h, F0, F1, fl, n, warp, nbulk, parts);
}

// Bulk pass P2: explicit update of the cells with two HLL edges (a7); h^{n+1} = h^n there, so
// h^n/h^{n+1} = 1 exactly and the update is U - (dt/h)(F_R - F_L).
__device__ __noinline__ void bulk_p2(const Prm& p, const CtaShared& sh, double* __restrict__ rho, double* __restrict__ mom,
                                     const double* __restrict__ h, const double* __restrict__ F0,
                                     const double* __restrict__ F1, const uint8_t* __restrict__ fl, int n, int warp,
                                     int nbulk, int ntrg, double dt, double dt_hav) {
  constexpr int U = 4;  // cells per lane per round, all loads first (shared-memory latency)
  const int lane = threadIdx.x & 31;
  const double h_av = p.h_av;
  for (int i0 = warp * 32 * U; i0 < n; i0 += nbulk * 32 * U) {
    double r[U], m[U], hn[U], a0[U], b0[U], a1[U], b1[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * 32 + lane, j = i < n ? i : 0;
      ok[u] = i < n && !((fl[j] & (F_REG | F_SPEC)) || (fl[j + 1] & F_SPEC));
      r[u] = rho[j]; m[u] = mom[j]; hn[u] = h[j];
      a0[u] = F0[j]; b0[u] = F0[j + 1]; a1[u] = F1[j]; b1[u] = F1[j + 1];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * 32 + lane;
      if (!ok[u]) continue;
      if (ntrg && (find_trg(sh, ntrg, i) || find_trg(sh, ntrg, i + 1))) continue;
      const double cfac = hn[u] == h_av ? dt_hav : dt / hn[u];
      rho[i] = r[u] - cfac * (b0[u] - a0[u]);
      mom[i] = m[u] - cfac * (b1[u] - a1[u]);
    }
  }
}

// window split part B: the results of this window's DTS jobs into the grid (as dts_block's
// epilogue: cells, width decisions, warm starts, counters of blocks owned by this window)
__device__ __forceinline__ void apply_dts_jobs(const Prm& p, CtaShared& sh, Arr& A, const Zone& Z, const DtsJob* jobs) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < sh.nblk; ++k) {
    const int jd = sh.dj[k];
    if (jd < 0) continue;
    const DtsJob& J = jobs[jd];
    const int a = sh.blkA[k], K = J.K;
    if (J.status) { if (lane == 0) set_status(sh, J.status); continue; }
    bool wm = false, rm = false;
    if (lane < K) {
      const double hn = A.h[a + lane], hn1 = J.hn[lane];
      wm = hn1 != hn && (width_marginal(hn1, p.eps_tiny * p.h_av) || width_marginal(hn1, p.eps_split * p.h_av));
      A.rho[a + lane] = J.un[lane][0]; A.mom[a + lane] = J.un[lane][1]; A.h[a + lane] = hn1;
      rm = hn1 < p.eps_tiny * p.h_av || hn1 > p.eps_split * p.h_av;
    }
    if (lane >= 1 && lane < K) {  // keep the converged boundary states for the next step
      Ifc* f = const_cast<Ifc*>(find_ifc(sh, a + lane));
      if (f) { f->pV = J.xs[lane][0]; f->pL = J.xs[lane][1]; }
    }
    const int mg = J.marg + __popc(__ballot_sync(0xffffffffu, wm));
    if (__any_sync(0xffffffffu, rm) && lane == 0) sh.remesh = 1;
    if (a >= Z.own_lo && a < Z.own_hi && lane == 0) {  // count a block once (its first cell's owner)
      sh.c_dts += (unsigned long long)J.it; sh.c_regions += 1ull;
      if ((unsigned long long)J.it > sh.c_dtsmax) sh.c_dtsmax = (unsigned long long)J.it;
      sh.c_margin += (unsigned long long)mg;
      sh.c_solves += (unsigned long long)J.solves;
    }
    __syncwarp();
  }
  for (int k = lane; k < sh.nifc; k += 32) { sh.ws0[k] = sh.ifc[k].pV; sh.ws1[k] = sh.ifc[k].pL; }
  __syncwarp();
}

// The end of a large step: status check, remesh (a10; R9, R10), counters and the new cell count.
__device__ __forceinline__ double step_tail(const Eos& e, const Prm& p, CtaShared& sh, Arr& A, int n, const int ntrg,
                                            const double dt, const Zone& Z) {
  double* const rho = A.rho;
  double* const mom = A.mom;
  double* const h = A.h;
  double* const F0 = A.F0;
  double* const F1 = A.F1;
  double* const X = A.X;
  uint8_t* const fl = A.fl;
  const int C = A.C;
  const int tid = threadIdx.x, T = blockDim.x;
  {
    const int stop2 = sh.status;
    __syncthreads();
    if (stop2) return -1.0;
  }
  // ---------------- remesh (a10; R9, R10): events -> shifts -> scatter ----------------
  int n_new = n;
  EIS_FCLK(5);
  if (sh.remesh) {
    if (tid == 0) { sh.nmev = 0; sh.nsev = 0; sh.ngrp = 0; }
    __syncthreads();
    for (int i = tid; i < n; i += T) {
      const double r_ = rho[i];
      const int ph = phase_of(e, r_);
      if (!(r_ > 0.0)) zone_status(sh, Z, i, ST_NONPOS);
      else if (ph == SPIN) zone_status(sh, Z, i, ST_SPINODAL);
      if (h[i] < p.eps_tiny * p.h_av) {  // merge partner: same-phase neighbour; both -> smaller, ties left
        const bool sl = i > 0 && !created_at(sh, ntrg, i) && phase_of(e, rho[i - 1]) == ph;
        const bool sr = i < n - 1 && !created_at(sh, ntrg, i + 1) && phase_of(e, rho[i + 1]) == ph;
        int j = -1;
        if (sl && sr) j = (h[i + 1] < h[i - 1]) ? i : i - 1;
        else if (sl) j = i - 1;
        else if (sr) j = i;
        if (j >= 0) { const int k = atomicAdd(&sh.nmev, 1); if (k < MAXEV) sh.mev[k] = j; else set_status(sh, ST_CAPACITY); }
      }
      if (h[i] > p.eps_split * p.h_av) {
        const int k = atomicAdd(&sh.nsev, 1);
        if (k < MAXEV) sh.sev[k] = i; else set_status(sh, ST_CAPACITY);
      }
    }
    __syncthreads();
    if (tid == 0 && sh.status == 0) {  // small serial bookkeeping: groups, splits, new size
      int nm = sh.nmev, ns = sh.nsev;
      for (int a = 1; a < nm; ++a) { int v = sh.mev[a], b = a - 1; while (b >= 0 && sh.mev[b] > v) { sh.mev[b + 1] = sh.mev[b]; --b; } sh.mev[b + 1] = v; }
      for (int a = 1; a < ns; ++a) { int v = sh.sev[a], b = a - 1; while (b >= 0 && sh.sev[b] > v) { sh.sev[b + 1] = sh.sev[b]; --b; } sh.sev[b + 1] = v; }
      int ng = 0, merges = 0, splits = 0, im = 0, is = 0;
      // walk merge edges (deduplicated) and split cells in increasing cell order
      while (im < nm || is < ns) {
        const int jm = im < nm ? sh.mev[im] : (1 << 29), js = is < ns ? sh.sev[is] : (1 << 29);
        Grp gr;
        if (jm <= js) {  // merge group [jm, g1]: consecutive merge edges (R10)
          int g1 = jm + 1;
          ++im;
          while (im < nm && sh.mev[im] <= g1) { if (sh.mev[im] == g1) ++g1; ++im; }
          double hs = 0.0, s0 = 0.0, s1 = 0.0;
          for (int k = jm; k <= g1; ++k) { hs += h[k]; s0 += h[k] * rho[k]; s1 += h[k] * mom[k]; }
          gr.g0 = jm; gr.g1 = g1; gr.h = hs; gr.r = s0 / hs; gr.m = s1 / hs;
          gr.split = hs > p.eps_split * p.h_av;
          merges += g1 - jm;
          while (is < ns && sh.sev[is] <= g1) ++is;  // split candidates inside the group
        } else {
          gr.g0 = gr.g1 = js; gr.h = h[js]; gr.r = rho[js]; gr.m = mom[js]; gr.split = 1;
          ++is;
        }
        splits += gr.split;
        if (ng < MAXEV) sh.grp[ng++] = gr; else set_status(sh, ST_CAPACITY);
      }
      sh.ngrp = ng;
      int ncre = 0;
      for (int k = 0; k < ntrg; ++k) ncre += sh.trg[k].acc;
      int nn = n + ncre;
      for (int k = 0; k < ng; ++k) nn += sh.grp[k].split - (sh.grp[k].g1 - sh.grp[k].g0);
      if (nn > C) set_status(sh, ST_CAPACITY);
      sh.n_new = nn;
      sh.c_merges += merges;
      sh.c_splits += splits;
    }
    __syncthreads();
    if (tid == 0) { sh.olo = Z.own_lo; sh.ohi = Z.own_hi; }
    __syncthreads();
    if (sh.status == 0 && (sh.ngrp > 0 || sh.c_creations > 0)) {
      if (tid == 0) { sh.olo = 1 << 30; sh.ohi = -1; }
      __syncthreads();
      for (int i = tid; i < n; i += T) {  // scatter into (F0, F1, X)
        int kg = -1;
        for (int k = 0; k < sh.ngrp; ++k)
          if (sh.grp[k].g0 <= i && i <= sh.grp[k].g1) kg = k;
        if (kg >= 0 && sh.grp[kg].g0 != i) continue;  // merged into its group head
        int pos = i + remesh_shift(sh, ntrg, i);
        if (created_at(sh, ntrg, i)) {  // created cell, width (w_r - w_l) dt
          const Trg* tr = find_trg(sh, ntrg, i);
          F0[pos - 1] = tr->rB; F1[pos - 1] = tr->mB; X[pos - 1] = (tr->wr - tr->wl) * dt;
          if (Z.own_lo < i && i <= Z.own_hi) {  // owned edge
            atomicMin(&sh.olo, pos - 1); atomicMax(&sh.ohi, pos); atomicAdd(&sh.o_cre, 1);
          }
        }
        if (Z.own_lo <= i && i < Z.own_hi) {  // owned head: its outputs are owned
          atomicMin(&sh.olo, pos);
          atomicMax(&sh.ohi, pos + ((kg >= 0 && sh.grp[kg].split) ? 2 : 1));
          if (kg >= 0) { atomicAdd(&sh.o_merges, sh.grp[kg].g1 - sh.grp[kg].g0); atomicAdd(&sh.o_splits, sh.grp[kg].split); }
        }
        if (kg >= 0) {
          const Grp& gr = sh.grp[kg];
          if (gr.split) {
            const double hh = 0.5 * gr.h;
            F0[pos] = gr.r; F1[pos] = gr.m; X[pos] = hh;
            F0[pos + 1] = gr.r; F1[pos + 1] = gr.m; X[pos + 1] = hh;
          } else { F0[pos] = gr.r; F1[pos] = gr.m; X[pos] = gr.h; }
        } else { F0[pos] = rho[i]; F1[pos] = mom[i]; X[pos] = h[i]; }
      }
      // boundary list: old boundaries shift with their right cell; each creation adds two
      __syncthreads();
      if (tid == 0) {
        int nif = sh.nifc;
        for (int k = 0; k < nif; ++k) sh.ifc[k].e += remesh_shift(sh, ntrg, sh.ifc[k].e);
        for (int k = 0; k < ntrg; ++k) {
          if (!sh.trg[k].acc) continue;
          const int pc = sh.trg[k].e + remesh_shift(sh, ntrg, sh.trg[k].e) - 1;  // created cell
          for (int q = 0; q < 2; ++q) {
            if (nif >= MAXIF) { set_status(sh, ST_CAPACITY); break; }
            int b = nif - 1;
            while (b >= 0 && sh.ifc[b].e > pc + q) { sh.ifc[b + 1] = sh.ifc[b]; --b; }
            sh.ifc[b + 1].e = pc + q;
            ++nif;
          }
        }
        sh.nifc = nif;
        if (sh.c_creations) sh.wsn = -1;  // ordinals changed: no warm start next step
        sh.nblk = 0;                      // flags are rebuilt below
      }
      n_new = sh.n_new;
      __syncthreads();
      for (int i = tid; i < n_new; i += T) { rho[i] = F0[i]; mom[i] = F1[i]; h[i] = X[i]; }  // copy back
      for (int i = tid; i <= C; i += T) fl[i] = 0;
      __syncthreads();
      for (int k = tid; k < sh.nifc; k += T) fl[sh.ifc[k].e] = F_IF;
    }
  }
  __syncthreads();
  EIS_FCLK(6);
  if (tid == 0) {
    EIS_TCLK(5);
    MemberStats& st = sh.st;
    st.steps += 1;
    st.cell_updates += n;
    st.creations += sh.o_cre;
    st.merges += sh.o_merges;
    st.splits += sh.o_splits;
    if (st.steps == 1 || dt < st.dt_min) st.dt_min = dt;
    if (dt > st.dt_max) st.dt_max = dt;
    sh.n = n_new;
    sh.ntrg = 0; sh.remesh = 0;
    sh.c_merges = 0; sh.c_splits = 0; sh.c_creations = 0;
    sh.o_cre = 0; sh.o_merges = 0; sh.o_splits = 0;
  }
  n = n_new;
  A.n = n;
  __syncthreads();
  return dt;
  }

template <int PH = 0>  // 0: the whole step; 1: window split part A (blocks exported as DTS jobs, no remesh)
__device__ __forceinline__ double step_body(const Eos& e, const Prm& p, CtaShared& sh, Arr& A, double t, double t_end,
                                            const Zone& Z) {
  double* const rho = A.rho;
  double* const mom = A.mom;
  double* const h = A.h;
  double* const F0 = A.F0;
  double* const F1 = A.F1;
  uint8_t* const fl = A.fl;
  int n = A.n;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  const int SW = nw - 1;  // solver warp
  const int half = lane >> 4, hl = lane & 15;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  // the solver warp joins the bulk when idle; a one-warp CTA (tiled windows) does all in order
  const int nbulk = (sh.nifc > 0 && nw > 1) ? nw - 1 : nw;
  if (tid == 0) { sh.olo = Z.own_lo; sh.ohi = Z.own_hi; }
  EIS_TCLK(0);
    double s_part = 0.0, h_part = INFINITY;

    if (warp == SW) {
      // ---------------- S1: tiny cells, implicit blocks, flags (O(#boundaries)) ----------------
      const int nif = sh.nifc;
      for (int k = 0; k < sh.nblk; ++k)  // clear last step's block flags
        for (int c = sh.blkA[k] + lane; c <= sh.blkB[k]; c += 32) fl[c] &= (uint8_t)~(F_TINY | F_REG);
      for (int k = lane; k < nif; k += 32) fl[sh.ifc[k].e] &= (uint8_t)~F_SPEC;
      __syncwarp();
      const bool valid = lane < nif;
      const int ek = valid ? sh.ifc[lane].e : -10;
      const int enext = lane + 1 < nif ? sh.ifc[lane + 1].e : -20;
      // cell ek lies between boundaries ek and ek + 1: tiny if narrower than eps_tiny h_av (R4)
      const bool tiny = p.mode != 1 && valid && enext == ek + 1 && h[ek] < p.eps_tiny * p.h_av;
      if (p.mode != 1 && lane == 0 && nif > 0) {  // a tiny cell at a domain end (R26)
        if (Z.left_real && sh.ifc[0].e == 1 && h[0] < p.eps_tiny * p.h_av) set_status(sh, ST_UNSUPPORTED);
        if (Z.right_real && sh.ifc[nif - 1].e == n - 1 && h[n - 1] < p.eps_tiny * p.h_av) set_status(sh, ST_UNSUPPORTED);
      }
      const unsigned mt = __ballot_sync(0xffffffffu, tiny);
      const int ntiny = __popc(mt);
      if (tiny) sh.tc[__popc(mt & lt_mask)] = ek;
      __syncwarp();
      // blocks: union of {k-1, k, k+1} over tiny k, overlapping ones merged (R11)
      const int cj = lane < ntiny ? sh.tc[lane] : 0;
      const int cprev = lane > 0 && lane < ntiny ? sh.tc[lane - 1] : -100;
      const int cnext = lane + 1 < ntiny ? sh.tc[lane + 1] : (1 << 29);
      const bool bstart = lane < ntiny && cprev + 1 < cj - 1;
      const bool bend = lane < ntiny && cj + 1 < cnext - 1;
      const unsigned ms = __ballot_sync(0xffffffffu, bstart), me = __ballot_sync(0xffffffffu, bend);
      const int nblk = __popc(ms);
      if (nblk > MAXBLK && lane == 0) set_status(sh, ST_CAPACITY);
      if (bstart && __popc(ms & lt_mask) < MAXBLK) sh.blkA[__popc(ms & lt_mask)] = cj - 1;
      if (bend && __popc(me & lt_mask) < MAXBLK) sh.blkB[__popc(me & lt_mask)] = cj + 1;
      __syncwarp();
      const int nb = nblk < MAXBLK ? nblk : MAXBLK;
      if (lane == 0) sh.nblk = nb;
      if (valid) {  // a boundary strictly inside a block is left to Algorithm 2
        bool interior = false;
        for (int k = 0; k < nb; ++k) interior |= (sh.blkA[k] < ek && ek <= sh.blkB[k]);
        sh.ifc[lane].interior = interior;
        if (!interior) fl[ek] |= F_SPEC;
      }
      __syncwarp();
      for (int k = 0; k < nb; ++k)
        for (int c = sh.blkA[k] + lane; c <= sh.blkB[k]; c += 32) fl[c] |= F_REG;
      __syncwarp();
      if (tiny) fl[ek] |= F_TINY;
      const bool warm = (nif == sh.wsn);
      if (valid) {
        sh.ifc[lane].pV = warm ? sh.ws0[lane] : -1.0;
        sh.ifc[lane].pL = warm ? sh.ws1[lane] : -1.0;
      }
      __syncwarp();
      EIS_FCLK(7);
      // ---------------- S2: explicit phase-boundary solves (App. A), half warps ----------------
      for (int k = half; k < nif; k += 2) {
        Ifc& f = sh.ifc[k];
        if (f.interior) continue;
        const int ed = f.e;
        const double rl = rho[ed - 1], rr = rho[ed];
        const int pl = phase_of(e, rl), pr = phase_of(e, rr);
        if (pl == pr || pl == SPIN || pr == SPIN) { if (hl == 0) zone_status_e(sh, Z, ed, pl == pr ? ST_INTERNAL : ST_SPINODAL); continue; }
        IfaceSol s = iface_solve_hw(e, p, rl, mom[ed - 1] / rl, rr, mom[ed] / rr, pl == VAP, f.pV, f.pL, hmask, hl, half * 16);
        if (hl == 0) {
          if (s.iters < 0) zone_status_e(sh, Z, ed, ST_NEWTON);
          f.F0 = s.F0; f.F1 = s.F1; f.w = s.w; f.pV = s.pV; f.pL = s.pL;
          if (Z.own_lo < ed && ed <= Z.own_hi) atomicAdd(&sh.c_solves, 1ull);
#ifdef EIS_S2_COUNT  // development: explicit boundary solves and their Newton iterations
          atomicAdd(reinterpret_cast<unsigned long long*>(&sh.dclk[3]), 1ull);
          atomicAdd(reinterpret_cast<unsigned long long*>(&sh.dclk[4]), (unsigned long long)s.iters);
          if (f.pV > 0.0 && warm) atomicAdd(reinterpret_cast<unsigned long long*>(&sh.dclk[2]), 1ull);
#endif
        }
      }
      __syncwarp();
    }
    EIS_FCLK(0);
    // ---------------- P1: edges (HLL a3, trigger a4), dt partials (a2) ----------------
    if (warp < nbulk) {
      double parts[2];
      bulk_p1(e, p, sh, Z, rho, mom, h, F0, F1, fl, n, warp, nbulk, parts);
      s_part = parts[0];
      h_part = parts[1];
    }
    s_part = warp_max(s_part);
    h_part = warp_min(h_part);
    if (lane == 0) { sh.part_s[warp] = s_part; sh.part_h[warp] = h_part; }  // folded after barrier A
    EIS_FCLK(1);
    EIS_ARRIVE(1);
    __syncthreads();  // ---------------- barrier A ----------------

    // lane-parallel fold of the per-warp partials (every warp computes the same dt)
    const double smax = warp_max(lane < nw ? sh.part_s[lane] : 0.0);
    const double hmin = warp_min(lane < nw ? sh.part_h[lane] : INFINITY);
    double dt = Z.dt_given > 0.0 ? Z.dt_given : p.cfl * hmin / smax;  // P:466 (tiles: the global dt)
    const double smax_step = Z.s_given > 0.0 ? Z.s_given : smax;       // LTS fine-level CFL (R29)
    if (t + dt > t_end) dt = t_end - t;
    const double dt_hav = dt / p.h_av;
    const int ntrg = sh.ntrg < MAXTRG ? sh.ntrg : MAXTRG;
    int remesh = 0;
    EIS_FCLK(2);

    if (warp == SW) {
      // ---------------- S4: dual time stepping on every block (a9) ----------------
#ifdef EIS_PHASE_CLOCK
      if (lane == 0) sh.tclk[6] = clock64();
#endif
      const int nblk = sh.nblk;
      if constexpr (PH == 1) {  // window split: each block becomes a DTS job (dts_jobs, one lane)
        for (int k = 0; k < nblk; ++k) {
          const int a = sh.blkA[k], b = sh.blkB[k], K = b - a + 1;
          if (lane == 0) sh.dj[k] = -1;
          if (b < Z.zlo || a >= Z.zhi) continue;  // a block wholly in the halo is not needed
          if (K > MAXB || b < a) { if (lane == 0) set_status(sh, ST_CAPACITY); continue; }
          int jd = 0;
          if (lane == 0) jd = atomicAdd(Z.djn, 1);
          jd = __shfl_sync(0xffffffffu, jd, 0);
          if (jd >= Z.djcap) { if (lane == 0) set_status(sh, ST_CAPACITY); continue; }
          DtsJob& J = Z.djobs[jd];
          if (lane < K) { J.un[lane][0] = rho[a + lane]; J.un[lane][1] = mom[a + lane]; J.hn[lane] = h[a + lane]; }
          if (lane >= 1 && lane < K) {  // warm start of interior boundaries from the last step
            const Ifc* f = find_ifc(sh, a + lane);
            J.xs[lane][0] = f ? f->pV : -1.0;
            J.xs[lane][1] = f ? f->pL : -1.0;
          }
          const unsigned tb = __ballot_sync(0xffffffffu, lane < K && (fl[a + lane] & F_TINY));
          if (lane == 0) {  // outer edges: the explicit step's fluxes and speeds
            double g0, g1, w;
            edge_view(sh, fl, F0, F1, a, 1, g0, g1, w);
            J.Fo[0][0] = g0; J.Fo[0][1] = g1; J.wo[0] = w;
            edge_view(sh, fl, F0, F1, b + 1, 0, g0, g1, w);
            J.Fo[1][0] = g0; J.Fo[1][1] = g1; J.wo[1] = w;
            J.dt = dt; J.K = K; J.tiny = (int)tb;
            sh.dj[k] = jd;
          }
          __syncwarp();
        }
      } else
      for (int k = 0; k < nblk; ++k) {
        const int a = sh.blkA[k], b = sh.blkB[k];
        if (b < Z.zlo || a >= Z.zhi) continue;  // tiles: a block wholly in the halo is not needed
        if (b - a + 1 > MAXB || b < a) { if (lane == 0) set_status(sh, ST_CAPACITY); continue; }
        long long it = 0, sv = 0;
        int mg = 0;
        const int err = p.mode == 2   ? lts_block(e, p, sh, rho, mom, h, F0, F1, fl, a, b, dt, smax_step, it, sv, remesh)
#ifndef EIS_NO_NEWTON
                        : p.mode == 3 ? newton_block(e, p, sh, rho, mom, h, F0, F1, fl, a, b, dt, it, sv, remesh)
#endif
                                      : dts_block(e, p, sh, rho, mom, h, F0, F1, fl, a, b, dt, it, sv, remesh, mg);
        if (err && lane == 0) set_status(sh, err);
        if (a >= Z.own_lo && a < Z.own_hi) {  // count a block once (its first cell's owner)
          if (lane == 0) {
            atomicAdd(&sh.c_dts, (unsigned long long)it); atomicAdd(&sh.c_regions, 1ull); atomicMax(&sh.c_dtsmax, (unsigned long long)it);
            if (mg) atomicAdd(&sh.c_margin, (unsigned long long)mg);
          }
          if (hl == 0 && sv) atomicAdd(&sh.c_solves, (unsigned long long)sv);
        }
      }
#ifdef EIS_PHASE_CLOCK
      if (lane == 0) sh.tclk[7] = clock64();
#endif
      EIS_FCLK(3);
      // ---------------- S5: cells next to explicit phase boundaries (a7) ----------------
      const int nif = sh.nifc;
      for (int q = lane; q < 2 * nif; q += 32) {
        const Ifc& f = sh.ifc[q >> 1];
        if (f.interior) continue;
        const int i = (q & 1) ? f.e : f.e - 1;
        if ((q & 1) == 0 && (fl[i] & F_SPEC)) continue;  // handled as the right cell of edge i
        if (fl[i] & F_REG) continue;
        if (ntrg && (find_trg(sh, ntrg, i) || find_trg(sh, ntrg, i + 1))) continue;  // creation pass
        double a0, a1, wa, b0, b1, wb;
        edge_view(sh, fl, F0, F1, i, 1, a0, a1, wa);
        edge_view(sh, fl, F0, F1, i + 1, 0, b0, b1, wb);
        int mg = 0;
        const int err = cell_update(rho, mom, h, i, a0, a1, wa, b0, b1, wb, dt, p, remesh, mg);
        if (err) zone_status(sh, Z, i, err);
        if (mg && i >= Z.own_lo && i < Z.own_hi) atomicAdd(&sh.c_margin, 1ull);
      }
      for (int k = lane; k < nif; k += 32) { sh.ws0[k] = sh.ifc[k].pV; sh.ws1[k] = sh.ifc[k].pL; }
      if (lane == 0) sh.wsn = nif;
      __syncwarp();
    }
    // ---------------- P2: explicit update of cells with two HLL edges (a7) ----------------
    if (warp < nbulk) bulk_p2(p, sh, rho, mom, h, F0, F1, fl, n, warp, nbulk, ntrg, dt, dt_hav);
    if (remesh) sh.remesh = 1;
    EIS_ARRIVE(3);
    __syncthreads();  // ---------------- barrier B ----------------
    EIS_FCLK(4);

    // ---------------- creations (a6): acceptance (R16), solves, neighbour updates ----------------
    if (ntrg) {
      for (int k = tid; k < ntrg; k += T) {
        int run = 0;
        while (find_trg(sh, ntrg, sh.trg[k].e - run - 1)) ++run;  // leftmost wins
        sh.trg[k].acc = (run & 1) ? 0 : 1;
      }
      __syncthreads();
      for (int k = warp * 2 + half; k < ntrg; k += nw * 2) {
        Trg& tr = sh.trg[k];
        if (!tr.acc) continue;
        const int ed = tr.e;
        const double rl = rho[ed - 1], rr = rho[ed];  // still U^n: these cells were deferred
        CreateSol s = create_solve_hw(e, p, phase_of(e, rl), rl, mom[ed - 1] / rl, rr, mom[ed] / rr, hmask, hl, half * 16);
        if (hl == 0) {
          if (s.iters < 0) set_status(sh, ST_CREATION);
          tr.Fl0 = s.Fl0; tr.Fl1 = s.Fl1; tr.wl = s.wl; tr.Fr0 = s.Fr0; tr.Fr1 = s.Fr1; tr.wr = s.wr;
          tr.rB = s.rB; tr.mB = s.mB;
          atomicAdd(&sh.c_creations, 1);
          if ((s.wr - s.wl) * dt > p.eps_split * p.h_av) set_status(sh, ST_UNSUPPORTED);  // never with C <= 1
        }
      }
      __syncthreads();
      for (int q = tid; q < 2 * ntrg; q += T) {
        const int ed = sh.trg[q >> 1].e;
        const int i = (q & 1) ? ed : ed - 1;
        if ((q & 1) == 0 && find_trg(sh, ntrg, i)) continue;  // handled as the right cell of edge i
        double a0, a1, wa, b0, b1, wb;
        edge_view(sh, fl, F0, F1, i, 1, a0, a1, wa);
        edge_view(sh, fl, F0, F1, i + 1, 0, b0, b1, wb);
        int rm = 0, mg = 0;
        const int err = cell_update(rho, mom, h, i, a0, a1, wa, b0, b1, wb, dt, p, rm, mg);
        if (err) zone_status(sh, Z, i, err);
        if (mg && i >= Z.own_lo && i < Z.own_hi) atomicAdd(&sh.c_margin, 1ull);
      }
      if (tid == 0) sh.remesh = 1;
      __syncthreads();
    }
    if constexpr (PH == 1) {  // window split, part A: the blocks were exported; remesh after the DTS jobs
      const int stop2 = sh.status;
      __syncthreads();
      return stop2 ? -1.0 : dt;
    } else {
      return step_tail(e, p, sh, A, n, ntrg, dt, Z);
    }
  }

// ------------------------------------------------------------------------------------------
// The member-resident kernel.  Dynamic shared memory: CtaShared | 6 x (cap+1) doubles |
// (cap+1) flag bytes.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ Arr carve(unsigned char* smem_raw, int C) {
  double* arr = reinterpret_cast<double*>(smem_raw + ((sizeof(CtaShared) + 15) & ~size_t(15)));
  Arr A;
  A.rho = arr; A.mom = arr + (C + 1); A.h = arr + 2 * (C + 1);
  A.F0 = arr + 3 * (C + 1); A.F1 = arr + 4 * (C + 1); A.X = arr + 5 * (C + 1);
  A.fl = reinterpret_cast<uint8_t*>(arr + 6 * (C + 1));
  A.C = C;
  A.n = 0;
  return A;
}

__device__ __forceinline__ void reset_counters(CtaShared& sh) {
  sh.wsn = -1; sh.nblk = 0; sh.ntrg = 0; sh.remesh = 0;
  sh.c_merges = 0; sh.c_splits = 0; sh.c_creations = 0;
  sh.c_dts = 0; sh.c_solves = 0; sh.c_regions = 0; sh.c_dtsmax = 0; sh.c_margin = 0;
  sh.o_cre = 0; sh.o_merges = 0; sh.o_splits = 0;
}

template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
resident_steps(const __grid_constant__ Eos e, const __grid_constant__ Prm p, const __grid_constant__ Members g,
               long long n_steps, double t_end) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CtaShared& sh = *reinterpret_cast<CtaShared*>(smem_raw);
  Arr A = carve(smem_raw, (int)g.cap);
  const int tid = threadIdx.x, T = blockDim.x, warp = tid >> 5, nw = T >> 5;
  const long long m = blockIdx.x;
  const long long base = m * g.cap;
  if (tid == 0) {
    sh.n = (int)g.n[m];
    sh.status = g.status[m];
    reset_counters(sh);
    sh.st = g.stats[m];
  }
  __syncthreads();
  A.n = sh.n;
  for (int i = tid; i < A.n; i += T) {
    A.rho[i] = g.rho[base + i];
    A.mom[i] = g.mom[base + i];
    A.h[i] = g.h[base + i];
  }
  for (int i = tid; i <= A.C; i += T) A.fl[i] = 0;
  double t = g.t[m];
  __syncthreads();
  if (warp == nw - 1) build_boundary_list(e, sh, A.rho, A.fl, A.n);
  __syncthreads();
  Zone Z;
  Z.zlo = 0; Z.zhi = 1 << 30; Z.own_lo = 0; Z.own_hi = 1 << 30; Z.dt_given = -1.0; Z.s_given = -1.0;
  Z.left_real = true; Z.right_real = true;
  for (long long step = 0; step < n_steps; ++step) {
    const bool stop = sh.status != 0 || !(t < t_end);
    __syncthreads();  // every thread has read sh.status before anyone can write it
    if (stop) break;
    const double dt = step_body(e, p, sh, A, t, t_end, Z);
#ifdef EIS_PHASE_CLOCK
    if (g.dbg && tid == 0) {
      long long* d = g.dbg + 8 * m;
      for (int i = 1; i <= 5; ++i) d[i - 1] += sh.tclk[i] - sh.tclk[0];
      d[5] += sh.tclk[7] - sh.tclk[6];
      d[6] += 1;
    }
#endif
    if (dt < 0.0) break;
    t += dt;
  }
  // ---------------- write back (one HBM round trip per call) ----------------
  __syncthreads();
  const int n = sh.n;
  for (int i = tid; i < n; i += T) {
    g.rho[base + i] = A.rho[i];
    g.mom[base + i] = A.mom[i];
    g.h[base + i] = A.h[i];
  }
  __syncthreads();
  if (tid == 0) {
    MemberStats st = sh.st;
    st.dts_iters += (long long)sh.c_dts;
    st.iface_solves += (long long)sh.c_solves;
    st.regions += (long long)sh.c_regions;
    st.margins += (long long)sh.c_margin;
    if ((long long)sh.c_dtsmax > st.dts_max) st.dts_max = (long long)sh.c_dtsmax;
    g.n[m] = n;
    g.t[m] = t;
    g.status[m] = sh.status;
    g.stats[m] = st;
  }
}

}  // namespace eis
