// eis_tiled.cuh — the tiled streaming kernels for huge grids (BASELINE configs[4], C5) and for
// ensembles of large members (C4; each member its own run of tiles).
//
// A grid is cut into fixed-size tiles (1400 owned cells by default), each stored with slack
// (capt cells) so that creations and splits insert locally; ping-pong buffers (step n reads
// buffer cur, writes 1-cur).  A step is three launches (plus tiled_members_finish for ensembles):
//   tiled_fast (one CTA per tile, high occupancy): stages the tile's own cells in shared memory
//     with a TMA bulk copy, streams them plus HALO cells of each neighbour through registers in
//     warp windows and, where the tile is plain (no cell of another phase, spinodal or creation
//     candidate), completes its step: HLL fluxes (a3), update (a7), the next step's CFL
//     partials (a2).  Otherwise it lists a window of <= WMAX owned cells around the special
//     cells, or the whole tile.  Widths are not stored for tiles whose widths are all h_av.
//   tiled_win (persistent one-warp CTAs): the member-resident step body (the whole method,
//     a1-a11) on each listed window plus halos, assembled in place into the tile output.
//   tiled_slow (persistent CTAs, dynamic work list): the same on whole tiles, then the last CTA
//     folds the CFL partials into the next dt (R5/R6).
// The halo is computed redundantly by both neighbours with identical inputs and code, so every
// decision at a tile boundary (boundary solves, creations, DTS blocks, merges) is taken
// identically on both sides; ownership: a created cell at a tile boundary and a merge group
// headed left of it belong to the left tile.
#pragma once
#include "eis_resident.cuh"

namespace eis {

constexpr int HALO = 10;  // halo cells per side: >= MAXB + 2 keeps every needed block exact

struct TileStats {
  long long cell_updates, dts_iters, iface_solves, creations, splits, merges, regions;
  long long dts_max, full_steps, win_steps;  // steps this tile took the whole-tile / window full step
  long long margins;                         // decision_margin_warnings (eis.h)
};

struct Tiles {
  double *rho[2], *mom[2], *h[2];  // ntiles x capt, ping-pong
  int* cnt[2];                     // live cells per tile
  int* hu[2];                      // per tile: 1 = every width is h_av (widths not stored)
  double* ws;                      // per tile: ws0[MAXIF], ws1[MAXIF], wsn  (2*MAXIF + 1 doubles)
  double* part;                    // per tile: S_max, h_min of the tile's new cells
  TileStats* tstats;
  double* scal;                    // per member (stride SCS): [0] t  [1] dt of the coming step
                                   //   [2] dt_min  [3] dt_max  [4] dt used (rank mode)  [5] S_max of the coming step
  int* mctl;                       // per member (stride MCS): [0] cur buffer  [1] status  [2] steps
  int* ctl;                        // global counters (below)
  double* xbuf;                    // rank mode: exchange buffer (layout XB_* below), else null
  int* slow;                       // work list of tiles needing the full step of the whole tile
  int* wlist;                      // work list of (tile, window begin, window end, ready tag)
  double* partf;                   // per window tile: S_max, h_min, all-h_av of its fast cells
  double* part2;                   // per tiled_slow CTA: S_max, h_min
  // peer mode (eis_set_exchange_peers): the exchange done by the kernels themselves over peer
  // memory (NVLink): xpeer_l / xpeer_r are the neighbours' exchange buffers (null at the domain
  // ends), xpeers[q] rank q's (for the CFL pair); null xpeers: the caller exchanges (NCCL)
  double* xpeer_l;
  double* xpeer_r;
  double* const* xpeers;
  int xrank, xworld;
  long long* wdbg;                 // diagnostics (EIS_WINDOW_DEBUG): per window job of the last step
                                   // {cycles, dts iterations, window cells, boundaries, start clock,
                                   //  6 phase cycles (EIS_PHASE_CLOCK builds, else 0)}
  int ntiles, capt, nbr_left, nbr_right;
  int wmax;                        // largest window (owned cells) of a window full step (<= WMAX)
  int poll;                        // a window kernel polls beside tiled_fast (EIS_WIN_POLL_PER_SM)
  int M, tpm;                      // members (independent grids) and tiles per member: tile k
                                   // belongs to member k / tpm; halos never cross members
  int split;                       // window split: part A, dts_jobs (one lane per block), part B
  int djcap;                       //   DTS job capacity
  DtsJob* djobs;                   //   DTS jobs of the step (counter ctl[10])
  unsigned char* wsave;            //   per window job: its grid between parts A and B (WSAVE bytes)
  // window prediction (tl.spec; window split only): the window step predicts the tile's special
  // range of the NEXT step, so that part A and the DTS jobs of the predicted windows run beside
  // tiled_fast on a second stream; tiled_fast compares its own classification with the
  // prediction (equal: the early result is used; else the window takes the late path)
  int spec;
  int* pred[2];                    //   per tile, by step parity: [slot, q_lo, q_hi, -] (slot -1: none);
                                   //   q = special range in positions relative to the first owned cell
  int* plist[2];                   //   predicted tiles by slot (-1: that window predicted nothing), by step parity
  int* mlist;                      //   list indices of this step's windows whose prediction failed (late part A)
};
constexpr int SCS = 8, MCS = 4;
// ctl: [1] any member status  [2] done-counter  [3] launches  [4] tile-list length  [5] next tile job
//      [6] window-list length  [7] next window job  [8] window jobs of the last step
//      [9] tiled_fast CTAs finished (the window kernel running beside tiled_fast polls it)
//      [10] DTS jobs of the step (window split)  [11] next window job of part B
//      [13] early window jobs of this step (= the last step's listed windows: a window's early slot is
//           its list index of the step that predicted it)  [15] next early job
//      [17] DTS jobs solved by the early dts_jobs launch  [18] hits, [19] window jobs (cumulative)
//      [20] listed windows of this step whose prediction failed (the late part A's jobs, mlist)
//      [14] early window jobs of the next step
constexpr int NCTL = 32;
// end of a step: the work-list counters (the predictions made become the next step's)
__device__ __forceinline__ void ctl_step_reset(const Tiles& tl) {
  tl.ctl[2] = 0; tl.ctl[4] = 0; tl.ctl[5] = 0; tl.ctl[6] = 0; tl.ctl[7] = 0; tl.ctl[9] = 0; tl.ctl[10] = 0; tl.ctl[11] = 0;
  tl.ctl[15] = 0; tl.ctl[17] = 0; tl.ctl[20] = 0;
  if (tl.spec && tl.ctl[8] > 0) tl.ctl[14] = 4 * tl.ctl[8] <= tl.ntiles ? tl.ctl[8] : 0;  // (ctl[8]: this step's listed windows;
                                                                                  //  predictions were made if they were sparse)
}
__device__ __forceinline__ void ctl_step_roll(const Tiles& tl) {  // once per step taken, with ctl[3] += 1
  tl.ctl[13] = tl.ctl[14]; tl.ctl[14] = 0;
}

// Exchange buffer (rank mode, one grid decomposed over ranks): four halo records of
// HALO cells (rho, mom, h) + a count, then the CFL pair (-S_max, h_min) to be min-reduced.
constexpr int WDBG_FIELDS = 11;
constexpr int XB_REC = 3 * HALO + 1;
constexpr int XB_SEND_LEFT = 0, XB_SEND_RIGHT = XB_REC, XB_RECV_LEFT = 2 * XB_REC, XB_RECV_RIGHT = 3 * XB_REC;
constexpr int XB_DT = 4 * XB_REC;
constexpr int XB_DOUBLES = 4 * XB_REC + 2;
// peer mode, appended (double-buffered by the parity of the publication tag, so a neighbour one
// publication ahead never overwrites what this rank has not consumed yet): the neighbours'
// records [parity][left, right][XB_REC] and the ranks' CFL pairs [parity][rank][-S_max, h_min,
// tag, status]
constexpr int XB_MAXRANKS = 8;
constexpr int XB_PREC = XB_DOUBLES;                          // + (2 par + side) * XB_REC
constexpr int XB_PPAIR = XB_PREC + 4 * XB_REC;               // + (par * XB_MAXRANKS + rank) * 4
constexpr int XB_DOUBLES_PEER = XB_PPAIR + 2 * XB_MAXRANKS * 4;
// ctl[12]: publications of this rank (init + every step) = the tag of the last one

constexpr int WS_STRIDE = 2 * MAXIF + 1;

// S_max and h_min (over non-tiny cells, R5/R6) of cells [lo, hi) of a smem grid of n cells
__device__ __forceinline__ void cfl_partials(const Eos& e, const Prm& p, const double* rho, const double* mom,
                                             const double* h, int n, int lo, int hi, bool left_real,
                                             bool right_real, double& s_out, double& h_out) {
  double s = 0.0, hm = INFINITY;
  for (int i = lo + (int)threadIdx.x; i < hi; i += blockDim.x) {
    const double r = rho[i];
    const int ph = phase_of(e, r);
    s = fmax(s, fabs(mom[i] * rcp_fast(r)) + sound(e, ph));  // u as in bulk_p1 / tiled_fast
    bool tiny = false;
    if (p.mode != 1 && h[i] < p.eps_tiny * p.h_av) {
      const bool same_l = (i > 0) ? phase_of(e, rho[i - 1]) == ph : false;
      const bool same_r = (i < n - 1) ? phase_of(e, rho[i + 1]) == ph : false;
      tiny = !same_l && !same_r;
    }
    if (!tiny) hm = fmin(hm, h[i]);
  }
  (void)left_real; (void)right_real;
  s_out = warp_max(s);
  h_out = warp_min(hm);
}

// Peer mode: this rank's step-end exchange, by one CTA after every record of the step is written
// (the last CTA of tiled_slow / tiled_init_dt): its send records into the neighbours' receive
// slots, its CFL pair (-S_max, h_min) and status into every rank's pair table, then -- after a
// system-scope fence -- the tag.  Consumed by tiled_finish (eis_step_finish).
__device__ void xpublish(const Tiles& tl, double neg_s, double hm, int status) {
  __shared__ long long tag_s;
  const int tid = threadIdx.x;
  __syncthreads();
  if (tid == 0) tag_s = (long long)(++tl.ctl[12]);
  __syncthreads();
  const long long tag = tag_s;
  const int par = (int)(tag & 1);
  for (int q = tid; q < XB_REC; q += blockDim.x) {  // my send-left -> left rank's right slot, etc.
    if (tl.xpeer_l) tl.xpeer_l[XB_PREC + (2 * par + 1) * XB_REC + q] = tl.xbuf[XB_SEND_LEFT + q];
    if (tl.xpeer_r) tl.xpeer_r[XB_PREC + (2 * par + 0) * XB_REC + q] = tl.xbuf[XB_SEND_RIGHT + q];
  }
  for (int q = tid; q < tl.xworld; q += blockDim.x) {
    double* pr = tl.xpeers[q] + XB_PPAIR + (par * XB_MAXRANKS + tl.xrank) * 4;
    pr[0] = neg_s; pr[1] = hm; pr[3] = (double)status;
  }
  __threadfence_system();
  __syncthreads();
  for (int q = tid; q < tl.xworld; q += blockDim.x) {
    volatile double* pt = tl.xpeers[q] + XB_PPAIR + (par * XB_MAXRANKS + tl.xrank) * 4 + 2;
    *pt = (double)tag;
  }
  __threadfence_system();
}

// Last CTA of a step: fold the per-CTA partials into the next dt, advance t.
__device__ void tiles_finish_step(const Prm& p, const Tiles& tl, int nparts, double dt_used, double t_end) {
  __shared__ double rs[32], rh[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double s = 0.0, hm = INFINITY;
  for (int k = tid; k < nparts; k += blockDim.x) {
    s = fmax(s, tl.part2[2 * k]);
    hm = fmin(hm, tl.part2[2 * k + 1]);
  }
  s = warp_max(s);
  hm = warp_min(hm);
  if (lane == 0) { rs[warp] = s; rh[warp] = hm; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 0; w < nw; ++w) { s = fmax(s, rs[w]); hm = fmin(hm, rh[w]); }
    tl.ctl[8] = tl.ctl[6];  // window jobs of this step (diagnostics)
    ctl_step_reset(tl);
  }
  if (tl.xbuf) {  // rank mode: the global dt needs the other ranks (eis_step_finish)
    if (tid == 0) {
      tl.xbuf[XB_DT] = -s;
      tl.xbuf[XB_DT + 1] = hm;
      tl.scal[4] = dt_used;
      __threadfence();
    }
    __syncthreads();
    if (tl.xpeers) xpublish(tl, tl.xbuf[XB_DT], tl.xbuf[XB_DT + 1], 0);
    return;
  }
  if (tid == 0) {
    const double t_new = tl.scal[0] + dt_used;
    double dt = p.cfl * hm / s;
    if (t_new + dt > t_end) dt = t_end - t_new;
    tl.scal[0] = t_new;
    tl.scal[1] = dt;
    tl.scal[5] = s;  // S_max of the next step (LTS fine-level CFL, R29)
    if (tl.mctl[2] == 0 || dt_used < tl.scal[2]) tl.scal[2] = dt_used;
    if (dt_used > tl.scal[3]) tl.scal[3] = dt_used;
    tl.mctl[0] = 1 - tl.mctl[0];
    tl.mctl[2] += 1;
    tl.ctl[3] += 1;
    ctl_step_roll(tl);
    __threadfence();
  }
}

// Geometry of tile k in the step reading buffer `in`: own cells and up to HALO halo cells per
// side (from the neighbour tiles, or from the exchange buffer at a rank boundary), seen as one
// virtual array [0, n) = left halo | own | right halo.
struct TGeo {
  long long base, bl, br;
  int k, m, in, out, cnt, cl, nL, nR, n;
  bool xl, xr, hu_in;
  bool first, last;  // the member's first / last tile (a domain end unless a rank neighbour)
  bool huL, huR;     // tile_geo_spec: the neighbour tiles' uniform-width flags (read buffer)
};
// (the tile metadata of both buffers is loaded before `cur` is known: one dependent global
// round trip fewer at the start of every tile)
// (PLAIN: no rank neighbour, the exchange buffer is never read; GEO = 1: one grid, GEO = 2: the
// member m2 and the tile j2 within it given (a 2D launch) -- no division by the tiles per member
// at the start of every CTA: tiled_fast's instantiations for the usual contexts)
template <bool PLAIN = false, int GEO = 0>
__device__ __forceinline__ TGeo tile_geo_spec(const Tiles& tl, int k, int m2 = 0, int j2 = 0) {
  const int m = GEO == 1 ? 0 : (GEO == 2 ? m2 : k / tl.tpm);
  const bool hasl = GEO == 1 ? k != 0 : (GEO == 2 ? j2 != 0 : k % tl.tpm != 0);
  const bool hasr = GEO == 1 ? k + 1 != tl.ntiles : (GEO == 2 ? j2 + 1 != tl.tpm : (k + 1) % tl.tpm != 0);
  const int c0 = tl.cnt[0][k], c1 = tl.cnt[1][k], h0 = tl.hu[0][k], h1 = tl.hu[1][k];
  const int l0 = hasl ? tl.cnt[0][k - 1] : 0, l1 = hasl ? tl.cnt[1][k - 1] : 0;
  const int r0 = hasr ? tl.cnt[0][k + 1] : 0, r1 = hasr ? tl.cnt[1][k + 1] : 0;
  const int hl0 = hasl ? tl.hu[0][k - 1] : 0, hl1 = hasl ? tl.hu[1][k - 1] : 0;  // (dropped where unused)
  const int hr0 = hasr ? tl.hu[0][k + 1] : 0, hr1 = hasr ? tl.hu[1][k + 1] : 0;
  const int cur = tl.mctl[MCS * m];
  TGeo g;
  g.k = k; g.m = m; g.in = cur; g.out = 1 - cur;
  g.first = !hasl; g.last = !hasr;
  g.base = (long long)k * tl.capt; g.bl = g.base - tl.capt; g.br = g.base + tl.capt;
  g.cnt = cur ? c1 : c0;
  g.hu_in = (cur ? h1 : h0) != 0;
  g.huL = (cur ? hl1 : hl0) != 0;
  g.huR = (cur ? hr1 : hr0) != 0;
  g.xl = !PLAIN && (g.first && tl.nbr_left); g.xr = !PLAIN && (g.last && tl.nbr_right);
  g.cl = cur ? l1 : l0;
  g.nL = hasl ? min(HALO, g.cl) : (g.xl ? (int)tl.xbuf[XB_RECV_LEFT + 3 * HALO] : 0);
  g.nR = hasr ? min(HALO, cur ? r1 : r0) : (g.xr ? (int)tl.xbuf[XB_RECV_RIGHT + 3 * HALO] : 0);
  g.n = g.nL + g.cnt + g.nR;
  return g;
}
// address of virtual cell i's density (the momentum is at +mo, in the same array family)
__device__ __forceinline__ const double* vcell(const Tiles& tl, const TGeo& g, int i, long long& mo) {
  if (i < g.nL) {
    if (g.xl) { mo = HALO; return tl.xbuf + XB_RECV_LEFT + HALO - g.nL + i; }
    mo = tl.mom[g.in] - tl.rho[g.in];
    return tl.rho[g.in] + g.bl + g.cl - g.nL + i;
  }
  if (i >= g.nL + g.cnt && g.xr) { mo = HALO; return tl.xbuf + XB_RECV_RIGHT + (i - g.nL - g.cnt); }
  mo = tl.mom[g.in] - tl.rho[g.in];
  return tl.rho[g.in] + (i < g.nL + g.cnt ? g.base + (i - g.nL) : g.br + (i - g.nL - g.cnt));
}

// ------------------------------------------------------------------------------------------
// tiled_fast: one CTA per tile.  Warp windows of 64 virtual cells s-2 .. s+61, two per lane
// (c0 = s-2+2l, c1 = c0+1; ghosts clamp at the grid ends, R15): u = m/rho and p (a1), the HLL
// fluxes of the lane's left edge (c0; the left state by shuffle from the previous lane) and of
// its internal edge (c1) (a3), the creation pre-filter on both (a4, R7), the right flux of c1
// by shuffle and the updates of the pairs of lanes 1..30, cells s .. s+59 (a7; lanes 0
// and 31 are halo, so every store is an aligned 16-byte pair) written to the output tile with
// the next step's CFL partials (a2) -- the same expressions as step_body's bulk passes, so a
// plain tile's result is the full step's bit for bit.  Interior windows load and store cell
// pairs as 16-byte vectors (from the shared-memory copy of the tile; the two halo windows from
// global memory).  FB windows per warp iteration (1: more would spill at 64 registers).  Outputs
// of a tile that turns out not plain are overwritten by the window / whole-tile full step.
// ------------------------------------------------------------------------------------------
#ifndef EIS_FB
#define EIS_FB 1
#endif
#ifndef EIS_FAST_STATIC_IN
#define EIS_FAST_STATIC_IN 1
#endif
#ifndef EIS_FAST_TMA
#define EIS_FAST_TMA 1  // the tile's own cells staged in shared memory by cp.async.bulk (0: L2 prefetch)
#endif
#ifndef EIS_FAST_PIPE
#define EIS_FAST_PIPE 0
#endif
// (Measured, round 2: four cells per lane -- 120-cell windows, 80 registers, 6 CTAs/SM, no
// spills -- is 20 % slower on C5 (1.22 vs 1.01 ms): the kernel needs the warps more than it saves
// on shuffles and per-window overhead.)
constexpr int FB = EIS_FB;  // windows per warp per batch
constexpr int FW = 60;      // cells updated per window: the pairs of lanes 1..30

// one window batch of one warp after its loads: the arithmetic, specialised by the phase (LIQ)
// and by uniform widths (HU).  A cell of another phase (or spinodal, or non-positive) and the
// right cell of a creation-candidate edge are "special": their index range [slo, shi] decides
// between the fast result and a full step of a window around them.
template <bool HU, bool LIQ, bool MASKED>
__device__ __forceinline__ void fast_pairs(const Eos& e, const double2 (&rv)[FB], const double2 (&mv)[FB], int w0,
                                           int nw, int nwin, int n, int own_lo, int own_hi, double dt, double dt_hav,
                                           double h_av, const double* ih, double* orho, double* omom, double* oh,
                                           unsigned bmask, int& slo, int& shi, bool& unif, double& snum, double& sden,
                                           double& h_part) {
  const int lane = threadIdx.x & 31;
  const double a = LIQ ? e.a_l : e.a_v;
  const double rho_tilde = e.rho_tilde, rho_min = e.rho_min, a_v2 = e.a_v2, a_l2 = e.a_l2, p0 = e.p0, rho0 = e.rho0;
  const double rmin2 = rho_min * rho_min, inv_rt = 1.0 / rho_tilde;
#pragma unroll
  for (int b = 0; b < FB; ++b) {
    if (w0 + nw * b >= nwin) break;  // warp-uniform
    if (MASKED && !(bmask >> b & 1)) continue;  // a window of the other specialisation
    const int c0 = FW * (w0 + nw * b) - 2 + 2 * lane, c1 = c0 + 1;
    const double r0 = rv[b].x, r1 = rv[b].y, m0 = mv[b].x, m1 = mv[b].y;
    const double u0 = m0 * rcp_fast(r0), u1 = m1 * rcp_fast(r1);
    // lanes beyond the grid hold clamped copies of real cells: every cell of [0, n) is checked
    const bool sp0 = LIQ ? !(r0 >= rho_min) : !(r0 <= rho_tilde && r0 > 0.0);
    bool sp1 = LIQ ? !(r1 >= rho_min) : !(r1 <= rho_tilde && r1 > 0.0);
    const double q0 = LIQ ? p0 + a_l2 * (r0 - rho0) : a_v2 * r0;
    const double q1 = LIQ ? p0 + a_l2 * (r1 - rho0) : a_v2 * r1;
    const double rl = __shfl_up_sync(0xffffffffu, r1, 1), ml = __shfl_up_sync(0xffffffffu, m1, 1);
    const double ul = __shfl_up_sync(0xffffffffu, u1, 1), pl = __shfl_up_sync(0xffffffffu, q1, 1);
    double fl0, fl1, fi0, fi1;  // edge c0 (left of c0), edge c1 (between c0 and c1)
    hll_fast(a, rl, ml, ul, pl, r0, m0, u0, q0, fl0, fl1);
    hll_fast(a, r0, m0, u0, q0, r1, m1, u1, q1, fi0, fi1);
    bool cl;  // creation pre-filters (R7) as bulk_p1; ghost / duplicate edges have du = 0
    {
      const double du = u0 - ul, x = rl * r0;
      cl = lane > 0 && (LIQ ? !(du * x <= e.a_l * (x - rmin2) - 1e-9 * x) : (du < -e.a_v * (2.0 - (rl + r0) * inv_rt) + 1e-9));
    }
    {
      const double du = u1 - u0, x = r0 * r1;
      sp1 |= LIQ ? !(du * x <= e.a_l * (x - rmin2) - 1e-9 * x) : (du < -e.a_v * (2.0 - (r0 + r1) * inv_rt) + 1e-9);
    }
    if (sp0 || cl) { const int cc = c0 < 0 ? 0 : (c0 >= n ? n - 1 : c0); slo = min(slo, cc); shi = max(shi, cc); }
    if (sp1) { const int cc = c1 < 0 ? 0 : (c1 >= n ? n - 1 : c1); slo = min(slo, cc); shi = max(shi, cc); }
    const double fr0 = __shfl_down_sync(0xffffffffu, fl0, 1), fr1 = __shfl_down_sync(0xffffffffu, fl1, 1);
    // P2, h^{n+1} = h^n: the pair of lanes 1..30 (own_lo is even, so both or neither
    // cell of a pair are own except the last cell of a tile with an odd end)
    const bool inner = lane >= 1 && lane <= 30;
    const bool up0 = inner && c0 >= own_lo && c0 < own_hi;
    const bool up1 = inner && c1 >= own_lo && c1 < own_hi;
    double ca = dt_hav, cb = dt_hav, ha = h_av, hb = h_av;
    if (!HU) {
      if (up0) { ha = ih[c0]; if (ha != h_av) ca = dt / ha; }
      if (up1) { hb = ih[c1]; if (hb != h_av) cb = dt / hb; }
    }
    const double n0 = r0 - ca * (fi0 - fl0), k0 = m0 - ca * (fi1 - fl1);
    const double n1 = r1 - cb * (fr0 - fi0), k1 = m1 - cb * (fr1 - fi1);
    if (up0 && up1) {  // c0 even: 16-byte aligned pair in the output tile
      *reinterpret_cast<double2*>(orho + c0) = make_double2(n0, n1);
      *reinterpret_cast<double2*>(omom + c0) = make_double2(k0, k1);
    } else if (up0) {
      orho[c0] = n0; omom[c0] = k0;
    }
    if (up0) {
      if (!HU) { oh[c0] = ha; unif &= ha == h_av; h_part = fmin(h_part, ha); }
      const double am = fabs(k0);
      if (am * sden > snum * n0) { snum = am; sden = n0; }
    }
    if (up1) {
      if (!HU) { oh[c1] = hb; unif &= hb == h_av; h_part = fmin(h_part, hb); }
      const double am = fabs(k1);
      if (am * sden > snum * n1) { snum = am; sden = n1; }
    }
  }
}

#ifndef EIS_WMAX
#define EIS_WMAX 150  // (window CTA shared memory: 16 one-warp CTAs per SM fit, the register limit)
#endif
constexpr int WMAX = EIS_WMAX;  // owned cells of a full-step window (larger: the whole tile)

// SPEC: window prediction compiled in (a template parameter: the kernel of contexts without
// predictions keeps the round-2 code generation -- 1 % on C5)
// PLAIN: one rank and no polling window kernel (the usual context): the exchange-buffer halos,
// send records, fences and ready tags are compiled out
template <bool HU, int IN, bool SPEC, bool PLAIN>  // IN: the buffer read (static, so the array bases stay parameter-bank operands)
__device__ __forceinline__ void tiled_fast_body(const Eos& e, const Prm& p, const Tiles& tl, const TGeo& g, double dt) {
  const bool gxl = !PLAIN && g.xl, gxr = !PLAIN && g.xr, tpoll = !PLAIN && tl.poll;
  const int BIN = IN >= 0 ? IN : g.in, BOUT = 1 - BIN;  // IN = -1: dynamic
  __shared__ double ps[32], ph[32];
  __shared__ int fl_or, s_lo, s_hi;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int k = g.k, n = g.n, own_lo = g.nL, own_hi = g.nL + g.cnt;
  const double h_av = p.h_av, dt_hav = dt / h_av;
  const double* const rin = tl.rho[BIN];
  const long long mo_t = tl.mom[BIN] - rin;
#if EIS_FAST_TMA
  // the tile's own cells staged in shared memory by the bulk-copy engine (one mbarrier, one
  // phase): interior windows then read shared memory; the halo windows read global memory
  extern __shared__ __align__(16) double tsm[];
  __shared__ __align__(8) unsigned long long tbar;
  const int capr = (tl.capt + 1) & ~1;
  const double* const s_rho = tsm - own_lo;  // indexed by the virtual cell
  const double* const s_mom = tsm + capr - own_lo;
  const unsigned tbar_a = (unsigned)__cvta_generic_to_shared(&tbar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tbar_a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const unsigned bytes = (unsigned)(((g.cnt + 1) & ~1) * 8);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tbar_a), "r"(2 * bytes) : "memory");
    if (bytes) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"((unsigned)__cvta_generic_to_shared(tsm)), "l"(rin + g.base), "r"(bytes), "r"(tbar_a) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"((unsigned)__cvta_generic_to_shared(tsm + capr)), "l"(rin + g.base + mo_t), "r"(bytes),
                   "r"(tbar_a) : "memory");
      // a tile with stored widths reads them from global memory in the window loop (only rho and
      // rho u are staged): bring them to L2 now (ncu source page: 11 % of the kernel's stall
      // samples sat on those loads)
      if (!HU) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tl.h[BIN] + g.base), "r"(bytes) : "memory");
    }
    fl_or = 0; s_lo = 1 << 30; s_hi = -1;
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  asm volatile("{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
               " @!P1 bra WAIT_%=;\n}" ::"r"(tbar_a) : "memory");
#else
  if (tid == 0) {  // the whole tile's requests in flight at once: bulk L2 prefetch of rho and mom
    const unsigned bytes = (unsigned)(((g.cnt + 1) & ~1) * 8);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rin + g.base), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rin + g.base + mo_t), "r"(bytes) : "memory");
    fl_or = 0; s_lo = 1 << 30; s_hi = -1;
  }
#endif
  // segment bases of the virtual array: left halo | own | right halo (density; momentum at +mo)
  const double* const segL = gxl ? tl.xbuf + XB_RECV_LEFT + HALO - g.nL : rin + g.bl + g.cl - g.nL;
  const long long moL = gxl ? HALO : mo_t;
  const double* const segO = rin + g.base - g.nL;
  const double* const segR = gxr ? tl.xbuf + XB_RECV_RIGHT - own_hi : rin + g.br - own_hi;
  const long long moR = gxr ? HALO : mo_t;
  double* const orho = tl.rho[BOUT] + g.base - own_lo;  // indexed by the virtual cell
  double* const omom = tl.mom[BOUT] + g.base - own_lo;
  double* const oh = tl.h[BOUT] + g.base - own_lo;
  const double* const ih = tl.h[BIN] + g.base - own_lo;
  int slo = 1 << 30, shi = -1;  // special cells (see fast_windows)
  bool unif = true;      // output widths all h_av
  int phases = 0;        // 1 vapour, 2 liquid: the warps' specialisations
  double snum = 0.0, sden = 1.0;  // max |m|/rho of the new cells, by cross-multiplication
  double h_part = HU ? h_av : INFINITY;
  const int nwin = (n + FW - 1) / FW;  // windows update cells [0, 60 nwin)
  // loads of the window batch starting at window w: placeholders past the tile
  auto load_batch = [&](int w, double2 (&rv)[FB], double2 (&mv)[FB]) {
#pragma unroll
    for (int b = 0; b < FB; ++b) {
      const int wi = w + nw * b;
      const int c0 = FW * wi - 2 + 2 * lane;
      rv[b] = make_double2(1.0, 1.0); mv[b] = make_double2(0.0, 0.0);
      if (wi < nwin) {
        if (FW * wi - 2 >= own_lo && FW * wi + 62 <= own_hi) {  // interior window: aligned pairs
#if EIS_FAST_TMA
          rv[b] = *reinterpret_cast<const double2*>(s_rho + c0);
          mv[b] = *reinterpret_cast<const double2*>(s_mom + c0);
#else
          rv[b] = *reinterpret_cast<const double2*>(segO + c0);
          mv[b] = *reinterpret_cast<const double2*>(segO + c0 + mo_t);
#endif
        } else {
          const int ca = c0 < 0 ? 0 : (c0 >= n ? n - 1 : c0), cb = c0 + 1 < 0 ? 0 : (c0 + 1 >= n ? n - 1 : c0 + 1);
          const double* pa = ca < own_lo ? segL : (ca < own_hi ? segO : segR);
          const long long ma = ca < own_lo ? moL : (ca < own_hi ? mo_t : moR);
          const double* pb = cb < own_lo ? segL : (cb < own_hi ? segO : segR);
          const long long mb = cb < own_lo ? moL : (cb < own_hi ? mo_t : moR);
          rv[b] = make_double2(pa[ca], pb[cb]);
          mv[b] = make_double2(pa[ca + ma], pb[cb + mb]);
        }
      }
    }
  };
  double2 rv[FB], mv[FB];
#if EIS_FAST_PIPE
  load_batch(warp, rv, mv);
#endif
  for (int w0 = warp; w0 < nwin; w0 += nw * FB) {
#if EIS_FAST_PIPE
    double2 rn[FB], mn[FB];  // the next batch's loads in flight during this batch's arithmetic
    load_batch(w0 + nw * FB, rn, mn);
#else
    load_batch(w0, rv, mv);
#endif
    // specialisation per window: liquid if any of its 64 loaded cells is liquid.  Every edge
    // lies inside some window's loaded cells, so a phase boundary always leaves a special cell
    // (the cell of the other phase) and the tile takes a window or whole-tile full step.
    unsigned lmask = 0, vmask = 0;
#pragma unroll
    for (int b = 0; b < FB; ++b) {
      if (w0 + nw * b >= nwin) break;  // warp-uniform
      vmask |= __any_sync(0xffffffffu, rv[b].x >= e.rho_min || rv[b].y >= e.rho_min) ? 0u : 1u << b;
      lmask |= vmask >> b & 1 ? 0u : 1u << b;
    }
    phases |= (lmask ? 2 : 0) | (vmask ? 1 : 0);
    if (!vmask)
      fast_pairs<HU, true, false>(e, rv, mv, w0, nw, nwin, n, own_lo, own_hi, dt, dt_hav, h_av, ih, orho, omom, oh,
                                  lmask, slo, shi, unif, snum, sden, h_part);
    else if (!lmask)
      fast_pairs<HU, false, false>(e, rv, mv, w0, nw, nwin, n, own_lo, own_hi, dt, dt_hav, h_av, ih, orho, omom, oh,
                                   vmask, slo, shi, unif, snum, sden, h_part);
    else if constexpr (FB > 1) {  // a batch whose windows differ in phase (rare): each window with its own
      fast_pairs<HU, true, true>(e, rv, mv, w0, nw, nwin, n, own_lo, own_hi, dt, dt_hav, h_av, ih, orho, omom, oh,
                                 lmask, slo, shi, unif, snum, sden, h_part);
      fast_pairs<HU, false, true>(e, rv, mv, w0, nw, nwin, n, own_lo, own_hi, dt, dt_hav, h_av, ih, orho, omom, oh,
                                  vmask, slo, shi, unif, snum, sden, h_part);
    }
#if EIS_FAST_PIPE
#pragma unroll
    for (int b = 0; b < FB; ++b) { rv[b] = rn[b]; mv[b] = mn[b]; }
#endif
  }
  // S_max of this lane's new cells: |m| rcp(rho) (+ a below, as cfl_partials; one phase)
  const double s_lane = warp_max(snum * rcp_fast(sden));
  const double h_lane = HU ? h_av : warp_min(h_part);
  const int flags = (__all_sync(0xffffffffu, unif) ? 0 : 8) | phases;
  slo = __reduce_min_sync(0xffffffffu, slo);
  shi = __reduce_max_sync(0xffffffffu, shi);
  if (lane == 0) {
    ps[warp] = s_lane; ph[warp] = h_lane;
    if (flags) atomicOr(&fl_or, flags);
    if (shi >= 0) { atomicMin(&s_lo, slo); atomicMax(&s_hi, shi); }
  }
  __syncthreads();
  const int f = fl_or;
  // owned cells within HALO (+1 for the edge) of a special cell need the full step: window [wa, wb)
  const int wa = max(own_lo, s_lo - 1 - HALO), wb = min(own_hi, s_hi + 2 + HALO);
  // both phases in the tile: its windows of one phase see the other phase's cells as special
  // (so wa < wb); the window full step handles the boundary, the fast cells are single-phase
  const bool mixed = (f & 3) == 3;
  const bool fast = !mixed && wa >= wb;
  const bool window = !fast && wa < wb && wb - wa <= tl.wmax;
  unif = !(f & 8);
  if (window) {  // partials and width uniformity of the fast cells (outside [wa, wb)), from the
                 // output just written (the window full step only moves them): as cfl_partials
    if (tpoll) __threadfence();  // output read by a window CTA running concurrently (polling mode)
    double sf = 0.0, hf = INFINITY;
    bool uf = true;
    for (int c = own_lo + tid; c < own_hi; c += blockDim.x) {
      if (c >= wa && c < wb) continue;
      const double r = orho[c], hh = HU ? h_av : oh[c];
      sf = fmax(sf, fabs(omom[c] * rcp_fast(r)) + sound(e, phase_of(e, r)));
      hf = fmin(hf, hh);
      uf &= hh == h_av;
    }
    sf = warp_max(sf);
    hf = warp_min(hf);
    uf = __all_sync(0xffffffffu, uf);
    if (lane == 0) { ps[warp] = sf; ph[warp] = hf; if (!uf) atomicOr(&fl_or, 16); }
    __syncthreads();
    if (tid == 0) {
      double s = 0.0, hm = INFINITY;
      for (int w = 0; w < nw; ++w) { s = fmax(s, ps[w]); hm = fmin(hm, ph[w]); }
      tl.partf[3 * k] = s; tl.partf[3 * k + 1] = hm; tl.partf[3 * k + 2] = (fl_or & 16) ? 0.0 : 1.0;
    }
  }
  if (fast && (gxl || gxr)) {  // rank mode: send records of the first / last HALO owned cells
    for (int q = tid; q < 2 * HALO; q += blockDim.x) {
      const bool left = q < HALO;
      if (left ? !gxl : !gxr) continue;
      const int c = left ? own_lo + q : own_hi - 2 * HALO + q;
      double* sb = tl.xbuf + (left ? XB_SEND_LEFT : XB_SEND_RIGHT) + (left ? q : q - HALO);
      sb[0] = orho[c]; sb[HALO] = omom[c]; sb[2 * HALO] = HU ? h_av : oh[c];
    }
  }
  if (tid == 0) {
    if (fast) {
      double s = 0.0, hm = INFINITY;
      for (int w = 0; w < nw; ++w) { s = fmax(s, ps[w]); hm = fmin(hm, ph[w]); }
      tl.part[2 * k] = s + ((f & 3) == 1 ? e.a_v : e.a_l);
      tl.part[2 * k + 1] = hm;
      tl.cnt[BOUT][k] = g.cnt;
      tl.hu[BOUT][k] = unif ? 1 : 0;
      tl.ws[(size_t)k * WS_STRIDE + 2 * MAXIF] = 0.0;  // no boundary: no warm start
      // fire-and-forget reduction: no load in the CTA's last instructions
      atomicAdd(reinterpret_cast<unsigned long long*>(&tl.tstats[k].cell_updates), (unsigned long long)g.cnt);
      if (gxl) tl.xbuf[XB_SEND_LEFT + 3 * HALO] = HALO;
      if (gxr) tl.xbuf[XB_SEND_RIGHT + 3 * HALO] = HALO;
    } else {
      tl.part[2 * k] = 0.0;  // neutral: the full-step kernels fold this tile's own partials
      tl.part[2 * k + 1] = INFINITY;
      if (window) {  // a window of the tile, published with this step's tag after its data
        const int j = atomicAdd(&tl.ctl[6], 1);
        tl.wlist[4 * j] = k; tl.wlist[4 * j + 1] = wa; tl.wlist[4 * j + 2] = wb;
        if (SPEC) {  // was this window predicted (its part A and DTS jobs already under way)?
          const int* pr = tl.pred[tl.ctl[3] & 1] + 4 * k;
          const int jp = pr[0];
          const bool hit = jp >= 0 && jp < tl.ctl[13] && pr[1] == s_lo - own_lo && pr[2] == s_hi - own_lo;
          tl.wlist[4 * j + 3] = hit ? jp : -1;
          atomicAdd(&tl.ctl[19], 1);
          if (hit) atomicAdd(&tl.ctl[18], 1);
          else tl.mlist[atomicAdd(&tl.ctl[20], 1)] = j;
        }
        if (tpoll) {  // only a concurrently polling window kernel reads the entry before this kernel ends
          __threadfence();
          *reinterpret_cast<volatile int*>(&tl.wlist[4 * j + 3]) = tl.ctl[3] + 1;
        }
      } else {
        tl.slow[atomicAdd(&tl.ctl[4], 1)] = k;
      }
    }
  }
}

template <int MAXT, int MINB, bool SPEC = false, bool PLAIN = false, int GEO = 0>
__global__ void __launch_bounds__(MAXT, MINB)
tiled_fast(const __grid_constant__ Eos e, const __grid_constant__ Prm p, const __grid_constant__ Tiles tl,
           double t_end) {
  const int kt = GEO == 2 ? (int)blockIdx.y * tl.tpm + (int)blockIdx.x : (int)blockIdx.x;
  const TGeo g = tile_geo_spec<PLAIN, GEO>(tl, kt, (int)blockIdx.y, (int)blockIdx.x);
  const double t = tl.scal[SCS * g.m];
  // no prediction for the next step unless this step's window step makes one (later in the stream)
  if (SPEC && threadIdx.x == 0) tl.pred[1 - (tl.ctl[3] & 1)][4 * kt] = -1;
  if (tl.mctl[MCS * g.m + 1] == 0 && t < t_end) {  // else the member does not step (uniform in the CTA)
    double dt = tl.scal[SCS * g.m + 1];
    if (t + dt > t_end) dt = t_end - t;  // as step_body
#if EIS_FAST_STATIC_IN
    if (g.in) {
      if (g.hu_in) tiled_fast_body<true, 1, SPEC, PLAIN>(e, p, tl, g, dt);
      else tiled_fast_body<false, 1, SPEC, PLAIN>(e, p, tl, g, dt);
    } else {
      if (g.hu_in) tiled_fast_body<true, 0, SPEC, PLAIN>(e, p, tl, g, dt);
      else tiled_fast_body<false, 0, SPEC, PLAIN>(e, p, tl, g, dt);
    }
#else
    if (g.hu_in) tiled_fast_body<true, -1, SPEC, PLAIN>(e, p, tl, g, dt);
    else tiled_fast_body<false, -1, SPEC, PLAIN>(e, p, tl, g, dt);
#endif
  }
  if (!PLAIN && tl.poll) {  // count finished CTAs for the polling window kernel (every CTA, always)
    __syncthreads();
    if (threadIdx.x == 0) { __threadfence(); atomicAdd(&tl.ctl[9], 1); }
  }
}

// ------------------------------------------------------------------------------------------
// The full step of tile k (shared memory): load tile + halos, step_body, owned output after
// the remesh, CFL partials, warm-start table, stats.  Returns (via s_out/h_out on thread 0)
// the tile's partials; a status is raised on tl.ctl[1].
// ------------------------------------------------------------------------------------------
// per-tile counters as fire-and-forget reductions (no load in the CTA's critical path)
__device__ __forceinline__ void tstats_add(const Tiles& tl, int k, long long cells, const CtaShared& sh, bool window) {
  TileStats& ts = tl.tstats[k];
  auto add = [](long long* a, long long v) {
    if (v) atomicAdd(reinterpret_cast<unsigned long long*>(a), (unsigned long long)v);
  };
  add(&ts.cell_updates, cells);
  add(&ts.dts_iters, (long long)sh.c_dts);
  add(&ts.iface_solves, (long long)sh.c_solves);
  add(&ts.regions, (long long)sh.c_regions);
  add(&ts.margins, (long long)sh.c_margin);
  if (sh.c_dtsmax) atomicMax(reinterpret_cast<unsigned long long*>(&ts.dts_max), (unsigned long long)sh.c_dtsmax);
  add(window ? &ts.win_steps : &ts.full_steps, 1);
  add(&ts.creations, sh.st.creations);  // owned events only (step_body)
  add(&ts.splits, sh.st.splits);
  add(&ts.merges, sh.st.merges);
}

__device__ __forceinline__ void tile_full(const Eos& e, const Prm& p, const Tiles& tl, CtaShared& sh, Arr& A, int capg,
                                          int k, double t_end, double& s_out, double& h_out) {
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  const TGeo g = tile_geo_spec(tl, k);
  const double t = tl.scal[SCS * g.m], dt_given = tl.scal[SCS * g.m + 1];
  const int n = g.n, nL = g.nL, cnt = g.cnt;
  if (tid == 0) {
    sh.status = 0;
    reset_counters(sh);
    memset(&sh.st, 0, sizeof(sh.st));
    const double* ws = tl.ws + (size_t)k * WS_STRIDE;
    sh.wsn = (int)ws[2 * MAXIF];
    for (int q = 0; q < MAXIF; ++q) { sh.ws0[q] = ws[q]; sh.ws1[q] = ws[MAXIF + q]; }
  }
  const int huL = g.huL, huR = g.huR;
  for (int i = tid; i < n; i += T) {
    long long mo;
    const double* pr = vcell(tl, g, i, mo);
    A.rho[i] = pr[0];
    A.mom[i] = pr[mo];
    double hh;
    if (i < nL) hh = g.xl ? pr[2 * HALO] : (huL ? p.h_av : tl.h[g.in][g.bl + g.cl - nL + i]);
    else if (i < nL + cnt) hh = g.hu_in ? p.h_av : tl.h[g.in][g.base + i - nL];
    else hh = g.xr ? pr[2 * HALO] : (huR ? p.h_av : tl.h[g.in][g.br + i - nL - cnt]);
    A.h[i] = hh;
  }
  for (int i = tid; i <= capg; i += T) A.fl[i] = 0;
  A.n = n;
  __syncthreads();
  if (warp == nw - 1) build_boundary_list(e, sh, A.rho, A.fl, n);
  __syncthreads();
  Zone Z;
  Z.own_lo = nL; Z.own_hi = nL + cnt;
  Z.zlo = max(nL - 2, 0); Z.zhi = min(nL + cnt + 2, n);
  Z.dt_given = dt_given;
  Z.s_given = tl.scal[SCS * g.m + 5];
  Z.left_real = (g.first && !tl.nbr_left); Z.right_real = (g.last && !tl.nbr_right);
  const double dt = step_body(e, p, sh, A, t, t_end, Z);
  __syncthreads();
  const int olo = sh.olo, ohi = sh.ohi;
  const int nout = ohi - olo;
  int st = sh.status;
  if (dt >= 0.0 && st == 0 && (nout > tl.capt || nout < (tl.tpm > 1 ? HALO : 3))) st = ST_CAPACITY;
  bool unif = true;
  if (dt >= 0.0 && st == 0) {
    bool u = true;  // widths all h_av?  then they are not stored
    for (int i = olo + tid; i < ohi; i += T) u &= A.h[i] == p.h_av;
    unif = __syncthreads_and(u);
    const long long ob = g.base;
    for (int i = tid; i < nout; i += T) {
      tl.rho[g.out][ob + i] = A.rho[olo + i];
      tl.mom[g.out][ob + i] = A.mom[olo + i];
      if (!unif) tl.h[g.out][ob + i] = A.h[olo + i];
    }
    if (g.xl) {  // my first HALO owned cells go to the left rank (its right halo)
      double* sb = tl.xbuf + XB_SEND_LEFT;
      for (int i = tid; i < HALO; i += T) { sb[i] = A.rho[olo + i]; sb[HALO + i] = A.mom[olo + i]; sb[2 * HALO + i] = A.h[olo + i]; }
      if (tid == 0) sb[3 * HALO] = HALO;
    }
    if (g.xr) {  // my last HALO owned cells go to the right rank (its left halo)
      double* sb = tl.xbuf + XB_SEND_RIGHT;
      for (int i = tid; i < HALO; i += T) {
        const int j = ohi - HALO + i;
        sb[i] = A.rho[j]; sb[HALO + i] = A.mom[j]; sb[2 * HALO + i] = A.h[j];
      }
      if (tid == 0) sb[3 * HALO] = HALO;
    }
    double s, hm;
    cfl_partials(e, p, A.rho, A.mom, A.h, A.n, olo, ohi, false, false, s, hm);
    if (lane == 0) { sh.part_s[warp] = s; sh.part_h[warp] = hm; }
  }
  __syncthreads();
  if (tid == 0) {
    s_out = 0.0; h_out = INFINITY;
    if (st != 0) { atomicCAS(&tl.mctl[MCS * g.m + 1], 0, st); atomicCAS(&tl.ctl[1], 0, st); }
    if (dt >= 0.0 && st == 0) {
      for (int w = 0; w < nw; ++w) { s_out = fmax(s_out, sh.part_s[w]); h_out = fmin(h_out, sh.part_h[w]); }
      tl.part[2 * k] = s_out;
      tl.part[2 * k + 1] = h_out;
      tl.cnt[g.out][k] = nout;
      tl.hu[g.out][k] = unif ? 1 : 0;
      double* ws = tl.ws + (size_t)k * WS_STRIDE;
      for (int q = 0; q < MAXIF; ++q) { ws[q] = sh.ws0[q]; ws[MAXIF + q] = sh.ws1[q]; }
      ws[2 * MAXIF] = (double)sh.wsn;
      tstats_add(tl, k, cnt, sh, false);
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// The full step of a window [wa, wb) of tile k's owned cells (virtual indices) that holds every
// special cell of the tile with a margin of HALO: step_body on the window plus HALO cells each
// side (shared memory), then the tile's output is assembled in place: the fast results left of
// the window stay, the window's remeshed cells follow, the fast results right of it shift by
// the change in cell count.  Cells outside the window are plain (one phase, both edges HLL, no
// block, creation or remesh event within HALO cells), so their fast results are step_body's.
// ------------------------------------------------------------------------------------------
constexpr int WCAP = WMAX + 2 * HALO + MAXEV + MAXTRG + 2;  // window grid capacity (even)

// Fast cells of a window tile: out[s, e) moves to out[s + d, e + d) (d = 0: stays), and their
// CFL partials (plain cells: |m| rcp(rho) + a, never tiny) and width uniformity are folded on
// the way.  Block-wide, chunks of FP_U x blockDim cells with all loads in flight; chunks run
// against the direction of the move, so overlapping ranges are safe.
constexpr int FP_U = 4;
__device__ __forceinline__ void fast_part_pass(const Eos& e, double* orho, double* omom, double* oh, double h_av,
                                               int s, int en, int d, double& sf, double& hf, bool& uf) {
  if (s >= en) return;
  const int T = blockDim.x, tid = threadIdx.x, CH = FP_U * T;
  const int nch = (en - s + CH - 1) / CH;
  for (int q = 0; q < nch; ++q) {
    const int lo = d > 0 ? max(s, en - (q + 1) * CH) : s + q * CH;
    const int hi = d > 0 ? en - q * CH : min(en, s + (q + 1) * CH);
    double r[FP_U], m[FP_U], h[FP_U];
#pragma unroll
    for (int u = 0; u < FP_U; ++u) {
      const int i = lo + tid + u * T;
      r[u] = 1.0; m[u] = 0.0; h[u] = h_av;
      if (i < hi) { r[u] = orho[i]; m[u] = omom[i]; if (oh) h[u] = oh[i]; }
    }
#pragma unroll
    for (int u = 0; u < FP_U; ++u) {
      if (lo + tid + u * T < hi) {
        sf = fmax(sf, fabs(m[u] * rcp_fast(r[u])) + sound(e, phase_of(e, r[u])));
        hf = fmin(hf, h[u]);
        uf &= h[u] == h_av;
      }
    }
    if (d != 0) {
      __syncthreads();
#pragma unroll
      for (int u = 0; u < FP_U; ++u) {
        const int i = lo + tid + u * T;
        if (i < hi) { orho[i + d] = r[u]; omom[i + d] = m[u]; if (oh) oh[i + d] = h[u]; }
      }
      __syncthreads();
    }
  }
}

// Window split (tl.split): part A (PH = 1) runs the step body up to the remesh with the blocks
// exported as DTS jobs and saves the window (CtaShared, n, dt, rho / mom / h) to the job's
// slot; dts_jobs solves every job of the step, one lane each; part B (PH = 2) restores the slot,
// applies the DTS results, finishes the step (remesh) and assembles the tile output.
constexpr size_t WSAVE_SH = (sizeof(CtaShared) + 15) & ~size_t(15);
// the saved prefix of the window CTA's shared memory: CtaShared | rho | mom | h (carve layout)
constexpr size_t WSAVE = (WSAVE_SH + 3 * 8 * (size_t)(WCAP + 1) + 15) & ~size_t(15);
// one TMA bulk copy each way (cp.async.bulk, shared <-> global): a window is saved and restored
// in one transfer instead of a loop of dependent loads
__device__ __forceinline__ void window_save(const Tiles& tl, CtaShared& sh, const Arr& A, int j, double dt) {
  if (threadIdx.x == 0) { sh.sv_n = A.n; sh.sv_dt = dt; }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned char* slot = tl.wsave + (size_t)j * WSAVE;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(slot), "r"((unsigned)__cvta_generic_to_shared(&sh)), "r"((unsigned)WSAVE) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // shared memory free for the next job
  }
  __syncthreads();
}
// (the CTA's mbarrier `bar` is initialised once by the kernel and used phase after phase: `par` is
// the parity of the phase this restore completes, flipped here for the next one -- an mbarrier
// must not be initialised again while it is a valid object)
__device__ __forceinline__ double window_restore(const Tiles& tl, CtaShared& sh, Arr& A, int j, unsigned bar, unsigned& par) {
  if (threadIdx.x == 0) {
    const unsigned char* slot = tl.wsave + (size_t)j * WSAVE;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((unsigned)WSAVE) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((unsigned)__cvta_generic_to_shared(&sh)), "l"(slot), "r"((unsigned)WSAVE), "r"(bar) : "memory");
  }
  asm volatile("{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               " @!P1 bra WAIT_%=;\n}" ::"r"(bar), "r"(par) : "memory");
  par ^= 1u;
  A.n = sh.sv_n;
  return sh.sv_dt;
}

// Window prediction: after a window's full step, which cells of this tile will tiled_fast flag
// as special in the NEXT step?  tiled_fast's own tests (fast_pairs: the cell tests of the warp
// window's specialisation and the creation pre-filter of every edge inside a warp window),
// evaluated on the window grid after the step (cells [0, nl); local cell i will be virtual cell
// v0 + i of the next step's tile, n_next cells in all); the cells outside the grid are the
// tile's plain cells, taken to keep the phase of the grid's end cells.  One warp.  Returns the
// range [qlo, qhi] of flagged cells as local indices (qhi < 0: none).  A guess by design: the
// next tiled_fast decides (a wrong guess only sends that window down the late path).
__device__ __forceinline__ void predict_special(const Eos& e, const double* rho, const double* mom, int nl, int v0,
                                                int n_next, int& qlo, int& qhi) {
  const int lane = threadIdx.x & 31;
  const double rho_min = e.rho_min, rho_tilde = e.rho_tilde, rmin2 = rho_min * rho_min, inv_rt = 1.0 / rho_tilde;
  const int nwin = (n_next + FW - 1) / FW;
  const int w_lo = max(0, (v0 - 61 + FW - 1) / FW), w_hi = min(nwin - 1, (v0 + nl - 1 + 2) / FW);
  const bool left_liq = rho[0] >= rho_min, right_liq = rho[nl - 1] >= rho_min;
  unsigned liqm = 0;  // bit w - w_lo: warp window w takes the liquid specialisation
  for (int w = w_lo; w <= w_hi && w - w_lo < 32; ++w) {
    const int ca = FW * w - 2, cb = FW * w + 61;  // its loaded cells (clamped to the grid by tiled_fast)
    bool any = (max(ca, 0) < v0 && left_liq) || (min(cb, n_next - 1) >= v0 + nl && right_liq);
    for (int c = ca + lane; c <= cb; c += 32) {
      const int i = c - v0;
      if (i >= 0 && i < nl) any |= rho[i] >= rho_min;
    }
    if (__any_sync(0xffffffffu, any)) liqm |= 1u << (w - w_lo);
  }
  int lo = 1 << 30, hi = -1;
  for (int i = lane; i < nl; i += 32) {
    const int v = v0 + i;
    const double r = rho[i];
    bool flagged = false;
    const int wa = max(w_lo, (v - 61 + FW - 1) / FW), wb = min(w_hi, (v + 2) / FW);
    for (int w = wa; w <= wb; ++w) {
      const bool L = liqm >> (w - w_lo) & 1u;
      flagged |= L ? !(r >= rho_min) : !(r <= rho_tilde && r > 0.0);
      if (i >= 1 && v >= FW * w - 1) {  // the edge (v - 1, v) lies inside window w
        const double rl = rho[i - 1];
        const double du = mom[i] * rcp_fast(r) - mom[i - 1] * rcp_fast(rl), x = rl * r;
        flagged |= L ? !(du * x <= e.a_l * (x - rmin2) - 1e-9 * x) : (du < -e.a_v * (2.0 - (rl + r) * inv_rt) + 1e-9);
      }
    }
    if (flagged) { lo = min(lo, i); hi = max(hi, i); }
  }
  qlo = __reduce_min_sync(0xffffffffu, lo);
  qhi = __reduce_max_sync(0xffffffffu, hi);
}

// The next window job of part PH from list SRC (0: tiled_fast's window list; 1: the predicted
// windows, part A beside tiled_fast).  Returns its index (< 0: the list is exhausted) with the
// tile, the window and its save slot.  With predictions on, a listed window whose prediction
// held (tiled_fast stored its early slot in the entry) skips the late part A and part B reads
// the early slot; the others use the slots above ntiles.
template <int PH, int SRC>
__device__ __forceinline__ int claim_window_job(const Tiles& tl, double t_end, int& k, int& wa, int& wb, int& slot) {
  for (;;) {
    if constexpr (SRC == 1) {
      const int j = atomicAdd(&tl.ctl[15], 1);
      if (j >= tl.ctl[13]) return -1;
      const int par = tl.ctl[3] & 1;
      k = tl.plist[par][j];
      if (k < 0) continue;  // that window made no prediction
      const int* pr = tl.pred[par] + 4 * k;
      const int qlo = pr[1], qhi = pr[2];
      const TGeo g = tile_geo_spec(tl, k);
      if (!(tl.mctl[MCS * g.m + 1] == 0 && tl.scal[SCS * g.m] < t_end)) continue;  // the member does not step
      const int own_lo = g.nL, own_hi = g.nL + g.cnt;
      wa = max(own_lo, own_lo + qlo - 1 - HALO);  // as tiled_fast's classification
      wb = min(own_hi, own_lo + qhi + 2 + HALO);
      if (wa >= wb || wb - wa > tl.wmax) continue;  // tiled_fast would not list such a window
      slot = j;
      return j;
    } else {
      int j = atomicAdd(&tl.ctl[PH == 2 ? 11 : 7], 1);
      if (PH == 1 && tl.spec) {  // the late part A: only the windows whose prediction failed
        if (j >= tl.ctl[20]) return -1;
        j = tl.mlist[j];
      } else if (j >= tl.ctl[6]) return -1;
      k = tl.wlist[4 * j]; wa = tl.wlist[4 * j + 1]; wb = tl.wlist[4 * j + 2];
      slot = j;
      if (tl.spec) {
        const int jp = tl.wlist[4 * j + 3];
        slot = jp >= 0 ? jp : tl.ntiles + j;
      }
      return j;
    }
  }
}

// PF: after the step body, thread 0 claims the next window job and loads its list entry into
// registers (jn, kn, wan, wbn; jn = -1 when the list is exhausted); the loads complete during the
// assembly and the caller publishes them, so the next job starts without those round trips.
template <bool PF, int PH = 0, int SRC = 0>
__device__ __forceinline__ void tile_window(const Eos& e, const Prm& p, const Tiles& tl, CtaShared& sh, Arr& A, int capw,
                                            int slot, int k, int wa, int wb, double t_end, int& jn, int& kn, int& wan,
                                            int& wbn, int& slotn, unsigned wbar = 0, unsigned* wpar = nullptr, int jlist = 0) {
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  const TGeo g = tile_geo_spec(tl, k);
  const double t = tl.scal[SCS * g.m], dt_given = tl.scal[SCS * g.m + 1];
  const int nL = g.nL, cnt = g.cnt;
  const int s0 = max(0, wa - HALO), s1 = min(g.n, wb + HALO), n = s1 - s0;
  const int spec_npar = (PH == 2 && tl.spec) ? 1 - (tl.ctl[3] & 1) : 0;           // window prediction (below)
  const bool spec_sparse = PH == 2 && tl.spec && 4 * tl.ctl[6] <= tl.ntiles;
  if (PH != 2 && tid == 0) {
    sh.status = 0;
    reset_counters(sh);
    memset(&sh.st, 0, sizeof(sh.st));
#ifdef EIS_DTS_CLOCK
    for (int q = 0; q < 5; ++q) sh.dclk[q] = 0;
#endif
    const double* ws = tl.ws + (size_t)k * WS_STRIDE;
    sh.wsn = (int)ws[2 * MAXIF];
    for (int q = 0; q < MAXIF; ++q) { sh.ws0[q] = ws[q]; sh.ws1[q] = ws[MAXIF + q]; }
  }
  const int huL = g.huL, huR = g.huR;
  if (PH != 2) {
    // the window's cells: every load of the thread first, then the shared-memory stores (the
    // loads of one thread are independent, so they are all in flight together)
    constexpr int LU = (WCAP + 31) / 32;
    double lr[LU], lm[LU], lh[LU];
#pragma unroll
    for (int u = 0; u < LU; ++u) {
      const int i = tid + 32 * u, v = s0 + i;
      lr[u] = 0.0; lm[u] = 0.0; lh[u] = 0.0;
      if (i < n) {
        long long mo;
        const double* pr = vcell(tl, g, v, mo);
        lr[u] = pr[0];
        lm[u] = pr[mo];
        if (v < nL) lh[u] = g.xl ? pr[2 * HALO] : (huL ? p.h_av : tl.h[g.in][g.bl + g.cl - nL + v]);
        else if (v < nL + cnt) lh[u] = g.hu_in ? p.h_av : tl.h[g.in][g.base + v - nL];
        else lh[u] = g.xr ? pr[2 * HALO] : (huR ? p.h_av : tl.h[g.in][g.br + v - nL - cnt]);
      }
    }
#pragma unroll
    for (int u = 0; u < LU; ++u) {
      const int i = tid + 32 * u;
      if (i < n) { A.rho[i] = lr[u]; A.mom[i] = lm[u]; A.h[i] = lh[u]; }
    }
    for (int i = tid; i <= capw; i += T) A.fl[i] = 0;
    A.n = n;
    __syncthreads();
    if (warp == nw - 1) build_boundary_list(e, sh, A.rho, A.fl, n);
    __syncthreads();
  }
  EIS_TCLK(0);
  Zone Z;
  Z.own_lo = wa - s0; Z.own_hi = wb - s0;
  Z.zlo = max(Z.own_lo - 2, 0); Z.zhi = min(Z.own_hi + 2, n);
  Z.dt_given = dt_given;
  Z.s_given = tl.scal[SCS * g.m + 5];
  Z.left_real = (g.first && !tl.nbr_left && s0 == 0);
  Z.right_real = (g.last && !tl.nbr_right && s1 == g.n);
  Z.djobs = tl.djobs; Z.djn = &tl.ctl[10]; Z.djcap = tl.djcap;
  double dt;
  if constexpr (PH == 0) {
    dt = step_body<0>(e, p, sh, A, t, t_end, Z);
  } else if constexpr (PH == 1) {  // part A: up to the remesh, blocks exported; the window saved
    dt = step_body<1>(e, p, sh, A, t, t_end, Z);
    window_save(tl, sh, A, slot, dt);
    if (PF && tid == 0) jn = claim_window_job<PH, SRC>(tl, t_end, kn, wan, wbn, slotn);
    __syncthreads();
    return;
  } else {  // part B: the saved window, the DTS results, the rest of the step
    dt = window_restore(tl, sh, A, slot, wbar, *wpar);
    __syncthreads();
    if (dt >= 0.0 && sh.status == 0) {
      apply_dts_jobs(p, sh, A, Z, tl.djobs);
      __syncthreads();
      dt = step_tail(e, p, sh, A, A.n, sh.ntrg < MAXTRG ? sh.ntrg : MAXTRG, dt, Z);
    }
  }
  if (PF && tid == 0) jn = claim_window_job<PH, SRC>(tl, t_end, kn, wan, wbn, slotn);
  __syncthreads();
  const int olo = sh.olo, ohi = sh.ohi;
  const int nw_out = ohi - olo;
  const int d = nw_out - (wb - wa);
  const int nout = cnt + d;
  int st = sh.status;
  if (dt >= 0.0 && st == 0 && (nout > tl.capt || nout < (tl.tpm > 1 ? HALO : 3))) st = ST_CAPACITY;
  __syncthreads();
  double s_th = 0.0, h_th = INFINITY;
  bool unif = true;
  if (dt >= 0.0 && st == 0) {
    double* const orho = tl.rho[g.out] + g.base;
    double* const omom = tl.mom[g.out] + g.base;
    double* const oh = tl.h[g.out] + g.base;
    const int pa = wa - nL;  // output position of the window's first cell
    // fast cells: left of the window stay, right of it shift by d; their partials and width
    // uniformity were folded by tiled_fast (tl.partf)
    double sf = 0.0, hf = INFINITY;
    bool uf = true;
    if (d != 0) fast_part_pass(e, orho, omom, g.hu_in ? nullptr : oh, p.h_av, wb - nL, cnt, d, sf, hf, uf);
    sf = tl.partf[3 * k]; hf = tl.partf[3 * k + 1]; uf = tl.partf[3 * k + 2] != 0.0;
    bool uw = true;
    for (int i = olo + tid; i < ohi; i += T) uw &= A.h[i] == p.h_av;
    unif = __syncthreads_and(uw && uf);
    for (int i = tid; i < nw_out; i += T) {
      orho[pa + i] = A.rho[olo + i];
      omom[pa + i] = A.mom[olo + i];
      if (!unif) oh[pa + i] = A.h[olo + i];
    }
    if (!unif && g.hu_in)
      for (int q = tid; q < nout; q += T)
        if (q < pa || q >= pa + nw_out) oh[q] = p.h_av;
    // CFL partials: the window's cells (tiny test inside the window grid) and the fast cells
    double s, hm;
    cfl_partials(e, p, A.rho, A.mom, A.h, A.n, olo, ohi, false, false, s, hm);
    s_th = fmax(s, sf);
    h_th = fmin(hm, hf);
    __syncthreads();
    if (g.xl || g.xr) {  // rank mode: send records of the first / last HALO output cells
      for (int q = tid; q < 2 * HALO; q += T) {
        const bool left = q < HALO;
        if (left ? !g.xl : !g.xr) continue;
        const int c = left ? q : nout - 2 * HALO + q;
        double* sb = tl.xbuf + (left ? XB_SEND_LEFT : XB_SEND_RIGHT) + (left ? q : q - HALO);
        sb[0] = orho[c]; sb[HALO] = omom[c]; sb[2 * HALO] = unif ? p.h_av : oh[c];
      }
      if (tid == 0) {
        if (g.xl) tl.xbuf[XB_SEND_LEFT + 3 * HALO] = HALO;
        if (g.xr) tl.xbuf[XB_SEND_RIGHT + 3 * HALO] = HALO;
      }
    }
  }
  // the tile's window of the next step, predicted (only while at most a quarter of the tiles hold a
  // window: part A of many windows is throughput work that costs tiled_fast more than the hidden
  // DTS latency is worth -- measured on C3); the early slot is this window's list index
  if (tl.spec && PH == 2 && T == 32) {
    int pk = -1, plo = 0, phi = 0;
    if (dt >= 0.0 && st == 0 && spec_sparse) {
      const int nLn = g.first ? 0 : HALO, nRn = g.last ? 0 : HALO;  // next step's halos (neighbours hold >= HALO cells)
      const int pa = wa - nL;
      int qlo, qhi;
      predict_special(e, A.rho, A.mom, A.n, nLn + pa - olo, nLn + nout + nRn, qlo, qhi);
      plo = pa + qlo - olo; phi = pa + qhi - olo;  // positions relative to the first owned cell
      const int lo2 = max(0, plo - 1 - HALO), hi2 = min(nout, phi + 2 + HALO);
      if (qhi >= 0 && lo2 < hi2 && hi2 - lo2 <= tl.wmax) pk = k;
    }
    if (tid == 0) {
      tl.plist[spec_npar][jlist] = pk;
      if (pk >= 0) { int* pr = tl.pred[spec_npar] + 4 * k; pr[1] = plo; pr[2] = phi; pr[0] = jlist; }
    }
  }
  if (lane == 0) { sh.part_s[warp] = s_th; sh.part_h[warp] = h_th; }
  __syncthreads();
  if (tid == 0) {
    if (st != 0) { atomicCAS(&tl.mctl[MCS * g.m + 1], 0, st); atomicCAS(&tl.ctl[1], 0, st); }
    if (dt >= 0.0 && st == 0) {
      double so = 0.0, ho = INFINITY;
      for (int w = 0; w < nw; ++w) { so = fmax(so, sh.part_s[w]); ho = fmin(ho, sh.part_h[w]); }
      tl.part[2 * k] = so;
      tl.part[2 * k + 1] = ho;
      tl.cnt[g.out][k] = nout;
      tl.hu[g.out][k] = unif ? 1 : 0;
      double* ws = tl.ws + (size_t)k * WS_STRIDE;
      for (int q = 0; q < MAXIF; ++q) { ws[q] = sh.ws0[q]; ws[MAXIF + q] = sh.ws1[q]; }
      ws[2 * MAXIF] = (double)sh.wsn;
      tstats_add(tl, k, cnt, sh, true);
    }
  }
  __syncthreads();
}

// EIS_WINDOW_DEBUG record of window job j (thread 0, after its full step)
__device__ __forceinline__ void window_dbg(const Tiles& tl, const CtaShared& sh, int j, int wa, int wb, long long c0) {
  long long* d = tl.wdbg + WDBG_FIELDS * (long long)j;
  d[0] = clock64() - c0; d[1] = (long long)sh.c_dts; d[2] = wb - wa;
  d[3] = sh.nifc; d[4] = c0;
#ifdef EIS_PHASE_CLOCK
  // phases: load+list | to arrival at A | arrival A -> arrival B | S4 (DTS) | B -> step end | assembly
  long long* q = d + 5;
  q[0] = sh.tclk[0] - c0;
  q[1] = sh.tclk[1] - sh.tclk[0];
  q[2] = sh.tclk[3] - sh.tclk[1];
  q[3] = sh.tclk[7] - sh.tclk[6];
  q[4] = sh.tclk[5] - sh.tclk[3];
  q[5] = clock64() - sh.tclk[5];
#endif
#ifdef EIS_DTS_CLOCK
  for (int q = 0; q < 5; ++q) d[5 + q] = sh.dclk[q];
  d[10] = (long long)sh.c_solves;
#endif
#if defined(EIS_FINE_CLOCK) && defined(EIS_PHASE_CLOCK)
  // load+list | S1+S2 | P1 | barrier A + dt | S4+S5+P2+barrier B | creations | remesh + assembly
  d[4] = sh.tclk[0] - c0;
  d[5] = sh.fclk[7] - sh.tclk[0]; d[6] = sh.fclk[1] - sh.fclk[0]; d[7] = sh.fclk[2] - sh.fclk[1];
  d[8] = sh.fclk[4] - sh.fclk[2]; d[9] = sh.fclk[0] - sh.fclk[7]; d[10] = clock64() - sh.fclk[5];
#endif
}

// tiled_win: persistent CTAs over the window list.  POLL (the instance launched beside
// tiled_fast on a second stream): a job index is waited for until its entry carries this step's
// tag, or until every tiled_fast CTA has finished and the index is past the list (or a status
// was raised).  The instance launched after tiled_fast (POLL = false) drains the same list.
// dts_jobs (window split): Algorithm 2 on every block exported by the window kernel's part A
// this step, one lane per block (dts_thread: the boundary solves of a block run on its lane),
// so the blocks of all windows iterate side by side instead of one block per window warp.
// (Tried: two lanes per block, each solving every other interior edge with the fluxes exchanged
// by shuffles -- 4 % slower on C5: the per-lane chain is the boundary solver's math either way.)
// blocks of more than 3 cells (rare: overlapping regions R11, merged blocks): out of line, so
// the usual block's code keeps its registers
__device__ __noinline__ void run_dts_job_gen(const Eos& e, const Prm& p, DtsJob& J) { run_dts_job<MAXB>(e, p, J); }
#ifdef EIS_DTS_DEBUG
__global__ void dts_dbg_print() {
  printf("dtsdbg solves %llu newton_its %llu evals %llu armijo_evals %llu retries %llu lin_exits %llu\n", g_dbg[0], g_dbg[1],
         g_dbg[2], g_dbg[3], g_dbg[4], g_dbg[5]);
  for (int i = 0; i < 8; ++i) g_dbg[i] = 0;
}
#endif
// (window prediction: the early launch, beside tiled_fast, solves the jobs of the predicted
// windows and leaves their count in ctl[17]; the launch after the late part A solves the rest)
__global__ void __launch_bounds__(32)
dts_jobs(const __grid_constant__ Eos e, const __grid_constant__ Prm p, const __grid_constant__ Tiles tl, int early) {
  const int n = tl.ctl[10] < tl.djcap ? tl.ctl[10] : tl.djcap;
  const int q0 = early ? 0 : tl.ctl[17];
  if (early && blockIdx.x == 0 && threadIdx.x == 0) tl.ctl[17] = n;  // (every job of part A beside tiled_fast is listed by now)
  for (int q = q0 + blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    DtsJob& J = tl.djobs[q];
#ifdef EIS_DTS_DEBUG  // development: the longest jobs of a step
    const long long c0 = clock64();
#endif
    if (J.K == 3) run_dts_job<3>(e, p, J);  // one tiny cell: the usual block
    else run_dts_job_gen(e, p, J);
#ifdef EIS_DTS_DEBUG
    const long long dc = clock64() - c0;
    if (dc > 400000) printf("dtsjob q %d K %d it %lld solves %d cycles %lld hn %.3e %.3e %.3e tiny %d\n", q, J.K, J.it, J.solves, dc,
                            J.hn[0], J.hn[1], J.hn[2], J.tiny);
#endif
  }
}

template <int MAXT, int MINB, bool POLL, int PH = 0, int SRC = 0>
__global__ void __launch_bounds__(MAXT, MINB)
tiled_win(const __grid_constant__ Eos e, const __grid_constant__ Prm p, const __grid_constant__ Tiles tl,
          double t_end) {
  static_assert(!POLL || PH <= 1, "a polling instance runs the whole window step or part A");
  static_assert(SRC == 0 || (!POLL && PH == 1), "the predicted windows only run part A");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CtaShared& sh = *reinterpret_cast<CtaShared*>(smem_raw);
  Arr A = carve(smem_raw, WCAP);
  const int tid = threadIdx.x;
  const int tag = tl.ctl[3] + 1;
  volatile int* vctl = tl.ctl;
  if constexpr (!POLL) {  // the next job is claimed during the current one's assembly (tile_window<true>)
    // window prediction: an empty job list (no early jobs; every listed window predicted) ends the
    // CTA before its first atomic
    if (SRC == 1 && tl.ctl[13] == 0) return;
    if (SRC == 0 && PH == 1 && tl.spec && tl.ctl[20] == 0) return;
    __shared__ __align__(8) unsigned long long wbar_s;  // part B: the restores' mbarrier, one phase per job
    const unsigned wbar = (unsigned)__cvta_generic_to_shared(&wbar_s);
    unsigned wpar = 0;
    if (PH == 2 && tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wbar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid == 0) {
      int k = 0, wa = 0, wb = 0, slot = 0;
      sh.pf_j = claim_window_job<PH, SRC>(tl, t_end, k, wa, wb, slot);
      sh.pf_k = k; sh.pf_wa = wa; sh.pf_wb = wb; sh.pf_slot = slot;
    }
    __syncthreads();
    for (;;) {
      const int j = sh.pf_j, k = sh.pf_k, wa = sh.pf_wa, wb = sh.pf_wb, slot = sh.pf_slot;
      if (j < 0) break;
      __syncthreads();  // every lane has read the job before thread 0 replaces it
      const long long c0 = clock64();
      int jn = -1, kn = 0, wan = 0, wbn = 0, slotn = 0;
      tile_window<true, PH, SRC>(e, p, tl, sh, A, WCAP, slot, k, wa, wb, t_end, jn, kn, wan, wbn, slotn, wbar, &wpar, j);
      if (tl.wdbg && tid == 0 && SRC == 0) window_dbg(tl, sh, j, wa, wb, c0);
      if (tid == 0) { sh.pf_j = jn; sh.pf_k = kn; sh.pf_wa = wan; sh.pf_wb = wbn; sh.pf_slot = slotn; }
      __syncthreads();
    }
  } else {
    for (;;) {
      __syncthreads();
      if (tid == 0) {
        int j = atomicAdd(&tl.ctl[7], 1);
        volatile int* ready = reinterpret_cast<volatile int*>(&tl.wlist[4 * j + 3]);
        if (POLL) {
#ifdef EIS_POLL_DEBUG
          long long spins = 0;
#endif
          for (;;) {
            if (j < vctl[6] && *ready == tag) break;
            if (vctl[1] != 0 || (vctl[9] >= tl.ntiles && j >= vctl[6])) { j = -1; break; }
            __nanosleep(256);
#ifdef EIS_POLL_DEBUG
            if (++spins == 4000000) {
              printf("poll stuck: cta %d j %d ctl6 %d ctl7 %d ctl9 %d ntiles %d tag %d ready %d ctl1 %d\n", blockIdx.x, j,
                     vctl[6], vctl[7], vctl[9], tl.ntiles, tag, j < 4 * tl.ntiles ? *ready : -7, vctl[1]);
              j = -1; break;
            }
#endif
          }
        } else if (j >= vctl[6]) {
          j = -1;
        }
        __threadfence();
        sh.n_new = j;
      }
      __syncthreads();
      const int j = sh.n_new;
      if (j < 0) break;
      const long long c0 = clock64();
      int jn, kn, wan, wbn, slotn;
      tile_window<false, PH>(e, p, tl, sh, A, WCAP, j, tl.wlist[4 * j], tl.wlist[4 * j + 1], tl.wlist[4 * j + 2], t_end,
                             jn, kn, wan, wbn, slotn);
      if (tl.wdbg && tid == 0) window_dbg(tl, sh, j, tl.wlist[4 * j + 1], tl.wlist[4 * j + 2], c0);
    }
  }
}

// ------------------------------------------------------------------------------------------
// tiled_slow: persistent CTAs take listed tiles one at a time (dynamic: DTS-heavy tiles vary a
// lot), fold the fast tiles' partials in strides, and the last CTA finishes the step.
// ------------------------------------------------------------------------------------------
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
tiled_slow(const __grid_constant__ Eos e, const __grid_constant__ Prm p, const __grid_constant__ Tiles tl,
           double t_end) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CtaShared& sh = *reinterpret_cast<CtaShared*>(smem_raw);
  const int capg = tl.capt + 2 * HALO + MAXEV + 1;  // even array stride (16-byte aligned rows)
  Arr A = carve(smem_raw, capg);
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  const bool one = tl.M == 1;  // one grid: this kernel folds the CFL partials and ends the step
  const double t = tl.scal[0], dt_given = tl.scal[1];
  if (one && (tl.mctl[1] != 0 || !(t < t_end))) {  // uniform across the grid: nothing to do
    if (blockIdx.x == 0 && tid == 0) { tl.ctl[6] = 0; tl.ctl[7] = 0; tl.ctl[9] = 0; tl.ctl[10] = 0; tl.ctl[11] = 0; tl.ctl[15] = 0; tl.ctl[17] = 0; tl.ctl[20] = 0; }  // (a no-op step's counters)
    // peer mode: a stopped rank still publishes a neutral pair while the others step (t is
    // global, so at t_end every rank stops together and nobody waits)
    if (blockIdx.x == 0 && tl.xbuf && tl.xpeers && t < t_end) xpublish(tl, 0.0, INFINITY, tl.mctl[1]);
    return;
  }
  double dt = dt_given;
  if (t + dt > t_end) dt = t_end - t;
  // fast tiles' partials (slow tiles hold neutral values here)
  double s = 0.0, hm = INFINITY;
  for (int q = blockIdx.x * T + tid; one && q < tl.ntiles; q += gridDim.x * T) {
    s = fmax(s, tl.part[2 * q]);
    hm = fmin(hm, tl.part[2 * q + 1]);
  }
  s = warp_max(s);
  hm = warp_min(hm);
  if (lane == 0) { sh.part_s[warp] = s; sh.part_h[warp] = hm; }
  __syncthreads();
  double cta_s = 0.0, cta_h = INFINITY;  // thread 0
  if (tid == 0)
    for (int w = 0; w < nw; ++w) { cta_s = fmax(cta_s, sh.part_s[w]); cta_h = fmin(cta_h, sh.part_h[w]); }
  const int njobs = tl.ctl[4];
  for (;;) {
    __syncthreads();
    if (tid == 0) sh.n_new = atomicAdd(&tl.ctl[5], 1);
    __syncthreads();
    const int j = sh.n_new;
    if (j >= njobs) break;
    double sk = 0.0, hk = INFINITY;
    tile_full(e, p, tl, sh, A, capg, tl.slow[j], t_end, sk, hk);
    if (tid == 0) { cta_s = fmax(cta_s, sk); cta_h = fmin(cta_h, hk); }
  }
  if (!one) return;  // members: tiled_members_finish folds and ends the step
  __shared__ int last;
  if (tid == 0) {
    tl.part2[2 * blockIdx.x] = cta_s;
    tl.part2[2 * blockIdx.x + 1] = cta_h;
    __threadfence();
    last = atomicAdd(&tl.ctl[2], 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    if (tl.mctl[1] == 0) tiles_finish_step(p, tl, (int)gridDim.x, dt, t_end);
    else {
      if (tid == 0) { ctl_step_reset(tl); }
      if (tl.xbuf && tl.xpeers) xpublish(tl, 0.0, INFINITY, tl.mctl[1]);  // (neutral pair, status)
    }
  }
}

// initial partials of every tile (one CTA per tile) and, by the last CTA, dt_0
template <int MAXT>
__global__ void __launch_bounds__(MAXT)
tiled_init_dt(const __grid_constant__ Eos e, const __grid_constant__ Prm p, const __grid_constant__ Tiles tl,
              double t_end) {
  const int k = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int m = k / tl.tpm;
  const bool first = k % tl.tpm == 0, lastt = (k + 1) % tl.tpm == 0;
  const int cur = tl.mctl[MCS * m];
  const long long base = (long long)k * tl.capt;
  const int cnt = tl.cnt[cur][k];
  __shared__ double rs[32], rh[32];
  __shared__ int last;
  double s = 0.0, hm = INFINITY;
  for (int i = tid; i < cnt; i += blockDim.x) {
    const long long g = base + i;
    const double r = tl.rho[cur][g];
    const int ph = phase_of(e, r);
    s = fmax(s, fabs(tl.mom[cur][g] * rcp_fast(r)) + sound(e, ph));
    bool tiny = false;
    const double hg = tl.hu[cur][k] ? p.h_av : tl.h[cur][g];
    if (p.mode != 1 && hg < p.eps_tiny * p.h_av) {  // neighbours may live in the next tiles
      const double rl = i > 0 ? tl.rho[cur][g - 1] : (!first ? tl.rho[cur][base - tl.capt + tl.cnt[cur][k - 1] - 1] : -1.0);
      const double rr = i < cnt - 1 ? tl.rho[cur][g + 1] : (!lastt ? tl.rho[cur][base + tl.capt] : -1.0);
      const bool same_l = rl > 0.0 && phase_of(e, rl) == ph, same_r = rr > 0.0 && phase_of(e, rr) == ph;
      tiny = !same_l && !same_r;
    }
    if (!tiny) hm = fmin(hm, hg);
  }
  s = warp_max(s);
  hm = warp_min(hm);
  if (lane == 0) { rs[warp] = s; rh[warp] = hm; }
  __syncthreads();
  // initial halos for the first exchange (before the last-CTA election: peer mode publishes
  // them with the initial CFL pair)
  if (tl.xbuf && (k == 0 || k == tl.ntiles - 1)) {  // initial halos for the first exchange
    const int cur2 = tl.mctl[0];
    if (k == 0 && tl.nbr_left) {
      double* sb = tl.xbuf + XB_SEND_LEFT;
      for (int i = tid; i < HALO; i += blockDim.x) {
        sb[i] = tl.rho[cur2][base + i]; sb[HALO + i] = tl.mom[cur2][base + i];
        sb[2 * HALO + i] = tl.hu[cur2][k] ? p.h_av : tl.h[cur2][base + i];
      }
      if (tid == 0) sb[3 * HALO] = HALO;
    }
    if (k == tl.ntiles - 1 && tl.nbr_right) {
      double* sb = tl.xbuf + XB_SEND_RIGHT;
      for (int i = tid; i < HALO; i += blockDim.x) {
        const long long j = base + cnt - HALO + i;
        sb[i] = tl.rho[cur2][j]; sb[HALO + i] = tl.mom[cur2][j]; sb[2 * HALO + i] = tl.hu[cur2][k] ? p.h_av : tl.h[cur2][j];
      }
      if (tid == 0) sb[3 * HALO] = HALO;
    }
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 0; w < nw; ++w) { s = fmax(s, rs[w]); hm = fmin(hm, rh[w]); }
    tl.part[2 * k] = s;
    tl.part[2 * k + 1] = hm;
    __threadfence();
    last = tl.M == 1 && atomicAdd(&tl.ctl[2], 1) == tl.ntiles - 1;  // members: tiled_members_finish
  }
  __syncthreads();
  if (last) {
    __threadfence();
    s = 0.0; hm = INFINITY;
    for (int q = tid; q < tl.ntiles; q += blockDim.x) { s = fmax(s, tl.part[2 * q]); hm = fmin(hm, tl.part[2 * q + 1]); }
    s = warp_max(s);
    hm = warp_min(hm);
    __syncthreads();
    if (lane == 0) { rs[warp] = s; rh[warp] = hm; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 0; w < nw; ++w) { s = fmax(s, rs[w]); hm = fmin(hm, rh[w]); }
      if (tl.xbuf) {
        tl.xbuf[XB_DT] = -s;
        tl.xbuf[XB_DT + 1] = hm;
      } else {
        double dt = p.cfl * hm / s;
        if (tl.scal[0] + dt > t_end) dt = t_end - tl.scal[0];
        tl.scal[1] = dt;
        tl.scal[5] = s;
      }
      tl.ctl[2] = 0;
    }
    __syncthreads();
    if (tl.xbuf && tl.xpeers) xpublish(tl, tl.xbuf[XB_DT], tl.xbuf[XB_DT + 1], tl.mctl[1]);
  }
}

// Members (independent grids, tl.M > 1), after tiled_slow: one warp per member folds its tiles'
// partials into its next dt (R5/R6) and, if it stepped (after_step, status 0,
// t < t_end), advances t, flips its buffers and counts the step.  Block 0 resets the step's
// work-list counters.  Each member keeps its own dt and t (R25).
__global__ void tiled_members_finish(const __grid_constant__ Prm p, const __grid_constant__ Tiles tl, double t_end,
                                     int after_step) {
  const int lane = threadIdx.x & 31;
  const int m = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    tl.ctl[8] = tl.ctl[6];
    ctl_step_reset(tl);
    if (after_step) { tl.ctl[3] += 1; ctl_step_roll(tl); }
  }
  if (m >= tl.M) return;
  double s = 0.0, hm = INFINITY;
  for (int j = lane; j < tl.tpm; j += 32) {
    const int k = m * tl.tpm + j;
    s = fmax(s, tl.part[2 * k]);
    hm = fmin(hm, tl.part[2 * k + 1]);
  }
  s = warp_max(s);
  hm = warp_min(hm);
  if (lane != 0) return;
  double* sc = tl.scal + SCS * m;
  int* mc = tl.mctl + MCS * m;
  if (mc[1] != 0) return;
  double t_new = sc[0];
  if (after_step) {
    if (!(t_new < t_end)) return;  // the member did not step
    double dt_used = sc[1];
    if (t_new + dt_used > t_end) dt_used = t_end - t_new;  // as the tile kernels
    t_new += dt_used;
    if (mc[2] == 0 || dt_used < sc[2]) sc[2] = dt_used;
    if (dt_used > sc[3]) sc[3] = dt_used;
    mc[0] = 1 - mc[0];
    mc[2] += 1;
  }
  double dt = p.cfl * hm / s;
  if (t_new + dt > t_end) dt = t_end - t_new;
  sc[0] = t_new;
  sc[1] = dt;
  sc[5] = s;
}

// members still stepping (status 0, t < t_end) -> ctl[10] (run_to polling)
__global__ void tiled_members_active(const __grid_constant__ Tiles tl, double t_end) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = m < tl.M && tl.mctl[MCS * m + 1] == 0 && tl.scal[SCS * m] < t_end;
  const unsigned b = __ballot_sync(0xffffffffu, act);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(&tl.ctl[10], __popc(b));
}

// rank mode, after the exchange: dt from the min-reduced pair; after a step also advance t and
// flip the buffers (what the last CTA does in single-rank mode)
// (one warp)  Peer mode: wait until every rank's publication of this step has arrived (its tag in
// this rank's pair table; a system-scope acquire), fold the ranks' pairs into XB_DT and copy the
// neighbours' records into the receive slots the next step's kernels read.  A rank that never
// publishes (a dead peer) ends the wait after ~2 s with status ST_INTERNAL instead of a hang.
__device__ bool xconsume(const Tiles& tl) {
  const int lane = threadIdx.x & 31;
  const long long tag = (long long)tl.ctl[12];  // publications so far: the same on every rank
  const int par = (int)(tag & 1);
  bool ok = true;
  if (lane < tl.xworld) {
    volatile const double* pt = tl.xbuf + XB_PPAIR + (par * XB_MAXRANKS + lane) * 4 + 2;
    const long long c0 = clock64();
    while (*pt != (double)tag)
      if (clock64() - c0 > 4000000000ll) { ok = false; break; }
  }
  ok = __all_sync(0xffffffffu, ok);
  if (!ok) {
    if (lane == 0) { atomicCAS(&tl.mctl[1], 0, (int)ST_INTERNAL); atomicCAS(&tl.ctl[1], 0, (int)ST_INTERNAL); }
    return false;
  }
  __threadfence_system();
  double ns = INFINITY, hm = INFINITY;  // the min over ranks of (-S_max_r, h_min_r), as the all-reduce
  if (lane < tl.xworld) {
    volatile const double* pr = tl.xbuf + XB_PPAIR + (par * XB_MAXRANKS + lane) * 4;
    ns = pr[0]; hm = pr[1];
  }
  ns = warp_min(ns);  // (compare-select: exact, order-free)
  hm = warp_min(hm);
  if (lane == 0) { tl.xbuf[XB_DT] = ns; tl.xbuf[XB_DT + 1] = hm; }
  for (int q = lane; q < XB_REC; q += 32) {
    volatile const double* rl = tl.xbuf + XB_PREC + (2 * par + 0) * XB_REC;
    volatile const double* rr = tl.xbuf + XB_PREC + (2 * par + 1) * XB_REC;
    if (tl.nbr_left) tl.xbuf[XB_RECV_LEFT + q] = rl[q];
    if (tl.nbr_right) tl.xbuf[XB_RECV_RIGHT + q] = rr[q];
  }
  __syncwarp();
  return true;
}

__global__ void tiled_finish(const __grid_constant__ Prm p, const __grid_constant__ Tiles tl, double t_end, int after_step) {
  if (tl.mctl[1] != 0) return;
  if (after_step && !(tl.scal[0] < t_end)) return;  // the step was a no-op (on every rank: t is global)
  if (tl.xpeers && !xconsume(tl)) return;
  if (threadIdx.x != 0) return;
  const double S = -tl.xbuf[XB_DT], hm = tl.xbuf[XB_DT + 1];
  double t_new = tl.scal[0];
  if (after_step) {
    const double dt_used = tl.scal[4];
    t_new += dt_used;
    if (tl.mctl[2] == 0 || dt_used < tl.scal[2]) tl.scal[2] = dt_used;
    if (dt_used > tl.scal[3]) tl.scal[3] = dt_used;
    tl.mctl[0] = 1 - tl.mctl[0];
    tl.mctl[2] += 1;
    tl.ctl[3] += 1;
    ctl_step_roll(tl);
  }
  ctl_step_reset(tl);
  double dt = p.cfl * hm / S;
  if (t_new + dt > t_end) dt = t_end - t_new;
  tl.scal[0] = t_new;
  tl.scal[1] = dt;
  tl.scal[5] = S;
}

}  // namespace eis
