// eis_tiled.cuh — the tiled streaming kernel for one huge grid (BASELINE configs[4], C5).
//
// The grid is cut into tiles of about TILE cells, each stored with slack (capt cells) so that
// creations and splits insert locally.  One launch = one large step of the whole grid: every
// CTA loads its tile plus H halo cells from each neighbour tile (ping-pong buffers: step n
// reads buffer cur, writes 1-cur), runs the same step body as the member-resident kernel with
// the global dt, and writes back the cells it owns after the remesh.  The halo is computed
// redundantly by both neighbours with identical inputs and code, so every decision at a tile
// boundary (boundary solves, creations, DTS blocks, merges) is taken identically on both sides;
// ownership rules: a created cell at a tile boundary and a merge group headed left of it belong
// to the left tile.  The CTA also reduces S_max / h_min of its new cells; the last CTA to finish
// folds all tiles into the next step's dt (CFL, R5/R6), so a step costs one launch and one
// read + one write of the state (24 B + 24 B per cell).
#pragma once
#include "eis_resident.cuh"

namespace eis {

constexpr int HALO = 10;  // halo cells per side: >= MAXB + 2 keeps every needed block exact

struct TileStats {
  long long cell_updates, dts_iters, iface_solves, creations, splits, merges, regions;
};

struct Tiles {
  double *rho[2], *mom[2], *h[2];  // ntiles x capt, ping-pong
  int* cnt[2];                     // live cells per tile
  double* ws;                      // per tile: ws0[MAXIF], ws1[MAXIF], wsn  (2*MAXIF + 1 doubles)
  double* part;                    // per tile: S_max, h_min of the tile's new cells
  TileStats* tstats;
  double* scal;                    // [0] t  [1] dt of the next step  [2] dt_min  [3] dt_max
  int* ctl;                        // [0] cur  [1] status  [2] done-counter  [3] steps
  double* xbuf;                    // rank mode: exchange buffer (layout XB_* below), else null
  int ntiles, capt, nbr_left, nbr_right;
};

// Exchange buffer (rank mode, one grid decomposed over ranks): four halo records of
// HALO cells (rho, mom, h) + a count, then the CFL pair (-S_max, h_min) to be min-reduced.
constexpr int XB_REC = 3 * HALO + 1;
constexpr int XB_SEND_LEFT = 0, XB_SEND_RIGHT = XB_REC, XB_RECV_LEFT = 2 * XB_REC, XB_RECV_RIGHT = 3 * XB_REC;
constexpr int XB_DT = 4 * XB_REC;
constexpr int XB_DOUBLES = 4 * XB_REC + 2;

constexpr int WS_STRIDE = 2 * MAXIF + 1;

// S_max and h_min (over non-tiny cells, R5/R6) of cells [lo, hi) of a smem grid of n cells
__device__ __forceinline__ void cfl_partials(const Eos& e, const Prm& p, const double* rho, const double* mom,
                                             const double* h, int n, int lo, int hi, bool left_real,
                                             bool right_real, double& s_out, double& h_out) {
  double s = 0.0, hm = INFINITY;
  for (int i = lo + (int)threadIdx.x; i < hi; i += blockDim.x) {
    const double r = rho[i];
    const int ph = phase_of(e, r);
    s = fmax(s, fabs(mom[i] / r) + sound(e, ph));
    bool tiny = false;
    if (p.mode == 0 && h[i] < p.eps_tiny * p.h_av) {
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

// Last CTA of a step: fold the per-tile partials into the next dt, advance t.
__device__ void tiles_finish_step(const Prm& p, const Tiles& tl, double dt_used, double t_end) {
  __shared__ double rs[32], rh[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double s = 0.0, hm = INFINITY;
  for (int k = tid; k < tl.ntiles; k += blockDim.x) {
    s = fmax(s, tl.part[2 * k]);
    hm = fmin(hm, tl.part[2 * k + 1]);
  }
  s = warp_max(s);
  hm = warp_min(hm);
  if (lane == 0) { rs[warp] = s; rh[warp] = hm; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 0; w < nw; ++w) { s = fmax(s, rs[w]); hm = fmin(hm, rh[w]); }
    if (tl.xbuf) {  // rank mode: the global dt needs the other ranks (eis_step_finish)
      tl.xbuf[XB_DT] = -s;
      tl.xbuf[XB_DT + 1] = hm;
      tl.scal[4] = dt_used;
      __threadfence();
      return;
    }
    const double t_new = tl.scal[0] + dt_used;
    double dt = p.cfl * hm / s;
    if (t_new + dt > t_end) dt = t_end - t_new;
    tl.scal[0] = t_new;
    tl.scal[1] = dt;
    if (tl.ctl[3] == 0 || dt_used < tl.scal[2]) tl.scal[2] = dt_used;
    if (dt_used > tl.scal[3]) tl.scal[3] = dt_used;
    tl.ctl[0] = 1 - tl.ctl[0];
    tl.ctl[3] += 1;
    tl.ctl[2] = 0;
    __threadfence();
  }
}

template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
tiled_step(const __grid_constant__ Eos e, const __grid_constant__ Prm p, const __grid_constant__ Tiles tl,
           double t_end) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CtaShared& sh = *reinterpret_cast<CtaShared*>(smem_raw);
  const int capg = tl.capt + 2 * HALO + MAXEV;
  Arr A = carve(smem_raw, capg);
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  const int k = blockIdx.x;
  const int cur = tl.ctl[0];
  const double t = tl.scal[0], dt_given = tl.scal[1];
  if (tl.ctl[1] != 0 || !(t < t_end)) return;  // uniform across the grid: nothing to do
  const int in = cur, out = 1 - cur;
  const long long base = (long long)k * tl.capt;
  const int cnt = tl.cnt[in][k];
  const bool xl = (k == 0 && tl.nbr_left), xr = (k == tl.ntiles - 1 && tl.nbr_right);  // halo from a rank
  const int nL = k > 0 ? min(HALO, tl.cnt[in][k - 1]) : (xl ? (int)tl.xbuf[XB_RECV_LEFT + 3 * HALO] : 0);
  const int nR = k < tl.ntiles - 1 ? min(HALO, tl.cnt[in][k + 1]) : (xr ? (int)tl.xbuf[XB_RECV_RIGHT + 3 * HALO] : 0);
  if (tid == 0) {
    sh.status = 0;
    reset_counters(sh);
    memset(&sh.st, 0, sizeof(sh.st));
    const double* ws = tl.ws + (size_t)k * WS_STRIDE;
    sh.wsn = (int)ws[2 * MAXIF];
    for (int q = 0; q < MAXIF; ++q) { sh.ws0[q] = ws[q]; sh.ws1[q] = ws[MAXIF + q]; }
  }
  const int n = nL + cnt + nR;
  {  // load: left halo | own | right halo (coalesced)
    const long long bl = base - tl.capt, br = base + tl.capt;
    const int cl = k > 0 ? tl.cnt[in][k - 1] : 0;
    for (int i = tid; i < n; i += T) {
      if (xl && i < nL) {  // left halo received from the left rank (its last cells)
        const double* rb = tl.xbuf + XB_RECV_LEFT;
        const int j = HALO - nL + i;
        A.rho[i] = rb[j]; A.mom[i] = rb[HALO + j]; A.h[i] = rb[2 * HALO + j];
        continue;
      }
      if (xr && i >= nL + cnt) {  // right halo received from the right rank (its first cells)
        const double* rb = tl.xbuf + XB_RECV_RIGHT;
        const int j = i - nL - cnt;
        A.rho[i] = rb[j]; A.mom[i] = rb[HALO + j]; A.h[i] = rb[2 * HALO + j];
        continue;
      }
      long long g;
      if (i < nL) g = bl + (cl - nL + i);
      else if (i < nL + cnt) g = base + (i - nL);
      else g = br + (i - nL - cnt);
      A.rho[i] = tl.rho[in][g];
      A.mom[i] = tl.mom[in][g];
      A.h[i] = tl.h[in][g];
    }
    for (int i = tid; i <= capg; i += T) A.fl[i] = 0;
  }
  A.n = n;
  __syncthreads();
  if (warp == nw - 1) build_boundary_list(e, sh, A.rho, A.fl, n);
  __syncthreads();
  Zone Z;
  Z.own_lo = nL; Z.own_hi = nL + cnt;
  Z.zlo = max(nL - 2, 0); Z.zhi = min(nL + cnt + 2, n);
  Z.dt_given = dt_given;
  Z.left_real = (k == 0 && !tl.nbr_left); Z.right_real = (k == tl.ntiles - 1 && !tl.nbr_right);
  const double dt = step_body(e, p, sh, A, t, t_end, Z);
  // ---------------- owned output, partials of the next dt, side tables ----------------
  __syncthreads();
  const int olo = sh.olo, ohi = sh.ohi;
  const int nout = ohi - olo;
  int st = sh.status;
  if (dt >= 0.0 && st == 0 && (nout > tl.capt || nout < (tl.ntiles > 1 ? HALO : 3))) st = ST_CAPACITY;
  if (dt >= 0.0 && st == 0) {
    const long long ob = base;
    for (int i = tid; i < nout; i += T) {
      tl.rho[out][ob + i] = A.rho[olo + i];
      tl.mom[out][ob + i] = A.mom[olo + i];
      tl.h[out][ob + i] = A.h[olo + i];
    }
    if (xl) {  // my first HALO owned cells go to the left rank (its right halo)
      double* sb = tl.xbuf + XB_SEND_LEFT;
      for (int i = tid; i < HALO; i += T) { sb[i] = A.rho[olo + i]; sb[HALO + i] = A.mom[olo + i]; sb[2 * HALO + i] = A.h[olo + i]; }
      if (tid == 0) sb[3 * HALO] = HALO;
    }
    if (xr) {  // my last HALO owned cells go to the right rank (its left halo)
      double* sb = tl.xbuf + XB_SEND_RIGHT;
      for (int i = tid; i < HALO; i += T) {
        const int j = ohi - HALO + i;
        sb[i] = A.rho[j]; sb[HALO + i] = A.mom[j]; sb[2 * HALO + i] = A.h[j];
      }
      if (tid == 0) sb[3 * HALO] = HALO;
    }
    double s, hm;
    cfl_partials(e, p, A.rho, A.mom, A.h, A.n, olo, ohi, Z.left_real, Z.right_real, s, hm);
    if (lane == 0) { sh.part_s[warp] = s; sh.part_h[warp] = hm; }
  }
  __syncthreads();
  if (tid == 0) {
    if (st != 0) atomicCAS(&tl.ctl[1], 0, st);
    if (dt >= 0.0 && st == 0) {
      double s = 0.0, hm = INFINITY;
      for (int w = 0; w < nw; ++w) { s = fmax(s, sh.part_s[w]); hm = fmin(hm, sh.part_h[w]); }
      tl.part[2 * k] = s;
      tl.part[2 * k + 1] = hm;
      tl.cnt[out][k] = nout;
      double* ws = tl.ws + (size_t)k * WS_STRIDE;
      for (int q = 0; q < MAXIF; ++q) { ws[q] = sh.ws0[q]; ws[MAXIF + q] = sh.ws1[q]; }
      ws[2 * MAXIF] = (double)sh.wsn;
      TileStats& ts = tl.tstats[k];
      ts.cell_updates += cnt;
      ts.dts_iters += (long long)sh.c_dts;
      ts.iface_solves += (long long)sh.c_solves;
      ts.regions += (long long)sh.c_regions;
      ts.creations += sh.st.creations;  // owned events only (step_body)
      ts.splits += sh.st.splits;
      ts.merges += sh.st.merges;
    }
    __threadfence();
    sh.remesh = atomicAdd(&tl.ctl[2], 1) == tl.ntiles - 1;  // reuse as "I am the last CTA"
  }
  __syncthreads();
  if (sh.remesh) {
    __threadfence();
    if (tl.ctl[1] == 0) tiles_finish_step(p, tl, dt, t_end);
    else if (tid == 0) tl.ctl[2] = 0;
  }
}

// initial partials of every tile (one CTA per tile) and, by the last CTA, dt_0
template <int MAXT>
__global__ void __launch_bounds__(MAXT)
tiled_init_dt(const __grid_constant__ Eos e, const __grid_constant__ Prm p, const __grid_constant__ Tiles tl,
              double t_end) {
  const int k = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int cur = tl.ctl[0];
  const long long base = (long long)k * tl.capt;
  const int cnt = tl.cnt[cur][k];
  __shared__ double rs[32], rh[32];
  __shared__ int last;
  double s = 0.0, hm = INFINITY;
  for (int i = tid; i < cnt; i += blockDim.x) {
    const long long g = base + i;
    const double r = tl.rho[cur][g];
    const int ph = phase_of(e, r);
    s = fmax(s, fabs(tl.mom[cur][g] / r) + sound(e, ph));
    bool tiny = false;
    if (p.mode == 0 && tl.h[cur][g] < p.eps_tiny * p.h_av) {  // neighbours may live in the next tiles
      const double rl = i > 0 ? tl.rho[cur][g - 1] : (k > 0 ? tl.rho[cur][base - tl.capt + tl.cnt[cur][k - 1] - 1] : -1.0);
      const double rr = i < cnt - 1 ? tl.rho[cur][g + 1] : (k < tl.ntiles - 1 ? tl.rho[cur][base + tl.capt] : -1.0);
      const bool same_l = rl > 0.0 && phase_of(e, rl) == ph, same_r = rr > 0.0 && phase_of(e, rr) == ph;
      tiny = !same_l && !same_r;
    }
    if (!tiny) hm = fmin(hm, tl.h[cur][g]);
  }
  s = warp_max(s);
  hm = warp_min(hm);
  if (lane == 0) { rs[warp] = s; rh[warp] = hm; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 0; w < nw; ++w) { s = fmax(s, rs[w]); hm = fmin(hm, rh[w]); }
    tl.part[2 * k] = s;
    tl.part[2 * k + 1] = hm;
    __threadfence();
    last = atomicAdd(&tl.ctl[2], 1) == tl.ntiles - 1;
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
      }
      tl.ctl[2] = 0;
    }
  }
  if (tl.xbuf && (k == 0 || k == tl.ntiles - 1)) {  // initial halos for the first exchange
    const int cur2 = tl.ctl[0];
    if (k == 0 && tl.nbr_left) {
      double* sb = tl.xbuf + XB_SEND_LEFT;
      for (int i = tid; i < HALO; i += blockDim.x) {
        sb[i] = tl.rho[cur2][base + i]; sb[HALO + i] = tl.mom[cur2][base + i]; sb[2 * HALO + i] = tl.h[cur2][base + i];
      }
      if (tid == 0) sb[3 * HALO] = HALO;
    }
    if (k == tl.ntiles - 1 && tl.nbr_right) {
      double* sb = tl.xbuf + XB_SEND_RIGHT;
      for (int i = tid; i < HALO; i += blockDim.x) {
        const long long j = base + cnt - HALO + i;
        sb[i] = tl.rho[cur2][j]; sb[HALO + i] = tl.mom[cur2][j]; sb[2 * HALO + i] = tl.h[cur2][j];
      }
      if (tid == 0) sb[3 * HALO] = HALO;
    }
  }
}

// rank mode, after the exchange: dt from the min-reduced pair; after a step also advance t and
// flip the buffers (what the last CTA does in single-rank mode)
__global__ void tiled_finish(const __grid_constant__ Prm p, const __grid_constant__ Tiles tl, double t_end, int after_step) {
  if (tl.ctl[1] != 0) return;
  const double S = -tl.xbuf[XB_DT], hm = tl.xbuf[XB_DT + 1];
  double t_new = tl.scal[0];
  if (after_step) {
    if (!(t_new < t_end)) return;  // the step was a no-op
    const double dt_used = tl.scal[4];
    t_new += dt_used;
    if (tl.ctl[3] == 0 || dt_used < tl.scal[2]) tl.scal[2] = dt_used;
    if (dt_used > tl.scal[3]) tl.scal[3] = dt_used;
    tl.ctl[0] = 1 - tl.ctl[0];
    tl.ctl[3] += 1;
    tl.ctl[2] = 0;
  }
  double dt = p.cfl * hm / S;
  if (t_new + dt > t_end) dt = t_end - t_new;
  tl.scal[0] = t_new;
  tl.scal[1] = dt;
}

}  // namespace eis
