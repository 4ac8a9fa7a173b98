// eis_dts.cuh — Algorithm 2 (dual time stepping; moving widths §3.4, P:744-766;
// residual and stop rule P:1128-1132, readings R8, R11-R13) on one implicit block of K <= MAXB
// cells by one warp, generic over the conservation law.
//
// One loop serves both systems the library runs: the isothermal two-phase model (NV = 2, the
// hot path of every layout: eis_resident.cuh dts_block) and the 3-equation Euler system of the
// paper's Lax shock-tube test (NV = 3, eis_lax.cuh).  A system `Sys` supplies
//   static constexpr int NV;                      conserved variables per cell
//   int  edge(j, W, Fe, we, half, hl, hmask)      interior edge j (between block cells j-1 and
//        j) at the iterate W[q*MAXB + i]: called by all 16 lanes of a half warp (the two-phase
//        boundary solver is half-warp cooperative); lane hl == 0 writes Fe[q*(MAXB+1) + j] and
//        the edge speed we[j] and returns a status (0: ok)
//   int  check(lane, w)                           admissibility of the new iterate of this
//        lane's cell (0 or a status)
//   void store(W, lane, w)                        caches derived values of the iterate (in the
//        scratch past the loop's arrays)
// The caller sets the outer edges (Fe[.][0], Fe[.][K], we[0], we[K]: the explicit step's, flux
// bounding P:601) and each lane's DtsCell; the loop returns U^{n+1}, h^{n+1}.
#pragma once
#include "eis_device.cuh"

namespace eis {

constexpr int MAXB = 8;  // cells per implicit block

template <int NV>
struct DtsCell {         // lane i < K: block cell i
  double un[NV];         // U^n
  double hn;             // h^n
  double theta;          // dtau / dt of this cell (theta_nb, or alpha for a tiny cell: P:1127, R12)
  double tol;            // its stop tolerance: tol_tiny for a tiny cell, tol_nb otherwise
};

// The relaxed update of P:763 (R13) and Part 2's conservative update with explicit roundings
// (no contraction left to the compiler): dts_warp and dts_thread evaluate these same functions,
// so the two loops give the same bits.
__device__ __forceinline__ double dts_relax(double w, double i1r, double qr, double a0, double un, double a1, double fL,
                                            double fR) {
  const double target = __fma_rn(a0, un, -__dmul_rn(a1, __dsub_rn(fR, fL)));  // (h^n/h) U^n - (dt/h) dF
  return __fma_rn(w, i1r, __dmul_rn(qr, target));                              // W/(1+r) + r/(1+r) target
}
__device__ __forceinline__ double dts_resid(double rsc, double nq, double w) { return fabs(__dmul_rn(rsc, __dsub_rn(nq, w))); }
__device__ __forceinline__ double dts_tol(double tol, double w) { return __dmul_rn(tol, fmax(fabs(w), 1.0)); }
// the rounding-error bound of W^{l+1} - W^l on the residual's scale (decision margins)
__device__ __forceinline__ double dts_margin(double rsc, double w, double qr, double a0, double un, double a1, double fL,
                                             double fR) {
  const double m = __fma_rn(a1, __dadd_rn(fabs(fL), fabs(fR)), fabs(__dmul_rn(a0, un)));
  return __dmul_rn(__dmul_rn(MARGIN_EPS, rsc), __fma_rn(qr, m, fabs(w)));
}
__device__ __forceinline__ double dts_final(double hn, double hn1, double un, double dt, double fL, double fR) {
  return __fma_rn(__ddiv_rn(hn, hn1), un, -__dmul_rn(__ddiv_rn(dt, hn1), __dsub_rn(fR, fL)));
}

// One implicit block of a window of the tiled layout, exported by the window kernel's part A,
// solved by dts_jobs (one lane), read back by part B (eis_tiled.cuh).
struct DtsJob {
  double un[MAXB][2];      // in: U^n (rho, rho u); out: U^{n+1}
  double hn[MAXB];         // in: h^n; out: h^{n+1}
  double Fo[2][2], wo[2];  // outer edges (left = edge a, right = edge b + 1): flux and speed
  double xs[MAXB + 1][2];  // interior boundaries' star pressures: in warm starts (-1: none), out converged
  double dt;
  long long it;            // out: Part-1 iterations
  int K, tiny;             // cells; bit i: cell i tiny
  int solves, status, marg, pad;  // out: boundary solves, status, stop decisions within their margin
};

// shared scratch of the loop (doubles): the iterate W[NV][MAXB], edge fluxes Fe[NV][MAXB + 1],
// edge speeds we[MAXB + 1]
template <int NV>
__host__ __device__ constexpr int dts_scratch() { return NV * MAXB + NV * (MAXB + 1) + (MAXB + 1); }

// Part 1 (iterate to the stop rule) and Part 2 (fluxes at U*, conservative update).  Returns
// the warp-uniform status; l_out = Part-1 iterations; marg += stop decisions taken within their
// rounding-error bound.  On lane < K with status 0, u1/h1 hold the cell's
// U^{n+1} and h^{n+1}.
template <class Sys>
__device__ __forceinline__ int dts_warp(Sys& S, double* sc, const int K, const double dt, const long long max_iter,
                                        const DtsCell<Sys::NV>& c, double (&u1)[Sys::NV], double& h1,
                                        long long& l_out, int& marg) {
  constexpr int NV = Sys::NV;
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  double* const W = sc;
  double* const Fe = sc + NV * MAXB;
  double* const we = Fe + NV * (MAXB + 1);
  const bool own = lane < K;
  double w[NV];
  double r = 0.0, dtau = 1.0;
#pragma unroll
  for (int q = 0; q < NV; ++q) w[q] = own ? c.un[q] : 0.0;
  if (own) {
    dtau = c.theta * dt;
    r = dtau / dt;
#pragma unroll
    for (int q = 0; q < NV; ++q) W[q * MAXB + lane] = w[q];
    S.store(W, lane, w);
  }
  // loop invariants of the relaxed update and of the residual (one reciprocal each)
  const double i1r = 1.0 / (1.0 + r), qr = r * i1r, rsc = (1.0 + r) / dtau;
  __syncwarp();
  long long l = 0;
  int err = 0;
  bool prev_cont_robust = true;  // decision margin of the last "continue"
  for (int part = 0; part < 2 && !err; ++part) {  // part 0: Part-1 iterations; part 1: fluxes at U*
    for (;;) {
      for (int j0 = 1; j0 < K; j0 += 2) {  // (a) interior edges at W^l, two per round (half warps)
        const int j = j0 + half;
        if (j < K) {
          const int s = S.edge(j, W, Fe, we, half, hl, hmask);
          if (s) err = s;
        }
      }
      err = __reduce_max_sync(0xffffffffu, err);
      __syncwarp();
      if (err || part == 1) break;
      // (b) relaxed moving-cell update (P:683-688 with the widths of P:763, R13) and this lane's
      // residual, res = |(1 + r)(W^{l+1} - W^l)| / (dtau max(|W^l|, 1)) < tol multiplied out
      bool conv = true, rstop = true, rcont = false;
      int bad = 0;
      if (own) {
        const double hl_ = __dadd_rn(c.hn, __dmul_rn(we[lane + 1] - we[lane], dt));
        if (!(hl_ > 0.0)) bad = ST_WIDTH;
        const double ih = 1.0 / hl_, a0 = c.hn * ih, a1 = dt * ih;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const double fL = Fe[q * (MAXB + 1) + lane], fR = Fe[q * (MAXB + 1) + lane + 1];
          const double nq = dts_relax(w[q], i1r, qr, a0, c.un[q], a1, fL, fR);
          const double d = dts_resid(rsc, nq, w[q]), t = dts_tol(c.tol, w[q]);
          conv = conv && d < t;
          // decision margin: the rounding-error bound of W^{l+1} - W^l on the residual's scale
          const double eb = dts_margin(rsc, w[q], qr, a0, c.un[q], a1, fL, fR);
          rstop = rstop && d < t - eb;
          rcont = rcont || d >= t + eb;
          w[q] = nq;
        }
        const int s = S.check(lane, w);
        if (s && !bad) bad = s;
      }
      // max over tiny cells < tol_tiny and over the others < tol_nb  <=>  every lane below its own
      conv = __all_sync(0xffffffffu, conv);
      rstop = __all_sync(0xffffffffu, rstop);
      rcont = __any_sync(0xffffffffu, rcont);
      if (conv && (!rstop || !prev_cont_robust)) marg += 1;
      prev_cont_robust = rcont;
      bad = __reduce_max_sync(0xffffffffu, bad);
      if (own) {
#pragma unroll
        for (int q = 0; q < NV; ++q) W[q * MAXB + lane] = w[q];
        S.store(W, lane, w);
      }
      __syncwarp();
      ++l;
      if (bad) { err = bad; break; }
      if (conv) break;
      if (l >= max_iter) { err = ST_DTS_CAP; break; }
    }
  }
  if (!err && own) {  // Part 2 (b): conservative update with F_left, F*, F_right
    const double hn1 = __dadd_rn(c.hn, __dmul_rn(we[lane + 1] - we[lane], dt));
    if (!(hn1 > 0.0)) err = ST_WIDTH;
    else {
#pragma unroll
      for (int q = 0; q < NV; ++q)
        u1[q] = dts_final(c.hn, hn1, c.un[q], dt, Fe[q * (MAXB + 1) + lane], Fe[q * (MAXB + 1) + lane + 1]);
      h1 = hn1;
    }
  }
  err = __reduce_max_sync(0xffffffffu, err);
  __syncwarp();
  l_out = l;
  return err;
}

// ------------------------------------------------------------------------------------------
// The same Algorithm 2 by ONE thread per block (lane-parallel over blocks: the window path of
// the tiled layout gathers the blocks of every window of a step into one launch, dts_jobs,
// one lane per block).  Identical expressions in the identical order as dts_warp, so the two
// give the same bits.  KMAX: compile-time bound of K (arrays stay in registers for KMAX = 3).
// A per-thread system `Sys` supplies
//   int  edges(K, W, Fe, we)     every interior edge j = 1 .. K-1 between cells j-1 and j at the
//        iterate W: fluxes Fe[j][NV] and edge speeds we[j]; returns the largest status (0: ok)
//   int  check(i, w)             admissibility of cell i's new iterate
//   void store(i, w)             caches derived values of cell i's iterate
// Fe[KMAX+1][NV], we[KMAX+1]: the caller sets the outer edges 0 and K.
// ------------------------------------------------------------------------------------------
template <class Sys, int KMAX>
__device__ __forceinline__ int dts_thread(Sys& S, const int K, const double dt, const long long max_iter,
                                          const DtsCell<Sys::NV> (&c)[KMAX], double (&Fe)[KMAX + 1][Sys::NV],
                                          double (&we)[KMAX + 1], double (&u1)[KMAX][Sys::NV], double (&h1)[KMAX],
                                          long long& l_out, int& marg) {
  constexpr int NV = Sys::NV;
  double W[KMAX][NV], i1r[KMAX], qr[KMAX], rsc[KMAX];
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    double r = 0.0, dtau = 1.0;
#pragma unroll
    for (int q = 0; q < NV; ++q) W[i][q] = 0.0;
    if (i < K) {
      dtau = c[i].theta * dt;
      r = dtau / dt;
#pragma unroll
      for (int q = 0; q < NV; ++q) W[i][q] = c[i].un[q];
      S.store(i, W[i]);
    }
    i1r[i] = 1.0 / (1.0 + r); qr[i] = r * i1r[i]; rsc[i] = (1.0 + r) / dtau;
  }
  long long l = 0;
  int err = 0;
  bool prev_cont_robust = true;
  for (int part = 0; part < 2 && !err; ++part) {
    for (;;) {
      {  // (a) interior edges at W^l
        const int s = S.edges(K, W, Fe, we);
        if (s > err) err = s;
      }
      if (err || part == 1) break;
      bool conv = true, rstop = true, rcont = false;
      int bad = 0;
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {  // (b) relaxed moving-cell update, residual
        if (i < K) {
          int bi = 0;
          const double hl_ = __dadd_rn(c[i].hn, __dmul_rn(we[i + 1] - we[i], dt));
          if (!(hl_ > 0.0)) bi = ST_WIDTH;
          const double ih = 1.0 / hl_, a0 = c[i].hn * ih, a1 = dt * ih;
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const double fL = Fe[i][q], fR = Fe[i + 1][q], w = W[i][q];
            const double nq = dts_relax(w, i1r[i], qr[i], a0, c[i].un[q], a1, fL, fR);
            const double d = dts_resid(rsc[i], nq, w), t = dts_tol(c[i].tol, w);
            conv = conv && d < t;
            const double eb = dts_margin(rsc[i], w, qr[i], a0, c[i].un[q], a1, fL, fR);
            rstop = rstop && d < t - eb;
            rcont = rcont || d >= t + eb;
            W[i][q] = nq;
          }
          const int s = S.check(i, W[i]);
          if (s && !bi) bi = s;
          if (bi > bad) bad = bi;
          S.store(i, W[i]);
        }
      }
      if (conv && (!rstop || !prev_cont_robust)) marg += 1;
      prev_cont_robust = rcont;
      ++l;
      if (bad) { err = bad; break; }
      if (conv) break;
      if (l >= max_iter) { err = ST_DTS_CAP; break; }
    }
  }
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {  // Part 2 (b): conservative update with F_left, F*, F_right
    if (!err && i < K) {
      const double hn1 = __dadd_rn(c[i].hn, __dmul_rn(we[i + 1] - we[i], dt));
      if (!(hn1 > 0.0)) err = ST_WIDTH;
      else {
#pragma unroll
        for (int q = 0; q < NV; ++q) u1[i][q] = dts_final(c[i].hn, hn1, c[i].un[q], dt, Fe[i][q], Fe[i + 1][q]);
        h1[i] = hn1;
      }
    }
  }
  l_out = l;
  return err;
}

}  // namespace eis
