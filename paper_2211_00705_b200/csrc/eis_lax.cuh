// eis_lax.cuh — the paper's first test on the GPU: batches of Lax shock tubes of
// the full 1D Euler equations (ideal gas) on a fixed mesh with one small cell of
// width alpha*h (readings L1-L7), exact Riemann fluxes and dual time
// stepping on the cells k-1, k, k+1 through THE SAME warp loop as the two-phase hot path
// (eis_dts.cuh dts_warp, instantiated for NV = 3).
//
// One CTA per case, the mesh (N + 1 <= 4095 cells) resident in shared memory for the whole run:
// per step a block reduction for dt, one exact Riemann solve per face (a thread per face), the
// explicit update of the cells outside the block, then warp 0 runs Algorithm 2 on the block.
//
// The exact Riemann solver is written here from the gas dynamics, not from the oracle: the star
// pressure by Newton from the two-rarefaction pressure (a lower bound of p*, from which the
// iterates of the increasing, concave wave-curve function rise monotonically: no floor and no
// damping), shock curves in mass-flux form Q_K = sqrt(rho_K ((g+1) p + (g-1) p_K) / 2), star
// densities behind shocks from mass conservation across the shock, rarefaction fans from the
// Riemann invariant and the isentrope.
#pragma once

#include <cuda_runtime.h>

#include <cmath>

#include "eis.h"
#include "eis_dts.cuh"

namespace eis {
namespace lax {

struct Side { double r, u, p, c; };  // primitive state and sound speed of one side

// the velocity jump across side K's outer wave at star pressure ps, and its derivative:
// shock (ps > p_K, Rankine-Hugoniot): f = (ps - p_K) / Q_K; rarefaction (isentrope + Riemann
// invariant): f = 2 c_K / (g - 1) ((ps / p_K)^z - 1), z = (g - 1) / (2 g)
__device__ __forceinline__ void wave(double g, const Side& K, double ps, double& f, double& df) {
  if (ps > K.p) {
    const double B = 0.5 * ((g + 1.0) * ps + (g - 1.0) * K.p);
    const double Q = sqrt(K.r * B);
    f = (ps - K.p) / Q;
    df = (1.0 - 0.25 * (g + 1.0) * (ps - K.p) / B) / Q;
  } else {
    const double s = exp((g - 1.0) / (2.0 * g) * log(ps / K.p));
    f = 2.0 * K.c / (g - 1.0) * (s - 1.0);
    df = K.c * s / (g * ps);
  }
}

// star pressure and velocity of the Riemann problem (L, R): 0, EIS_E_NONPOS_DENSITY (vacuum is
// generated) or EIS_E_NEWTON (reading L4: converged when the Newton correction is <= 2e-15 p)
__device__ int star(double g, const Side& L, const Side& R, double& ps, double& us) {
  const double du = R.u - L.u;
  const double z = (g - 1.0) / (2.0 * g);
  const double num = L.c + R.c - 0.5 * (g - 1.0) * du;
  if (!(num > 0.0)) return EIS_E_NONPOS_DENSITY;
  double p = pow(num / (L.c * pow(L.p, -z) + R.c * pow(R.p, -z)), 1.0 / z);  // two rarefactions
  double fl, dfl, fr, dfr, d = INFINITY;
  for (int it = 0; it < 60 && !(fabs(d) <= 2e-15 * p); ++it) {
    wave(g, L, p, fl, dfl);
    wave(g, R, p, fr, dfr);
    d = (fl + fr + du) / (dfl + dfr);
    p -= d;
  }
  if (!(fabs(d) <= 2e-15 * p) || !(p > 0.0)) return EIS_E_NEWTON;
  wave(g, L, p, fl, dfl);
  wave(g, R, p, fr, dfr);
  ps = p;
  us = 0.5 * (L.u + R.u) + 0.5 * (fr - fl);
  return 0;
}

// the self-similar solution on the t-axis (x/t = 0), primitive (r, u, p)
__device__ void on_axis(double g, const Side& L, const Side& R, double ps, double us, double& r, double& u, double& p) {
  const double z = (g - 1.0) / (2.0 * g);
  if (us >= 0.0) {  // the axis lies left of the contact: the left wave decides
    if (ps > L.p) {  // shock moving at S = u_L - Q_L / rho_L; rho* (u* - S) = Q_L
      const double Q = sqrt(L.r * 0.5 * ((g + 1.0) * ps + (g - 1.0) * L.p));
      const double S = L.u - Q / L.r;
      if (S >= 0.0) { r = L.r; u = L.u; p = L.p; }
      else { r = Q / (us - S); u = us; p = ps; }
    } else if (L.u - L.c >= 0.0) {  // rarefaction head right of the axis
      r = L.r; u = L.u; p = L.p;
    } else if (us - L.c * exp(z * log(ps / L.p)) <= 0.0) {  // tail left of the axis: star state
      r = L.r * exp(log(ps / L.p) / g); u = us; p = ps;
    } else {  // inside the fan: u - c = 0 and u + 2c/(g-1) = u_L + 2 c_L/(g-1)
      const double c = (g - 1.0) / (g + 1.0) * (L.u + 2.0 * L.c / (g - 1.0));
      r = L.r * exp(2.0 / (g - 1.0) * log(c / L.c)); u = c; p = L.p * exp(g * log(r / L.r));
    }
  } else {  // right of the contact: the right wave decides
    if (ps > R.p) {  // shock moving at S = u_R + Q_R / rho_R; rho* (S - u*) = Q_R
      const double Q = sqrt(R.r * 0.5 * ((g + 1.0) * ps + (g - 1.0) * R.p));
      const double S = R.u + Q / R.r;
      if (S <= 0.0) { r = R.r; u = R.u; p = R.p; }
      else { r = Q / (S - us); u = us; p = ps; }
    } else if (R.u + R.c <= 0.0) {  // rarefaction head left of the axis
      r = R.r; u = R.u; p = R.p;
    } else if (us + R.c * exp(z * log(ps / R.p)) >= 0.0) {  // tail right of the axis: star state
      r = R.r * exp(log(ps / R.p) / g); u = us; p = ps;
    } else {  // inside the fan: u + c = 0 and u - 2c/(g-1) = u_R - 2 c_R/(g-1)
      const double c = -(g - 1.0) / (g + 1.0) * (R.u - 2.0 * R.c / (g - 1.0));
      r = R.r * exp(2.0 / (g - 1.0) * log(c / R.c)); u = -c; p = R.p * exp(g * log(r / R.r));
    }
  }
}

// Godunov flux of the face between the conserved states (r, m, E) of its two cells:
// F = (m, m u + p, u (g/(g-1) p + m u / 2)); 0 or a status.  One compiled copy (noinline), so the
// warp and the one-thread DTS loops see the same flux bits.
__device__ __noinline__ int face_flux(double g, double r0, double m0, double E0, double r1, double m1, double E1, double F[3]) {
  if (!(r0 > 0.0) || !(r1 > 0.0)) return EIS_E_NONPOS_DENSITY;
  Side L, R;
  L.r = r0; L.u = m0 / r0; L.p = (g - 1.0) * (E0 - 0.5 * m0 * L.u);
  R.r = r1; R.u = m1 / r1; R.p = (g - 1.0) * (E1 - 0.5 * m1 * R.u);
  if (!(L.p > 0.0) || !(R.p > 0.0)) return EIS_E_NONPOS_DENSITY;
  L.c = sqrt(g * L.p / L.r);
  R.c = sqrt(g * R.p / R.r);
  double ps, us;
  const int s = star(g, L, R, ps, us);
  if (s) return s;
  double r, u, p;
  on_axis(g, L, R, ps, us, r, u, p);
  const double m = r * u;
  F[0] = m;
  F[1] = m * u + p;
  F[2] = u * (g / (g - 1.0) * p + 0.5 * m * u);
  return 0;
}

// the Euler system for the generic DTS loop: fixed mesh (edge speeds 0), exact fluxes
struct EulerDts {
  static constexpr int NV = 3;
  double g;
  __device__ __forceinline__ int edge(int j, double* W, double* Fe, double* we, int, int hl, unsigned) {
    if (hl) return 0;
    double F[3];
    const int s = face_flux(g, W[j - 1], W[MAXB + j - 1], W[2 * MAXB + j - 1], W[j], W[MAXB + j], W[2 * MAXB + j], F);
    Fe[j] = F[0]; Fe[MAXB + 1 + j] = F[1]; Fe[2 * (MAXB + 1) + j] = F[2];
    we[j] = 0.0;
    return s;
  }
  __device__ __forceinline__ int check(int, const double (&)[3]) const { return 0; }  // (positivity: the next flux)
  __device__ __forceinline__ void store(double*, int, const double (&)[3]) {}
};

// the same for the per-thread loop (dts_thread): one thread owns the block
struct EulerDtsT {
  static constexpr int NV = 3;
  double g;
  template <int KMAX>
  __device__ __forceinline__ int edges(int K, const double (&W)[KMAX][3], double (&Fe)[KMAX + 1][3], double (&we)[KMAX + 1]) {
    int err = 0;
#pragma unroll
    for (int j = 1; j < KMAX; ++j) {
      if (j < K) {
        we[j] = 0.0;
        const int s = face_flux(g, W[j - 1][0], W[j - 1][1], W[j - 1][2], W[j][0], W[j][1], W[j][2], Fe[j]);
        if (s > err) err = s;
      }
    }
    return err;
  }
  __device__ __forceinline__ int check(int, const double (&)[3]) const { return 0; }
  __device__ __forceinline__ void store(int, const double (&)[3]) {}
};

constexpr int LAX_THREADS = 256;
constexpr int LAX_MAX_N = 4094;

__global__ void __launch_bounds__(LAX_THREADS)
lax_cases(const eis_lax_case* __restrict__ cases, long long stride, double* rho_out, double* mom_out, double* E_out,
          eis_lax_stats* __restrict__ stats) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[LAX_THREADS / 32];
  __shared__ double dsc[dts_scratch<3>()];
  __shared__ int s_status;
  __shared__ long long s_l;
  __shared__ int s_marg;
  const eis_lax_case c = cases[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = (int)c.n, nc = N + 1, k = N / 2;
  const double g = c.gamma, hh = (c.x_right - c.x_left) / (double)N, hk = c.alpha * hh;
  const bool blk = c.implicit_block != 0;
  double* U[3] = {sm, sm + nc, sm + 2 * nc};                                   // conserved, per cell
  double* F[3] = {sm + 3 * nc, sm + 4 * nc + 1, sm + 5 * nc + 2};              // F[q][f]: left face of cell f
  for (int i = tid; i < nc; i += blockDim.x) {  // L1: the small cell k and the cells right of it hold the right state
    const bool left = i < k;
    const double r = left ? c.rho_l : c.rho_r, u = left ? c.u_l : c.u_r, p = left ? c.p_l : c.p_r;
    U[0][i] = r; U[1][i] = r * u; U[2][i] = p / (g - 1.0) + 0.5 * r * u * u;
  }
  if (tid == 0) { s_status = 0; s_marg = 0; }
  long long steps = 0, dts_iters = 0, dts_max = 0, solves = 0;
  double t = 0.0;
  __syncthreads();
  while (t < c.t_end) {
    // ---- dt (L2): max |u| + c over the regular cells; h_min with the small cell only without
    // the block (every status check is a __syncthreads_or: the break is uniform over the CTA)
    int err = 0;
    double smax = 0.0;
    for (int i = tid; i < nc; i += blockDim.x) {
      if (blk && i == k) continue;
      const double r = U[0][i], u = U[1][i] / r, p = (g - 1.0) * (U[2][i] - 0.5 * U[1][i] * u);
      if (!(r > 0.0) || !(p > 0.0)) { err = EIS_E_NONPOS_DENSITY; continue; }
      smax = fmax(smax, fabs(u) + sqrt(g * p / r));
    }
    for (int o = 16; o > 0; o >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
    if (lane == 0) red[warp] = smax;
    if (err) atomicCAS(&s_status, 0, err);
    if (__syncthreads_or(err)) break;
    smax = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) smax = fmax(smax, red[w]);
    double dt = c.cfl * (blk ? hh : fmin(hh, hk)) / smax;
    if (t + dt > c.t_end) dt = c.t_end - t;  // L6
    // ---- exact fluxes from U^n on every face, transmissive ends (L3)
    for (int f = tid; f <= nc; f += blockDim.x) {
      const int a = f == 0 ? 0 : f - 1, b = f == nc ? nc - 1 : f;
      double G[3];
      const int s = face_flux(g, U[0][a], U[1][a], U[2][a], U[0][b], U[1][b], U[2][b], G);
      if (s) { err = s; atomicCAS(&s_status, 0, s); }
      F[0][f] = G[0]; F[1][f] = G[1]; F[2][f] = G[2];
    }
    if (__syncthreads_or(err)) break;
    // ---- explicit update of every cell outside the block (fixed mesh)
    for (int i = tid; i < nc; i += blockDim.x) {
      if (blk && i >= k - 1 && i <= k + 1) continue;
      const double q = dt / (i == k ? hk : hh);
      for (int v = 0; v < 3; ++v) U[v][i] = U[v][i] - q * (F[v][i + 1] - F[v][i]);
    }
    if (blk && warp == 0 && c.dts_loop) {  // ---- Algorithm 2 on {k-1, k, k+1}, one thread (dts_thread)
      int e = 0;
      if (lane == 0) {
        DtsCell<3> cell[3];
        double Fe[4][3], we[4] = {0.0, 0.0, 0.0, 0.0}, u1[3][3], h1[3];
        for (int i = 0; i < 3; ++i) {
          for (int v = 0; v < 3; ++v) { cell[i].un[v] = U[v][k - 1 + i]; Fe[i + 1][v] = 0.0; }
          cell[i].hn = i == 1 ? hk : hh;
          cell[i].theta = i == 1 ? c.alpha : c.theta_nb;
          cell[i].tol = i == 1 ? c.tol_tiny : c.tol_nb;
        }
        for (int v = 0; v < 3; ++v) { Fe[0][v] = F[v][k - 1]; Fe[3][v] = F[v][k + 2]; }
        EulerDtsT S{g};
        long long l = 0;
        int marg = 0;
        e = dts_thread<EulerDtsT, 3>(S, 3, dt, c.dts_max_iter, cell, Fe, we, u1, h1, l, marg);
        if (!e)
          for (int i = 0; i < 3; ++i)
            for (int v = 0; v < 3; ++v) U[v][k - 1 + i] = u1[i][v];
        if (e) atomicCAS(&s_status, 0, e);
        s_l = l;
        s_marg += marg;
      }
      err = __shfl_sync(0xffffffffu, e, 0);
    } else if (blk && warp == 0) {  // ---- Algorithm 2 on {k-1, k, k+1} (the warp loop, dts_warp, NV = 3)
      double* Fe = dsc + 3 * MAXB;
      double* we = Fe + 3 * (MAXB + 1);
      if (lane < 3) {  // outer faces keep the explicit fluxes (flux bounding)
        Fe[lane * (MAXB + 1)] = F[lane][k - 1];
        Fe[lane * (MAXB + 1) + 3] = F[lane][k + 2];
      }
      if (lane == 0) { we[0] = 0.0; we[3] = 0.0; }
      DtsCell<3> cell{};
      if (lane < 3) {
        for (int v = 0; v < 3; ++v) cell.un[v] = U[v][k - 1 + lane];  // (the block cells still hold U^n)
        cell.hn = lane == 1 ? hk : hh;
        cell.theta = lane == 1 ? c.alpha : c.theta_nb;  // P:1127, theta_k = alpha
        cell.tol = lane == 1 ? c.tol_tiny : c.tol_nb;
      }
      __syncwarp();
      EulerDts S{g};
      double u1[3] = {0.0, 0.0, 0.0}, h1 = 0.0;
      long long l = 0;
      int marg = 0;
      const int e = dts_warp(S, dsc, 3, dt, c.dts_max_iter, cell, u1, h1, l, marg);
      if (!e && lane < 3)
        for (int v = 0; v < 3; ++v) U[v][k - 1 + lane] = u1[v];
      if (lane == 0) {
        if (e) atomicCAS(&s_status, 0, e);  // (ST_* are the eis_status values)
        s_l = l;
        s_marg += marg;
      }
      err = e;
    }
    if (__syncthreads_or(err)) break;
    if (blk) {
      const long long l = s_l;
      dts_iters += l;
      if (l > dts_max) dts_max = l;
      solves += 2 * (l + 1);
    }
    solves += nc + 1;
    t += dt;
    ++steps;
  }
  __syncthreads();
  const long long base = (long long)blockIdx.x * stride;
  for (int i = tid; i < nc; i += blockDim.x) {
    rho_out[base + i] = U[0][i];
    mom_out[base + i] = U[1][i];
    E_out[base + i] = U[2][i];
  }
  if (tid == 0) {
    eis_lax_stats s;
    s.steps = steps; s.dts_iters = dts_iters; s.dts_max = dts_max; s.riemann_solves = solves;
    s.t = t; s.status = s_status; s.margins = s_marg;
    stats[blockIdx.x] = s;
  }
}

inline size_t smem_bytes(int N) { return sizeof(double) * (3 * (size_t)(N + 1) + 3 * (size_t)(N + 2)); }

}  // namespace lax
}  // namespace eis
