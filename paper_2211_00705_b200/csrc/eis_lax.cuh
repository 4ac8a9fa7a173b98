// eis_lax.cuh — the paper's first test on the GPU: batches of Lax shock tubes of
// the full 1D Euler equations (ideal gas) on a fixed mesh with one small cell of width alpha*h,
// exact Riemann fluxes and dual time stepping, Algorithm 2, on the cells
// k-1, k, k+1 -- the same DTS loop as the two-phase kernels, for a 3-equation system.
//
// One CTA per case, the mesh (N + 1 <= 4095 cells) resident in shared memory for the whole run:
// per step a block reduction for dt, one exact Riemann solve per face (a thread per face), the
// explicit update of the cells outside the block, then warp 0 runs the DTS loop: lanes 0 and 1
// solve the two interior faces in parallel, lanes 0..2 update the three block cells, the
// residual is a warp max.  Readings L1-L7.
#pragma once

#include <cuda_runtime.h>

#include <cmath>

#include "eis.h"

namespace eis {
namespace lax {

// f_K(p) and f_K'(p) of the gamma-law Riemann problem: shock branch from the Rankine-Hugoniot
// conditions, rarefaction branch from the isentrope and the Riemann invariant
__device__ __forceinline__ void fk(double g, double p, double rk, double pk, double ck, double& f, double& df) {
  if (p > pk) {
    const double A = 2.0 / ((g + 1.0) * rk), B = (g - 1.0) / (g + 1.0) * pk;
    const double q = sqrt(A / (B + p));
    f = (p - pk) * q;
    df = q * (1.0 - (p - pk) / (2.0 * (B + p)));
  } else {
    const double e = (g - 1.0) / (2.0 * g);
    f = 2.0 * ck / (g - 1.0) * (pow(p / pk, e) - 1.0);
    df = 1.0 / (rk * ck) * pow(p / pk, -(g + 1.0) / (2.0 * g));
  }
}

// Godunov flux of the exact solution at x/t = 0 for primitive states (rho, u, p); returns 0,
// EIS_E_NONPOS_DENSITY (non-positive state or vacuum) or EIS_E_NEWTON.  Star pressure by Newton
// from the primitive-variable estimate, stop when 2|dp|/(p_new + p) <= 1e-14 (reading L4).
__device__ int exact_flux(double g, double rl, double ul, double pl, double rr, double ur, double pr, double F[3]) {
  if (!(rl > 0.0) || !(rr > 0.0) || !(pl > 0.0) || !(pr > 0.0)) return EIS_E_NONPOS_DENSITY;
  const double cl = sqrt(g * pl / rl), cr = sqrt(g * pr / rr);
  if (2.0 / (g - 1.0) * (cl + cr) <= ur - ul) return EIS_E_NONPOS_DENSITY;  // vacuum
  const double pfloor = 1e-8 * fmin(pl, pr);
  double p = 0.5 * (pl + pr) - 0.125 * (ur - ul) * (rl + rr) * (cl + cr);
  if (p < pfloor) p = pfloor;
  bool ok = false;
  for (int it = 1; it <= 100; ++it) {
    double fL, dfL, fR, dfR;
    fk(g, p, rl, pl, cl, fL, dfL);
    fk(g, p, rr, pr, cr, fR, dfR);
    double pn = p - (fL + fR + ur - ul) / (dfL + dfR);
    if (pn < pfloor) pn = pfloor;
    const double change = 2.0 * fabs(pn - p) / (pn + p);
    p = pn;
    if (change <= 1e-14) { ok = true; break; }
  }
  if (!ok) return EIS_E_NEWTON;
  double fL, dfL, fR, dfR;
  fk(g, p, rl, pl, cl, fL, dfL);
  fk(g, p, rr, pr, cr, fR, dfR);
  const double u = 0.5 * (ul + ur) + 0.5 * (fR - fL);
  // the state at x/t = 0
  const double gm = (g - 1.0) / (g + 1.0);
  double r, v, q;
  if (0.0 <= u) {  // left of the contact
    if (p > pl) {
      const double sl = ul - cl * sqrt((g + 1.0) / (2.0 * g) * p / pl + (g - 1.0) / (2.0 * g));
      if (0.0 <= sl) { r = rl; v = ul; q = pl; }
      else { r = rl * (p / pl + gm) / (gm * p / pl + 1.0); v = u; q = p; }
    } else {
      const double cs = cl * pow(p / pl, (g - 1.0) / (2.0 * g));
      if (0.0 <= ul - cl) { r = rl; v = ul; q = pl; }
      else if (0.0 >= u - cs) { r = rl * pow(p / pl, 1.0 / g); v = u; q = p; }
      else {
        const double c = 2.0 / (g + 1.0) * (cl + 0.5 * (g - 1.0) * (ul - 0.0));
        v = 2.0 / (g + 1.0) * (cl + 0.5 * (g - 1.0) * ul + 0.0);
        r = rl * pow(c / cl, 2.0 / (g - 1.0));
        q = pl * pow(c / cl, 2.0 * g / (g - 1.0));
      }
    }
  } else {
    if (p > pr) {
      const double sr = ur + cr * sqrt((g + 1.0) / (2.0 * g) * p / pr + (g - 1.0) / (2.0 * g));
      if (0.0 >= sr) { r = rr; v = ur; q = pr; }
      else { r = rr * (p / pr + gm) / (gm * p / pr + 1.0); v = u; q = p; }
    } else {
      const double cs = cr * pow(p / pr, (g - 1.0) / (2.0 * g));
      if (0.0 >= ur + cr) { r = rr; v = ur; q = pr; }
      else if (0.0 <= u + cs) { r = rr * pow(p / pr, 1.0 / g); v = u; q = p; }
      else {
        const double c = 2.0 / (g + 1.0) * (cr - 0.5 * (g - 1.0) * (ur - 0.0));
        v = 2.0 / (g + 1.0) * (-cr + 0.5 * (g - 1.0) * ur + 0.0);
        r = rr * pow(c / cr, 2.0 / (g - 1.0));
        q = pr * pow(c / cr, 2.0 * g / (g - 1.0));
      }
    }
  }
  const double En = q / (g - 1.0) + 0.5 * r * v * v;
  F[0] = r * v;
  F[1] = r * v * v + q;
  F[2] = v * (En + q);
  return 0;
}

// flux of a face from the conserved states of its two cells
__device__ __forceinline__ int face_flux(double g, double r0, double m0, double e0, double r1, double m1, double e1,
                                         double F[3]) {
  if (!(r0 > 0.0) || !(r1 > 0.0)) return EIS_E_NONPOS_DENSITY;
  const double u0 = m0 / r0, u1 = m1 / r1;
  const double p0 = (g - 1.0) * (e0 - 0.5 * m0 * m0 / r0), p1 = (g - 1.0) * (e1 - 0.5 * m1 * m1 / r1);
  return exact_flux(g, r0, u0, p0, r1, u1, p1, F);
}

__device__ __forceinline__ double warp_max_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

constexpr int LAX_THREADS = 256;
constexpr int LAX_MAX_N = 4094;

__global__ void __launch_bounds__(LAX_THREADS)
lax_cases(const eis_lax_case* __restrict__ cases, long long stride, double* rho_out, double* mom_out, double* E_out,
          eis_lax_stats* __restrict__ stats) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[LAX_THREADS / 32];
  __shared__ int s_status;
  __shared__ double Un[3][3], W[3][3], G[4][3];
  __shared__ long long s_l;
  const eis_lax_case c = cases[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = (int)c.n, nc = N + 1, k = N / 2;
  const double g = c.gamma, hh = (c.x_right - c.x_left) / (double)N, hk = c.alpha * hh;
  const bool blk = c.implicit_block != 0;
  double* U0 = sm;
  double* U1 = U0 + nc;
  double* U2 = U1 + nc;
  double* F0 = U2 + nc;        // F*[f]: flux at the left face of cell f, f = 0..nc
  double* F1 = F0 + nc + 1;
  double* F2 = F1 + nc + 1;
  for (int i = tid; i < nc; i += blockDim.x) {  // L1: the small cell k and the cells right of it hold the right state
    const bool left = i < k;
    const double r = left ? c.rho_l : c.rho_r, u = left ? c.u_l : c.u_r, p = left ? c.p_l : c.p_r;
    U0[i] = r; U1[i] = r * u; U2[i] = p / (g - 1.0) + 0.5 * r * u * u;
  }
  if (tid == 0) s_status = 0;
  long long steps = 0, dts_iters = 0, dts_max = 0, solves = 0;
  double t = 0.0;
  __syncthreads();
  while (t < c.t_end) {
    // ---- dt (L2): max |u| + c over the regular cells (all cells and h_min without the block)
    // (every status check is a __syncthreads_or: the break is uniform over the CTA)
    int err = 0;
    double smax = 0.0;
    for (int i = tid; i < nc; i += blockDim.x) {
      if (blk && i == k) continue;
      const double r = U0[i], u = U1[i] / r, p = (g - 1.0) * (U2[i] - 0.5 * U1[i] * U1[i] / r);
      if (!(r > 0.0) || !(p > 0.0)) { err = EIS_E_NONPOS_DENSITY; continue; }
      smax = fmax(smax, fabs(u) + sqrt(g * p / r));
    }
    smax = warp_max_d(smax);
    if (lane == 0) red[warp] = smax;
    if (err) atomicCAS(&s_status, 0, err);
    if (__syncthreads_or(err)) break;
    smax = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) smax = fmax(smax, red[w]);
    const double hmin = blk ? hh : fmin(hh, hk);
    double dt = c.cfl * hmin / smax;
    if (t + dt > c.t_end) dt = c.t_end - t;  // L6
    // ---- exact fluxes from U^n on every face, transmissive ends (L3)
    for (int f = tid; f <= nc; f += blockDim.x) {
      const int a = f == 0 ? 0 : f - 1, b = f == nc ? nc - 1 : f;
      double F[3];
      const int s = face_flux(g, U0[a], U1[a], U2[a], U0[b], U1[b], U2[b], F);
      if (s) { err = s; atomicCAS(&s_status, 0, s); }
      F0[f] = F[0]; F1[f] = F[1]; F2[f] = F[2];
    }
    if (tid < 9 && blk) Un[tid / 3][tid % 3] = (tid % 3 == 0 ? U0 : tid % 3 == 1 ? U1 : U2)[k - 1 + tid / 3];
    if (__syncthreads_or(err)) break;
    // ---- explicit update of every cell outside the block (fixed mesh)
    for (int i = tid; i < nc; i += blockDim.x) {
      if (blk && i >= k - 1 && i <= k + 1) continue;
      const double q = dt / (i == k ? hk : hh);
      U0[i] = U0[i] - q * (F0[i + 1] - F0[i]);
      U1[i] = U1[i] - q * (F1[i + 1] - F1[i]);
      U2[i] = U2[i] - q * (F2[i + 1] - F2[i]);
    }
    long long l = 0;
    if (blk && warp == 0) {  // ---- Algorithm 2 on {k-1, k, k+1}
      const double theta = lane == 1 ? c.alpha : c.theta_nb;  // P:1127, theta_k = alpha
      const double hi = lane == 1 ? hk : hh;
      if (lane < 9) W[lane / 3][lane % 3] = Un[lane / 3][lane % 3];
      if (lane < 3) {  // outer faces keep the explicit fluxes
        G[0][lane] = (lane == 0 ? F0 : lane == 1 ? F1 : F2)[k - 1];
        G[3][lane] = (lane == 0 ? F0 : lane == 1 ? F1 : F2)[k + 2];
      }
      __syncwarp();
      for (int part = 0; part < 2 && !err; ++part) {  // part 1: fluxes at the accepted iterate
        for (;;) {
          if (lane < 2) {  // (a) the two interior faces in parallel
            double F[3];
            const int s = face_flux(g, W[lane][0], W[lane][1], W[lane][2], W[lane + 1][0], W[lane + 1][1],
                                    W[lane + 1][2], F);
            if (s) err = s;
            G[lane + 1][0] = F[0]; G[lane + 1][1] = F[1]; G[lane + 1][2] = F[2];
          }
          err = __reduce_max_sync(0xffffffffu, err);
          __syncwarp();
          if (err || part == 1) break;
          double rj = 0.0, wn[3];  // (b) the update of P:683-688 and the residual of P:1128-1131
          if (lane < 3) {
            const double r = theta, dtau = theta * dt;
            for (int q = 0; q < 3; ++q) {
              const double target = Un[lane][q] - dt / hi * (G[lane + 1][q] - G[lane][q]);
              wn[q] = W[lane][q] / (1.0 + r) + r / (1.0 + r) * target;
              rj = fmax(rj, fabs((1.0 + r) * (wn[q] - W[lane][q]) / (dtau * fmax(fabs(W[lane][q]), 1.0))));
            }
          }
          __syncwarp();
          if (lane < 3) { W[lane][0] = wn[0]; W[lane][1] = wn[1]; W[lane][2] = wn[2]; }
          const double r_nb = warp_max_d(lane == 0 || lane == 2 ? rj : 0.0);
          const double r_t = __shfl_sync(0xffffffffu, rj, 1);
          __syncwarp();
          ++l;
          if (r_nb < c.tol_nb && r_t < c.tol_tiny) break;
          if (l >= c.dts_max_iter) { err = EIS_E_DTS_CAP; break; }
        }
      }
      if (!err && lane < 3) {  // Part 2: conservative update with the outer explicit fluxes
        const int i = k - 1 + lane;
        const double q = dt / hi;
        U0[i] = Un[lane][0] - q * (G[lane + 1][0] - G[lane][0]);
        U1[i] = Un[lane][1] - q * (G[lane + 1][1] - G[lane][1]);
        U2[i] = Un[lane][2] - q * (G[lane + 1][2] - G[lane][2]);
      }
      if (lane == 0) {
        if (err) atomicCAS(&s_status, 0, err);
        s_l = l;
      }
    }
    if (__syncthreads_or(err)) break;
    if (blk) {
      l = s_l;
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
    rho_out[base + i] = U0[i];
    mom_out[base + i] = U1[i];
    E_out[base + i] = U2[i];
  }
  if (tid == 0) {
    eis_lax_stats s;
    s.steps = steps; s.dts_iters = dts_iters; s.dts_max = dts_max; s.riemann_solves = solves;
    s.t = t; s.status = s_status; s.reserved = 0;
    stats[blockIdx.x] = s;
  }
}

inline size_t smem_bytes(int N) { return sizeof(double) * (3 * (size_t)(N + 1) + 3 * (size_t)(N + 2)); }

}  // namespace lax
}  // namespace eis
