// tools/newton_latency.cu — latency of one half-warp phase-boundary solve (development tool).
// One warp per CTA, both half warps solve a C3-like boundary (liquid | vapour bubble) R times,
// cold (HLLC start) and warm (start at the previous root); prints cycles per solve and the
// Newton iteration counts.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2211_00705_b200/csrc
#include <cstdio>
#include <cmath>
#include "eis_device.cuh"

using namespace eis;

__global__ void k(const __grid_constant__ Eos e, const __grid_constant__ Prm p, int R, int warm, long long* cyc, int* its, double* out) {
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  // liquid at 999 kg/m^3 moving away at 150 m/s from a vapour cell of 0.01 kg/m^3 at rest
  double rl = 999.0 + 0.3 * blockIdx.x * 1e-3, ul = -150.0, rv = 0.01, uv = 0.0;
  double x0 = -1, x1 = -1;
  IfaceSol s0 = iface_solve_hw(e, p, rl, ul, rv, uv, false, x0, x1, hmask, hl, half * 16);
  if (warm) { x0 = s0.pV; x1 = s0.pL; }
  long long t0 = clock64();
  int itsum = 0;
  double acc = 0;
  for (int r = 0; r < R; ++r) {
    IfaceSol s = iface_solve_hw(e, p, rl, ul + 1e-9 * r, rv, uv, false, x0, x1, hmask, hl, half * 16);
    itsum += s.iters;
    acc += s.F1;
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[blockIdx.x] = (t1 - t0) / R; its[blockIdx.x] = itsum; out[blockIdx.x] = acc; }
}

int main_solve(Eos& e, Prm& p, long long* cyc, int* its, double* out);
int main() {
  Eos e;
  e.a_v2 = 1.352e5; e.a_v = sqrt(e.a_v2); e.a_l = 1500; e.a_l2 = 1500.0 * 1500.0; e.rho0 = 998; e.p0 = 2339;
  e.tau = 1.0 / sqrt(2 * M_PI) * pow(e.a_v2, -1.5); e.rho_min = 993.998960444; e.rho_tilde = 0.0323381031;
  e.inv_av2 = 1 / e.a_v2; e.inv_al2 = 1 / e.a_l2; e.inv_p0 = 1 / e.p0; e.inv_av = 1 / e.a_v; e.inv_rho0 = 1 / e.rho0;
  Prm p;
  p.cfl = 0.9; p.eps_split = 2; p.eps_tiny = 0.5; p.theta_nb = 0.9; p.tol_nb = 1e-3; p.tol_tiny = 0.1;
  p.newton_rtol = 1e-13; p.newton_gtol = 1e-12; p.newton_stol = sqrt(1e-13); p.h_av = 1e-3; p.dts_max_iter = 1000000; p.newton_max_iter = 50;
  p.armijo_max = 30; p.mode = 0;
  long long* cyc; int* its; double* out;
  cudaMallocManaged(&cyc, 8 * 1024); cudaMallocManaged(&its, 4 * 1024); cudaMallocManaged(&out, 8 * 1024);
  return main_solve(e, p, cyc, its, out);
}
int main_solve(Eos& e, Prm& p, long long* cyc, int* its, double* out) {
  for (int warm = 0; warm < 2; ++warm) {
    for (int blocks : {1, 148, 592}) {
      k<<<blocks, 32>>>(e, p, 100, warm, cyc, its, out);
      cudaDeviceSynchronize();
      printf("{\"warm\": %d, \"ctas\": %d, \"cycles_per_solve\": %lld, \"newton_iters_per_solve\": %.2f}\n", warm, blocks,
             cyc[0], its[0] / 100.0);
    }
  }
  extern int main_eval_only(Eos&, long long*, double*);
  return main_eval_only(e, cyc, out);
}
__global__ void k_eval(const __grid_constant__ Eos e, int R, long long* cyc, double* out);
// (appended) per-evaluation latency probe
__global__ void k_eval(const __grid_constant__ Eos e, int R, long long* cyc, double* out) {
  IfaceProb P;
  P.rV = 0.01; P.uV = 0.0; P.rL = 999.0; P.uL = -150.0; P.sV = 1.0; P.du = 150.0;
  double G[2], J[4], aux[2], da[4], acc = 0, x0 = 500.0 + threadIdx.x, x1 = 600.0;
  long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
    iface_eval(e, P, x0, x1, G, J, aux, da);
    x0 += 1e-9 * G[0]; x1 += 1e-9 * J[3];  // dependent chain
    acc += aux[0];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / R; out[0] = acc + x0 + x1; }
}

__global__ void k_lin(const __grid_constant__ Eos e, const __grid_constant__ Prm p, int R, long long* cyc, double* out) {
  // warm-started one-evaluation solve (iface_try_lin, the DTS inner solve): start at the root
  double rl = 999.0, ul = -150.0, rv = 0.01, uv = 0.0;
  IfaceSol s0 = iface_solve_t(e, p, rl, ul, rv, uv, false, -1.0, -1.0);
  double x0 = s0.pV, x1 = s0.pL, acc = 0;
  int ok = 0;
  long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
    IfaceSol s;
    const bool b = iface_try_lin(e, p, rl, ul + 1e-12 * (r & 7) + 1e-13 * acc, rv, uv, false, x0, x1, s);
    ok += b;
    acc += 1e-30 * s.F1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / R; out[0] = acc + ok; out[1] = ok; }
}
int main_eval_only(Eos& e, long long* cyc, double* out) {
  Prm p;
  p.cfl = 0.9; p.eps_split = 2; p.eps_tiny = 0.5; p.theta_nb = 0.9; p.tol_nb = 1e-3; p.tol_tiny = 0.1;
  p.newton_rtol = 1e-13; p.newton_gtol = 1e-12; p.newton_stol = sqrt(1e-13); p.h_av = 1e-3; p.dts_max_iter = 1000000; p.newton_max_iter = 50;
  p.armijo_max = 30; p.mode = 0; p.lin_gtol = 1e-6;
  k_lin<<<1, 1>>>(e, p, 200, cyc, out);
  cudaDeviceSynchronize();
  printf("{\"try_lin_cycles\": %lld, \"accepted\": %.0f}\n", cyc[0], out[1]);

  for (int th : {1, 32}) {
    k_eval<<<1, th>>>(e, 200, cyc, out);
    cudaDeviceSynchronize();
    printf("{\"iface_eval_cycles\": %lld, \"threads\": %d}\n", cyc[0], th);
  }
  return 0;
}
