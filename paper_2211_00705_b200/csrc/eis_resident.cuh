// eis_resident.cuh — the member-resident large-step kernel (ensembles C1-C4).
//
// One CTA owns one member (an independent 1D grid, R25) for a whole eis_step / eis_run_to
// call: the grid is loaded from HBM into shared memory once, advanced n_steps large steps of
// Algorithm 1 with the moving mesh (§3.4), phase creation (App. B) and
// dual time stepping (Alg. 2), and written back once.  HBM traffic is paid per call,
// not per step; inside a step the kernel is bound by the FP64 pipe and shared memory.
//
// Per-step passes:
//   A  decode: phase, u = m/rho, S_max, tiny flags, h_min, implicit blocks, dt   (a1, a2, a8)
//   B  edges: HLL flux, interface detection, creation trigger                      (a3, a4)
//   C  special edges: creation acceptance, interface + creation Newton, half-warp  (a5, a6)
//   D  explicit moving-cell update of all non-block cells                         (a7)
//   E  dual time stepping, one warp per implicit block                            (a9)
//   F  remesh: insert, merge, split (block scan + scatter), only when flagged     (a10)
#pragma once
#include "eis_device.cuh"

namespace eis {

constexpr int MAXSPEC = 32;  // special edges (interfaces + creations) per member per step
constexpr int MAXBLK = 16;   // implicit blocks per member per step
constexpr int MAXB = 8;      // cells per implicit block
constexpr int DTS_SCRATCH = 64;  // doubles of per-warp DTS scratch (inside the u array)

// per-edge / per-cell flag byte
enum : uint8_t {
  F_PH = 0x03,      // phase of cell i
  F_TINY = 0x04,    // cell i tiny (pass A) | remesh: merge partner is the left neighbour
  F_REG = 0x08,     // cell i in an implicit block (pass A) | remesh: partner is the right one
  F_SPEC = 0x10,    // edge i is special (interface or accepted creation)
  F_TRIG = 0x20,    // edge i triggered the creation test
  F_CREATE = 0x40,  // edge i carries an accepted creation
  F_MERGE = 0x80    // remesh: cells i and i+1 are merged
};

struct Spec {
  double Fl0, Fl1, wl;  // flux / speed seen by the cell LEFT of the edge
  double Fr0, Fr1, wr;  // ... by the cell RIGHT of the edge (== left for an interface)
  double rB, mB;        // created cell state
  int e, kind;          // kind: 1 interface, 2 accepted creation, 3 pending trigger, 0 void
};

struct MemberStats {
  long long steps, cell_updates, dts_iters, iface_solves, creations, splits, merges, regions;
  double dt_min, dt_max;
};

struct Members {  // global (HBM) state, member-major SoA
  double *rho, *mom, *h;
  long long* n;
  double* t;
  int* status;
  MemberStats* stats;
  long long cap;
};

struct CtaShared {
  double dt;
  double red[64];
  int n, nspec, nblk, status, remesh;
  int c_merges, c_splits, c_creations;
  int blkA[MAXBLK];
  int warp_sums[33];
  Spec spec[MAXSPEC];
};

__device__ __forceinline__ void set_status(CtaShared& sh, int code) { atomicCAS(&sh.status, 0, code); }

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// look up the special-edge record of edge e (linear search, nspec is tiny)
__device__ __forceinline__ const Spec* find_spec(const CtaShared& sh, int e) {
  for (int k = 0; k < sh.nspec; ++k)
    if (sh.spec[k].e == e && (sh.spec[k].kind == 1 || sh.spec[k].kind == 2)) return &sh.spec[k];
  return nullptr;
}

// Block-wide exclusive scan of one int per thread (thread order), returns the prefix and
// the total through *total.  Uses sh.warp_sums.
__device__ __forceinline__ int block_excl_scan(CtaShared& sh, int v, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh.warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = lane < nw ? sh.warp_sums[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sh.warp_sums[lane] = s;  // inclusive warp prefix
    if (lane == 31) sh.warp_sums[32] = s;
  }
  __syncthreads();
  int base = warp > 0 ? sh.warp_sums[warp - 1] : 0;
  *total = sh.warp_sums[32];
  int r = base + x - v;
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------------------------------
// Algorithm 2 on one implicit block [a, b] by one warp (
// R11-R13).  Interior edges are solved by the two half warps in parallel (lane-parallel
// Armijo), cell updates by lanes 0..K-1, residual (R8) by warp max.
// ------------------------------------------------------------------------------------------
__device__ __noinline__ void dts_block(const Eos& e, const Prm& p, CtaShared& sh, double* rho, double* mom, double* h,
                          const double* F0, const double* F1, const uint8_t* fl, double* sc, int a, int b,
                          double dt, long long& it_out, long long& solves) {
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  const int K = b - a + 1;
  double* W0 = sc;                // [MAXB]
  double* W1 = sc + MAXB;         // [MAXB]
  double* Fe0 = sc + 2 * MAXB;    // [MAXB+1]
  double* Fe1 = Fe0 + MAXB + 1;
  double* we = Fe1 + MAXB + 1;
  double* xs0 = we + MAXB + 1;
  double* xs1 = xs0 + MAXB + 1;
  // outer fluxes F_left = F_{a-1/2}(U^n), F_right = F_{b+1/2}(U^n): flux bounding
  if (lane == 0) {
    for (int s = 0; s < 2; ++s) {
      int ed = s == 0 ? a : b + 1;
      int j = s == 0 ? 0 : K;
      const Spec* sp = (fl[ed] & F_SPEC) ? find_spec(sh, ed) : nullptr;
      if (sp) {
        Fe0[j] = s == 0 ? sp->Fr0 : sp->Fl0;
        Fe1[j] = s == 0 ? sp->Fr1 : sp->Fl1;
        we[j] = s == 0 ? sp->wr : sp->wl;
      } else {
        Fe0[j] = F0[ed]; Fe1[j] = F1[ed]; we[j] = 0.0;
      }
    }
  }
  double rn0 = 0, rn1 = 0, hn = 0, r = 0, dtau = 1, w0 = 0, w1 = 0;
  bool tin = false;
  int ph0 = 0;
  if (lane < K) {
    rn0 = rho[a + lane]; rn1 = mom[a + lane]; hn = h[a + lane];
    tin = fl[a + lane] & F_TINY;
    ph0 = fl[a + lane] & F_PH;
    double theta = tin ? hn / p.h_av : p.theta_nb;  // theta_k = alpha = h_k^n/h_av (R12)
    dtau = theta * dt;
    r = dtau / dt;
    w0 = rn0; w1 = rn1;
    W0[lane] = w0; W1[lane] = w1;
  }
  if (lane <= K) { xs0[lane] = -1.0; xs1[lane] = -1.0; }
  __syncwarp();
  long long l = 0;
  int err = 0;
  for (int part = 0; part < 2 && !err; ++part) {
    // part 0: Part 1 iterations; part 1: Part 2 (fluxes at U*, conservative update)
    for (;;) {
      // (a) interior edges at W^l
      for (int j0 = 1; j0 < K; j0 += 2) {
        int j = j0 + half;
        if (j < K) {
          double rl = W0[j - 1], ml = W1[j - 1], rr = W0[j], mr = W1[j];
          int pl = fl[a + j - 1] & F_PH, pr = fl[a + j] & F_PH;
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
      if (part == 1) break;
      // (b) relaxed moving-cell update (P:763 form, R13) and residual
      double res_nb = 0.0, res_t = 0.0;
      int bad = 0;
      if (lane < K) {
        double hl_ = hn + (we[lane + 1] - we[lane]) * dt;
        if (!(hl_ > 0.0)) bad = ST_WIDTH;
        double q = r / (1.0 + r);
        double n0 = w0 / (1.0 + r) + q * ((hn / hl_) * rn0 - (dt / hl_) * (Fe0[lane + 1] - Fe0[lane]));
        double n1 = w1 / (1.0 + r) + q * ((hn / hl_) * rn1 - (dt / hl_) * (Fe1[lane + 1] - Fe1[lane]));
        double r0 = fabs((1.0 + r) * (n0 - w0) / (dtau * fmax(fabs(w0), 1.0)));
        double r1 = fabs((1.0 + r) * (n1 - w1) / (dtau * fmax(fabs(w1), 1.0)));
        double ri = fmax(r0, r1);
        if (tin) res_t = ri; else res_nb = ri;
        w0 = n0; w1 = n1;
        if (!(w0 > 0.0) || phase_of(e, w0) != ph0) bad = bad ? bad : ST_SPINODAL;
      }
      res_nb = warp_max(res_nb);
      res_t = warp_max(res_t);
      bad = __reduce_max_sync(0xffffffffu, bad);
      __syncwarp();
      if (lane < K) { W0[lane] = w0; W1[lane] = w1; }
      __syncwarp();
      ++l;
      if (bad) { err = bad; break; }
      if (res_nb < p.tol_nb && res_t < p.tol_tiny) break;
      if (l >= p.dts_max_iter) { err = ST_DTS_CAP; break; }
    }
  }
  if (!err && lane < K) {  // Part 2 (b): conservative update with F_left, F*, F_right
    double hn1 = hn + (we[lane + 1] - we[lane]) * dt;
    if (!(hn1 > 0.0)) err = ST_WIDTH;
    else {
      rho[a + lane] = (hn / hn1) * rn0 - (dt / hn1) * (Fe0[lane + 1] - Fe0[lane]);
      mom[a + lane] = (hn / hn1) * rn1 - (dt / hn1) * (Fe1[lane + 1] - Fe1[lane]);
      h[a + lane] = hn1;
      if (hn1 < p.eps_tiny * p.h_av || hn1 > p.eps_split * p.h_av) sh.remesh = 1;
    }
  }
  err = __reduce_max_sync(0xffffffffu, err);
  if (err && lane == 0) set_status(sh, err);
  it_out = l;
}

// ------------------------------------------------------------------------------------------
// The kernel.  Dynamic shared memory: CtaShared | 6 x (cap+1) doubles | (cap+1) flag bytes.
// Barrier discipline: sh.status is only READ between two barriers with no write in between
// (CHECK_STOP), so every thread takes the same branch.
// ------------------------------------------------------------------------------------------
#define EIS_CHECK_STOP()                 \
  {                                      \
    __syncthreads();                     \
    const int stop_ = sh.status;         \
    __syncthreads();                     \
    if (stop_) break;                    \
  }

__device__ __forceinline__ void or_flag(uint8_t* fl, int i, uint8_t bits) {
  atomicOr(reinterpret_cast<unsigned int*>(fl + (i & ~3)), (unsigned)bits << (8 * (i & 3)));
}

template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
resident_steps(const Eos e, const Prm p, Members g, long long n_steps, double t_end) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CtaShared& sh = *reinterpret_cast<CtaShared*>(smem_raw);
  const int C = (int)g.cap;
  double* arr = reinterpret_cast<double*>(smem_raw + ((sizeof(CtaShared) + 15) & ~size_t(15)));
  double* rho = arr;
  double* mom = arr + (C + 1);
  double* h = arr + 2 * (C + 1);
  double* U = arr + 3 * (C + 1);   // velocities (passes A-C) | DTS scratch (E) | remesh output (F)
  double* F0 = arr + 4 * (C + 1);  // edge fluxes (B-E) | remesh output (F)
  double* F1 = arr + 5 * (C + 1);
  uint8_t* fl = reinterpret_cast<uint8_t*>(arr + 6 * (C + 1));
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  const long long m = blockIdx.x;
  const long long base = m * g.cap;

  if (tid == 0) {
    sh.n = (int)g.n[m];
    sh.status = g.status[m];
  }
  __syncthreads();
  int n = sh.n;
  for (int i = tid; i < n; i += T) {
    rho[i] = g.rho[base + i];
    mom[i] = g.mom[base + i];
    h[i] = g.h[base + i];
  }
  double t = g.t[m];
  MemberStats st = g.stats[m];  // thread 0's copy is authoritative
  long long dts_acc = 0, solves_acc = 0, regions_acc = 0;

  for (long long step = 0; step < n_steps; ++step) {
    EIS_CHECK_STOP();
    if (!(t < t_end)) break;
    // ---------------- pass A: decode (a1), S_max, tiny (a8), h_min, dt (a2) ----------------
    if (tid == 0) { sh.nspec = 0; sh.nblk = 0; sh.remesh = 0; sh.c_merges = 0; sh.c_splits = 0; sh.c_creations = 0; }
    double smax = 0.0, hmin = INFINITY;
    for (int i = tid; i < n; i += T) {
      double r_ = rho[i], m_ = mom[i];
      int ph = phase_of(e, r_);
      if (!(r_ > 0.0)) set_status(sh, ST_NONPOS);
      else if (ph == SPIN) set_status(sh, ST_SPINODAL);
      double u = m_ / r_;
      U[i] = u;
      smax = fmax(smax, fabs(u) + sound(e, ph));  // S over all cells (R5)
      fl[i] = (uint8_t)ph;
    }
    if (tid == 0) fl[n] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += T) {
      int ph = fl[i] & F_PH;
      bool same_l = i > 0 && (fl[i - 1] & F_PH) == ph;
      bool same_r = i < n - 1 && (fl[i + 1] & F_PH) == ph;
      bool tiny = h[i] < p.eps_tiny * p.h_av && !same_l && !same_r;  // R4, R10
      if (tiny && p.mode == 0) {
        fl[i] |= F_TINY;
        if (i == 0 || i == n - 1) set_status(sh, ST_UNSUPPORTED);  // R26
      }
      if (p.mode == 1 || !tiny) hmin = fmin(hmin, h[i]);  // h_min over non-tiny cells (R6)
    }
    smax = warp_max(smax);
    hmin = warp_min(hmin);
    if (lane == 0) { sh.red[warp] = smax; sh.red[32 + warp] = hmin; }
    __syncthreads();
    if (tid == 0) {
      double s = 0.0, hm = INFINITY;
      for (int w = 0; w < nw; ++w) { s = fmax(s, sh.red[w]); hm = fmin(hm, sh.red[32 + w]); }
      double dt = p.cfl * hm / s;
      if (t + dt > t_end) dt = t_end - t;
      sh.dt = dt;
    }
    if (p.mode == 0) {  // implicit blocks: union of {k-1, k, k+1} (R11)
      for (int i = tid; i < n; i += T) {
        bool reg = (fl[i] & F_TINY) || (i > 0 && (fl[i - 1] & F_TINY)) || (i < n - 1 && (fl[i + 1] & F_TINY));
        if (reg) fl[i] |= F_REG;
      }
    }
    EIS_CHECK_STOP();
    const double dt = sh.dt;
    if (p.mode == 0) {
      for (int i = tid; i < n; i += T) {
        if ((fl[i] & F_REG) && (i == 0 || !(fl[i - 1] & F_REG))) {
          int k = atomicAdd(&sh.nblk, 1);
          if (k < MAXBLK) sh.blkA[k] = i; else set_status(sh, ST_CAPACITY);
        }
      }
    }
    // ---------------- pass B: edge fluxes from U^n (a3), creation trigger (a4) ----------------
    for (int ed = tid; ed <= n; ed += T) {
      int L = ed > 0 ? ed - 1 : 0, R = ed < n ? ed : n - 1;  // transmissive ghosts (R15)
      uint8_t fL = fl[L], fR = fl[R];
      if (ed > 0 && ed < n && (fL & F_REG) && (fR & F_REG)) continue;  // left to Algorithm 2
      int pL = fL & F_PH, pR = fR & F_PH;
      if (pL == pR) {
        double rl = rho[L], ml = mom[L], ul = U[L], rr = rho[R], mr = mom[R], ur = U[R];
        double f0, f1;
        hll(e, pL, rl, ml, ul, rr, mr, ur, f0, f1);
        F0[ed] = f0; F1[ed] = f1;
        if (ed > 0 && ed < n && !(fL & F_REG) && !(fR & F_REG) && creation_trigger(e, pL, rl, ul, rr, ur)) {
          int k = atomicAdd(&sh.nspec, 1);
          if (k < MAXSPEC) { sh.spec[k].e = ed; sh.spec[k].kind = 3; } else set_status(sh, ST_CAPACITY);
          or_flag(fl, ed, F_TRIG);
        }
      } else {
        int k = atomicAdd(&sh.nspec, 1);
        if (k < MAXSPEC) { sh.spec[k].e = ed; sh.spec[k].kind = 1; } else set_status(sh, ST_CAPACITY);
        or_flag(fl, ed, F_SPEC);
      }
    }
    EIS_CHECK_STOP();
    // ---------------- pass C: creation acceptance (R16), special-edge solves (a5, a6) ----------------
    const int nspec = sh.nspec;
    for (int k = tid; k < nspec; k += T) {
      if (sh.spec[k].kind != 3) continue;
      int ed = sh.spec[k].e, run = 0;  // leftmost wins: accepted iff an even number of
      while (ed - run - 1 >= 1 && (fl[ed - run - 1] & F_TRIG)) ++run;  // triggered edges precede it
      sh.spec[k].kind = (run & 1) ? 0 : 2;
    }
    __syncthreads();
    for (int k = tid; k < nspec; k += T)
      if (sh.spec[k].kind == 2) or_flag(fl, sh.spec[k].e, F_SPEC | F_CREATE);
    __syncthreads();
    {
      const int half = lane >> 4, hl = lane & 15;
      const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
      for (int k = warp * 2 + half; k < nspec; k += nw * 2) {
        Spec& sp = sh.spec[k];
        const int kind = sp.kind;
        if (kind != 1 && kind != 2) continue;
        const int ed = sp.e, L = ed - 1, R = ed;
        const double rl = rho[L], ul = U[L], rr = rho[R], ur = U[R];
        if (kind == 1) {
          IfaceSol s = iface_solve_hw(e, p, rl, ul, rr, ur, (fl[L] & F_PH) == VAP, -1.0, -1.0, hmask, hl, half * 16);
          if (hl == 0) {
            if (s.iters < 0) set_status(sh, ST_NEWTON);
            sp.Fl0 = sp.Fr0 = s.F0; sp.Fl1 = sp.Fr1 = s.F1; sp.wl = sp.wr = s.w;
            ++solves_acc;
          }
        } else {
          CreateSol s = create_solve_hw(e, p, fl[L] & F_PH, rl, ul, rr, ur, hmask, hl, half * 16);
          if (hl == 0) {
            if (s.iters < 0) set_status(sh, ST_CREATION);
            sp.Fl0 = s.Fl0; sp.Fl1 = s.Fl1; sp.wl = s.wl;
            sp.Fr0 = s.Fr0; sp.Fr1 = s.Fr1; sp.wr = s.wr;
            sp.rB = s.rB; sp.mB = s.mB;
            atomicAdd(&sh.c_creations, 1);
            sh.remesh = 1;
          }
        }
      }
    }
    EIS_CHECK_STOP();
    // ---------------- pass D: explicit moving-cell update (a7) ----------------
    for (int i = tid; i < n; i += T) {
      const uint8_t f = fl[i];
      if (f & F_REG) continue;
      double FL0 = F0[i], FL1 = F1[i], wL = 0.0, FR0 = F0[i + 1], FR1 = F1[i + 1], wR = 0.0;
      if (f & F_SPEC) {
        const Spec* s = find_spec(sh, i);
        if (s) { FL0 = s->Fr0; FL1 = s->Fr1; wL = s->wr; }
      }
      if (fl[i + 1] & F_SPEC) {
        const Spec* s = find_spec(sh, i + 1);
        if (s) { FR0 = s->Fl0; FR1 = s->Fl1; wR = s->wl; }
      }
      const double hn = h[i];
      const double hn1 = hn + (wR - wL) * dt;
      if (!(hn1 > 0.0)) { set_status(sh, ST_WIDTH); continue; }
      const double q = hn / hn1, c = dt / hn1;
      rho[i] = q * rho[i] - c * (FR0 - FL0);
      mom[i] = q * mom[i] - c * (FR1 - FL1);
      h[i] = hn1;
      if (hn1 < p.eps_tiny * p.h_av || hn1 > p.eps_split * p.h_av) sh.remesh = 1;
    }
    // ---------------- pass E: dual time stepping (a9), one warp per implicit block ----------------
    {
      const int nblk = sh.nblk < MAXBLK ? sh.nblk : MAXBLK;
      for (int k = warp; k < nblk; k += nw) {
        const int a = sh.blkA[k];
        int b = a;
        while (b + 1 < n && (fl[b + 1] & F_REG)) ++b;
        if (b - a + 1 > MAXB) { if (lane == 0) set_status(sh, ST_CAPACITY); continue; }
        long long it = 0, sv = 0;
        dts_block(e, p, sh, rho, mom, h, F0, F1, fl, U + warp * DTS_SCRATCH, a, b, dt, it, sv);
        if (lane == 0) { dts_acc += it; regions_acc += 1; }
        if ((lane & 15) == 0) solves_acc += sv;
      }
    }
    EIS_CHECK_STOP();
    // ---------------- pass F: remesh (a10; R9, R10), only when flagged ----------------
    int n_new = n;
    if (sh.remesh) {
      for (int i = tid; i < n; i += T) {  // post-update phases; keep the edge bits
        const int ph = phase_of(e, rho[i]);
        if (!(rho[i] > 0.0)) set_status(sh, ST_NONPOS);
        else if (ph == SPIN) set_status(sh, ST_SPINODAL);
        fl[i] = (uint8_t)((fl[i] & (F_SPEC | F_CREATE)) | ph);
      }
      if (tid == 0) fl[n] &= (F_SPEC | F_CREATE);
      __syncthreads();
      for (int i = tid; i < n; i += T) {  // merge partner: same-phase neighbour; both -> smaller, ties left
        uint8_t f = fl[i];
        if (h[i] < p.eps_tiny * p.h_av) {
          const int ph = f & F_PH;
          const bool sl = i > 0 && !(f & F_CREATE) && (fl[i - 1] & F_PH) == ph;
          const bool sr = i < n - 1 && !(fl[i + 1] & F_CREATE) && (fl[i + 1] & F_PH) == ph;
          int side = 0;
          if (sl && sr) side = (h[i + 1] < h[i - 1]) ? 2 : 1;
          else if (sl) side = 1;
          else if (sr) side = 2;
          if (side == 1) fl[i] = f | F_TINY;
          if (side == 2) fl[i] = f | F_REG;
        }
      }
      __syncthreads();
      for (int i = tid; i < n - 1; i += T)
        if ((fl[i] & F_REG) || (fl[i + 1] & F_TINY)) or_flag(fl, i, F_MERGE);
      __syncthreads();
      int carry = 0;
      for (int c0 = 0; c0 < n; c0 += T) {  // counts in cell order -> scan -> scatter into (U, F0, F1)
        const int i = c0 + tid;
        int cnt = 0;
        double gr = 0, gm = 0, gh = 0;
        bool head = false, split = false;
        if (i < n) {
          const uint8_t f = fl[i];
          if (f & F_CREATE) cnt += 1;
          head = !(i > 0 && (fl[i - 1] & F_MERGE));
          if (head) {
            if (!(f & F_MERGE)) { gr = rho[i]; gm = mom[i]; gh = h[i]; }
            else {  // merge group: h-weighted average summed left to right (R10)
              double hs = 0.0, s0 = 0.0, s1 = 0.0;
              int j = i, merged = 0;
              for (;;) {
                hs += h[j]; s0 += h[j] * rho[j]; s1 += h[j] * mom[j];
                if (!(fl[j] & F_MERGE)) break;
                ++j; ++merged;
              }
              gr = s0 / hs; gm = s1 / hs; gh = hs;
              atomicAdd(&sh.c_merges, merged);
            }
            split = gh > p.eps_split * p.h_av;
            cnt += split ? 2 : 1;
            if (split) atomicAdd(&sh.c_splits, 1);
          }
        }
        int tot = 0;
        int pos = block_excl_scan(sh, cnt, &tot) + carry;
        if (i < n) {
          if (fl[i] & F_CREATE) {
            const Spec* s = find_spec(sh, i);
            if (pos < C && s) { U[pos] = s->rB; F0[pos] = s->mB; F1[pos] = (s->wr - s->wl) * dt; }
            ++pos;
          }
          if (head) {
            if (split) {
              const double hh = 0.5 * gh;
              if (pos + 1 < C) { U[pos] = gr; F0[pos] = gm; F1[pos] = hh; U[pos + 1] = gr; F0[pos + 1] = gm; F1[pos + 1] = hh; }
            } else if (pos < C) { U[pos] = gr; F0[pos] = gm; F1[pos] = gh; }
          }
        }
        carry += tot;
      }
      if (tid == 0 && carry > C) set_status(sh, ST_CAPACITY);
      n_new = carry;
      double* t0 = rho; double* t1 = mom; double* t2 = h;  // (U, F0, F1) become the state
      rho = U; mom = F0; h = F1;
      U = t0; F0 = t1; F1 = t2;
    }
    __syncthreads();
    if (tid == 0) {
      st.steps += 1;
      st.cell_updates += n;
      st.creations += sh.c_creations;
      st.merges += sh.c_merges;
      st.splits += sh.c_splits;
      if (st.steps == 1 || dt < st.dt_min) st.dt_min = dt;
      if (dt > st.dt_max) st.dt_max = dt;
      sh.n = n_new;
    }
    n = n_new;
    t += dt;
  }
  // ---------------- write back (one HBM round trip per call) ----------------
  __syncthreads();
  n = sh.n;
  for (int i = tid; i < n; i += T) {
    g.rho[base + i] = rho[i];
    g.mom[base + i] = mom[i];
    g.h[base + i] = h[i];
  }
  for (int o = 16; o > 0; o >>= 1) {
    dts_acc += __shfl_xor_sync(0xffffffffu, dts_acc, o);
    solves_acc += __shfl_xor_sync(0xffffffffu, solves_acc, o);
    regions_acc += __shfl_xor_sync(0xffffffffu, regions_acc, o);
  }
  long long* red = reinterpret_cast<long long*>(sh.red);  // 64 slots
  __syncthreads();
  if (lane == 0) { red[warp] = dts_acc; red[32 + warp] = solves_acc; }
  __syncthreads();
  if (tid == 0) {
    long long da = 0, sa = 0;
    for (int w = 0; w < nw; ++w) { da += red[w]; sa += red[32 + w]; }
    st.dts_iters += da;
    st.iface_solves += sa;
  }
  __syncthreads();
  if (lane == 0) red[warp] = regions_acc;
  __syncthreads();
  if (tid == 0) {
    long long rr = 0;
    for (int w = 0; w < nw; ++w) rr += red[w];
    st.regions += rr;
    g.n[m] = n;
    g.t[m] = t;
    g.status[m] = sh.status;
    g.stats[m] = st;
  }
}

}  // namespace eis
