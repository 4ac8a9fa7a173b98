// eis_api.cu — the C ABI of libeis.so (include/eis.h): contexts, stream-ordered launches of
// the member-resident kernel, state transfer and reporting kernels.  Host code here only
// validates, allocates and launches; every step of the method runs in the kernels of
// eis_resident.cuh / eis_device.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "eis.h"
#include "eis_resident.cuh"
#include "eis_tiled.cuh"
#include "eis_lax.cuh"

#ifndef EIS_WIN_MINB
#define EIS_WIN_MINB 16  // one-warp window CTAs per SM (register budget 128)
#endif
#ifndef EIS_FAST_T
#define EIS_FAST_T 128  // tiled_fast threads per CTA (one CTA per tile)
#endif
#ifndef EIS_FAST_MINB
#define EIS_FAST_MINB 8  // tiled_fast CTAs of 128 threads per SM (register budget 64)
#endif

using namespace eis;

struct eis_ctx {
  long long tile_full_steps = 0, tile_win_steps = 0;
  // kernel timing (eis_set_timing): events around each step kernel, summed on request
  int timing = 0;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::array<int, 5>> ev_marks;  // per recorded launch group: event indices + kind
  std::vector<std::array<int, 6>> ev_spec;   // development (EIS_SPEC_TIMING): step start, early part A end, early dts_jobs end, late part A end, late dts end, part B end
  long long n_kernels = 0;                     // kernels launched by the step calls while timing is on
  size_t ev_used = 0;
  eis_eos eos_in;
  eis_params prm_in;
  eis_grid grid;
  Eos e;
  Prm p;
  cudaStream_t stream;
  int threads, minb;
  size_t smem;
  Members g;
  double *d_rho, *d_mom, *d_h, *d_t;
  long long* d_n;
  int* d_status;
  MemberStats* d_stats;
  uint8_t* d_u8;    // scratch: phases for get_state
  double* d_pack;   // scratch for packed host transfers (3 * M * cap)
  long long* d_cnt; // scratch: per-member interface counts / offsets
  eis_interface* d_if;
  long long if_cap;
  long long* d_ifoff = nullptr;  // per-member offsets of eis_interfaces (n_members entries)
  int state_set;
  // tiled layout (one huge grid, C5): tile buffers; d_rho/d_mom/d_h stay the contiguous staging
  int tiled, tile_cells;
  Tiles tl;
  double *t_rho[2], *t_mom[2], *t_h[2], *t_ws, *t_part, *t_scal;
  int *t_cnt[2], *t_hu[2], *t_ctl, *t_mctl = nullptr, *t_slow, *t_wlist;
  int *t_pred[2] = {nullptr, nullptr}, *t_plist[2] = {nullptr, nullptr}, *t_mlist = nullptr;  // window prediction (Tiles::spec)
  int win_grid_early = 0;                  //   CTAs of the early part A (beside tiled_fast)
  int fast_plain, fast_one;                // tiled_fast instantiations (EIS_FAST_PLAIN / EIS_FAST_ONE = 0: the general ones)
  long long* t_wdbg = nullptr;
  double *t_part2, *t_partf;
  int slow_grid, win_grid, win_grid_poll;
  double** d_xpeers = nullptr;  // peer mode: the ranks' exchange buffers (device array)
  int dts_grid = 0;                        // window split: dts_jobs CTAs (one warp each)
  int dts_tpb = 32;                        //   threads per dts_jobs CTA (EIS_DTS_TPB, development)
  DtsJob* t_djobs = nullptr;
  unsigned char* t_wsave = nullptr;
  cudaStream_t stream2 = nullptr;          // tiled: the window kernel beside tiled_fast
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  size_t smem_win;
  size_t smem_fast = 0;  // tiled_fast staging (EIS_FAST_TMA builds)
  TileStats* t_stats;
  long long* t_off;
  int staging_fresh;
  eis_status sticky;
  char msg[512];
};

static eis_status fail(eis_ctx* c, eis_status s, const char* fmt, const char* extra = "") {
  if (c) {
    snprintf(c->msg, sizeof(c->msg), fmt, extra);
    if (s == EIS_E_CUDA || s == EIS_E_ARG) c->sticky = s;
  }
  return s;
}

#define CU(call)                                                                       \
  do {                                                                                 \
    cudaError_t err_ = (call);                                                         \
    if (err_ != cudaSuccess) return fail(c, EIS_E_CUDA, "CUDA error: %s", cudaGetErrorString(err_)); \
  } while (0)

// ------------------------------------------------------------------------------------------
// Thresholds (R3), host side, once per context.  Maxwell equal area along the path liquid ->
// spinodal linear in rho -> vapour: Phi(rt) = a_l^2 ln(rho_min/rho0) + s ln(rt/rho_min)
// + a_v^2 ln(rho_V0/rt) with s = (a_v^2 rt - p_min)/(rt - rho_min).  Solved in x = ln(rt) by
// a sign-change search outward from rho_V0 followed by regula falsi (Illinois).
// ------------------------------------------------------------------------------------------
static double maxwell_phi(double x, double a_v2, double a_l2, double rho0, double p0, double p_min, double rho_min) {
  const double rt = std::exp(x);
  const double s = (a_v2 * rt - p_min) / (rt - rho_min);
  return a_l2 * std::log(rho_min / rho0) + s * std::log(rt / rho_min) + a_v2 * std::log((p0 / a_v2) / rt);
}

extern "C" eis_status eis_thresholds_of(const eis_eos* in, eis_thresholds* out) {
  if (!in || !out || !(in->a_v2 > 0) || !(in->a_l > 0) || !(in->rho0 > 0) || !(in->p0 > 0)) return EIS_E_ARG;
  const double a_l2 = in->a_l * in->a_l;
  const double rho_min = in->rho0 + (in->p_min - in->p0) / a_l2;
  if (!(rho_min > 0) || !(in->p_min < in->p0)) return EIS_E_ARG;
  double rt = in->rho_tilde;
  if (!(rt > 0)) {
    const double lo0 = std::log(in->p0 / in->a_v2), hi0 = std::log(rho_min);
    auto F = [&](double x) { return maxwell_phi(x, in->a_v2, a_l2, in->rho0, in->p0, in->p_min, rho_min); };
    // walk up from rho_V0 in growing steps until the sign changes
    double xa = lo0 + 1e-12, fa = F(xa), xb = xa, fb = fa, step = 1e-6;
    bool found = false;
    while (xb < hi0) {
      xb = std::fmin(xa + step, hi0 - 1e-12);
      fb = F(xb);
      if ((fa < 0) != (fb < 0)) { found = true; break; }
      xa = xb; fa = fb; step *= 1.5;
      if (xb >= hi0 - 1e-12) break;
    }
    if (!found) return EIS_E_ARG;
    int side = 0;
    for (int it = 0; it < 200; ++it) {
      double xc = (xa * fb - xb * fa) / (fb - fa);
      double fc = F(xc);
      if (fc == 0 || std::fabs(xb - xa) < 1e-15 * std::fabs(xb)) { xa = xb = xc; break; }
      if ((fc < 0) == (fb < 0)) { xb = xc; fb = fc; if (side == -1) fa *= 0.5; side = -1; }
      else { xa = xc; fa = fc; if (side == 1) fb *= 0.5; side = 1; }
    }
    rt = std::exp(0.5 * (xa + xb));
  }
  if (!(rt < rho_min)) return EIS_E_ARG;
  out->rho_min = rho_min;
  out->rho_tilde = rt;
  out->p_tilde = in->a_v2 * rt;
  out->tau = in->tau > 0 ? in->tau : 1.0 / std::sqrt(2.0 * M_PI) * std::pow(in->a_v2, -1.5);
  out->a_v = std::sqrt(in->a_v2);
  return EIS_OK;
}

// ------------------------------------------------------------------------------------------
// small kernels: state fill / validation / packing / reporting
// ------------------------------------------------------------------------------------------
__global__ void k_fill(double* a, long long count, double v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) a[i] = v;
}
__global__ void k_fill_ll(long long* a, long long count, long long v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) a[i] = v;
}
// one CTA per member: validate the initial state (rho > 0, not spinodal), reset counters
// member status from the initial state (status zeroed before): grid (members, chunks of a
// member's cells), so one huge grid is checked by many CTAs
constexpr int VALIDATE_CHUNK = 8192;
__global__ void k_validate(const Eos e, Members g, double t0) {
  __shared__ int bad;
  const long long m = blockIdx.x;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const long long n_in = g.n[m];
  const long long n = n_in < 0 ? 0 : (n_in > g.cap ? g.cap : n_in);  // never read past the member's row
  for (long long lo = (long long)blockIdx.y * VALIDATE_CHUNK; lo < n; lo += (long long)gridDim.y * VALIDATE_CHUNK) {
    const long long hi = min(n, lo + VALIDATE_CHUNK);
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      double r = g.rho[m * g.cap + i];
      if (!(r > 0.0)) atomicMax(&bad, ST_NONPOS);
      else if (phase_of(e, r) == SPIN) atomicMax(&bad, ST_SPINODAL);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int st = bad;
    if (blockIdx.y == 0) {
      if (n_in < 3 || n_in > g.cap) st = ST_CAPACITY;
      g.t[m] = t0;
      MemberStats z;
      memset(&z, 0, sizeof(z));
      g.stats[m] = z;
    }
    if (st) atomicMax(&g.status[m], st);
  }
}
// copy live cells, zero the rest, phases (255 past the end)
// grid (members, chunks of a member's cells) as k_validate, so one huge grid packs on many CTAs
__global__ void k_pack(const Eos e, Members g, double* rho, double* mom, double* h, uint8_t* ph) {
  const long long m = blockIdx.x;
  const long long n = g.n[m];
  for (long long i = (long long)blockIdx.y * blockDim.x + threadIdx.x; i < g.cap; i += (long long)gridDim.y * blockDim.x) {
    const long long k = m * g.cap + i;
    const bool live = i < n;
    const double r = live ? g.rho[k] : 0.0;
    if (rho) rho[k] = r;
    if (mom) mom[k] = live ? g.mom[k] : 0.0;
    if (h) h[k] = live ? g.h[k] : 0.0;
    if (ph) ph[k] = live ? (uint8_t)phase_of(e, r) : (uint8_t)255;
  }
}
// interfaces: one thread per member, widths summed left to right (fixed order, one add per cell)
__global__ void k_iface(const Eos e, Members g, long long M, double x_left, const long long* off,
                        long long* cnt, eis_interface* out, long long cap_out) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (m >= M) return;
  const long long n = g.n[m];
  const double* rho = g.rho + m * g.cap;
  const double* h = g.h + m * g.cap;
  long long k = off ? off[m] : 0, c = 0;
  double x = x_left;
  int pa = phase_of(e, rho[0]);
  for (long long i = 0; i < n; ++i) {
    x = __dadd_rn(x, h[i]);
    if (i + 1 < n) {
      const int pb = phase_of(e, rho[i + 1]);
      if (pa != pb) {
        if (out && k < cap_out) { out[k].member = m; out[k].edge = i + 1; out[k].x = x; out[k].left_phase = pa; out[k].right_phase = pb; }
        ++k; ++c;
      }
      pa = pb;
    }
  }
  if (cnt) cnt[m] = c;
}

// the phase-boundary Riemann problem of each reported boundary's two adjacent cells (App. A),
// one half warp per boundary, cold-started from the HLLC estimate
__global__ void k_iface_solve(const Eos e, const Prm p, Members g, eis_interface* out, long long total) {
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  const long long j = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 4;
  if (j >= total) return;  // a whole half warp: the solver's syncs stay within it
  const eis_interface b = out[j];
  const long long i = b.member * g.cap + b.edge;
  const double rl = g.rho[i - 1], ml = g.mom[i - 1], rr = g.rho[i], mr = g.mom[i];
  const bool vap_left = b.left_phase == VAP;
  const bool ok = (b.left_phase == VAP || b.left_phase == LIQ) && (b.right_phase == VAP || b.right_phase == LIQ);
  IfaceSol s;
  s.iters = -1;
  if (ok) s = iface_solve_hw(e, p, rl, ml / rl, rr, mr / rr, vap_left, -1.0, -1.0, hmask, hl, half * 16);
  if (hl == 0) {
    const bool conv = ok && s.iters >= 0;
    out[j].w = conv ? s.w : 0.0;
    out[j].z = conv ? -s.F0 : 0.0;  // F_PB = (-z, ...)
    out[j].p_vap = conv ? s.pV : 0.0;
    out[j].p_liq = conv ? s.pL : 0.0;
    out[j].solve_status = conv ? 0 : EIS_E_NEWTON;
    out[j].reserved = 0;
  }
}

// member-major staging -> tiles: tile k = member m's j-th tile (m = k / tpm) gets the member's
// cells [j tile, (j+1) tile), the last tile the remainder (fixed-size tiles: any tile-aligned
// split of a grid over ranks reproduces the single-grid tiling exactly).  A member whose cell
// count does not fit its tiles gets status ST_CAPACITY.
__global__ void k_to_tiles(Members g, Tiles tl, int cur, int tile_cells) {
  const int k = blockIdx.x, m = k / tl.tpm, j = k % tl.tpm;
  const long long n = g.n[m];
  const long long lo = (long long)j * tile_cells, hi = j == tl.tpm - 1 ? n : lo + tile_cells;
  const long long base = (long long)k * tl.capt, src = (long long)m * g.cap;
  const bool fits = hi - lo >= (tl.tpm > 1 ? HALO : 3) && hi - lo <= tl.capt;
  for (long long i = lo + threadIdx.x; fits && i < hi; i += blockDim.x) {
    tl.rho[cur][base + i - lo] = g.rho[src + i];
    tl.mom[cur][base + i - lo] = g.mom[src + i];
    tl.h[cur][base + i - lo] = g.h[src + i];
  }
  if (threadIdx.x == 0) {
    if (!fits) atomicCAS(&tl.mctl[MCS * m + 1], 0, (int)ST_CAPACITY);
    tl.cnt[cur][k] = fits ? (int)(hi - lo) : 0;
    tl.hu[cur][k] = 0;  // widths stored; the first step finds out whether they are all h_av
    double* ws = tl.ws + (size_t)k * WS_STRIDE;
    ws[2 * MAXIF] = -1.0;
    TileStats z;
    memset(&z, 0, sizeof(z));
    tl.tstats[k] = z;
  }
}
// tiles -> member-major staging, given each tile's offset inside its member (off[k]) and each
// member's cell count (off[ntiles + m])
__global__ void k_from_tiles(Members g, Tiles tl, const long long* off, double h_av) {
  const int k = blockIdx.x, m = k / tl.tpm;
  const int cur = tl.mctl[MCS * m];
  const int cnt = tl.cnt[cur][k];
  const bool hu = tl.hu[cur][k] != 0;
  const long long base = (long long)k * tl.capt, o = (long long)m * g.cap + off[k];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    g.rho[o + i] = tl.rho[cur][base + i];
    g.mom[o + i] = tl.mom[cur][base + i];
    g.h[o + i] = hu ? h_av : tl.h[cur][base + i];
  }
  if (k % tl.tpm == 0 && threadIdx.x == 0) {
    g.n[m] = off[tl.ntiles + m];
    g.t[m] = tl.scal[SCS * m];
    g.status[m] = tl.mctl[MCS * m + 1];
  }
}

static unsigned grid_for(long long count) {
  long long b = (count + 255) / 256;
  return (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b));
}

// ------------------------------------------------------------------------------------------
// tiled layout (one huge grid): allocation, staging <-> tiles
// ------------------------------------------------------------------------------------------
// the side stream of the window kernel that runs beside tiled_fast: highest priority, so its
// CTAs take the first SM slots tiled_fast frees (it is launched after tiled_fast, and only waits
// for work tiled_fast publishes: no kernel waits on a kernel launched after it)
static cudaError_t make_side_stream(cudaStream_t* s) {
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, hi);
}

static eis_status create_tiled(eis_ctx* c, eis_ctx** out) {
  const eis_grid* grid = &c->grid;
  const long long cap = grid->cell_capacity;
  c->tile_cells = grid->tile_cells > 0 ? grid->tile_cells : 1400;
  if (c->tile_cells < 4 * HALO || c->tile_cells > 8192) { delete c; return EIS_E_ARG; }
  const int capt = c->tile_cells + 32 + (c->tile_cells & 1);  // even: 16-byte aligned tile rows
  long long tpm = (grid->n_cells + c->tile_cells - 1) / c->tile_cells;  // tiles per member
  if (tpm > 1 && grid->n_cells - (tpm - 1) * c->tile_cells < HALO) --tpm;  // tiny remainder joins the last tile
  if (tpm < 1) tpm = 1;
  // ensembles with the default tile size: equal tiles per member (C4: 3 x 1366 instead of 1400,
  // 1400, 1296; +1 % measured), the tile count unchanged
  if (grid->n_members > 1 && grid->tile_cells <= 0 && tpm > 1) {
    const long long eq = ((grid->n_cells + tpm - 1) / tpm + 1) & ~1LL;
    if (eq >= 4 * HALO && eq <= c->tile_cells && (grid->n_cells + eq - 1) / eq == tpm && grid->n_cells - (tpm - 1) * eq >= HALO)
      c->tile_cells = (int)eq;
  }
  const long long M = grid->n_members, ntiles = M * tpm;
  if (ntiles > (1 << 30)) { delete c; return EIS_E_ARG; }
  if (M > 1 && (grid->nbr_left || grid->nbr_right)) { delete c; return EIS_E_ARG; }  // rank mode: one grid
  c->threads = grid->threads > 0 ? grid->threads : 256;
  if (c->threads != 256) { delete c; return EIS_E_ARG; }
  const int capg = capt + 2 * HALO + MAXEV + 1;  // as tiled_step
  c->smem = ((sizeof(CtaShared) + 15) & ~size_t(15)) + 6 * 8 * (size_t)(capg + 1) + (((size_t)capg + 1 + 15) & ~size_t(15));
  if (cudaSetDevice(grid->device) != cudaSuccess) { delete c; return EIS_E_CUDA; }
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, grid->device);
  if ((int)c->smem + 1024 > max_optin) { delete c; return EIS_E_CAPACITY; }
  if (cudaFuncSetAttribute(tiled_slow<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem) != cudaSuccess) {
    delete c; return EIS_E_CUDA;
  }
#if EIS_FAST_TMA
  c->smem_fast = 2 * sizeof(double) * (size_t)((capt + 1) & ~1);
  if (cudaFuncSetAttribute(tiled_fast<EIS_FAST_T, EIS_FAST_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)c->smem_fast) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)c->smem_fast) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_fast<EIS_FAST_T, EIS_FAST_MINB, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)c->smem_fast) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)c->smem_fast) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_fast<EIS_FAST_T, EIS_FAST_MINB, false, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)c->smem_fast) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)c->smem_fast) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_fast<EIS_FAST_T, EIS_FAST_MINB, false, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)c->smem_fast) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)c->smem_fast) != cudaSuccess) { delete c; return EIS_E_CUDA; }
#endif
  c->smem_win = ((sizeof(CtaShared) + 15) & ~size_t(15)) + 6 * 8 * (size_t)(WCAP + 1) + (((size_t)WCAP + 1 + 15) & ~size_t(15));
  if (cudaFuncSetAttribute(tiled_win<32, EIS_WIN_MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_win) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_win<32, EIS_WIN_MINB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_win) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_win<32, EIS_WIN_MINB, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_win) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_win<32, EIS_WIN_MINB, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_win) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_win<32, EIS_WIN_MINB, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_win) != cudaSuccess ||
      cudaFuncSetAttribute(tiled_win<32, EIS_WIN_MINB, false, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_win) != cudaSuccess) {
    delete c; return EIS_E_CUDA;
  }
  {  // load every tiled kernel now (CUDA lazy loading would load one at its first launch)
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, tiled_fast<EIS_FAST_T, EIS_FAST_MINB>) != cudaSuccess || cudaFuncGetAttributes(&fa, tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true>) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, tiled_fast<EIS_FAST_T, EIS_FAST_MINB, false, true>) != cudaSuccess || cudaFuncGetAttributes(&fa, tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true, true>) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, tiled_fast<EIS_FAST_T, EIS_FAST_MINB, false, true, 1>) != cudaSuccess || cudaFuncGetAttributes(&fa, tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true, true, 1>) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, tiled_fast<EIS_FAST_T, EIS_FAST_MINB, false, true, 2>) != cudaSuccess || cudaFuncGetAttributes(&fa, tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true, true, 2>) != cudaSuccess || cudaFuncGetAttributes(&fa, tiled_win<32, EIS_WIN_MINB, true>) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, tiled_win<32, EIS_WIN_MINB, false>) != cudaSuccess || cudaFuncGetAttributes(&fa, tiled_slow<256, 4>) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, tiled_win<32, EIS_WIN_MINB, false, 1>) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, tiled_win<32, EIS_WIN_MINB, false, 1, 1>) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, tiled_win<32, EIS_WIN_MINB, false, 2>) != cudaSuccess || cudaFuncGetAttributes(&fa, dts_jobs) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, tiled_finish) != cudaSuccess || cudaFuncGetAttributes(&fa, tiled_init_dt<256>) != cudaSuccess) {
      delete c; return EIS_E_CUDA;
    }
  }
  int nsm = 0, per_sm = 0, per_sm_w = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, grid->device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tiled_slow<256, 4>, 256, c->smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_w, tiled_win<32, EIS_WIN_MINB, false>, 32, c->smem_win);
  c->slow_grid = (int)std::min<long long>(ntiles, (long long)std::max(nsm, 1) * std::max(per_sm, 1));
  c->win_grid = (int)std::min<long long>(ntiles, (long long)std::max(nsm, 1) * std::max(per_sm_w, 1));
  // the polling instance beside tiled_fast: off by default (measured on C5: 1, 2, 4 CTAs/SM
  // beside tiled_fast cost tiled_fast more than the overlap saves); EIS_WIN_POLL_PER_SM=k
  c->win_grid_poll = 0;
  if (const char* ev = getenv("EIS_WIN_POLL_PER_SM")) c->win_grid_poll = std::max(0, atoi(ev)) * std::max(1, nsm);
  // window split (dual time stepping only; EIS_WIN_SPLIT=0: every window step in one kernel)
  int split = c->p.mode == 0;  // (with a polling instance: part A polls beside tiled_fast)
  if (const char* ev = getenv("EIS_WIN_SPLIT")) split = split && atoi(ev) != 0;
  c->dts_grid = std::max(nsm, 1) * 16;
  c->dts_tpb = 32;
  if (const char* ev = getenv("EIS_DTS_TPB")) c->dts_tpb = std::max(1, std::min(32, atoi(ev)));
  const size_t tc = (size_t)ntiles * capt;
  const size_t mc = (size_t)M * cap;  // member-major staging
  bool ok = cudaMalloc(&c->d_rho, mc * 8) == cudaSuccess && cudaMalloc(&c->d_mom, mc * 8) == cudaSuccess &&
            cudaMalloc(&c->d_h, mc * 8) == cudaSuccess && cudaMalloc(&c->d_t, M * 8) == cudaSuccess &&
            cudaMalloc(&c->d_n, M * 8) == cudaSuccess && cudaMalloc(&c->d_status, M * 4) == cudaSuccess &&
            cudaMalloc(&c->d_stats, M * sizeof(MemberStats)) == cudaSuccess && cudaMalloc(&c->d_cnt, M * 8 + 8) == cudaSuccess;
  for (int b = 0; b < 2 && ok; ++b)
    ok = cudaMalloc(&c->t_rho[b], tc * 8) == cudaSuccess && cudaMalloc(&c->t_mom[b], tc * 8) == cudaSuccess &&
         cudaMalloc(&c->t_h[b], tc * 8) == cudaSuccess && cudaMalloc(&c->t_cnt[b], ntiles * 4) == cudaSuccess &&
         cudaMalloc(&c->t_hu[b], ntiles * 4) == cudaSuccess;
  ok = ok && cudaMalloc(&c->t_ws, (size_t)ntiles * WS_STRIDE * 8) == cudaSuccess &&
       cudaMalloc(&c->t_part, (size_t)ntiles * 16) == cudaSuccess &&
       cudaMalloc(&c->t_stats, (size_t)ntiles * sizeof(TileStats)) == cudaSuccess &&
       cudaMalloc(&c->t_scal, (size_t)M * SCS * 8) == cudaSuccess && cudaMalloc(&c->t_ctl, NCTL * 4) == cudaSuccess &&
       cudaMalloc(&c->t_mctl, (size_t)M * MCS * 4) == cudaSuccess &&
       cudaMalloc(&c->t_slow, (size_t)ntiles * 4) == cudaSuccess &&
       cudaMalloc(&c->t_wlist, (size_t)ntiles * 16) == cudaSuccess &&
       make_side_stream(&c->stream2) == cudaSuccess &&
       cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
       cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) == cudaSuccess &&
       cudaMalloc(&c->t_partf, (size_t)ntiles * 24) == cudaSuccess &&
       cudaMalloc(&c->t_part2, (size_t)c->slow_grid * 16) == cudaSuccess &&
       cudaMalloc(&c->t_off, (ntiles + M) * 8) == cudaSuccess;
  const long long djcap = 4 * ntiles;  // DTS jobs per step (windows hold one block, rarely more)
  // window prediction (window split, one rank, no polling instance; EIS_WIN_SPEC=0: off): part A
  // and the DTS jobs of the predicted windows run beside tiled_fast on the side stream
  const int spec_ok = split && c->win_grid_poll == 0 && !grid->nbr_left && !grid->nbr_right;
  int spec = spec_ok && M > 1;  // default: ensembles (C4 +15 %); one grid (C5): +4 % at 20 steps, see DESIGN 6.2
  if (const char* ev = getenv("EIS_WIN_SPEC")) spec = spec_ok && atoi(ev) != 0;
  c->win_grid_early = std::max(nsm, 1) * (M > 1 ? 8 : 16);  // (C5: 16 per SM 1.35 ms/step, 8: 1.46, 4: 1.55; C4: 8 0.591, 16 0.597)
  if (const char* ev = getenv("EIS_WIN_EARLY_PER_SM")) c->win_grid_early = std::max(1, atoi(ev)) * std::max(1, nsm);
  c->win_grid_early = (int)std::min<long long>(ntiles, c->win_grid_early);
  c->fast_plain = 1; c->fast_one = 1;  // (eis_create zero-fills the context: defaults are set here)
  if (const char* ev = getenv("EIS_FAST_PLAIN")) c->fast_plain = atoi(ev) != 0;
  if (const char* ev = getenv("EIS_FAST_ONE")) c->fast_one = atoi(ev) != 0;
  if (ok && split)
    ok = cudaMalloc(&c->t_djobs, (size_t)djcap * sizeof(DtsJob)) == cudaSuccess &&
         cudaMalloc(&c->t_wsave, (size_t)ntiles * WSAVE * (spec ? 2 : 1)) == cudaSuccess;
  if (ok && spec) ok = cudaMalloc(&c->t_mlist, (size_t)ntiles * 4) == cudaSuccess;
  for (int b = 0; b < 2 && ok && spec; ++b)
    ok = cudaMalloc(&c->t_pred[b], (size_t)ntiles * 16) == cudaSuccess && cudaMalloc(&c->t_plist[b], (size_t)ntiles * 4) == cudaSuccess;
  if (!ok || cudaMemset(c->t_ctl, 0, NCTL * 4) != cudaSuccess) { eis_destroy(c); return EIS_E_CUDA; }
  c->g.rho = c->d_rho; c->g.mom = c->d_mom; c->g.h = c->d_h; c->g.n = c->d_n; c->g.t = c->d_t;
  c->g.status = c->d_status; c->g.stats = c->d_stats; c->g.cap = cap;
  c->g.dbg = nullptr;
  Tiles& tl = c->tl;
  for (int b = 0; b < 2; ++b) { tl.rho[b] = c->t_rho[b]; tl.mom[b] = c->t_mom[b]; tl.h[b] = c->t_h[b]; tl.cnt[b] = c->t_cnt[b]; tl.hu[b] = c->t_hu[b]; }
  tl.slow = c->t_slow; tl.part2 = c->t_part2; tl.wlist = c->t_wlist; tl.partf = c->t_partf;
  tl.wdbg = nullptr;
  if (getenv("EIS_WINDOW_DEBUG")) {
    if (cudaMalloc(&c->t_wdbg, (size_t)ntiles * WDBG_FIELDS * 8) != cudaSuccess ||
        cudaMemset(c->t_wdbg, 0, (size_t)ntiles * WDBG_FIELDS * 8) != cudaSuccess) { eis_destroy(c); return EIS_E_CUDA; }
    tl.wdbg = c->t_wdbg;
  }
  tl.poll = c->win_grid_poll > 0 ? 1 : 0;
  tl.split = split; tl.djcap = split ? (int)djcap : 0; tl.djobs = c->t_djobs; tl.wsave = c->t_wsave;
  tl.spec = spec;
  for (int b = 0; b < 2; ++b) { tl.pred[b] = c->t_pred[b]; tl.plist[b] = c->t_plist[b]; }
  tl.mlist = c->t_mlist;
  tl.wmax = WMAX;  // EIS_TILED_WMAX: a smaller bound (0: every special tile takes the whole-tile step)
  if (const char* ev = getenv("EIS_TILED_WMAX")) tl.wmax = std::max(0, std::min(WMAX, atoi(ev)));
  tl.ws = c->t_ws; tl.part = c->t_part; tl.tstats = c->t_stats; tl.scal = c->t_scal; tl.ctl = c->t_ctl;
  tl.mctl = c->t_mctl;
  tl.ntiles = (int)ntiles; tl.capt = capt; tl.M = (int)M; tl.tpm = (int)tpm;
  tl.xbuf = nullptr;
  tl.xpeer_l = nullptr; tl.xpeer_r = nullptr; tl.xpeers = nullptr; tl.xrank = 0; tl.xworld = 1;
  tl.nbr_left = grid->nbr_left != 0; tl.nbr_right = grid->nbr_right != 0;
  *out = c;
  return EIS_OK;
}

__global__ void k_tiles_reset(Tiles tl, const int* status, double t0) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m == 0) for (int q = 0; q < NCTL; ++q) if (q != 12) tl.ctl[q] = 0;  // [12]: peer-mode publications,
                                                                        // counted over the context's life
  if (m >= tl.M) return;
  if (status[m]) atomicCAS(&tl.ctl[1], 0, status[m]);
  int* mc = tl.mctl + MCS * m;
  mc[0] = 0; mc[1] = status[m]; mc[2] = 0; mc[3] = 0;
  double* sc = tl.scal + SCS * m;
  sc[0] = t0;
  for (int q = 1; q < SCS; ++q) sc[q] = 0.0;
}

// tiles -> contiguous staging (member 0), when the staging copy is stale
static eis_status tiles_to_staging(eis_ctx* c) {
  if (c->staging_fresh) return EIS_OK;
  const int nt = c->tl.ntiles, M = c->tl.M, tpm = c->tl.tpm;
  std::vector<int> mctl((size_t)M * MCS);
  CU(cudaMemcpyAsync(mctl.data(), c->t_mctl, (size_t)M * MCS * 4, cudaMemcpyDeviceToHost, c->stream));
  std::vector<int> cnt0(nt), cnt1(nt);
  CU(cudaMemcpyAsync(cnt0.data(), c->t_cnt[0], nt * 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(cnt1.data(), c->t_cnt[1], nt * 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  std::vector<long long> off((size_t)nt + M);  // tile offset inside its member, then member sizes
  for (int m = 0; m < M; ++m) {
    const std::vector<int>& cnt = mctl[(size_t)MCS * m] ? cnt1 : cnt0;
    long long o = 0;
    for (int j = 0; j < tpm; ++j) { off[(size_t)m * tpm + j] = o; o += cnt[(size_t)m * tpm + j]; }
    if (o > c->grid.cell_capacity) return fail(c, EIS_E_CAPACITY, "tiled grid exceeds cell_capacity%s");
    off[(size_t)nt + m] = o;
  }
  CU(cudaMemcpyAsync(c->t_off, off.data(), ((size_t)nt + M) * 8, cudaMemcpyHostToDevice, c->stream));
  k_from_tiles<<<nt, 256, 0, c->stream>>>(c->g, c->tl, c->t_off, c->p.h_av);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(c->stream));
  c->staging_fresh = 1;
  return EIS_OK;
}

static eis_status tiled_stats(eis_ctx* c, eis_stats* out) {
  const int nt = c->tl.ntiles, M = c->tl.M;
  std::vector<TileStats> ts(nt);
  std::vector<double> scal((size_t)M * SCS);
  std::vector<int> mctl((size_t)M * MCS);
  CU(cudaMemcpyAsync(ts.data(), c->t_stats, nt * sizeof(TileStats), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(scal.data(), c->t_scal, (size_t)M * SCS * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(mctl.data(), c->t_mctl, (size_t)M * MCS * 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  memset(out, 0, sizeof(*out));
  long long full = 0, win = 0;
  for (const TileStats& s : ts) {
    out->cell_updates += s.cell_updates; out->dts_iters += s.dts_iters; out->iface_solves += s.iface_solves;
    out->creations += s.creations; out->splits += s.splits; out->merges += s.merges; out->regions += s.regions;
    out->dts_iter_max = std::max(out->dts_iter_max, (int64_t)s.dts_max);
    out->decision_margin_warnings += s.margins;
    full += s.full_steps;
    win += s.win_steps;
  }
  c->tile_full_steps = full;
  c->tile_win_steps = win;
  out->t_min = INFINITY; out->t_max = -INFINITY; out->dt_min = INFINITY; out->dt_max = 0.0;
  for (int m = 0; m < M; ++m) {
    const double* sc = &scal[(size_t)SCS * m];
    const int steps = mctl[(size_t)MCS * m + 2];
    out->steps += steps;
    out->t_min = std::fmin(out->t_min, sc[0]); out->t_max = std::fmax(out->t_max, sc[0]);
    if (steps) { out->dt_min = std::fmin(out->dt_min, sc[2]); out->dt_max = std::fmax(out->dt_max, sc[3]); }
  }
  if (!(out->dt_min < INFINITY)) out->dt_min = 0.0;
  return EIS_OK;
}

// per member (tiled): its tiles' counters, its steps, t, dt range
static eis_status tiled_member_stats(eis_ctx* c, eis_stats* out) {
  const int nt = c->tl.ntiles, M = c->tl.M, tpm = c->tl.tpm;
  std::vector<TileStats> ts(nt);
  std::vector<double> scal((size_t)M * SCS);
  std::vector<int> mctl((size_t)M * MCS);
  CU(cudaMemcpyAsync(ts.data(), c->t_stats, nt * sizeof(TileStats), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(scal.data(), c->t_scal, (size_t)M * SCS * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(mctl.data(), c->t_mctl, (size_t)M * MCS * 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (int m = 0; m < M; ++m) {
    eis_stats& o = out[m];
    memset(&o, 0, sizeof(o));
    for (int j = 0; j < tpm; ++j) {
      const TileStats& s = ts[(size_t)m * tpm + j];
      o.cell_updates += s.cell_updates; o.dts_iters += s.dts_iters; o.iface_solves += s.iface_solves;
      o.creations += s.creations; o.splits += s.splits; o.merges += s.merges; o.regions += s.regions;
      o.dts_iter_max = std::max(o.dts_iter_max, (int64_t)s.dts_max);
      o.decision_margin_warnings += s.margins;
    }
    const double* sc = &scal[(size_t)SCS * m];
    o.steps = mctl[(size_t)MCS * m + 2];
    o.t_min = o.t_max = sc[0];
    o.dt_min = sc[2]; o.dt_max = sc[3];
  }
  return EIS_OK;
}

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
extern "C" eis_status eis_create(const eis_eos* eos, const eis_params* prm, const eis_grid* grid, eis_ctx** out) {
  if (!out) return EIS_E_ARG;
  *out = nullptr;
  if (!eos || !prm || !grid) return EIS_E_ARG;
  if (grid->n_members < 1 || grid->n_cells < 3 || grid->cell_capacity < grid->n_cells || !(grid->x_right > grid->x_left))
    return EIS_E_ARG;
  if (!(prm->cfl > 0) || !(prm->eps_tiny > 0) || !(prm->eps_split > prm->eps_tiny) || !(prm->theta_nb > 0) ||
      prm->newton_max_iter < 1 || prm->armijo_max < 0 || prm->armijo_max > 31 || prm->dts_max_iter < 1 ||
      (prm->mode != EIS_MODE_SPLIT && prm->mode != EIS_MODE_EXPLICIT && prm->mode != EIS_MODE_LTS &&
       prm->mode != EIS_MODE_NEWTON))
    return EIS_E_ARG;
  eis_thresholds th;
  if (eis_thresholds_of(eos, &th) != EIS_OK) return EIS_E_ARG;
  eis_ctx* c = new eis_ctx();
  memset(c, 0, sizeof(*c));
  c->eos_in = *eos;
  c->prm_in = *prm;
  c->grid = *grid;
  c->stream = (cudaStream_t)grid->stream;
  Eos& e = c->e;
  e.a_v2 = eos->a_v2; e.a_v = th.a_v; e.a_l = eos->a_l; e.a_l2 = eos->a_l * eos->a_l; e.rho0 = eos->rho0;
  e.p0 = eos->p0; e.tau = th.tau; e.rho_min = th.rho_min; e.rho_tilde = th.rho_tilde;
  e.inv_av2 = 1.0 / e.a_v2; e.inv_al2 = 1.0 / e.a_l2; e.inv_p0 = 1.0 / e.p0; e.inv_av = 1.0 / e.a_v; e.inv_rho0 = 1.0 / e.rho0;
  Prm& p = c->p;
  p.cfl = prm->cfl; p.eps_split = prm->eps_split; p.eps_tiny = prm->eps_tiny; p.theta_nb = prm->theta_nb;
  p.tol_nb = prm->tol_nb; p.tol_tiny = prm->tol_tiny; p.newton_rtol = prm->newton_rtol; p.newton_gtol = prm->newton_gtol;
  p.newton_stol = std::sqrt(prm->newton_rtol);
  p.lin_gtol = std::sqrt(prm->newton_gtol);  // R14d: the quadratic regime starts below sqrt(gtol)
  if (const char* ev = getenv("EIS_NEWTON_STOL")) p.newton_stol = atof(ev);  // development knobs
  if (const char* ev = getenv("EIS_LIN_GTOL")) p.lin_gtol = atof(ev);
  p.h_av = grid->h_av > 0 ? grid->h_av : (grid->x_right - grid->x_left) / (double)grid->n_cells;  // fixed (R9)
  p.dts_max_iter = prm->dts_max_iter; p.newton_max_iter = prm->newton_max_iter; p.armijo_max = prm->armijo_max;
  p.mode = prm->mode;

  const long long M = grid->n_members, cap = grid->cell_capacity;
  // AUTO: members of more than 2048 cells (C4, C5) stream through the tiled layout (measured:
  // C4 1.8x the member-resident kernel, whose CTA then fills an SM alone); smaller members
  // (C1-C3) stay resident in shared memory for the whole call
  c->tiled = grid->layout == EIS_LAYOUT_TILED || (grid->layout == EIS_LAYOUT_AUTO && cap > 2048);
  if (grid->layout < 0 || grid->layout > 2) { delete c; return EIS_E_ARG; }
  if (c->tiled) return create_tiled(c, out);
  if (cap > 16384) { delete c; return EIS_E_ARG; }
  // CTA size: 128 threads (3 bulk warps + the solver warp, 128 registers per thread) up to
  // 2048 cells; larger members 512 threads (128 registers: the solver code does not spill;
  // measured on C4 against 256 and 1024 threads)
  int T = grid->threads;
  if (T <= 0) {
    T = cap <= 2048 ? 128 : 512;
    if (grid->n_cells < 128) T = 64;
  }
  if (T % 32 || T < 64 || T > 1024) { delete c; return EIS_E_ARG; }  // >= 1 bulk warp + the solver warp
  c->threads = T;
  c->smem = ((sizeof(CtaShared) + 15) & ~size_t(15)) + 6 * 8 * (size_t)(cap + 1) + (((size_t)cap + 1 + 15) & ~size_t(15));
  int dev = grid->device;
  if (cudaSetDevice(dev) != cudaSuccess) { delete c; return EIS_E_CUDA; }
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if ((int)c->smem > max_optin) { delete c; return EIS_E_CAPACITY; }
  // tuning knob (development): CTAs per SM the 256-thread variant is compiled for (2 or 4)
  c->minb = 4;
  if (const char* ev = getenv("EIS_RESIDENT_MINB")) { int v = atoi(ev); if (v == 2 || v == 4) c->minb = v; }
  cudaError_t e1 = cudaFuncSetAttribute(resident_steps<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem);
  cudaError_t e3 = cudaFuncSetAttribute(resident_steps<512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem);
  cudaError_t e4 = cudaFuncSetAttribute(resident_steps<256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem);
  cudaError_t e2 = cudaFuncSetAttribute(resident_steps<1024, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem);
  cudaError_t e5 = cudaFuncSetAttribute(resident_steps<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem);
  if (e5 != cudaSuccess) { delete c; return EIS_E_CUDA; }
  if (cudaFuncSetAttribute(resident_steps<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem) != cudaSuccess) {
    delete c; return EIS_E_CUDA;
  }
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess) { delete c; return EIS_E_CUDA; }
  const size_t cells = (size_t)M * cap;
  bool ok = cudaMalloc(&c->d_rho, cells * 8) == cudaSuccess && cudaMalloc(&c->d_mom, cells * 8) == cudaSuccess &&
            cudaMalloc(&c->d_h, cells * 8) == cudaSuccess && cudaMalloc(&c->d_t, M * 8) == cudaSuccess &&
            cudaMalloc(&c->d_n, M * 8) == cudaSuccess && cudaMalloc(&c->d_status, M * 4) == cudaSuccess &&
            cudaMalloc(&c->d_stats, M * sizeof(MemberStats)) == cudaSuccess &&
            cudaMalloc(&c->d_cnt, (M + 1) * 8) == cudaSuccess;
  if (!ok) { eis_destroy(c); return EIS_E_CUDA; }
  c->g.rho = c->d_rho; c->g.mom = c->d_mom; c->g.h = c->d_h; c->g.n = c->d_n; c->g.t = c->d_t;
  c->g.dbg = nullptr;
#ifdef EIS_PHASE_CLOCK
  if (cudaMalloc(&c->g.dbg, (size_t)M * 64) != cudaSuccess || cudaMemset(c->g.dbg, 0, (size_t)M * 64) != cudaSuccess) {
    eis_destroy(c); return EIS_E_CUDA;
  }
#endif
  c->g.status = c->d_status; c->g.stats = c->d_stats; c->g.cap = cap;
  *out = c;
  return EIS_OK;
}

extern "C" void eis_destroy(eis_ctx* c) {
  if (!c) return;
  cudaFree(c->d_rho); cudaFree(c->d_mom); cudaFree(c->d_h); cudaFree(c->d_t); cudaFree(c->d_n);
  cudaFree(c->d_status); cudaFree(c->d_stats); cudaFree(c->d_u8); cudaFree(c->d_pack); cudaFree(c->d_cnt);
  cudaFree(c->d_if);
  cudaFree(c->d_ifoff);
  if (!c->tiled) cudaFree(c->g.dbg);
  for (int b = 0; b < 2; ++b) { cudaFree(c->t_rho[b]); cudaFree(c->t_mom[b]); cudaFree(c->t_h[b]); cudaFree(c->t_cnt[b]); cudaFree(c->t_hu[b]); }
  cudaFree(c->t_slow); cudaFree(c->t_part2); cudaFree(c->t_wlist); cudaFree(c->t_wdbg); cudaFree(c->t_partf);
  cudaFree(c->t_djobs); cudaFree(c->t_wsave);
  for (int b = 0; b < 2; ++b) { cudaFree(c->t_pred[b]); cudaFree(c->t_plist[b]); }
  cudaFree(c->t_mlist);
  cudaFree(c->d_xpeers);
  cudaFree(c->t_ws); cudaFree(c->t_part); cudaFree(c->t_stats); cudaFree(c->t_scal); cudaFree(c->t_ctl); cudaFree(c->t_mctl); cudaFree(c->t_off);
  for (cudaEvent_t ev : c->ev_pool) cudaEventDestroy(ev);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  delete c;
}

extern "C" eis_status eis_set_timing(eis_ctx* c, int32_t enable) {
  if (!c) return EIS_E_ARG;
  c->timing = enable != 0;
  c->ev_marks.clear();
  c->ev_spec.clear();
  c->ev_used = 0;
  c->n_kernels = 0;
  return EIS_OK;
}

extern "C" eis_status eis_get_timing(eis_ctx* c, double* ms, int64_t* launches) {
  if (!c || !ms || !launches) return EIS_E_ARG;
  CU(cudaStreamSynchronize(c->stream));
  for (int q = 0; q < 4; ++q) ms[q] = 0.0;
  *launches = (int64_t)c->n_kernels;
  if (!c->ev_spec.empty()) {  // development: mean offsets from the step start (ms)
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (const auto& sm : c->ev_spec)
      for (int q = 1; q < 6; ++q) {
        float t = 0.f;
        if (sm[q] >= 0 && cudaEventElapsedTime(&t, c->ev_pool[sm[0]], c->ev_pool[sm[q]]) == cudaSuccess) acc[q] += t;
      }
    const double n = (double)c->ev_spec.size();
    fprintf(stderr, "EIS_SPEC_TIMING (ms from the step start, mean of %d steps): early A end %.4f  early dts end %.4f  late A end %.4f  late dts end %.4f  part B end %.4f\n",
            (int)n, acc[1] / n, acc[2] / n, acc[3] / n, acc[4] / n, acc[5] / n);
  }
  for (const auto& m : c->ev_marks) {
    float t = 0.f;
    if (m[4] == 0) {  // resident: one kernel
      CU(cudaEventElapsedTime(&t, c->ev_pool[m[0]], c->ev_pool[m[1]]));
      ms[3] += t;
      continue;
    }
    for (int q = 0; q < 3; ++q) {
      CU(cudaEventElapsedTime(&t, c->ev_pool[m[q]], c->ev_pool[m[q + 1]]));
      ms[q] += t;
    }
  }
  return EIS_OK;
}

extern "C" eis_status eis_window_diag(eis_ctx* c, int64_t* out, int64_t capacity, int64_t* count) {
  if (!c || !count) return EIS_E_ARG;
  if (!c->tiled || !c->t_wdbg) return fail(c, EIS_E_ARG, "eis_window_diag: tiled context created with EIS_WINDOW_DEBUG set%s");
  int ctl[9];
  CU(cudaMemcpyAsync(ctl, c->t_ctl, sizeof(ctl), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  *count = ctl[8];
  if (out && capacity > 0) {
    const long long n = std::min<long long>(capacity, ctl[8]);
    CU(cudaMemcpyAsync(out, c->t_wdbg, (size_t)n * WDBG_FIELDS * 8, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  return EIS_OK;
}

extern "C" eis_status eis_window_prediction(eis_ctx* c, int64_t* windows, int64_t* predicted, int32_t* enabled) {
  if (!c || !windows || !predicted || !enabled) return EIS_E_ARG;
  if (!c->tiled) return fail(c, EIS_E_ARG, "eis_window_prediction: not a tiled context%s");
  int ctl[NCTL];
  CU(cudaMemcpyAsync(ctl, c->t_ctl, sizeof(ctl), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  *windows = ctl[19]; *predicted = ctl[18]; *enabled = c->tl.spec;
  return EIS_OK;
}

extern "C" eis_status eis_tile_info(eis_ctx* c, int64_t* n_tiles, int64_t* full_tile_steps, int64_t* window_steps) {
  if (!c || !n_tiles || !full_tile_steps || !window_steps) return EIS_E_ARG;
  if (!c->tiled) return fail(c, EIS_E_ARG, "eis_tile_info: not a tiled context%s");
  eis_stats st;
  const eis_status s = tiled_stats(c, &st);
  if (s) return s;
  *n_tiles = c->tl.ntiles;
  *full_tile_steps = c->tile_full_steps;
  *window_steps = c->tile_win_steps;
  return EIS_OK;
}

extern "C" const char* eis_last_error(const eis_ctx* c) { return c ? c->msg : "null context"; }

static eis_status ensure_pack(eis_ctx* c) {
  if (!c->d_pack) {
    const size_t cells = (size_t)c->grid.n_members * c->grid.cell_capacity;
    CU(cudaMalloc(&c->d_pack, cells * 3 * 8));
    CU(cudaMalloc(&c->d_u8, cells));
  }
  return EIS_OK;
}

extern "C" eis_status eis_set_state(eis_ctx* c, const double* rho, const double* mom, const double* width,
                                    const int64_t* n_cells, int32_t where, double t0) {
  if (!c) return EIS_E_ARG;
  if (!rho || !mom || (where != EIS_HOST && where != EIS_DEVICE)) return fail(c, EIS_E_ARG, "set_state: bad argument%s");
  CU(cudaSetDevice(c->grid.device));
  const long long M = c->grid.n_members, cap = c->grid.cell_capacity;
  size_t bytes = (size_t)M * cap * 8;
  const cudaMemcpyKind kind = where == EIS_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  // every host-side argument check before the first copy is queued (the caller's buffers are
  // then never read after an error return)
  if (n_cells && where == EIS_HOST)
    for (long long m = 0; m < M; ++m)
      if (n_cells[m] < 3 || n_cells[m] > cap) return fail(c, EIS_E_ARG, "set_state: n_cells out of range%s");
  if (c->tiled) {
    if ((c->tl.nbr_left || c->tl.nbr_right) && !c->tl.xbuf)
      return fail(c, EIS_E_ORDER, "rank mode: eis_set_exchange_buffer before eis_set_state%s");
    if (M == 1) {  // one grid: a misfit is an argument error (members get a status, k_to_tiles)
      long long nn = c->grid.n_cells;
      if (n_cells && where == EIS_HOST) nn = n_cells[0];
      const long long lo_last = (long long)(c->tl.tpm - 1) * c->tile_cells;
      if (nn - lo_last < HALO || nn - lo_last > c->tl.capt) return fail(c, EIS_E_ARG, "set_state: n_cells does not fit the tiling%s");
    }
  }
  if (M == 1 && where == EIS_HOST) {  // one grid from the host: only its live cells cross the link
    const long long nn = n_cells ? n_cells[0] : c->grid.n_cells;
    if (nn >= 3 && nn <= cap) bytes = (size_t)nn * 8;
  }
  CU(cudaMemcpyAsync(c->d_rho, rho, bytes, kind, c->stream));
  CU(cudaMemcpyAsync(c->d_mom, mom, bytes, kind, c->stream));
  if (width) CU(cudaMemcpyAsync(c->d_h, width, bytes, kind, c->stream));
  else k_fill<<<grid_for(M * cap), 256, 0, c->stream>>>(c->d_h, M * cap, c->p.h_av);
  if (n_cells) {
    CU(cudaMemcpyAsync(c->d_n, n_cells, M * 8, kind, c->stream));
  } else {
    k_fill_ll<<<grid_for(M), 256, 0, c->stream>>>(c->d_n, M, c->grid.n_cells);
  }
  CU(cudaMemsetAsync(c->d_status, 0, (size_t)M * 4, c->stream));
  {
    const long long ny = std::min<long long>(65535, (c->grid.cell_capacity + VALIDATE_CHUNK - 1) / VALIDATE_CHUNK);
    k_validate<<<dim3((unsigned)M, (unsigned)std::max<long long>(ny, 1)), 256, 0, c->stream>>>(c->e, c->g, t0);
  }
  CU(cudaGetLastError());
  if (c->tiled) {
    k_tiles_reset<<<(unsigned)((M + 127) / 128), 128, 0, c->stream>>>(c->tl, c->d_status, t0);
    CU(cudaMemsetAsync(c->t_wlist, 0, (size_t)c->tl.ntiles * 16, c->stream));  // window ready tags
    for (int b = 0; b < 2 && c->tl.spec; ++b) CU(cudaMemsetAsync(c->t_pred[b], 0xff, (size_t)c->tl.ntiles * 16, c->stream));  // no predictions
    k_to_tiles<<<c->tl.ntiles, 256, 0, c->stream>>>(c->g, c->tl, 0, c->tile_cells);
    tiled_init_dt<256><<<c->tl.ntiles, 256, 0, c->stream>>>(c->e, c->p, c->tl, INFINITY);
    if (M > 1) tiled_members_finish<<<(unsigned)((M * 32 + 255) / 256), 256, 0, c->stream>>>(c->p, c->tl, INFINITY, 0);
    CU(cudaGetLastError());
    c->staging_fresh = 1;
  }
  if (where == EIS_HOST) CU(cudaStreamSynchronize(c->stream));
  c->state_set = 1;
  c->sticky = EIS_OK;
  c->msg[0] = 0;
  return EIS_OK;
}

static eis_status collect_stats(eis_ctx* c, eis_stats* out) {
  const long long M = c->grid.n_members;
#ifdef EIS_PHASE_CLOCK
  if (c->g.dbg) {  // development: mean cycles per step (all members)
    std::vector<long long> d((size_t)M * 8);
    CU(cudaMemcpyAsync(d.data(), c->g.dbg, (size_t)M * 64, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    double acc[7] = {0};
    for (long long m = 0; m < M; ++m) for (int i = 0; i < 7; ++i) acc[i] += (double)d[8 * m + i];
    const double ns = acc[6] > 0 ? acc[6] : 1;
    fprintf(stderr, "[phase] steps %.0f | cycles/step from start: solver@A %.0f warp0@A %.0f solver@B %.0f warp0@B %.0f end %.0f | S4 %.0f\n",
            acc[6], acc[0] / ns, acc[1] / ns, acc[2] / ns, acc[3] / ns, acc[4] / ns, acc[5] / ns);
  }
#endif
  std::vector<MemberStats> ms(M);
  std::vector<double> t(M);
  CU(cudaMemcpyAsync(ms.data(), c->d_stats, M * sizeof(MemberStats), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(t.data(), c->d_t, M * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  memset(out, 0, sizeof(*out));
  out->t_min = INFINITY; out->t_max = -INFINITY; out->dt_min = INFINITY; out->dt_max = 0;
  for (long long m = 0; m < M; ++m) {
    const MemberStats& s = ms[m];
    out->steps += s.steps; out->cell_updates += s.cell_updates; out->dts_iters += s.dts_iters;
    out->iface_solves += s.iface_solves; out->creations += s.creations; out->splits += s.splits;
    out->merges += s.merges; out->regions += s.regions;
    out->dts_iter_max = std::max(out->dts_iter_max, (int64_t)s.dts_max);
    out->decision_margin_warnings += s.margins;
    out->t_min = std::fmin(out->t_min, t[m]); out->t_max = std::fmax(out->t_max, t[m]);
    if (s.steps) out->dt_min = std::fmin(out->dt_min, s.dt_min);
    out->dt_max = std::fmax(out->dt_max, s.dt_max);
  }
  return EIS_OK;
}

// one large step of the tiled grid: the streaming pass over every tile, then the full step of
// the listed tiles (and, by its last CTA, the next dt)
static int timing_event(eis_ctx* c, cudaStream_t st = nullptr) {  // an event from the pool, recorded on a stream
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t ev;
    if (cudaEventCreate(&ev) != cudaSuccess) return -1;
    c->ev_pool.push_back(ev);
  }
  const int i = (int)c->ev_used++;
  cudaEventRecord(c->ev_pool[i], st ? st : c->stream);
  return i;
}

// development (EIS_SYNC_DEBUG=1): synchronise after every launch of a step and name the first failure
static void dbg_sync(eis_ctx* c, const char* what) {
  static const int on = getenv("EIS_SYNC_DEBUG") ? atoi(getenv("EIS_SYNC_DEBUG")) : 0;
  if (!on) return;
  cudaError_t e1 = cudaStreamSynchronize(c->stream2), e2 = cudaStreamSynchronize(c->stream);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    fprintf(stderr, "EIS_SYNC_DEBUG: after %s: %s / %s\n", what, cudaGetErrorString(e1), cudaGetErrorString(e2));
    int ctl[NCTL];
    if (cudaMemcpy(ctl, c->t_ctl, sizeof(ctl), cudaMemcpyDeviceToHost) == cudaSuccess)
      for (int q = 0; q < NCTL; ++q) fprintf(stderr, " ctl[%d]=%d", q, ctl[q]);
    fprintf(stderr, "\n");
    abort();
  }
}

static void tiled_launch(eis_ctx* c, double t_end) {
  std::array<int, 5> m{-1, -1, -1, -1, 1};
  // a step captured into a CUDA graph (rank mode: step_local -> halo exchange -> step_finish
  // replayed without the host) records no timing events: the pool's events belong to eager steps
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cap);
  const int timing_saved = c->timing;
  if (cap != cudaStreamCaptureStatusNone) c->timing = 0;
  // tiled_fast, then (side stream, high priority) a window kernel that takes window jobs as
  // tiled_fast publishes them; after tiled_fast a full-occupancy instance drains the rest
  if (c->win_grid_poll > 0 || c->tl.spec) cudaEventRecord(c->ev_fork, c->stream);
  if (c->timing) m[0] = timing_event(c);
  static const int spec_timing_on = getenv("EIS_SPEC_TIMING") ? atoi(getenv("EIS_SPEC_TIMING")) : 0;
  const bool spec_timing = spec_timing_on && c->timing && c->tl.split;
  std::array<int, 6> sm{m[0], -1, -1, -1, -1, -1};
  if (c->tl.spec) {  // the predicted windows: part A and their DTS jobs beside tiled_fast
    cudaStreamWaitEvent(c->stream2, c->ev_fork, 0);
    tiled_win<32, EIS_WIN_MINB, false, 1, 1><<<c->win_grid_early, 32, c->smem_win, c->stream2>>>(c->e, c->p, c->tl, t_end);
    if (spec_timing) sm[1] = timing_event(c, c->stream2);
    dts_jobs<<<c->dts_grid * 32 / c->dts_tpb, c->dts_tpb, 0, c->stream2>>>(c->e, c->p, c->tl, 1);
    if (spec_timing) sm[2] = timing_event(c, c->stream2);
    cudaEventRecord(c->ev_join, c->stream2);
    dbg_sync(c, "early part A + dts_jobs");
  }
  const int plain_ok = c->fast_plain, one_ok = c->fast_one;
  const bool plain = plain_ok && !c->tl.nbr_left && !c->tl.nbr_right && !c->tl.poll;  // (no exchange buffer, no polling kernel)
  const bool one = one_ok && plain && c->tl.M == 1;
  if (one && c->tl.spec)
    tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true, true, 1><<<c->tl.ntiles, EIS_FAST_T, c->smem_fast, c->stream>>>(c->e, c->p, c->tl, t_end);
  else if (one)
    tiled_fast<EIS_FAST_T, EIS_FAST_MINB, false, true, 1><<<c->tl.ntiles, EIS_FAST_T, c->smem_fast, c->stream>>>(c->e, c->p, c->tl, t_end);
  else if (one_ok && plain && c->tl.M <= 65535 && c->tl.spec)  // ensembles: (tile in member, member) as a 2D grid
    tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true, true, 2><<<dim3((unsigned)c->tl.tpm, (unsigned)c->tl.M), EIS_FAST_T, c->smem_fast, c->stream>>>(c->e, c->p, c->tl, t_end);
  else if (one_ok && plain && c->tl.M <= 65535)
    tiled_fast<EIS_FAST_T, EIS_FAST_MINB, false, true, 2><<<dim3((unsigned)c->tl.tpm, (unsigned)c->tl.M), EIS_FAST_T, c->smem_fast, c->stream>>>(c->e, c->p, c->tl, t_end);
  else if (c->tl.spec && plain)
    tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true, true><<<c->tl.ntiles, EIS_FAST_T, c->smem_fast, c->stream>>>(c->e, c->p, c->tl, t_end);
  else if (c->tl.spec)
    tiled_fast<EIS_FAST_T, EIS_FAST_MINB, true><<<c->tl.ntiles, EIS_FAST_T, c->smem_fast, c->stream>>>(c->e, c->p, c->tl, t_end);
  else if (plain)
    tiled_fast<EIS_FAST_T, EIS_FAST_MINB, false, true><<<c->tl.ntiles, EIS_FAST_T, c->smem_fast, c->stream>>>(c->e, c->p, c->tl, t_end);
  else
    tiled_fast<EIS_FAST_T, EIS_FAST_MINB><<<c->tl.ntiles, EIS_FAST_T, c->smem_fast, c->stream>>>(c->e, c->p, c->tl, t_end);
  dbg_sync(c, "tiled_fast");
  if (c->timing) m[1] = timing_event(c);
  if (c->win_grid_poll > 0) {
    cudaStreamWaitEvent(c->stream2, c->ev_fork, 0);
    if (c->tl.split)  // part A of the windows as tiled_fast publishes them
      tiled_win<32, EIS_WIN_MINB, true, 1><<<c->win_grid_poll, 32, c->smem_win, c->stream2>>>(c->e, c->p, c->tl, t_end);
    else
      tiled_win<32, EIS_WIN_MINB, true><<<c->win_grid_poll, 32, c->smem_win, c->stream2>>>(c->e, c->p, c->tl, t_end);
    cudaEventRecord(c->ev_join, c->stream2);
  }
  if (c->tl.split) {  // part A, the DTS jobs (one lane per block), part B
    if (c->tl.spec) cudaStreamWaitEvent(c->stream, c->ev_join, 0);  // the early jobs are solved (and counted)
    tiled_win<32, EIS_WIN_MINB, false, 1><<<c->win_grid, 32, c->smem_win, c->stream>>>(c->e, c->p, c->tl, t_end);
    dbg_sync(c, "part A");
    if (spec_timing) sm[3] = timing_event(c);
    if (c->win_grid_poll > 0) cudaStreamWaitEvent(c->stream, c->ev_join, 0);  // every part A done
    dts_jobs<<<c->dts_grid * 32 / c->dts_tpb, c->dts_tpb, 0, c->stream>>>(c->e, c->p, c->tl, 0);
    dbg_sync(c, "dts_jobs");
    if (spec_timing) sm[4] = timing_event(c);
#ifdef EIS_DTS_DEBUG
    dts_dbg_print<<<1, 1, 0, c->stream>>>();
#endif
    tiled_win<32, EIS_WIN_MINB, false, 2><<<c->win_grid, 32, c->smem_win, c->stream>>>(c->e, c->p, c->tl, t_end);
    dbg_sync(c, "part B");
    if (spec_timing) { sm[5] = timing_event(c); c->ev_spec.push_back(sm); }
  } else {
    tiled_win<32, EIS_WIN_MINB, false><<<c->win_grid, 32, c->smem_win, c->stream>>>(c->e, c->p, c->tl, t_end);
  }
  if (c->win_grid_poll > 0 && !c->tl.split) cudaStreamWaitEvent(c->stream, c->ev_join, 0);
  if (c->timing) m[2] = timing_event(c);
  tiled_slow<256, 4><<<c->slow_grid, 256, c->smem, c->stream>>>(c->e, c->p, c->tl, t_end);
  dbg_sync(c, "tiled_slow");
  if (c->tl.M > 1)
    tiled_members_finish<<<(unsigned)(((long long)c->tl.M * 32 + 255) / 256), 256, 0, c->stream>>>(c->p, c->tl, t_end, 1);
  if (c->timing) {
    m[3] = timing_event(c); c->ev_marks.push_back(m);
    c->n_kernels += 2 + (c->tl.split ? 3 : 1) + (c->win_grid_poll > 0 ? 1 : 0) + (c->tl.M > 1 ? 1 : 0) + (c->tl.spec ? 2 : 0);
  }
  c->timing = timing_saved;
}

static eis_status launch(eis_ctx* c, long long n_steps, double t_end, eis_stats* out) {
  if (!c) return EIS_E_ARG;
  if (c->sticky) return c->sticky;
  if (!c->state_set) return fail(c, EIS_E_ORDER, "step before set_state%s");
  if (n_steps < 0) return fail(c, EIS_E_ARG, "negative step count%s");
  CU(cudaSetDevice(c->grid.device));
  if (c->tiled) {
    c->staging_fresh = 0;
    const long long M = c->tl.M;
    for (long long s = 0; s < n_steps; ++s) {
      tiled_launch(c, t_end);
      if ((s & 63) == 63 && t_end < INFINITY) {  // poll: stop launching once t_end is reached
        if (M == 1) {
          double tt;
          int st;
          CU(cudaMemcpyAsync(&tt, c->t_scal, 8, cudaMemcpyDeviceToHost, c->stream));
          CU(cudaMemcpyAsync(&st, c->t_mctl + 1, 4, cudaMemcpyDeviceToHost, c->stream));
          CU(cudaStreamSynchronize(c->stream));
          if (!(tt < t_end) || st != 0) break;
        } else {
          int act;
          CU(cudaMemsetAsync(c->t_ctl + 10, 0, 4, c->stream));
          tiled_members_active<<<(unsigned)((M + 255) / 256), 256, 0, c->stream>>>(c->tl, t_end);
          CU(cudaMemcpyAsync(&act, c->t_ctl + 10, 4, cudaMemcpyDeviceToHost, c->stream));
          CU(cudaMemsetAsync(c->t_ctl + 10, 0, 4, c->stream));  // (the next step counts its DTS jobs from 0)
          CU(cudaStreamSynchronize(c->stream));
          if (act == 0) break;
        }
      }
    }
    CU(cudaGetLastError());
    if (out) return tiled_stats(c, out);
    return EIS_OK;
  }
  if (n_steps > 0) {
    const unsigned M = (unsigned)c->grid.n_members;
    std::array<int, 5> m{-1, -1, -1, -1, 0};
    if (c->timing) m[0] = timing_event(c);
    if (c->threads <= 128 && M <= 148)  // few members (C1, C2, the paper's tests): no register cap
      resident_steps<128, 1><<<M, c->threads, c->smem, c->stream>>>(c->e, c->p, c->g, n_steps, t_end);
    else if (c->threads <= 128)
      resident_steps<128, 4><<<M, c->threads, c->smem, c->stream>>>(c->e, c->p, c->g, n_steps, t_end);
    else if (c->threads <= 256 && c->minb == 4)
      resident_steps<256, 4><<<M, c->threads, c->smem, c->stream>>>(c->e, c->p, c->g, n_steps, t_end);
    else if (c->threads <= 256)
      resident_steps<256, 2><<<M, c->threads, c->smem, c->stream>>>(c->e, c->p, c->g, n_steps, t_end);
    else if (c->threads <= 512)
      resident_steps<512, 1><<<M, c->threads, c->smem, c->stream>>>(c->e, c->p, c->g, n_steps, t_end);
    else
      resident_steps<1024, 1><<<M, c->threads, c->smem, c->stream>>>(c->e, c->p, c->g, n_steps, t_end);
    if (c->timing) { m[1] = timing_event(c); c->ev_marks.push_back(m); c->n_kernels += 1; }
    CU(cudaGetLastError());
  }
  if (out) return collect_stats(c, out);
  return EIS_OK;
}

extern "C" eis_status eis_step(eis_ctx* c, int64_t n_steps, eis_stats* out) {
  return launch(c, n_steps, INFINITY, out);
}

extern "C" eis_status eis_run_to(eis_ctx* c, double t_end, int64_t max_steps, eis_stats* out) {
  return launch(c, max_steps, t_end, out);
}

static dim3 pack_grid(const eis_ctx* c) {
  const long long ny = std::min<long long>(65535, std::max<long long>(1, (c->grid.cell_capacity + 255) / 256 / 8));
  return dim3((unsigned)c->grid.n_members, (unsigned)(c->grid.n_members > 1 ? 1 : ny));
}

extern "C" eis_status eis_get_state(eis_ctx* c, double* rho, double* mom, double* width, uint8_t* phase,
                                    int64_t* n_cells, double* t, int32_t where) {
  if (!c) return EIS_E_ARG;
  if (c->sticky) return c->sticky;
  if (!c->state_set) return fail(c, EIS_E_ORDER, "get_state before set_state%s");
  if (where != EIS_HOST && where != EIS_DEVICE) return fail(c, EIS_E_ARG, "get_state: bad where%s");
  CU(cudaSetDevice(c->grid.device));
  if (c->tiled) { eis_status s0 = tiles_to_staging(c); if (s0) return s0; }
  const long long M = c->grid.n_members, cap = c->grid.cell_capacity;
  const size_t cells = (size_t)M * cap;
  if (where == EIS_DEVICE) {
    k_pack<<<pack_grid(c), 256, 0, c->stream>>>(c->e, c->g, rho, mom, width, phase);
    CU(cudaGetLastError());
    if (n_cells) CU(cudaMemcpyAsync(n_cells, c->d_n, M * 8, cudaMemcpyDeviceToDevice, c->stream));
    if (t) CU(cudaMemcpyAsync(t, c->d_t, M * 8, cudaMemcpyDeviceToDevice, c->stream));
    return EIS_OK;
  }
  eis_status s = ensure_pack(c);
  if (s) return s;
  double* pr = c->d_pack;
  k_pack<<<pack_grid(c), 256, 0, c->stream>>>(c->e, c->g, rho ? pr : nullptr, mom ? pr + cells : nullptr,
                                             width ? pr + 2 * cells : nullptr, phase ? c->d_u8 : nullptr);
  CU(cudaGetLastError());
  size_t ncopy = cells;  // one grid: only its live cells cross the link (the rest is unspecified)
  if (M == 1) {
    long long nn = 0;
    CU(cudaMemcpyAsync(&nn, c->d_n, 8, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (nn > 0 && nn <= cap) ncopy = (size_t)nn;
  }
  if (rho) CU(cudaMemcpyAsync(rho, pr, ncopy * 8, cudaMemcpyDeviceToHost, c->stream));
  if (mom) CU(cudaMemcpyAsync(mom, pr + cells, ncopy * 8, cudaMemcpyDeviceToHost, c->stream));
  if (width) CU(cudaMemcpyAsync(width, pr + 2 * cells, ncopy * 8, cudaMemcpyDeviceToHost, c->stream));
  if (phase) CU(cudaMemcpyAsync(phase, c->d_u8, ncopy, cudaMemcpyDeviceToHost, c->stream));
  if (n_cells) CU(cudaMemcpyAsync(n_cells, c->d_n, M * 8, cudaMemcpyDeviceToHost, c->stream));
  if (t) CU(cudaMemcpyAsync(t, c->d_t, M * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (ncopy < cells) {  // the contract's tail (include/eis.h): zeros and phase 255 past n_cells
    const size_t tail = cells - ncopy;
    if (rho) memset(rho + ncopy, 0, tail * 8);
    if (mom) memset(mom + ncopy, 0, tail * 8);
    if (width) memset(width + ncopy, 0, tail * 8);
    if (phase) memset(phase + ncopy, 255, tail);
  }
  return EIS_OK;
}

extern "C" eis_status eis_interfaces(eis_ctx* c, eis_interface* out, int64_t capacity, int64_t* count) {
  if (!c || !count) return EIS_E_ARG;
  if (c->sticky) return c->sticky;
  if (!c->state_set) return fail(c, EIS_E_ORDER, "interfaces before set_state%s");
  CU(cudaSetDevice(c->grid.device));
  if (c->tiled) { eis_status s0 = tiles_to_staging(c); if (s0) return s0; }
  const long long M = c->grid.n_members;
  const unsigned nb = (unsigned)((M + 127) / 128);
  k_iface<<<nb, 128, 0, c->stream>>>(c->e, c->g, M, c->grid.x_left, nullptr, c->d_cnt, nullptr, 0);
  CU(cudaGetLastError());
  std::vector<long long> cnt(M), off(M);
  CU(cudaMemcpyAsync(cnt.data(), c->d_cnt, M * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  long long total = 0;
  for (long long m = 0; m < M; ++m) { off[m] = total; total += cnt[m]; }
  *count = total;
  if (out && capacity > 0 && total > 0) {
    if (c->if_cap < total) {
      cudaFree(c->d_if);
      c->d_if = nullptr;
      CU(cudaMalloc(&c->d_if, total * sizeof(eis_interface)));
      c->if_cap = total;
    }
    if (!c->d_ifoff) CU(cudaMalloc(&c->d_ifoff, M * 8));
    long long* d_off = c->d_ifoff;
    CU(cudaMemcpyAsync(d_off, off.data(), M * 8, cudaMemcpyHostToDevice, c->stream));
    k_iface<<<nb, 128, 0, c->stream>>>(c->e, c->g, M, c->grid.x_left, d_off, nullptr, c->d_if, total);
    k_iface_solve<<<(unsigned)((total + 7) / 8), 128, 0, c->stream>>>(c->e, c->p, c->g, c->d_if, total);
    CU(cudaGetLastError());
    const long long ncopy = total < capacity ? total : capacity;
    CU(cudaMemcpyAsync(out, c->d_if, ncopy * sizeof(eis_interface), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  return (out && total > capacity) ? EIS_E_CAPACITY : EIS_OK;
}

extern "C" eis_status eis_member_status(eis_ctx* c, int32_t* out) {
  if (!c || !out) return EIS_E_ARG;
  if (!c->state_set) return fail(c, EIS_E_ORDER, "member_status before set_state%s");
  if (c->tiled) {
    std::vector<int> mctl((size_t)c->tl.M * MCS);
    CU(cudaMemcpyAsync(mctl.data(), c->t_mctl, mctl.size() * 4, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    for (int m = 0; m < c->tl.M; ++m) out[m] = mctl[(size_t)MCS * m + 1];
    return EIS_OK;
  }
  CU(cudaMemcpyAsync(out, c->d_status, c->grid.n_members * 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return EIS_OK;
}

extern "C" eis_status eis_member_stats(eis_ctx* c, eis_stats* out) {
  if (!c || !out) return EIS_E_ARG;
  if (!c->state_set) return fail(c, EIS_E_ORDER, "member_stats before set_state%s");
  if (c->tiled) return tiled_member_stats(c, out);
  const long long M = c->grid.n_members;
  std::vector<MemberStats> ms(M);
  std::vector<double> t(M);
  CU(cudaMemcpyAsync(ms.data(), c->d_stats, M * sizeof(MemberStats), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(t.data(), c->d_t, M * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (long long m = 0; m < M; ++m) {
    const MemberStats& s = ms[m];
    eis_stats& o = out[m];
    o.steps = s.steps; o.cell_updates = s.cell_updates; o.dts_iters = s.dts_iters; o.iface_solves = s.iface_solves;
    o.creations = s.creations; o.splits = s.splits; o.merges = s.merges; o.regions = s.regions;
    o.t_min = o.t_max = t[m]; o.dt_min = s.dt_min; o.dt_max = s.dt_max; o.dts_iter_max = s.dts_max;
    o.decision_margin_warnings = s.margins;
  }
  return EIS_OK;
}

// ------------------------------------------------------------------------------------------
// rank mode (one tiled grid decomposed over ranks): exchange buffer + split step
// ------------------------------------------------------------------------------------------
static_assert(EIS_XB_DOUBLES_PEER == XB_DOUBLES_PEER && EIS_XB_MAXRANKS == XB_MAXRANKS, "exchange layout (include/eis.h)");
// peer mode: the neighbours' exchange buffers and every rank's (device pointers this context's
// device can access: peer-mapped / symmetric memory), each of EIS_XB_DOUBLES_PEER doubles
extern "C" eis_status eis_set_exchange_peers(eis_ctx* c, double* left, double* right, double* const* all,
                                             int32_t rank, int32_t world) {
  if (!c || !c->tiled || !c->tl.xbuf || !all || world < 1 || world > XB_MAXRANKS || rank < 0 || rank >= world)
    return EIS_E_ARG;
  if ((c->tl.nbr_left != 0) != (left != nullptr) || (c->tl.nbr_right != 0) != (right != nullptr)) return EIS_E_ARG;
  for (int q = 0; q < world; ++q) if (!all[q]) return EIS_E_ARG;
  if (all[rank] != c->tl.xbuf) return EIS_E_ARG;  // this rank's entry is its own exchange buffer
  CU(cudaSetDevice(c->grid.device));
  if (!c->d_xpeers) CU(cudaMalloc(&c->d_xpeers, XB_MAXRANKS * sizeof(double*)));
  CU(cudaMemcpy(c->d_xpeers, all, world * sizeof(double*), cudaMemcpyHostToDevice));
  c->tl.xpeer_l = left; c->tl.xpeer_r = right;
  c->tl.xpeers = c->d_xpeers; c->tl.xrank = rank; c->tl.xworld = world;
  return EIS_OK;
}

extern "C" eis_status eis_set_exchange_buffer(eis_ctx* c, double* xbuf) {
  if (!c || !c->tiled || !xbuf) return EIS_E_ARG;
  c->tl.xbuf = xbuf;
  return EIS_OK;
}

extern "C" eis_status eis_step_local(eis_ctx* c, double t_end) {
  if (!c || !c->tiled || !c->tl.xbuf) return EIS_E_ARG;
  if (c->sticky) return c->sticky;
  if (!c->state_set) return fail(c, EIS_E_ORDER, "step before set_state%s");
  CU(cudaSetDevice(c->grid.device));
  c->staging_fresh = 0;
  tiled_launch(c, t_end);
  CU(cudaGetLastError());
  return EIS_OK;
}

extern "C" eis_status eis_step_finish(eis_ctx* c, double t_end, int32_t after_step) {
  if (!c || !c->tiled || !c->tl.xbuf) return EIS_E_ARG;
  if (c->sticky) return c->sticky;
  CU(cudaSetDevice(c->grid.device));
  tiled_finish<<<1, 32, 0, c->stream>>>(c->p, c->tl, t_end, after_step);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cap);
  if (c->timing && cap == cudaStreamCaptureStatusNone) c->n_kernels += 1;
  CU(cudaGetLastError());
  return EIS_OK;
}

// ---------------------------------------------------------------------------------------------
// Lax shock tube batches (include/eis.h): validation, one launch, stats back.
// ---------------------------------------------------------------------------------------------
extern "C" eis_status eis_lax_run(const eis_lax_case* cases, int64_t n_cases, int64_t stride, double* rho,
                                  double* mom, double* E, eis_lax_stats* stats, void* stream) {
  if (!cases || !stats || !rho || !mom || !E || n_cases <= 0 || n_cases > (int64_t)INT32_MAX) return EIS_E_ARG;
  int64_t nmax = 0;
  for (int64_t i = 0; i < n_cases; ++i) {
    const eis_lax_case& c = cases[i];
    if (c.n < 6 || (c.n & 1) || c.n > lax::LAX_MAX_N || c.n + 2 > stride || !(c.alpha > 0.0) ||
        !(c.theta_nb > 0.0) || !(c.cfl > 0.0) || !(c.gamma > 1.0) || !(c.x_right > c.x_left) ||
        !(c.t_end >= 0.0) || c.dts_max_iter < 1)
      return EIS_E_ARG;
    nmax = std::max(nmax, c.n);
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = lax::smem_bytes((int)nmax);
  if (cudaFuncSetAttribute(lax::lax_cases, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return EIS_E_CUDA;
  eis_lax_case* d_cases = nullptr;
  eis_lax_stats* d_stats = nullptr;
  if (cudaMallocAsync(&d_cases, sizeof(eis_lax_case) * n_cases, st) != cudaSuccess) return EIS_E_CUDA;
  if (cudaMallocAsync(&d_stats, sizeof(eis_lax_stats) * n_cases, st) != cudaSuccess) {
    cudaFreeAsync(d_cases, st);
    return EIS_E_CUDA;
  }
  cudaMemcpyAsync(d_cases, cases, sizeof(eis_lax_case) * n_cases, cudaMemcpyHostToDevice, st);
  lax::lax_cases<<<(unsigned)n_cases, lax::LAX_THREADS, smem, st>>>(d_cases, stride, rho, mom, E, d_stats);
  const cudaError_t le = cudaGetLastError();
  cudaMemcpyAsync(stats, d_stats, sizeof(eis_lax_stats) * n_cases, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_cases, st);
  cudaFreeAsync(d_stats, st);
  const cudaError_t se = cudaStreamSynchronize(st);
  return le == cudaSuccess && se == cudaSuccess ? EIS_OK : EIS_E_CUDA;
}
