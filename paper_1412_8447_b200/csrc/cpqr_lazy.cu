// cpqr_lazy.cu -- bound-pruned ("lazy") variant of the panel CPQR of
// cpqr_panel.cu: per step only the columns whose norm bound can reach the
// step's maximum are brought up to date; panel_finalize_kernel catches every
// column up at the end of a panel on the DMMA pipe.  Same pivots as
// evaluating every column every step (cpqr.hpp:48-85).
#include <cstdio>

#include "cpqr_panel.cuh"

namespace lrb {
namespace cpqr_detail {
namespace {

// Spin waits of the lazy kernel with a watchdog: a wait that exceeds ~4 s of
// SM clock reports where it stood and traps (a launch error instead of a hang).
__device__ __noinline__ void lazy_stuck(const char* what, long long s, unsigned int have, unsigned int want) {
  printf("cpqr_lazy watchdog: cta %d stuck in %s at step %lld (have %u, want %u)\n", (int)blockIdx.x, what, s, have,
         want);
  __trap();
}
__device__ __forceinline__ void lazy_grid_wait(const unsigned int* bar, unsigned int target, long long s) {
  if (threadIdx.x == 0) {
    unsigned int v;
    const long long t0 = clock64();
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (clock64() - t0 > (8ll << 30)) lazy_stuck("grid barrier", s, v, target);
    } while (v < target);
  }
  __syncthreads();
}
__device__ __forceinline__ void lazy_tag_wait(const unsigned int* tag, unsigned int want, long long s) {
  unsigned int t;
  const long long t0 = clock64();
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(t) : "l"(tag) : "memory");
    if (clock64() - t0 > (8ll << 30)) lazy_stuck("candidate tag", s, t, want);
  } while (!tag_ready(t, want));
}

// ============================================================ lazy (bound-pruned) variant
// The eager kernel above reads every trailing column every step, but the
// argmax of step s+1 only needs the exact downdated norms of the columns that
// can win it.  A downdate never increases a value (fl(x - r^2) <= x), and an
// exact recompute (cpqr.hpp:78-84) only replaces a value that fell below 1e-6
// of the last exact one by the exact trailing norm, which exceeds the value it
// replaced by at most the accumulated downdate roundoff (< 1e-12 nx after 512
// steps).  So ub = nr + 1e-10 nx, the value at a column's last evaluation,
// bounds all of its later values, and a column with ub < L cannot be the
// maximum once some evaluated column reaches L.  Per step every CTA evaluates
// -- catches up through the step's reflector, replaying each missed step's F
// entry, R(s, j), downdate and recompute check in order, the eager pass's
// arithmetic -- only its columns with ub >= L, L = beta * M_s (M_s: this
// step's winning norm^2, beta from the recent ratios M_s / M_{s-1}).  If the
// best value found is below L the round is repeated with L = that value
// (everything skipped is then strictly smaller).  The columns never evaluated
// in a panel are caught up at its end by panel_finalize_kernel on the DMMA
// pipe (D = V^T A_p, then the same recurrence), which also applies the rank-NB
// update.  The pivot sequence is the one of evaluating every column every step.


constexpr double kLazyGapInit = 0.1, kLazyGapMin = 0.02, kLazyGapMax = 0.5;
constexpr double kLazyGapHit = 0.98, kLazyGapMiss = 1.9;  // 0.98^32 ~ 1 / 1.9: one retry per ~30 steps

// Reflector of column b for step s1 from A_p - V F^T (c_used panel reflectors
// applied) into the candidate buffer cd, plus w = V^T v when the next step
// continues this panel (the eager kernel's `stage`, as a function).
__device__ __forceinline__ void stage_candidate(const PanelArgs& a, double* cd, int64_t s1, long long b, int c_used,
                                bool same_panel, const double* Vs, double* scr, double* fb, double* sh_alpha,
                                double* sh_red) {
  const int64_t m = a.m, ld = a.ld;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (b >= a.n || s1 >= m) {
    __syncthreads();
    return;
  }
  const double* x = a.W + b * ld;
  double xl[kRowsPerThread];
#pragma unroll
  for (int q = 0; q < kRowsPerThread; ++q) {
    const int64_t r = threadIdx.x + PT * q;
    xl[q] = (r >= s1 && r < m) ? __ldcg(x + r) : 0.0;
  }
  if (threadIdx.x < NB) fb[threadIdx.x] = threadIdx.x < c_used ? __ldcg(a.F + b * NB + threadIdx.x) : 0.0;
  __syncthreads();
  double xr[kRowsPerThread];
  double part = 0.0;
#pragma unroll
  for (int q = 0; q < kRowsPerThread; ++q) {
    const int64_t r = threadIdx.x + PT * q;
    xr[q] = 0.0;
    if (r >= s1 && r < m) {
      double v0 = xl[q], v1 = 0.0, v2 = 0.0, v3 = 0.0;
      int i = 0;
      for (; i + 4 <= c_used; i += 4) {
        v0 = fma(-Vs[i * ld + r], fb[i], v0);
        v1 = fma(-Vs[(i + 1) * ld + r], fb[i + 1], v1);
        v2 = fma(-Vs[(i + 2) * ld + r], fb[i + 2], v2);
        v3 = fma(-Vs[(i + 3) * ld + r], fb[i + 3], v3);
      }
      for (; i < c_used; ++i) v0 = fma(-Vs[i * ld + r], fb[i], v0);
      const double v = (v0 + v1) + (v2 + v3);
      xr[q] = v;
      if (r == s1) *sh_alpha = v;
    }
    part = fma(xr[q], xr[q], part);
  }
  const double cn2 = cta_sum(part, sh_red);
  const double colnorm = sqrt(cn2);
  const double alpha = *sh_alpha;
  const bool apply = colnorm > 0.0;
  double beta = alpha, tau = 0.0, scale = 1.0;
  if (apply) {
    beta = alpha >= 0.0 ? -colnorm : colnorm;
    tau = (beta - alpha) / beta;
    scale = alpha - beta;
  }
  double vr[kRowsPerThread];
#pragma unroll
  for (int q = 0; q < kRowsPerThread; ++q) {
    const int64_t r = threadIdx.x + PT * q;
    vr[q] = 0.0;
    if (r >= s1 && r < m) vr[q] = apply ? ((r == s1) ? 1.0 : xr[q] / scale) : xr[q];
    if (r < ld) cd[kHdr + r] = vr[q];
  }
  if (threadIdx.x == 0) {
    cd[0] = alpha;
    cd[1] = beta;
    cd[2] = tau;
    cd[3] = apply ? 1.0 : 0.0;
  }
  if (same_panel) {
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q)
      if (threadIdx.x + PT * q < ld) scr[threadIdx.x + PT * q] = vr[q];
    __syncthreads();
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t rr = s1 + lane; rr < m; rr += 32) {
      const double vt = scr[rr];
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[t] = fma(Vs[(warp + PW * t) * ld + rr], vt, acc[t]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = warp + PW * t;
      const double w = warp_sum(i < c_used ? acc[t] : 0.0);
      if (lane == 0) cd[kHdr + ld + i] = w;
    }
  }
  __syncthreads();
}

struct LazyCtx {
  const PanelArgs& a;
  int lvl;               // catch up through panel reflector lvl - 1
  const int* elist;      // slots to evaluate (any order)
  int ecnt;
  int64_t c0;
  int warp, lane;
  const double* Vs;      // [NB][ld] panel reflectors (zero outside their support; zero when not applied)
  const double* swall;   // [NB][NB] w of each step
  const double* sM;      // [NBL][NBL] F = M D' (see below)
  double* snr;
  double* snx;
  int* spos;
  int* scj;
  unsigned long long recomputes;
};

// Catch-up of the listed slots, one warp per column (rows base + 2(lane +
// 32 k) + {0, 1} in registers, one read of the column for all missed steps):
//   D(cc)  = A_p(:, j)^T v_cc for every missed panel step cc in [cj, lvl) at
//            once (independent dot products), reduced over the warp by a
//            transpose-reduce (lane 2cc ends with D(cc));
//   F(cc)  = sum_{cj <= i <= cc} M(cc, i) D'(i),  D'(i) = D(i) - w_i^T F(j, <cj):
//            the xLAQPS recurrence F(c) = tau_c (D(c) - w_c^T F(<c)) solved
//            once per panel step for every column (M lower triangular,
//            M(c, c) = tau_c, M(c, i) = -tau_c sum_{i<=t<c} w_c[t] M(t, i));
//   R(s_cc, j) = A_p(s_cc, j) - V(s_cc, <=cc) F(j, <=cc);
//   nr -= R^2 in step order with the exact recompute below 1e-6 nx
//            (cpqr.hpp:68-84) -- the only sequential part, a scalar chain.
// The panel rows [t0, t0 + NBL) all sit in the lanes' first chunk (k = 0).
template <int TC0, int NLD>
__device__ __forceinline__ void lazy_cols(LazyCtx& x, double& bv, long long& bp) {
  constexpr int KP = NLD - TC0;  // row pairs per lane
  constexpr int D = 2;           // columns in flight per warp
  const PanelArgs& a = x.a;
  const int64_t ld = a.ld, m = a.m, t0 = a.t0;
  const int lane = x.lane, lvl = x.lvl;
  const int base = 64 * TC0;
  const int my = lane >> 1;  // the panel step this lane reduces / solves for
  struct Slot {
    double c[KP][2];
    double fl;
    double nr, nx;
    int j, lp, cj;
    bool ok;
  };
  auto fetch = [&](Slot& cb, int qi) {
    const int q = x.warp + PW * qi;
    cb.ok = q < x.ecnt;
    cb.j = cb.ok ? x.elist[q] : (int)x.c0;
    const int li = cb.j - (int)x.c0;
    const double* src = a.W + (size_t)cb.j * (size_t)ld + base + 2 * lane;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const double2 xx = __ldcg(reinterpret_cast<const double2*>(src + 64 * k));
      cb.c[k][0] = xx.x;
      cb.c[k][1] = xx.y;
    }
    cb.cj = cb.ok ? x.scj[li] : lvl;
    // F(j, lane & 15) (the entries below cj are the ones used), broadcast later
    cb.fl = (lane & 15) < cb.cj ? __ldcg(a.F + (size_t)cb.j * NB + (lane & 15)) : 0.0;
    cb.nr = x.snr[li];
    cb.nx = x.snx[li];
    cb.lp = x.spos[li];
  };
  auto process = [&](Slot& cb) {
    if (!cb.ok) return;  // warp-uniform (one column per warp)
    const int j = cb.j, cj = cb.cj;
    // ---- dot products of the missed reflectors
    double p[NBL];
#pragma unroll
    for (int cc = 0; cc < NBL; ++cc) {
      p[cc] = 0.0;
      if (cc >= cj && cc < lvl) {
        const double2* v2 = reinterpret_cast<const double2*>(x.Vs + (size_t)cc * ld + base);
        double q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const double2 vx = v2[lane + 32 * k];
          q0 = fma(cb.c[k][0], vx.x, q0);
          q1 = fma(cb.c[k][1], vx.y, q1);
        }
        p[cc] = q0 + q1;
      }
    }
    // ---- transpose-reduce: after the rounds of 16, 8, 4, 2 lane l holds the
    // partial of entry 8 b4 + 4 b3 + 2 b2 + b1 (b_i: bits of l), then + lane ^ 1
#pragma unroll
    for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const double send = up ? p[i] : p[i + h];
        const double keep = up ? p[i + h] : p[i];
        p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    const double dme = p[0] + __shfl_xor_sync(0xffffffffu, p[0], 1);  // D(my)
    // ---- F(j, <cj) from the earlier evaluations; D' = D - w^T F(<cj)
    double fr[NBL];
    const double* Fj = a.F + (size_t)j * NB;
#pragma unroll
    for (int t = 0; t < NBL; ++t) fr[t] = __shfl_sync(0xffffffffu, cb.fl, t);
    double dp = dme;
#pragma unroll
    for (int t = 0; t < NBL; ++t) dp = fma(-x.swall[my * NB + t], fr[t], dp);
    // ---- F(my) = sum_{cj <= i <= my} M(my, i) D'(i); the full F row in every lane
    double fm = 0.0;
#pragma unroll
    for (int i = 0; i < NBL; ++i) {
      const double di = __shfl_sync(0xffffffffu, dp, 2 * i);
      if (i >= cj) fm = fma(x.sM[my * NBL + i], di, fm);
    }
    const bool mine = my >= cj && my < lvl;
#pragma unroll
    for (int i = 0; i < NBL; ++i) {
      const double fi = __shfl_sync(0xffffffffu, fm, 2 * i);
      if (i >= cj && i < lvl) fr[i] = fi;
    }
    if (mine && !(lane & 1)) a.F[(size_t)j * NB + my] = fm;
    // ---- R(s_my, j): A_p(s_my, j) from the lane holding that row (chunk 0)
    const int rel = (int)(t0 - base) + my;
    const double x0 = __shfl_sync(0xffffffffu, cb.c[0][0], rel >> 1);
    const double x1 = __shfl_sync(0xffffffffu, cb.c[0][1], rel >> 1);
    double r = (rel & 1) ? x1 : x0;
#pragma unroll
    for (int i = 0; i < NBL; ++i) r = fma(-x.Vs[(size_t)i * ld + t0 + my], fr[i], r);
    // ---- the downdate chain in step order (every lane, same values)
    double nr = cb.nr, nx = cb.nx;
    __syncwarp();  // F(j, <lvl) visible to the recompute
#pragma unroll
    for (int cc = 0; cc < NBL; ++cc) {
      if (cc >= cj && cc < lvl) {
        const double xc = __shfl_sync(0xffffffffu, r, 2 * cc);
        double nn = nr - xc * xc;
        if (nn < 1e-6 * nx) {  // exact norm of rows s_cc+1.. of A_p - V F(<=cc) (rows still A_p)
          const int64_t sc = t0 + cc;
          const double* col = a.W + (size_t)j * ld;
          double acc = 0.0;
          for (int64_t rr = sc + 1 + lane; rr < m; rr += 32) {
            double xv = __ldcg(col + rr);
            for (int i = 0; i <= cc; ++i) xv = fma(-x.Vs[(size_t)i * ld + rr], __ldcg(Fj + i), xv);
            acc = fma(xv, xv, acc);
          }
          nn = warp_sum(acc);
          nx = nn;
          if (lane == 0) ++x.recomputes;
        }
        nr = nn;
      }
    }
    if (mine && !(lane & 1)) a.W[(size_t)j * ld + t0 + my] = r;  // R rows after the recomputes read A_p
    const int li = j - (int)x.c0;
    if (lane == 0) {
      x.snr[li] = nr;
      x.snx[li] = nx;
      x.scj[li] = lvl;
    }
    const long long key = ((long long)cb.lp << 32) | (long long)j;
    if (better(nr, key, bv, bp)) { bv = nr; bp = key; }
  };
  const int per_warp = max(0, (x.ecnt - x.warp + PW - 1) / PW);
  Slot buf[D];
#pragma unroll
  for (int u = 0; u < D - 1; ++u)
    if (u < per_warp) fetch(buf[u], u);
  for (int q0 = 0; q0 < per_warp; q0 += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int q = q0 + u;
      if (q >= per_warp) break;
      if (q + D - 1 < per_warp) fetch(buf[(u + D - 1) % D], q + D - 1);
      process(buf[u]);
    }
  }
  // (every lane of a warp holds the same candidate)
}

template <int TC0, int NLD, bool LIST>
__global__ void __launch_bounds__(PT, 1) cpqr_lazy_kernel(PanelArgs a) {
  unsigned int bar_target = 0;
  extern __shared__ double dyn[];
  __shared__ double sh_red[PW];
  __shared__ double sh_bv[PW];
  __shared__ long long sh_bp[PW];
  __shared__ double sh_hdr[kHdr];
  __shared__ long long sh_piv[2];
  __shared__ double sh_gbv, sh_thr;
  __shared__ double sh_cbv;     // this CTA's best candidate of the current step (kept across retry rounds)
  __shared__ long long sh_cbp;
  __shared__ double swall[NB * NB];
  __shared__ double stau[NB];
  __shared__ double sM[NBL * NBL];  // F = M D' for the catch-ups (lower triangular, row c set at step c)
  __shared__ double fb[NB];
  __shared__ double sh_alpha;
  __shared__ double sh_gap;  // 1 - beta of the adaptive threshold (carried across launches in lstats[2])
  __shared__ int sh_cnt[2 * PT];
  __shared__ int sh_nact, sh_nzero, sh_ecnt;
  __shared__ unsigned long long sh_zkey;

  const int G = gridDim.x, cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = a.m, n = a.n, ld = a.ld;
  const int64_t c0 = n * cta / G, c1 = n * (cta + 1) / G;
  const int64_t cand_sz = kHdr + ld + NB;
  const int nld = (int)(ld >> 6);
  const int C = (int)(a.t1 - a.t0);
  double* vv = dyn;
  double* Vs = dyn + ld;
  double* scr = Vs + NB * ld;
  double* snr = scr + ld;
  double* snx = snr + a.maxcols;
  int* spos = reinterpret_cast<int*>(snx + a.maxcols);
  int* alist = spos + a.maxcols;
  int* zlist = alist + a.maxcols;
  int* scj = zlist + a.maxcols;
  int* elist = scj + a.maxcols;
  for (int64_t i = threadIdx.x; i < (NB + 2) * ld; i += PT) dyn[i] = 0.0;
  for (int i = threadIdx.x; i < NB * NB; i += PT) swall[i] = 0.0;
  for (int i = threadIdx.x; i < NBL * NBL; i += PT) sM[i] = 0.0;
  if (threadIdx.x == 0) {
    const double g = __longlong_as_double((long long)__ldcg(a.lstats + 2));
    sh_gap = (g >= kLazyGapMin && g <= kLazyGapMax) ? g : kLazyGapInit;  // zeroed at the start of a CPQR
  }
  unsigned int ep = __ldcg(a.epoch);
  unsigned long long my_recomputes = 0, my_evals = 0, my_retries = 0;
  __syncthreads();

  // ------------------------------------------------------------ init (first launch): exact norms
  if (a.init) {
    int bad = 0;
    for (int64_t j = c0 + warp; j < c1; j += PW) {
      const double* col = a.W + j * ld;
      double acc = 0.0;
      for (int t = 0; t < nld; ++t) {
        const double2 xx = *reinterpret_cast<const double2*>(col + 64 * t + 2 * lane);
        bad |= !isfinite(xx.x) | !isfinite(xx.y);
        acc = fma(xx.x, xx.x, acc);
        acc = fma(xx.y, xx.y, acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) {
        a.nrm[j] = acc;
        a.nrmx[j] = acc == 0.0 ? -0.0 : acc;  // -0: identically zero, stays zero for the whole CPQR
        a.posof[j] = (int)j;
      }
      if (acc == 0.0) {
        a.F[j * NB + lane] = 0.0;
        if (lane == 0) atomicAdd(a.nzero, 1);
      }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(a.flags, 1);
    grid_barrier(a.bar, bar_target);
    if (__ldcg(a.flags) != 0) return;
  }
  for (int64_t j = c0 + threadIdx.x; j < c1; j += PT) {
    snr[j - c0] = __ldcg(a.nrm + j);
    snx[j - c0] = __ldcg(a.nrmx + j);
    spos[j - c0] = __ldcg(a.posof + j);
    scj[j - c0] = 0;
  }
  __syncthreads();
  if constexpr (!LIST) {
    if (threadIdx.x == 0) {
      sh_nact = (int)(c1 - c0);
      sh_nzero = 0;
    }
    __syncthreads();
  } else {  // ordered compaction of the owned slots into the active and zero lists
    const int64_t nloc = c1 - c0, chunk = (nloc + PT - 1) / PT;
    const int64_t b0 = min(nloc, chunk * threadIdx.x), b1 = min(nloc, b0 + chunk);
    int na = 0, nz = 0;
    for (int64_t t = b0; t < b1; ++t) {
      if (snx[t] == 0.0 && signbit(snx[t])) ++nz;
      else ++na;
    }
    sh_cnt[threadIdx.x] = na;
    sh_cnt[PT + threadIdx.x] = nz;
    __syncthreads();
    if (threadIdx.x == 0) {
      int sa = 0, sz = 0;
      for (int t = 0; t < PT; ++t) {
        const int ta = sh_cnt[t], tz = sh_cnt[PT + t];
        sh_cnt[t] = sa;
        sh_cnt[PT + t] = sz;
        sa += ta;
        sz += tz;
      }
      sh_nact = sa;
      sh_nzero = sz;
    }
    __syncthreads();
    int oa = sh_cnt[threadIdx.x], oz = sh_cnt[PT + threadIdx.x];
    for (int64_t t = b0; t < b1; ++t) {
      if (snx[t] == 0.0 && signbit(snx[t])) zlist[oz++] = (int)(c0 + t);
      else alist[oa++] = (int)(c0 + t);
    }
    __syncthreads();
  }

  // the CTA's best of (bv, bp) over its threads, the zero slots' offer at norm 0
  // included, into sh_cbv / sh_cbp (combined with the current values when `keep`)
  auto cta_best = [&](double bv, long long bp, bool keep) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (better(ov, op, bv, bp)) { bv = ov; bp = op; }
    }
    if (lane == 0) { sh_bv[warp] = bv; sh_bp[warp] = bp; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double cv = keep ? sh_cbv : -INFINITY;
      long long cp = keep ? sh_cbp : INT64_MAX;
      for (int w = 0; w < PW; ++w)
        if (better(sh_bv[w], sh_bp[w], cv, cp)) { cv = sh_bv[w]; cp = sh_bp[w]; }
      if (LIST && sh_nzero > 0 && sh_zkey != ~0ull && better(0.0, (long long)sh_zkey, cv, cp)) {
        cv = 0.0;
        cp = (long long)sh_zkey;
      }
      sh_cbv = cv;
      sh_cbp = cp;
    }
    __syncthreads();
  };
  // identically-zero slots: relabel (the one at logical position s takes p) and
  // offer the lowest logical position at norm 0
  auto zero_slots = [&](bool relabel, int s_, int p_) {
    if (!(LIST && sh_nzero > 0)) return;
    if (threadIdx.x == 0) sh_zkey = ~0ull;
    __syncthreads();
    unsigned long long zk = ~0ull;
    for (int t = threadIdx.x; t < sh_nzero; t += PT) {
      const int z = zlist[t] - (int)c0;
      if (snr[z] == -INFINITY) continue;
      int lp = spos[z];
      if (relabel && lp == s_) spos[z] = lp = p_;
      const unsigned long long key = ((unsigned long long)lp << 32) | (unsigned long long)(c0 + z);
      zk = key < zk ? key : zk;
    }
    if (zk != ~0ull) atomicMin(&sh_zkey, zk);
    __syncthreads();
  };
  // the step's evaluation list: active slots below level lvl with ub >= thr
  // (and, once per step, the relabelling of the slot at logical position s_)
  // the step's evaluation list: active slots below level lvl with ub >= thr
  // (and, once per step, the relabelling of the slot at logical position s_;
  // the slot sp_ being pivoted this step is skipped).  Run by warps w0..PW-1,
  // no block barrier (sh_ecnt zeroed by the caller before its last barrier).
  auto list_warps = [&](double thr, int lvl, bool relabel, int s_, int p_, int sp_, int w0) {
    if (warp < w0) return;
    const int nthr = PT - 32 * w0, tid = threadIdx.x - 32 * w0;
    const int cnt = sh_nact;
    for (int i0 = 0; i0 < cnt; i0 += nthr) {
      const int i = i0 + tid;
      bool take = false;
      int j = 0;
      if (i < cnt) {
        j = LIST ? alist[i] : (int)c0 + i;
        const int li = j - (int)c0;
        const double nr = snr[li];
        if (nr != -INFINITY && j != sp_) {
          if (relabel && spos[li] == s_) spos[li] = p_;
          take = scj[li] < lvl && nr + kLazyBoundEps * snx[li] >= thr;
        }
      }
      const unsigned mask = __ballot_sync(0xffffffffu, take);
      int basei = 0;
      if (lane == 0 && mask) basei = atomicAdd(&sh_ecnt, __popc(mask));
      basei = __shfl_sync(0xffffffffu, basei, 0);
      if (take) elist[basei + __popc(mask & ((1u << lane) - 1))] = j;
    }
  };
  auto build_list = [&](double thr, int lvl) {  // (retry rounds) every warp, with barriers
    if (threadIdx.x == 0) sh_ecnt = 0;
    __syncthreads();
    list_warps(thr, lvl, false, 0, 0, -1, 0);
    __syncthreads();
  };
  auto run_pass = [&](int lvl, double& bv, long long& bp) {
    LazyCtx x{a, lvl, elist, sh_ecnt, c0, warp, lane, Vs, swall, sM, snr, snx, spos, scj, 0ull};
    lazy_cols<TC0, NLD>(x, bv, bp);
    my_recomputes += x.recomputes;
    my_evals += (unsigned long long)sh_ecnt;
  };
  auto publish = [&](unsigned int e) {  // the CTA's candidate of round e: partial + staged reflector + tag
    if (threadIdx.x == 0) {
      a.pval[(int64_t)(e & 1) * G + cta] = sh_cbv;
      a.ppos[(int64_t)(e & 1) * G + cta] = sh_cbp;
    }
  };

  // ------------------------------------------------------------ candidates for step t0 (exact norms)
  {
    double bv = -INFINITY;
    long long bp = INT64_MAX;
    for (int i = threadIdx.x; i < sh_nact; i += PT) {
      const int j = LIST ? alist[i] : (int)c0 + i;
      const int li = j - (int)c0;
      const long long key = ((long long)spos[li] << 32) | (long long)j;
      if (snr[li] != -INFINITY && better(snr[li], key, bv, bp)) { bv = snr[li]; bp = key; }
    }
    zero_slots(false, 0, 0);
    cta_best(bv, bp, false);
    publish(ep);
    __syncthreads();
    grid_arrive(a.bar, bar_target);
    stage_candidate(a, a.cand + ((int64_t)(ep & 1) * G + cta) * cand_sz, a.t0, sh_cbp & 0xffffffffll, 0, false, Vs,
                    scr, fb, &sh_alpha, sh_red);
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ctag + cta), "r"(ep + 1u) : "memory");
    lazy_grid_wait(a.bar, bar_target, -1);
  }

  const bool tr = a.trace != nullptr && threadIdx.x == 0;
  unsigned long long tprev = tr ? gtimer() : 0;
  const unsigned long long tk0 = tprev, ck0 = tr ? clock64() : 0;
  auto stamp = [&](int slot) {
    if (tr) {
      const unsigned long long t = gtimer();
      a.trace[cta * 8 + slot] += t - tprev;
      tprev = t;
    }
  };
  double Lprev = -INFINITY;
  bool check = false;
  for (int64_t s = a.t0; s < a.t1; ++s) {
    const int c = (int)(s - a.t0);
    bool retried = false;
    for (;;) {
      // (1) global argmax over the per-CTA partials of round ep
      if (warp == 0) {
        const int par = (int)(ep & 1);
        double pv[kMaxG / 32];
        long long pp[kMaxG / 32];
#pragma unroll
        for (int r = 0; r < kMaxG / 32; ++r) {
          const int cc = lane + 32 * r;
          pv[r] = cc < G ? __ldcg(a.pval + (int64_t)par * G + cc) : -INFINITY;
          pp[r] = cc < G ? __ldcg(a.ppos + (int64_t)par * G + cc) : INT64_MAX;
        }
        double bv = pv[0];
        long long bp = pp[0];
        int bc = lane;
#pragma unroll
        for (int r = 1; r < kMaxG / 32; ++r)
          if (better(pv[r], pp[r], bv, bp)) { bv = pv[r]; bp = pp[r]; bc = lane + 32 * r; }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
          const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
          if (better(ov, op, bv, bp)) { bv = ov; bp = op; bc = oc; }
        }
        if (lane == 0) {
          sh_piv[0] = bp;
          sh_piv[1] = bc;
          sh_gbv = bv;  // (the winner's tag is awaited when its reflector is read, step 3a)
        }
      }
      __syncthreads();
      if (!(check && sh_gbv < Lprev)) break;
      // (1b) retry: the last pass skipped columns that may beat the best value it
      // found; evaluate them against that value (level c: through reflector c - 1)
      const double thr = sh_gbv;
      build_list(thr, c);
      double bv = -INFINITY;
      long long bp = INT64_MAX;
      run_pass(c, bv, bp);
      cta_best(bv, bp, true);
      publish(ep + 1);
      __syncthreads();
      grid_arrive(a.bar, bar_target);
      stage_candidate(a, a.cand + ((int64_t)((ep + 1) & 1) * G + cta) * cand_sz, s, sh_cbp & 0xffffffffll, c, c > 0,
                      Vs, scr, fb, &sh_alpha, sh_red);
      if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ctag + cta), "r"(ep + 2u) : "memory");
      lazy_grid_wait(a.bar, bar_target, s);
      ++ep;
      ++my_retries;
      retried = true;
      Lprev = thr;
    }
    const int64_t p = sh_piv[0] >> 32;
    const int64_t sp = sh_piv[0] & 0xffffffffll;
    const double Ms = sh_gbv;
    const double* cd = a.cand + ((int64_t)(ep & 1) * G + sh_piv[1]) * cand_sz;

    const bool owner = (sp >= c0 && sp < c1);
    const bool last = c == C - 1;  // last step of the panel: relabel only (panel_finalize_kernel applies it)
    // (2) threshold for the next pass, L = beta M_s.  A miss (the next maximum below L) costs a
    // retry round over everything skipped, a low beta costs extra columns every step, and where
    // the balance lies depends on the spectrum (C4: beta ~ 0.9, a Gaussian matrix: ~ 0.97).  beta
    // follows the retries: the gap 1 - beta shrinks 2% after a step without one and grows by
    // kLazyGapMiss after one, which settles near one retry in ~30 steps.
    if (threadIdx.x == 0) {
      if (check) sh_gap = fmin(kLazyGapMax, fmax(kLazyGapMin, retried ? sh_gap * (a.gap_miss > 1.0 ? a.gap_miss : kLazyGapMiss) : sh_gap * kLazyGapHit));
      const double beta = a.beta > 0.0 ? a.beta : 1.0 - sh_gap;
      sh_thr = last ? INFINITY : beta * Ms;
      sh_ecnt = 0;
      if (owner) {  // the pivot's slot leaves the active set (the reference's swap is a relabelling)
        snr[sp - c0] = -INFINITY;
        spos[sp - c0] = (int)s;
      }
    }
    __syncthreads();
    const double thr = sh_thr;
    if (warp == 0) {
      // (3a) the winner's reflector -> vv, Vs(:, c), w of this step, tau (after its tag)
      if (lane == 0) {
        lazy_tag_wait(a.ctag + sh_piv[1], ep + 1u, s);
      }
      __syncwarp();
      const double tau_b = __ldcg(cd + 2);
      const bool apply_b = __ldcg(cd + 3) != 0.0 && tau_b != 0.0;
      if (s > 0 && lane == 0) vv[s - 1] = 0.0;
      for (int64_t i = s + lane; i < m; i += 32) {
        const double vi = __ldcg(cd + kHdr + i);
        vv[i] = vi;
        Vs[c * ld + i] = apply_b ? vi : 0.0;
      }
      if (lane < kHdr) sh_hdr[lane] = __ldcg(cd + lane);
      swall[c * NB + lane] = lane < c ? __ldcg(cd + kHdr + ld + lane) : 0.0;
      if (lane == 0) stau[c] = apply_b ? tau_b : 0.0;
    } else {
      // (3b) meanwhile: relabel and the evaluation list (level c + 1, ub >= thr)
      list_warps(thr, c + 1, true, (int)s, (int)p, (int)sp, 1);
    }
    __syncthreads();
    if (threadIdx.x <= c) {  // row c of M: M(c, c) = tau_c, M(c, i) = -tau_c sum_{i<=t<c} w_c[t] M(t, i)
      const int i = threadIdx.x;
      double v = 0.0;
      for (int t = i; t < c; ++t) v = fma(swall[c * NB + t], sM[t * NBL + i], v);
      sM[c * NBL + i] = i == c ? stau[c] : -stau[c] * v;
    }
    __syncthreads();
    stamp(1);  // argmax + candidate loads + list
    if (cta == 0) {
      if (threadIdx.x == 0) a.tau[s] = stau[c];
      if (threadIdx.x < NB) a.wall[c * NB + threadIdx.x] = swall[c * NB + threadIdx.x];
    }
    if (!last) {
      zero_slots(true, (int)s, (int)p);
      double bv = -INFINITY;
      long long bp = INT64_MAX;
      run_pass(c + 1, bv, bp);
      stamp(2);  // pass
      cta_best(bv, bp, false);
      publish(ep + 1);
      if (owner) {  // the pivot slot: R(s, s) = beta, the reflector below; F row -> 0
        double* ps = a.W + sp * ld;
        const double beta = sh_hdr[1];
        for (int64_t i = s + threadIdx.x; i < m; i += PT) ps[i] = (sh_hdr[3] != 0.0 && i == s) ? beta : vv[i];
        if (threadIdx.x < NB) a.F[sp * NB + threadIdx.x] = 0.0;
      }
      if (cta == 0)
        for (int64_t i = threadIdx.x; i < ld; i += PT) a.Vg[i * NB + c] = Vs[c * ld + i];
      __syncthreads();
      stamp(3);  // CTA argmax, pivot write-back
      grid_arrive(a.bar, bar_target);
      stage_candidate(a, a.cand + ((int64_t)((ep + 1) & 1) * G + cta) * cand_sz, s + 1, sh_cbp & 0xffffffffll, c + 1,
                      true, Vs, scr, fb, &sh_alpha, sh_red);
      if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ctag + cta), "r"(ep + 2u) : "memory");
      stamp(4);  // stage
      lazy_grid_wait(a.bar, bar_target, s);
      stamp(5);  // grid barrier
      ++ep;
      Lprev = thr;
      check = true;
    } else {  // last step of the panel: relabel only; panel_finalize_kernel applies this reflector
      zero_slots(true, (int)s, (int)p);
      if (owner) {
        double* ps = a.W + sp * ld;
        const double beta = sh_hdr[1];
        for (int64_t i = s + threadIdx.x; i < m; i += PT) ps[i] = (sh_hdr[3] != 0.0 && i == s) ? beta : vv[i];
        if (threadIdx.x < NB) a.F[sp * NB + threadIdx.x] = 0.0;
      }
      if (cta == 0)
        for (int64_t i = threadIdx.x; i < ld; i += PT) a.Vg[i * NB + c] = Vs[c * ld + i];
      __syncthreads();
    }
  }
  for (int64_t j = c0 + threadIdx.x; j < c1; j += PT) {
    a.nrm[j] = snr[j - c0];
    a.nrmx[j] = snx[j - c0];
    a.posof[j] = spos[j - c0];
    a.cjg[j] = scj[j - c0];
  }
  if (cta == 0 && threadIdx.x == 0) {  // every CTA read the old values before the first barrier
    *a.epoch = ep + 1u;
    a.lstats[2] = (unsigned long long)__double_as_longlong(sh_gap);
  }
  if (tr) {
    a.trace[cta * 8 + 6] += clock64() - ck0;
    a.trace[cta * 8 + 7] += gtimer() - tk0;
  }
  const unsigned int wcount = __reduce_add_sync(0xffffffffu, (unsigned int)my_recomputes);
  if (lane == 0 && wcount) atomicAdd(a.recomputes, (unsigned long long)wcount);
  if (threadIdx.x == 0 && a.lstats) {
    atomicAdd(a.lstats + 1, my_evals);
    if (cta == 0) atomicAdd(a.lstats, my_retries);
  }
}

// End of a lazy panel [t0, t1): every active column catches up on the panel
// reflectors it has not seen (all of them for the columns no step evaluated),
// then (upd) rows t1..r1 get the rank-C update A_p -= V F^T.  One warp per
// 8-column group, on the DMMA pipe in the transposed forms
//   D^T (8 cols x 32) = A_p(t0:ld, cols)^T V        (dots v_c^T a_j)
//   W^T(cols, rows)  -= F(cols, 0:C) V(rows, 0:C)^T (update)
// in which a lane owns rows r0 + 2(lane & 3) + {0, 1} of column j0 + lane / 4
// (one 16-byte load) and D / F entries i = 8 nt + 2 (lane & 3) + e (the mma K
// index mapped onto rows, resp. reflectors, accordingly).  Between them, per
// column and missed step cc in order (the four lanes of a column reduce their
// F entries by two shuffles): F(j, cc) = tau_cc (D(cc) - F(j, <cc) w_cc),
// R(s_cc, j) = A_p(s_cc, j) - V(s_cc, <=cc) F(j, <=cc), nr -= R^2 and the exact
// recompute below 1e-6 nx (cpqr.hpp:68-84), as the step passes do.
constexpr int FU = 8;       // 8-row blocks in flight per lane


__global__ void __launch_bounds__(FW * 32, 1) panel_finalize_kernel(FinArgs f) {
  extern __shared__ double fsm[];
  const int64_t ld = f.ld, t0 = f.t0;
  const int nrow = (int)(ld - t0);
  const int vcs = nrow + 8;                  // Vc row stride (== 8 mod 16: conflict-free 16-byte loads)
  double* Vr = fsm;                          // [nrow][FVR]: V(t0 + r, i), reflector-contiguous
  double* Vc = Vr + (size_t)nrow * FVR;      // [NBL][vcs]: V(t0 + r, i), row-contiguous
  double* sw = Vc + (size_t)NBL * vcs;       // [NB][NB]
  double* st = sw + NB * NB;                 // [NB]
  {  // the panel's V from the row-major global copy, 16-byte loads, 4 in flight per thread
    const int tot = nrow * (NBL / 2);
    for (int e0 = threadIdx.x; e0 < tot; e0 += 4 * blockDim.x) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * blockDim.x;
        v[u] = e < tot ? __ldcg(reinterpret_cast<const double2*>(f.Vg + (t0 + e / (NBL / 2)) * NB) + e % (NBL / 2))
                       : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e >= tot) break;
        const int r = e / (NBL / 2), i = 2 * (e % (NBL / 2));
        const double x0 = i < f.C ? v[u].x : 0.0, x1 = i + 1 < f.C ? v[u].y : 0.0;
        *reinterpret_cast<double2*>(Vr + r * FVR + i) = make_double2(x0, x1);
        Vc[i * vcs + r] = x0;
        Vc[(i + 1) * vcs + r] = x1;
      }
    }
  }
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) sw[e] = f.wall[e];
  if (threadIdx.x < NB) st[threadIdx.x] = (int)threadIdx.x < f.C ? f.tau[threadIdx.x] : 0.0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane & 3, cg8 = lane >> 2;
  const int ntl = (f.C + 7) >> 3;  // 8-reflector tiles of this panel (<= 2)
  const int64_t ngroups = (f.n + 7) >> 3;
  unsigned long long rec = 0;
  for (int64_t gi = (int64_t)blockIdx.x * FW + warp; gi < ngroups; gi += (int64_t)gridDim.x * FW) {
    const int64_t j = gi * 8 + cg8;
    const bool colok = j < f.n;
    double nr = colok ? f.nrm[j] : -INFINITY;
    double nx = colok ? f.nrmx[j] : 0.0;
    const int cj = colok ? f.cj[j] : f.C;
    // pivoted slots (-inf) and identically-zero columns (nx = -0) take no update
    const bool active = colok && nr != -INFINITY && !(nx == 0.0 && signbit(nx)) && cj < f.C;
    if (!__any_sync(0xffffffffu, active)) continue;
    double* wc = f.W + (size_t)(colok ? j : 0) * ld;
    // A_p(t0 + cc, j) and F(j, <cj): issued before the dot-product loop
    double xap[NBL];
#pragma unroll
    for (int cc = 0; cc < NBL; ++cc) xap[cc] = (active && cc >= cj && cc < f.C) ? __ldcg(wc + t0 + cc) : 0.0;
    double fv[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = 8 * nt + 2 * q + e;
        fv[nt][e] = (active && i < cj) ? __ldcg(f.F + (size_t)j * NB + i) : 0.0;
      }
    // ---- D^T = A_p(t0:ld, cols)^T V (rows whose V entries are zero contribute 0)
    double dacc[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) dacc[nt][0] = dacc[nt][1] = 0.0;
    const int nb8 = nrow >> 3;
    for (int b0 = 0; b0 < nb8; b0 += FU) {
      double2 w2[FU];
#pragma unroll
      for (int u = 0; u < FU; ++u)
        w2[u] = (b0 + u < nb8 && active) ? __ldcg(reinterpret_cast<const double2*>(wc + t0 + 8 * (b0 + u) + 2 * q))
                                          : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < FU; ++u) {
        if (b0 + u >= nb8) break;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          if (nt >= ntl) break;
          const double2 vb = *reinterpret_cast<const double2*>(Vc + (8 * nt + cg8) * vcs + 8 * (b0 + u) + 2 * q);
          dmma_8x8x4(dacc[nt][0], dacc[nt][1], w2[u].x, vb.x);
          dmma_8x8x4(dacc[nt][0], dacc[nt][1], w2[u].y, vb.y);
        }
      }
    }
    // ---- per-column recurrence over the missed steps
    const int cmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)(active ? cj : f.C));
    for (int cc = cmin; cc < f.C; ++cc) {
      const bool act = active && cc >= cj;
      const int64_t sc = t0 + cc;
      const double* vrow = Vr + (size_t)cc * FVR;  // V(sc, :)
      double p0 = 0.0, p1 = 0.0, dsel = 0.0;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 8 * nt + 2 * q + e;
          p0 = fma(fv[nt][e], sw[cc * NB + i], p0);
          p1 = fma(fv[nt][e], vrow[i], p1);
          if (i == cc) dsel = dacc[nt][e];
        }
      p0 += __shfl_xor_sync(0xffffffffu, p0, 1);
      p0 += __shfl_xor_sync(0xffffffffu, p0, 2);
      p1 += __shfl_xor_sync(0xffffffffu, p1, 1);
      p1 += __shfl_xor_sync(0xffffffffu, p1, 2);
      const double d = __shfl_sync(0xffffffffu, dsel, (lane & ~3) | ((cc >> 1) & 3));
      const double tc = st[cc];
      const bool apply = tc != 0.0;
      const double fnew = apply ? tc * (d - p0) : 0.0;
      double xa = 0.0;
#pragma unroll
      for (int t = 0; t < NBL; ++t)
        if (t == cc) xa = xap[t];
      const double xs = xa - p1 - (apply ? 1.0 : 0.0) * fnew;
      const bool own = q == ((cc >> 1) & 3);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (act && own && 8 * nt + 2 * q + e == cc) fv[nt][e] = fnew;
      if (act && own) f.F[(size_t)j * NB + cc] = fnew;
      if (act && q == 0) wc[sc] = xs;
      double nn = nr - xs * xs;
      const bool need = act && nn < 1e-6 * nx;
      unsigned ball = __ballot_sync(0xffffffffu, need && q == 0);
      if (ball) {
        __syncwarp();
        while (ball) {  // exact trailing norms, one flagged column at a time by the whole warp
          const int g = (__ffs(ball) - 1) >> 2;
          ball &= ball - 1;
          const int64_t jg = gi * 8 + g;
          const double* col = f.W + (size_t)jg * ld;
          const double* Fj = f.F + (size_t)jg * NB;
          double acc = 0.0;
          for (int64_t r = sc + 1 + lane; r < f.m; r += 32) {
            double xv = __ldcg(col + r);
            for (int i = 0; i <= cc; ++i) xv = fma(-Vr[(size_t)(r - t0) * FVR + i], __ldcg(Fj + i), xv);
            acc = fma(xv, xv, acc);
          }
          acc = warp_sum(acc);
          if (cg8 == g) {
            nn = acc;
            nx = acc;
          }
          if (lane == 0) ++rec;
        }
      }
      if (act) nr = nn;
    }
    if (active && q == 0) {
      f.nrm[j] = nr;
      f.nrmx[j] = nx;
    }
    // ---- update rows t1..r1: W^T(cols, rows) += (-F)(cols, refl) V(rows, refl)^T
    if (f.upd) {
      const int u0 = (int)(f.t1 - t0) >> 3, u1 = (int)(f.r1 - t0) >> 3;
      for (int b0 = u0; b0 < u1; b0 += FU) {
        double2 w2[FU];
#pragma unroll
        for (int u = 0; u < FU; ++u)
          w2[u] = (b0 + u < u1 && active) ? __ldcg(reinterpret_cast<const double2*>(wc + t0 + 8 * (b0 + u) + 2 * q))
                                           : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < FU; ++u) {
          if (b0 + u >= u1) break;
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            if (nt >= ntl) break;
            const double2 vb = *reinterpret_cast<const double2*>(Vr + (size_t)(8 * (b0 + u) + cg8) * FVR + 8 * nt + 2 * q);
            dmma_8x8x4(w2[u].x, w2[u].y, -fv[nt][0], vb.x);
            dmma_8x8x4(w2[u].x, w2[u].y, -fv[nt][1], vb.y);
          }
        }
#pragma unroll
        for (int u = 0; u < FU; ++u)
          if (b0 + u < u1 && active) *reinterpret_cast<double2*>(wc + t0 + 8 * (b0 + u) + 2 * q) = w2[u];
      }
    }
  }
  const unsigned int wcount = __reduce_add_sync(0xffffffffu, (unsigned int)rec);
  if (lane == 0 && wcount) atomicAdd(f.recomputes, (unsigned long long)wcount);
}

}  // namespace

PanelKernT lazy_kernel_for(int nld, int tc, bool list) {
#define LRB_LAZY_K(L)                                                                                       \
  {cpqr_lazy_kernel<0, 4, L>, cpqr_lazy_kernel<1, 4, L>, cpqr_lazy_kernel<2, 4, L>, cpqr_lazy_kernel<3, 4, L>}, \
      {cpqr_lazy_kernel<0, 5, L>, cpqr_lazy_kernel<1, 5, L>, cpqr_lazy_kernel<2, 5, L>,                       \
       cpqr_lazy_kernel<3, 5, L>, cpqr_lazy_kernel<4, 5, L>},                                                  \
      {cpqr_lazy_kernel<0, 8, L>, cpqr_lazy_kernel<1, 8, L>, cpqr_lazy_kernel<2, 8, L>,                       \
       cpqr_lazy_kernel<3, 8, L>, cpqr_lazy_kernel<4, 8, L>, cpqr_lazy_kernel<5, 8, L>,                       \
       cpqr_lazy_kernel<6, 8, L>, cpqr_lazy_kernel<7, 8, L>}
  struct KernSet {
    PanelKernT k4[4], k5[5], k8[8];
  };
  static const KernSet lz[2] = {{LRB_LAZY_K(false)}, {LRB_LAZY_K(true)}};
#undef LRB_LAZY_K
  const KernSet& k = lz[list ? 1 : 0];
  if (nld == 8) return k.k8[tc];
  if (nld == 5) return k.k5[tc];
  if (nld == 4) return k.k4[tc];
  return nullptr;
}

void lazy_set_attributes() {
  for (int l = 0; l < 2; ++l)
    for (int nld : {4, 5, 8})
      for (int tc = 0; tc < nld; ++tc) {
        PanelKernT kf = lazy_kernel_for(nld, tc, l == 1);
        cudaFuncAttributes fa{};
        LRB_CUDA(cudaFuncGetAttributes(&fa, kf));
        LRB_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(227 * 1024 - fa.sharedSizeBytes)));
      }
  LRB_CUDA(cudaFuncSetAttribute(panel_finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)finalize_smem_bytes(512, 0)));
}

void launch_panel_finalize(const FinArgs& f, int grid, cudaStream_t st) {
  panel_finalize_kernel<<<grid, FW * 32, finalize_smem_bytes(f.ld, f.t0), st>>>(f);
  LRB_CHECK_LAUNCH();
}

}  // namespace cpqr_detail
}  // namespace lrb
