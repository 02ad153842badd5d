// cpqr_panel.cu -- truncated column-pivoted Householder QR with delayed
// (panel) trailing updates, for the short-wide working matrices of the path
// (the sketch Y and C^T: m <= 512 rows, tens of thousands of columns).
//
// Same observable semantics as cpqr.hpp:32-114 (and as cpqr.cu): first
// maximum of the running squared norms (ties -> lowest position), full column
// swaps, reflector beta = -sign(alpha)|x|, tau = (beta-alpha)/beta,
// v = x/(alpha-beta), downdate norm2 -= R(s,j)^2 and exact recompute below
// 1e-6 of the last exact value.  Only the order of the floating-point work
// differs (roundoff-level, like any reordering of the right-looking update).
//
// Why: the right-looking kernel streams the trailing matrix in AND out every
// step.  Here the reflectors of a panel of NB steps are accumulated in the
// compact form  A_cur = A_p - V F^T  (A_p: the matrix at panel start,
// F = A_p^T V T built one column per step as in LAPACK's xLAQPS):
//   per step, per trailing column j (one read of A_p(s:m, j), no write):
//     F(j, c)   = tau (A_p(s:m, j)^T v - sum_{i<c} F(j, i) w_i),  w = V^T v
//     R(s, j)   = A_p(s, j) - sum_{i<=c} V(s, i) F(j, i)          (row s only)
//     norm2(j) -= R(s, j)^2  (exact recompute from A_p - V F^T when flagged)
//   per panel: A_p(s1:m, :) -= V(s1:m, :) F(:, :)^T (panel_update_dmma_kernel).
// HBM traffic per step is one read of the trailing block (half of the
// right-looking pass) plus 256 B of F per column; the panel update is one
// read+write every NB steps.
//
// Column swaps are logical: a column keeps its slot (and its CTA) for the
// whole factorization; each slot carries its logical position (the position
// the reference's swaps would have moved it to; ties in the argmax go to the
// lowest logical position) and a pivoted slot leaves the active set (norm
// -inf, F row 0).  No step waits on a column move; one permutation pass at
// the end puts the <= 2k displaced columns at their positions.
//
// Structure per panel: ONE persistent cooperative launch for the NB steps
// (per step: batched argmax of per-CTA partials -> the winner's staged
// reflector -> fused pass over owned columns -> per-CTA argmax + staging of
// the CTA's best column's reflector for the next step -> one grid barrier),
// then panel_update_dmma_kernel for the block update.
#include <cooperative_groups.h>
#include <chrono>
#include <cstdio>
#include <vector>
#include <algorithm>

#include "cpqr_panel.cuh"

namespace cg = cooperative_groups;

namespace lrb {

namespace cpqr_detail {
namespace {

struct Col {
  double c[CH][2];
  double f;   // F(j, lane) (lane < c), 0 otherwise
  double nr, nx;
};

// state of one step's pass, shared by every column of a warp
struct PassCtx {
  const PanelArgs& a;
  int64_t s;
  int c;
  int64_t p;             // logical position of this step's pivot (the column at position s moves there)
  bool apply;
  double tau, vr_c;
  int64_t c0, cnt;       // cnt: active slots of the CTA (alist)
  int warp, lane;
  const double* vv;
  const double* Vs;
  const double* wsh;     // w = V^T v (NB)
  const double* vrow;    // V(s, 0:NB)
  double* snr;           // this CTA's running / last exact squared norms (shared memory, index j - c0)
  double* snx;
  int* spos;             // logical positions of the owned slots (shared memory, index j - c0)
  const int* alist;      // the CTA's slots that are not identically zero, ascending; null: all of them
  unsigned long long recomputes;
};



// One step's pass over a warp's column slots (pivoted slots: loads only).
// TC0 = first active 64-row chunk (s / 64, constant over a 32-step panel),
// NLD = ld / 64; TC0 = -1: runtime chunk range.
// Specialised layout: a column is handled by a group of L lanes (16 for 5-8
// active 64-row chunks, 8 for 2-4, 4 for one), 32 / L columns per warp
// instruction; lane l of a group holds rows base + 2(l + L k) + {0, 1},
// k < KP (<= 16 row pairs), and F(j, l S .. l S + S - 1) (S = NB / L).  The
// pass is latency-bound per warp (load -> dot -> log2(L)-round reduction ->
// norm), so several columns per instruction buy memory-level parallelism:
// 16 lanes instead of 32 on the early panels took the CPQR of Y from 19.4 to
// 16.9 ms.
template <int TC0, int NLD, bool LIST>
__device__ __forceinline__ void pass_cols(PassCtx& x, double& bv, long long& bp) {
  constexpr bool SPEC = TC0 >= 0;
  constexpr int NA = SPEC ? NLD - TC0 : CH;
  // lanes per column: a power of two with at most 16 row pairs per lane
  constexpr int L = !SPEC ? 32 : (NA >= 5 ? 16 : (NA >= 2 ? 8 : 4));
  constexpr int KP = SPEC ? 32 * NA / L : CH;  // row pairs per lane
  constexpr int GPW = 32 / L;
  constexpr int S = NB / L;
  constexpr int D = S == 1 ? 4 : (S <= 2 ? (KP > 8 ? 2 : 3) : 2);  // warp-iterations in flight
  const PanelArgs& a = x.a;
  const int64_t s = x.s, ld = a.ld, m = a.m;
  const int lane = x.lane, c = x.c;
  const int l = lane & (L - 1), g = lane / L;
  const int gbase = lane & ~(L - 1);
  const int tc0 = SPEC ? TC0 : (int)(s >> 6);
  const int nld = SPEC ? NLD : (int)(ld >> 6);
  const int base = SPEC ? 64 * TC0 : 0;
  // rows of this lane: base + 2(l + L k) + e; the generic layout (L = 32) keeps
  // chunk k at rows 64k + 2 lane and predicates k in [tc0, nld)
  auto active = [&](int k) { return SPEC ? k < KP : (k >= tc0 && k < nld); };
  const int rel = (int)(s - base);
  const int kk_s = rel / (2 * L), lo_s = (rel >> 1) & (L - 1), e_s = rel & 1;
  // per-lane slices of w and V(s, :)
  double wl[S], vl[S];
#pragma unroll
  for (int t = 0; t < S; ++t) {
    wl[t] = x.wsh[l * S + t];
    vl[t] = x.vrow[l * S + t];
  }
  const int lc = c / S, tcs = c % S;  // owner lane / slot of F(j, c)
  // the warp's slots c0 + warp + PW q (or, with identically-zero slots
  // present, alist[warp + PW q]), visited in alternating direction (the
  // previous step's last columns are L2-hot; 32-bit indices, n < 2^31)
  const int first = (int)(x.c0 + x.warp);
  const int n_valid = ((int)x.cnt - x.warp + PW - 1) / PW;
  const int jstart = (s & 1) ? first + PW * (n_valid - 1) : first;
  const int dj = (s & 1) ? -PW : PW;
  const double* Wb = a.W + base + 2 * l;
  const double* Fb = a.F + l * S;
  struct Slot {
    double c[KP][2];
    double f[S];
    double nr, nx;
    int j, lp;
    bool ok;
  };
  const int keep_from = n_valid - (int)(((long long)n_valid * a.keep1024) >> 10);
  const uint64_t pol_keep = l2_policy(true), pol_stream = l2_policy(false);
  auto fetch = [&](Slot& cb, int qi) {
    const int q = qi * GPW + g;
    cb.ok = q < n_valid;
    // an owned column for the (unused) loads of an idle lane group
    cb.j = jstart + dj * (cb.ok ? q : 0);
    if constexpr (LIST) cb.j = cb.ok ? x.alist[cb.j - (int)x.c0] : (int)x.c0;
    const double* src = Wb + (size_t)cb.j * (size_t)ld;
    const uint64_t pol = q >= keep_from ? pol_keep : pol_stream;
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (active(k)) {
        const double2 xx = ld_l2hint(reinterpret_cast<const double2*>(src + 2 * L * k), pol);
        cb.c[k][0] = xx.x;
        cb.c[k][1] = xx.y;
      }
    const double* fr = Fb + (size_t)cb.j * NB;
#pragma unroll
    for (int t = 0; t < S; ++t) cb.f[t] = (l * S + t < c) ? fr[t] : 0.0;
    cb.nr = x.snr[cb.j - x.c0];
    cb.nx = x.snx[cb.j - x.c0];
    cb.lp = x.spos[cb.j - x.c0];
    if (cb.nr == -INFINITY) cb.ok = false;  // pivoted slot (its rows hold R / reflector values)
  };
  const double2* v2 = reinterpret_cast<const double2*>(x.vv + base);
  auto process = [&](Slot& cb) {
    double d0 = 0.0, d1 = 0.0, xs = 0.0;
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (active(k)) {
        const double2 vx = v2[l + L * k];
        d0 = fma(cb.c[k][0], vx.x, d0);
        d1 = fma(cb.c[k][1], vx.y, d1);
        if (k == kk_s) xs = e_s ? cb.c[k][1] : cb.c[k][0];
      }
    double e0 = d0 + d1, e1 = 0.0;
#pragma unroll
    for (int t = 0; t < S; ++t) {
      e0 = fma(-cb.f[t], wl[t], e0);
      e1 = fma(cb.f[t], vl[t], e1);
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) {
      e0 += __shfl_xor_sync(0xffffffffu, e0, o);
      e1 += __shfl_xor_sync(0xffffffffu, e1, o);
    }
    const double fnew = x.apply ? x.tau * e0 : 0.0;
    // R(s, j) = A_p(s, j) - sum_{i<c} V(s,i) F(j,i) - V(s,c) F(j,c)
    xs = __shfl_sync(0xffffffffu, xs, gbase | lo_s);
    xs = xs - e1 - x.vr_c * fnew;
    const int j = cb.j;
    if (cb.ok && l == lo_s) a.W[(size_t)j * ld + s] = xs;
    if (cb.ok && l == lc) a.F[(size_t)j * NB + c] = fnew;
#pragma unroll
    for (int t = 0; t < S; ++t)
      if (l == lc && t == tcs) cb.f[t] = fnew;
    double nr = cb.nr - xs * xs;
    double nx = cb.nx;
    const bool need = cb.ok && nr < 1e-6 * nx;
    if (__any_sync(0xffffffffu, need)) {  // rare: exact norm from A_p - V F^T (L2-hot re-read)
      __syncwarp();
      const double qq = group_recompute<L>(a.W + (size_t)j * ld, a.F + (size_t)j * NB, s, m, ld, c, x.Vs, l);
      if (need) {
        nr = qq;
        nx = qq;
        if (l == 0) ++x.recomputes;  // one count per column (its group leader)
      }
    }
    if (cb.ok) {
      // the column at logical position s takes the pivot's position p (the reference's swap)
      const int lp = cb.lp == (int)s ? (int)x.p : cb.lp;
      if (l == 0) {
        x.snr[j - x.c0] = nr;
        x.snx[j - x.c0] = nx;
        x.spos[j - x.c0] = lp;
      }
      const long long key = ((long long)lp << 32) | (long long)j;  // ties -> lowest logical position
      if (better(nr, key, bv, bp)) { bv = nr; bp = key; }
    }
  };
  const int iters = (n_valid + GPW - 1) / GPW;
  Slot buf[D];
#pragma unroll
  for (int u = 0; u < D - 1; ++u)
    if (u < iters) fetch(buf[u], u);
  for (int q0 = 0; q0 < iters; q0 += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int q = q0 + u;
      if (q >= iters) break;
      if (q + D - 1 < iters) fetch(buf[(u + D - 1) % D], q + D - 1);
      process(buf[u]);
    }
  }
  // per-lane best -> warp best (the caller publishes lane 0's)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
    if (better(ov, op, bv, bp)) { bv = ov; bp = op; }
  }
}

// TC0 / NLD: the panel's first active 64-row chunk (t0 / 64; a 32-step panel
// never crosses a chunk) and ld / 64, or -1 for the generic runtime version
// LIST: identically-zero slots may exist (they leave the pass; one launch with
// LIST = true finds out, see cpqr_panel)
template <int TC0, int NLD, bool LIST>
__global__ void __launch_bounds__(PT, 1) cpqr_panel_kernel(PanelArgs a) {
  unsigned int bar_target = 0;
  extern __shared__ double dyn[];
  __shared__ double sh_red[PW];
  __shared__ double sh_bv[PW];
  __shared__ long long sh_bp[PW];
  __shared__ double sh_hdr[kHdr];
  __shared__ long long sh_piv[2];
  __shared__ double wsh[NB];    // w = V^T v of the current step
  __shared__ double vrow[NB];   // V(s, 0:NB)
  __shared__ double fb[NB];     // F row of the staged candidate column
  __shared__ double sh_alpha;
  __shared__ int sh_cnt[2 * PT];
  __shared__ int sh_nact, sh_nzero;
  __shared__ unsigned long long sh_zkey;

  const int G = gridDim.x, cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = a.m, n = a.n, ld = a.ld;
  const int64_t c0 = n * cta / G, c1 = n * (cta + 1) / G;
  const int64_t cand_sz = kHdr + ld + NB;
  const int nld = (int)(ld >> 6);
  double* vv = dyn;              // [ld] current reflector, zero outside [s, m)
  double* Vs = dyn + ld;         // [NB][ld] panel reflectors (column-major, zero outside support)
  double* scr = Vs + NB * ld;    // [ld] staging scratch
  double* snr = scr + ld;        // [maxcols] norms of the owned slots for this launch
  double* snx = snr + a.maxcols;
  int* spos = reinterpret_cast<int*>(snx + a.maxcols);  // [maxcols] their logical positions
  int* alist = spos + a.maxcols;  // active slots of this launch
  int* zlist = alist + a.maxcols;  // identically-zero slots (skipped by the pass)
  for (int64_t i = threadIdx.x; i < (NB + 2) * ld; i += PT) dyn[i] = 0.0;
  unsigned long long my_recomputes = 0;
  __syncthreads();

  // candidate staging: reflector of column b for step s1 from A_p - V F^T
  // (c_used = number of panel reflectors already applied); w = V^T v when the
  // next step continues this panel
  auto stage = [&](double* cd, int64_t s1, long long b, int c_used, bool same_panel) {
    if (b >= n || s1 >= m) {
      __syncthreads();
      return;
    }
    const double* x = a.W + b * ld;
    double xl[kRowsPerThread];  // issued before the F row is published
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
      const int64_t r = threadIdx.x + PT * q;
      xl[q] = (r >= s1 && r < m) ? x[r] : 0.0;
    }
    if (threadIdx.x < NB) fb[threadIdx.x] = threadIdx.x < c_used ? a.F[b * NB + threadIdx.x] : 0.0;
    __syncthreads();
    // rows r = threadIdx.x + PT * q (ld <= 512 <= 2 PT)
    double xr[kRowsPerThread];
    double part = 0.0;
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
      const int64_t r = threadIdx.x + PT * q;
      xr[q] = 0.0;
      if (r >= s1 && r < m) {
        // four independent chains over the panel's reflectors (latency)
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
        if (r == s1) sh_alpha = v;
      }
      part = fma(xr[q], xr[q], part);
    }
    const double cn2 = cta_sum(part, sh_red);  // (its barriers publish sh_alpha)
    const double colnorm = sqrt(cn2);
    const double alpha = sh_alpha;
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
    // w_i = V(:, i)^T v for the reflectors of this panel (warp i, i < c_used)
    if (same_panel) {
      double* vtmp = scr;
#pragma unroll
      for (int q = 0; q < kRowsPerThread; ++q)
        if (threadIdx.x + PT * q < ld) vtmp[threadIdx.x + PT * q] = vr[q];
      __syncthreads();
      static_assert(NB == 4 * PW, "four reflectors per warp");
      double acc[4] = {0.0, 0.0, 0.0, 0.0};  // reflectors warp + PW t, interleaved
      for (int64_t rr = s1 + lane; rr < m; rr += 32) {
        const double vt = vtmp[rr];
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
  };

  // ------------------------------------------------------------ init (first launch)
  if (a.init) {
    double bv = -INFINITY;
    long long bp = INT64_MAX;
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
        a.F[j * NB + lane] = 0.0;  // its panel updates are no-ops
        if (lane == 0) atomicAdd(a.nzero, 1);
      }
      const long long key = (j << 32) | j;
      if (better(acc, key, bv, bp)) { bv = acc; bp = key; }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(a.flags, 1);
    if (lane == 0) { sh_bv[warp] = bv; sh_bp[warp] = bp; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double cv = sh_bv[0];
      long long cp = sh_bp[0];
      for (int w = 1; w < PW; ++w)
        if (better(sh_bv[w], sh_bp[w], cv, cp)) { cv = sh_bv[w]; cp = sh_bp[w]; }
      a.pval[cta] = cv;  // parity 0 = step 0
      a.ppos[cta] = cp;
      sh_piv[0] = cp;
    }
    __syncthreads();
    stage(a.cand + (int64_t)cta * cand_sz, 0, sh_piv[0] & 0xffffffffll, 0, false);
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ctag + cta), "r"(1u) : "memory");
    grid_barrier(a.bar, bar_target);
    if (__ldcg(a.flags) != 0) return;
  }
  // the owned columns' norms live in shared memory for this launch
  for (int64_t j = c0 + threadIdx.x; j < c1; j += PT) {
    snr[j - c0] = __ldcg(a.nrm + j);
    snx[j - c0] = __ldcg(a.nrmx + j);
    spos[j - c0] = __ldcg(a.posof + j);
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
  if (a.entry) {  // first eager launch after lazy panels: exact norms, no candidate staged yet
    double bv = -INFINITY;
    long long bp = INT64_MAX;
    for (int i = threadIdx.x; i < sh_nact; i += PT) {
      const int j = LIST ? alist[i] : (int)c0 + i;
      const int li = j - (int)c0;
      const long long key = ((long long)spos[li] << 32) | (long long)j;
      if (snr[li] != -INFINITY && better(snr[li], key, bv, bp)) { bv = snr[li]; bp = key; }
    }
    if (threadIdx.x == 0) sh_zkey = ~0ull;
    __syncthreads();
    if (LIST) {  // the lowest logical position among the live zero slots competes at norm 0
      unsigned long long zk = ~0ull;
      for (int t = threadIdx.x; t < sh_nzero; t += PT) {
        const int z = zlist[t] - (int)c0;
        if (snr[z] == -INFINITY) continue;
        const unsigned long long key = ((unsigned long long)spos[z] << 32) | (unsigned long long)(c0 + z);
        zk = key < zk ? key : zk;
      }
      if (zk != ~0ull) atomicMin(&sh_zkey, zk);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (better(ov, op, bv, bp)) { bv = ov; bp = op; }
    }
    if (lane == 0) { sh_bv[warp] = bv; sh_bp[warp] = bp; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double cv = sh_bv[0];
      long long cp = sh_bp[0];
      for (int w = 1; w < PW; ++w)
        if (better(sh_bv[w], sh_bp[w], cv, cp)) { cv = sh_bv[w]; cp = sh_bp[w]; }
      if (LIST && sh_zkey != ~0ull && better(0.0, (long long)sh_zkey, cv, cp)) {
        cv = 0.0;
        cp = (long long)sh_zkey;
      }
      a.pval[(a.t0 & 1) * G + cta] = cv;
      a.ppos[(a.t0 & 1) * G + cta] = cp;
      sh_piv[0] = cp;
    }
    __syncthreads();
    stage(a.cand + ((a.t0 & 1) * G + cta) * cand_sz, a.t0, sh_piv[0] & 0xffffffffll, 0, false);
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ctag + cta), "r"((unsigned int)(a.t0 + 1)) : "memory");
    grid_barrier(a.bar, bar_target);
  }

  // ------------------------------------------------------------ steps of this panel
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
  for (int64_t s = a.t0; s < a.t1; ++s) {
    const int c = (int)(s - a.t0);  // panel column of this step's reflector
    const int par = (int)(s & 1), nxt = par ^ 1;
    // (1) global argmax over the per-CTA partials
    if (warp == 0) {
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
        // the winner stages its reflector after arriving at the barrier: wait for its tag
        unsigned int t;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(t) : "l"(a.ctag + bc) : "memory");
        } while (!tag_ready(t, (unsigned int)(s + 1)));
      }
    }
    __syncthreads();
    const int64_t p = sh_piv[0] >> 32;            // logical position of the pivot
    const int64_t sp = sh_piv[0] & 0xffffffffll;  // its slot
    const double* cd = a.cand + ((int64_t)par * G + sh_piv[1]) * cand_sz;

    // (2) the winner's reflector -> vv, Vs(:, c), w, V(s, :)
    {
      const double tau_b = __ldcg(cd + 2);
      const bool apply_b = __ldcg(cd + 3) != 0.0;
      if (s > 0 && threadIdx.x == 0) vv[s - 1] = 0.0;
      for (int64_t i = s + threadIdx.x; i < m; i += PT) {
        const double vi = __ldcg(cd + kHdr + i);
        vv[i] = vi;
        Vs[c * ld + i] = (apply_b && tau_b != 0.0) ? vi : 0.0;
      }
      if (threadIdx.x < kHdr) sh_hdr[threadIdx.x] = __ldcg(cd + threadIdx.x);
      if (threadIdx.x < NB) wsh[threadIdx.x] = threadIdx.x < c ? __ldcg(cd + kHdr + ld + threadIdx.x) : 0.0;
      // V(s, 0:c) of the earlier reflectors (V(s, c) = 1 when applied: vr_c below)
      if (threadIdx.x < NB) vrow[threadIdx.x] = threadIdx.x < c ? Vs[threadIdx.x * ld + s] : 0.0;
    }
    // (3) the pivot's slot leaves the active set (its norm -> -inf; no data moves:
    // the reference's column swap is the relabelling s <-> p of logical positions)
    const bool owner = (sp >= c0 && sp < c1);
    if (owner && threadIdx.x == 0) {
      snr[sp - c0] = -INFINITY;
      spos[sp - c0] = (int)s;
    }
    __syncthreads();
    if (tr && a.tstep) a.tstep[(s * G + cta) * 4 + 1] = gtimer();
    stamp(1);  // argmax + candidate / swap loads
    const double tau = sh_hdr[2];
    const bool apply = sh_hdr[3] != 0.0 && tau != 0.0;
    if (cta == 0 && threadIdx.x == 0) a.tau[s] = tau;
    const double vr_c = apply ? 1.0 : 0.0;  // V(s, c)

    // (4) fused pass over owned positions j in (s, n): read-only except row s and F(j, c)
    double bv = -INFINITY;
    long long bp = INT64_MAX;
    {
      PassCtx x{a,    s,    c,     p,    apply, tau,  vr_c, c0,   sh_nact, warp, lane,
                vv,   Vs,   wsh,   vrow, snr,   snx,  spos, alist, 0ull};
      pass_cols<TC0, NLD, LIST>(x, bv, bp);
      my_recomputes += x.recomputes;
    }

    if (tr && a.tstep) a.tstep[(s * G + cta) * 4 + 2] = gtimer();
    // identically-zero slots: the one at logical position s takes p; the lowest
    // logical position among them is this CTA's candidate at norm 0
    if (LIST && sh_nzero > 0) {
      if (threadIdx.x == 0) sh_zkey = ~0ull;
      __syncthreads();
      unsigned long long zk = ~0ull;
      for (int t = threadIdx.x; t < sh_nzero; t += PT) {
        const int z = zlist[t] - (int)c0;
        if (snr[z] == -INFINITY) continue;  // pivoted (only once every other column is exhausted)
        int lp = spos[z];
        if (lp == (int)s) spos[z] = lp = (int)p;
        const unsigned long long key = ((unsigned long long)lp << 32) | (unsigned long long)(c0 + z);
        zk = key < zk ? key : zk;
      }
      if (zk != ~0ull) atomicMin(&sh_zkey, zk);
    }
    stamp(2);  // pass
    // (5) CTA argmax, pivot column write-back, V row-major copy for the panel GEMM
    if (lane == 0) { sh_bv[warp] = bv; sh_bp[warp] = bp; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double cv = sh_bv[0];
      long long cp = sh_bp[0];
      for (int w = 1; w < PW; ++w)
        if (better(sh_bv[w], sh_bp[w], cv, cp)) { cv = sh_bv[w]; cp = sh_bp[w]; }
      if (LIST && sh_nzero > 0 && sh_zkey != ~0ull && better(0.0, (long long)sh_zkey, cv, cp)) {
        cv = 0.0;
        cp = (long long)sh_zkey;
      }
      a.pval[(int64_t)nxt * G + cta] = cv;
      a.ppos[(int64_t)nxt * G + cta] = cp;
      sh_piv[0] = cp;
    }
    if (owner) {  // the pivot slot: R(s, s) = beta, the reflector below; F row -> 0 (panel update no-op)
      double* ps = a.W + sp * ld;
      const double beta = sh_hdr[1];
      for (int64_t i = s + threadIdx.x; i < m; i += PT) ps[i] = (sh_hdr[3] != 0.0 && i == s) ? beta : vv[i];
      if (threadIdx.x < NB) a.F[sp * NB + threadIdx.x] = 0.0;
    }
    if (cta == 0)
      for (int64_t i = threadIdx.x; i < ld; i += PT) a.Vg[i * NB + c] = Vs[c * ld + i];
    __syncthreads();
    stamp(3);  // CTA argmax, pivot write-back
    // publish the partial, then stage the next candidate while the other CTAs
    // finish (the candidate is published by its own tag, not by the barrier)
    grid_arrive(a.bar, bar_target);
    if (s + 1 < a.k) {
      stage(a.cand + ((int64_t)nxt * G + cta) * cand_sz, s + 1, sh_piv[0] & 0xffffffffll, c + 1, s + 1 < a.t1);
      if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ctag + cta), "r"((unsigned int)(s + 2))
                     : "memory");
    }
    stamp(4);  // stage
    if (tr && a.tstep) a.tstep[(s * G + cta) * 4 + 3] = (gtimer() & ~3ull) | (owner ? 1 : 0);
    grid_wait(a.bar, bar_target);
    if (tr && a.tstep && s + 1 < a.k) a.tstep[((s + 1) * G + cta) * 4] = gtimer();
    stamp(5);  // grid barrier
  }
  // the owned slots' state back to global for the next launch / the final permutation
  for (int64_t j = c0 + threadIdx.x; j < c1; j += PT) {
    a.nrm[j] = snr[j - c0];
    a.nrmx[j] = snx[j - c0];
    a.posof[j] = spos[j - c0];
  }
  if (tr) {  // SM clock over this launch: cycles / ns
    a.trace[cta * 8 + 6] += clock64() - ck0;
    a.trace[cta * 8 + 7] += gtimer() - tk0;
  }
  // every group leader of the warp holds its columns' count
  const unsigned int wcount = __reduce_add_sync(0xffffffffu, (unsigned int)my_recomputes);
  if (lane == 0 && wcount) atomicAdd(a.recomputes, (unsigned long long)wcount);
}

// Panel update on the DMMA pipe: W(r0:r1, :) -= V(r0:r1, 0:nc) F(:, 0:nc)^T as
// m8n8k4 tiles with the W tile itself as the accumulator.  A warp owns an
// 8-column group and walks the 8-row blocks; -V's A fragments are pre-swizzled
// in shared memory ([row block][k step][lane]), F's B fragments sit in
// registers, and U row blocks of W are loaded before any is multiplied.
constexpr int PUW = 16;  // warps per CTA
constexpr int PUU = 8;   // row blocks in flight per warp
__global__ void __launch_bounds__(PUW * 32, 1)
    panel_update_dmma_kernel(double* __restrict__ W, int64_t ld, int64_t r0, int64_t r1, int64_t n,
                             const double* __restrict__ Vg, const double* __restrict__ F, int nc) {
  extern __shared__ double vfrag[];
  const int nrb = (int)((r1 - r0) >> 3);
  for (int e = threadIdx.x; e < nrb * 256; e += blockDim.x) {
    const int rb = e >> 8, ks = (e >> 5) & 7, ln = e & 31;
    const int kc = 4 * ks + (ln & 3);
    vfrag[e] = kc < nc ? -Vg[(r0 + 8 * rb + (ln >> 2)) * NB + kc] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ngroups = (n + 7) >> 3;
  for (int64_t gi = (int64_t)blockIdx.x * PUW + warp; gi < ngroups; gi += (int64_t)gridDim.x * PUW) {
    const int64_t j0 = gi * 8;
    double b[8];
    const int64_t jb = j0 + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int kc = 4 * ks + (lane & 3);
      b[ks] = (jb < n && kc < nc) ? __ldg(F + jb * NB + kc) : 0.0;
    }
    // F rows all zero (pivoted or identically-zero columns): the update is a no-op
    bool nz = false;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) nz |= b[ks] != 0.0;
    if (!__any_sync(0xffffffffu, nz)) continue;
    const int64_t jc = j0 + 2 * (lane & 3);
    const bool v0 = jc < n, v1 = jc + 1 < n;
    double* w0 = W + jc * ld + r0 + (lane >> 2);
    double* w1 = w0 + ld;
    for (int rb0 = 0; rb0 < nrb; rb0 += PUU) {
      double c[PUU][2];
#pragma unroll
      for (int u = 0; u < PUU; ++u) {
        const bool ok = rb0 + u < nrb;
        c[u][0] = (ok && v0) ? __ldcs(w0 + 8 * (rb0 + u)) : 0.0;
        c[u][1] = (ok && v1) ? __ldcs(w1 + 8 * (rb0 + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PUU; ++u) {
        if (rb0 + u < nrb) {
          const double* af = vfrag + ((rb0 + u) * 8) * 32 + lane;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) dmma_8x8x4(c[u][0], c[u][1], af[ks * 32], b[ks]);
        }
      }
#pragma unroll
      for (int u = 0; u < PUU; ++u)
        if (rb0 + u < nrb) {
          if (v0) __stcs(w0 + 8 * (rb0 + u), c[u][0]);
          if (v1) __stcs(w1 + 8 * (rb0 + u), c[u][1]);
        }
    }
  }
}

// Final permutation: piv[posof[j]] = j; slots with posof[j] != j are listed
// (at most 2 per step; overflow -> flags bit 2, never expected)
__global__ void perm_scatter_kernel(const int* __restrict__ posof, int64_t n, int64_t* __restrict__ piv,
                                    int* __restrict__ list, int* __restrict__ count, int cap, int* flags) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int p = posof[j];
    piv[p] = j;
    if (p != (int)j) {
      const int e = atomicAdd(count, 1);
      if (e < cap) list[e] = (int)j;
      else atomicOr(flags, 4);
    }
  }
}

__global__ void iota_positions_kernel(int* posof, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    posof[j] = (int)j;
}

// listed slots -> scratch (scatter = false), scratch -> their logical positions (scatter = true)
__global__ void move_slots_kernel(double* __restrict__ W, int64_t ld, const int* __restrict__ list,
                                  const int* __restrict__ count, const int* __restrict__ posof,
                                  double* __restrict__ tmp, bool scatter) {
  const int cnt = *count;
  for (int e = blockIdx.x; e < cnt; e += gridDim.x) {
    const int j = list[e];
    double* src = scatter ? tmp + (size_t)e * ld : W + (size_t)j * ld;
    double* dst = scatter ? W + (size_t)posof[j] * ld : tmp + (size_t)e * ld;
    for (int64_t r = threadIdx.x; r < ld; r += blockDim.x) dst[r] = src[r];
  }
}

}  // namespace
}  // namespace cpqr_detail
using namespace cpqr_detail;

bool cpqr_panel_supported(int64_t m, int64_t n, int64_t ld, bool padded) {
  static const bool off = [] {
    const char* e = getenv("LRB_CPQR_PANEL");
    return e && atoi(e) == 0;
  }();
  // specialised widths only (the generic-width panel kernel is slower than cpqr.cu's)
  // shared memory: V panel + 2 vectors + the state of ceil(n / SMs) column slots
  const int64_t maxcols = (n + num_sms() - 1) / num_sms() + 1;
  const bool fits = panel_smem_bytes(ld, maxcols) <= (size_t)kSmemLimit;
  return !off && padded && (ld == 256 || ld == 320 || ld == 512) && m <= ld && fits;
}

void cpqr_panel(Workspace& ws, int64_t m, int64_t n, double* W, int64_t ld, int64_t k, int64_t* pivots,
                double* tau, int* d_flags, long long* d_recomputes, cudaStream_t st) {
  using KernT = void (*)(PanelArgs);
  static const bool evdiag0 = getenv("LRB_CPQR_EVENTS") != nullptr;
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  const auto host_t0 = std::chrono::steady_clock::now();
  if (evdiag0) {
    LRB_CUDA(cudaEventCreate(&ev_begin));
    LRB_CUDA(cudaEventCreate(&ev_end));
    LRB_CUDA(cudaEventRecord(ev_begin, st));
  }
  // specialised kernels per (ld / 64, first active chunk); ld in {256, 320, 512}
#define LRB_PANEL_K(L)                                                                                        \
  {cpqr_panel_kernel<0, 4, L>, cpqr_panel_kernel<1, 4, L>, cpqr_panel_kernel<2, 4, L>, cpqr_panel_kernel<3, 4, L>}, \
      {cpqr_panel_kernel<0, 5, L>, cpqr_panel_kernel<1, 5, L>, cpqr_panel_kernel<2, 5, L>,                        \
       cpqr_panel_kernel<3, 5, L>, cpqr_panel_kernel<4, 5, L>},                                                   \
      {cpqr_panel_kernel<0, 8, L>, cpqr_panel_kernel<1, 8, L>, cpqr_panel_kernel<2, 8, L>,                        \
       cpqr_panel_kernel<3, 8, L>, cpqr_panel_kernel<4, 8, L>, cpqr_panel_kernel<5, 8, L>,                        \
       cpqr_panel_kernel<6, 8, L>, cpqr_panel_kernel<7, 8, L>},                                                   \
      cpqr_panel_kernel<-1, -1, L>
  struct KernSet {
    KernT k4[4], k5[5], k8[8], gen;
  };
  // [0]: dense (no identically-zero columns), [1]: with the zero-slot lists
  static const KernSet ks[2] = {{LRB_PANEL_K(false)}, {LRB_PANEL_K(true)}};
#undef LRB_PANEL_K
  const int nld = (int)(ld / 64);
  auto kern_for = [&](int64_t t0, bool list, bool lazy) -> KernT {
    if (lazy) return lazy_kernel_for(nld, (int)(t0 / 64), list);
    const KernSet& k = ks[list ? 1 : 0];
    const int tc = (int)(t0 / 64);
    if (nld == 8) return k.k8[tc];
    if (nld == 5) return k.k5[tc];
    if (nld == 4) return k.k4[tc];
    return k.gen;
  };
  static bool attr = false;
  if (!attr) {
    auto set = [](KernT kf) {
      cudaFuncAttributes fa{};
      LRB_CUDA(cudaFuncGetAttributes(&fa, kf));
      LRB_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(fa.maxDynamicSharedSizeBytes > 0 ? 227 * 1024 - fa.sharedSizeBytes
                                                                           : kSmemLimit)));
    };
    for (const KernSet& k : ks) {
      for (KernT kf : k.k4) set(kf);
      for (KernT kf : k.k5) set(kf);
      for (KernT kf : k.k8) set(kf);
      set(k.gen);
    }
    lazy_set_attributes();
    LRB_CUDA(cudaFuncSetAttribute(panel_update_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * 256 * 64)));
    attr = true;
  }
  // one CTA per SM (the shared memory holds the panel's V)
  static const int grid_cap = getenv("LRB_CPQR_GRID") ? atoi(getenv("LRB_CPQR_GRID")) : 0;  // diagnostic
  int G = std::min(grid_cap > 0 ? std::min(grid_cap, num_sms()) : num_sms(), kMaxG);
  G = (int)std::min<int64_t>(G, std::max<int64_t>(1, (n + PW - 1) / PW));
  const int64_t maxcols = (n + G - 1) / G + 1;
  // Bound-pruned (lazy) steps for wide sweeps, where the eager pass streams the
  // whole trailing block every step; for narrower ones (n < 32768) the eager
  // pass is cheaper than the lazy panels' end-of-panel catch-up (measured:
  // 510 x 65536 C4 sample 17.2 -> 14.7 ms, 210 x 20000 2.7 -> 4.3 ms).
  // LRB_CPQR_LAZY=0 / 1 forces either (read per call: tests switch it in-process).
  const char* lz_env = getenv("LRB_CPQR_LAZY");
  const bool lazy_want = lz_env ? atoi(lz_env) != 0 : n >= 32768;
  static const double lazy_beta = getenv("LRB_CPQR_BETA") ? atof(getenv("LRB_CPQR_BETA")) : 0.0;
  const bool lazy = lazy_want && lazy_smem_bytes(ld, maxcols) <= (size_t)kSmemLimit;
  const size_t smem = lazy ? lazy_smem_bytes(ld, maxcols) : panel_smem_bytes(ld, maxcols);
  if (smem > (size_t)kSmemLimit) throw CudaError("cpqr_panel: too many columns per CTA for the shared norms");
  const size_t cand_sz = kHdr + (size_t)ld + NB;
  const size_t nd = 2 * (size_t)n + 2 * (size_t)G + 2 * (size_t)G * cand_sz + (size_t)n * NB + (size_t)ld * NB;
  const size_t ndisp = 2 * (size_t)k + 2;  // slots away from their final position: <= 2 per step
  const size_t bytes = sizeof(double) * (nd + ndisp * (size_t)ld) + sizeof(long long) * 2 * (size_t)G + 256 +
                       sizeof(int) * ((size_t)n + ndisp + 2) + sizeof(unsigned int) * (size_t)G +
                       // lazy: wall, stats, epoch, catch-up levels
                       sizeof(double) * NB * NB + 4 * sizeof(unsigned long long) + sizeof(int) * ((size_t)n + 2) + 8;
  uint8_t* base = static_cast<uint8_t*>(ws.get(WsSlot::kCpqrState, bytes));
  PanelArgs a{};
  a.W = W;
  a.m = m;
  a.n = n;
  a.ld = ld;
  a.k = k;
  a.piv = pivots;
  a.tau = tau;
  double* d = reinterpret_cast<double*>(base);
  a.nrm = d;
  a.nrmx = d + n;
  a.pval = d + 2 * n;
  a.cand = a.pval + 2 * G;
  a.F = a.cand + 2 * (size_t)G * cand_sz;
  a.Vg = a.F + (size_t)n * NB;
  a.ppos = reinterpret_cast<long long*>(a.Vg + (size_t)ld * NB);
  a.bar = reinterpret_cast<unsigned int*>(a.ppos + 2 * (size_t)G);
  double* disp_cols = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(a.bar) + 256);
  a.posof = reinterpret_cast<int*>(disp_cols + ndisp * (size_t)ld);
  int* disp_list = a.posof + n;
  int* disp_count = disp_list + ndisp;
  a.ctag = reinterpret_cast<unsigned int*>(disp_count + 2);
  a.nzero = disp_count + 1;
  {  // lazy state after the tags (8-byte aligned)
    uintptr_t pz = reinterpret_cast<uintptr_t>(a.ctag + G);
    pz = (pz + 7) & ~uintptr_t(7);
    a.wall = reinterpret_cast<double*>(pz);
    a.lstats = reinterpret_cast<unsigned long long*>(a.wall + NB * NB);
    a.epoch = reinterpret_cast<unsigned int*>(a.lstats + 3);
    a.cjg = reinterpret_cast<int*>(a.lstats + 4);
    a.beta = lazy_beta;
    static const double gap_miss = getenv("LRB_CPQR_GAPMISS") ? atof(getenv("LRB_CPQR_GAPMISS")) : 0.0;  // diagnostic
    a.gap_miss = gap_miss;
    if (lazy) LRB_CUDA(cudaMemsetAsync(a.lstats, 0, 4 * sizeof(unsigned long long), st));
  }
  LRB_CUDA(cudaMemsetAsync(a.nzero, 0, sizeof(int), st));
  LRB_CUDA(cudaMemsetAsync(a.ctag, 0xFF, sizeof(unsigned int) * (size_t)G, st));  // no candidate staged yet
  a.maxcols = maxcols;
  a.flags = d_flags;
  a.recomputes = reinterpret_cast<unsigned long long*>(d_recomputes);
  static const bool trace = getenv("LRB_CPQR_TRACE") != nullptr;
  static const bool trace_panels = getenv("LRB_CPQR_TRACE_PANELS") != nullptr;
  std::vector<unsigned long long> prev;
  a.trace = nullptr;
  a.tstep = nullptr;
  if (trace) {
    LRB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.trace), 8 * sizeof(unsigned long long) * G, st));
    LRB_CUDA(cudaMemsetAsync(a.trace, 0, 8 * sizeof(unsigned long long) * G, st));
    if (trace_panels)
      LRB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.tstep), 4 * sizeof(unsigned long long) * G * k, st));
  }
  // LRB_CPQR_EVENTS: CUDA events around every launch (kernel vs gap time, diagnostic)
  static const bool evdiag = getenv("LRB_CPQR_EVENTS") != nullptr;
  std::vector<cudaEvent_t> ev;
  auto evrec = [&]() {
    if (!evdiag) return;
    cudaEvent_t e;
    LRB_CUDA(cudaEventCreate(&e));
    LRB_CUDA(cudaEventRecord(e, st));
    ev.push_back(e);
  };
  evrec();
  // the first launch runs the list variant and counts identically-zero
  // columns; later launches take the dense variant when there are none
  bool list = true;
  thread_local int* h_nzero = nullptr;  // mapped pinned word (no copy-engine queueing)
  if (!h_nzero) LRB_CUDA(cudaMallocHost(&h_nzero, sizeof(int)));
  // lazy panels (NBL steps) while the trailing block is tall; the last
  // LRB_CPQR_EAGER_ROWS (default 0: measured no gain at 128-256) rows of ld run the eager kernel, whose
  // per-step pass is cheap once the sweep is short (its first launch stages
  // the entry candidate itself: a.entry)
  static const int64_t eager_rows = getenv("LRB_CPQR_EAGER_ROWS") ? atoll(getenv("LRB_CPQR_EAGER_ROWS")) : 0;
  const int64_t lazy_end = lazy ? std::max<int64_t>(0, ((ld - eager_rows) / 64) * 64) : 0;
  int launches = 0;
  bool prev_lazy = false;
  for (int64_t t0 = 0, t1 = 0; t0 < k; t0 = t1) {
    const bool lz = lazy && t0 < lazy_end;
    t1 = std::min<int64_t>(k, t0 + (lz ? NBL : NB));
    a.entry = (!lz && prev_lazy) ? 1 : 0;
    prev_lazy = lz;
    if (++launches == 2) {
      LRB_CUDA(cudaStreamSynchronize(st));
      list = *h_nzero > 0;
    }
    a.t0 = t0;
    a.t1 = t1;
    a.init = t0 == 0 ? 1 : 0;
    {  // L2 keep share of the sweep (measured, profiles/r02_cpqr_profile.md): sweeps that fit
      // in ~110 MB are kept whole; larger ones keep their last ~40 MB (more evicts the
      // lines the streaming part still reuses).  LRB_CPQR_L2KEEP=<MB> overrides.
      static const double keep_env = getenv("LRB_CPQR_L2KEEP") ? atof(getenv("LRB_CPQR_L2KEEP")) : -1.0;
      const double sweep = 8.0 * (double)(ld - 64 * (t0 / 64)) * (double)std::max<int64_t>(1, n - t0);
      const double keep_mb = keep_env >= 0.0 ? keep_env : (sweep <= 110e6 ? 1e9 : 40.0);
      a.keep1024 = (int)std::min(1024.0, 1024.0 * keep_mb * 1e6 / sweep);
    }
    LRB_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned int), st));
    // eager tags count steps, lazy ones rounds (>= steps): waiters accept tags >= the wanted
    // one, so the lazy panels' tags are cleared before the eager tail
    if (a.entry) LRB_CUDA(cudaMemsetAsync(a.ctag, 0xFF, sizeof(unsigned int) * (size_t)G, st));
    evrec();
    void* params[] = {&a};
    LRB_CUDA(cudaLaunchCooperativeKernel((void*)kern_for(t0, list, lz), dim3(G), dim3(PT), params, smem, st));
    LRB_CHECK_LAUNCH();
    if (t0 == 0) copy_bytes_mapped(h_nzero, a.nzero, sizeof(int), st);
    evrec();
    if (trace && trace_panels) {  // per-panel phase means / maxima over CTAs (diagnostic)
      std::vector<unsigned long long> h(8 * (size_t)G);
      LRB_CUDA(cudaMemcpyAsync(h.data(), a.trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
      LRB_CUDA(cudaStreamSynchronize(st));
      if (t0 == 0) prev.assign(h.size(), 0ull);
      fprintf(stderr, "cpqr_panel t0=%4ld us/step (mean/max):", (long)t0);
      for (int slot = 1; slot <= 5; ++slot) {
        double sum = 0, mx = 0;
        for (int g = 0; g < G; ++g) {
          const double v = (double)(h[g * 8 + slot] - prev[g * 8 + slot]) / 1e3 / (double)(t1 - t0);
          sum += v;
          mx = std::max(mx, v);
        }
        fprintf(stderr, " %.2f/%.2f", sum / G, mx);
      }
      fprintf(stderr, "\n");
      prev = h;
    }
    if (lz) {  // catch every column up on this panel's reflectors, then the rank-NB update
      FinArgs fa{};
      fa.W = W;
      fa.ld = ld;
      fa.m = m;
      fa.n = n;
      fa.t0 = t0;
      fa.t1 = t1;
      fa.r1 = std::min<int64_t>(ld, (m + 7) & ~int64_t(7));
      fa.C = (int)(t1 - t0);
      fa.upd = (t1 < k && t1 < m && t1 < n && fa.r1 > t1) ? 1 : 0;
      fa.Vg = a.Vg;
      fa.F = a.F;
      fa.tau = tau + t0;
      fa.wall = a.wall;
      fa.nrm = a.nrm;
      fa.nrmx = a.nrmx;
      fa.cj = a.cjg;
      fa.recomputes = a.recomputes;
      const int64_t ngroups = (n + 7) / 8;
      const int fg = (int)std::min<int64_t>((ngroups + FW - 1) / FW, num_sms());
      launch_panel_finalize(fa, fg, st);
    }
    // A_p(t1:m, t1:n) -= V(t1:m, 0:c) F(t1:n, 0:c)^T  (rows/cols of later panels only)
    if (!lz && t1 < k && t1 < m && t1 < n) {
      // every slot (pivoted ones have F = 0); rows t1..m rounded up to 8 (padding rows stay 0)
      const int64_t r1 = std::min<int64_t>(ld, (m + 7) & ~int64_t(7));
      const int64_t ngroups = (n + 7) / 8;
      const int ug = (int)std::min<int64_t>((ngroups + PUW - 1) / PUW, num_sms());  // persistent
      const size_t usm = sizeof(double) * 256 * (size_t)((r1 - t1) / 8);
      panel_update_dmma_kernel<<<ug, PUW * 32, usm, st>>>(W, ld, t1, r1, n, a.Vg, a.F, (int)(t1 - t0));
      LRB_CHECK_LAUNCH();
    }
    evrec();
  }
  if (evdiag) {  // per panel: [memset] [cooperative kernel] [update]
    LRB_CUDA(cudaStreamSynchronize(st));
    double tm = 0, tk = 0, tu = 0;
    for (size_t i = 0; i + 3 < ev.size(); i += 3) {
      float x = 0;
      LRB_CUDA(cudaEventElapsedTime(&x, ev[i], ev[i + 1])); tm += x;
      LRB_CUDA(cudaEventElapsedTime(&x, ev[i + 1], ev[i + 2])); tk += x;
      LRB_CUDA(cudaEventElapsedTime(&x, ev[i + 2], ev[i + 3])); tu += x;
    }
    fprintf(stderr, "cpqr_panel events: memset+gap %.3f ms, panel kernels %.3f ms, updates %.3f ms\n", tm, tk, tu);
    for (auto e : ev) cudaEventDestroy(e);
  }
  // logical -> physical: pivots, and the few slots not at their final position
  // move there through a scratch copy (the reference's swapped layout)
  LRB_CUDA(cudaMemsetAsync(disp_count, 0, sizeof(int), st));
  const int pg = (int)std::min<int64_t>((n + 255) / 256, 4 * (int64_t)num_sms());
  if (k == 0) iota_positions_kernel<<<pg, 256, 0, st>>>(a.posof, n);
  perm_scatter_kernel<<<pg, 256, 0, st>>>(a.posof, n, pivots, disp_list, disp_count, (int)ndisp,
                                                        d_flags);
  LRB_CHECK_LAUNCH();
  const int dg = (int)std::min<size_t>(ndisp, 4 * (size_t)num_sms());
  move_slots_kernel<<<dg, 256, 0, st>>>(W, ld, disp_list, disp_count, a.posof, disp_cols, false);
  move_slots_kernel<<<dg, 256, 0, st>>>(W, ld, disp_list, disp_count, a.posof, disp_cols, true);
  LRB_CHECK_LAUNCH();
  if (evdiag0) {
    const double host_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    LRB_CUDA(cudaEventRecord(ev_end, st));
    LRB_CUDA(cudaEventSynchronize(ev_end));
    float x = 0;
    LRB_CUDA(cudaEventElapsedTime(&x, ev_begin, ev_end));
    fprintf(stderr, "cpqr_panel events: whole call %.3f ms on the stream, host enqueue %.3f ms\n", x, host_ms);
    cudaEventDestroy(ev_begin);
    cudaEventDestroy(ev_end);
  }
  if (trace) {
    std::vector<unsigned long long> h(8 * (size_t)G);
    LRB_CUDA(cudaMemcpyAsync(h.data(), a.trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    LRB_CUDA(cudaStreamSynchronize(st));
    const char* names[6] = {"", "loads", "pass", "argmax+wb", "stage", "barrier"};
    for (int slot = 1; slot <= 5; ++slot) {
      double mn = 1e30, mx = 0, sum = 0;
      int arg = 0;
      for (int g = 0; g < G; ++g) {
        const double v = h[g * 8 + slot] / 1e3 / k;
        mn = std::min(mn, v);
        sum += v;
        if (v > mx) { mx = v; arg = g; }
      }
      fprintf(stderr, "cpqr_panel trace %-10s us/step: min %.2f mean %.2f max %.2f (cta %d)\n", names[slot], mn,
              sum / G, mx, arg);
    }
    {
      double cyc = 0, ns = 0;
      for (int g = 0; g < G; ++g) { cyc += (double)h[g * 8 + 6]; ns += (double)h[g * 8 + 7]; }
      fprintf(stderr, "cpqr_panel trace SM clock %.0f MHz over %.3f ms\n", 1e3 * cyc / ns, ns / G / 1e6);
    }
    if (lazy) {
      unsigned long long ls[2];
      LRB_CUDA(cudaMemcpyAsync(ls, a.lstats, sizeof ls, cudaMemcpyDeviceToHost, st));
      LRB_CUDA(cudaStreamSynchronize(st));
      fprintf(stderr, "cpqr_lazy: %llu retry rounds, %.1f columns evaluated per step (%.2f%% of n)\n", ls[0],
              (double)ls[1] / (double)std::max<int64_t>(1, k), 100.0 * (double)ls[1] / (double)std::max<int64_t>(1, k) / (double)n);
    }
    if (a.tstep) {  // per step: the last-arriving CTA's phases vs the CTA mean (steps 1..k-1)
      std::vector<unsigned long long> t(4 * (size_t)G * k);
      LRB_CUDA(cudaMemcpyAsync(t.data(), a.tstep, t.size() * 8, cudaMemcpyDeviceToHost, st));
      LRB_CUDA(cudaStreamSynchronize(st));
      for (int64_t b0 = 0; b0 < k; b0 += 64) {
        const int64_t b1 = std::min<int64_t>(k, b0 + 64);
        double wait = 0, dl[3] = {0, 0, 0}, dstart = 0;
        int cnt = 0, own_p = 0, own_s = 0;
        for (int64_t s = std::max<int64_t>(b0, 1); s < b1; ++s) {
          if (s % NB == 0) continue;  // first step of a launch: no departure stamp
          double mean[4] = {0, 0, 0, 0};
          int am = 0;
          for (int g = 0; g < G; ++g) {
            const unsigned long long* q = &t[(s * G + g) * 4];
            for (int e = 0; e < 4; ++e) mean[e] += ((double)q[e] - (double)t[(s * G) * 4]) / G;
            if (q[3] > t[(s * G + am) * 4 + 3]) am = g;
          }
          const unsigned long long* L = &t[(s * G + am) * 4];
          own_p += (int)(L[3] & 1);
          own_s += (int)((L[3] >> 1) & 1);
          const double base0 = (double)t[(s * G) * 4];
          wait += (double)L[3] - base0 - mean[3];
          dstart += (double)L[0] - base0 - mean[0];
          for (int e = 1; e < 4; ++e)
            dl[e - 1] += ((double)L[e] - (double)L[e - 1]) - (mean[e] - mean[e - 1]);
          ++cnt;
        }
        if (!cnt) continue;
        const double ns = 1e3 * cnt;
        fprintf(stderr, "cpqr_panel steps %4ld-%4ld last CTA vs mean (us): arrival %+.2f = start %+.2f loads %+.2f "
                "pass %+.2f tail %+.2f; last CTA owns p %d / s %d of %d\n", (long)b0, (long)b1, wait / ns, dstart / ns,
                dl[0] / ns, dl[1] / ns, dl[2] / ns, own_p, own_s, cnt);
      }
      cudaFreeAsync(a.tstep, st);
    }
    cudaFreeAsync(a.trace, st);
  }
}

}  // namespace lrb
