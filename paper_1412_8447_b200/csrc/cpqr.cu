// cpqr.cu -- truncated column-pivoted Householder QR on B200.
//
// Restates cpqr.hpp:32-114 exactly in its observable pivot semantics:
//   * pivot = first maximum of the running squared norms over positions
//     [step, n) (strict >, cpqr.hpp:49-51): ties go to the lowest position;
//   * full-column swap of data, norm2, norm2_exact and pivot (cpqr.hpp:52-57);
//   * reflector beta = -sign(alpha)|x|, tau = (beta-alpha)/beta, v = x/(alpha-beta)
//     (cpqr.hpp:59-66), applied as W -= (tau v)(v^T W) (cpqr.hpp:68-75);
//   * downdate norm2 -= W(step,j)^2 and exact recompute below 1e-6 of the last
//     exact value (cpqr.hpp:78-84).
//
// B200 design: ONE persistent cooperative kernel runs all k steps.  Columns
// are statically partitioned over CTAs (and round-robin over warps); a warp
// owns a whole column and keeps up to 64*CH rows in registers (the sketch Y
// and C^T have <= 512 rows: one 16-byte load per lane per 64 rows moves a
// column in and out exactly once per step), with the next column's loads
// issued before the current one is reduced (register double buffering).
// Each step is one fused HBM pass
//   dot(v, col) -> rank-1 update -> row-s downdate -> (rare) exact recompute
//   -> per-warp / per-CTA argmax on (norm2 desc, position asc)
// followed by a single grid barrier.  At the end of a step every CTA builds
// the Householder reflector of ITS best column (fresh norm, beta, tau, v) and
// stages it in a double-buffered candidate slot; the next step only reads the
// winner's slot, so the serial part of a step is one batched L2 round trip.
// Sweep direction alternates per step so the columns written last are read
// first while still in L2.  Rows > 64*CH (tall deterministic IDs) stream
// through L2 in two passes.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace lrb {

namespace {

constexpr int kMaxWarps = 32;  // shared reductions sized for up to 1024 threads
constexpr int kGridWarpsPerCta = 8;  // grid sizing estimate (columns per CTA)
constexpr int kMaxSmemRows = 6144;  // v and tau*v kept in shared memory up to this height
constexpr int kMaxG = 512;          // partial slots read by one warp (16 per lane)
constexpr int kHdr = 4;             // candidate header: alpha, beta, tau, apply

struct CpqrArgs {
  double* W;
  int64_t m, n, ld, k;
  int64_t* piv;
  double* nrm;
  double* nrmx;
  double* tau;
  double* pval;      // [2][G]
  long long* ppos;   // [2][G]
  double* cand;      // [2][G][kHdr + m]: reflector of each CTA's best column
  double* scratch;   // [G][4*m]: old-s column, pivot R rows, (v, tau*v if not in smem)
  int* flags;
  unsigned long long* recomputes;
  int nopivot;  // unpivoted Householder QR (orth_rows fallback): position s is always the pivot
  unsigned int* bar;  // grid barrier counter (zeroed before the launch)
};

// Grid barrier of the co-resident (cooperative) grid: one release reduction
// per CTA on a monotonic counter, an acquire spin (cooperative groups'
// grid.sync measured ~9 us per barrier on this part; this is one L2 round
// trip after the last arrival).
__device__ __forceinline__ void cpqr_grid_barrier(unsigned int* bar, unsigned int& target) {
  target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

constexpr int kSU = 4;  // streamed 64-row chunks in flight per lane (tall matrices)

__device__ __forceinline__ bool better(double v1, long long p1, double v2, long long p2) {
  return v1 > v2 || (v1 == v2 && p1 < p2);
}

// fixed-order CTA sum (all threads receive the result)
__device__ double cta_sum(double x, double* sh) {
  x = warp_sum(x);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[w] = x;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
  return t;
}

// Reflector of column jb (rows s0..m-1, cpqr.hpp:59-66) into candidate slot cd.
// When colnorm == 0 the slot carries x itself (the column is left untouched).
__device__ void stage_candidate(const CpqrArgs& a, double* cd, int64_t s0, long long jb, double* sh) {
  const int64_t m = a.m;
  if (jb >= a.n || s0 >= m) {
    __syncthreads();
    return;
  }
  const double* x = a.W + jb * a.ld;
  double part = 0.0;
  for (int64_t i = s0 + threadIdx.x; i < m; i += blockDim.x) part = fma(x[i], x[i], part);
  const double cn2 = cta_sum(part, sh);
  const double colnorm = sqrt(cn2);
  const double alpha = x[s0];
  const bool apply = colnorm > 0.0;
  double beta = alpha, tau = 0.0, scale = 1.0;
  if (apply) {
    beta = alpha >= 0.0 ? -colnorm : colnorm;
    tau = (beta - alpha) / beta;
    scale = alpha - beta;
  }
  for (int64_t i = s0 + threadIdx.x; i < m; i += blockDim.x)
    cd[kHdr + i] = apply ? ((i == s0) ? 1.0 : x[i] / scale) : x[i];
  if (threadIdx.x == 0) {
    cd[0] = alpha;
    cd[1] = beta;
    cd[2] = tau;
    cd[3] = apply ? 1.0 : 0.0;
  }
}

// per-warp column state
template <int CH>
struct Col {
  double c[CH][2];
  double nr, nx;
};

template <int CH>
__device__ __forceinline__ void load_col(Col<CH>& col, const double* src, bool cross_cta, int64_t s, int64_t m,
                                         int lane) {
#pragma unroll
  for (int t = 0; t < CH; ++t) {
    const int64_t i = 64 * t + 2 * lane;
    col.c[t][0] = col.c[t][1] = 0.0;
    if (64 * (t + 1) > s && i < m) {
      if (i + 1 < m) {
        const double2 xx = cross_cta ? __ldcg(reinterpret_cast<const double2*>(src + i))
                                     : *reinterpret_cast<const double2*>(src + i);
        col.c[t][0] = xx.x;
        col.c[t][1] = xx.y;
      } else {
        col.c[t][0] = cross_cta ? __ldcg(src + i) : src[i];
      }
    }
  }
}

template <int CH, bool PF, bool FAST, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) cpqr_kernel(CpqrArgs a) {
  unsigned int bar_target = 0;
  extern __shared__ double dyn[];
  __shared__ double sh_red[kMaxWarps];
  __shared__ double sh_bv[kMaxWarps];
  __shared__ long long sh_bp[kMaxWarps];
  constexpr int kWarps = NT / 32;
  constexpr int kThreads = NT;
  __shared__ double sh_hdr[kHdr];
  __shared__ long long sh_piv[2];    // p, winner cta
  __shared__ long long sh_state[2];  // piv[p], piv[s]
  __shared__ double sh_nst[4];       // nrm[p], nrmx[p], nrm[s], nrmx[s]

  const int G = gridDim.x, cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = a.m, n = a.n, ld = a.ld, k = a.k;
  const int64_t c0 = n * cta / G, c1 = n * (cta + 1) / G;
  const int64_t cand_sz = kHdr + m;
  double* scr = a.scratch + (int64_t)cta * 4 * ld;
  double* olds = scr;       // old column at position s (when swapped into p)
  double* pivr = scr + ld;  // pivot column rows < s
  const bool vs = ld <= kMaxSmemRows;
  double* vv = vs ? dyn : scr + 2 * ld;      // v[i] for i >= s (v[s] = 1)
  double* tv = vs ? dyn + ld : scr + 3 * ld;  // tau * v
  if (FAST) {
    for (int64_t i = threadIdx.x; i < ld; i += kThreads) {
      vv[i] = 0.0;
      tv[i] = 0.0;
      olds[i] = 0.0;
    }
  }
  const int nchunks = (int)((m + 63) / 64);
  const int64_t cnt = (c1 - c0 - warp + kWarps - 1) / kWarps;  // columns of this warp
  unsigned long long my_recomputes = 0;

  // ------------------------------------------------------------ init
  {
    double bv = -INFINITY;
    long long bp = INT64_MAX;
    int bad = 0;
    for (int64_t j = c0 + warp; j < c1; j += kWarps) {
      const double* col = a.W + j * ld;
      double acc = 0.0;
      for (int t = 0; t < nchunks; ++t) {
        const int64_t i = 64 * t + 2 * lane;
        if (i + 1 < m) {
          const double2 x = *reinterpret_cast<const double2*>(col + i);
          bad |= !isfinite(x.x) | !isfinite(x.y);
          acc = fma(x.x, x.x, acc);
          acc = fma(x.y, x.y, acc);
        } else if (i < m) {
          const double x = col[i];
          bad |= !isfinite(x);
          acc = fma(x, x, acc);
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) {
        a.nrm[j] = acc;
        a.nrmx[j] = acc;
        a.piv[j] = j;
      }
      if (better(acc, j, bv, bp)) { bv = acc; bp = j; }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(a.flags, 1);
    if (lane == 0) { sh_bv[warp] = bv; sh_bp[warp] = bp; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double cv = sh_bv[0];
      long long cp = sh_bp[0];
      for (int w = 1; w < kWarps; ++w)
        if (better(sh_bv[w], sh_bp[w], cv, cp)) { cv = sh_bv[w]; cp = sh_bp[w]; }
      if (a.nopivot) {  // the owner of column 0 wins
        cp = (0 >= c0 && 0 < c1) ? 0 : INT64_MAX;
        cv = cp == 0 ? INFINITY : -INFINITY;
      }
      a.pval[cta] = cv;
      a.ppos[cta] = cp;
      sh_piv[0] = cp;
    }
    __syncthreads();
    stage_candidate(a, a.cand + (int64_t)cta * cand_sz, 0, sh_piv[0], sh_red);
  }
  cpqr_grid_barrier(a.bar, bar_target);
  if (__ldcg(a.flags) != 0) return;

  // ------------------------------------------------------------ steps
  for (int64_t s = 0; s < k; ++s) {
    const int par = (int)(s & 1), nxt = par ^ 1;
    // (1) global argmax over the per-CTA partials: one batched load per lane
    if (warp == 0) {
      double pv[kMaxG / 32];
      long long pp[kMaxG / 32];
#pragma unroll
      for (int r = 0; r < kMaxG / 32; ++r) {
        const int c = lane + 32 * r;
        pv[r] = c < G ? __ldcg(a.pval + (int64_t)par * G + c) : -INFINITY;
        pp[r] = c < G ? __ldcg(a.ppos + (int64_t)par * G + c) : INT64_MAX;
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
      if (lane == 0) { sh_piv[0] = bp; sh_piv[1] = bc; }
    }
    __syncthreads();
    const int64_t p = sh_piv[0];
    const double* cd = a.cand + ((int64_t)par * G + sh_piv[1]) * cand_sz;

    // (2) the winner's reflector -> v, tau*v (one batched L2 round trip)
    {
      const double tau_b = __ldcg(cd + 2);
      const bool apply_b = __ldcg(cd + 3) != 0.0;
      if (FAST && s > 0 && threadIdx.x == 0) {  // keep v, tau*v zero above row s
        vv[s - 1] = 0.0;
        tv[s - 1] = 0.0;
      }
      for (int64_t i = s + threadIdx.x; i < m; i += kThreads) {
        const double vi = __ldcg(cd + kHdr + i);
        vv[i] = vi;
        tv[i] = apply_b ? tau_b * vi : 0.0;
      }
      if (threadIdx.x < kHdr) sh_hdr[threadIdx.x] = __ldcg(cd + threadIdx.x);
    }
    // (3) swap bookkeeping by the owner of position p
    const bool owner = (p >= c0 && p < c1);
    const bool swapped = owner && p != s;
    if (swapped) {
      for (int64_t i = threadIdx.x; i < m; i += kThreads) olds[i] = __ldcg(a.W + s * ld + i);
      for (int64_t i = threadIdx.x; i < s; i += kThreads) pivr[i] = a.W[p * ld + i];
      if (threadIdx.x == 0) {
        sh_state[0] = a.piv[p];
        sh_state[1] = __ldcg(a.piv + s);
        sh_nst[0] = a.nrm[p];
        sh_nst[1] = a.nrmx[p];
        sh_nst[2] = __ldcg(a.nrm + s);
        sh_nst[3] = __ldcg(a.nrmx + s);
      }
    }
    __syncthreads();
    const double tau = sh_hdr[2];
    const bool apply = sh_hdr[3] != 0.0;
    if (cta == 0 && threadIdx.x == 0) a.tau[s] = tau;

    // (4) fused trailing pass over owned positions j in (s, n)
    double bv = -INFINITY;
    long long bp = INT64_MAX;
    auto col_of = [&](int64_t it) { return c0 + warp + kWarps * ((s & 1) ? (cnt - 1 - it) : it); };
    auto next_valid = [&](int64_t it) {
      while (it < cnt && col_of(it) <= s) ++it;
      return it;
    };
    auto fetch = [&](Col<CH>& cb, int64_t j) {
      const bool from_s = swapped && j == p;
      load_col<CH>(cb, from_s ? olds : a.W + j * ld, false, s, m, lane);
      cb.nr = from_s ? sh_nst[2] : a.nrm[j];
      cb.nx = from_s ? sh_nst[3] : a.nrmx[j];
    };
    auto process = [&](Col<CH>& cb, int64_t j) {
      const bool from_s = swapped && j == p;
      const double* src = from_s ? olds : a.W + j * ld;
      double* dst = a.W + j * ld;
      double dot = 0.0;
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        const int64_t i = 64 * t + 2 * lane;
        if (64 * (t + 1) > s && i < m) {
          if (i >= s) dot = fma(cb.c[t][0], vv[i], dot);
          if (i + 1 >= s && i + 1 < m) dot = fma(cb.c[t][1], vv[i + 1], dot);
        }
      }
      // streamed rows (tall matrices): kSU chunks' loads issued before their FMAs
      // (the FMA order, hence the result, is that of the one-chunk loop)
      for (int t = CH; t < nchunks; t += kSU) {
        double xv[kSU][2];
#pragma unroll
        for (int u = 0; u < kSU; ++u) {
          const int64_t i = 64 * (t + u) + 2 * lane;
          const bool in = t + u < nchunks;
          xv[u][0] = (in && i < m && i >= s) ? src[i] : 0.0;
          xv[u][1] = (in && i + 1 < m && i + 1 >= s) ? src[i + 1] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kSU; ++u) {
          const int64_t i = 64 * (t + u) + 2 * lane;
          if (t + u < nchunks) {
            if (i < m && i >= s) dot = fma(xv[u][0], vv[i], dot);
            if (i + 1 < m && i + 1 >= s) dot = fma(xv[u][1], vv[i + 1], dot);
          }
        }
      }
      dot = warp_sum(dot);
      double xs = 0.0, tail2 = 0.0;
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        const int64_t i = 64 * t + 2 * lane;
        if (64 * (t + 1) > s && i < m) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t r = i + e;
            if (r >= s && r < m) {
              double c = cb.c[t][e];
              if (apply) c = fma(-tv[r], dot, c);
              cb.c[t][e] = c;
              if (r == s) xs = c;
              else tail2 = fma(c, c, tail2);
            }
          }
          if (i + 1 < m) *reinterpret_cast<double2*>(dst + i) = make_double2(cb.c[t][0], cb.c[t][1]);
          else dst[i] = cb.c[t][0];
        }
      }
      for (int t = CH; t < nchunks; t += kSU) {
        double xv[kSU][2];
#pragma unroll
        for (int u = 0; u < kSU; ++u)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t r = 64 * (t + u) + 2 * lane + e;
            xv[u][e] = (t + u < nchunks && r < m) ? src[r] : 0.0;
          }
#pragma unroll
        for (int u = 0; u < kSU; ++u)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t r = 64 * (t + u) + 2 * lane + e;
            if (t + u < nchunks && r < m) {
              double c = xv[u][e];
              if (r >= s) {
                if (apply) c = fma(-tv[r], dot, c);
                if (r == s) xs = c;
                else tail2 = fma(c, c, tail2);
              }
              dst[r] = c;  // rows < s copied through unchanged (needed when from_s)
            }
          }
      }
      if (from_s)  // rows < s of the swapped-in column that sit in skipped cached chunks
        for (int64_t r = lane; r < s && r < 64 * (int64_t)CH; r += 32) dst[r] = olds[r];
      xs = __shfl_sync(0xffffffffu, xs, (int)((s % 64) / 2));
      double nr = cb.nr - xs * xs;
      double nx = cb.nx;
      if (nr < 1e-6 * nx) {
        nr = warp_sum(tail2);
        nx = nr;
        ++my_recomputes;
      }
      if (lane == 0) {
        a.nrm[j] = nr;
        a.nrmx[j] = nx;
        if (from_s) a.piv[j] = sh_state[1];
      }
      if (better(nr, j, bv, bp)) { bv = nr; bp = j; }
    };
    // FAST path: ld % 64 == 0, ld <= 64*CH, rows [m, ld) are zero and
    // vv/tv are zero outside [s, m): no per-element predicates at all.
    const int t0 = (int)(s >> 6);
    const int nld = (int)(ld >> 6);
    auto fetch_fast = [&](Col<CH>& cb, int64_t j) {
      const bool from_s = swapped && j == p;
      const double* src = from_s ? olds : a.W + j * ld;
      const int ts = from_s ? 0 : t0;
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        if (t >= ts && t < nld) {
          const double2 xx = *reinterpret_cast<const double2*>(src + 64 * t + 2 * lane);
          cb.c[t][0] = xx.x;
          cb.c[t][1] = xx.y;
        }
      }
      cb.nr = from_s ? sh_nst[2] : a.nrm[j];
      cb.nx = from_s ? sh_nst[3] : a.nrmx[j];
    };
    auto process_fast = [&](Col<CH>& cb, int64_t j) {
      const bool from_s = swapped && j == p;
      const int ts = from_s ? 0 : t0;
      double* dst = a.W + j * ld;
      const double2* v2 = reinterpret_cast<const double2*>(vv);
      const double2* tv2 = reinterpret_cast<const double2*>(tv);
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int t = 0; t < CH; ++t)
        if (t >= ts && t < nld) {
          const double2 vx = v2[32 * t + lane];
          d0 = fma(cb.c[t][0], vx.x, d0);
          d1 = fma(cb.c[t][1], vx.y, d1);
        }
      const double dot = warp_sum(d0 + d1);
      double xs = 0.0;
#pragma unroll
      for (int t = 0; t < CH; ++t)
        if (t >= ts && t < nld) {
          if (apply) {
            const double2 tx = tv2[32 * t + lane];
            cb.c[t][0] = fma(-tx.x, dot, cb.c[t][0]);
            cb.c[t][1] = fma(-tx.y, dot, cb.c[t][1]);
          }
          if (t == t0) xs = (s & 1) ? cb.c[t][1] : cb.c[t][0];
          *reinterpret_cast<double2*>(dst + 64 * t + 2 * lane) = make_double2(cb.c[t][0], cb.c[t][1]);
        }
      xs = __shfl_sync(0xffffffffu, xs, (int)((s & 63) >> 1));
      double nr = cb.nr - xs * xs;
      double nx = cb.nx;
      if (nr < 1e-6 * nx) {  // rare: exact recompute from the registers (rows > s)
        double q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int t = 0; t < CH; ++t)
          if (t >= t0 && t < nld) {
            const int64_t r = 64 * t + 2 * lane;
            if (r > s) q0 = fma(cb.c[t][0], cb.c[t][0], q0);
            if (r + 1 > s) q1 = fma(cb.c[t][1], cb.c[t][1], q1);
          }
        nr = warp_sum(q0 + q1);
        nx = nr;
        ++my_recomputes;
      }
      if (lane == 0) {
        a.nrm[j] = nr;
        a.nrmx[j] = nx;
        if (from_s) a.piv[j] = sh_state[1];
      }
      if (better(nr, j, bv, bp)) { bv = nr; bp = j; }
    };

    if constexpr (FAST && !PF) {
      Col<CH> A;
      for (int64_t it = next_valid(0); it < cnt; it = next_valid(it + 1)) {
        fetch_fast(A, col_of(it));
        process_fast(A, col_of(it));
      }
    } else if constexpr (FAST) {
      Col<CH> A, B;
      int64_t it = next_valid(0);
      if (it < cnt) fetch_fast(A, col_of(it));
      while (it < cnt) {
        const int64_t it2 = next_valid(it + 1);
        if (it2 < cnt) fetch_fast(B, col_of(it2));
        process_fast(A, col_of(it));
        if (it2 >= cnt) break;
        const int64_t it3 = next_valid(it2 + 1);
        if (it3 < cnt) fetch_fast(A, col_of(it3));
        process_fast(B, col_of(it2));
        it = it3;
      }
    } else if constexpr (!PF) {
      Col<CH> A;
      for (int64_t it = next_valid(0); it < cnt; it = next_valid(it + 1)) {
        fetch(A, col_of(it));
        process(A, col_of(it));
      }
    } else {
      Col<CH> A, B;
      int64_t it = next_valid(0);
      if (it < cnt) fetch(A, col_of(it));
      while (it < cnt) {
        const int64_t it2 = next_valid(it + 1);
        if (it2 < cnt) fetch(B, col_of(it2));
        process(A, col_of(it));
        if (it2 >= cnt) break;
        const int64_t it3 = next_valid(it2 + 1);
        if (it3 < cnt) fetch(A, col_of(it3));
        process(B, col_of(it2));
        it = it3;
      }
    }

    // (5) CTA argmax, pivot column write-back, candidate staging
    if (lane == 0) { sh_bv[warp] = bv; sh_bp[warp] = bp; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double cv = sh_bv[0];
      long long cp = sh_bp[0];
      for (int w = 1; w < kWarps; ++w)
        if (better(sh_bv[w], sh_bp[w], cv, cp)) { cv = sh_bv[w]; cp = sh_bp[w]; }
      if (a.nopivot) {  // the owner of position s + 1 wins
        cp = (s + 1 >= c0 && s + 1 < c1) ? s + 1 : INT64_MAX;
        cv = cp == s + 1 ? INFINITY : -INFINITY;
      }
      a.pval[(int64_t)nxt * G + cta] = cv;
      a.ppos[(int64_t)nxt * G + cta] = cp;
      sh_piv[0] = cp;
    }
    if (owner) {
      double* ps = a.W + s * ld;
      if (swapped) {
        for (int64_t i = threadIdx.x; i < s; i += kThreads) ps[i] = pivr[i];
        if (threadIdx.x == 0) {
          a.piv[s] = sh_state[0];
          a.nrm[s] = sh_nst[0];
          a.nrmx[s] = sh_nst[1];
        }
      }
      const double beta = sh_hdr[1];
      for (int64_t i = s + threadIdx.x; i < m; i += kThreads) ps[i] = (apply && i == s) ? beta : vv[i];
    }
    __syncthreads();
    stage_candidate(a, a.cand + ((int64_t)nxt * G + cta) * cand_sz, s + 1, sh_piv[0], sh_red);
    cpqr_grid_barrier(a.bar, bar_target);
  }
  if (lane == 0 && my_recomputes) atomicAdd(a.recomputes, (unsigned long long)my_recomputes);
}

__global__ void extract_s_kernel(int64_t m, int64_t n, const double* __restrict__ W, int64_t ld, int64_t k,
                                 double* __restrict__ s, int64_t lds) {
  const int64_t total = k * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % k, j = t / k;
    double v = (i > j) ? 0.0 : W[i + j * ld];
    if (W[i + i * ld] < 0.0) v = -v;
    s[i + j * lds] = v;
  }
}

// q(:, c) = H_0 ... H_{k-1} e_c, then the sign fix; one warp per column
__global__ void form_q_kernel(int64_t m, const double* __restrict__ W, int64_t ld, int64_t k,
                              const double* __restrict__ tau, double* __restrict__ q, int64_t ldq) {
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= k) return;
  double* qc = q + c * ldq;
  for (int64_t i = lane; i < m; i += 32) qc[i] = (i == c) ? 1.0 : 0.0;
  __syncwarp();
  for (int64_t st = k - 1; st >= 0; --st) {
    const double t = tau[st];
    if (t == 0.0) continue;
    const double* v = W + st * ld;  // v(st) = 1, v(i>st) = W(i, st)
    double d = 0.0;
    for (int64_t i = st + lane; i < m; i += 32) d = fma(qc[i], i == st ? 1.0 : v[i], d);
    d = warp_sum(d);
    for (int64_t i = st + lane; i < m; i += 32) qc[i] = fma(-(t * (i == st ? 1.0 : v[i])), d, qc[i]);
    __syncwarp();
  }
  if (W[c + c * ld] < 0.0)
    for (int64_t i = lane; i < m; i += 32) qc[i] = -qc[i];
}


template <int CH, bool PF, bool FAST, int NT, int MINB>
int launch_cpqr(CpqrArgs& args, size_t smem, int Gmax, cudaStream_t st) {
  auto kern = cpqr_kernel<CH, PF, FAST, NT, MINB>;
  if (smem > 48 * 1024) LRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  LRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
  per_sm = std::max(1, std::min(per_sm, MINB));
  int G = std::min(per_sm * num_sms(), Gmax);
  // never more CTAs than NT/32-warp groups of columns
  G = (int)std::min<int64_t>(G, std::max<int64_t>(1, (args.n + NT / 32 - 1) / (NT / 32)));
  void* params[] = {&args};
  LRB_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(G), dim3(NT), params, smem, st));
  LRB_CHECK_LAUNCH();
  return G;
}

int cpqr_grid(int64_t n) {
  const int64_t max_g = std::max<int64_t>(1, (n + kGridWarpsPerCta - 1) / kGridWarpsPerCta);
  return (int)std::min<int64_t>(std::min(4 * num_sms(), kMaxG), max_g);
}

// CPQR kernel variant for the fast path (env LRB_CPQR_VARIANT selects for experiments)
int cpqr_fast_variant() {
  static int v = [] {
    const char* e = getenv("LRB_CPQR_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

}  // namespace

void cpqr_inplace(Workspace& ws, int64_t m, int64_t n, double* W, int64_t ld, int64_t k, int64_t* pivots,
                  double* tau, int* d_flags, long long* d_recomputes, bool padded, cudaStream_t st, bool nopivot) {
  if (!nopivot && cpqr_panel_supported(m, n, ld, padded)) {
    cpqr_panel(ws, m, n, W, ld, k, pivots, tau, d_flags, d_recomputes, st);
    return;
  }
  const int Gmax = cpqr_grid(n);
  const size_t cand_sz = kHdr + (size_t)m;
  // state: nrm, nrmx (n each), pval (2G), cand (2 G cand_sz), scratch (G 4m), ppos (2G)
  const size_t nd = 2 * (size_t)n + 2 * (size_t)Gmax + 2 * (size_t)Gmax * cand_sz + 4 * (size_t)Gmax * ld;
  const size_t bytes = sizeof(double) * nd + sizeof(long long) * 2 * (size_t)Gmax + 256;
  uint8_t* base = static_cast<uint8_t*>(ws.get(WsSlot::kCpqrState, bytes));
  CpqrArgs a{};
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
  a.cand = a.pval + 2 * Gmax;
  a.scratch = a.cand + 2 * (size_t)Gmax * cand_sz;
  a.ppos = reinterpret_cast<long long*>(a.scratch + 4 * (size_t)Gmax * ld);
  a.flags = d_flags;
  a.recomputes = reinterpret_cast<unsigned long long*>(d_recomputes);
  a.nopivot = nopivot ? 1 : 0;
  a.bar = reinterpret_cast<unsigned int*>(a.ppos + 2 * (size_t)Gmax);  // in the 256 B tail of the state
  LRB_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned int), st));
  const size_t smem = ld <= kMaxSmemRows ? 2 * sizeof(double) * (size_t)ld : 0;
  const bool fast = padded && ld % 64 == 0 && ld <= 512;
  if (fast) {
    switch (cpqr_fast_variant()) {
      // measured (tools/bench_cpqr.py, 510 x 65536): 1 CTA x 16 warps per SM with
      // register double buffering is fastest (fewer CTAs -> cheaper grid barrier)
      case 1: launch_cpqr<8, false, true, 512, 2>(a, smem, Gmax, st); break;   // 32 warps/SM, no prefetch
      case 2: launch_cpqr<8, false, true, 256, 4>(a, smem, Gmax, st); break;   // 4 CTAs/SM, no prefetch
      case 3: launch_cpqr<8, true, true, 256, 2>(a, smem, Gmax, st); break;    // 2 CTAs x 8 warps, prefetch
      default: launch_cpqr<8, true, true, 512, 1>(a, smem, Gmax, st); break;   // 1 CTA x 16 warps, prefetch
    }
  } else if (m <= 512) {
    launch_cpqr<8, true, false, 256, 2>(a, smem, Gmax, st);
  } else {
    launch_cpqr<16, false, false, 256, 2>(a, smem, Gmax, st);
  }
}

void cpqr_extract_s(int64_t m, int64_t n, const double* W, int64_t ld, int64_t k, double* s, int64_t lds,
                    cudaStream_t st) {
  (void)m;
  const int64_t total = k * n;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 16 * num_sms()));
  extract_s_kernel<<<g, 256, 0, st>>>(m, n, W, ld, k, s, lds);
  LRB_CHECK_LAUNCH();
}

void cpqr_form_q(int64_t m, int64_t n, const double* W, int64_t ld, int64_t k, const double* tau, double* q,
                 int64_t ldq, cudaStream_t st) {
  (void)n;
  const int wpb = 8;
  form_q_kernel<<<(unsigned)((k + wpb - 1) / wpb), wpb * 32, 0, st>>>(m, W, ld, k, tau, q, ldq);
  LRB_CHECK_LAUNCH();
}

}  // namespace lrb
