// cpqr_panel.cuh -- state and device helpers shared by the eager panel CPQR
// (cpqr_panel.cu) and its bound-pruned variant (cpqr_lazy.cu).
#pragma once
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace lrb {
namespace cpqr_detail {

constexpr int NB = 32;       // panel width (one F entry per lane)
constexpr int CH = 8;        // 64-row chunks held in registers: ld <= 512
constexpr int PT = 256;      // threads per CTA (8 warps, one CTA per SM; up to 255 registers)
constexpr int kRowsPerThread = (64 * CH + PT - 1) / PT;
constexpr int PW = PT / 32;
constexpr int kMaxG = 256;       // per-CTA partials read by one warp (8 per lane)
constexpr int kHdr = 4;      // candidate header: alpha, beta, tau, apply
// dynamic shared memory: (NB+2) ld doubles (v, V, scratch) + per owned slot two
// norms and a logical position; the opt-in ceiling (227 KB) also holds the static arrays
constexpr int kSmemLimit = 216 * 1024;
inline size_t panel_smem_bytes(int64_t ld, int64_t maxcols) {
  // + logical positions, active list, zero list (ints)
  return sizeof(double) * ((size_t)(NB + 2) * ld + 2 * (size_t)maxcols) + sizeof(int) * 3 * (size_t)maxcols;
}

struct PanelArgs {
  double* W;
  int64_t m, n, ld, k;
  int64_t t0, t1;            // steps [t0, t1) of this launch (t1 - t0 <= NB)
  int init;                  // first launch: norms, pivots, first candidate
  int64_t* piv;
  double* nrm;
  double* nrmx;
  double* tau;
  double* pval;              // [2][G]
  long long* ppos;           // [2][G]
  double* cand;              // [2][G][kHdr + ld + NB]: reflector + w of each CTA's best column
  double* F;                 // [n][NB] row-major
  double* Vg;                // [ld][NB] row-major copy of the panel's V (GEMM operand)
  int* flags;
  unsigned long long* recomputes;
  unsigned long long* trace;  // optional per-phase ns of CTA 0 (LRB_CPQR_TRACE), 8 slots
  unsigned long long* tstep;  // optional per-step barrier arrival / departure times [k][G][2]
  unsigned int* bar;          // grid barrier counter (zeroed before each launch)
  int64_t maxcols;            // columns per CTA bound (shared-memory norm arrays)
  int* posof;                 // [n] logical position of each column slot (between launches)
  unsigned int* ctag;         // [G] step + 1 of the candidate each CTA last staged (release-published)
  int* nzero;                 // identically-zero columns found by the first launch
  int keep1024;               // the last keep1024/1024 of each warp's sweep is loaded L2::evict_last
  // lazy (bound-pruned) variant only
  int* cjg;                   // [n] panel reflectors already applied to each slot (between launches)
  double* wall;               // [NB][NB] w of each panel step (row c: V(:, i)^T v_c, i < c)
  unsigned int* epoch;        // rounds published so far (candidate tags / buffer parity across launches)
  double beta;                // > 0: fixed threshold factor; <= 0: adaptive
  int entry;                  // eager kernel after lazy panels: stage the step-t0 candidate first
  double gap_miss;            // growth of 1 - beta after a retry round (0: default)
  unsigned long long* lstats; // [0] retry rounds, [1] columns evaluated by the step passes, [2] 1 - beta (double bits)
};

// Grid barrier for the co-resident (cooperative) grid: one release atomic per
// CTA on a monotonic counter and an acquire spin without back-off.  (The
// cooperative-groups grid.sync measured ~9 us per barrier here; this one is
// the latency of an L2 atomic round trip plus the last arrival.)
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int& target) {
  target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    // release: the CTA's writes (ordered before this thread by the barrier) become visible gpu-wide
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// the two halves of grid_barrier: publish (after the CTA's partial is
// written) and wait -- the candidate staging runs in between
__device__ __forceinline__ void grid_arrive(unsigned int* bar, unsigned int& target) {
  target += gridDim.x;
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void grid_wait(const unsigned int* bar, unsigned int target) {
  if (threadIdx.x == 0) {
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// A CTA's candidate tag is monotonic within one CPQR call (reset to ~0u: none
// staged yet).  A waiter accepts any tag >= the one it needs: the owner may
// already have staged its next round's candidate (other buffer parity) while a
// slow CTA is still reading this round's -- waiting for equality would then
// deadlock the grid.
__device__ __forceinline__ bool tag_ready(unsigned int t, unsigned int want) {
  return t != ~0u && (int)(t - want) >= 0;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ bool better(double v1, long long p1, double v2, long long p2) {
  return v1 > v2 || (v1 == v2 && p1 < p2);
}

// column loads with an L2 eviction priority: the columns a warp visits last in
// step s are the ones it visits first in step s + 1 (the sweep alternates
// direction), so they are kept (evict_last) and the rest streamed (evict_first)
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t p;
  if (keep)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_l2hint(const double2* ptr, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(ptr), "l"(pol));
  return r;
}

__device__ __forceinline__ double cta_sum(double x, double* sh) {
  x = warp_sum(x);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[w] = x;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < PW; ++i) t += sh[i];
  return t;
}


// group version of the recompute (L lanes per column): rows s+1..m-1 of the
// column re-read from W (L2-hot), F(j, 0:c] from global (written by the group)
template <int L>
__device__ __forceinline__ double group_recompute(const double* col, const double* Fj, int64_t s, int64_t m,
                                               int64_t ld, int c, const double* Vs, int l) {
  double q = 0.0;
  for (int64_t r = s + 1 + l; r < m; r += L) {
    double x = col[r];
    for (int i = 0; i <= c; ++i) x = fma(-Vs[i * ld + r], Fj[i], x);
    q = fma(x, x, q);
  }
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  return q;
}

// ---------------------------------------------------------------- lazy variant (cpqr_lazy.cu)
constexpr double kLazyBoundEps = 1e-10;  // ub = nr + kLazyBoundEps * nx
constexpr int NBL = 16;                  // steps per lazy panel (catch-ups span at most NBL - 1 steps)
inline size_t lazy_smem_bytes(int64_t ld, int64_t maxcols) {
  // eager layout + per slot the catch-up level and the step's evaluation list
  return panel_smem_bytes(ld, maxcols) + sizeof(int) * 2 * (size_t)maxcols;
}
struct FinArgs {
  double* W;
  int64_t ld, m, n, t0, t1, r1;
  int C, upd;
  const double* Vg;     // [ld][NB] row-major
  double* F;            // [n][NB]
  const double* tau;    // tau of steps t0 .. t1
  const double* wall;   // [NB][NB]
  double* nrm;
  double* nrmx;
  const int* cj;
  unsigned long long* recomputes;
};
constexpr int FW = 16;  // panel_finalize_kernel: warps per CTA
constexpr int FVR = 24;  // row stride of its reflector-contiguous V copy (== 8 mod 16: conflict-free 16-byte loads)
inline size_t finalize_smem_bytes(int64_t ld, int64_t t0) {
  // V(t0:ld, 0:NBL) twice (reflector- and row-contiguous), w of each step, tau
  return sizeof(double) * ((size_t)(ld - t0) * FVR + (size_t)NBL * (size_t)(ld - t0 + 8) + NB * NB + NB);
}
using PanelKernT = void (*)(PanelArgs);
// the lazy kernel for ld = 64 nld and first active chunk tc
PanelKernT lazy_kernel_for(int nld, int tc, bool list);
void lazy_set_attributes();
void launch_panel_finalize(const FinArgs& f, int grid, cudaStream_t st);

}  // namespace cpqr_detail
}  // namespace lrb
