// gemm_tn.cu -- FP64 "TN" GEMM on the sm_100a DMMA pipe:
//
//     out(M x N) = alpha * P^T Q (+ beta * out)     P: K x M, Q: K x N
//
// with every operand column-major and K contiguous ("K-major").  This one
// shape class carries all dense contractions of the ID/CUR path:
//   sketch        Y   = Omega A          P = Omega^T (m x l), Q = A
//   ID coeffs     T   = S11^-1 S12       P = (S11^-1)^T,      Q = S12
//   C^+ A R^+     X^T = A^T C, W = X R^T, Gram / CholeskyQR2 products
//   error         ||A - C (U R)||_F       fused residual epilogue
//
// Design (B200): 128x128x16 CTA tile, 8 consumer warps each owning a 64x32
// warp tile (8x4 DMMA.8x8x4 tiles, 64 fp64 accumulators per thread) plus one
// TMA producer warp.  Operand tiles arrive through a 5-stage TMA ring
// (cp.async.bulk.tensor, 128B swizzle, mbarrier complete_tx); each 16-deep
// k-slice is read from shared memory with conflict-free LDS.128 by mapping
// MMA k-step t / quad q to physical k = 4q + t (the same permutation on both
// operands leaves the product unchanged).  One CTA per SM (160 KB smem,
// <=224 regs/thread); grid rasterised along the smaller tile dimension so
// CTAs sharing an operand tile run together and hit L2.
#include "common.cuh"
#include "kernels.h"

namespace lrb {

namespace {

constexpr int BM = 128, BN = 128, BK = 16;
constexpr int STAGES = 5;
constexpr int CONSUMER_WARPS = 8;
constexpr int THREADS = (CONSUMER_WARPS + 1) * 32;
constexpr int TILE_BYTES = BM * BK * 8;  // 16 KB per operand per stage
constexpr int STAGE_BYTES = 2 * TILE_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct EpiArgs {
  double* out;
  int64_t ldo;
  double alpha, beta;
  // residual epilogue
  const double* resid;  // R(M x N), ld
  int64_t ldr;
  double* partials;     // one (err2) per CTA
  // split-K partial epilogue
  double* ws;           // splits x M x N (ld M)
};

template <int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmp, const __grid_constant__ CUtensorMap tmq, int M, int N,
                   int K, int tiles_m, int tiles_n, int m_fast, int kt_per_split, EpiArgs ep, int upper, int tri) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bid = blockIdx.x;
  int tm, tn;
  if (upper) {  // tiles on or above the diagonal only (Gram products; tiles_m == tiles_n)
    int t = bid;
    tn = 0;
    while (t > tn) { t -= tn + 1; ++tn; }
    tm = t;
  } else if (m_fast) { tm = bid % tiles_m; tn = bid / tiles_m; }
  else { tn = bid % tiles_n; tm = bid / tiles_n; }
  const int m0 = tm * BM, n0 = tn * BN;
  const int KT = (K + BK - 1) / BK;
  // triangular operands: K-tiles that only meet structural zeros are skipped
  // (tri & 1: P(k, i) = 0 for k < i; tri & 2: Q(k, j) = 0 for k > j)
  int kt_begin = blockIdx.y * kt_per_split;
  int kt_end = min(KT, kt_begin + kt_per_split);
  if (tri & 1) kt_begin = max(kt_begin, m0 / BK);
  if (tri & 2) kt_end = min(kt_end, (n0 + BN) / BK);
  const int nkt = max(0, kt_end - kt_begin);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CONSUMER_WARPS) {
    // ---------------- TMA producer (one lane)
    if (lane == 0) {
      tma_prefetch_desc(&tmp);
      tma_prefetch_desc(&tmq);
      for (int i = 0; i < nkt; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sp = smem + s * STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        const int k = (kt_begin + i) * BK;
        tma_load_2d(sp, &tmp, &full[s], k, m0);
        tma_load_2d(sp + TILE_BYTES, &tmq, &full[s], k, n0);
      }
    }
    return;
  }

  // ---------------- DMMA consumers
  const int wm = warp & 1, wn = warp >> 1;
  const int q = lane & 3, r8 = lane >> 2;  // quad index, row-in-group
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // byte offsets within a swizzled [row][16 doubles] tile: row*128 + ((chunk ^ (row&7)) * 16)
  const uint32_t a_row0 = (wm * 64 + r8) * 128;
  const uint32_t b_row0 = (wn * 32 + r8) * 128;

  for (int i = 0; i < nkt; ++i) {
    const int s = i % STAGES;
    const uint32_t ph = (i / STAGES) & 1;
    mbar_wait(&full[s], ph);
    const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
    const uint32_t sb = sa + TILE_BYTES;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t chunk = ((2 * q + h) ^ r8) * 16;
      double2 a[8], b[4];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        const uint32_t addr = sa + a_row0 + rr * 8 * 128 + chunk;
        asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(a[rr].x), "=d"(a[rr].y) : "r"(addr));
      }
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const uint32_t addr = sb + b_row0 + cc * 8 * 128 + chunk;
        asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(b[cc].x), "=d"(b[cc].y) : "r"(addr));
      }
#pragma unroll
      for (int rr = 0; rr < 8; ++rr)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) dmma_8x8x4(acc[rr][cc][0], acc[rr][cc][1], a[rr].x, b[cc].x);
#pragma unroll
      for (int rr = 0; rr < 8; ++rr)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) dmma_8x8x4(acc[rr][cc][0], acc[rr][cc][1], a[rr].y, b[cc].y);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- epilogue: acc[rr][cc][v] = out(m, n)
  const int mb = m0 + wm * 64 + r8;
  const int nb = n0 + wn * 32 + 2 * q;
  if constexpr (EPI == kEpiStore) {
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int m = mb + rr * 8;
      if (m >= M) continue;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int n = nb + cc * 8 + v;
          if (n < N) {
            double* o = ep.out + (int64_t)m + (int64_t)n * ep.ldo;
            double x = ep.alpha * acc[rr][cc][v];
            if (ep.beta != 0.0) x += ep.beta * *o;
            *o = x;
          }
        }
    }
  } else if constexpr (EPI == kEpiSplitK) {
    double* ws = ep.ws + (int64_t)blockIdx.y * M * N;
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int m = mb + rr * 8;
      if (m >= M) continue;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int n = nb + cc * 8 + v;
          if (n < N) ws[(int64_t)m + (int64_t)n * M] = acc[rr][cc][v];
        }
    }
  } else {  // kEpiResid: sum (R - acc)^2 over the tile
    double e2 = 0.0;
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int m = mb + rr * 8;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int n = nb + cc * 8 + v;
          if (m < M && n < N) {
            const double d = ep.resid[(int64_t)m + (int64_t)n * ep.ldr] - acc[rr][cc][v];
            e2 = fma(d, d, e2);
          }
        }
    }
    e2 = warp_sum(e2);
    __shared__ double red[CONSUMER_WARPS];
    if (lane == 0) red[warp] = e2;
    // named barrier over the 8 consumer warps only (the producer has exited)
    asm volatile("bar.sync 1, %0;\n" ::"r"(CONSUMER_WARPS * 32));
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < CONSUMER_WARPS; ++w) t += red[w];
      ep.partials[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
  }
}

// deterministic split-K reduction: out = alpha * sum_s ws[s] + beta * out
__global__ void splitk_reduce_kernel(const double* __restrict__ ws, int splits, int M, int N, double* out,
                                     int64_t ldo, double alpha, double beta, int upper) {
  const int64_t total = (int64_t)M * N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    if (upper && (t % M) / BM > (t / M) / BN) continue;  // tile below the diagonal: not computed
    double s = 0.0;
    for (int p = 0; p < splits; ++p) s += ws[p * total + t];
    const int64_t m = t % M, n = t / M;
    double* o = out + m + n * ldo;
    double x = alpha * s;
    if (beta != 0.0) x += beta * *o;
    *o = x;
  }
}

template <int EPI>
void launch(const CUtensorMap& tp, const CUtensorMap& tq, int M, int N, int K, int splits, const EpiArgs& ep,
            cudaStream_t st, bool upper = false, int tri = 0) {
  static bool attr = false;
  if (!attr) {
    LRB_CUDA(cudaFuncSetAttribute(gemm_tn_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    attr = true;
  }
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int KT = (K + BK - 1) / BK;
  const int kt_per_split = (KT + splits - 1) / splits;
  dim3 grid(upper ? tiles_n * (tiles_n + 1) / 2 : tiles_m * tiles_n, splits);
  gemm_tn_kernel<EPI><<<grid, THREADS, SMEM_BYTES, st>>>(tp, tq, M, N, K, tiles_m, tiles_n, tiles_m <= tiles_n ? 1 : 0,
                                                         kt_per_split, ep, upper ? 1 : 0, tri);
  LRB_CHECK_LAUNCH();
}

}  // namespace

int gemm_tn_grid_ctas(int M, int N) { return ((M + BM - 1) / BM) * ((N + BN - 1) / BN); }

void gemm_tn(Workspace& ws, int M, int N, int K, const double* P, int64_t ldp, const double* Q, int64_t ldq,
             double* out, int64_t ldo, double alpha, double beta, int splits, cudaStream_t st, bool upper, int tri) {
  if (upper && M != N) throw CudaError("gemm_tn: upper-tile mode needs a square output");
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    scale_matrix(M, N, out, ldo, beta, st);
    return;
  }
  const CUtensorMap tp = make_tmap_f64(P, K, M, ldp, BK, BM, true);
  const CUtensorMap tq = make_tmap_f64(Q, K, N, ldq, BK, BN, true);
  EpiArgs ep{};
  ep.out = out;
  ep.ldo = ldo;
  ep.alpha = alpha;
  ep.beta = beta;
  const int KT = (K + BK - 1) / BK;
  if (splits <= 0) {
    // auto: when the output tiles are fewer than two waves of CTAs (one CTA
    // per SM), split K so that tiles x splits fills two waves as exactly as
    // possible (e.g. 10 upper Gram tiles -> 29 splits, 290 CTAs; powers of two
    // gave 320 = 2.2 waves), each split keeping >= 8 K-tiles
    const int tiles = upper ? ((N + BN - 1) / BN) * ((N + BN - 1) / BN + 1) / 2 : gemm_tn_grid_ctas(M, N);
    splits = 1;
    if (tiles < 2 * num_sms()) splits = std::max(1, std::min(KT / 8, (2 * num_sms()) / tiles));
  }
  splits = std::max(1, std::min(splits, KT));
  if (splits == 1) {
    launch<kEpiStore>(tp, tq, M, N, K, 1, ep, st, upper, tri);
    return;
  }
  double* w = ws.get_doubles(WsSlot::kSplitK, (size_t)splits * M * N);
  ep.ws = w;
  launch<kEpiSplitK>(tp, tq, M, N, K, splits, ep, st, upper, tri);
  const int64_t total = (int64_t)M * N;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8 * num_sms());
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(w, splits, M, N, out, ldo, alpha, beta, upper ? 1 : 0);
  LRB_CHECK_LAUNCH();
}

void gemm_tn_resid_sq(Workspace& ws, int M, int N, int K, const double* P, int64_t ldp, const double* Q,
                      int64_t ldq, const double* R, int64_t ldr, double* partials_out, int* num_partials,
                      cudaStream_t st) {
  const CUtensorMap tp = make_tmap_f64(P, K, M, ldp, BK, BM, true);
  const CUtensorMap tq = make_tmap_f64(Q, K, N, ldq, BK, BN, true);
  EpiArgs ep{};
  ep.resid = R;
  ep.ldr = ldr;
  ep.partials = partials_out;
  launch<kEpiResid>(tp, tq, M, N, K, 1, ep, st);
  *num_partials = gemm_tn_grid_ctas(M, N);
}

}  // namespace lrb
