// ozaki.cu -- FP64 GEMM emulated on the sm_100a INT8 tensor cores (tcgen05
// kind::i8, TMEM accumulators, TMA operand staging), Ozaki scheme II style:
//
//   1. scale: every column of P (K x M) and Q (K x N) (K contiguous) gets a
//      power-of-two shift so |x| 2^s < 2^beta, and x' = rint(x 2^s) is an exact
//      integer (|x'| <= 2^beta, beta chosen so K 2^(2 beta) < M_crt / 2);
//   2. residues: x' mod m_t for 16 pairwise-coprime moduli m_t <= 256, stored
//      as symmetric int8 planes in the same K-major layout;
//   3. 16 INT8 GEMMs: C_t = P_t^T Q_t with exact int32 accumulation
//      (|terms| <= 2^14, K <= 2^17), reduced mod m_t in the epilogue;
//   4. CRT: C' = sum_t c_t (M/m_t) ((M/m_t)^-1 mod m_t) mod M in int128 (M <
//      2^127), C = C' 2^-(s_i + t_j) rounded to double.
// The integer product is exact; the only error is the input truncation to
// beta >= 53 bits relative to each column's largest entry, so the result is
// as accurate as an FP64 GEMM (accumulation itself is exact here).  The scaled
// residue planes of an operand can be kept and reused: A enters both big
// contractions of the CUR with the same per-column scaling.
#include <climits>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace lrb {

namespace {

constexpr int kMod[kOzakiModuli] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
// the same list as a compile-time function usable in unrolled device loops
__host__ __device__ constexpr int kmod(int t) {
  return t == 0 ? 256 : t == 1 ? 255 : t == 2 ? 253 : t == 3 ? 251 : t == 4 ? 247 : t == 5 ? 241 : t == 6 ? 239
       : t == 7 ? 233 : t == 8 ? 229 : t == 9 ? 227 : t == 10 ? 223 : t == 11 ? 217 : t == 12 ? 211
       : t == 13 ? 199 : t == 14 ? 197 : 193;
}
// CRT constants for the 16 moduli (checked against crt_host() at first use)
__host__ __device__ constexpr int kcrt_inv(int t) {
  return t == 0 ? 33 : t == 1 ? 224 : t == 2 ? 195 : t == 3 ? 157 : t == 4 ? 135 : t == 5 ? 5 : t == 6 ? 184 : t == 7 ? 231 : t == 8 ? 30 : t == 9 ? 125 : t == 10 ? 34 : t == 11 ? 69 : t == 12 ? 138 : t == 13 ? 45 : t == 14 ? 125 : 116;
}
__host__ __device__ constexpr unsigned long long kcrt_lo(int t) {
  return t == 0 ? 0x4f49e5694da9b2e1ull : t == 1 ? 0xdc260b74c26c1f00ull : t == 2 ? 0x9d2149451d00b500ull : t == 3 ? 0xce517cd98d6cd300ull : t == 4 ? 0xbf00edc53ccce700ull : t == 5 ? 0xf38f4acb35d0f100ull : t == 6 ? 0x6fb4e8e030e92f00ull : t == 7 ? 0x400adf7d96273900ull : t == 8 ? 0xe460060ca2d64d00ull : t == 9 ? 0x22287b63959c6b00ull : t == 10 ? 0x1d07eaa91a043f00ull : t == 11 ? 0xbe46a92f8bfd4900ull : t == 12 ? 0x163067a0850cfb00ull : t == 13 ? 0x64b68a2d6a571700ull : t == 14 ? 0x20dcc75b5bd36d00ull : 0x104ccb7d161a2100ull;
}
__host__ __device__ constexpr unsigned long long kcrt_hi(int t) {
  return t == 0 ? 0x2984652cbaccc5ull : t == 1 ? 0x29ae133ffac78cull : t == 2 ? 0x2a026c7210ffc4ull : t == 3 ? 0x2a581dc182587full : t == 4 ? 0x2b07aa28241161ull : t == 5 ? 0x2c19e9e0e86b0aull : t == 6 ? 0x2c7863cd5e0b89ull : t == 7 ? 0x2d9d8cd3c1274dull : t == 8 ? 0x2e698658032147ull : t == 9 ? 0x2ed235339261dbull : t == 10 ? 0x2fa93501fc538aull : t == 11 ? 0x30fa914fe6fd5eull : t == 12 ? 0x325f1d5499d7afull : t == 13 ? 0x3568b59c98d3f7ull : t == 14 ? 0x35f384c67897beull : 0x3711c48aea8303ull;
}
__constant__ int c_mod[kOzakiModuli];
__constant__ double c_inv_mod[kOzakiModuli];
__constant__ unsigned long long c_Mt[kOzakiModuli][2];  // M / m_t (low, high limbs)
__constant__ int c_crt_inv[kOzakiModuli];               // (M / m_t)^-1 mod m_t
__constant__ unsigned long long c_Mcrt[2];
// c_t = (M / m_t) ((M / m_t)^-1 mod m_t) < M as 32-bit limbs; C' = sum_t r_t c_t mod M
__constant__ uint32_t c_crt_c[kOzakiModuli][4];
__constant__ unsigned long long c_crt_k0[2];  // 128 sum_t c_t mod 2^128 (residue offset r + 128)
__constant__ double c_crt_invM, c_crt_k0M;    // 1 / M, 128 sum_t c_t / M

typedef unsigned __int128 u128;
typedef __int128 i128;

struct CrtHost {
  u128 M = 1;
  u128 Mt[kOzakiModuli];
  int inv[kOzakiModuli];
  double log2M = 0.0;
};

u128 mod_pow_inv(u128 a, int m) {
  // inverse of (a mod m) modulo m by brute force (m <= 256)
  const int r = (int)(a % (u128)m);
  for (int x = 1; x < m; ++x)
    if ((r * x) % m == 1) return (u128)x;
  return 0;
}

const CrtHost& crt_host() {
  static CrtHost h = [] {
    CrtHost c;
    for (int t = 0; t < kOzakiModuli; ++t) c.M *= (u128)kMod[t];
    for (int t = 0; t < kOzakiModuli; ++t) {
      c.Mt[t] = c.M / (u128)kMod[t];
      c.inv[t] = (int)mod_pow_inv(c.Mt[t], kMod[t]);
    }
    c.log2M = 0.0;
    for (int t = 0; t < kOzakiModuli; ++t) c.log2M += std::log2((double)kMod[t]);
    return c;
  }();
  return h;
}

void upload_constants() {
  static bool done = false;
  if (done) return;
  const CrtHost& h = crt_host();
  for (int t = 0; t < kOzakiModuli; ++t)
    if (kmod(t) != kMod[t] || kcrt_inv(t) != h.inv[t] || kcrt_lo(t) != (unsigned long long)h.Mt[t] ||
        kcrt_hi(t) != (unsigned long long)(h.Mt[t] >> 64))
      throw CudaError("ozaki: compiled CRT constants disagree with the moduli");
  double inv[kOzakiModuli];
  unsigned long long mt[kOzakiModuli][2], mm[2];
  for (int t = 0; t < kOzakiModuli; ++t) {
    inv[t] = 1.0 / kMod[t];
    mt[t][0] = (unsigned long long)(h.Mt[t]);
    mt[t][1] = (unsigned long long)(h.Mt[t] >> 64);
  }
  mm[0] = (unsigned long long)h.M;
  mm[1] = (unsigned long long)(h.M >> 64);
  LRB_CUDA(cudaMemcpyToSymbol(c_mod, kMod, sizeof kMod));
  LRB_CUDA(cudaMemcpyToSymbol(c_inv_mod, inv, sizeof inv));
  LRB_CUDA(cudaMemcpyToSymbol(c_Mt, mt, sizeof mt));
  LRB_CUDA(cudaMemcpyToSymbol(c_crt_inv, h.inv, sizeof h.inv));
  LRB_CUDA(cudaMemcpyToSymbol(c_Mcrt, mm, sizeof mm));
  uint32_t cl[kOzakiModuli][4];
  u128 k0 = 0;
  double k0M = 0.0;
  for (int t = 0; t < kOzakiModuli; ++t) {
    const u128 ct = h.Mt[t] * (u128)h.inv[t];  // < M: inv < m_t
    for (int i = 0; i < 4; ++i) cl[t][i] = (uint32_t)(ct >> (32 * i));
    k0 += (u128)128 * ct;  // mod 2^128
    k0M += 128.0 * ((double)ct / (double)h.M);
  }
  const unsigned long long k0w[2] = {(unsigned long long)k0, (unsigned long long)(k0 >> 64)};
  const double invM = 1.0 / (double)h.M;
  LRB_CUDA(cudaMemcpyToSymbol(c_crt_c, cl, sizeof cl));
  LRB_CUDA(cudaMemcpyToSymbol(c_crt_k0, k0w, sizeof k0w));
  LRB_CUDA(cudaMemcpyToSymbol(c_crt_invM, &invM, sizeof invM));
  LRB_CUDA(cudaMemcpyToSymbol(c_crt_k0M, &k0M, sizeof k0M));
  done = true;
}

// ------------------------------------------------------------ 1+2: scale and split
// Pass 1 (colmax_kernel): max|x| per column into an int64 bit pattern (non-
// negative doubles order like their bit patterns) with atomicMax.
// Pass 2 (split_kernel): x' = rint(x 2^s) once per element in FP64, then the
// 16 residues without per-modulus FP64 work:
//   * moduli in 8 pairs, P = m1 m2 < 2^16: r = x' - rint(x'/P) P (DFMA, exact
//     integer, |r| < 2^17), moved into FP32 as the bit pattern 1.5*2^23 + r;
//   * per modulus in FP32: q = rint(r/m) by the magic-add trick, then
//     y = 1.5*2^23 + r - q m (FFMA, exact) whose low mantissa byte is the
//     symmetric residue (|r/m - q| < 1/2 is never misrounded: the fp32
//     reciprocal error |r| 2^-24/m < 2^-14 is below 1/(2m), the distance of
//     r/m from a half-integer for odd m; 1/256 is exact);
//   * bytes of 4 consecutive K entries are packed per plane (PRMT), one
//     coalesced 4-byte store per plane.
constexpr int kSplitRows = 8;  // K entries per thread per tile
constexpr int kOzakiNonFinite = INT_MIN;  // shift sentinel of a column with NaN / Inf
constexpr int kSplitThreads = 256;
constexpr int kSplitTile = kSplitRows * kSplitThreads;

constexpr int kMaxRowsPerThread = 32;  // colmax: 8192-row tiles, 16 double2 loads in flight per thread
__global__ void __launch_bounds__(256) colmax_kernel(int64_t K, int64_t cols, const double* __restrict__ X,
                                                     int64_t ldx, bool vec2, unsigned long long* __restrict__ cmax) {
  __shared__ unsigned long long sh[8];
  constexpr int64_t kTile = (int64_t)kMaxRowsPerThread * kSplitThreads;
  const int64_t tiles_k = (K + kTile - 1) / kTile;
  for (int64_t t = blockIdx.x; t < tiles_k * cols; t += gridDim.x) {
    const int64_t j = t / tiles_k, i0 = (t % tiles_k) * kTile;
    const double* x = X + j * ldx;
    // max of |x| as a bit pattern: NaN / Inf patterns exceed every finite one,
    // so a non-finite column is recognised by the split (fmax would drop NaN)
    unsigned long long mx = 0;
    if (vec2 && i0 + kTile <= K) {
      double2 r[kMaxRowsPerThread / 2];
#pragma unroll
      for (int e = 0; e < kMaxRowsPerThread / 2; ++e)
        r[e] = __ldcs(reinterpret_cast<const double2*>(x + i0 + 2 * (e * kSplitThreads + threadIdx.x)));
#pragma unroll
      for (int e = 0; e < kMaxRowsPerThread / 2; ++e) {
        mx = max(mx, (unsigned long long)__double_as_longlong(fabs(r[e].x)));
        mx = max(mx, (unsigned long long)__double_as_longlong(fabs(r[e].y)));
      }
    } else {
      for (int64_t i = i0 + threadIdx.x; i < K && i < i0 + kTile; i += kSplitThreads)
        mx = max(mx, (unsigned long long)__double_as_longlong(fabs(x[i])));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = sh[0];
      for (int w = 1; w < kSplitThreads / 32; ++w) m = max(m, sh[w]);
      if (m > 0) atomicMax(cmax + j, m);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// One tile of kSplitRows consecutive K entries of a column: scale, reduce mod
// the pairs, then the 16 residues (see above), stored 8 bytes per plane.
template <bool UNS>
__device__ __forceinline__ void split_tile(const double (&v)[kSplitRows], double sc1, double sc2,
                                           int8_t* __restrict__ out, int64_t plane_stride) {
  constexpr double M52 = 6755399441055744.0;  // 1.5 * 2^52
  constexpr float M23 = 12582912.0f;          // 1.5 * 2^23
  double xp[kSplitRows];
#pragma unroll
  for (int q = 0; q < kSplitRows; ++q) xp[q] = rint((v[q] * sc1) * sc2);  // exact, |xp| <= 2^beta
#pragma unroll
  for (int g = 0; g < kOzakiModuli / 2; ++g) {
    const double P = (double)(kmod(2 * g) * kmod(2 * g + 1));
    const double invP = 1.0 / P;
    uint32_t b0[kSplitRows], b1[kSplitRows];
#pragma unroll
    for (int q = 0; q < kSplitRows; ++q) {
      const double qg = fma(xp[q], invP, M52) - M52;
      const double r = fma(-qg, P, xp[q]);  // exact, |r| < 2^17
      if constexpr (UNS) {
        const int iP = kmod(2 * g) * kmod(2 * g + 1);
        const double bias = M52 + (double)(iP * ((131072 + iP - 1) / iP));  // M52 + B_P
        const uint32_t u = (uint32_t)__double2loint(r + bias);             // r + B_P in [0, 2^18)
        const uint32_t m0 = (uint32_t)kmod(2 * g), m1 = (uint32_t)kmod(2 * g + 1);
        b0[q] = u - m0 * __umulhi(u, (uint32_t)((0x100000000ull + m0 - 1) / m0));  // u mod m
        b1[q] = u - m1 * __umulhi(u, (uint32_t)((0x100000000ull + m1 - 1) / m1));
      } else {
        const int lo = __double2loint(r + M52);
        const float fb = __int_as_float(0x4B400000 + lo);  // 1.5*2^23 + r
        const float rf = fb - M23;                           // r
        const float m0 = (float)kmod(2 * g), m1 = (float)kmod(2 * g + 1);
        const float q0 = fmaf(rf, 1.0f / m0, M23) - M23;
        const float q1 = fmaf(rf, 1.0f / m1, M23) - M23;
        b0[q] = (uint32_t)__float_as_int(fmaf(-q0, m0, fb));  // 1.5*2^23 + residue, exact
        b1[q] = (uint32_t)__float_as_int(fmaf(-q1, m1, fb));
      }
    }
    static_assert(kSplitRows == 8, "two packed words per plane");
    __stcs(reinterpret_cast<uint2*>(out + (2 * g) * plane_stride),
           make_uint2(pack4(b0[0], b0[1], b0[2], b0[3]), pack4(b0[4], b0[5], b0[6], b0[7])));
    __stcs(reinterpret_cast<uint2*>(out + (2 * g + 1) * plane_stride),
           make_uint2(pack4(b1[0], b1[1], b1[2], b1[3]), pack4(b1[4], b1[5], b1[6], b1[7])));
  }
}

// UNS: residues t = x' mod m in [0, m) for the u8 operand: the pair remainder
// comes out of the FP64 stage already biased positive (u = r + B_P, B_P a
// multiple of P >= 2^17, folded into the low-word constant) and t = u - m
// umulhi(u, ceil(2^32/m)) is exact for u < 2^24.  Two integer ops per
// modulus instead of three FP32 ones plus the rebias.
template <bool UNS>
__global__ void __launch_bounds__(256) split_kernel(int64_t K, int64_t cols, const double* __restrict__ X,
                                                    int64_t ldx, bool vec2, int beta,
                                                    const unsigned long long* __restrict__ cmax,
                                                    int8_t* __restrict__ planes, int64_t ldp, int64_t plane_stride,
                                                    int* __restrict__ shift) {
  // a CTA walks whole columns (j += gridDim.x) tile by tile: no index
  // division, one scale per column, and a software pipeline: the next tile's
  // 4 values are in flight while this tile's 64 residues are computed and stored
  const int tiles_k = (int)((K + kSplitTile - 1) / kSplitTile);
  const int64_t r_off = (int64_t)kSplitRows * threadIdx.x;
  auto load = [&](int64_t j, int tk, double (&v)[kSplitRows]) {
    const int64_t i0 = (int64_t)tk * kSplitTile + r_off;
    const double* x = X + j * ldx + i0;
    if (vec2 && i0 + kSplitRows <= K) {
#pragma unroll
      for (int h = 0; h < kSplitRows / 2; ++h) {
        const double2 a = __ldcs(reinterpret_cast<const double2*>(x + 2 * h));
        v[2 * h] = a.x;
        v[2 * h + 1] = a.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < kSplitRows; ++q) v[q] = i0 + q < K ? x[q] : 0.0;
    }
  };
  double v[kSplitRows], vn[kSplitRows];
  int64_t j = blockIdx.x;
  int tk = 0;
  if (j < cols) load(j, 0, v);
  while (j < cols) {
    const double mx = __longlong_as_double((long long)cmax[j]);
    int e = 0;
    if (mx > 0.0 && isfinite(mx)) frexp(mx, &e);  // mx < 2^e
    const int sft = (mx > 0.0 && isfinite(mx)) ? beta - e : 0;
    // non-finite column: the sentinel makes every product entry NaN (crt_kernel)
    if (threadIdx.x == 0) shift[j] = isfinite(mx) ? sft : kOzakiNonFinite;
    const double sc1 = ldexp(1.0, sft / 2), sc2 = ldexp(1.0, sft - sft / 2);
    int8_t* colp = planes + j * ldp;
    for (; tk < tiles_k; ++tk) {
      // prefetch the next tile (this column's next one, or the next column's first)
      const bool last = tk + 1 == tiles_k;
      const int64_t jn = last ? j + gridDim.x : j;
      const int tkn = last ? 0 : tk + 1;
      if (jn < cols) load(jn, tkn, vn);
      const int64_t i0 = (int64_t)tk * kSplitTile + r_off;
      if (i0 < K) split_tile<UNS>(v, sc1, sc2, colp + i0, plane_stride);
#pragma unroll
      for (int q = 0; q < kSplitRows; ++q) v[q] = vn[q];
    }
    tk = 0;
    j += gridDim.x;
  }
}

// ------------------------------------------------------------ 3: tcgen05 INT8 GEMM
// One CTA owns a 128 x 512 output tile of one plane (two 128x256 UMMAs into
// all 512 TMEM columns).  Clusters of 4 CTAs stacked along M share the same
// 512 Q columns: each CTA TMA-loads a 128-column slice of the Q stage and
// multicasts it to the whole cluster, so a CTA pulls 8 KB (own P) + 8 KB (its
// Q slice) from L2 per 64-byte K step for 128x512x64 MACs -- about 32 B per
// 1024 MMA clocks, inside the per-SM share of L2 bandwidth.  Stage release is
// cluster-wide: every CTA's MMA commit arrives on the stage's empty barrier
// in all four CTAs (count 4).
constexpr int IBM = 128, IBN = 512, IBK = 64;  // tile; K in bytes (= int8 elements) per stage
constexpr int ICL = 4;                         // cluster size along M (largest; 2 and 1 for short M)
constexpr int ISTAGES = 5;
constexpr int IA_BYTES = IBM * IBK, IB_BYTES = IBN * IBK;
constexpr int ISTAGE_BYTES = IA_BYTES + IB_BYTES;
constexpr int ITHREADS = 6 * 32;  // warp 0 TMA, warp 1 MMA + TMEM, warps 2-5 epilogue
constexpr int ISMEM = ISTAGES * ISTAGE_BYTES + 1024 + 256;
constexpr uint32_t kTmemCols = 512;

__device__ __forceinline__ uint64_t smem_desc_sw64(uint32_t saddr) {
  // K-major, SWIZZLE_64B: 8-row x 64 B atoms, SBO = 512 B between atoms, LBO unused (1), version 1, layout 4
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

__device__ __forceinline__ uint64_t smem_desc_sw128_mn(uint32_t saddr) {
  // MN-major, SWIZZLE_128B (canonical ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16-byte units): 128 bytes
  // (= 128 int8 rows of the tile) contiguous along M, K rows at a 128-byte pitch, 8-row groups
  // SBO = 1024 B apart; one 128-byte group along M (n = 1), so LBO (the tile size) is never used
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4, %5}], [%2], %6;\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

// CL: CTAs per cluster along M sharing the Q tile by multicast (4 when the M
// tiles come in fours; 2 / 1 for short M, e.g. C3's l = 210 = 2 tiles, which a
// 4-cluster would pad to 4 tiles of mostly zero rows)
template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(ITHREADS, 1)
    imma_gemm_kernel(const __grid_constant__ CUtensorMap tmp, const __grid_constant__ CUtensorMap tmq, int M, int N,
                     int K, int8_t* __restrict__ out, int64_t ldo, int64_t out_plane_stride, uint32_t ab_fmt,
                     int p_mn) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ISTAGES * ISTAGE_BYTES);
  uint64_t* empty = full + ISTAGES;
  uint64_t* tmem_full = empty + ISTAGES;
  uint32_t* tmem_base_sh = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int plane = blockIdx.z;
  const uint32_t rank = cluster_rank();
  const int m0 = blockIdx.x * IBM, n0 = blockIdx.y * IBN;
  const int nkb = (K + IBK - 1) / IBK;

  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < ISTAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], CL);
      }
      mbar_init(tmem_full, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_base_sh)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  cluster_sync_all();  // barriers of every CTA initialised before any multicast lands
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmp);
      tma_prefetch_desc(&tmq);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ISTAGES;
        const uint32_t ph = (i / ISTAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);  // stage s free in all four CTAs
        uint8_t* sp = smem + s * ISTAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], ISTAGE_BYTES);
        // P stage: K-major planes [K][M] (box 64 K-bytes x 128 rows, 64B swizzle) or, p_mn, the
        // planes of the transposed operand [M][K] (box 128 M-bytes x 64 K rows, 128B swizzle)
        if (p_mn) tma_load_3d(sp, &tmp, &full[s], m0, i * IBK, plane);
        else tma_load_3d(sp, &tmp, &full[s], i * IBK, m0, plane);
        // this CTA's 512 / CL columns of the Q stage, in TMA boxes of at most 256 columns
        constexpr int kBox = IBN / CL < 256 ? IBN / CL : 256;
#pragma unroll
        for (int t = 0; t < IBN / CL / kBox; ++t)
          tma_load_3d_mc(sp + IA_BYTES + rank * (IB_BYTES / CL) + t * kBox * IBK, &tmq, &full[s], i * IBK,
                         n0 + (int)rank * (IBN / CL) + t * kBox, plane, (uint16_t)((1u << CL) - 1));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::i8: D s32; A/B u8 (0) or s8 (1) per operand (ab_fmt bits 7, 10)
      // bit 15: A (our P) is MN-major in shared memory
      const uint32_t idesc = (2u << 4) | ab_fmt | (p_mn ? (1u << 15) : 0u) | ((uint32_t)(256 >> 3) << 17) |
                             ((uint32_t)(IBM >> 4) << 24);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ISTAGES;
        const uint32_t ph = (i / ISTAGES) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t sa = smem_u32(smem + s * ISTAGE_BYTES);
        const uint32_t sb = sa + IA_BYTES;
#pragma unroll
        for (int kk = 0; kk < IBK / 32; ++kk) {
          // 32 K entries further: 32 bytes along a K-major row, 32 rows of 128 bytes MN-major
          const uint64_t da = p_mn ? smem_desc_sw128_mn(sa + kk * 32 * IBM) : smem_desc_sw64(sa + kk * 32);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint64_t db = smem_desc_sw64(sb + h * 256 * IBK + kk * 32);
            const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + h * 256),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
        }
        // frees stage s in every CTA of the cluster once these MMAs have read it
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                smem_u32(&empty[s])),
            "h"((uint16_t)((1u << CL) - 1))
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(tmem_full))
                   : "memory");
    }
    __syncwarp();
  } else {
    // epilogue: TMEM lane quadrant (warp % 4) -> rows 32q .. 32q+31
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int q = warp & 3;
    const int row = m0 + 32 * q + lane;
    const int mod = c_mod[plane];
    const double inv = c_inv_mod[plane];
    int8_t* o = out + (int64_t)plane * out_plane_stride;
    const int ncols = min(IBN, N - n0);
    for (int c0 = 0; c0 < ncols; c0 += 16) {
      uint32_t v[16];
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (row < M) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int col = n0 + c0 + e;
          if (col < N) {
            const double x = (double)(int)v[e];
            const int r = (int)fma(-rint(x * inv), (double)mod, x);  // |r| <= m/2 (+1 at an inexact tie)
            o[(int64_t)col * ldo + row] = (int8_t)r;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  cluster_sync_all();  // no CTA leaves while cluster peers may still signal its barriers
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
  }
}

// ------------------------------------------------------------ 4: CRT reconstruction
__global__ void crt_kernel(int64_t M, int64_t N, const int8_t* __restrict__ res, int64_t ldr, int64_t plane_stride,
                           const int* __restrict__ shift_p, const int* __restrict__ shift_q, double* __restrict__ out,
                           int64_t ldo, double alpha, double beta) {
  const i128 Mc = (i128)(((u128)c_Mcrt[1] << 64) | (u128)c_Mcrt[0]);
  const i128 half = Mc >> 1;
  // 2D walk (rows fastest): no per-element 64-bit index division; moduli,
  // inverses and M / m_t are compile-time constants of the unrolled loop
  for (int64_t j = blockIdx.y; j < N; j += gridDim.y) {
    const int sq = shift_q[j];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
      const int8_t* r = res + j * ldr + i;
      // T = sum_t (r_t + 128) c_t exactly in four 64-bit limb accumulators
      // (32x32 -> 64 multiply-adds; each limb sum < 2^44), then one quotient
      // q = round((T - K0) / M) in FP64 (|C'| <= 0.39 M at the largest K, far
      // from the rounding boundary) and C' = T - K0 - q M in wrapping 128-bit
      // arithmetic; the final +-M step only guards the quotient
      unsigned long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
      for (int p = 0; p < kOzakiModuli; ++p) {
        const uint32_t rp = (uint32_t)((int)r[p * plane_stride] + 128);
        a0 += (unsigned long long)c_crt_c[p][0] * rp;
        a1 += (unsigned long long)c_crt_c[p][1] * rp;
        a2 += (unsigned long long)c_crt_c[p][2] * rp;
        a3 += (unsigned long long)c_crt_c[p][3] * rp;
      }
      const double td = fma(fma(fma((double)a3, 4294967296.0, (double)a2), 4294967296.0, (double)a1), 4294967296.0,
                            (double)a0);
      const long long q = __double2ll_rn(fma(td, c_crt_invM, -c_crt_k0M));
      const u128 T = (u128)a0 + ((u128)a1 << 32) + ((u128)a2 << 64) + ((u128)a3 << 96);
      const u128 K0 = ((u128)c_crt_k0[1] << 64) | (u128)c_crt_k0[0];
      i128 s = (i128)(T - K0 - (u128)(i128)q * (u128)Mc);
      if (s > half) s -= Mc;
      else if (s < -half) s += Mc;
      // int128 -> double (round to nearest via the high/low split), then unscale
      const bool neg = s < 0;
      const u128 a = neg ? (u128)(-s) : (u128)s;
      const double hi = (double)(unsigned long long)(a >> 64);
      const double lo = (double)(unsigned long long)a;
      double v = fma(hi, 18446744073709551616.0, lo);
      if (neg) v = -v;
      const int sp = shift_p[i];
      v = (sp == kOzakiNonFinite || sq == kOzakiNonFinite) ? CUDART_NAN : ldexp(v, -(sp + sq));
      double* o = out + i + j * ldo;
      *o = beta == 0.0 ? alpha * v : alpha * v + beta * *o;
    }
  }
}

// Same reconstruction, four consecutive rows per thread: one 4-byte load per
// plane instead of four byte loads (the residue planes have ldr % 16 == 0).
__global__ void __launch_bounds__(256, 3) crt4_kernel(int64_t M, int64_t N, const int8_t* __restrict__ res, int64_t ldr, int64_t plane_stride,
                            const int* __restrict__ shift_p, const int* __restrict__ shift_q, double* __restrict__ out,
                            int64_t ldo, double alpha, double beta) {
  const i128 Mc = (i128)(((u128)c_Mcrt[1] << 64) | (u128)c_Mcrt[0]);
  const i128 half = Mc >> 1;
  const u128 K0 = ((u128)c_crt_k0[1] << 64) | (u128)c_crt_k0[0];
  // flattened (row group, column) work items so short columns keep every lane busy
  const int64_t G = (M + 3) / 4;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < G * N; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = w / G;
    const int64_t i0 = 4 * (w - j * G);
    const int sq = shift_q[j];
    {
      const int8_t* r = res + j * ldr + i0;
      unsigned long long a[4][4];
#pragma unroll
      for (int e = 0; e < 4; ++e) a[e][0] = a[e][1] = a[e][2] = a[e][3] = 0ull;
#pragma unroll
      for (int p = 0; p < kOzakiModuli; ++p) {
        const uint32_t w = __ldcs(reinterpret_cast<const unsigned int*>(r + p * plane_stride));
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t rp = ((w >> (8 * e)) & 0xffu) ^ 0x80u;  // signed residue + 128
          a[e][0] += (unsigned long long)c_crt_c[p][0] * rp;
          a[e][1] += (unsigned long long)c_crt_c[p][1] * rp;
          a[e][2] += (unsigned long long)c_crt_c[p][2] * rp;
          a[e][3] += (unsigned long long)c_crt_c[p][3] * rp;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t i = i0 + e;
        if (i >= M) break;
        const double td = fma(fma(fma((double)a[e][3], 4294967296.0, (double)a[e][2]), 4294967296.0,
                                  (double)a[e][1]), 4294967296.0, (double)a[e][0]);
        const long long q = __double2ll_rn(fma(td, c_crt_invM, -c_crt_k0M));
        const u128 T = (u128)a[e][0] + ((u128)a[e][1] << 32) + ((u128)a[e][2] << 64) + ((u128)a[e][3] << 96);
        i128 sv = (i128)(T - K0 - (u128)(i128)q * (u128)Mc);
        if (sv > half) sv -= Mc;
        else if (sv < -half) sv += Mc;
        const bool neg = sv < 0;
        const u128 au = neg ? (u128)(-sv) : (u128)sv;
        double v = fma((double)(unsigned long long)(au >> 64), 18446744073709551616.0,
                       (double)(unsigned long long)au);
        if (neg) v = -v;
        const int sp = shift_p[i];
        v = (sp == kOzakiNonFinite || sq == kOzakiNonFinite) ? CUDART_NAN : ldexp(v, -(sp + sq));
        double* o = out + i + j * ldo;
        *o = beta == 0.0 ? alpha * v : alpha * v + beta * *o;
      }
    }
  }
}

CUtensorMap make_tmap_i8_planes(const int8_t* base, int64_t K, int64_t cols, int64_t ld, int64_t plane_stride,
                                int box_rows) {
  using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    LRB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)cols, (cuuint64_t)kOzakiModuli};
  cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)plane_stride};
  cuuint32_t box[3] = {(cuuint32_t)IBK, (cuuint32_t)box_rows, 1};  // IBK bytes = the 64B swizzle span
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (int8 planes) failed: " + std::to_string((int)r));
  return map;
}

// The planes of an operand split along its columns ([plane][col][K], K contiguous), read as the
// M-major operand of a product that contracts over its COLUMNS: box = 128 K-bytes (the product's M
// rows) x IBK columns (the product's K), 128B swizzle.
CUtensorMap make_tmap_i8_planes_mn(const int8_t* base, int64_t K, int64_t cols, int64_t ld, int64_t plane_stride) {
  using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    LRB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)cols, (cuuint64_t)kOzakiModuli};
  cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)plane_stride};
  cuuint32_t box[3] = {(cuuint32_t)IBM, (cuuint32_t)IBK, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (int8 planes, M-major) failed: " + std::to_string((int)r));
  return map;
}

// Opt-in (LRB_SPLIT_FUSED=1), slower than the two passes on B200 -- see ozaki_split_into.
// Column max and split in one pass over X (kSplitCluster CTAs per column):
// each CTA keeps its kSplitTilesPerCta tiles of the column in registers,
// the column's max|x| is reduced across the cluster through distributed
// shared memory, then the tiles are split from registers.  X is read once
// instead of twice (colmax_kernel + split_kernel); K <= 65536, vec2 layout.
constexpr int kSplitCluster = 8;
constexpr int kSplitTilesPerCta = 4;
template <bool UNS>
__global__ void __cluster_dims__(kSplitCluster, 1, 1) __launch_bounds__(kSplitThreads, 3)
split_fused_kernel(int64_t K, int64_t cols, const double* __restrict__ X, int64_t ldx, int beta,
                   int8_t* __restrict__ planes, int64_t ldp, int64_t plane_stride, int* __restrict__ shift) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  // this CTA's rows of the column, staged by cp.async: thread t's 8 rows of a
  // tile at 64t bytes, its four 16-byte pieces XOR-swizzled by (t >> 1) & 3 so
  // the per-thread 16-byte shared loads are conflict-free
  extern __shared__ __align__(16) double xs[];
  __shared__ unsigned long long sh[kSplitThreads / 32];
  __shared__ unsigned long long slot[2];
  const int rank = (int)cluster.block_rank();
  const int64_t nclusters = gridDim.x / kSplitCluster;
  const int tiles_k = (int)((K + kSplitTile - 1) / kSplitTile);
  const int64_t r_off = (int64_t)kSplitRows * threadIdx.x;
  const int swz = (threadIdx.x >> 1) & 3;
  int it = 0;
  for (int64_t j = blockIdx.x / kSplitCluster; j < cols; j += nclusters, ++it) {
    const double* xc = X + j * ldx;
#pragma unroll
    for (int u = 0; u < kSplitTilesPerCta; ++u) {
      const int tk = rank * kSplitTilesPerCta + u;
      const int64_t i0 = (int64_t)tk * kSplitTile + r_off;
      double* d = xs + u * kSplitTile + r_off;
      if (tk < tiles_k && i0 + kSplitRows <= K) {
#pragma unroll
        for (int h = 0; h < kSplitRows / 2; ++h) {
          const uint32_t dst = (uint32_t)__cvta_generic_to_shared(d + 2 * (h ^ swz));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(xc + i0 + 2 * h) : "memory");
        }
      } else {
#pragma unroll
        for (int h = 0; h < kSplitRows / 2; ++h) {
          const int64_t i = i0 + 2 * h;
          d[2 * (h ^ swz)] = (tk < tiles_k && i < K) ? xc[i] : 0.0;
          d[2 * (h ^ swz) + 1] = (tk < tiles_k && i + 1 < K) ? xc[i + 1] : 0.0;
        }
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    auto tile = [&](int u, double (&v)[kSplitRows]) {
      const double* d = xs + u * kSplitTile + r_off;
#pragma unroll
      for (int h = 0; h < kSplitRows / 2; ++h) {
        const double2 a = *reinterpret_cast<const double2*>(d + 2 * (h ^ swz));
        v[2 * h] = a.x;
        v[2 * h + 1] = a.y;
      }
    };
    unsigned long long mx = 0;
#pragma unroll
    for (int u = 0; u < kSplitTilesPerCta; ++u) {
      double v[kSplitRows];
      tile(u, v);
#pragma unroll
      for (int q = 0; q < kSplitRows; ++q) mx = max(mx, (unsigned long long)__double_as_longlong(fabs(v[q])));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = sh[0];
      for (int w = 1; w < kSplitThreads / 32; ++w) m = max(m, sh[w]);
      slot[it & 1] = m;
    }
    // slot[it & 1] is rewritten two columns later, after the next cluster
    // barrier, which every CTA reaches only once it has read this column's slots
    cluster.sync();
    unsigned long long cm = 0;
#pragma unroll
    for (int r = 0; r < kSplitCluster; ++r) cm = max(cm, *cluster.map_shared_rank(&slot[it & 1], r));
    const double mxd = __longlong_as_double((long long)cm);
    int e = 0;
    if (mxd > 0.0 && isfinite(mxd)) frexp(mxd, &e);
    const int sft = (mxd > 0.0 && isfinite(mxd)) ? beta - e : 0;
    if (rank == 0 && threadIdx.x == 0) shift[j] = isfinite(mxd) ? sft : kOzakiNonFinite;
    const double sc1 = ldexp(1.0, sft / 2), sc2 = ldexp(1.0, sft - sft / 2);
    int8_t* colp = planes + j * ldp;
#pragma unroll 1
    for (int u = 0; u < kSplitTilesPerCta; ++u) {
      const int tk = rank * kSplitTilesPerCta + u;
      const int64_t i0 = (int64_t)tk * kSplitTile + r_off;
      if (tk < tiles_k && i0 < K) {
        double v[kSplitRows];
        tile(u, v);
        split_tile<UNS>(v, sc1, sc2, colp + i0, plane_stride);
      }
    }
  }
  cluster.sync();  // no CTA leaves while a peer may still read its slots
}

}  // namespace

int ozaki_beta(int64_t K) {
  // K 2^(2 beta) < M_crt / 2  (exact int32 partial sums need K <= 2^17)
  const double lm = crt_host().log2M - 1.0 - std::log2((double)std::max<int64_t>(K, 1));
  const int b = (int)std::floor(lm / 2.0);
  return std::min(b, 60);  // |x'| <= 2^60 keeps the residue reduction exact
}

size_t ozaki_plane_bytes(int64_t K, int64_t cols) {
  const int64_t ld = (K + 15) / 16 * 16;
  return (size_t)ld * cols * kOzakiModuli;
}

void ozaki_split_into(const double* X, int64_t ldx, const OzakiOperand& op, cudaStream_t st) {
  upload_constants();
  const int64_t K = op.K, cols = op.cols;
  if (K < 1 || cols < 1) return;
  if (op.unsigned_res && K > kOzakiMaxKUnsigned) throw CudaError("ozaki_split: unsigned residues need K <= 65536");
  const bool vec2 = (reinterpret_cast<uintptr_t>(X) % 16 == 0) && (ldx % 2 == 0);
  // "1": cluster-fused split (reads X once, but measured slower: 22-25 ms vs
  // 14 ms for the two passes at C4 -- the register-resident column leaves 16
  // warps per SM and no load/compute overlap; kept for A/B and tests)
  const char* fe = std::getenv("LRB_SPLIT_FUSED");
  const bool fused_off = !(fe && fe[0] == '1');
  if (!fused_off && vec2 && K >= (int64_t)kSplitCluster * kSplitTile &&
      K <= (int64_t)kSplitCluster * kSplitTilesPerCta * kSplitTile) {
    auto kern = op.unsigned_res ? split_fused_kernel<true> : split_fused_kernel<false>;
    constexpr int kFusedSmem = kSplitTilesPerCta * kSplitTile * (int)sizeof(double);  // 64 KB
    static thread_local bool attr = false;
    if (!attr) {
      LRB_CUDA(cudaFuncSetAttribute(split_fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem));
      LRB_CUDA(cudaFuncSetAttribute(split_fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem));
      attr = true;
    }
    // persistent clusters: only as many as are co-resident (GPC packing of
    // 8-CTA clusters leaves fewer than 3 * SMs / 8), or the excess run as a tail
    static thread_local int max_cl = 0;
    if (!max_cl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kSplitCluster * 64);
      cfg.blockDim = dim3(kSplitThreads);
      cfg.dynamicSmemBytes = kFusedSmem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kSplitCluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      LRB_CUDA(cudaOccupancyMaxActiveClusters(&max_cl, split_fused_kernel<false>, &cfg));
      max_cl = std::max(1, max_cl);
      if (std::getenv("LRB_WS_DEBUG")) std::fprintf(stderr, "[lrb] split_fused: %d co-resident clusters\n", max_cl);
    }
    const int budget_cl = g_sm_budget > 0 ? std::max(1, max_cl * g_sm_budget / kNumSMsB200) : max_cl;
    const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>(cols, std::min(max_cl, budget_cl)));
    kern<<<(int)(ncl * kSplitCluster), kSplitThreads, kFusedSmem, st>>>(K, cols, X, ldx, op.beta, op.planes, op.ld,
                                                                 op.plane_stride, op.shift);
    LRB_CHECK_LAUNCH();
    return;
  }
  unsigned long long* cmax = nullptr;
  LRB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cmax), sizeof(unsigned long long) * cols, st));
  LRB_CUDA(cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * cols, st));
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(cols, 8 * num_sms()));  // split: whole columns per CTA
  const int64_t mtiles = (K + kMaxRowsPerThread * kSplitThreads - 1) / (kMaxRowsPerThread * kSplitThreads) * cols;
  const int gm = (int)std::max<int64_t>(1, std::min<int64_t>(mtiles, 8 * num_sms()));
  colmax_kernel<<<gm, kSplitThreads, 0, st>>>(K, cols, X, ldx, vec2, cmax);
  LRB_CHECK_LAUNCH();
  auto kern = op.unsigned_res ? split_kernel<true> : split_kernel<false>;
  kern<<<g, kSplitThreads, 0, st>>>(K, cols, X, ldx, vec2, op.beta, cmax, op.planes, op.ld, op.plane_stride,
                                            op.shift);
  LRB_CHECK_LAUNCH();
  LRB_CUDA(cudaFreeAsync(cmax, st));
}

void ozaki_split(int64_t K, int64_t cols, const double* X, int64_t ldx, int beta, OzakiOperand& op, cudaStream_t st) {
  op.K = K;
  op.cols = cols;
  op.ld = (K + 15) / 16 * 16;
  op.plane_stride = op.ld * cols;
  op.beta = beta;
  ozaki_split_into(X, ldx, op, st);
}

OzakiOperand ozaki_cols(const OzakiOperand& op, int64_t off, int64_t cols) {
  OzakiOperand v = op;
  v.planes = op.planes + off * op.ld;
  v.shift = op.shift + off;
  v.cols = cols;
  return v;
}

void ozaki_gemm_tn(Workspace& ws, const OzakiOperand& P, const OzakiOperand& Q, int64_t M, int64_t N, double* out,
                   int64_t ldo, double alpha, double beta, cudaStream_t st) {
  upload_constants();
  if (P.K != Q.K || M > P.cols || N > Q.cols) throw CudaError("ozaki_gemm_tn: operand shape mismatch");
  if (P.K > (int64_t(1) << 17)) throw CudaError("ozaki_gemm_tn: K > 2^17 would overflow the int32 accumulators");
  static bool attr = false;
  if (!attr) {
    LRB_CUDA(cudaFuncSetAttribute(imma_gemm_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, ISMEM));
    LRB_CUDA(cudaFuncSetAttribute(imma_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ISMEM));
    LRB_CUDA(cudaFuncSetAttribute(imma_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ISMEM));
    attr = true;
  }
  const int tiles_m0 = (int)((M + IBM - 1) / IBM);
  // the cluster size that wastes no M tile (padding 2 tiles to 4 doubled C3's sketch work)
  const int cl = tiles_m0 % 4 == 0 ? 4 : (tiles_m0 % 2 == 0 ? 2 : (tiles_m0 == 1 ? 1 : 4));
  const CUtensorMap tp = make_tmap_i8_planes(P.planes, P.K, P.cols, P.ld, P.plane_stride, IBM);
  const CUtensorMap tq = make_tmap_i8_planes(Q.planes, Q.K, Q.cols, Q.ld, Q.plane_stride, std::min(256, IBN / cl));
  const int64_t ldr = (M + 15) / 16 * 16;  // 4-byte aligned residue columns for crt4_kernel
  int8_t* res = static_cast<int8_t*>(ws.get(WsSlot::kTmp7, (size_t)ldr * N * kOzakiModuli));
  const int tiles_m = (int)((M + IBM - 1) / IBM), tiles_n = (int)((N + IBN - 1) / IBN);
  // clusters of cl CTAs along M: pad the M grid (extra CTAs compute zero rows and store nothing)
  dim3 grid((tiles_m + cl - 1) / cl * cl, tiles_n, kOzakiModuli);
  if (P.unsigned_res && Q.unsigned_res) throw CudaError("ozaki_gemm_tn: at most one unsigned-residue operand");
  if ((P.unsigned_res || Q.unsigned_res) && P.K > kOzakiMaxKUnsigned)
    throw CudaError("ozaki_gemm_tn: K too large for an unsigned-residue operand");
  const uint32_t ab_fmt = (P.unsigned_res ? 0u : (1u << 7)) | (Q.unsigned_res ? 0u : (1u << 10));
  auto kern = cl == 4 ? imma_gemm_kernel<4> : (cl == 2 ? imma_gemm_kernel<2> : imma_gemm_kernel<1>);
  kern<<<grid, ITHREADS, ISMEM, st>>>(tp, tq, (int)M, (int)N, (int)P.K, res, ldr, ldr * N, ab_fmt, 0);
  LRB_CHECK_LAUNCH();
  const int64_t items = (M + 3) / 4 * N;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, 8 * num_sms()));
  crt4_kernel<<<gx, 256, 0, st>>>(M, N, res, ldr, ldr * N, P.shift, Q.shift, out, ldo, alpha, beta);
  LRB_CHECK_LAUNCH();
}

namespace {
// out(j, r) = X(j, r) 2^-shift[j]: the column scales of the split operand folded into its partner
__global__ void scale_rows_pow2_kernel(int64_t K, int64_t cols, const double* __restrict__ X, int64_t ldx,
                                       const int* __restrict__ shift, double* __restrict__ out, int64_t ldo) {
  for (int64_t r = blockIdx.y; r < cols; r += gridDim.y)
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
      const int sft = shift[j];
      out[j + r * ldo] = sft == kOzakiNonFinite ? CUDART_NAN : ldexp(X[j + r * ldx], -sft);
    }
}
}  // namespace

void ozaki_fold_scales(int64_t K, int64_t cols, const double* X, int64_t ldx, const int* shift, double* out,
                       int64_t ldo, cudaStream_t st) {
  if (K <= 0 || cols <= 0) return;
  dim3 grid((unsigned)std::min<int64_t>((K + 255) / 256, 1024), (unsigned)std::min<int64_t>(cols, 65535));
  scale_rows_pow2_kernel<<<grid, 256, 0, st>>>(K, cols, X, ldx, shift, out, ldo);
  LRB_CHECK_LAUNCH();
}

namespace {
// bits the two operands of a length-K contraction may share: K 2^(ba + bq) < M_crt / 2
int ozaki_room(int64_t K) {
  return (int)std::floor(crt_host().log2M - 1.0 - std::log2((double)std::max<int64_t>(K, 1)));
}
}  // namespace

int ozaki_partner_beta(int64_t K, int beta_a) { return std::min(ozaki_room(K) - beta_a, 60); }

// out (A.K x N) = A_int Q with A_int the integer matrix behind A's planes (A.K x A.cols, entry (i, j) =
// rint(a_ij 2^shift_j)) and Q (A.cols x N) split along ITS columns: the contraction runs over A's
// columns, so A's planes are the M-major operand of the INT8 GEMM.  A's column scales are not
// applied here (the caller folded 2^-shift_j into Q's rows: ozaki_fold_scales); zero_shift: A.K zeros.
void ozaki_gemm_a_cols(Workspace& ws, const OzakiOperand& A, const OzakiOperand& Q, int64_t N, double* out,
                       int64_t ldo, const int* zero_shift, cudaStream_t st) {
  upload_constants();
  const int64_t M = A.K, K = A.cols;
  if (Q.K != K || N > Q.cols) throw CudaError("ozaki_gemm_a_cols: operand shape mismatch");
  if (K > (int64_t(1) << 17)) throw CudaError("ozaki_gemm_a_cols: K > 2^17 would overflow the int32 accumulators");
  if (A.unsigned_res && Q.unsigned_res) throw CudaError("ozaki_gemm_a_cols: at most one unsigned-residue operand");
  if ((A.unsigned_res || Q.unsigned_res) && K > kOzakiMaxKUnsigned)
    throw CudaError("ozaki_gemm_a_cols: K too large for an unsigned-residue operand");
  if (A.beta + Q.beta > ozaki_room(K)) throw CudaError("ozaki_gemm_a_cols: operand bits exceed the CRT range");
  static bool attr = false;
  if (!attr) {
    LRB_CUDA(cudaFuncSetAttribute(imma_gemm_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, ISMEM));
    LRB_CUDA(cudaFuncSetAttribute(imma_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ISMEM));
    LRB_CUDA(cudaFuncSetAttribute(imma_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ISMEM));
    attr = true;
  }
  const int tiles_m = (int)((M + IBM - 1) / IBM), tiles_n = (int)((N + IBN - 1) / IBN);
  const int cl = tiles_m % 4 == 0 ? 4 : (tiles_m % 2 == 0 ? 2 : (tiles_m == 1 ? 1 : 4));
  const CUtensorMap tp = make_tmap_i8_planes_mn(A.planes, A.K, A.cols, A.ld, A.plane_stride);
  const CUtensorMap tq = make_tmap_i8_planes(Q.planes, Q.K, Q.cols, Q.ld, Q.plane_stride, std::min(256, IBN / cl));
  const int64_t ldr = (M + 15) / 16 * 16;
  int8_t* res = static_cast<int8_t*>(ws.get(WsSlot::kTmp7, (size_t)ldr * N * kOzakiModuli));
  dim3 grid((tiles_m + cl - 1) / cl * cl, tiles_n, kOzakiModuli);
  const uint32_t ab_fmt = (A.unsigned_res ? 0u : (1u << 7)) | (Q.unsigned_res ? 0u : (1u << 10));
  auto kern = cl == 4 ? imma_gemm_kernel<4> : (cl == 2 ? imma_gemm_kernel<2> : imma_gemm_kernel<1>);
  kern<<<grid, ITHREADS, ISMEM, st>>>(tp, tq, (int)M, (int)N, (int)K, res, ldr, ldr * N, ab_fmt, 1);
  LRB_CHECK_LAUNCH();
  const int64_t items = (M + 3) / 4 * N;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, 8 * num_sms()));
  crt4_kernel<<<gx, 256, 0, st>>>(M, N, res, ldr, ldr * N, zero_shift, Q.shift, out, ldo, 1.0, 0.0);
  LRB_CHECK_LAUNCH();
}

}  // namespace lrb
