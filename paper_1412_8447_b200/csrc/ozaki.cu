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
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace lrb {

namespace {

constexpr int kMod[kOzakiModuli] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
__constant__ int c_mod[kOzakiModuli];
__constant__ double c_inv_mod[kOzakiModuli];
__constant__ unsigned long long c_Mt[kOzakiModuli][2];  // M / m_t (low, high limbs)
__constant__ int c_crt_inv[kOzakiModuli];               // (M / m_t)^-1 mod m_t
__constant__ unsigned long long c_Mcrt[2];

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
  done = true;
}

// ------------------------------------------------------------ 1+2: scale and split
// One block per column (grid-stride): pass 1 finds max|x| (HBM), pass 2 re-reads
// the column (L2) and writes 16 residue bytes per 16-element K chunk.
__global__ void __launch_bounds__(256) residue_kernel(int64_t K, int64_t cols, const double* __restrict__ X,
                                                      int64_t ldx, int beta, int8_t* __restrict__ planes,
                                                      int64_t ldp, int64_t plane_stride, int* __restrict__ shift) {
  __shared__ double sh[8];
  __shared__ int sh_shift;
  for (int64_t j = blockIdx.x; j < cols; j += gridDim.x) {
    const double* x = X + j * ldx;
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i < K; i += blockDim.x) mx = fmax(mx, fabs(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t = fmax(t, sh[w]);
      int e = 0;
      if (t > 0.0) {
        frexp(t, &e);  // t < 2^e
      }
      const int s = t > 0.0 ? beta - e : 0;
      sh_shift = s;
      shift[j] = s;
    }
    __syncthreads();
    const int s = sh_shift;
    // 16 consecutive K entries per thread -> one 16-byte store per plane
    for (int64_t i0 = 16 * (int64_t)threadIdx.x; i0 < K; i0 += 16 * (int64_t)blockDim.x) {
      alignas(16) int8_t r[kOzakiModuli][16];
#pragma unroll 4
      for (int e = 0; e < 16; ++e) {
        const int64_t i = i0 + e;
        const double v = i < K ? rint(ldexp(x[i], s)) : 0.0;  // exact integer, |v| <= 2^beta
#pragma unroll
        for (int t = 0; t < kOzakiModuli; ++t) {
          const double m = (double)c_mod[t];
          double q = floor(v * c_inv_mod[t]);
          double rr = fma(-q, m, v);  // exact: |rr| < 2m
          if (rr < 0.0) rr += m;
          if (rr >= m) rr -= m;
          int ri = (int)rr;
          if (ri > (c_mod[t] - 1) / 2) ri -= c_mod[t];  // symmetric: [-128, 127] (m = 256) / [-(m-1)/2, (m-1)/2]
          r[t][e] = (int8_t)ri;
        }
      }
#pragma unroll
      for (int t = 0; t < kOzakiModuli; ++t)
        *reinterpret_cast<int4*>(planes + t * plane_stride + j * ldp + i0) = *reinterpret_cast<const int4*>(r[t]);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ 3: tcgen05 INT8 GEMM
constexpr int IBM = 128, IBN = 256, IBK = 128;  // tile (K in bytes = int8 elements)
constexpr int ISTAGES = 4;
constexpr int IA_BYTES = IBM * IBK, IB_BYTES = IBN * IBK;
constexpr int ISTAGE_BYTES = IA_BYTES + IB_BYTES;
constexpr int ITHREADS = 6 * 32;  // warp 0 TMA, warp 1 MMA + TMEM, warps 2-5 epilogue
constexpr int ISMEM = ISTAGES * ISTAGE_BYTES + 1024 + 256;
constexpr uint32_t kTmemCols = 256;

__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  // K-major, SWIZZLE_128B: 8-row x 128 B atoms, SBO = 1024 B between atoms, LBO unused (1), version 1
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
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

__global__ void __launch_bounds__(ITHREADS, 1)
    imma_gemm_kernel(const __grid_constant__ CUtensorMap tmp, const __grid_constant__ CUtensorMap tmq, int M, int N,
                     int K, int tiles_m, int tiles_n, int m_fast, int8_t* __restrict__ out, int64_t ldo,
                     int64_t out_plane_stride) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ISTAGES * ISTAGE_BYTES);
  uint64_t* empty = full + ISTAGES;
  uint64_t* tmem_full = empty + ISTAGES;
  uint32_t* tmem_base_sh = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int plane = blockIdx.z;
  // rasterise along the smaller tile dimension so CTAs sharing an operand tile run together
  const int tm = m_fast ? blockIdx.x % tiles_m : blockIdx.x / tiles_n;
  const int tn = m_fast ? blockIdx.x / tiles_m : blockIdx.x % tiles_n;
  const int m0 = tm * IBM, n0 = tn * IBN;
  const int nkb = (K + IBK - 1) / IBK;

  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < ISTAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(tmem_full, 1);
      fence_barrier_init();
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_base_sh)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmp);
      tma_prefetch_desc(&tmq);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ISTAGES;
        const uint32_t ph = (i / ISTAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sp = smem + s * ISTAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], ISTAGE_BYTES);
        tma_load_3d(sp, &tmp, &full[s], i * IBK, m0, plane);
        tma_load_3d(sp + IA_BYTES, &tmq, &full[s], i * IBK, n0, plane);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::i8: D s32, A/B signed int8, K-major, N = 256, M = 128
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(IBN >> 3) << 17) |
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
          const uint64_t da = smem_desc_sw128(sa + kk * 32);
          const uint64_t db = smem_desc_sw128(sb + kk * 32);
          const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        // frees the smem stage once these MMAs have read it
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&empty[s]))
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
    int8_t* o = out + (int64_t)plane * out_plane_stride;
    for (int c0 = 0; c0 < IBN; c0 += 16) {
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
            int r = (int)v[e] % mod;
            if (r > (mod - 1) / 2) r -= mod;
            else if (r < -(mod / 2)) r += mod;
            o[(int64_t)col * ldo + row] = (int8_t)r;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
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
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M * N; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % M, j = t / M;
    i128 s = 0;
#pragma unroll
    for (int p = 0; p < kOzakiModuli; ++p) {
      const int m = c_mod[p];
      int d = ((int)res[p * plane_stride + j * ldr + i] * c_crt_inv[p]) % m;
      if (d > m / 2) d -= m;
      else if (d < -(m / 2)) d += m;
      const i128 Mt = (i128)(((u128)c_Mt[p][1] << 64) | (u128)c_Mt[p][0]);
      s += (i128)d * Mt;  // |term| <= M/2
      if (s > half) s -= Mc;
      else if (s < -half) s += Mc;
    }
    // int128 -> double (round to nearest via the high/low split), then unscale
    const bool neg = s < 0;
    const u128 a = neg ? (u128)(-s) : (u128)s;
    const double hi = (double)(unsigned long long)(a >> 64);
    const double lo = (double)(unsigned long long)a;
    double v = fma(hi, 18446744073709551616.0, lo);
    if (neg) v = -v;
    v = ldexp(v, -(shift_p[i] + shift_q[j]));
    double* o = out + i + j * ldo;
    *o = beta == 0.0 ? alpha * v : alpha * v + beta * *o;
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
  cuuint32_t box[3] = {(cuuint32_t)IBK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (int8 planes) failed: " + std::to_string((int)r));
  return map;
}

}  // namespace

int ozaki_beta(int64_t K) {
  // K 2^(2 beta) < M_crt / 2  (exact int32 partial sums need K <= 2^17)
  const double lm = crt_host().log2M - 1.0 - std::log2((double)std::max<int64_t>(K, 1));
  int b = (int)std::floor(lm / 2.0) - 0;
  return std::min(b, 62);
}

size_t ozaki_plane_bytes(int64_t K, int64_t cols) {
  const int64_t ld = (K + 15) / 16 * 16;
  return (size_t)ld * cols * kOzakiModuli;
}

void ozaki_split(int64_t K, int64_t cols, const double* X, int64_t ldx, int beta, OzakiOperand& op, cudaStream_t st) {
  upload_constants();
  op.K = K;
  op.cols = cols;
  op.ld = (K + 15) / 16 * 16;
  op.plane_stride = op.ld * cols;
  op.beta = beta;
  const int g = (int)std::min<int64_t>(cols, 8 * num_sms());
  residue_kernel<<<g, 256, 0, st>>>(K, cols, X, ldx, beta, op.planes, op.ld, op.plane_stride, op.shift);
  LRB_CHECK_LAUNCH();
}

void ozaki_gemm_tn(Workspace& ws, const OzakiOperand& P, const OzakiOperand& Q, int64_t M, int64_t N, double* out,
                   int64_t ldo, double alpha, double beta, cudaStream_t st) {
  upload_constants();
  if (P.K != Q.K || M > P.cols || N > Q.cols) throw CudaError("ozaki_gemm_tn: operand shape mismatch");
  if (P.K > (int64_t(1) << 17)) throw CudaError("ozaki_gemm_tn: K > 2^17 would overflow the int32 accumulators");
  static bool attr = false;
  if (!attr) {
    LRB_CUDA(cudaFuncSetAttribute(imma_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ISMEM));
    attr = true;
  }
  const CUtensorMap tp = make_tmap_i8_planes(P.planes, P.K, P.cols, P.ld, P.plane_stride, IBM);
  const CUtensorMap tq = make_tmap_i8_planes(Q.planes, Q.K, Q.cols, Q.ld, Q.plane_stride, IBN);
  const int64_t ldr = M;
  int8_t* res = static_cast<int8_t*>(ws.get(WsSlot::kTmp7, (size_t)M * N * kOzakiModuli));
  const int tiles_m = (int)((M + IBM - 1) / IBM), tiles_n = (int)((N + IBN - 1) / IBN);
  dim3 grid(tiles_m * tiles_n, 1, kOzakiModuli);
  imma_gemm_kernel<<<grid, ITHREADS, ISMEM, st>>>(tp, tq, (int)M, (int)N, (int)P.K, tiles_m, tiles_n,
                                                   tiles_m <= tiles_n ? 1 : 0, res, ldr, M * N);
  LRB_CHECK_LAUNCH();
  const int64_t total = M * N;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 16 * num_sms()));
  crt_kernel<<<g, 256, 0, st>>>(M, N, res, ldr, M * N, P.shift, Q.shift, out, ldo, alpha, beta);
  LRB_CHECK_LAUNCH();
}

}  // namespace lrb
