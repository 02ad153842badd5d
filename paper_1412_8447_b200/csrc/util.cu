#include <cstdio>
#include <cstdlib>
// util.cu -- workspace, TMA descriptors and the HBM-bound data-movement
// kernels (gathers for C / R / A_skel, transposes, validation, reductions).
// All reductions use a fixed grid and a fixed tree so results are bitwise
// reproducible run to run (test_sketch.cpp:170-183).
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace lrb {

thread_local int g_sm_budget = 0;


unsigned long long g_kernel_launches = 0;

// ---------------------------------------------------------------- workspace
Workspace::~Workspace() { release_all(); }

void Workspace::release_all() {
  for (auto& p : ptr_)
    if (p) {
      cudaFree(p);
      p = nullptr;
    }
  for (auto& c : cap_) c = 0;
}

void* Workspace::try_get(WsSlot s, size_t bytes) {
  const size_t i = static_cast<size_t>(s);
  if (bytes == 0) bytes = 16;
  if (cap_[i] >= bytes) return ptr_[i];
  static const bool dbg = getenv("LRB_WS_DEBUG") != nullptr;
  if (dbg) fprintf(stderr, "workspace slot %zu grows %zu -> %zu bytes (try)\n", i, cap_[i], bytes);
  if (ptr_[i]) {
    LRB_CUDA(cudaDeviceSynchronize());
    LRB_CUDA(cudaFree(ptr_[i]));
    ptr_[i] = nullptr;
    cap_[i] = 0;
  }
  const size_t rounded = (bytes + (1u << 20) - 1) & ~size_t((1u << 20) - 1);
  if (cudaMalloc(&ptr_[i], rounded) != cudaSuccess) {
    cudaGetLastError();
    ptr_[i] = nullptr;
    return nullptr;
  }
  cap_[i] = rounded;
  return ptr_[i];
}

void* Workspace::get(WsSlot s, size_t bytes) {
  const size_t i = static_cast<size_t>(s);
  if (bytes == 0) bytes = 16;
  if (cap_[i] < bytes) {
    static const bool dbg = getenv("LRB_WS_DEBUG") != nullptr;
    if (dbg) fprintf(stderr, "workspace slot %zu grows %zu -> %zu bytes\n", i, cap_[i], bytes);
    if (ptr_[i]) {
      LRB_CUDA(cudaDeviceSynchronize());
      LRB_CUDA(cudaFree(ptr_[i]));
      ptr_[i] = nullptr;
    }
    const size_t rounded = (bytes + (1u << 20) - 1) & ~size_t((1u << 20) - 1);
    LRB_CUDA(cudaMalloc(&ptr_[i], rounded));
    cap_[i] = rounded;
  }
  return ptr_[i];
}

// ---------------------------------------------------------------- tensor maps
namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    LRB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
}  // namespace

CUtensorMap make_tmap_f64(const double* base, int64_t rows, int64_t cols, int64_t ld, int box_rows, int box_cols,
                          bool swizzle128) {
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") rows=" + std::to_string(rows) +
                    " cols=" + std::to_string(cols) + " ld=" + std::to_string(ld));
  return map;
}

// ---------------------------------------------------------------- kernels
namespace {

__global__ void scale_kernel(int M, int N, double* a, int64_t lda, double beta) {
  const int64_t total = (int64_t)M * N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    double* p = a + (t % M) + (t / M) * lda;
    *p = beta == 0.0 ? 0.0 : beta * *p;
  }
}

__global__ void copy_kernel(int64_t m, int64_t n, const double* __restrict__ s, int64_t lds, double* __restrict__ d,
                            int64_t ldd) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      d[i + j * ldd] = s[i + j * lds];
}

__global__ void copy_upper_kernel(int64_t k, const double* __restrict__ s, int64_t lds, double* __restrict__ d,
                                  int64_t ldd) {
  const int64_t total = k * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % k, j = t / k;
    d[i + j * ldd] = i <= j ? s[i + j * lds] : 0.0;
  }
}

// 32x32 tiles through shared memory (padded against bank conflicts)
__global__ void transpose_kernel(int64_t m, int64_t n, const double* __restrict__ s, int64_t lds,
                                 double* __restrict__ d, int64_t ldd) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, j = j0 + r;
    if (i < m && j < n) tile[r][threadIdx.x] = s[i + j * lds];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + threadIdx.x, i = i0 + r;  // out(j, i) = s(i, j)
    if (i < m && j < n) d[j + i * ldd] = tile[threadIdx.x][r];
  }
}

__global__ void gather_columns_kernel(int64_t m, int64_t k, const double* __restrict__ a, int64_t lda,
                                      const int64_t* __restrict__ idx, double* __restrict__ out, int64_t ldo) {
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y) {
    const int64_t col = idx[j];  // negative: a zero column (masked gather for sharded assembly)
    const double* src = a + (col >= 0 ? col : 0) * lda;
    double* dst = out + j * ldo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      dst[i] = col >= 0 ? src[i] : 0.0;
  }
}

// R = A(idx, :): a thread keeps one row index and walks columns (no index
// division per element; 4 independent column loads in flight).  Each load
// touches its own 32-byte sector of A (the gather is sector-bound), stores are
// coalesced along the k rows of a column.
__global__ void gather_rows_kernel(int64_t k, int64_t n, const double* __restrict__ a, int64_t lda,
                                   const int64_t* __restrict__ idx, double* __restrict__ out, int64_t ldo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const double* src = a + idx[i];
  double* dst = out + i;
  const int64_t step = gridDim.y;
  int64_t j = blockIdx.y;
  for (; j + 3 * step < n; j += 4 * step) {
    const double v0 = __ldcs(src + j * lda), v1 = __ldcs(src + (j + step) * lda);
    const double v2 = __ldcs(src + (j + 2 * step) * lda), v3 = __ldcs(src + (j + 3 * step) * lda);
    dst[j * ldo] = v0;
    dst[(j + step) * ldo] = v1;
    dst[(j + 2 * step) * ldo] = v2;
    dst[(j + 3 * step) * ldo] = v3;
  }
  for (; j < n; j += step) dst[j * ldo] = __ldcs(src + j * lda);
}

__global__ void gather_rows_t_kernel(int64_t k, int64_t n, const double* __restrict__ a, int64_t lda,
                                     const int64_t* __restrict__ idx, double* __restrict__ out, int64_t ldo) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, j = j0 + r;
    if (i < k && j < n) tile[r][threadIdx.x] = a[idx[i] + j * lda];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + threadIdx.x, i = i0 + r;
    if (i < k && j < n) out[j + i * ldo] = tile[threadIdx.x][r];
  }
}

__global__ void check_finite_kernel(int64_t m, int64_t n, const double* __restrict__ a, int64_t lda, int* flag) {
  int bad = 0;
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      bad |= !isfinite(a[i + j * lda]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// fixed-order block reduction helpers (blockDim.x == 256)
__device__ double block_sum_256(double v, double* sh) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < 8; ++w) t += sh[w];
  __syncthreads();
  return t;
}
__device__ double block_max_256(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < 8; ++w) t = fmax(t, sh[w]);
  __syncthreads();
  return t;
}

__global__ void frob2_kernel(int64_t m, int64_t n, const double* __restrict__ a, int64_t lda,
                             double* __restrict__ partials) {
  __shared__ double sh[8];
  double acc = 0.0;
  const int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[(t % m) + (t / m) * lda];
    acc = fma(x, x, acc);
  }
  const double s = block_sum_256(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void maxabs_kernel(int64_t m, int64_t n, const double* __restrict__ a, int64_t lda,
                              double* __restrict__ partials) {
  __shared__ double sh[8];
  double acc = 0.0;
  const int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    acc = fmax(acc, fabs(a[(t % m) + (t / m) * lda]));
  const double s = block_max_256(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(const double* __restrict__ p, int n, double* out, int op_max) {
  __shared__ double sh[8];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc = op_max ? fmax(acc, p[i]) : acc + p[i];
  const double s = op_max ? block_max_256(acc, sh) : block_sum_256(acc, sh);
  if (threadIdx.x == 0) out[0] = s;
}

inline int grid_for(int64_t total, int block = 256) {
  const int64_t g = (total + block - 1) / block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 16 * num_sms()));
}

}  // namespace

void scale_matrix(int M, int N, double* a, int64_t lda, double beta, cudaStream_t st) {
  if (beta == 1.0 || M <= 0 || N <= 0) return;
  scale_kernel<<<grid_for((int64_t)M * N), 256, 0, st>>>(M, N, a, lda, beta);
  LRB_CHECK_LAUNCH();
}

void copy_matrix(int64_t m, int64_t n, const double* src, int64_t lds, double* dst, int64_t ldd, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  if (lds == m && ldd == m) {
    LRB_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, st));
    return;
  }
  dim3 grid((unsigned)std::min<int64_t>((m + 255) / 256, 64), (unsigned)std::min<int64_t>(n, 65535));
  copy_kernel<<<grid, 256, 0, st>>>(m, n, src, lds, dst, ldd);
  LRB_CHECK_LAUNCH();
}

void copy_upper(int64_t k, const double* src, int64_t lds, double* dst, int64_t ldd, cudaStream_t st) {
  if (k <= 0) return;
  copy_upper_kernel<<<grid_for(k * k), 256, 0, st>>>(k, src, lds, dst, ldd);
  LRB_CHECK_LAUNCH();
}

void transpose_matrix(int64_t m, int64_t n, const double* src, int64_t lds, double* dst, int64_t ldd,
                      cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  dim3 grid((unsigned)((m + 31) / 32), (unsigned)((n + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(m, n, src, lds, dst, ldd);
  LRB_CHECK_LAUNCH();
}

void gather_columns(int64_t m, int64_t k, const double* a, int64_t lda, const int64_t* idx, double* out, int64_t ldo,
                    cudaStream_t st) {
  if (m <= 0 || k <= 0) return;
  dim3 grid((unsigned)std::min<int64_t>((m + 255) / 256, 64), (unsigned)std::min<int64_t>(k, 65535));
  gather_columns_kernel<<<grid, 256, 0, st>>>(m, k, a, lda, idx, out, ldo);
  LRB_CHECK_LAUNCH();
}

void gather_rows(int64_t k, int64_t n, const double* a, int64_t lda, const int64_t* idx, double* out, int64_t ldo,
                 cudaStream_t st) {
  if (k <= 0 || n <= 0) return;
  const unsigned gx = (unsigned)((k + 255) / 256);
  const unsigned gy = (unsigned)std::max<int64_t>(1, std::min<int64_t>(n, (8 * num_sms() + gx - 1) / gx * 4));
  gather_rows_kernel<<<dim3(gx, gy), 256, 0, st>>>(k, n, a, lda, idx, out, ldo);
  LRB_CHECK_LAUNCH();
}

void gather_rows_t(int64_t k, int64_t n, const double* a, int64_t lda, const int64_t* idx, double* out, int64_t ldo,
                   cudaStream_t st) {
  if (k <= 0 || n <= 0) return;
  dim3 grid((unsigned)((k + 31) / 32), (unsigned)((n + 31) / 32));
  gather_rows_t_kernel<<<grid, dim3(32, 8), 0, st>>>(k, n, a, lda, idx, out, ldo);
  LRB_CHECK_LAUNCH();
}

void check_finite(int64_t m, int64_t n, const double* a, int64_t lda, int* flag, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  dim3 grid((unsigned)std::min<int64_t>((m + 255) / 256, 16), (unsigned)std::min<int64_t>(n, 8192));
  check_finite_kernel<<<grid, 256, 0, st>>>(m, n, a, lda, flag);
  LRB_CHECK_LAUNCH();
}

void sum_partials(const double* p, int n, double* out, cudaStream_t st) {
  sum_partials_kernel<<<1, 256, 0, st>>>(p, n, out, 0);
  LRB_CHECK_LAUNCH();
}

void frob2(int64_t m, int64_t n, const double* a, int64_t lda, double* partials, double* out, cudaStream_t st) {
  const int g = 4 * num_sms();
  frob2_kernel<<<g, 256, 0, st>>>(m, n, a, lda, partials);
  LRB_CHECK_LAUNCH();
  sum_partials_kernel<<<1, 256, 0, st>>>(partials, g, out, 0);
  LRB_CHECK_LAUNCH();
}

void max_abs(int64_t m, int64_t n, const double* a, int64_t lda, double* partials, double* out, cudaStream_t st) {
  const int g = 4 * num_sms();
  maxabs_kernel<<<g, 256, 0, st>>>(m, n, a, lda, partials);
  LRB_CHECK_LAUNCH();
  sum_partials_kernel<<<1, 256, 0, st>>>(partials, g, out, 1);
  LRB_CHECK_LAUNCH();
}

namespace {
__global__ void copy_bytes_kernel(char* __restrict__ dst, const char* __restrict__ src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
}  // namespace

void copy_bytes_mapped(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  copy_bytes_kernel<<<1, 32, 0, st>>>(static_cast<char*>(dst), static_cast<const char*>(src), (int)bytes);
  LRB_CHECK_LAUNCH();
}

}  // namespace lrb
