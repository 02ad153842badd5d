// sparse.cu -- BASELINE config 5: randomized CUR of a CSR matrix (SURVEY.md
// section 8a row 26; the reference is dense-only, core.hpp:14-17, so parity is
// pinned on down-scaled instances densified through the dense oracle).
//
//   CSR -> CSC            stable radix sort by column (rows stay ascending per
//                         column: deterministic, no atomics in the data path)
//   Y = Omega A           SpMM, one warp per column of A: Y(:,j) = sum over the
//                         column's nonzeros a_ij * Omega(:, i); Omega columns are
//                         contiguous (l doubles) so each nonzero is one
//                         coalesced 2.5 KB read; fixed summation order
//   C = A(:, J), R = A(I, :)  sparse column / row extracts (+ dense copies for
//                         the k x k factorizations)
//   A^T Q (for U)         the same SpMM with Q^T as the dense operand
// All kernels are HBM / L2 bound (1e7 nonzeros at config 5).
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace lrb {

namespace {

__global__ void expand_rows_kernel(int64_t m, const int64_t* __restrict__ row_ptr, int64_t* __restrict__ rows) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < m;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5)
    for (int64_t t = row_ptr[i] + lane; t < row_ptr[i + 1]; t += 32) rows[t] = i;
}

__global__ void iota_kernel(int64_t n, int64_t* __restrict__ v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    v[t] = t;
}

__global__ void permute_kernel(int64_t nnz, const int64_t* __restrict__ perm, const int64_t* __restrict__ rows,
                               const double* __restrict__ val, int64_t* __restrict__ row_out,
                               double* __restrict__ val_out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = perm[t];
    row_out[t] = rows[p];
    val_out[t] = val[p];
  }
}

// col_ptr[c] = first t with key[t] >= c (keys sorted), for c in [0, n]
__global__ void bounds_kernel(int64_t nnz, int64_t n, const int64_t* __restrict__ key, int64_t* __restrict__ ptr) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= n; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (key[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    ptr[c] = lo;
  }
}

// out(:, j) = sum_{t in col j} val[t] * B(:, row[t]); one warp per column, lanes over rows
template <int RPL>  // rows of B per lane held in registers (p <= 32*RPL)
__global__ void spmm_csc_kernel(int64_t p, int64_t n, const double* __restrict__ B, int64_t ldb,
                                const int64_t* __restrict__ col_ptr, const int64_t* __restrict__ row_idx,
                                const double* __restrict__ val, double* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double acc[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) acc[r] = 0.0;
    const int64_t t0 = col_ptr[j], t1 = col_ptr[j + 1];
    for (int64_t t = t0; t < t1; ++t) {
      const double a = val[t];
      const double* b = B + row_idx[t] * ldb;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int64_t i = lane + 32 * r;
        if (i < p) acc[r] = fma(a, __ldg(b + i), acc[r]);
      }
    }
    double* o = out + j * ldo;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int64_t i = lane + 32 * r;
      if (i < p) o[i] = acc[r];
    }
  }
}

// general p: chunks of 512 rows
__global__ void spmm_csc_chunk_kernel(int64_t p, int64_t n, const double* __restrict__ B, int64_t ldb,
                                      const int64_t* __restrict__ col_ptr, const int64_t* __restrict__ row_idx,
                                      const double* __restrict__ val, double* __restrict__ out, int64_t ldo,
                                      int64_t r0) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double acc[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) acc[r] = 0.0;
    for (int64_t t = col_ptr[j]; t < col_ptr[j + 1]; ++t) {
      const double a = val[t];
      const double* b = B + row_idx[t] * ldb + r0;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int64_t i = lane + 32 * r;
        if (r0 + i < p) acc[r] = fma(a, b[i], acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int64_t i = lane + 32 * r;
      if (r0 + i < p) out[j * ldo + r0 + i] = acc[r];
    }
  }
}

// counts[t] = ptr[sel[t]+1] - ptr[sel[t]]; out_ptr = exclusive scan (single block, k small)
__global__ void select_ptr_kernel(int64_t k, const int64_t* __restrict__ ptr, const int64_t* __restrict__ sel,
                                  int64_t* __restrict__ out_ptr) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t acc = 0;
  for (int64_t t = 0; t < k; ++t) {
    out_ptr[t] = acc;
    acc += ptr[sel[t] + 1] - ptr[sel[t]];
  }
  out_ptr[k] = acc;
}

// copy the selected compressed segments (columns of CSC or rows of CSR)
__global__ void extract_kernel(int64_t k, const int64_t* __restrict__ ptr, const int64_t* __restrict__ idx,
                               const double* __restrict__ val, const int64_t* __restrict__ sel,
                               const int64_t* __restrict__ out_ptr, int64_t* __restrict__ out_idx,
                               double* __restrict__ out_val) {
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < k;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t s0 = ptr[sel[t]], s1 = ptr[sel[t] + 1], o = out_ptr[t];
    for (int64_t q = s0 + lane; q < s1; q += 32) {
      out_idx[o + q - s0] = idx[q];
      out_val[o + q - s0] = val[q];
    }
  }
}

// dense (rows x k, ld) columns from a CSC extract: dense(idx, t) = val  (col-major, pre-zeroed)
__global__ void scatter_cols_kernel(int64_t k, const int64_t* __restrict__ ptr, const int64_t* __restrict__ idx,
                                    const double* __restrict__ val, double* __restrict__ dense, int64_t ld) {
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < k;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5)
    for (int64_t q = ptr[t] + lane; q < ptr[t + 1]; q += 32) dense[idx[q] + t * ld] = val[q];
}

// dense (k x cols, ld) rows from a CSR extract: dense(t, idx) = val
__global__ void scatter_rows_kernel(int64_t k, const int64_t* __restrict__ ptr, const int64_t* __restrict__ idx,
                                    const double* __restrict__ val, double* __restrict__ dense, int64_t ld) {
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < k;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5)
    for (int64_t q = ptr[t] + lane; q < ptr[t + 1]; q += 32) dense[t + idx[q] * ld] = val[q];
}

// partial sums of x*y over an m x n block (fixed grid -> deterministic)
__global__ void dot_kernel(int64_t m, int64_t n, const double* __restrict__ x, int64_t ldx,
                           const double* __restrict__ y, int64_t ldy, double* __restrict__ partials) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      acc = fma(x[i + j * ldx], y[i + j * ldy], acc);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    partials[blockIdx.x + (int64_t)blockIdx.y * gridDim.x] = t;
  }
}

inline int warps_grid(int64_t items, int wpb = 8) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((items + wpb - 1) / wpb, 64 * num_sms()));
}

}  // namespace

void csr_to_csc(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int64_t* col_idx, const double* val,
                int64_t* col_ptr, int64_t* row_idx, double* cval, cudaStream_t st) {
  if (nnz == 0) {
    LRB_CUDA(cudaMemsetAsync(col_ptr, 0, sizeof(int64_t) * (n + 1), st));
    return;
  }
  int64_t *rows = nullptr, *perm_in = nullptr, *perm_out = nullptr, *keys_out = nullptr;
  LRB_CUDA(cudaMallocAsync(&rows, sizeof(int64_t) * nnz, st));
  LRB_CUDA(cudaMallocAsync(&perm_in, sizeof(int64_t) * nnz, st));
  LRB_CUDA(cudaMallocAsync(&perm_out, sizeof(int64_t) * nnz, st));
  LRB_CUDA(cudaMallocAsync(&keys_out, sizeof(int64_t) * nnz, st));
  expand_rows_kernel<<<warps_grid(m), 256, 0, st>>>(m, row_ptr, rows);
  LRB_CHECK_LAUNCH();
  iota_kernel<<<warps_grid(nnz / 8 + 1), 256, 0, st>>>(nnz, perm_in);
  LRB_CHECK_LAUNCH();
  int end_bit = 1;
  while (end_bit < 64 && (int64_t(1) << end_bit) <= n) ++end_bit;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, col_idx, keys_out, perm_in, perm_out, nnz, 0, end_bit, st);
  void* tmp = nullptr;
  LRB_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
  LRB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, col_idx, keys_out, perm_in, perm_out, nnz, 0, end_bit,
                                           st));  // stable: rows stay ascending within a column
  ++g_kernel_launches;
  permute_kernel<<<warps_grid(nnz / 8 + 1), 256, 0, st>>>(nnz, perm_out, rows, val, row_idx, cval);
  LRB_CHECK_LAUNCH();
  bounds_kernel<<<warps_grid(n / 8 + 1), 256, 0, st>>>(nnz, n, keys_out, col_ptr);
  LRB_CHECK_LAUNCH();
  LRB_CUDA(cudaFreeAsync(tmp, st));
  LRB_CUDA(cudaFreeAsync(rows, st));
  LRB_CUDA(cudaFreeAsync(perm_in, st));
  LRB_CUDA(cudaFreeAsync(perm_out, st));
  LRB_CUDA(cudaFreeAsync(keys_out, st));
}

void spmm_csc(int64_t p, int64_t n, const double* B, int64_t ldb, const int64_t* col_ptr, const int64_t* row_idx,
              const double* val, double* out, int64_t ldo, cudaStream_t st) {
  if (p <= 0 || n <= 0) return;
  const int g = warps_grid(n);
  if (p <= 64) spmm_csc_kernel<2><<<g, 256, 0, st>>>(p, n, B, ldb, col_ptr, row_idx, val, out, ldo);
  else if (p <= 128) spmm_csc_kernel<4><<<g, 256, 0, st>>>(p, n, B, ldb, col_ptr, row_idx, val, out, ldo);
  else if (p <= 256) spmm_csc_kernel<8><<<g, 256, 0, st>>>(p, n, B, ldb, col_ptr, row_idx, val, out, ldo);
  else if (p <= 512) spmm_csc_kernel<16><<<g, 256, 0, st>>>(p, n, B, ldb, col_ptr, row_idx, val, out, ldo);
  else {
    for (int64_t r0 = 0; r0 < p; r0 += 512) {
      spmm_csc_chunk_kernel<<<g, 256, 0, st>>>(p, n, B, ldb, col_ptr, row_idx, val, out, ldo, r0);
      LRB_CHECK_LAUNCH();
    }
    return;
  }
  LRB_CHECK_LAUNCH();
}

void sparse_select(int64_t k, const int64_t* ptr, const int64_t* idx, const double* val, const int64_t* sel,
                   int64_t* out_ptr, int64_t* out_idx, double* out_val, cudaStream_t st) {
  select_ptr_kernel<<<1, 32, 0, st>>>(k, ptr, sel, out_ptr);
  LRB_CHECK_LAUNCH();
  extract_kernel<<<warps_grid(k), 256, 0, st>>>(k, ptr, idx, val, sel, out_ptr, out_idx, out_val);
  LRB_CHECK_LAUNCH();
}

void sparse_scatter_cols(int64_t rows, int64_t k, const int64_t* ptr, const int64_t* idx, const double* val,
                         double* dense, int64_t ld, cudaStream_t st) {
  LRB_CUDA(cudaMemset2DAsync(dense, ld * sizeof(double), 0, rows * sizeof(double), k, st));
  scatter_cols_kernel<<<warps_grid(k), 256, 0, st>>>(k, ptr, idx, val, dense, ld);
  LRB_CHECK_LAUNCH();
}

void sparse_scatter_rows(int64_t k, int64_t cols, const int64_t* ptr, const int64_t* idx, const double* val,
                         double* dense, int64_t ld, cudaStream_t st) {
  LRB_CUDA(cudaMemset2DAsync(dense, ld * sizeof(double), 0, k * sizeof(double), cols, st));
  scatter_rows_kernel<<<warps_grid(k), 256, 0, st>>>(k, ptr, idx, val, dense, ld);
  LRB_CHECK_LAUNCH();
}

void dot_sum(int64_t m, int64_t n, const double* x, int64_t ldx, const double* y, int64_t ldy, double* partials,
             int* num_partials, cudaStream_t st) {
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 8)),
            (unsigned)std::max<int64_t>(1, std::min<int64_t>(n, 512)));
  dot_kernel<<<grid, 256, 0, st>>>(m, n, x, ldx, y, ldy, partials);
  LRB_CHECK_LAUNCH();
  *num_partials = (int)(grid.x * grid.y);
}

}  // namespace lrb
