// jacobi.cu -- one-sided (Hestenes) Jacobi SVD on the GPU, restating the
// convergence rules of svd.hpp:39-93 and the assembly of svd.hpp:132-183:
//   * per sweep: exact column norms, eps^2 floor relative to the largest,
//     negligible columns zeroed (svd.hpp:47-58);
//   * a pair is skipped when either norm is zero or |a_pq|/sqrt(a_pp a_qq)
//     <= 1e-14; the rotation and the running norm updates use the reference
//     formulas (svd.hpp:62-88); convergence when the sweep's worst coupling is
//     <= 1e-14, at most 60 sweeps (ConvergenceError otherwise);
//   * sigma = column norms, stable descending order, u = b/sigma above the
//     eps*max(m,n)*sigma_1 cutoff, deterministic basis completion otherwise.
// The pair order is the parallel round-robin (circle) ordering instead of
// the reference's cyclic p<q order, so results agree to rounding (the
// sweep's pairs are disjoint and run as independent CTAs).  This is the
// general / fallback path; the CUR hot path uses CholeskyQR2 (see api.cpp).
#include <algorithm>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace lrb {

namespace {

constexpr double kRelTol = 1e-14;
constexpr int kMaxSweeps = 60;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  __syncthreads();
  return t;
}

__global__ void col_norm2_kernel(int64_t m, int64_t n, const double* __restrict__ b, double* __restrict__ nrm) {
  __shared__ double sh[32];
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc = fma(b[i + j * m], b[i + j * m], acc);
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) nrm[j] = s;
  }
}

// floor2 = max(norm2) * eps^2; zero negligible columns; reset worst
__global__ void sweep_start_kernel(int64_t m, int64_t n, double* __restrict__ b, double* __restrict__ nrm,
                                   double* __restrict__ state) {
  __shared__ double sh_floor;
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int64_t j = 0; j < n; ++j) mx = (j == 0 || nrm[j] > mx) ? nrm[j] : mx;
    const double eps = 2.220446049250313e-16;
    sh_floor = mx * eps * eps;
    state[0] = sh_floor;
    reinterpret_cast<unsigned long long*>(state)[1] = 0ull;  // worst (as bits of a nonnegative double)
  }
  __syncthreads();
  const double floor2 = sh_floor;
  for (int64_t j = 0; j < n; ++j) {
    if (nrm[j] <= floor2 && nrm[j] != 0.0) {
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) b[i + j * m] = 0.0;
      __syncthreads();
      if (threadIdx.x == 0) nrm[j] = 0.0;
      __syncthreads();
    }
  }
}

// one CTA per pair of the round
__global__ void jacobi_round_kernel(int64_t m, int64_t n, int64_t N, int64_t round, double* __restrict__ b,
                                    double* __restrict__ v, double* __restrict__ nrm, double* __restrict__ state) {
  __shared__ double sh[32];
  const int64_t t = blockIdx.x;
  int64_t p, q;
  if (t == 0) { p = N - 1; q = round; }
  else { p = (round + t) % (N - 1); q = (round - t + N - 1) % (N - 1); }
  if (p > q) { const int64_t x = p; p = q; q = x; }
  if (q >= n) return;  // dummy player
  const double app = nrm[p], aqq = nrm[q];
  if (app == 0.0 || aqq == 0.0) return;
  double* bp = b + p * m;
  double* bq = b + q * m;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc = fma(bp[i], bq[i], acc);
  const double apq = block_sum(acc, sh);
  const double rel = fabs(apq) / sqrt(app * aqq);
  if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(state) + 1, __double_as_longlong(rel));
  if (rel <= kRelTol) return;
  const double theta = (aqq - app) / (2.0 * apq);
  const double tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
  const double c = 1.0 / sqrt(1.0 + tt * tt);
  const double s = c * tt;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double x = bp[i], y = bq[i];
    bp[i] = c * x - s * y;
    bq[i] = s * x + c * y;
  }
  double* vp = v + p * n;
  double* vq = v + q * n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = vp[i], y = vq[i];
    vp[i] = c * x - s * y;
    vq[i] = s * x + c * y;
  }
  const double floor2 = state[0];
  double np = c * c * app - 2.0 * c * s * apq + s * s * aqq;
  double nq = s * s * app + 2.0 * c * s * apq + c * c * aqq;
  np = np > 0.0 ? np : 0.0;
  nq = nq > 0.0 ? nq : 0.0;
  const bool dp = np <= floor2 && np != 0.0, dq = nq <= floor2 && nq != 0.0;
  if (dp) for (int64_t i = threadIdx.x; i < m; i += blockDim.x) bp[i] = 0.0;
  if (dq) for (int64_t i = threadIdx.x; i < m; i += blockDim.x) bq[i] = 0.0;
  if (threadIdx.x == 0) {
    nrm[p] = dp ? 0.0 : np;
    nrm[q] = dq ? 0.0 : nq;
  }
}

__global__ void identity_kernel(int64_t n, double* v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n; t += (int64_t)gridDim.x * blockDim.x)
    v[t] = (t % n) == (t / n) ? 1.0 : 0.0;
}

// u(:, j) = b(:, order[j]) / sigma_j (or 0 below cutoff), v_out(:, j) = v(:, order[j])
__global__ void assemble_kernel(int64_t m, int64_t n, const double* __restrict__ b, const double* __restrict__ v,
                                const int64_t* __restrict__ order, const double* __restrict__ sig, double cutoff,
                                double* __restrict__ u, double* __restrict__ vout, double* __restrict__ sigma) {
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const int64_t src = order[j];
    const double sj = sig[src];
    if (threadIdx.x == 0) sigma[j] = sj;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) u[i + j * m] = sj > cutoff ? b[i + src * m] / sj : 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) vout[i + j * n] = v[i + src * n];
  }
}

// svd.hpp:97-120, one CTA (rare path: only for numerically zero singular values)
__global__ void complete_basis_kernel(int64_t m, int64_t n, double* __restrict__ u, const int64_t* __restrict__ zc,
                                      int64_t nz, double* __restrict__ e) {
  __shared__ double sh[32];
  __shared__ int accept;
  int64_t candidate = 0;
  for (int64_t zi = 0; zi < nz; ++zi) {
    const int64_t col = zc[zi];
    for (; candidate < m; ++candidate) {
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) e[i] = (i == candidate) ? 1.0 : 0.0;
      __syncthreads();
      for (int64_t j = 0; j < n; ++j) {
        bool pending = false;
        for (int64_t t = 0; t < nz; ++t)
          if (zc[t] == j) { pending = j >= col; break; }
        if (pending) continue;
        double acc = 0.0;
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc = fma(u[i + j * m], e[i], acc);
        const double d = block_sum(acc, sh);
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) e[i] -= d * u[i + j * m];
        __syncthreads();
      }
      double acc = 0.0;
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc = fma(e[i], e[i], acc);
      const double nrm = sqrt(block_sum(acc, sh));
      if (threadIdx.x == 0) accept = nrm > 0.5;
      __syncthreads();
      if (accept) {
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) u[i + col * m] = e[i] / nrm;
        __syncthreads();
        ++candidate;
        break;
      }
    }
  }
}

}  // namespace

bool jacobi_svd(Workspace& ws, int64_t m, int64_t n, const double* a, int64_t lda, double* u, double* sigma,
                double* v, cudaStream_t st) {
  // b (m x n working copy, ld m), vv (n x n), nrm (n), state (2)
  double* b = nullptr;
  double* vv = nullptr;
  double* nrm = nullptr;
  double* state = nullptr;
  LRB_CUDA(cudaMallocAsync(&b, sizeof(double) * m * n, st));
  LRB_CUDA(cudaMallocAsync(&vv, sizeof(double) * n * n, st));
  LRB_CUDA(cudaMallocAsync(&nrm, sizeof(double) * (n + 4), st));
  state = nrm + n;
  copy_matrix(m, n, a, lda, b, m, st);
  identity_kernel<<<std::max<int64_t>(1, std::min<int64_t>((n * n + 255) / 256, 1024)), 256, 0, st>>>(n, vv);
  LRB_CHECK_LAUNCH();
  const int64_t N = n + (n & 1);
  const int blk = m >= 4096 ? 512 : 256;
  bool converged = false;
  for (int sweep = 0; sweep < kMaxSweeps && !converged; ++sweep) {
    col_norm2_kernel<<<(unsigned)std::min<int64_t>(n, 4 * num_sms()), 256, 0, st>>>(m, n, b, nrm);
    LRB_CHECK_LAUNCH();
    sweep_start_kernel<<<1, 256, 0, st>>>(m, n, b, nrm, state);
    LRB_CHECK_LAUNCH();
    if (N >= 2)
      for (int64_t r = 0; r < N - 1; ++r) {
        jacobi_round_kernel<<<(unsigned)(N / 2), blk, 0, st>>>(m, n, N, r, b, vv, nrm, state);
        LRB_CHECK_LAUNCH();
      }
    unsigned long long worst_bits = 0;
    LRB_CUDA(cudaMemcpyAsync(&worst_bits, reinterpret_cast<unsigned long long*>(state) + 1, sizeof(worst_bits),
                             cudaMemcpyDeviceToHost, st));
    LRB_CUDA(cudaStreamSynchronize(st));
    double worst;
    memcpy(&worst, &worst_bits, sizeof(worst));
    converged = worst <= kRelTol;
  }
  if (!converged) {
    cudaFreeAsync(b, st);
    cudaFreeAsync(vv, st);
    cudaFreeAsync(nrm, st);
    return false;
  }
  // sigma = column norms; stable descending order (svd.hpp:150-158)
  col_norm2_kernel<<<(unsigned)std::min<int64_t>(n, 4 * num_sms()), 256, 0, st>>>(m, n, b, nrm);
  LRB_CHECK_LAUNCH();
  std::vector<double> h(n);
  LRB_CUDA(cudaMemcpyAsync(h.data(), nrm, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  LRB_CUDA(cudaStreamSynchronize(st));
  for (auto& x : h) x = std::sqrt(x);
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), int64_t(0));
  std::stable_sort(order.begin(), order.end(), [&](int64_t i, int64_t j) { return h[i] > h[j]; });
  const double eps = 2.220446049250313e-16;
  const double cutoff = h[order[0]] * eps * (double)std::max(m, n);
  std::vector<int64_t> zc;
  for (int64_t j = 0; j < n; ++j)
    if (!(h[order[j]] > cutoff)) zc.push_back(j);
  int64_t* d_order = nullptr;
  double* d_sig = nullptr;
  LRB_CUDA(cudaMallocAsync(&d_order, sizeof(int64_t) * (n + zc.size() + 1), st));
  LRB_CUDA(cudaMallocAsync(&d_sig, sizeof(double) * n, st));
  LRB_CUDA(cudaMemcpyAsync(d_order, order.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  LRB_CUDA(cudaMemcpyAsync(d_sig, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  assemble_kernel<<<(unsigned)std::min<int64_t>(n, 4 * num_sms()), 256, 0, st>>>(m, n, b, vv, d_order, d_sig,
                                                                                  cutoff, u, v, sigma);
  LRB_CHECK_LAUNCH();
  if (!zc.empty()) {
    LRB_CUDA(cudaMemcpyAsync(d_order + n, zc.data(), sizeof(int64_t) * zc.size(), cudaMemcpyHostToDevice, st));
    complete_basis_kernel<<<1, 256, 0, st>>>(m, n, u, d_order + n, (int64_t)zc.size(), b);
    LRB_CHECK_LAUNCH();
  }
  LRB_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(d_order, st);
  cudaFreeAsync(d_sig, st);
  cudaFreeAsync(b, st);
  cudaFreeAsync(vv, st);
  cudaFreeAsync(nrm, st);
  return true;
}

}  // namespace lrb
