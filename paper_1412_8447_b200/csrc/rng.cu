// rng.cu -- Gaussian test/sketch matrices with the reference stream semantics
// (rng.hpp:14-94): element (i,j) of a rows x cols matrix uses linear stream
// index e = i*cols + j of a counter-mode SplitMix64 stream; pairs (e, e+1)
// with e even feed one Box-Muller transform, r*cos(theta) -> e, r*sin(theta)
// -> e+1.  The integer stream is bit-exact; the transcendental functions are
// CUDA's (log 1 ulp, sin/cos <= 2 ulp), so entries agree with glibc to a few
// ulp rather than bitwise (hard part 4).
#include "common.cuh"
#include "kernels.h"

namespace lrb {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t stream_value(uint64_t seed, uint64_t index) {
  return mix64(seed + (index + 1) * 0x9E3779B97F4A7C15ULL);
}

// one thread per stream pair; `transposed` writes out(j, i) (coalesced)
__global__ void gaussian_kernel(int64_t rows, int64_t cols, uint64_t seed, double* __restrict__ out, int64_t ldo,
                                int transposed) {
  const int64_t total = rows * cols;
  const int64_t npairs = (total + 1) / 2;
  const double two_pi = 2.0 * 3.14159265358979323846;
  for (int64_t pr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pr < npairs;
       pr += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t e = (uint64_t)pr * 2;
    const double u1 = (double)((stream_value(seed, e) >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(stream_value(seed, e + 1) >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = two_pi * u2;
    double sn, cs;
    sincos(angle, &sn, &cs);
    const int64_t i0 = (int64_t)e / cols, j0 = (int64_t)e % cols;
    const double v0 = radius * cs;
    if (transposed) out[j0 + i0 * ldo] = v0;
    else out[i0 + j0 * ldo] = v0;
    if ((int64_t)e + 1 < total) {
      const int64_t i1 = ((int64_t)e + 1) / cols, j1 = ((int64_t)e + 1) % cols;
      const double v1 = radius * sn;
      if (transposed) out[j1 + i1 * ldo] = v1;
      else out[i1 + j1 * ldo] = v1;
    }
  }
}

}  // namespace

void gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out, int64_t ldo, bool transposed,
                     cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  const int64_t npairs = (rows * cols + 1) / 2;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((npairs + 255) / 256, 32 * num_sms()));
  gaussian_kernel<<<g, 256, 0, st>>>(rows, cols, seed, out, ldo, transposed ? 1 : 0);
  LRB_CHECK_LAUNCH();
}

// sketch.hpp:84-100 srft_operator, stored transposed (out[i + j*ldo] = Omega(j, i)):
// Omega(j, i) = sqrt(m/ell) * (cas(2 pi ((rows_j i) mod m) / m) / sqrt(m)) * sign_i,
// sign_i = -1 if stream_value(sign_seed, i) is odd (hartley.hpp:60-73).
__global__ void srft_operator_t_kernel(int64_t m, int64_t ell, uint64_t sign_seed, const int64_t* __restrict__ rows,
                                       double* __restrict__ out, int64_t ldo) {
  const double hs = 1.0 / sqrt((double)m), scale = sqrt((double)m / (double)ell);
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * ell; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % m, j = t / m;
    const double sg = (stream_value(sign_seed, (uint64_t)i) & 1u) ? -1.0 : 1.0;
    const double ang = two_pi * (double)((rows[j] * i) % m) / (double)m;
    double sn, cs;
    sincos(ang, &sn, &cs);
    out[i + j * ldo] = scale * ((hs * (cs + sn)) * sg);
  }
}

void srft_operator_t(int64_t m, int64_t ell, uint64_t sign_seed, const int64_t* rows, double* out, int64_t ldo,
                     cudaStream_t st) {
  if (m <= 0 || ell <= 0) return;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((m * ell + 255) / 256, 32 * num_sms()));
  srft_operator_t_kernel<<<g, 256, 0, st>>>(m, ell, sign_seed, rows, out, ldo);
  LRB_CHECK_LAUNCH();
}

}  // namespace lrb
