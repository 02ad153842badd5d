// verify.cu -- device pieces of the verifiers (verify.hpp:58-166): the row
// scatter of the permuted stack [0; F E] of Lemma 2 (verify.hpp:108-117).
#include "common.cuh"
#include "kernels.h"

namespace lrb {

namespace {
// out(piv[l], :) = l < k ? (top ? top(l, :) : 0) : res(l - k, :)   (out m x b)
__global__ void scatter_stack_kernel(int64_t m, int64_t b, int64_t k, const int64_t* __restrict__ piv,
                                     const double* __restrict__ top, int64_t ldt, const double* __restrict__ res,
                                     int64_t ldr, double* __restrict__ out, int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * b) return;
  const int64_t l = e % m, j = e / m;
  const double v = l < k ? (top ? top[j * ldt + l] : 0.0) : res[j * ldr + (l - k)];
  out[j * ldo + piv[l]] = v;
}
}  // namespace

void scatter_stack(int64_t m, int64_t b, int64_t k, const int64_t* piv, const double* top, int64_t ldt,
                   const double* res, int64_t ldr, double* out, int64_t ldo, cudaStream_t st) {
  const int64_t tot = m * b;
  scatter_stack_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(m, b, k, piv, top, ldt, res, ldr, out, ldo);
  LRB_CHECK_LAUNCH();
}

}  // namespace lrb
