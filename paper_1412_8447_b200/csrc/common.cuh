// common.cuh -- shared device/host helpers for the B200 ID/CUR kernels.
// sm_100a only: DMMA (mma.sync .f64 -> SASS DMMA.8x8x4), TMA bulk tensor
// copies with mbarrier completion, cooperative grid sync.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

namespace lrb {

// ------------------------------------------------------------------ errors
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define LRB_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::lrb::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

// every kernel launch site calls this: error check + launch accounting
extern unsigned long long g_kernel_launches;
#define LRB_CHECK_LAUNCH()                     \
  do {                                         \
    ++::lrb::g_kernel_launches;                \
    LRB_CUDA(cudaGetLastError());              \
  } while (0)

constexpr int kNumSMsB200 = 148;

// SMs of the partition the calling thread is enqueueing for (a green-context
// stream, see api.cu tsid_cur_split), else 0 = the whole device
extern thread_local int g_sm_budget;

inline int num_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : kNumSMsB200;
  }();
  return g_sm_budget > 0 && g_sm_budget < n ? g_sm_budget : n;
}

// ------------------------------------------------------------ device utils
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// D = A(8x4,row) * B(4x8,col) + D, fp64.  Fragment ownership (lane l):
//   a = A[l/4][l%4], b = B[l%4][l/4], d = {D[l/4][2(l%4)], D[l/4][2(l%4)+1]}
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra.uni DONE;\n"
      "bra.uni LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 2D TMA tile load: global (tensor map) -> shared, completion on mbarrier
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ------------------------------------------------------- warp reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------ tensor maps
// Column-major fp64 matrix (rows x cols, ld) viewed as a 2D tensor with the
// row index fastest.  Box = {box_rows, box_cols}; 128B swizzle requires
// box_rows * 8 == 128.
CUtensorMap make_tmap_f64(const double* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                          int box_cols, bool swizzle128);

}  // namespace lrb
