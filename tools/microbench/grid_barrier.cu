// Grid-barrier latency on the B200: a co-resident grid (one CTA per SM) runs
// N barriers back to back; variants of arrival / spin.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o grid_barrier grid_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int V>
__global__ void bar_kernel(unsigned int* bar, int iters, unsigned long long* out) {
  unsigned int target = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (V == 0) {
      cg::this_grid().sync();
      continue;
    }
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      if (V == 1) {  // release red + acquire spin
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned int v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while (v < target);
      } else if (V == 2) {  // release red + relaxed spin + acquire fence
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned int v;
        do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while (v < target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (V == 3) {  // fence + relaxed red + volatile spin + fence
        __threadfence();
        atomicAdd(bar, 1u);
        volatile unsigned int* vb = bar;
        while (*vb < target) {}
        __threadfence();
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

template <int V>
void run(int G, int iters) {
  unsigned int* bar;
  unsigned long long* out;
  cudaMalloc(&bar, 4);
  cudaMalloc(&out, 8);
  cudaMemset(bar, 0, 4);
  void* args[] = {&bar, &iters, &out};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchCooperativeKernel((void*)bar_kernel<V>, G, 256, args, 0, 0);  // warm
  cudaMemset(bar, 0, 4);
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((void*)bar_kernel<V>, G, 256, args, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"variant\": %d, \"ctas\": %d, \"us_per_barrier\": %.3f}\n", V, G, 1e3 * ms / iters);
  cudaFree(bar);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int G : {sms / 2, sms}) {
    run<0>(G, 2000);
    run<1>(G, 2000);
    run<2>(G, 2000);
    run<3>(G, 2000);
  }
  return 0;
}
