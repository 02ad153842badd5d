// Probe: green-context SM partitions from the runtime API -- primary-context
// memory, <<<>>> and cooperative launches on green-context streams, and
// whether two partitions run kernels concurrently.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o green_ctx green_ctx.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
#include <set>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
  printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(r)); \
  return 1; } } while (0)

__global__ void smid_kernel(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

__global__ void coop_kernel(int* out, unsigned int* bar) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  cooperative_groups::this_grid().sync();
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

__global__ void spin_kernel(long long cycles, unsigned long long* t) {
  const long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  while (clock64() - t0 < cycles) {}
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && blockIdx.x == 0) { t[0] = g0; t[1] = g1; }
}

__global__ void __cluster_dims__(4, 1, 1) cluster_kernel(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

int main() {
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  int* d = nullptr;
  RK(cudaMalloc(&d, 4096 * sizeof(int)));
  unsigned long long* t = nullptr;
  RK(cudaMalloc(&t, 4 * sizeof(unsigned long long)));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource res{};
  CK(cuDeviceGetDevResource(dev, &res, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", res.sm.smCount);
  CUdevResource groups[1], rest{};
  unsigned nb = 1;
  CK(cuDevSmResourceSplitByCount(groups, &nb, &res, &rest, 0, 48));
  printf("split: group %u SMs, remaining %u SMs\n", groups[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc da, db;
  CK(cuDevResourceGenerateDesc(&da, &groups[0], 1));
  CK(cuDevResourceGenerateDesc(&db, &rest, 1));
  CUgreenCtx ga, gb;
  CK(cuGreenCtxCreate(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sa, sb;
  CK(cuGreenCtxStreamCreate(&sa, ga, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&sb, gb, CU_STREAM_NON_BLOCKING, 0));
  // (1) plain launch on partition A, primary-context memory
  smid_kernel<<<512, 64, 0, (cudaStream_t)sa>>>(d);
  RK(cudaGetLastError());
  RK(cudaStreamSynchronize((cudaStream_t)sa));
  std::vector<int> h(512);
  RK(cudaMemcpy(h.data(), d, 512 * sizeof(int), cudaMemcpyDeviceToHost));
  std::set<int> sms(h.begin(), h.end());
  printf("plain launch on A: %zu distinct SMs\n", sms.size());
  // (2) cooperative launch with the partition's SM count
  int G = (int)groups[0].sm.smCount;
  void* args[] = {&d, &t};
  cudaError_t ce = cudaLaunchCooperativeKernel((void*)coop_kernel, dim3(G), dim3(256), args, 0, (cudaStream_t)sa);
  printf("cooperative launch G=%d on A: %s\n", G, cudaGetErrorString(ce));
  if (ce == cudaSuccess) {
    RK(cudaStreamSynchronize((cudaStream_t)sa));
    RK(cudaMemcpy(h.data(), d, G * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> s2(h.begin(), h.begin() + G);
    printf("cooperative kernel ran on %zu distinct SMs\n", s2.size());
  }
  int occ = 0;
  RK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, coop_kernel, 256, 0));
  // (3) concurrency: 200M-cycle spin on A and on B at once
  spin_kernel<<<G, 32, 0, (cudaStream_t)sa>>>(200000000LL, t);
  spin_kernel<<<(int)rest.sm.smCount, 32, 0, (cudaStream_t)sb>>>(200000000LL, t + 2);
  RK(cudaGetLastError());
  RK(cudaDeviceSynchronize());
  unsigned long long ht[4];
  RK(cudaMemcpy(ht, t, sizeof ht, cudaMemcpyDeviceToHost));
  printf("spin A [%.3f, %.3f] ms, B [%.3f, %.3f] ms (relative to A start)\n", 0.0, (ht[1] - ht[0]) / 1e6,
         ((double)ht[2] - (double)ht[0]) / 1e6, ((double)ht[3] - (double)ht[0]) / 1e6);
  // (4) cross-stream event from the primary-context stream into a green stream
  cudaEvent_t ev;
  RK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  RK(cudaEventRecord(ev, 0));
  RK(cudaStreamWaitEvent((cudaStream_t)sa, ev, 0));
  smid_kernel<<<4, 32, 0, (cudaStream_t)sa>>>(d);
  RK(cudaStreamSynchronize((cudaStream_t)sa));
  printf("event wait across contexts: ok\n");
  // (5) 4-CTA cluster kernel on each partition (200 clusters)
  for (int pass = 0; pass < 2; ++pass) {
    cudaStream_t st = (cudaStream_t)(pass ? sb : sa);
    cluster_kernel<<<800, 64, 0, st>>>(d);
    cudaError_t e1 = cudaGetLastError();
    cudaError_t e2 = cudaStreamSynchronize(st);
    RK(cudaMemcpy(h.data(), d, 512 * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> s3(h.begin(), h.begin() + 512);
    printf("cluster kernel on %s: launch %s, sync %s, %zu distinct SMs\n", pass ? "B" : "A", cudaGetErrorString(e1),
           cudaGetErrorString(e2), s3.size());
  }
  return 0;
}
