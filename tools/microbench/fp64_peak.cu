// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 .f64) and DFMA.
// Prints one JSON line per measurement. Used to fill MEASURED_PEAKS-style FP64 numbers
// (the driver-written MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("{\"device\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\",\"smem_optin\":%zu,\"l2\":%d,\"regs_per_sm\":%d}\n",
         p.name, p.multiProcessorCount, p.major, p.minor, p.sharedMemPerBlockOptin, p.l2CacheSize, p.regsPerMultiprocessor);
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16, 32}) {
    for (int cps : {1, 2}) {
      int iters = 20000;
      dmma_loop<<<sms * cps, warps * 32>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<<<sms * cps, warps * 32>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = 2.0 * 256 * 8 * (double)iters * warps * sms * cps;
      printf("{\"kind\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"ctas_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", warps, cps, ms, flop / ms / 1e9);
    }
  }
  for (int warps : {8, 16, 32}) {
    int iters = 20000;
    dfma_loop<<<sms * 2, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 16 * (double)iters * warps * 32 * sms * 2;
    printf("{\"kind\":\"dfma\",\"warps_per_cta\":%d,\"ctas_per_sm\":2,\"ms\":%.3f,\"tflops\":%.3f}\n", warps, ms, flop / ms / 1e9);
  }
  size_t n = (size_t)1 << 28;  // 4 GiB per buffer in double2
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kind\":\"copy\",\"GBps\":%.1f}\n", 2.0 * n * 16 / ms / 1e6);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"status\":\"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
