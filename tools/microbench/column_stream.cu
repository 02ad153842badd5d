// Streaming-read microbenchmark in the CPQR pass's access pattern: one CTA per
// SM, W warps, each warp walks its columns (c0 + warp + W*it) of a 512-row
// column-major FP64 matrix with a D-deep register ring (8 x 16 B per lane per
// column), reducing each column with a warp dot.  Reports GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o column_stream column_stream.cu
#include <cstdio>

template <int W, int D>
__global__ void __launch_bounds__(W * 32, 1) stream_kernel(const double* __restrict__ a, int n, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = (int)((long long)n * blockIdx.x / gridDim.x), c1 = (int)((long long)n * (blockIdx.x + 1) / gridDim.x);
  const int cnt = (c1 - c0 - warp + W - 1) / W;
  double acc = 0.0;
  double2 buf[D][8];
  auto fetch = [&](double2 (&b)[8], int it) {
    const double* col = a + (size_t)(c0 + warp + W * it) * 512;
#pragma unroll
    for (int k = 0; k < 8; ++k) b[k] = __ldcs(reinterpret_cast<const double2*>(col + 64 * k + 2 * lane));
  };
#pragma unroll
  for (int u = 0; u < D - 1; ++u)
    if (u < cnt) fetch(buf[u], u);
  for (int q0 = 0; q0 < cnt; q0 += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int q = q0 + u;
      if (q >= cnt) break;
      if (q + D - 1 < cnt) fetch(buf[(u + D - 1) % D], q + D - 1);
      double d = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) d += buf[u][k].x * 1.0001 + buf[u][k].y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      acc += d;
    }
  }
  if (lane == 0) out[blockIdx.x * W + warp] = acc;
}

template <int W, int D>
void run(const double* a, int n, double* out, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  stream_kernel<W, D><<<sms, W * 32>>>(a, n, out);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) stream_kernel<W, D><<<sms, W * 32>>>(a, n, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double gb = 5.0 * 512.0 * 8.0 * n / 1e9;
  printf("{\"warps\": %d, \"ring\": %d, \"GBps\": %.1f}\n", W, D, gb / (ms * 1e-3));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n = 65536;
  double *a, *out;
  cudaMalloc(&a, (size_t)512 * n * 8);
  cudaMalloc(&out, 64 * 1024 * 8);
  cudaMemset(a, 0, (size_t)512 * n * 8);
  run<8, 2>(a, n, out, sms);
  run<8, 3>(a, n, out, sms);
  run<8, 4>(a, n, out, sms);
  run<8, 6>(a, n, out, sms);
  run<16, 2>(a, n, out, sms);
  run<16, 3>(a, n, out, sms);
  run<16, 4>(a, n, out, sms);
  run<32, 2>(a, n, out, sms);
  return 0;
}
