#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void thr(double* o, double s, int n, long long* cyc) {
  double a[CH];
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3 + i;
  __syncthreads();
  long long c0 = clock64();
  for (int t = 0; t < n; ++t)
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = fma(a[i], s, 0.5);
  __syncthreads();
  long long c1 = clock64();
  double r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  o[threadIdx.x] = r;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
int main() {
  double* o; long long* cyc; cudaMalloc(&o, 8192); cudaMallocManaged(&cyc, 8);
  const int n = 4096;
  for (int warps : {1, 2, 4, 8, 16}) {
    thr<8><<<1, 32 * warps>>>(o, 0.999, n, cyc); cudaDeviceSynchronize();
    thr<8><<<1, 32 * warps>>>(o, 0.999, n, cyc); cudaDeviceSynchronize();
    double per = double(*cyc) / (n * 8.0);
    printf("warps=%2d  8 chains: %.2f cycles per warp-DFMA per warp, SM rate %.1f DFMA lanes/clk\n", warps, per, 32.0 * warps / per);
  }
  for (int warps : {1, 4}) {
    thr<16><<<1, 32 * warps>>>(o, 0.999, n, cyc); cudaDeviceSynchronize();
    thr<16><<<1, 32 * warps>>>(o, 0.999, n, cyc); cudaDeviceSynchronize();
    double per = double(*cyc) / (n * 16.0);
    printf("warps=%2d 16 chains: %.2f cycles per warp-DFMA per warp, SM rate %.1f DFMA lanes/clk\n", warps, per, 32.0 * warps / per);
  }
  return 0;
}
