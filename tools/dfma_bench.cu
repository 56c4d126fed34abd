#include <cstdio>
#include <cuda_runtime.h>
__global__ void thr(double* o, double s, int n) {  // 8 independent chains per thread
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int t = 0; t < n; ++t)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 0.5);
  double r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  o[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void lat(double* o, double s, int n, long long* cyc) {  // one dependent chain
  double a = threadIdx.x * 1e-3;
  long long c0 = clock64();
  for (int t = 0; t < n; ++t) a = fma(a, s, 0.5);
  long long c1 = clock64();
  o[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
__global__ void lat_rcp(double* o, double s, int n, long long* cyc) {
  double a = 1.5 + threadIdx.x * 1e-3;
  long long c0 = clock64();
  for (int t = 0; t < n; ++t) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); a = r + 1.0; }
  long long c1 = clock64();
  o[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
__global__ void lat_lds(double* o, int n, long long* cyc) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
  __syncthreads();
  int p = 0;
  long long c0 = clock64();
  for (int t = 0; t < n; ++t) p = idx[p];
  long long c1 = clock64();
  o[threadIdx.x] = p;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
__global__ void lat_sync(double* o, int n, long long* cyc) {
  long long c0 = clock64();
  for (int t = 0; t < n; ++t) __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, 1 << 26);
  long long* cyc; cudaMallocManaged(&cyc, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); thr<<<sms * 4, 256>>>(o, 0.999, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA throughput: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1.965 GHz)\n", 2.0 * 8 * n * sms * 4 * 256 / ms / 1e9,
           8.0 * n * sms * 4 * 256 / (ms * 1e-3) / sms / 1.965e9);
  }
  lat<<<1, 32>>>(o, 0.999, n, cyc); cudaDeviceSynchronize(); printf("DFMA latency: %.1f cycles\n", double(*cyc) / n);
  lat_rcp<<<1, 32>>>(o, 0.999, n, cyc); cudaDeviceSynchronize(); printf("rcp64+DADD latency: %.1f cycles\n", double(*cyc) / n);
  lat_lds<<<1, 32>>>(o, n, cyc); cudaDeviceSynchronize(); printf("LDS latency: %.1f cycles\n", double(*cyc) / n);
  lat_sync<<<1, 512>>>(o, n, cyc); cudaDeviceSynchronize(); printf("syncthreads(512): %.1f cycles\n", double(*cyc) / n);
  return 0;
}
