#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void f2(unsigned long long& d, unsigned long long a, unsigned long long b) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__global__ void k1(float* o, float s, int n) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
  for (int t = 0; t < n; ++t)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 0.5f);
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  o[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k2(float* o, float s, int n) {
  unsigned long long a[8];
  float2 sv = make_float2(s, s), hv = make_float2(0.5f, 0.5f);
  unsigned long long S = *reinterpret_cast<unsigned long long*>(&sv);
  for (int i = 0; i < 8; ++i) { float2 x = make_float2(threadIdx.x * 0.001f + i, i); a[i] = *reinterpret_cast<unsigned long long*>(&x); }
  for (int t = 0; t < n; ++t)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      unsigned long long d = *reinterpret_cast<unsigned long long*>(&hv);
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a[i]), "l"(S));
      a[i] = d;
    }
  float r = 0; for (int i = 0; i < 8; ++i) { float2 x = *reinterpret_cast<float2*>(&a[i]); r += x.x + x.y; }
  o[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 20000, blocks = sms * 4, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k1<<<blocks, threads>>>(o, 0.999f, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * n * double(blocks) * threads;
    printf("FFMA : %.2f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
    cudaEventRecord(e0); k2<<<blocks, threads>>>(o, 0.999f, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 4.0 * 8 * n * double(blocks) * threads;
    printf("FFMA2: %.2f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
  }
  return 0;
}
