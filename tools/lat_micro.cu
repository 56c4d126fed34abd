#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double fast_rsqrt(double d) {
  if (!(d > 1e-30 && d < 1e30)) return rsqrt(d);
  double r = double(rsqrtf(float(d)));
  const double h = 0.5 * d;
  r = r * fma(-h, r * r, 1.5);
  r = r * fma(-h, r * r, 1.5);
  return r;
}
template <int V>
__global__ void k(double* o, double s, int n, long long* cyc) {
  double a = 1.5 + threadIdx.x * 1e-6;
  long long c0 = clock64();
  for (int t = 0; t < n; ++t) {
    if (V == 0) a = __shfl_sync(0xffffffffu, a, t & 31) * s + 1.0;            // shfl + DFMA
    if (V == 1) a = rsqrt(a) + 1.0;                                           // library rsqrt
    if (V == 2) a = fast_rsqrt(a) + 1.0;                                      // float seed + 2 Newton
    if (V == 3) a = double(rsqrtf(float(a))) + 1.0;                           // seed only
    if (V == 4) a = a * s + 1.0;                                              // DFMA
    if (V == 5) a = (a * s) * s;                                              // 2 DMUL
    if (V == 6) { float f = float(a); a = double(f) + 1.0; }                  // F2F round trip
  }
  long long c1 = clock64();
  o[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
int main() {
  double* o; long long* cyc; cudaMalloc(&o, 8192); cudaMallocManaged(&cyc, 8);
  const char* names[] = {"shfl.f64 + DFMA", "rsqrt(double) + DADD", "fast_rsqrt + DADD", "f32 rsqrt seed (F2F,MUFU,F2F) + DADD", "DFMA", "2 DMUL", "F2F.F32.F64 + F2F.F64.F32 + DADD"};
  const int n = 1024;
#define RUN(V) k<V><<<1, 32>>>(o, 0.999, n, cyc); cudaDeviceSynchronize(); k<V><<<1, 32>>>(o, 0.999, n, cyc); cudaDeviceSynchronize(); printf("%-40s %.1f cycles\n", names[V], double(*cyc) / n);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6)
  return 0;
}
