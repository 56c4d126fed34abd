// Microbenchmark of the per-pivot building blocks of a one-CTA 64-pivot
// factorisation (512 threads): barrier, shared column exchange, FP64 rsqrt,
// shuffle, FP64 update chains.  Prints cycles per pivot measured in-kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/chol_micro tools/chol_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void __launch_bounds__(512) micro(double* out, long long* cyc, double seed) {
  __shared__ double2 col[2][64];
  __shared__ double dinf[2];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double2 a[6];
  for (int s = 0; s < 6; ++s) a[s] = make_double2(seed + tid + s, seed - s);
  if (tid < 64) col[0][tid] = make_double2(1.0 + tid, 0.5);
  if (tid == 0) dinf[0] = 2.0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int k = 0; k < 64; ++k) {
    __syncthreads();
    const double2* ck = col[k & 1];
    double2* cn = col[(k + 1) & 1];
    if (V == 0) {  // barrier + one LDS + one STS
      const double2 c = ck[lane];
      if (w == (k & 15)) cn[lane] = make_double2(c.x + 1.0, c.y);
    } else if (V == 1) {  // + rsqrt by one lane, published
      const double2 c = ck[lane];
      const double invd = dinf[k & 1];
      if (w == (k & 15)) {
        cn[lane] = make_double2(c.x * invd, c.y);
        if (lane == 0) dinf[(k + 1) & 1] = rsqrt(c.x + 3.0);
      }
    } else if (V == 2) {  // + shuffle before rsqrt
      const double2 c = ck[lane];
      const double invd = dinf[k & 1];
      if (w == (k & 15)) {
        cn[lane] = make_double2(c.x * invd, c.y);
        const double d = __shfl_sync(0xffffffffu, c.x, k & 31);
        if (lane == 0) dinf[(k + 1) & 1] = rsqrt(d + 3.0);
      }
    } else if (V == 3) {  // + 6 complex updates per thread (all warps), owner publishes after its first
      const double2 ci0 = ck[lane], ci1 = ck[lane + 32];
      const double invd = dinf[k & 1];
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const double2 cj = ck[(w + 16 * s) & 63];
        const double2 ci = (s & 1) ? ci1 : ci0;
        const double tr = ci.x * cj.x + ci.y * cj.y, tim = ci.y * cj.x - ci.x * cj.y;
        a[s].x = fma(-tr, invd * 1e-3, a[s].x);
        a[s].y = fma(-tim, invd * 1e-3, a[s].y);
        if (s == 0 && w == (k & 15)) {
          cn[lane] = a[0];
          cn[lane + 32] = a[1];
          const double d = __shfl_sync(0xffffffffu, a[0].x, k & 31);
          if (lane == 0) dinf[(k + 1) & 1] = rsqrt(fabs(d) + 3.0);
        }
      }
    } else if (V == 4) {  // updates only, no publish chain
      const double2 ci0 = ck[lane], ci1 = ck[lane + 32];
      const double invd = dinf[k & 1];
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const double2 cj = ck[(w + 16 * s) & 63];
        const double2 ci = (s & 1) ? ci1 : ci0;
        const double tr = ci.x * cj.x + ci.y * cj.y, tim = ci.y * cj.x - ci.x * cj.y;
        a[s].x = fma(-tr, invd * 1e-3, a[s].x);
        a[s].y = fma(-tim, invd * 1e-3, a[s].y);
      }
    } else if (V == 5) {  // barrier only
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double acc = 0;
  for (int s = 0; s < 6; ++s) acc += a[s].x + a[s].y;
  out[tid] = acc;
  if (tid == 0) cyc[0] = t1 - t0;
}

template <int V>
void run(double* out, long long* cyc, const char* name) {
  long long h = 0;
  for (int rep = 0; rep < 3; ++rep) {
    micro<V><<<1, 512>>>(out, cyc, 1.0);
    cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 100; ++rep) micro<V><<<1, 512>>>(out, cyc, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::printf("%-44s %7.1f cycles/pivot   %6.2f us/launch\n", name, double(h) / 64.0, ms * 10.0);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 512 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  run<5>(out, cyc, "barrier only");
  run<0>(out, cyc, "barrier + LDS + STS");
  run<1>(out, cyc, "+ rsqrt(double) by one lane");
  run<2>(out, cyc, "+ shuffle before rsqrt");
  run<4>(out, cyc, "6 cplx updates / thread, no publish");
  run<3>(out, cyc, "6 cplx updates + publish chain");
  std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
