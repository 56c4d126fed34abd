// Throughput of legacy warp-level mma.sync (m16n8k8 TF32, m16n8k16 BF16) on B200.
#include <cstdio>
#include <cuda_runtime.h>
template <int KIND>
__global__ void k(float* out, int n) {
  float c[8][4] = {};
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  for (int t = 0; t < n; ++t) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int sms = 148, n = 4096;
  for (int kind = 0; kind < 2; ++kind)
    for (int warps : {4, 8, 16}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      if (kind == 0) k<0><<<sms * 4, 32 * warps>>>(o, 16); else k<1><<<sms * 4, 32 * warps>>>(o, 16);
      cudaEventRecord(e0);
      if (kind == 0) k<0><<<sms * 4, 32 * warps>>>(o, n); else k<1><<<sms * 4, 32 * warps>>>(o, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double macs = double(sms) * 4 * warps * n * 8 * (kind == 0 ? 16 * 8 * 8 : 16 * 8 * 16);
      printf("%s warps/CTA=%2d (4 CTAs/SM): %.0f TFLOP/s dense\n", kind == 0 ? "tf32 m16n8k8 " : "bf16 m16n8k16", warps, 2 * macs / ms / 1e9);
    }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
