// Micro-benchmark of the K4 inner loop shape (one warp = one Q = 32 voxel,
// thread = matrix row in registers, v broadcast from shared memory): what
// bounds an iteration — the FFMA2 pipe, the shared-memory broadcast loads, or
// the per-iteration reduction/publish tail.
//   MODE 0: LDS.128 broadcast of v (the K4 scheme) + publish + shuffle norm
//   MODE 1: v from registers (no loads) + publish + shuffle norm
//   MODE 2: LDS.64 broadcast
//   MODE 3: LDS.128 broadcast, no publish / norm (products only)
//   MODE 4: LDS.128, v replicated per quarter-warp (quarter q reads copy q)
//   MODE 6: MODE 0 with the norm reduction only every 4th iteration
//   loop2<NRM>: two rows per thread (16 lanes per voxel, 2 voxels per warp,
//   1 block of 256 threads per SM); norm every NRM-th iteration
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/k4_loop_micro.cu -o tools/k4_loop_micro
#include <cstdio>
#include <cuda_runtime.h>
using u64 = unsigned long long;
__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void ffma2(u64& d, u64 a, u64 b) { asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b)); }
__device__ __forceinline__ float2 unpk(u64 x) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(x));
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) loop(float* out, int iters) {
  __shared__ __align__(16) float2 vs[2][8][4][34];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float2 m[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) m[c] = make_float2(0.01f * ((lane * 7 + c) % 13) - 0.06f, 0.003f * (c - lane));
  float2 vr[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) vr[c] = make_float2(0.17f, 0.01f * c);
  for (int q = 0; q < 4; ++q) vs[0][w][q][lane] = make_float2(0.17f, 0.01f * lane);
  __syncwarp();
  if constexpr (MODE == 7 || MODE == 8) {
#pragma unroll
    for (int c = 0; c < 32; ++c) vr[c] = vs[0][w][0][c];
  }
  float2 up = make_float2(0.17f, 0.f);
  float own = 1.f;
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    __syncwarp();
    u64 acc[2] = {0ull, 0ull}, acc2[2] = {0ull, 0ull};
    if constexpr (MODE == 7 || MODE == 8) {  // opaque zero: the products cannot be hoisted
      u64 z;
      asm volatile("mov.b64 %0, 0;" : "=l"(z));
      acc[0] = acc[1] = acc2[0] = acc2[1] = z;
    }
    if constexpr (MODE == 1 || MODE == 7 || MODE == 8) {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        ffma2(acc[c & 1], pk(m[c].x, m[c].x), pk(vr[c].x, vr[c].y));
        ffma2(acc2[c & 1], pk(m[c].y, m[c].y), pk(vr[c].y, vr[c].x));
      }
    } else if constexpr (MODE == 2) {
      const float2* v = vs[b][w][0];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float2 x = v[c];
        ffma2(acc[c & 1], pk(m[c].x, m[c].x), pk(x.x, x.y));
        ffma2(acc2[c & 1], pk(m[c].y, m[c].y), pk(x.y, x.x));
      }
    } else {
      const float4* v4 = reinterpret_cast<const float4*>(vs[b][w][MODE == 4 ? (lane >> 3) : 0]);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const float4 x = v4[t];
        ffma2(acc[0], pk(m[2 * t].x, m[2 * t].x), pk(x.x, x.y));
        ffma2(acc2[0], pk(m[2 * t].y, m[2 * t].y), pk(x.y, x.x));
        ffma2(acc[1], pk(m[2 * t + 1].x, m[2 * t + 1].x), pk(x.z, x.w));
        ffma2(acc2[1], pk(m[2 * t + 1].y, m[2 * t + 1].y), pk(x.w, x.z));
      }
    }
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float2 x = unpk(acc[k]), y = unpk(acc2[k]);
      s = make_float2(s.x + (x.x - y.x), s.y + (x.y + y.y));
    }
    if constexpr (MODE == 6) {
      const float inv = rsqrtf(own);
      up = make_float2((0.9f * up.x + s.x) * inv, (0.9f * up.y + s.y) * inv);
      vs[b ^ 1][w][0][lane] = up;
      if ((it & 3) == 3) {
        float x = up.x * up.x + up.y * up.y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        own = x;
      }
    } else if constexpr (MODE == 3 || MODE == 8) {
      up = make_float2(up.x * 0.5f + s.x, up.y * 0.5f + s.y);
      if (up.x == 12345.f) vs[b ^ 1][w][0][lane] = up;  // keep the loads live
    } else {
      const float inv = rsqrtf(own);
      up = make_float2((0.9f * up.x + s.x) * inv, (0.9f * up.y + s.y) * inv);
      if constexpr (MODE == 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) vs[b ^ 1][w][q][lane] = up;
      } else {
        vs[b ^ 1][w][0][lane] = up;
      }
      float x = up.x * up.x + up.y * up.y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      own = x;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = up.x + up.y;
}

template <int MODE>
void run(float* o, int sms, const char* name) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000, blocks = sms * 2, threads = 256;
  loop<MODE><<<blocks, threads>>>(o, 10);
  float ms;
  cudaEventRecord(e0);
  loop<MODE><<<blocks, threads>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  // algorithmic flops: 8 Q^2 per voxel-iteration, one voxel per warp
  const double fl = 8.0 * 32 * 32 * iters * double(blocks) * (threads / 32);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc_per_iter = ms * 1e-3 * clk * 1e3 / iters;
  printf("%-34s %.3f ms  %.1f TFLOP/s  %.0f cycles/iteration per SM (4 warps/SMSP; FFMA2 floor 512)\n", name, ms,
         fl / ms / 1e9, cyc_per_iter);
}


template <int NRM, int TH = 256, int MB = 1>
__global__ void __launch_bounds__(TH, MB) loop2(float* out, int iters) {
  __shared__ __align__(16) float2 vs[2][TH / 16][34];
  const int lane = threadIdx.x & 31, vox = threadIdx.x >> 4, loc = threadIdx.x & 15;
  float2 m[2][32];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 32; ++c)
      m[r][c] = make_float2(0.01f * ((lane * 7 + c + r) % 13) - 0.06f, 0.003f * (c - lane - 16 * r));
  vs[0][vox][loc] = vs[0][vox][loc + 16] = make_float2(0.17f, 0.f);
  __syncwarp();
  float2 up[2] = {make_float2(0.17f, 0.f), make_float2(0.17f, 0.f)};
  float own = 1.f;
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    __syncwarp();
    u64 acc[2][2] = {}, acc2[2][2] = {};
    const float4* v4 = reinterpret_cast<const float4*>(vs[b][vox]);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const float4 x = v4[t];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        ffma2(acc[r][0], pk(m[r][2 * t].x, m[r][2 * t].x), pk(x.x, x.y));
        ffma2(acc2[r][0], pk(m[r][2 * t].y, m[r][2 * t].y), pk(x.y, x.x));
        ffma2(acc[r][1], pk(m[r][2 * t + 1].x, m[r][2 * t + 1].x), pk(x.z, x.w));
        ffma2(acc2[r][1], pk(m[r][2 * t + 1].y, m[r][2 * t + 1].y), pk(x.w, x.z));
      }
    }
    const float inv = rsqrtf(own);
    float x = 0.f;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float2 s = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float2 a = unpk(acc[r][k]), c = unpk(acc2[r][k]);
        s = make_float2(s.x + (a.x - c.x), s.y + (a.y + c.y));
      }
      up[r] = make_float2((0.9f * up[r].x + s.x) * inv, (0.9f * up[r].y + s.y) * inv);
      vs[b ^ 1][vox][loc + 16 * r] = up[r];
      x += up[r].x * up[r].x + up[r].y * up[r].y;
    }
    if (NRM == 1 || (it % NRM) == NRM - 1) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      own = x;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = up[0].x + up[1].y;
}

template <int NRM, int TH = 256, int MB = 1>
void run2(float* o, int sms, const char* name) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000, blocks = sms * MB, threads = TH;
  loop2<NRM, TH, MB><<<blocks, threads>>>(o, 10);
  float ms;
  cudaEventRecord(e0);
  loop2<NRM, TH, MB><<<blocks, threads>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 8.0 * 32 * 32 * iters * double(blocks) * (threads / 16);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc_per_iter = ms * 1e-3 * clk * 1e3 / iters * 16.0 / (TH / 16 * MB);
  printf("%-34s %.3f ms  %.1f TFLOP/s  %.0f cycles/iteration per SM (per 16 voxels/SM; FFMA2 floor 512)\n", name, ms,
         fl / ms / 1e9, cyc_per_iter);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, 1 << 24);
  for (int r = 0; r < 2; ++r) {
    run<0>(o, sms, "0 LDS.128 bcast + publish/norm");
    run<1>(o, sms, "1 v in registers + publish/norm");
    run<2>(o, sms, "2 LDS.64 bcast + publish/norm");
    run<3>(o, sms, "3 LDS.128 bcast, products only");
    run<4>(o, sms, "4 LDS.128 per-quarter copies");
    run<6>(o, sms, "6 LDS.128, norm every 4th");
    run<7>(o, sms, "7 v in regs (runtime) + publish/norm");
    run<8>(o, sms, "8 v in regs (runtime), products only");
    run2<1>(o, sms, "RPT2 LDS.128 + norm every it");
    run2<4>(o, sms, "RPT2 LDS.128 + norm every 4th");
    run2<1, 128, 3>(o, sms, "RPT2 128x3 + norm every it");
    run2<4, 128, 3>(o, sms, "RPT2 128x3 + norm every 4th");
    run2<1, 64, 6>(o, sms, "RPT2 64x6 + norm every it");
    run2<1, 192, 2>(o, sms, "RPT2 192x2 + norm every it");
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
