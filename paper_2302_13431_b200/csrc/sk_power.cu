// K4 — batched per-voxel power iteration (eigensolve.cpp:40-74) with the
// ESPIRiT map B = I - G/|Lambda| (spatial_gram.cpp:156-164) applied in
// registers, plus the per-voxel half of normalize_maps (maps.cpp:117-172)
// fused into the epilogue.
//
// Layout: G arrives as packed Hermitian planes [h][N] (h = Q(Q+1)/2; plane
// (p <= q) holds G(row p, col q) for every voxel, written by the K3
// expansion).  A block owns VPB consecutive voxels and stages their h x VPB
// tile in shared memory with VPB-wide coalesced row reads; each voxel is then
// unpacked into registers, one matrix ROW per thread (QP threads per voxel,
// QP = Q rounded up to a power of two, padding rows/cols are zero).
//
// Per iteration a thread does QP complex MACs (its row times v, v broadcast
// from shared memory as float4 pairs), the group reduces ||w||^2 with
// shuffles, and every thread rescales its own component.  The matrix never
// leaves registers across the `iters` iterations, so the stage is FP32-bound:
// 8 Q^2 flops per voxel-iteration against one 8*h-byte read per voxel.
//
// Exactly the reference's control flow: fixed iteration count; at it == 0 an
// annihilated all-ones start restarts from e_0; a norm below 1e-14 freezes v.
#include "sk_internal.h"

namespace skb {

namespace {

__device__ __forceinline__ void cmac(float2& acc, float2 m, float2 x) {
  acc.x = fmaf(m.x, x.x, acc.x);
  acc.x = fmaf(-m.y, x.y, acc.x);
  acc.y = fmaf(m.x, x.y, acc.y);
  acc.y = fmaf(m.y, x.x, acc.y);
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int QP>
struct Group {
  static constexpr int kThreads = 256;
  static constexpr int kVPB = kThreads / QP;  // voxels per block
  static constexpr int kStride = QP + 2;      // float2 per v row (16-B aligned, bank-skewed)
};

// Sum over the QP threads of one voxel.  QP <= 32: xor shuffles inside the
// aligned lane group.  QP == 64: two warps, combined through shared memory
// (uniform __syncthreads: every thread of the block calls this).
template <int QP>
__device__ __forceinline__ float group_sum(float x, float* red, int vox, int half) {
  if constexpr (QP <= 32) {
#pragma unroll
    for (int o = QP / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[vox * 2 + half] = x;
    __syncthreads();
    return red[vox * 2] + red[vox * 2 + 1];
  }
}

template <int QP>
__device__ __forceinline__ double group_sum_d(double x, double* red, int vox, int half) {
  if constexpr (QP <= 32) {
#pragma unroll
    for (int o = QP / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[vox * 2 + half] = x;
    __syncthreads();
    return red[vox * 2] + red[vox * 2 + 1];
  }
}

template <int QP>
__device__ __forceinline__ void group_sync() {
  if constexpr (QP <= 32)
    __syncwarp();
  else
    __syncthreads();
}

template <int QP>
__global__ void __launch_bounds__(256, (QP <= 32 ? 2 : 1)) power_kernel(PowerArgs a) {
  using G = Group<QP>;
  constexpr int VPB = G::kVPB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Q = a.q;
  const int h = Q * (Q + 1) / 2;
  // Persistent: the block walks voxel tiles with a double-buffered cp.async
  // prefetch of the next tile's h x VPB plane slab (VPB-wide coalesced rows).
  const int tile_elems = (h > QP ? h : QP) * VPB;
  float2* gbuf = reinterpret_cast<float2*>(smem_raw);             // [2][tile_elems]
  float2* vs = gbuf + 2 * tile_elems;                             // [VPB][kStride]
  double* redd = reinterpret_cast<double*>(vs + VPB * G::kStride);  // [VPB][2]
  float* red = reinterpret_cast<float*>(redd + VPB * 2);           // [VPB][2]

  const int vox = threadIdx.x / QP;
  const int p = threadIdx.x % QP;
  const int half = (threadIdx.x / 32) & 1;
  const i64 tiles = (a.n + VPB - 1) / VPB;

  auto load_tile = [&](i64 t, float2* dst) {
    const i64 jj0 = t * VPB;
    for (int e = threadIdx.x; e < h * VPB; e += blockDim.x) {
      const int pair = e / VPB, v = e % VPB;
      const bool ok = jj0 + v < a.n;
      cp_async8(dst + e, a.planes + (ok ? i64(pair) * a.n + jj0 + v : 0), ok ? 8 : 0);
    }
    cp_async_commit();
  };

  i64 tile = blockIdx.x;
  int buf = 0;
  if (tile < tiles) load_tile(tile, gbuf);
  for (; tile < tiles; tile += gridDim.x, buf ^= 1) {
  const i64 next = tile + gridDim.x;
  if (next < tiles) {
    load_tile(next, gbuf + (buf ^ 1) * tile_elems);
    cp_async_wait<1>();
  } else {
    cp_async_wait<0>();
  }
  __syncthreads();
  float2* gs = gbuf + buf * tile_elems;
  const i64 j0 = tile * VPB;
  const i64 j = j0 + vox;
  const bool live = j < a.n;

  // Unpack this thread's matrix row.
  float2 m[QP];
#pragma unroll
  for (int c = 0; c < QP; ++c) {
    float2 val = make_float2(0.f, 0.f);
    if (p < Q && c < Q) {
      if (p <= c) {
        val = gs[(p * Q - p * (p - 1) / 2 + (c - p)) * VPB + vox];
      } else {
        const float2 t = gs[(c * Q - c * (c - 1) / 2 + (p - c)) * VPB + vox];
        val = make_float2(t.x, -t.y);
      }
      if (p == c) val.y = 0.f;  // spatial_gram.cpp:140-146
    }
    m[c] = val;
  }
  // The tile buffer is free once every row is in registers: stream the lo
  // residual planes into it while the iterations run (hi/lo split, sk_expand.cu).
  if (a.planes_lo != nullptr) {
    __syncthreads();
    for (int e = threadIdx.x; e < h * VPB; e += blockDim.x) {
      const int pair = e / VPB, v = e % VPB;
      const bool ok = j0 + v < a.n;
      cp_async8(gs + e, a.planes_lo + (ok ? i64(pair) * a.n + j0 + v : 0), ok ? 8 : 0);
    }
    cp_async_commit();
  }

  float2* myv = vs + vox * G::kStride;
  const float init = rsqrtf(float(Q));
  float2 vp = (p < Q) ? make_float2(init, 0.f) : make_float2(0.f, 0.f);
  myv[p] = vp;
  bool done = false;
  group_sync<QP>();

  // M v with v broadcast from shared memory: v is staged into registers in
  // chunks of 8 complex values (4 LDS.128 in flight) feeding 4 independent
  // accumulator pairs, so the FMA pipe is not serialised on LDS latency.
  auto matvec = [&](float2& out) {
    const float4* v4 = reinterpret_cast<const float4*>(myv);
    float2 acc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] = make_float2(0.f, 0.f);
    constexpr int kChunk = QP < 8 ? QP : 8;
#pragma unroll
    for (int c0 = 0; c0 < QP; c0 += kChunk) {
      float4 vv[kChunk / 2];
#pragma unroll
      for (int t = 0; t < kChunk / 2; ++t) vv[t] = v4[c0 / 2 + t];
#pragma unroll
      for (int t = 0; t < kChunk / 2; ++t) {
        cmac(acc[(2 * t) & 3], m[c0 + 2 * t], make_float2(vv[t].x, vv[t].y));
        cmac(acc[(2 * t + 1) & 3], m[c0 + 2 * t + 1], make_float2(vv[t].z, vv[t].w));
      }
    }
    out = make_float2((acc[0].x + acc[1].x) + (acc[2].x + acc[3].x), (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y));
  };

  // Iteration 0, peeled: an annihilated all-ones start restarts from e_0
  // (eigensolve.cpp:56-63).  The e_0 candidate is formed by every thread (the
  // reductions stay warp/block-uniform) and selected per voxel.
  if (a.iters > 0) {
    float2 mv;
    matvec(mv);
    float2 w = make_float2(a.alpha * vp.x + a.beta * mv.x, a.alpha * vp.y + a.beta * mv.y);
    float n2 = group_sum<QP>(w.x * w.x + w.y * w.y, red, vox, half);
    const float2 v0 = (p == 0) ? make_float2(1.f, 0.f) : make_float2(0.f, 0.f);
    const float2 w0 = make_float2(a.alpha * v0.x + a.beta * m[0].x, a.alpha * v0.y + a.beta * m[0].y);
    const float n20 = group_sum<QP>(w0.x * w0.x + w0.y * w0.y, red, vox, half);
    if (n2 < 1e-28f) {  // ||B v|| < 1e-14
      vp = v0;
      w = w0;
      n2 = n20;
    }
    if (n2 < 1e-28f) done = true;  // B ~ 0 here: keep the current v
    if (!done) {
      const float inv = rsqrtf(n2);
      vp = make_float2(w.x * inv, w.y * inv);
    }
    group_sync<QP>();
    myv[p] = vp;
    group_sync<QP>();
  }
  // Iterations 1..iters-1, software-pipelined: the shared vector holds the
  // UNNORMALISED iterate u_k (u_1 = v_1).  The reduction ||u_k||^2 runs
  // alongside the mat-vec M u_k (independent instructions), and the scale is
  // applied afterwards: w = B (u_k / ||u_k||) = B v_k, exactly the reference
  // step.  ||B v_k|| is only known one iteration later, so the break test of
  // iteration k (||B v_k|| < 1e-14 -> keep v_k) is evaluated then, with v_k
  // kept in `vprev`.
  float2 up = vp;          // u_k
  float2 vprev = vp;       // v_k (normalised)
  for (int it = 1; it < a.iters; ++it) {
    const float n2 = group_sum<QP>(up.x * up.x + up.y * up.y, red, vox, half);  // ||u_k||^2 = ||B v_{k-1}||^2
    float2 mv;
    matvec(mv);                                                                 // M u_k
    if (it > 1 && n2 < 1e-28f && !done) {  // iteration it-1 should have stopped: keep v_{it-1}
      done = true;
    }
    const float inv = rsqrtf(n2);
    if (!done) {
      vprev = make_float2(up.x * inv, up.y * inv);  // v_k
      up = make_float2((a.alpha * up.x + a.beta * mv.x) * inv, (a.alpha * up.y + a.beta * mv.y) * inv);
    }
    group_sync<QP>();
    myv[p] = up;
    group_sync<QP>();
  }
  if (a.iters > 1) {
    const float n2 = group_sum<QP>(up.x * up.x + up.y * up.y, red, vox, half);  // ||B v_{iters-1}||^2
    if (!done) {
      if (n2 < 1e-28f) {
        vp = vprev;
      } else {
        const float inv = rsqrtf(n2);
        vp = make_float2(up.x * inv, up.y * inv);
      }
    } else {
      vp = vprev;
    }
    group_sync<QP>();
    myv[p] = vp;
    group_sync<QP>();
  }

  // Rayleigh quotient in FP64 on M = hi + lo: mv = Re(v^H M v) (the FP32
  // iterate v enters only to second order); value = Re(v^H B v).
  double mrx = 0.0, mry = 0.0;
#pragma unroll
  for (int c = 0; c < QP; ++c) {
    const float2 vc = myv[c];
    mrx = fma(double(m[c].x), double(vc.x), mrx);
    mrx = fma(-double(m[c].y), double(vc.y), mrx);
    mry = fma(double(m[c].x), double(vc.y), mry);
    mry = fma(double(m[c].y), double(vc.x), mry);
  }
  if (a.planes_lo != nullptr) {
    cp_async_wait<0>();
    __syncthreads();
    if (p < Q) {
      for (int c = 0; c < Q; ++c) {
        float2 lv;
        if (p <= c) {
          lv = gs[(p * Q - p * (p - 1) / 2 + (c - p)) * VPB + vox];
        } else {
          const float2 t = gs[(c * Q - c * (c - 1) / 2 + (p - c)) * VPB + vox];
          lv = make_float2(t.x, -t.y);
        }
        if (p == c) lv.y = 0.f;
        const float2 vc = myv[c];
        mrx += double(lv.x) * vc.x - double(lv.y) * vc.y;
        mry += double(lv.x) * vc.y + double(lv.y) * vc.x;
      }
    }
  }
  const double mv = group_sum_d<QP>(double(vp.x) * mrx + double(vp.y) * mry, redd, vox, half);
  const float vn2 = group_sum<QP>(vp.x * vp.x + vp.y * vp.y, red, vox, half);

  if (a.recon != nullptr) {
    // normalize_maps, per voxel: SoS (maps.cpp:117-128) then phase reference
    // against the apodised coil-combined calibration recon (maps.cpp:163-172).
    if (vn2 > 0.f) {
      const float inv = 1.0f / sqrtf(vn2);
      vp.x *= inv;
      vp.y *= inv;
    } else if (p == 0 && live && a.zeroed) {
      atomicAdd(a.zeroed, 1ull);
    }
    float2 r = make_float2(0.f, 0.f);
    if (p < Q && live) r = a.recon[i64(p) * a.n + j];
    const float ux = group_sum<QP>(vp.x * r.x + vp.y * r.y, red, vox, half);  // conj(v) * r
    const float uy = group_sum<QP>(vp.x * r.y - vp.y * r.x, red, vox, half);
    const float mag = sqrtf(ux * ux + uy * uy);
    if (mag > 0.f) {
      const float cx = ux / mag, cy = uy / mag;
      vp = make_float2(vp.x * cx - vp.y * cy, vp.x * cy + vp.y * cx);
    }
  }

  // Stage maps for channel-major coalesced stores: reuse the plane tile.
  __syncthreads();
  float2* ms = gs;  // [QP][VPB]
  ms[p * VPB + vox] = vp;
  __syncthreads();
  for (int e = threadIdx.x; e < Q * VPB; e += blockDim.x) {
    const int c = e / VPB, v = e % VPB;
    if (j0 + v < a.n) a.maps[i64(c) * a.n + j0 + v] = ms[c * VPB + v];
  }
  if (p == 0 && live) {
    const float lam = float(mv * double(a.lam_scale));
    if (a.lambda) a.lambda[j] = lam;
    if (a.value) a.value[j] = float(double(a.alpha) * vn2 + double(a.beta) * mv);
    if (a.mask) a.mask[j] = lam < a.mask_threshold ? 1 : 0;
  }
  __syncthreads();  // the staging buffer is the prefetch target two tiles on
  }
}

template <int QP>
void launch(sk_ctx* ctx, const PowerArgs& a) {
  using G = Group<QP>;
  const int h = a.q * (a.q + 1) / 2;
  const size_t tile = size_t(std::max(h, QP)) * G::kVPB * sizeof(float2);
  const size_t smem = 2 * tile + size_t(G::kVPB) * G::kStride * sizeof(float2) +
                      size_t(G::kVPB) * 2 * (sizeof(double) + sizeof(float));
  SKB_CUDA(cudaFuncSetAttribute(power_kernel<QP>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  SKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, power_kernel<QP>, G::kThreads, smem));
  const i64 tiles = (a.n + G::kVPB - 1) / G::kVPB;
  const i64 blocks = std::min<i64>(tiles, i64(std::max(per_sm, 1)) * ctx->sm_count);
  power_kernel<QP><<<unsigned(blocks), G::kThreads, smem, ctx->stream>>>(a);
  ++ctx->launches;
  SKB_LAUNCH("power_kernel");
}

}  // namespace

void power_iteration(sk_ctx* ctx, const PowerArgs& a) {
  if (a.n <= 0) return;
  if (a.q <= 4)
    launch<4>(ctx, a);
  else if (a.q <= 8)
    launch<8>(ctx, a);
  else if (a.q <= 16)
    launch<16>(ctx, a);
  else if (a.q <= 32)
    launch<32>(ctx, a);
  else if (a.q <= 64)
    launch<64>(ctx, a);
  else
    fail(9, "eig_power_field: more than 64 channels is outside the B200 path");
}

}  // namespace skb
