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
__device__ __forceinline__ void group_sync() {
  if constexpr (QP <= 32)
    __syncwarp();
  else
    __syncthreads();
}

template <int QP>
__global__ void __launch_bounds__(256) power_kernel(PowerArgs a) {
  using G = Group<QP>;
  constexpr int VPB = G::kVPB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Q = a.q;
  const int h = Q * (Q + 1) / 2;
  float2* gs = reinterpret_cast<float2*>(smem_raw);       // [h][VPB]
  float2* vs = gs + i64(h) * VPB;                          // [VPB][kStride]
  float* red = reinterpret_cast<float*>(vs + VPB * G::kStride);  // [VPB][2]

  const int vox = threadIdx.x / QP;
  const int p = threadIdx.x % QP;
  const int half = (threadIdx.x / 32) & 1;
  const i64 j0 = i64(blockIdx.x) * VPB;
  const i64 j = j0 + vox;
  const bool live = j < a.n;

  // Stage the block's tile of packed planes (VPB-wide coalesced rows).
  for (int e = threadIdx.x; e < h * VPB; e += blockDim.x) {
    const int pair = e / VPB, v = e % VPB;
    gs[e] = (j0 + v < a.n) ? a.planes[i64(pair) * a.n + j0 + v] : make_float2(0.f, 0.f);
  }
  __syncthreads();

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

  float2* myv = vs + vox * G::kStride;
  const float init = rsqrtf(float(Q));
  float2 vp = (p < Q) ? make_float2(init, 0.f) : make_float2(0.f, 0.f);
  myv[p] = vp;
  bool done = false;
  group_sync<QP>();

  auto matvec = [&](float2& out) {
    const float4* v4 = reinterpret_cast<const float4*>(myv);
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < QP; c += 2) {
      const float4 vv = v4[c / 2];
      cmac(acc0, m[c], make_float2(vv.x, vv.y));
      cmac(acc1, m[c + 1], make_float2(vv.z, vv.w));
    }
    out = make_float2(acc0.x + acc1.x, acc0.y + acc1.y);
  };

  for (int it = 0; it < a.iters; ++it) {
    float2 mv;
    matvec(mv);
    float2 w = make_float2(a.alpha * vp.x + a.beta * mv.x, a.alpha * vp.y + a.beta * mv.y);
    float nrm = sqrtf(group_sum<QP>(w.x * w.x + w.y * w.y, red, vox, half));
    if (it == 0) {
      // All-ones start annihilated: restart from e_0 (eigensolve.cpp:58-63).
      // The e_0 candidate is formed by every thread (the reductions must stay
      // warp/block-uniform) and selected per voxel.
      const float2 v0 = (p == 0) ? make_float2(1.f, 0.f) : make_float2(0.f, 0.f);
      const float2 w0 = make_float2(a.alpha * v0.x + a.beta * m[0].x, a.alpha * v0.y + a.beta * m[0].y);
      const float nrm0 = sqrtf(group_sum<QP>(w0.x * w0.x + w0.y * w0.y, red, vox, half));
      if (nrm < 1e-14f) {
        vp = v0;
        w = w0;
        nrm = nrm0;
      }
    }
    if (nrm < 1e-14f) done = true;  // B ~ 0 here: keep the current v
    if (!done) {
      const float inv = 1.0f / nrm;
      vp = make_float2(w.x * inv, w.y * inv);
    }
    group_sync<QP>();
    myv[p] = vp;
    group_sync<QP>();
  }

  // Rayleigh quotient: mv = Re(v^H M v); value = Re(v^H B v).
  float2 mvv;
  matvec(mvv);
  const float mv = group_sum<QP>(vp.x * mvv.x + vp.y * mvv.y, red, vox, half);
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
    const float lam = mv * a.lam_scale;
    if (a.lambda) a.lambda[j] = lam;
    if (a.value) a.value[j] = a.alpha * vn2 + a.beta * mv;
    if (a.mask) a.mask[j] = lam < a.mask_threshold ? 1 : 0;
  }
}

template <int QP>
void launch(sk_ctx* ctx, const PowerArgs& a) {
  using G = Group<QP>;
  const int h = a.q * (a.q + 1) / 2;
  const size_t tile = size_t(h) * G::kVPB * sizeof(float2);
  const size_t smem = std::max(tile, size_t(QP) * G::kVPB * sizeof(float2)) +
                      size_t(G::kVPB) * G::kStride * sizeof(float2) + size_t(G::kVPB) * 2 * sizeof(float);
  SKB_CUDA(cudaFuncSetAttribute(power_kernel<QP>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const i64 blocks = (a.n + G::kVPB - 1) / G::kVPB;
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
