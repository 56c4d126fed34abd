// K4 — batched per-voxel power iteration (eigensolve.cpp:40-74) with the
// ESPIRiT map B = I - G/|Lambda| (spatial_gram.cpp:156-164) applied in
// registers, plus the per-voxel half of normalize_maps (maps.cpp:117-172)
// fused into the epilogue.
//
// Layout: G arrives as packed Hermitian planes [h][N] (h = Q(Q+1)/2; plane
// (p <= q) holds G(row p, col q) for every voxel, written by the K3
// expansion) as an fp32 hi/lo pair.  Blocks are persistent and walk voxel
// tiles; the next tile's h x VPB slab of hi planes is prefetched with
// cp.async (double buffer) while the current tile iterates.  Each voxel is
// unpacked into registers: matrix row p is held by TPR threads (TPR = 1 by
// default; 2 halves the registers per thread and is kept as a measured,
// slower alternative), QP = Q rounded up to a power of two (padding rows/cols
// are zero).
//
// Per iteration a thread does QP/TPR complex MACs (its row segment times v, v
// broadcast from shared memory as float4 pairs) and rescales its own
// component; v and the per-warp partials of ||u||^2 are double-buffered so an
// iteration costs one voxel-scoped barrier (named barrier when a voxel spans
// several warps, __syncwarp otherwise).  The matrix never leaves
// registers across the `iters` iterations, so the stage is FP32-bound:
// 8 Q^2 flops per voxel-iteration against one read of the planes.  The final
// Rayleigh quotient is evaluated in FP64 on hi + lo (lo streamed into the
// free tile buffer during the iterations), which keeps per-voxel eigenvalues
// at ~FP64 accuracy.
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

template <int QP, int TPR>
struct Layout {
  static constexpr int kThreads = 256;
  static constexpr int kCols = QP / TPR;         // matrix columns held per thread
  static constexpr int kTPV = QP * TPR;          // threads per voxel
  static constexpr int kVPB = kThreads / kTPV;   // voxels per block
  static constexpr int kWPV = kTPV > 32 ? kTPV / 32 : 1;  // warps per voxel
  static constexpr int kStride = QP + 2;         // float2 per v row (16-B aligned, bank-skewed)
};

// Sum over the voxel's rows of a per-row value replicated in its TPR threads.
template <int QP, int TPR, typename T>
__device__ __forceinline__ T row_sum(T x, T* red, int vox, int hc) {
  using L = Layout<QP, TPR>;
  if (TPR > 1 && hc != 0) x = T(0);
  if constexpr (L::kTPV <= 32) {
#pragma unroll
    for (int o = L::kTPV / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    const int w = (threadIdx.x % L::kTPV) >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[vox * L::kWPV + w] = x;
    __syncthreads();
    T s = T(0);
#pragma unroll
    for (int k = 0; k < L::kWPV; ++k) s += red[vox * L::kWPV + k];
    return s;
  }
}

// Combine the TPR partial row sums (adjacent lanes).
template <int TPR, typename T>
__device__ __forceinline__ T pair_sum(T x) {
  if constexpr (TPR == 2) x += __shfl_xor_sync(0xffffffffu, x, 1);
  return x;
}

template <int QP, int TPR>
__device__ __forceinline__ void voxel_sync() {
  if constexpr (Layout<QP, TPR>::kTPV <= 32)
    __syncwarp();
  else
    __syncthreads();
}

// Barrier over the threads of one voxel only: a warp-level sync for
// single-warp voxels, a named barrier (id 1 + vox) for multi-warp voxels.
template <int QP, int TPR>
__device__ __forceinline__ void voxel_bar(int vox) {
  constexpr int kTPV = Layout<QP, TPR>::kTPV;
  if constexpr (kTPV <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + vox), "n"(kTPV) : "memory");
  }
}

template <int QP, int TPR>
constexpr int min_blocks() {
  return (QP == 64 && TPR == 1) ? 1 : (QP == 32 && TPR == 2) ? 3 : 2;
}

__device__ __forceinline__ int pair_index(int p, int c, int Q) { return p * Q - p * (p - 1) / 2 + (c - p); }

template <int QP, int TPR>
__global__ void __launch_bounds__(256, min_blocks<QP, TPR>()) power_kernel(PowerArgs a) {
  using Lt = Layout<QP, TPR>;
  constexpr int VPB = Lt::kVPB, COLS = Lt::kCols, WPV = Lt::kWPV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Q = a.q;
  const int h = Q * (Q + 1) / 2;
  const int tile_elems = (h > QP ? h : QP) * VPB;
  float2* gbuf = reinterpret_cast<float2*>(smem_raw);                     // [2][tile_elems]
  float2* vs = gbuf + 2 * tile_elems;                                     // [2][VPB][kStride]
  double* redd = reinterpret_cast<double*>(vs + 2 * VPB * Lt::kStride);   // [VPB][kWPV]
  float* red = reinterpret_cast<float*>(redd + VPB * WPV);                // [VPB][kWPV]
  float* red2 = red + VPB * WPV;                                          // [2][VPB][kWPV]

  const int vox = threadIdx.x / Lt::kTPV;
  const int local = threadIdx.x % Lt::kTPV;
  const int p = local / TPR;
  const int hc = local % TPR;
  const int c0 = hc * COLS;
  const i64 tiles = (a.n + VPB - 1) / VPB;

  auto load_tile = [&](i64 t, float2* dst, const float2* src) {
    const i64 jj0 = t * VPB;
    for (int e = threadIdx.x; e < h * VPB; e += blockDim.x) {
      const int pair = e / VPB, v = e % VPB;
      const bool ok = jj0 + v < a.n;
      cp_async8(dst + e, src + (ok ? i64(pair) * a.n + jj0 + v : 0), ok ? 8 : 0);
    }
    cp_async_commit();
  };

  i64 tile = blockIdx.x;
  int buf = 0;
  if (tile < tiles) load_tile(tile, gbuf, a.planes);
  for (; tile < tiles; tile += gridDim.x, buf ^= 1) {
    const i64 next = tile + gridDim.x;
    if (next < tiles) {
      load_tile(next, gbuf + (buf ^ 1) * tile_elems, a.planes);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    float2* gs = gbuf + buf * tile_elems;
    const i64 j0 = tile * VPB;
    const i64 j = j0 + vox;
    const bool live = j < a.n;

    // Unpack this thread's row segment (columns c0 .. c0 + COLS).
    float2 m[COLS];
#pragma unroll
    for (int c = 0; c < COLS; ++c) {
      const int cc = c0 + c;
      float2 val = make_float2(0.f, 0.f);
      if (p < Q && cc < Q) {
        if (p <= cc) {
          val = gs[pair_index(p, cc, Q) * VPB + vox];
        } else {
          const float2 t = gs[pair_index(cc, p, Q) * VPB + vox];
          val = make_float2(t.x, -t.y);
        }
        if (p == cc) val.y = 0.f;  // spatial_gram.cpp:140-146
      }
      m[c] = val;
    }
    // The tile buffer is free once every row is in registers: stream the lo
    // residual planes into it while the iterations run.
    if (a.planes_lo != nullptr) {
      __syncthreads();
      load_tile(tile, gs, a.planes_lo);
    }
    // M[p][0] for the e_0 restart (held by the hc == 0 thread of the row)
    float2 mp0 = m[0];
    if constexpr (TPR == 2) {
      mp0.x = __shfl_sync(0xffffffffu, m[0].x, threadIdx.x & ~1);
      mp0.y = __shfl_sync(0xffffffffu, m[0].y, threadIdx.x & ~1);
    }

    // v is double-buffered in shared memory (vb[0], vb[1]) together with the
    // per-warp partials of ||u||^2, so an iteration needs one voxel barrier.
    auto vb = [&](int b) { return vs + (b * VPB + vox) * Lt::kStride; };
    const float init = rsqrtf(float(Q));
    float2 vp = (p < Q) ? make_float2(init, 0.f) : make_float2(0.f, 0.f);
    if (hc == 0) vb(0)[p] = vp;
    bool done = false;
    voxel_sync<QP, TPR>();

    // Publish u into buffer b and its squared norm: returned directly for a
    // single-warp voxel, left as per-warp partials in red2[b] otherwise.
    auto publish = [&](float2 u, int b) -> float {
      if (hc == 0) vb(b)[p] = u;
      float x = (hc == 0) ? u.x * u.x + u.y * u.y : 0.f;
      if constexpr (Lt::kTPV <= 32) {
#pragma unroll
        for (int o = Lt::kTPV / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        return x;
      } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0) red2[(b * VPB + vox) * WPV + ((threadIdx.x % Lt::kTPV) >> 5)] = x;
        return 0.f;
      }
    };
    auto published_norm = [&](float own, int b) -> float {
      if constexpr (Lt::kTPV <= 32) {
        return own;
      } else {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < WPV; ++k) s += red2[(b * VPB + vox) * WPV + k];
        return s;
      }
    };

    // M v: v is staged into registers in chunks of 8 complex values (4
    // LDS.128 in flight) feeding 4 independent accumulator pairs.
    auto matvec = [&](const float2* v, float2& out) {
      const float4* v4 = reinterpret_cast<const float4*>(v + c0);
      float2 acc[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = make_float2(0.f, 0.f);
      constexpr int kChunk = COLS < 8 ? COLS : 8;
#pragma unroll
      for (int cb = 0; cb < COLS; cb += kChunk) {
        float4 vv[kChunk / 2];
#pragma unroll
        for (int t = 0; t < kChunk / 2; ++t) vv[t] = v4[cb / 2 + t];
#pragma unroll
        for (int t = 0; t < kChunk / 2; ++t) {
          cmac(acc[(2 * t) & 3], m[cb + 2 * t], make_float2(vv[t].x, vv[t].y));
          cmac(acc[(2 * t + 1) & 3], m[cb + 2 * t + 1], make_float2(vv[t].z, vv[t].w));
        }
      }
      out = make_float2(pair_sum<TPR>((acc[0].x + acc[1].x) + (acc[2].x + acc[3].x)),
                        pair_sum<TPR>((acc[0].y + acc[1].y) + (acc[2].y + acc[3].y)));
    };

    // Iteration 0, peeled: an annihilated all-ones start restarts from e_0
    // (eigensolve.cpp:56-63); the candidate is formed uniformly and selected.
    if (a.iters > 0) {
      float2 mv;
      matvec(vb(0), mv);
      float2 w = make_float2(a.alpha * vp.x + a.beta * mv.x, a.alpha * vp.y + a.beta * mv.y);
      float n2 = row_sum<QP, TPR>(w.x * w.x + w.y * w.y, red, vox, hc);
      const float2 v0 = (p == 0) ? make_float2(1.f, 0.f) : make_float2(0.f, 0.f);
      const float2 w0 = make_float2(a.alpha * v0.x + a.beta * mp0.x, a.alpha * v0.y + a.beta * mp0.y);
      const float n20 = row_sum<QP, TPR>(w0.x * w0.x + w0.y * w0.y, red, vox, hc);
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
    }
    // Iterations 1..iters-1, software-pipelined on the unnormalised iterate
    // u_k: ||u_k||^2 travels with u_k (published together), w = B(u_k/||u_k||)
    // = B v_k.  ||B v_k|| is known one iteration later, so the break test of
    // iteration k (||B v_k|| < 1e-14 -> keep v_k) is evaluated then, with v_k
    // in vprev.  Iteration k reads buffer k&1 and writes buffer (k+1)&1; the
    // barrier at the top of iteration k+1 orders both (every read of (k+1)&1
    // from iteration k-1 precedes the barrier at the top of iteration k).
    float2 up = vp, vprev = vp;
    float own = 0.f;
    if (a.iters > 1) own = publish(up, 1);  // iteration 0 read only vb[0]
    for (int it = 1; it < a.iters; ++it) {
      const int b = it & 1;
      voxel_bar<QP, TPR>(vox);
      const float n2 = published_norm(own, b);
      float2 mv;
      matvec(vb(b), mv);
      if (it > 1 && n2 < 1e-28f && !done) done = true;
      const float inv = rsqrtf(n2);
      if (!done) {
        vprev = make_float2(up.x * inv, up.y * inv);
        up = make_float2((a.alpha * up.x + a.beta * mv.x) * inv, (a.alpha * up.y + a.beta * mv.y) * inv);
      }
      own = publish(up, b ^ 1);
    }
    int fb = 0;  // buffer that receives the final v
    if (a.iters > 1) {
      voxel_bar<QP, TPR>(vox);
      const float n2 = published_norm(own, a.iters & 1);
      if (!done && !(n2 < 1e-28f)) {
        const float inv = rsqrtf(n2);
        vp = make_float2(up.x * inv, up.y * inv);
      } else {
        vp = vprev;
      }
      fb = (a.iters & 1) ^ 1;  // last read by iteration iters-1, before the barrier above
    }
    voxel_sync<QP, TPR>();
    float2* myv = vb(fb);
    if (hc == 0) myv[p] = vp;
    voxel_sync<QP, TPR>();

    // Rayleigh quotient in FP64 on M = hi + lo: mv = Re(v^H M v) (the FP32
    // iterate v enters only to second order); value = Re(v^H B v).
    double mrx = 0.0, mry = 0.0;
#pragma unroll
    for (int c = 0; c < COLS; ++c) {
      const float2 vc = myv[c0 + c];
      mrx = fma(double(m[c].x), double(vc.x), mrx);
      mrx = fma(-double(m[c].y), double(vc.y), mrx);
      mry = fma(double(m[c].x), double(vc.y), mry);
      mry = fma(double(m[c].y), double(vc.x), mry);
    }
    if (a.planes_lo != nullptr) {
      cp_async_wait<0>();
      __syncthreads();
      if (p < Q) {
        for (int c = c0; c < c0 + COLS && c < Q; ++c) {
          float2 lv;
          if (p <= c) {
            lv = gs[pair_index(p, c, Q) * VPB + vox];
          } else {
            const float2 t = gs[pair_index(c, p, Q) * VPB + vox];
            lv = make_float2(t.x, -t.y);
          }
          if (p == c) lv.y = 0.f;
          const float2 vc = myv[c];
          mrx += double(lv.x) * vc.x - double(lv.y) * vc.y;
          mry += double(lv.x) * vc.y + double(lv.y) * vc.x;
        }
      }
    }
    mrx = pair_sum<TPR>(mrx);
    mry = pair_sum<TPR>(mry);
    const double mv = row_sum<QP, TPR>(double(vp.x) * mrx + double(vp.y) * mry, redd, vox, hc);
    const float vn2 = row_sum<QP, TPR>(vp.x * vp.x + vp.y * vp.y, red, vox, hc);

    if (a.recon != nullptr) {
      // normalize_maps, per voxel: SoS (maps.cpp:117-128) then phase reference
      // against the apodised coil-combined calibration recon (maps.cpp:163-172).
      if (vn2 > 0.f) {
        const float inv = 1.0f / sqrtf(vn2);
        vp.x *= inv;
        vp.y *= inv;
      } else if (p == 0 && hc == 0 && live && a.zeroed) {
        atomicAdd(a.zeroed, 1ull);
      }
      float2 r = make_float2(0.f, 0.f);
      if (p < Q && live) r = a.recon[i64(p) * a.n + j];
      const float ux = row_sum<QP, TPR>(vp.x * r.x + vp.y * r.y, red, vox, hc);  // conj(v) * r
      const float uy = row_sum<QP, TPR>(vp.x * r.y - vp.y * r.x, red, vox, hc);
      const float mag = sqrtf(ux * ux + uy * uy);
      if (mag > 0.f) {
        const float cx = ux / mag, cy = uy / mag;
        vp = make_float2(vp.x * cx - vp.y * cy, vp.x * cy + vp.y * cx);
      }
    }

    // Stage maps for channel-major coalesced stores: reuse the plane tile.
    __syncthreads();
    float2* ms = gs;  // [QP][VPB]
    if (hc == 0) ms[p * VPB + vox] = vp;
    __syncthreads();
    for (int e = threadIdx.x; e < Q * VPB; e += blockDim.x) {
      const int c = e / VPB, v = e % VPB;
      if (j0 + v < a.n) a.maps[i64(c) * a.n + j0 + v] = ms[c * VPB + v];
    }
    if (p == 0 && hc == 0 && live) {
      const float lam = float(mv * double(a.lam_scale));
      if (a.lambda) a.lambda[j] = lam;
      if (a.value) a.value[j] = float(double(a.alpha) * vn2 + double(a.beta) * mv);
      if (a.mask) a.mask[j] = lam < a.mask_threshold ? 1 : 0;
    }
    __syncthreads();  // the staging buffer is the prefetch target two tiles on
  }
}

template <int QP, int TPR>
void launch(sk_ctx* ctx, const PowerArgs& a) {
  using Lt = Layout<QP, TPR>;
  const int h = a.q * (a.q + 1) / 2;
  const size_t tile = size_t(std::max(h, QP)) * Lt::kVPB * sizeof(float2);
  const size_t smem = 2 * tile + 2 * size_t(Lt::kVPB) * Lt::kStride * sizeof(float2) +
                      size_t(Lt::kVPB) * Lt::kWPV * (sizeof(double) + 3 * sizeof(float));
  SKB_CUDA(cudaFuncSetAttribute(power_kernel<QP, TPR>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  SKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, power_kernel<QP, TPR>, Lt::kThreads, smem));
  const i64 tiles = (a.n + Lt::kVPB - 1) / Lt::kVPB;
  const i64 blocks = std::min<i64>(tiles, i64(std::max(per_sm, 1)) * ctx->sm_count);
  power_kernel<QP, TPR><<<unsigned(blocks), Lt::kThreads, smem, ctx->stream>>>(a);
  ++ctx->launches;
  SKB_LAUNCH("power_kernel");
}

}  // namespace

void power_iteration(sk_ctx* ctx, const PowerArgs& a) {
  if (a.n <= 0) return;
  // Row split (threads per matrix row) per size class; SKB_POWER_TPR32 /
  // SKB_POWER_TPR64 select the alternative layout for experiments.
  static const int tpr32 = [] {
    const char* v = std::getenv("SKB_POWER_TPR32");
    return v && std::atoi(v) == 2 ? 2 : 1;
  }();
  static const int tpr64 = [] {
    const char* v = std::getenv("SKB_POWER_TPR64");
    return v && std::atoi(v) == 2 ? 2 : 1;
  }();
  if (a.q <= 4)
    launch<4, 1>(ctx, a);
  else if (a.q <= 8)
    launch<8, 1>(ctx, a);
  else if (a.q <= 16)
    launch<16, 1>(ctx, a);
  else if (a.q <= 32)
    tpr32 == 2 ? launch<32, 2>(ctx, a) : launch<32, 1>(ctx, a);
  else if (a.q <= 64)
    tpr64 == 2 ? launch<64, 2>(ctx, a) : launch<64, 1>(ctx, a);
  else
    fail(9, "eig_power_field: more than 64 channels is outside the B200 path");
}

}  // namespace skb
