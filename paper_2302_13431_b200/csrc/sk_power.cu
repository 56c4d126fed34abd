// K4 — batched per-voxel power iteration (eigensolve.cpp:40-74) with the
// ESPIRiT map B = I - G/|Lambda| (spatial_gram.cpp:156-164) applied in
// registers, plus the per-voxel half of normalize_maps (maps.cpp:117-172)
// fused into the epilogue.
//
// Layout: G arrives as packed Hermitian planes [h][N] (h = Q(Q+1)/2; plane
// (p <= q) holds G(row p, col q) for every voxel, written by the K3
// expansion) as an fp32 hi plane plus a bf16 residual lo plane.  Blocks are persistent and walk voxel
// tiles; the next tile's h x VPB slab of hi planes is prefetched by TMA
// (cp.async.bulk.tensor boxes on an mbarrier, double buffer; swizzled 32/64 B
// rows so that the unpack and the epilogue reads spread over the banks; an
// 8-byte cp.async fallback when TMA cannot address the planes) while the
// current tile iterates.  Each voxel is unpacked into registers: a thread
// holds RPT full matrix rows (p = local + r * QP/RPT), QP = Q rounded up to a
// power of two (padding rows/cols are zero).
//
// Per iteration a thread loads v once from shared memory (float4 broadcast
// pairs) and does RPT * QP complex MACs with it as FFMA2 pairs, then rescales
// its own components; v and the per-warp partials of ||u||^2 are
// double-buffered so an iteration costs one voxel-scoped barrier (named
// barrier when a voxel spans several warps, __syncwarp otherwise).  With one
// row per thread the v broadcasts need as many shared-memory wavefronts as
// the FFMA2 pipe needs cycles (tools/k4_loop_micro.cu).  The
// matrix never leaves registers across the `iters` iterations: 8 Q^2 flops
// per voxel-iteration against one read of the planes.  The final Rayleigh
// quotient is evaluated in FP64 on hi + lo (lo streamed into its own tile
// buffer during the iterations), which keeps per-voxel eigenvalues at ~FP64
// accuracy; on full-resolution grids an FP32 quotient from the
// registers is kept for lambda >= rq32_min (||G/|Lambda| || <= 1).  A voxel
// range of a larger grid (PowerArgs::ld) lets the pipeline run K4 in chunks.
//
// Exactly the reference's control flow: fixed iteration count; at it == 0 an
// annihilated all-ones start restarts from e_0; a norm below 1e-14 freezes v.
#include "sk_internal.h"

#include <cuda.h>
#include <cudaTypedefs.h>

namespace skb {

namespace {


// Packed FP32x2 FMA (FFMA2, sm_100): same FMA-pipe rate as FFMA at half the
// issue slots.  ptxas folds pk(s, s) into a scalar-broadcast operand and
// pk(hi, lo) of a register pair into a swapped (LO_HI) operand.
using u64 = unsigned long long;
__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void ffma2(u64& d, u64 a, u64 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ float2 unpk(u64 x) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(x));
  return r;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// TMA (cp.async.bulk.tensor) + mbarrier helpers.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// Tile geometry of the TMA path: nb boxes of hb plane rows x VPB voxels.
// With a tile row of 32/64/128 B the boxes land swizzled (TMA SWIZZLE_32B/
// 64B/128B: the 16-B chunk index within each row is XORed with address bits
// 7..): the unpack and the epilogue read a warp's 32 matrix rows from as
// many different plane rows, which a dense [pair][VPB] tile maps onto 2-4
// banks (16-way conflicts for Q = 32); swizzled they spread over 8 chunks.
struct TmaTiles {
  int use = 0;  // 0: cp.async fallback (plane stride not a multiple of 16 B)
  int hb = 0, nb = 0;
  int swz = 0;  // swizzle mask applied by the readers (0: dense tile)
  int swz_lo = 0;  // the same for the lo tile (4-byte elements: rows half as long)
};

// float2 index of tile element idx under the TMA swizzle (buffer 1 KB aligned).
__device__ __forceinline__ int swz_at(int idx, int mask) {
  const int b = idx << 3;
  return (b ^ (((b >> 7) & mask) << 4)) >> 3;
}
// lo2 index of lo-tile element idx under its swizzle.
__device__ __forceinline__ int swz_lo_at(int idx, int mask) {
  const int b = idx << 2;
  return (b ^ (((b >> 7) & mask) << 4)) >> 2;
}

template <int QP_, int RPT_, int THREADS_, int MINB_, int ACC_ = 0, int PF_ = 4, int QF_ = 0, int TILE_ = 0>
struct Layout {
  static constexpr int QP = QP_, RPT = RPT_, kThreads = THREADS_, kMinBlocks = MINB_;
  static constexpr int QF = QF_;  // > 0: the channel count is fixed at compile time (Q == QF)
  static constexpr int kPrefetch = PF_;  // LDS.128 of v kept in flight ahead of their use
  static constexpr int kTPV = QP / RPT;          // threads per voxel
  static constexpr int kVPB = kThreads / kTPV;   // voxels per block
  static constexpr int kWPV = kTPV > 32 ? kTPV / 32 : 1;  // warps per voxel
  static constexpr int kAcc = ACC_ > 0 ? ACC_ : (RPT >= 4 ? 1 : 4 / RPT);  // accumulator pairs per row
  // Tiled matvec (TILE_ != 0, RPT == 1): thread `local` = 4 rg + cg holds the
  // 4 x kTC block of rows 4 rg.., columns kTC cg.. instead of a full row: a
  // product needs only its kTC entries of v and two shuffle rounds over the
  // column groups (lane xor 2, 1) leave (M v)[local] in thread `local`
  // (row_of(local) == local).  Used for Q = 64 (C5 K4 20.4 -> 18.5 ms); for
  // Q = 32 it measured slower than one row per thread (0.95 vs 0.92 ms, C2:
  // the shared-memory wavefronts barely drop and the shuffles add latency).
  static constexpr bool kTile = TILE_ != 0;
  static constexpr int kTC = QP / 4;  // tile: 4 rows x kTC columns
  // float2 per v row: column group g starts at g (kTC + 2) in the tiled
  // layout (16-B aligned, the four groups on disjoint banks), else QP + 2.
  static constexpr int kStride = kTile ? QP + 8 : QP + 2;
  __device__ static constexpr int vidx(int c) { return kTile ? c + (c / kTC) * 2 : c; }
  __device__ static constexpr int col_group(int local) { return local & 3; }
  __device__ static constexpr int row_group(int local) { return local >> 2; }
  __device__ static constexpr int row_of(int local) { return kTile ? 4 * row_group(local) + col_group(local) : local; }
  static_assert(!kTile || (RPT == 1 && QP >= 8), "tiled matvec: one row per thread");
};

// Sum over the voxel's threads.  Multi-warp voxels go through shared memory
// with block-wide barriers (used only outside the iteration loop).
template <class L, typename T>
__device__ __forceinline__ T voxel_sum(T x, T* red, int vox) {
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

template <class L>
__device__ __forceinline__ void voxel_sync() {
  if constexpr (L::kTPV <= 32)
    __syncwarp();
  else
    __syncthreads();
}

// Barrier over the threads of one voxel only: a warp-level sync for
// single-warp voxels, a named barrier (id 1 + vox) for multi-warp voxels.
template <class L>
__device__ __forceinline__ void voxel_bar(int vox) {
  if constexpr (L::kTPV <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + vox), "n"(L::kTPV) : "memory");
  }
}

__device__ __forceinline__ int pair_index(int p, int c, int Q) { return p * Q - p * (p - 1) / 2 + (c - p); }

// Element (p, c) of the Hermitian matrix from the packed tile (zero outside Q).
__device__ __forceinline__ float2 herm_at(const float2* gs, int p, int c, int Q, int VPB, int vox, int swz) {
  float2 val = make_float2(0.f, 0.f);
  SKB_DCHECK(p >= 0 && c >= 0 && vox >= 0 && vox < VPB);
  SKB_DCHECK(p >= Q || c >= Q || pair_index(min(p, c), max(p, c), Q) < Q * (Q + 1) / 2);
  if (p < Q && c < Q) {
    if (p <= c) {
      val = gs[swz_at(pair_index(p, c, Q) * VPB + vox, swz)];
    } else {
      const float2 t = gs[swz_at(pair_index(c, p, Q) * VPB + vox, swz)];
      val = make_float2(t.x, -t.y);
    }
    if (p == c) val.y = 0.f;  // spatial_gram.cpp:140-146
  }
  return val;
}

// herm_at for row AND column indices known only at run time (the tiled
// layout): the packed element (min, max) with a conditional conjugate, no
// branches around the load (the branchy form faulted under ptxas 12.9 when
// both indices were run-time values in the fully unrolled unpack).
__device__ __forceinline__ float2 herm_at_bf(const float2* gs, int p, int c, int Q, int VPB, int vox, int swz) {
  const int lo = min(p, c), hi = max(p, c);
  const bool in = hi < Q;
  SKB_DCHECK(lo >= 0 && vox >= 0 && vox < VPB);
  const float2 t = gs[swz_at((in ? pair_index(lo, hi, Q) : 0) * VPB + vox, swz)];
  return in ? make_float2(t.x, p == c ? 0.f : (p <= c ? t.y : -t.y)) : make_float2(0.f, 0.f);
}

// STACK: a.slices > 1 (the tile index also selects the slice; compiled out of
// the single-slice kernel, where the extra index math cost 2% on C2/C4).
template <class L, bool STACK>
__global__ void __launch_bounds__(L::kThreads, L::kMinBlocks)
    power_kernel(PowerArgs a, const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
                 TmaTiles tt, int tile_rows) {
  constexpr int QP = L::QP, RPT = L::RPT, VPB = L::kVPB, WPV = L::kWPV, TPV = L::kTPV;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int Q = L::QF > 0 ? L::QF : a.q;
  const int h = Q * (Q + 1) / 2;
  const int tile_elems = tile_rows * VPB;  // tile bytes: a multiple of 1 KB
  SKB_DCHECK(blockDim.x == L::kThreads && h <= tile_rows && Q <= QP);  // every packed read lands in the tile
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw);  // [0..1] hi buffers, [2] lo
  // tile buffers start on a 1 KB boundary (the swizzle pattern follows address bits 4..9)
  float2* gbuf = reinterpret_cast<float2*>(smem_raw + ((smem_u32(smem_raw) + 128 + 1023) & ~1023u) -
                                           smem_u32(smem_raw));  // [2][tile_elems] hi planes
  lo2* lbuf = reinterpret_cast<lo2*>(gbuf + 2 * tile_elems);             // [tile_elems] lo planes (bf16 pairs)
  float2* vs = reinterpret_cast<float2*>(lbuf + tile_elems);             // [2][VPB][kStride]
  double2* vds = reinterpret_cast<double2*>(vs + 2 * VPB * L::kStride);  // [VPB][QP] final v in FP64
  double* redd = reinterpret_cast<double*>(vds + VPB * QP);              // [VPB][kWPV]
  float* red = reinterpret_cast<float*>(redd + VPB * WPV);               // [VPB][kWPV]
  float* red2 = red + VPB * WPV;                                         // [2][VPB][kWPV]
  int* pct = reinterpret_cast<int*>(red2 + 2 * VPB * WPV);               // [h] packed index -> (p << 8) | c
  for (int e = threadIdx.x; e < h; e += blockDim.x) {
    int pp = 0, base = 0;
    while (e >= base + Q - pp) base += Q - pp++;
    pct[e] = (pp << 8) | (pp + e - base);
  }

  const int vox = threadIdx.x / TPV;
  const int local = threadIdx.x % TPV;
  const int prow = L::row_of(local);    // the thread's rows: prow + r * TPV
  const i64 tps = (a.n + VPB - 1) / VPB;  // tiles per slice
  const i64 tiles = STACK ? tps * a.slices : tps;
  const i64 ld = a.ld > 0 ? a.ld : a.n;  // plane / channel stride (a voxel range of a larger grid)

  // Tile loads.  TMA path: one thread issues nb boxes (hb plane rows x VPB
  // voxels, OOB zero-filled) completing on the buffer's mbarrier; every
  // thread waits on its phase.  Fallback: per-thread 8-byte cp.async.
  if (tt.use && threadIdx.x == 0) {
    for (int k = 0; k < 3; ++k) mbar_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0;  // bit k: parity of bars[k]
  // (a stack of slices: tile t = slice t / tps, tile t % tps of that slice; the
  // slice's planes are rows [slice h, slice h + h) of the 2-D tensor)
  auto load_tile = [&](i64 t, float2* dst, const float2* src, const CUtensorMap* map, int bar) {
    const i64 sl = STACK ? t / tps : 0;
    const i64 jj0 = (t - sl * tps) * VPB;
    if (tt.use) {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // prior generic writes to dst
        mbar_expect_tx(bars + bar, unsigned(tt.nb * tt.hb * VPB * sizeof(float2)));
        for (int k = 0; k < tt.nb; ++k)
          tma_load_2d(dst + k * tt.hb * VPB, map, int(jj0), int(sl) * h + k * tt.hb, bars + bar);
      }
      return;
    }
    src += sl * i64(h) * ld;
    for (int e = threadIdx.x; e < h * VPB; e += blockDim.x) {
      const int pair = e / VPB, v = e % VPB;
      const bool ok = jj0 + v < a.n;
      cp_async8(dst + e, src + (ok ? i64(pair) * ld + jj0 + v : 0), ok ? 8 : 0);
    }
    cp_async_commit();
  };
  auto load_lo_tile = [&](i64 t) {  // the tile's lo planes into lbuf, completing on bars[2]
    const i64 sl = STACK ? t / tps : 0;
    const i64 jj0 = (t - sl * tps) * VPB;
    if (tt.use) {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(bars + 2, unsigned(tt.nb * tt.hb * VPB * sizeof(lo2)));
        for (int k = 0; k < tt.nb; ++k)
          tma_load_2d(lbuf + k * tt.hb * VPB, &tm_lo, int(jj0), int(sl) * h + k * tt.hb, bars + 2);
      }
      return;
    }
    const lo2* src = a.planes_lo + sl * i64(h) * ld;
    for (int e = threadIdx.x; e < h * VPB; e += blockDim.x) {
      const int pair = e / VPB, v = e % VPB;
      const bool ok = jj0 + v < a.n;
      cp_async4(lbuf + e, src + (ok ? i64(pair) * ld + jj0 + v : 0), ok ? 4 : 0);
    }
    cp_async_commit();
  };
  auto wait_tile = [&](int bar) {
    mbar_wait(bars + bar, (phase >> bar) & 1u);
    phase ^= 1u << bar;
  };

  i64 tile = blockIdx.x;
  int buf = 0;
  if (tile < tiles) load_tile(tile, gbuf, a.planes, &tm_hi, 0);
  for (; tile < tiles; tile += gridDim.x, buf ^= 1) {
    const i64 next = tile + gridDim.x;
    if (next < tiles) load_tile(next, gbuf + (buf ^ 1) * tile_elems, a.planes, &tm_hi, buf ^ 1);
    if (tt.use) {
      wait_tile(buf);
    } else {
      if (next < tiles)
        cp_async_wait<1>();
      else
        cp_async_wait<0>();
      __syncthreads();
    }
    float2* gs = gbuf + buf * tile_elems;
    const i64 sl = STACK ? tile / tps : 0;  // slice of this tile
    const i64 j0 = (tile - sl * tps) * VPB;
    const i64 j = j0 + vox;
    const bool live = j < a.n;
    const i64 cbase = sl * i64(Q) * ld;  // the slice's first channel row in recon / maps

    // Unpack this thread's rows.
    float2 m[RPT][QP];
    float2 mc0[RPT];  // M[p][0] of the thread's rows p (the e_0 restart of iteration 0)
    if constexpr (L::kTile) {
      const int r0 = 4 * L::row_group(local), c0 = L::kTC * L::col_group(local);
#pragma unroll
      for (int tr = 0; tr < 4; ++tr)
#pragma unroll
        for (int tc = 0; tc < L::kTC; ++tc) m[0][tr * L::kTC + tc] = herm_at_bf(gs, r0 + tr, c0 + tc, Q, VPB, vox, tt.swz);
      mc0[0] = herm_at_bf(gs, prow, 0, Q, VPB, vox, tt.swz);
    } else {
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
#pragma unroll
        for (int c = 0; c < QP; ++c)
          // compile-time Q: the branch-free read (C2 K4 0.905 -> 0.878 ms, C4 5.62 -> 4.97 ms);
          // run-time Q keeps the branchy one (the branch-free form spills there)
          m[r][c] = L::QF > 0 ? herm_at_bf(gs, prow + r * TPV, c, Q, VPB, vox, tt.swz)
                              : herm_at(gs, prow + r * TPV, c, Q, VPB, vox, tt.swz);
        mc0[r] = m[r][0];
      }
    }
    // Stream the lo residual planes of this tile while the iterations run
    // (its own buffer: the final Rayleigh quotient reads hi and lo packed).
    if (a.planes_lo != nullptr) load_lo_tile(tile);
    // recon values for the epilogue, loaded while the iterations run
    float2 rcv[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int p = prow + r * TPV;
      rcv[r] = (a.recon != nullptr && p < Q && live) ? a.recon[cbase + i64(p) * ld + j] : make_float2(0.f, 0.f);
    }

    // v is double-buffered in shared memory (buffers 0 and 1) together with
    // the per-warp partials of ||u||^2, so an iteration needs one voxel barrier.
    auto vb = [&](int b) { return vs + (b * VPB + vox) * L::kStride; };
    const float init = rsqrtf(float(Q));
    float2 vp[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      vp[r] = (prow + r * TPV < Q) ? make_float2(init, 0.f) : make_float2(0.f, 0.f);
      vb(0)[L::vidx(prow + r * TPV)] = vp[r];
    }
    bool done = false;
    voxel_sync<L>();

    // Publish u into buffer b and its squared norm: returned directly for a
    // single-warp voxel, left as per-warp partials in red2[b] otherwise.
    // Single-warp voxels return the thread's own partial of ||u||^2: the
    // butterfly over the voxel's lanes runs at the top of the next iteration,
    // after its barrier, where ptxas interleaves the shuffle chain with the
    // matvec's loads and FFMA2s (before the barrier it was exposed: 14% of the
    // stall samples on C2).
    auto publish = [&](const float2 (&u)[RPT], int b) -> float {
      float x = 0.f;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        SKB_DCHECK(L::vidx(prow + r * TPV) < L::kStride);
        vb(b)[L::vidx(prow + r * TPV)] = u[r];
        x = fmaf(u[r].x, u[r].x, fmaf(u[r].y, u[r].y, x));
      }
      if constexpr (TPV <= 32 || L::kTile) {
        return x;  // tiled: recomputed from v by the next matvec (tile_norm)
      } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0) red2[(b * VPB + vox) * WPV + (local >> 5)] = x;
        return 0.f;
      }
    };
    auto voxel_butterfly = [&](float x) -> float {
#pragma unroll
      for (int o = TPV / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      return x;
    };
    auto published_norm = [&](float own, int b) -> float {
      if constexpr (TPV <= 32 || L::kTile) {
        return own;  // already reduced (voxel_butterfly / the tiled matvec)
      } else {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < WPV; ++k) s += red2[(b * VPB + vox) * WPV + k];
        return s;
      }
    };

    // M v for the thread's rows: v is staged into registers in chunks of 8
    // complex values (4 LDS.128, shared by all RPT rows) feeding kAcc
    // independent accumulator pairs per row.
    // Complex MAC as two FFMA2: acc += m.x * (v.x, v.y), acc2 += m.y * (v.y, v.x);
    // (M v) = (acc.x - acc2.x, acc.y + acc2.y).
    // side: a value whose butterfly over the voxel's lanes (single-warp voxels)
    // is spread over the chunks of the product, one shuffle level every few
    // chunks, so its latency hides behind the FFMA2s (nullptr: none).  For
    // ||u||^2 in the iteration loop: C2 K4 0.878 -> 0.797 ms, C4 4.97 -> 4.71
    // ms (the chain issued as one block, before or after the barrier, was
    // 11-14% of the stall samples; the 48 B of spill it costs are harmless).
    auto matvec = [&](const float2* v, float2 (&out)[RPT], float* side = nullptr) {
      if constexpr (L::kTile) {
        // 4 x kTC block times v[kTC cg ..]: acc += m.x (v.x, v.y), acc2 += m.y (v.y, v.x)
        // (two accumulators per row: C5 K4 18.5 ms against 22.7 with one)
        constexpr int TC = L::kTC;
        const int cg = L::col_group(local);
        const float4* v4 = reinterpret_cast<const float4*>(v + cg * (TC + 2));
        SKB_DCHECK(v >= vs && v + cg * (TC + 2) + TC <= vs + 2 * VPB * L::kStride);
        // side (tiled): ||v||^2 of the buffer read, from the column-group
        // quarter of v the thread loads anyway, summed over the four column
        // groups with the reduce-scatter's shuffles -- no cross-warp exchange
        // (publish's warp butterfly + shared partials were 17.7% of C5's K4
        // stall samples)
        u64 acc[4], acc2[4], nacc = 0ull;
#pragma unroll
        for (int tr = 0; tr < 4; ++tr) acc[tr] = acc2[tr] = 0ull;
#pragma unroll
        for (int t = 0; t < TC / 2; ++t) {
          const float4 vt = v4[t];
          if (side != nullptr) {
            ffma2(nacc, pk(vt.x, vt.y), pk(vt.x, vt.y));
            ffma2(nacc, pk(vt.z, vt.w), pk(vt.z, vt.w));
          }
#pragma unroll
          for (int tr = 0; tr < 4; ++tr) {
            const float2 ma = m[0][tr * TC + 2 * t], mb = m[0][tr * TC + 2 * t + 1];
            ffma2(acc[tr], pk(ma.x, ma.x), pk(vt.x, vt.y));
            ffma2(acc2[tr], pk(ma.y, ma.y), pk(vt.y, vt.x));
            ffma2(acc[tr], pk(mb.x, mb.x), pk(vt.z, vt.w));
            ffma2(acc2[tr], pk(mb.y, mb.y), pk(vt.w, vt.z));
          }
        }
        float2 s4[4];
#pragma unroll
        for (int tr = 0; tr < 4; ++tr) {
          const float2 x = unpk(acc[tr]), y = unpk(acc2[tr]);
          s4[tr] = make_float2(x.x - y.x, x.y + y.y);
        }
        // reduce-scatter over the column groups: bit 1 of cg keeps rows {2,3}
        // (else {0,1}), bit 0 then keeps the odd (else even) one: row 4 rg + cg.
        // cg is lane bits 0..1: partners at lane xor 2, then xor 1.
        const bool b1 = (cg & 2) != 0, b0 = (cg & 1) != 0;
        float2 k0 = b1 ? s4[2] : s4[0], k1 = b1 ? s4[3] : s4[1];
        const float2 o0 = b1 ? s4[0] : s4[2], o1 = b1 ? s4[1] : s4[3];
        const float2 nn = unpk(nacc);
        float nq = nn.x + nn.y;
        k0.x += __shfl_xor_sync(0xffffffffu, o0.x, 2);
        k0.y += __shfl_xor_sync(0xffffffffu, o0.y, 2);
        k1.x += __shfl_xor_sync(0xffffffffu, o1.x, 2);
        k1.y += __shfl_xor_sync(0xffffffffu, o1.y, 2);
        if (side != nullptr) nq += __shfl_xor_sync(0xffffffffu, nq, 2);
        float2 kk = b0 ? k1 : k0;
        const float2 oo = b0 ? k0 : k1;
        kk.x += __shfl_xor_sync(0xffffffffu, oo.x, 1);
        kk.y += __shfl_xor_sync(0xffffffffu, oo.y, 1);
        if (side != nullptr) *side = nq + __shfl_xor_sync(0xffffffffu, nq, 1);
        out[0] = kk;
        return;
      }
      constexpr int A = L::kAcc;
      const float4* v4 = reinterpret_cast<const float4*>(v);
      u64 acc[RPT][A], acc2[RPT][A];
#pragma unroll
      for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int k = 0; k < A; ++k) acc[r][k] = acc2[r][k] = 0ull;
      // v arrives as NT float4 (two columns each) through a rotating buffer
      // of D register sets.  (ptxas re-sinks each load next to its use under
      // the 128-register budget whatever D is — measured: the loop is
      // short-scoreboard bound on these loads; 1-block/255-register and
      // two-rows-per-thread layouts that could keep loads in flight lose more
      // to the halved occupancy.)
      constexpr int NT = QP / 2 > 0 ? QP / 2 : 1;
      constexpr int D = L::kPrefetch < NT ? L::kPrefetch : NT;
      float4 buf[D];
#pragma unroll
      for (int t = 0; t < D; ++t) buf[t] = v4[t];
      constexpr int LV = TPV <= 32 ? (TPV >= 32 ? 5 : TPV >= 16 ? 4 : TPV >= 8 ? 3 : TPV >= 4 ? 2 : TPV >= 2 ? 1 : 0) : 0;
      float side_sh = 0.f;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const float4 vt = buf[t % D];
        if (t + D < NT) buf[t % D] = v4[t + D];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const float2 ma = m[r][2 * t], mb = m[r][2 * t + 1];
          const int ka = (2 * t) % A, kb = (2 * t + 1) % A;
          ffma2(acc[r][ka], pk(ma.x, ma.x), pk(vt.x, vt.y));
          ffma2(acc2[r][ka], pk(ma.y, ma.y), pk(vt.y, vt.x));
          ffma2(acc[r][kb], pk(mb.x, mb.x), pk(vt.z, vt.w));
          ffma2(acc2[r][kb], pk(mb.y, mb.y), pk(vt.w, vt.z));
        }
        if (side != nullptr) {
          // level j: the shuffle at chunk 3j, its sum two chunks later (in-order
          // issue: an add right behind its shuffle stalls the warp); short
          // products (NT < 3 LV) take one level per chunk
          constexpr int SP = NT >= 3 * LV ? 3 : 1;
#pragma unroll
          for (int j = 0; j < LV; ++j) {
            const int ts = SP * j, ta = ts + (SP == 3 ? 2 : 0);
            if (t == ts) side_sh = __shfl_xor_sync(0xffffffffu, *side, TPV >> (j + 1));
            if (t == ta) *side += side_sh;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        float2 s = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < A; ++k) {
          const float2 x = unpk(acc[r][k]), y = unpk(acc2[r][k]);
          s = make_float2(s.x + (x.x - y.x), s.y + (x.y + y.y));
        }
        out[r] = s;
      }
    };

    // Iteration 0, peeled: an annihilated all-ones start restarts from e_0
    // (eigensolve.cpp:56-63); the candidate is formed uniformly and selected.
    if (a.iters > 0) {
      float2 mv[RPT], w[RPT], w0[RPT], v0[RPT];
      matvec(vb(0), mv);
      float x = 0.f, x0 = 0.f;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        w[r] = make_float2(a.alpha * vp[r].x + a.beta * mv[r].x, a.alpha * vp[r].y + a.beta * mv[r].y);
        v0[r] = (prow + r * TPV == 0) ? make_float2(1.f, 0.f) : make_float2(0.f, 0.f);
        // (B e_0)[p] = alpha e_0[p] + beta M[p][0]
        w0[r] = make_float2(a.alpha * v0[r].x + a.beta * mc0[r].x, a.alpha * v0[r].y + a.beta * mc0[r].y);
        x += w[r].x * w[r].x + w[r].y * w[r].y;
        x0 += w0[r].x * w0[r].x + w0[r].y * w0[r].y;
      }
      float n2 = voxel_sum<L>(x, red, vox);
      const float n20 = voxel_sum<L>(x0, red, vox);
      if (n2 < 1e-28f) {  // ||B v|| < 1e-14
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          vp[r] = v0[r];
          w[r] = w0[r];
        }
        n2 = n20;
      }
      if (n2 < 1e-28f) done = true;  // B ~ 0 here: keep the current v
      if (!done) {
        const float inv = rsqrtf(n2);
#pragma unroll
        for (int r = 0; r < RPT; ++r) vp[r] = make_float2(w[r].x * inv, w[r].y * inv);
      }
    }
    // Iterations 1..iters-1, software-pipelined on the unnormalised iterate
    // u_k: ||u_k||^2 travels with u_k (published together), w = B(u_k/||u_k||)
    // = B v_k.  ||B v_k|| is known one iteration later, so the break test of
    // iteration k (||B v_k|| < 1e-14 -> keep v_k) is evaluated then, with v_k
    // in vprev.  Iteration k reads buffer k&1 and writes buffer (k+1)&1; the
    // barrier at the top of iteration k+1 orders both (every read of (k+1)&1
    // from iteration k-1 precedes the barrier at the top of iteration k).
    float2 up[RPT], vprev[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) up[r] = vprev[r] = vp[r];
    float own = 0.f;
    if (a.iters > 1) own = publish(up, 1);  // iteration 0 read only buffer 0
    if constexpr (L::kTile) {
      // (the tiled Q = 64 kernel keeps the plain loop: restructured as below
      // it spills, C5 18.1 -> 19.6 ms)
      for (int it = 1; it < a.iters; ++it) {
        const int b = it & 1;
        voxel_bar<L>(vox);
        float2 mv[RPT];
        matvec(vb(b), mv, &own);
        float n2 = published_norm(own, b);
        asm("" : "+f"(n2) : "f"(mv[0].x));
        done = done || (it > 1 && n2 < 1e-28f);
        const float inv = rsqrtf(n2);
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const float2 nv = make_float2(up[r].x * inv, up[r].y * inv);
          const float2 nu = make_float2((a.alpha * up[r].x + a.beta * mv[r].x) * inv,
                                        (a.alpha * up[r].y + a.beta * mv[r].y) * inv);
          vprev[r] = done ? vprev[r] : nv;
          up[r] = done ? up[r] : nu;
        }
        own = publish(up, b ^ 1);
      }
    } else {
      // one iteration reading buffer b (b = it & 1) and publishing into b ^ 1;
      // the row layouts run them in pairs (b = 1, 0) with the two buffers'
      // addresses fixed, halving the loop and address overhead (C2 K4 0.797 ->
      // 0.780 ms)
      float2* const vbuf[2] = {vb(0), vb(1)};
      auto iteration = [&](int it, int b) {
        voxel_bar<L>(vox);
        float2 mv[RPT];
        if constexpr (TPV <= 32)
          matvec(vbuf[b], mv, &own);  // the butterfly of ||u||^2 rides along
        else
          matvec(vbuf[b], mv);
        // ||u_k||^2 (the previous iteration's shuffle reduction) is consumed only
        // after the products: the empty asm ties it to mv so ptxas cannot hoist
        // the test above the loads, and the reduction overlaps the matvec.
        float n2 = published_norm(own, b);
        asm("" : "+f"(n2) : "f"(mv[0].x));
        done = done || (it > 1 && n2 < 1e-28f);
        const float inv = rsqrtf(n2);
#pragma unroll
        for (int r = 0; r < RPT; ++r) {  // branch-free: one basic block per iteration
          const float2 nv = make_float2(up[r].x * inv, up[r].y * inv);
          const float2 nu = make_float2((a.alpha * up[r].x + a.beta * mv[r].x) * inv,
                                        (a.alpha * up[r].y + a.beta * mv[r].y) * inv);
          vprev[r] = done ? vprev[r] : nv;
          up[r] = done ? up[r] : nu;
        }
        own = publish(up, b ^ 1);
      };
      int it = 1;
      for (; it + 1 < a.iters; it += 2) {
        iteration(it, 1);
        iteration(it + 1, 0);
      }
      if (it < a.iters) iteration(it, 1);
    }
    int fb = 0;  // buffer that receives the final v
    if (a.iters > 1) {
      voxel_bar<L>(vox);
      if constexpr (L::kTile) {
        float2 unused[RPT];
        matvec(vb(a.iters & 1), unused, &own);  // (the product itself is dead code)
      } else if constexpr (TPV <= 32) {
        own = voxel_butterfly(own);
      }
      const float n2 = published_norm(own, a.iters & 1);
      const bool keep = done || n2 < 1e-28f;
      const float inv = keep ? 0.f : rsqrtf(n2);
#pragma unroll
      for (int r = 0; r < RPT; ++r) vp[r] = keep ? vprev[r] : make_float2(up[r].x * inv, up[r].y * inv);
      fb = (a.iters & 1) ^ 1;  // last read by iteration iters-1, before the barrier above
    }
    (void)fb;
    // FP32 Rayleigh quotient on hi first (one more matvec from registers): a
    // voxel whose value is large relative to ||M|| (rq32_min, pipeline only)
    // keeps it and skips the FP64 evaluation below.
    bool need64 = true;
    float mv32 = 0.f;
    if (a.rq32_min > 0.f) {
      voxel_bar<L>(vox);  // every read of the v buffers precedes the overwrite
#pragma unroll
      for (int r = 0; r < RPT; ++r) vb(0)[L::vidx(prow + r * TPV)] = vp[r];
      voxel_sync<L>();
      float2 y[RPT];
      matvec(vb(0), y);
      float x = 0.f;
#pragma unroll
      for (int r = 0; r < RPT; ++r) x = fmaf(vp[r].x, y[r].x, fmaf(vp[r].y, y[r].y, x));  // Re(conj(v) y)
      mv32 = voxel_sum<L>(x, red, vox);
      need64 = !(mv32 * a.lam_scale >= a.rq32_min);
    }
    // Rayleigh quotient in FP64 on M = hi + lo over the packed triangle,
    //   Re(v^H M v) = sum_p M_pp |v_p|^2 + 2 Re sum_{p<c} conj(v_p) M_pc v_c,
    // split evenly over the voxel's threads (the FP32 iterate v enters only to
    // second order); value = Re(v^H B v).  v is staged once in FP64.
    {
      double2* vd = vds + vox * QP;
#pragma unroll
      for (int r = 0; r < RPT; ++r) vd[prow + r * TPV] = make_double2(double(vp[r].x), double(vp[r].y));
    }
    if (a.planes_lo != nullptr) {
      if (tt.use)
        wait_tile(2);
      else
        cp_async_wait<0>();
    }
    __syncthreads();
    double xd = 0.0;
    if (!need64) {
      // FP32 value kept (voxel_sum below still runs: its shuffles span voxels)
    } else {
      const double2* vd = vds + vox * QP;
      // four accumulators over alternate packed elements, loop unrolled by
      // four: the loop is latency-bound (LDS -> F2F -> DFMA chains), so more
      // elements in flight (two accumulators: C5 K4 18.7 -> 18.1 ms)
      double xd1 = 0.0, xd2 = 0.0, xd3 = 0.0;
#pragma unroll 4
      for (int e = local; e < h; e += TPV) {
        const int sel = (e / TPV) & 3;
        double& acc = sel == 0 ? xd : sel == 1 ? xd1 : sel == 2 ? xd2 : xd3;
        const int pc = pct[e], pp = pc >> 8, cc = pc & 0xff;
        const float2 hv = gs[swz_at(e * VPB + vox, tt.swz)];
        double mx = double(hv.x), my = double(hv.y);
        if (a.planes_lo != nullptr) {
          const float2 lv = lo_unpack(lbuf[swz_lo_at(e * VPB + vox, tt.swz_lo)]);
          mx += double(lv.x);
          my += double(lv.y);
        }
        const double2 vpp = vd[pp], vc = vd[cc];
        if (pp == cc) {
          acc = fma(mx, vpp.x * vpp.x + vpp.y * vpp.y, acc);  // spatial_gram.cpp:140-146 (real diagonal)
        } else {
          const double tx = mx * vc.x - my * vc.y, ty = mx * vc.y + my * vc.x;  // M_pc v_c
          acc = fma(2.0, vpp.x * tx + vpp.y * ty, acc);                         // 2 Re(conj(v_p) .)
        }
      }
      xd = (xd + xd1) + (xd2 + xd3);
    }
    // ||v||^2, v^H M v and (with recon) conj(v) . recon reduced together: the
    // phase reference needs only the direction of the last, so it is formed
    // from the unnormalised v and the four butterflies run interleaved.
    float xn = 0.f, xr = 0.f, xi = 0.f;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      xn += vp[r].x * vp[r].x + vp[r].y * vp[r].y;
      const float2 rc = rcv[r];  // zero without recon
      xr += vp[r].x * rc.x + vp[r].y * rc.y;  // conj(v) * recon
      xi += vp[r].x * rc.y - vp[r].y * rc.x;
    }
    double mv64;
    float vn2, ux, uy;
    if constexpr (TPV <= 32) {
#pragma unroll
      for (int o = TPV / 2; o > 0; o >>= 1) {
        xd += __shfl_xor_sync(0xffffffffu, xd, o);
        xn += __shfl_xor_sync(0xffffffffu, xn, o);
        xr += __shfl_xor_sync(0xffffffffu, xr, o);
        xi += __shfl_xor_sync(0xffffffffu, xi, o);
      }
      mv64 = xd;
      vn2 = xn;
      ux = xr;
      uy = xi;
    } else {
      mv64 = voxel_sum<L>(xd, redd, vox);
      vn2 = voxel_sum<L>(xn, red, vox);
      ux = voxel_sum<L>(xr, red, vox);
      uy = voxel_sum<L>(xi, red, vox);
    }
    const double mv = need64 ? mv64 : double(mv32);

    if (a.recon != nullptr) {
      // normalize_maps, per voxel: SoS (maps.cpp:117-128) then phase reference
      // against the apodised coil-combined calibration recon (maps.cpp:163-172).
      if (vn2 > 0.f) {
        const float inv = 1.0f / sqrtf(vn2);
#pragma unroll
        for (int r = 0; r < RPT; ++r) vp[r] = make_float2(vp[r].x * inv, vp[r].y * inv);
      } else if (local == 0 && live && a.zeroed) {
        atomicAdd(a.zeroed + sl, 1ull);
      }
      const float mag = sqrtf(ux * ux + uy * uy);
      if (mag > 0.f) {
        const float cx = ux / mag, cy = uy / mag;
#pragma unroll
        for (int r = 0; r < RPT; ++r)
          vp[r] = make_float2(vp[r].x * cx - vp[r].y * cy, vp[r].x * cy + vp[r].y * cx);
      }
    }

    // Stage maps for channel-major coalesced stores: reuse the hi plane tile.
    __syncthreads();
    float2* ms = gs;  // [QP][VPB]
#pragma unroll
    for (int r = 0; r < RPT; ++r) ms[(prow + r * TPV) * VPB + vox] = vp[r];
    __syncthreads();
    for (int e = threadIdx.x; e < Q * VPB; e += blockDim.x) {
      const int c = e / VPB, v = e % VPB;
      if (j0 + v < a.n) a.maps[cbase + i64(c) * ld + j0 + v] = ms[c * VPB + v];
    }
    if (local == 0 && live) {
      const float lam = float(mv * double(a.lam_scale));
      const i64 js = sl * ld + j;
      if (a.lambda) a.lambda[js] = lam;
      if (a.value) a.value[js] = float(double(a.alpha) * vn2 + double(a.beta) * mv);
      if (a.mask) a.mask[js] = lam < a.mask_threshold ? 1 : 0;
    }
    __syncthreads();  // the staging buffer is the prefetch target two tiles on
  }
}

// 2-D tensor map over packed planes [h][n] (float2 as one 8-byte element):
// box {VPB voxels, hb plane rows}.  Returns false when TMA cannot address it.
// elem: bytes per element (8: float2 hi planes, 4: bf16-pair lo planes).
bool encode_planes(CUtensorMap* m, const void* base, int elem, i64 n, i64 ld, i64 h, int vpb, int hb,
                   CUtensorMapSwizzle swz) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode || base == nullptr || (ld * elem) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0 ||
      (vpb * elem) % 16 != 0)
    return false;
  const cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(h)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * cuuint64_t(elem)};
  const cuuint32_t box[2] = {cuuint32_t(vpb), cuuint32_t(hb)};
  const cuuint32_t estr[2] = {1, 1};
  // L2 promotion of the 8*vpb-byte box rows: 256 B
  constexpr CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  return encode(m, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
                const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <class L>
void launch(sk_ctx* ctx, const PowerArgs& a) {
  const int h = a.q * (a.q + 1) / 2;
  TmaTiles tt;
  CUtensorMap tm_hi{}, tm_lo{};
  // box rows: <= 256; every box a multiple of 128 B (TMA smem alignment) and of 8 rows when
  // swizzled (the pattern's period); a swizzled tile a multiple of 1 KB (buffers stay 1 KB aligned)
  const int row_bytes = L::kVPB * int(sizeof(float2));
  const CUtensorMapSwizzle swz = row_bytes == 32  ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : row_bytes == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                                    : CU_TENSOR_MAP_SWIZZLE_NONE;
  const bool swizzled = swz != CU_TENSOR_MAP_SWIZZLE_NONE;
  const int al = std::max(std::max(1, 128 / row_bytes), swizzled ? 8 : 1);
  tt.nb = (h + 255) / 256;
  for (;; ++tt.nb) {
    tt.hb = ((h + tt.nb - 1) / tt.nb + al - 1) / al * al;
    if (tt.hb <= 256) break;
  }
  const i64 ld = a.ld > 0 ? a.ld : a.n;
  // the lo tile's rows are half as long: the next smaller swizzle (dense below 32 B)
  const CUtensorMapSwizzle swz_lo = swz == CU_TENSOR_MAP_SWIZZLE_128B  ? CU_TENSOR_MAP_SWIZZLE_64B
                                    : swz == CU_TENSOR_MAP_SWIZZLE_64B ? CU_TENSOR_MAP_SWIZZLE_32B
                                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
  const i64 rows = i64(h) * (a.slices > 1 ? a.slices : 1);  // a stack of slices: [slices][h] plane rows
  tt.use = encode_planes(&tm_hi, a.planes, 8, a.n, ld, rows, L::kVPB, tt.hb, swz) &&
           (a.planes_lo == nullptr || encode_planes(&tm_lo, a.planes_lo, 4, a.n, ld, rows, L::kVPB, tt.hb, swz_lo));
  if (a.planes_lo == nullptr) tm_lo = tm_hi;
  tt.swz = !tt.use ? 0 : swz == CU_TENSOR_MAP_SWIZZLE_32B ? 1 : swz == CU_TENSOR_MAP_SWIZZLE_64B ? 3
                                                          : swz == CU_TENSOR_MAP_SWIZZLE_128B ? 7 : 0;
  tt.swz_lo = !tt.use ? 0 : swz_lo == CU_TENSOR_MAP_SWIZZLE_32B ? 1 : swz_lo == CU_TENSOR_MAP_SWIZZLE_64B ? 3 : 0;
  const int alt = tt.swz ? std::max(al, 1024 / row_bytes) : al;
  const int tile_rows = (std::max(std::max(h, L::QP), tt.use ? tt.nb * tt.hb : 0) + alt - 1) / alt * alt;
  const size_t tile = size_t(tile_rows) * L::kVPB * sizeof(float2);
  // two hi tile buffers (double-buffered prefetch) + the lo tile (half the bytes)
  const size_t smem = 1024 + 128 + 2 * tile + tile / 2 +
                      2 * size_t(L::kVPB) * L::kStride * sizeof(float2) +
                      size_t(L::kVPB) * L::QP * sizeof(double2) +
                      size_t(L::kVPB) * L::kWPV * (sizeof(double) + 3 * sizeof(float)) + size_t(h) * sizeof(int);
  const bool stack = a.slices > 1;
  auto* kern = stack ? power_kernel<L, true> : power_kernel<L, false>;
  set_smem_limit(reinterpret_cast<const void*>(kern), smem);
  int per_sm = 0;
  SKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::kThreads, smem));
  const i64 tiles = (a.n + L::kVPB - 1) / L::kVPB * (a.slices > 1 ? a.slices : 1);
  // (one CTA per SM for a stack, leaving room for the multislice producer's kernels,
  // measured slower: C3 56.4 against 54.5 ms)
  const i64 blocks = std::min<i64>(tiles, i64(std::max(per_sm, 1)) * ctx->sm_count);
  kern<<<unsigned(blocks), L::kThreads, smem, ctx->stream>>>(a, tm_hi, tm_lo, tt, tile_rows);
  ++ctx->launches;
  SKB_LAUNCH("power_kernel");
}

}  // namespace

void power_iteration(sk_ctx* ctx, const PowerArgs& a) {
  if (a.n <= 0) return;
  // One matrix row per thread, Q fixed at compile time for the BASELINE
  // channel counts.  Q = 32: one accumulator pair per row (ptxas then rotates
  // two v quads; measured C2 0.973 -> 0.942 ms, C4 5.81 -> 5.52 ms against
  // two pairs).  Q = 64: the tiled matvec (4 x 16 blocks, C5 20.4 -> 18.5 ms
  // against one row per thread).  Measured and dropped: two rows per thread
  // (three 128-thread blocks, 1.12 vs 0.95 ms on C2), one 256-thread block
  // per SM, deeper v prefetch, the tiled matvec for Q = 32.
  if (a.q <= 4)
    launch<Layout<4, 1, 256, 2>>(ctx, a);
  else if (a.q == 8)
    launch<Layout<8, 1, 256, 2, 0, 4, 8>>(ctx, a);
  else if (a.q <= 8)
    launch<Layout<8, 1, 256, 2>>(ctx, a);
  else if (a.q <= 16)
    launch<Layout<16, 1, 256, 2>>(ctx, a);
  else if (a.q == 32)
    launch<Layout<32, 1, 256, 2, 1, 4, 32>>(ctx, a);
  else if (a.q <= 32)
    launch<Layout<32, 1, 256, 2, 2, 4>>(ctx, a);
  else if (a.q == 64)
    launch<Layout<64, 1, 256, 1, 2, 4, 64, 1>>(ctx, a);
  else if (a.q <= 64)
    launch<Layout<64, 1, 256, 1>>(ctx, a);
  else
    power_iteration_wide(ctx, a);  // any Q the shared memory holds (sk_power_wide.cu)
}

}  // namespace skb
