// K3 — G(x) lag expansion (spatial_gram.cpp:125-138) in FP64.
//
// G_pq(x) = sum_l k_pq[l] exp(-i 2 pi l . x) over the (4 tau + 1)^D lag box,
// evaluated separably axis by axis (last axis first).  Lags are symmetric
// (l in [-H, H], H = 2 tau), so each output is
//   x_0 + sum_{l=1..H} [ c_l (x_l + x_-l) + i s_l (x_l - x_-l) ],
// (c, s) = (cos, -sin)(2 pi l (j - j0) / N): half the MACs of a plain DFT.
//
// Arithmetic is FP64 and the final stage writes G as an fp32 value plus a
// bf16 residual (hi = fl32(G), lo = bf16(G - hi): 12 bytes per packed entry,
// G known to 2^-33 |G|): K4 iterates on hi alone (FP32, registers) and
// evaluates the Rayleigh quotient on hi + lo, so per-voxel eigenvalues stay
// accurate even where lambda ~ 1e-4.
//
//  * expand_row: stage along an axis with small inner extent (always the last
//    axis): a block stages RB rows' (S, D) in shared memory and each thread
//    owns one output index j with its (c, s) row in registers.
//  * expand_col: inner >= 32: a warp owns 32 consecutive inner indices, each
//    thread keeps its column's (S, D) in registers and sweeps all output rows
//    with the (c, s) table broadcast from shared memory (256-byte stores).
#include "sk_internal.h"

#include <cstdlib>
#include <string>

namespace skb {

namespace {

constexpr int kRB = 8;       // rows per expand_row block
constexpr int kColRows = 32; // table rows staged per chunk in expand_col

__device__ __forceinline__ void store_out(double2 v, double2* out64, float2* hi, lo2* lo, i64 idx) {
  if (out64) {
    out64[idx] = v;
  } else {
    const float hx = float(v.x), hy = float(v.y);
    hi[idx] = make_float2(hx, hy);
    lo[idx] = lo_pack(v.x - double(hx), v.y - double(hy));
  }
}

template <int H>
__global__ void __launch_bounds__(256) expand_row_kernel(const double2* __restrict__ in, i64 rows, i64 inner, int N,
                                                         const double2* __restrict__ cs, double2* out64, float2* hi,
                                                         lo2* lo) {
  constexpr int L = 2 * H + 1;
  __shared__ double2 sS[kRB][H + 1], sD[kRB][H + 1];  // [row][0] of sS holds x_0
  const i64 r0 = i64(blockIdx.x) * kRB;
  for (int e = threadIdx.x; e < kRB * (H + 1); e += blockDim.x) {
    const int r = e / (H + 1), l = e % (H + 1);
    const i64 row = r0 + r;
    double2 s = make_double2(0.0, 0.0), d = make_double2(0.0, 0.0);
    if (row < rows) {
      const i64 b = row / inner, i = row % inner;
      if (l == 0) {
        s = in[(b * L + H) * inner + i];
      } else {
        const double2 xp = in[(b * L + H + l) * inner + i], xm = in[(b * L + H - l) * inner + i];
        s = make_double2(xp.x + xm.x, xp.y + xm.y);
        d = make_double2(xp.x - xm.x, xp.y - xm.y);
      }
    }
    sS[r][l] = s;
    sD[r][l] = d;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    double2 t[H > 0 ? H : 1];
#pragma unroll
    for (int l = 0; l < H; ++l) t[l] = cs[i64(j) * H + l];
    for (int r = 0; r < kRB; ++r) {
      const i64 row = r0 + r;
      if (row >= rows) break;
      double ax = 0.0, ay = 0.0;
#pragma unroll
      for (int l = 0; l < H; ++l) {
        const double2 S = sS[r][l + 1], D = sD[r][l + 1];
        ax = fma(t[l].x, S.x, ax);
        ax = fma(-t[l].y, D.y, ax);
        ay = fma(t[l].x, S.y, ay);
        ay = fma(t[l].y, D.x, ay);
      }
      const double2 x0 = sS[r][0];
      const i64 b = row / inner, i = row % inner;
      store_out(make_double2(x0.x + ax, x0.y + ay), out64, hi, lo, (b * N + j) * inner + i);
    }
  }
}

// FULL: the whole (c, s) table (N x H) is staged once per CTA (dynamic shared
// memory, no per-chunk barriers); otherwise kColRows rows at a time.
template <int H, bool FULL>
__global__ void __launch_bounds__(256) expand_col_kernel(const double2* __restrict__ in, i64 inner, int N, int jc,
                                                         const double2* __restrict__ cs, double2* out64, float2* hi,
                                                         lo2* lo) {
  constexpr int L = 2 * H + 1;
  __shared__ __align__(16) double2 tab_chunk[FULL ? 1 : kColRows * (H > 0 ? H : 1)];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* tab = FULL ? reinterpret_cast<double2*>(smem_raw) : tab_chunk;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const i64 nchunk = (inner + 31) / 32;
  const i64 b = i64(blockIdx.x) / nchunk;
  const i64 i = (i64(blockIdx.x) % nchunk) * 32 + tx;
  const bool live = i < inner;
  double2 S[H > 0 ? H : 1], D[H > 0 ? H : 1], x0 = make_double2(0.0, 0.0);
  if (live) x0 = in[(b * L + H) * inner + i];
#pragma unroll
  for (int l = 0; l < H; ++l) {
    double2 xp = make_double2(0.0, 0.0), xm = make_double2(0.0, 0.0);
    if (live) {
      xp = in[(b * L + H + 1 + l) * inner + i];
      xm = in[(b * L + H - 1 - l) * inner + i];
    }
    S[l] = make_double2(xp.x + xm.x, xp.y + xm.y);
    D[l] = make_double2(xp.x - xm.x, xp.y - xm.y);
  }
  if constexpr (FULL) {
    for (int e = ty * 32 + tx; e < N * H; e += 256) tab[e] = cs[e];
    __syncthreads();
  }
  for (int j_begin = 0; j_begin < (FULL ? 1 : N); j_begin += kColRows) {
    const int j_count = min(kColRows, N - j_begin);
    if constexpr (!FULL) {
      __syncthreads();
      for (int e = ty * 32 + tx; e < kColRows * H; e += 256) {
        const int jj = e / H, l = e % H;
        tab[e] = jj < j_count ? cs[i64(j_begin + jj) * H + l] : make_double2(0.0, 0.0);
      }
      __syncthreads();
    }
    if (!live) continue;
    if constexpr (FULL) {
      // Mirrored pairs: rows jc + k and jc - k share c_l and negate s_l, so
      // A = sum c_l S_l and B = i sum s_l D_l give both outputs (A + B, A - B)
      // for half the FP64 MACs.
      // jc: the grid centre relative to the first output row (a z-slab may
      // start above or end below it).  Items: rows jp >= jc (mirror 2 jc - jp
      // when it is another output row), then the rows below jc whose mirror
      // lies past the last output row, alone.
      const int p0 = max(jc, 0), P = max(0, N - p0);
      const int S1 = jc > 0 ? max(0, min(min(jc, N), 2 * jc - N + 1)) : 0;
      for (int t = ty; t < P + S1; t += 8) {
        const bool single = t >= P;
        const int jp = single ? t - P : p0 + t;
        const int jm = single ? -1 : 2 * jc - jp;
        const double2* row = tab + jp * H;
        double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
#pragma unroll
        for (int l = 0; l < H; ++l) {
          const double2 tcs = row[l];
          ax = fma(tcs.x, S[l].x, ax);
          ay = fma(tcs.x, S[l].y, ay);
          bx = fma(-tcs.y, D[l].y, bx);
          by = fma(tcs.y, D[l].x, by);
        }
        store_out(make_double2(x0.x + (ax + bx), x0.y + (ay + by)), out64, hi, lo, (b * N + jp) * inner + i);
        if (jm >= 0 && jm < N && jm != jp)
          store_out(make_double2(x0.x + (ax - bx), x0.y + (ay - by)), out64, hi, lo, (b * N + jm) * inner + i);
      }
    } else {
      for (int jj = ty; jj < j_count; jj += 8) {
        const double2* row = tab + jj * H;
        double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
#pragma unroll
        for (int l = 0; l < H; l += 2) {
          const double2 t0 = row[l], t1 = row[l + 1];
          ax = fma(t0.x, S[l].x, ax);
          ax = fma(-t0.y, D[l].y, ax);
          ay = fma(t0.x, S[l].y, ay);
          ay = fma(t0.y, D[l].x, ay);
          bx = fma(t1.x, S[l + 1].x, bx);
          bx = fma(-t1.y, D[l + 1].y, bx);
          by = fma(t1.x, S[l + 1].y, by);
          by = fma(t1.y, D[l + 1].x, by);
        }
        store_out(make_double2(x0.x + (ax + bx), x0.y + (ay + by)), out64, hi, lo,
                  (b * N + j_begin + jj) * inner + i);
      }
    }
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  const unsigned d = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(bytes) : "memory");
}

// Persistent form of the FULL expand_col: the (c, s) table is staged once per
// CTA, and the next column block's 2H+1 input rows are prefetched into shared
// memory with cp.async while the current block is expanded (no per-CTA load
// bubble, no table reloads).  CPT columns per thread (a block is 32 CPT
// columns wide): every (c, s) tap is a warp-wide shared-memory broadcast
// feeding 4 CPT DFMAs; two columns per thread pay only for long tap rows
// (launch_stage).
template <int H, int CPT>
__global__ void __launch_bounds__(256) expand_col_persist_kernel(const double2* __restrict__ in, i64 inner, int N,
                                                                 int jc, int items, i64 nblocks,
                                                                 const double2* __restrict__ cs, double2* out64,
                                                                 float2* hi, lo2* lo) {
  constexpr int L = 2 * H + 1, W = 32 * CPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* tab = reinterpret_cast<double2*>(smem_raw);  // [items][H] (items = P + S1, computed by the host)
  double2* xin = tab + items * H;                       // [2][L][W]
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const i64 nchunk = (inner + W - 1) / W;
  auto issue = [&](i64 cb, int buf) {
    const i64 b = cb / nchunk, ib = (cb % nchunk) * W;
    for (int e = tid; e < L * W; e += 256) {
      const int l = e / W, c = e % W;
      const bool ok = ib + c < inner;
      cp_async16(xin + (buf * L + l) * W + c, in + (b * L + l) * inner + (ok ? ib + c : 0), ok ? 16 : 0);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  i64 cb = blockIdx.x;
  if (cb < nblocks) issue(cb, 0);
  const int p0 = max(jc, 0), P = max(0, N - p0);
  const int S1 = jc > 0 ? max(0, min(min(jc, N), 2 * jc - N + 1)) : 0;
  SKB_DCHECK(blockDim.x == 32 && blockDim.y == 8 && P + S1 <= items);  // the host sized tab for `items` rows
  // table rows in item order: item t < P is row p0 + t, item P + s is row s
  for (int e = tid; e < (P + S1) * H; e += 256) {
    const int t = e / H, l = e % H;
    tab[e] = cs[(t < P ? p0 + t : t - P) * H + l];
  }
  for (int buf = 0; cb < nblocks; cb += gridDim.x, buf ^= 1) {
    const i64 next = cb + gridDim.x;
    if (next < nblocks) {
      issue(next, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();  // xin[buf] (and, on the first pass, the table) visible to all
    const i64 b = cb / nchunk, i0 = (cb % nchunk) * W + tx;  // the thread's columns: i0 + 32 k
    double2 x0[CPT], S[CPT][H > 0 ? H : 1], D[CPT][H > 0 ? H : 1];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const double2* xb = xin + buf * L * W + tx + 32 * k;
      x0[k] = xb[H * W];
#pragma unroll
      for (int l = 0; l < H; ++l) {
        const double2 xp = xb[(H + 1 + l) * W], xm = xb[(H - 1 - l) * W];
        S[k][l] = make_double2(xp.x + xm.x, xp.y + xm.y);
        D[k][l] = make_double2(xp.x - xm.x, xp.y - xm.y);
      }
    }
    __syncthreads();  // every thread has its columns: xin[buf] may be refilled (issued next iteration)
    if (i0 >= inner) continue;
    for (int t = ty; t < P + S1; t += 8) {
      const bool single = t >= P;
      const int jp = single ? t - P : p0 + t;
      const int jm = single ? -1 : 2 * jc - jp;
      const double2* row = tab + t * H;
      double ax[CPT], ay[CPT], bx[CPT], by[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) ax[k] = ay[k] = bx[k] = by[k] = 0.0;
#pragma unroll
      for (int l = 0; l < H; ++l) {
        const double2 tcs = row[l];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          ax[k] = fma(tcs.x, S[k][l].x, ax[k]);
          ay[k] = fma(tcs.x, S[k][l].y, ay[k]);
          bx[k] = fma(-tcs.y, D[k][l].y, bx[k]);
          by[k] = fma(tcs.y, D[k][l].x, by[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const i64 i = i0 + 32 * k;
        if (i >= inner) continue;
        store_out(make_double2(x0[k].x + (ax[k] + bx[k]), x0[k].y + (ay[k] + by[k])), out64, hi, lo,
                  (b * N + jp) * inner + i);
        if (jm >= 0 && jm < N && jm != jp)
          store_out(make_double2(x0[k].x + (ax[k] - bx[k]), x0[k].y + (ay[k] - by[k])), out64, hi, lo,
                    (b * N + jm) * inner + i);
      }
    }
  }
}

template <int H>
void launch_stage(sk_ctx* ctx, const double2* in, i64 batch, i64 inner, int N, int jc, const double2* cs,
                  double2* out64, float2* hi, lo2* lo) {
  if (inner >= 32) {
    const i64 gx = (inner + 31) / 32 * batch;
    if (gx > 0x7fffffffLL) fail(SK_ERR_UNSUPPORTED, "expand: grid too large");
    const size_t full_bytes = size_t(N) * (H > 0 ? H : 1) * sizeof(double2);
    // items: output rows at or past the centre (with their mirrors) plus the
    // rows below it whose mirror lies past the last output row (kernel rules)
    const int p0 = std::max(jc, 0), P = std::max(0, N - p0);
    const int S1 = jc > 0 ? std::max(0, std::min(std::min(jc, N), 2 * jc - N + 1)) : 0;
    const int items = P + S1;
    const size_t tbytes = size_t(items) * (H > 0 ? H : 1) * sizeof(double2);
    const size_t pbytes = tbytes + size_t(2 * (2 * H + 1) * 32) * sizeof(double2);
    const size_t pbytes2 = tbytes + size_t(2 * (2 * H + 1) * 64) * sizeof(double2);
    if (H >= 12 && inner % 64 == 0 && pbytes2 <= 200 * 1024) {
      // two columns per thread, each (c, s) broadcast feeding eight DFMAs, for the long tap
      // rows only: C5 (H = 12) field 3.19 -> 2.95 ms; with H <= 10 the halved occupancy costs
      // more than the broadcasts saved (C2 0.241 -> 0.258 ms, C4 2.49 -> 2.61 ms, C3 +6%)
      set_smem_limit(reinterpret_cast<const void*>(expand_col_persist_kernel<H, 2>), pbytes2);
      const i64 nblocks = inner / 64 * batch;
      int per_sm = 1;
      SKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expand_col_persist_kernel<H, 2>, 256, pbytes2));
      const unsigned grid = unsigned(std::min<i64>(nblocks, i64(std::max(per_sm, 1)) * ctx->sm_count));
      expand_col_persist_kernel<H, 2><<<grid, dim3{32, 8}, pbytes2, ctx->stream>>>(in, inner, N, jc, items, nblocks,
                                                                                 cs, out64, hi, lo);
    } else if (H > 0 && pbytes <= 110 * 1024) {  // persistent, two CTAs per SM (C2 last stage 218 -> 146 us)
      set_smem_limit(reinterpret_cast<const void*>(expand_col_persist_kernel<H, 1>), pbytes);
      const i64 nblocks = gx;
      const unsigned grid = unsigned(std::min<i64>(nblocks, 2 * ctx->sm_count));
      expand_col_persist_kernel<H, 1><<<grid, dim3{32, 8}, pbytes, ctx->stream>>>(in, inner, N, jc, items, nblocks,
                                                                                 cs, out64, hi, lo);
    } else if (full_bytes <= 110 * 1024) {  // two CTAs per SM still fit
      set_smem_limit(reinterpret_cast<const void*>(expand_col_kernel<H, true>), full_bytes);
      expand_col_kernel<H, true><<<dim3{unsigned(gx)}, dim3{32, 8}, full_bytes, ctx->stream>>>(in, inner, N, jc, cs,
                                                                                               out64, hi, lo);
    } else {
      expand_col_kernel<H, false><<<dim3{unsigned(gx)}, dim3{32, 8}, 0, ctx->stream>>>(in, inner, N, jc, cs, out64,
                                                                                        hi, lo);
    }
  } else {
    const i64 rows = batch * inner;
    const int threads = N >= 256 ? 256 : (N >= 128 ? 128 : 64);
    expand_row_kernel<H><<<unsigned((rows + kRB - 1) / kRB), threads, 0, ctx->stream>>>(in, rows, inner, N, cs, out64,
                                                                                          hi, lo);
  }
  ++ctx->launches;
  SKB_LAUNCH("expand stage");
}

}  // namespace

void expand_stage_f64(sk_ctx* ctx, const double2* in, i64 batch, i64 inner, int H, int N, int jc, const double2* cs,
                      double2* out64, float2* hi, lo2* lo) {
  if (batch <= 0 || N <= 0 || inner <= 0) return;
  switch (H) {
    case 0: launch_stage<0>(ctx, in, batch, inner, N, jc, cs, out64, hi, lo); break;
    case 2: launch_stage<2>(ctx, in, batch, inner, N, jc, cs, out64, hi, lo); break;
    case 4: launch_stage<4>(ctx, in, batch, inner, N, jc, cs, out64, hi, lo); break;
    case 6: launch_stage<6>(ctx, in, batch, inner, N, jc, cs, out64, hi, lo); break;
    case 8: launch_stage<8>(ctx, in, batch, inner, N, jc, cs, out64, hi, lo); break;
    case 10: launch_stage<10>(ctx, in, batch, inner, N, jc, cs, out64, hi, lo); break;
    case 12: launch_stage<12>(ctx, in, batch, inner, N, jc, cs, out64, hi, lo); break;
    case 14: launch_stage<14>(ctx, in, batch, inner, N, jc, cs, out64, hi, lo); break;
    default: fail(SK_ERR_UNSUPPORTED, "G(x) expansion: kernel radius > 7 is outside the B200 path");
  }
}

}  // namespace skb
