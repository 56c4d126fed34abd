// Separable small-matrix transforms along one axis of a row-major volume:
//
//   out[b][j][i] = sum_a M[j][a] * in[b][a][i]        (M: N x L, complex64)
//
// Every centred transform on the hot path is one of these per axis, because
// the inputs are sparse boxes of a larger grid (the reference zero-pads and
// runs full FFTs): the Gram's channel spectra (calibration.cpp:96-109), the
// pruned inverse at the Gram lags, the G(x) lag-kernel expansion
// (spatial_gram.cpp:125-138), the apodised calibration recon (maps.cpp:141-159)
// and the periodic-sinc interpolation (maps.cpp:54-99).  The matrices are
// built in FP64 on the host (sk_runtime.cu) with exact integer phase
// reduction, so the device arithmetic is a plain complex GEMM-like contraction.
//
// Two mappings:
//  * column mode (inner >= 32): a warp owns 32 consecutive `i`; each thread
//    keeps its column's taps in registers and sweeps j; M rows come from
//    shared memory as warp-wide broadcasts.  Loads/stores are 256-byte
//    coalesced along i.
//  * row mode (inner < 32, e.g. the last axis): a block stages RB input rows
//    in shared memory, each thread owns output j and accumulates RB rows,
//    reading M^T[a][j] coalesced from global/L2.
#include "sk_internal.h"

namespace skb {

namespace {

__device__ __forceinline__ void cmac(float2& acc, float2 m, float2 x) {
  acc.x = fmaf(m.x, x.x, acc.x);
  acc.x = fmaf(-m.y, x.y, acc.x);
  acc.y = fmaf(m.x, x.y, acc.y);
  acc.y = fmaf(m.y, x.x, acc.y);
}

constexpr int kColJ = 64;  // output rows per column-mode block

template <int LT>
__global__ void __launch_bounds__(256) axis_col_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                       const float2* __restrict__ M, int L, int N, i64 inner,
                                                       int a0, int lt, bool accumulate) {
  __shared__ __align__(16) float2 sm[kColJ * LT];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const i64 nchunk = (inner + 31) / 32;
  const i64 b = i64(blockIdx.x) / nchunk;
  const i64 i = (i64(blockIdx.x) % nchunk) * 32 + tx;
  const int j_begin = blockIdx.y * kColJ;
  const int j_count = min(kColJ, N - j_begin);
  // Stage the M tile (j_count rows x lt taps), zero-padded to LT.
  for (int e = ty * 32 + tx; e < kColJ * LT; e += 256) {
    const int jj = e / LT, t = e % LT;
    sm[e] = (jj < j_count && t < lt) ? M[i64(j_begin + jj) * L + a0 + t] : make_float2(0.f, 0.f);
  }
  float2 x[LT];
  const bool live = i < inner;
#pragma unroll
  for (int t = 0; t < LT; ++t)
    x[t] = (live && t < lt) ? in[(b * L + a0 + t) * inner + i] : make_float2(0.f, 0.f);
  __syncthreads();
  if (!live) return;
  for (int jj = ty; jj < j_count; jj += 8) {
    const float4* row = reinterpret_cast<const float4*>(sm + jj * LT);
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < LT; t += 2) {
      const float4 m2 = row[t / 2];
      cmac(acc0, make_float2(m2.x, m2.y), x[t]);
      cmac(acc1, make_float2(m2.z, m2.w), x[t + 1]);
    }
    float2 acc = make_float2(acc0.x + acc1.x, acc0.y + acc1.y);
    float2* dst = out + (b * N + j_begin + jj) * inner + i;
    if (accumulate) {
      const float2 prev = *dst;
      acc.x += prev.x;
      acc.y += prev.y;
    }
    *dst = acc;
  }
}

constexpr int kRowRB = 16;   // input rows per row-mode block
constexpr int kRowTap = 64;  // taps staged per chunk

__global__ void __launch_bounds__(256) axis_row_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                       const float2* __restrict__ Mt, i64 rows, int L, int N,
                                                       i64 inner) {
  __shared__ __align__(16) float2 xs[kRowTap][kRowRB];  // [tap][row]
  const i64 r0 = i64(blockIdx.x) * kRowRB;
  for (int j0 = 0; j0 < N; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    float2 acc[kRowRB];
#pragma unroll
    for (int r = 0; r < kRowRB; ++r) acc[r] = make_float2(0.f, 0.f);
    for (int a0 = 0; a0 < L; a0 += kRowTap) {
      const int lt = min(kRowTap, L - a0);
      __syncthreads();
      for (int e = threadIdx.x; e < kRowTap * kRowRB; e += blockDim.x) {
        const int r = e / kRowTap, t = e % kRowTap;  // consecutive threads walk taps (contiguous for inner == 1)
        const i64 row = r0 + r;
        float2 v = make_float2(0.f, 0.f);
        if (row < rows && t < lt) {
          const i64 bb = row / inner, ii = row % inner;
          v = in[(bb * L + a0 + t) * inner + ii];
        }
        xs[t][r] = v;
      }
      __syncthreads();
      if (j < N) {
        for (int t = 0; t < lt; ++t) {
          const float2 m = Mt[i64(a0 + t) * N + j];
          const float4* xr = reinterpret_cast<const float4*>(&xs[t][0]);
#pragma unroll
          for (int r = 0; r < kRowRB; r += 2) {
            const float4 x2 = xr[r / 2];
            cmac(acc[r], m, make_float2(x2.x, x2.y));
            cmac(acc[r + 1], m, make_float2(x2.z, x2.w));
          }
        }
      }
    }
    if (j < N) {
#pragma unroll
      for (int r = 0; r < kRowRB; ++r) {
        const i64 row = r0 + r;
        if (row < rows) {
          const i64 bb = row / inner, ii = row % inner;
          out[(bb * N + j) * inner + ii] = acc[r];
        }
      }
    }
  }
}

// Symmetric-tap centred DFT along an axis (the G(x) lag expansion,
// spatial_gram.cpp:125-138): taps a = 0..2H hold lags l = a - H, and
//   out[b][j][i] = x_0 + sum_{l=1..H} [ c_jl (x_l + x_-l) + i s_jl (x_l - x_-l) ]
// with (c, s) = (cos, sign*sin)(2 pi l (j - j0) / N).  Pairing l with -l
// halves the FMAs of the generic contraction.  A thread owns one (b, i)
// column: it forms S_l = x_l + x_-l and D_l = x_l - x_-l once in registers,
// then sweeps its block's j range with the (c, s) table broadcast from
// shared memory; stores are 256-byte coalesced along i.
template <int H>
__global__ void __launch_bounds__(256) axis_symdft_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                          const float2* __restrict__ cs, int N, i64 inner) {
  // Each thread owns TWO columns (i, i + 32): every table entry read from
  // shared memory feeds 8 FMAs.
  __shared__ __align__(16) float2 tab[kColJ * H];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const i64 nchunk = (inner + 63) / 64;
  const i64 b = i64(blockIdx.x) / nchunk;
  const i64 i0 = (i64(blockIdx.x) % nchunk) * 64 + tx;
  constexpr int L = 2 * H + 1;
  float2 S[2][H], D[2][H], x0[2];
  bool live[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const i64 i = i0 + 32 * u;
    live[u] = i < inner;
    x0[u] = live[u] ? in[(b * L + H) * inner + i] : make_float2(0.f, 0.f);
#pragma unroll
    for (int l = 0; l < H; ++l) {
      float2 xp = make_float2(0.f, 0.f), xm = make_float2(0.f, 0.f);
      if (live[u]) {
        xp = in[(b * L + H + 1 + l) * inner + i];
        xm = in[(b * L + H - 1 - l) * inner + i];
      }
      S[u][l] = make_float2(xp.x + xm.x, xp.y + xm.y);
      D[u][l] = make_float2(xp.x - xm.x, xp.y - xm.y);
    }
  }
  float2* dst = out + b * N * inner + i0;
  // The block sweeps every output row; the (c, s) table streams through
  // shared memory in kColJ-row chunks.
  for (int j_begin = 0; j_begin < N; j_begin += kColJ) {
    const int j_count = min(kColJ, N - j_begin);
    __syncthreads();
    for (int e = ty * 32 + tx; e < kColJ * H; e += 256) {
      const int jj = e / H, l = e % H;
      tab[e] = jj < j_count ? cs[i64(j_begin + jj) * H + l] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int jj = ty; jj < j_count; jj += 8) {
      const float4* row = reinterpret_cast<const float4*>(tab + jj * H);
      float ax[2], ay[2], bx[2], by[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        ax[u] = x0[u].x;
        ay[u] = x0[u].y;
        bx[u] = 0.f;
        by[u] = 0.f;
      }
#pragma unroll
      for (int l = 0; l < H; l += 2) {
        const float4 t = row[l / 2];  // (c_l, s_l, c_l+1, s_l+1)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          ax[u] = fmaf(t.x, S[u][l].x, ax[u]);
          ax[u] = fmaf(-t.y, D[u][l].y, ax[u]);
          ay[u] = fmaf(t.x, S[u][l].y, ay[u]);
          ay[u] = fmaf(t.y, D[u][l].x, ay[u]);
          bx[u] = fmaf(t.z, S[u][l + 1].x, bx[u]);
          bx[u] = fmaf(-t.w, D[u][l + 1].y, bx[u]);
          by[u] = fmaf(t.z, S[u][l + 1].y, by[u]);
          by[u] = fmaf(t.w, D[u][l + 1].x, by[u]);
        }
      }
      float2* d = dst + i64(j_begin + jj) * inner;
      if (live[0]) d[0] = make_float2(ax[0] + bx[0], ay[0] + by[0]);
      if (live[1]) d[32] = make_float2(ax[1] + bx[1], ay[1] + by[1]);
    }
  }
}

}  // namespace

namespace {

// Both axes of a 2-D separable transform in one CTA per batch item (the
// Gram's channel spectra: E0 x E1 calibration -> P0 x P1 pad): the input, the
// two matrices and the axis-1 result stay in shared memory, so the two
// axis launches and the round trip of the intermediate through global memory
// are gone (K1 stage: C2 0.109 -> 0.098 ms, C1 0.047 -> 0.027 ms).
//   tmp[a0][j1] = sum_a1 M1[j1][a1] in[a0][a1];  out[j0][j1] = sum_a0 M0[j0][a0] tmp[a0][j1]
__global__ void __launch_bounds__(256) sep2d_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                    const float2* __restrict__ M0, const float2* __restrict__ M1,
                                                    int E0, int E1, int P0, int P1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* xs = reinterpret_cast<float2*>(smem_raw);  // [E0][E1]
  float2* tmp = xs + E0 * E1;                         // [E0][P1]
  float2* m1 = tmp + E0 * P1;                         // [E1][P1] (transposed: lanes run along j1)
  float2* m0 = m1 + P1 * E1;                          // [P0][E0]
  const float2* src = in + i64(blockIdx.x) * E0 * E1;
  float2* dst = out + i64(blockIdx.x) * P0 * P1;
  for (int e = threadIdx.x; e < E0 * E1; e += blockDim.x) xs[e] = src[e];
  for (int e = threadIdx.x; e < P1 * E1; e += blockDim.x) m1[(e % E1) * P1 + e / E1] = M1[e];
  for (int e = threadIdx.x; e < P0 * E0; e += blockDim.x) m0[e] = M0[e];
  __syncthreads();
  for (int e = threadIdx.x; e < E0 * P1; e += blockDim.x) {
    const int a0 = e / P1, j1 = e % P1;
    float2 acc = make_float2(0.f, 0.f), acc2 = acc;
    const float2* mc = m1 + j1;
    const float2* xr = xs + a0 * E1;
    int a1 = 0;
    for (; a1 + 1 < E1; a1 += 2) {
      cmac(acc, mc[a1 * P1], xr[a1]);
      cmac(acc2, mc[(a1 + 1) * P1], xr[a1 + 1]);
    }
    if (a1 < E1) cmac(acc, mc[a1 * P1], xr[a1]);
    tmp[e] = make_float2(acc.x + acc2.x, acc.y + acc2.y);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < P0 * P1; e += blockDim.x) {
    const int j0 = e / P1, j1 = e % P1;
    float2 acc = make_float2(0.f, 0.f), acc2 = acc;
    const float2* mr = m0 + j0 * E0;
    int a0 = 0;
    for (; a0 + 1 < E0; a0 += 2) {
      cmac(acc, mr[a0], tmp[a0 * P1 + j1]);
      cmac(acc2, mr[a0 + 1], tmp[(a0 + 1) * P1 + j1]);
    }
    if (a0 < E0) cmac(acc, mr[a0], tmp[a0 * P1 + j1]);
    dst[e] = make_float2(acc.x + acc2.x, acc.y + acc2.y);
  }
}

}  // namespace

size_t sep2d_smem(int E0, int E1, int P0, int P1) {
  return size_t(E0 * E1 + E0 * P1 + P1 * E1 + P0 * E0) * sizeof(float2);
}

void sep2d(sk_ctx* ctx, const float2* in, float2* out, i64 batch, int E0, int E1, int P0, int P1, const float2* M0,
           const float2* M1) {
  const size_t smem = sep2d_smem(E0, E1, P0, P1);
  set_smem_limit(reinterpret_cast<const void*>(sep2d_kernel), smem);
  sep2d_kernel<<<unsigned(batch), 256, smem, ctx->stream>>>(in, out, M0, M1, E0, E1, P0, P1);
  ++ctx->launches;
  SKB_LAUNCH("sep2d_kernel");
}

void apply_axis_symdft(sk_ctx* ctx, const float2* in, float2* out, const float2* cs, i64 batch, int H, int N,
                       i64 inner) {
  if (batch <= 0 || N <= 0 || inner <= 0) return;
  if (inner < 32 || H > 16 || (H & 1)) fail(9, "apply_axis_symdft: needs inner >= 32 and even H <= 16");
  const i64 gx = (inner + 63) / 64 * batch;
  if (gx > 0x7fffffffLL) fail(9, "apply_axis_symdft: grid too large");
  const dim3 grid{unsigned(gx)}, block{32, 8};
  switch (H) {
    case 2: axis_symdft_kernel<2><<<grid, block, 0, ctx->stream>>>(in, out, cs, N, inner); break;
    case 4: axis_symdft_kernel<4><<<grid, block, 0, ctx->stream>>>(in, out, cs, N, inner); break;
    case 6: axis_symdft_kernel<6><<<grid, block, 0, ctx->stream>>>(in, out, cs, N, inner); break;
    case 8: axis_symdft_kernel<8><<<grid, block, 0, ctx->stream>>>(in, out, cs, N, inner); break;
    case 10: axis_symdft_kernel<10><<<grid, block, 0, ctx->stream>>>(in, out, cs, N, inner); break;
    case 12: axis_symdft_kernel<12><<<grid, block, 0, ctx->stream>>>(in, out, cs, N, inner); break;
    case 14: axis_symdft_kernel<14><<<grid, block, 0, ctx->stream>>>(in, out, cs, N, inner); break;
    default: axis_symdft_kernel<16><<<grid, block, 0, ctx->stream>>>(in, out, cs, N, inner); break;
  }
  ++ctx->launches;
  SKB_LAUNCH("axis_symdft_kernel");
}

// Mt (L x N) is stored right after M (N x L) in the same allocation.
void apply_axis(sk_ctx* ctx, const float2* in, float2* out, const float2* M, i64 batch, int L, int N, i64 inner) {
  if (batch <= 0 || N <= 0 || inner <= 0) return;
  if (inner >= 32) {
    const dim3 block(32, 8);
    for (int a0 = 0; a0 < L; a0 += 64) {
      const int lt = std::min(64, L - a0);
      const i64 gx = (inner + 31) / 32 * batch;
      if (gx > 0x7fffffffLL) fail(9, "apply_axis: grid too large");
      const dim3 grid(unsigned(gx), unsigned((N + kColJ - 1) / kColJ));
      const bool acc = a0 > 0;
      if (lt <= 8)
        axis_col_kernel<8><<<grid, block, 0, ctx->stream>>>(in, out, M, L, N, inner, a0, lt, acc);
      else if (lt <= 16)
        axis_col_kernel<16><<<grid, block, 0, ctx->stream>>>(in, out, M, L, N, inner, a0, lt, acc);
      else if (lt <= 32)
        axis_col_kernel<32><<<grid, block, 0, ctx->stream>>>(in, out, M, L, N, inner, a0, lt, acc);
      else
        axis_col_kernel<64><<<grid, block, 0, ctx->stream>>>(in, out, M, L, N, inner, a0, lt, acc);
      ++ctx->launches;
      SKB_LAUNCH("axis_col_kernel");
    }
  } else {
    const i64 rows = batch * inner;
    const float2* Mt = M + i64(N) * L;
    const int threads = N >= 256 ? 256 : (N >= 128 ? 128 : 64);
    const i64 blocks = (rows + kRowRB - 1) / kRowRB;
    axis_row_kernel<<<unsigned(blocks), threads, 0, ctx->stream>>>(in, out, Mt, rows, L, N, inner);
    ++ctx->launches;
    SKB_LAUNCH("axis_row_kernel");
  }
}

}  // namespace skb
