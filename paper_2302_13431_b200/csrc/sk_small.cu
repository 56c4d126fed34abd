// Small dense FP64 product of the subspace nullspace solver (K2):
//
//  * cross_gram:  H = X^H Y for tall-skinny X, Y (n x b, b <= 256), as a
//    deterministic two-phase reduction (row-chunk partials, then a fixed-order
//    sum).  Used for CholQR's X^H X and for the Rayleigh-Ritz projection
//    wherever the b = 64 cluster kernels of sk_cholqr.cu do not apply
//    (n < 1024 or b != 64).
//
// (Round 1 also measured own one-CTA Cholesky variants - lazy, blocked,
// with the inverse, lane-pair and row TRSMs - against cuSOLVER POTRF +
// cuBLAS TRSM for these blocks; the library pair won once CUDA graphs hid
// its host cost, and the b = 64 path moved to sk_cholqr.cu.  DESIGN.md §4.)
#include "sk_internal.h"

#include <cstdio>
#include <cstdlib>

namespace skb {

namespace {

__device__ __forceinline__ double2 cfma_conj(double2 acc, double2 a, double2 b) {  // acc + conj(a) * b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}

constexpr int kTile = 32;
constexpr int kRows = 32;  // rows staged per step

// partial[chunk][j][i] (col-major b x b) = sum_{r in chunk} conj(X[r,i]) * Y[r,j]
__global__ void __launch_bounds__(256) cross_gram_partial_kernel(const double2* __restrict__ x, const double2* __restrict__ y,
                                                                 i64 n, int b, i64 rows_per_chunk,
                                                                 double2* __restrict__ partial) {
  __shared__ double2 xs[kRows][kTile + 1];
  __shared__ double2 ys[kRows][kTile + 1];
  const int tiles = (b + kTile - 1) / kTile;
  const int ti = blockIdx.x % tiles, tj = blockIdx.x / tiles;
  const i64 chunk = blockIdx.y;
  const i64 r0 = chunk * rows_per_chunk, r1 = min(n, r0 + rows_per_chunk);
  const int tx = threadIdx.x % kTile, ty = threadIdx.x / kTile;  // 32 x 8
  double2 acc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k] = make_double2(0.0, 0.0);
  constexpr int kPerThread = kRows * kTile / 256;  // 4 elements of each operand per thread and step
  for (i64 rs = r0; rs < r1; rs += kRows) {
    double2 xv_[kPerThread], yv_[kPerThread];  // all loads in flight before the shared stores
#pragma unroll
    for (int u = 0; u < kPerThread; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int rr = e % kRows, cc = e / kRows;  // lanes along rows: X is column-major (coalesced)
      const i64 r = rs + rr;
      const int ci = ti * kTile + cc, cj = tj * kTile + cc;
      xv_[u] = (r < r1 && ci < b) ? x[r + i64(ci) * n] : make_double2(0.0, 0.0);
      yv_[u] = (r < r1 && cj < b) ? y[r + i64(cj) * n] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPerThread; ++u) {
      const int e = threadIdx.x + 256 * u;
      xs[e % kRows][e / kRows] = xv_[u];
      ys[e % kRows][e / kRows] = yv_[u];
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < kRows; ++rr) {
      const double2 xv = xs[rr][tx];
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = cfma_conj(acc[k], xv, ys[rr][ty + 8 * k]);
    }
  }
  const int i = ti * kTile + tx;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = tj * kTile + ty + 8 * k;
    if (i < b && j < b) partial[chunk * b * b + i64(j) * b + i] = acc[k];
  }
}

__global__ void reduce_partials_kernel(const double2* __restrict__ partial, int chunks, int bb,
                                       double2* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < bb; e += gridDim.x * blockDim.x) {
    // fixed-order sum, eight loads in flight (the chunk order is the same for every run)
    double2 s = make_double2(0.0, 0.0);
    int c = 0;
    for (; c + 8 <= chunks; c += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = partial[i64(c + u) * bb + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        s.x += v[u].x;
        s.y += v[u].y;
      }
    }
    for (; c < chunks; ++c) {
      const double2 v = partial[i64(c) * bb + e];
      s.x += v.x;
      s.y += v.y;
    }
    out[e] = s;
  }
}

 // packed lower, i >= j

}  // namespace

void cross_gram(sk_ctx* ctx, const double2* x, const double2* y, i64 n, int b, double2* out) {
  const int tiles = (b + kTile - 1) / kTile;
  // ~1 wave of CTAs over the SMs
  i64 chunks = std::max<i64>(1, i64(ctx->sm_count) / (tiles * tiles));
  i64 rows = (n + chunks - 1) / chunks;
  rows = ((rows + kRows - 1) / kRows) * kRows;
  chunks = (n + rows - 1) / rows;
  double2* partial = ctx->arena.get<double2>("ss:partial", chunks * b * b);
  cross_gram_partial_kernel<<<dim3(unsigned(tiles * tiles), unsigned(chunks)), 256, 0, ctx->stream>>>(x, y, n, b, rows,
                                                                                                       partial);
  ++ctx->launches;
  SKB_LAUNCH("cross_gram_partial");
  reduce_partials_kernel<<<unsigned((b * b + 255) / 256), 256, 0, ctx->stream>>>(partial, int(chunks), b * b, out);
  ++ctx->launches;
  SKB_LAUNCH("reduce_partials");
}

}  // namespace skb
