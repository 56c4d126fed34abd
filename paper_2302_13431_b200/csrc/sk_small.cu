// Small dense FP64 kernels for the subspace nullspace solver (K2):
//
//  * cross_gram:  H = X^H Y for tall-skinny X, Y (n x b, b <= 128), as a
//    deterministic two-phase reduction (row-chunk partials, then a fixed-order
//    sum).  Used for CholQR's X^H X and for the Rayleigh-Ritz projection.
//  * chol_inv:    one CTA: S = L L^H (Cholesky, lower) and M = L^{-1}, both
//    packed in shared memory; writes M as a full column-major b x b matrix so
//    that V = Y M^H is one ZGEMM.  A non-positive pivot raises a device flag
//    (read at the next host synchronisation) instead of stopping the stream.
//
// These replace per-iteration cuBLAS HERK/TRSM + cuSOLVER POTRF calls whose
// launch and host-sync overhead dominated the stage at b ~ 96.
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
__device__ __forceinline__ double2 cfma_conj_rev(double2 acc, double2 a, double2 b) {  // acc + a * conj(b)
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y);
  acc.y = fma(-a.x, b.y, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {  // acc + a * b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
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

__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }  // packed lower, i >= j

// One CTA.  S (b x b col-major, Hermitian; lower used) -> Minv (b x b col-major,
// lower = L^{-1}, upper zero).  *flag |= 1 on a non-positive pivot.
__global__ void __launch_bounds__(256) chol_inv_kernel(const double2* __restrict__ s, int b,
                                                       double2* __restrict__ minv, int* __restrict__ flag) {
  extern __shared__ double2 sm[];
  double2* L = sm;                    // packed lower b(b+1)/2
  double2* M = sm + b * (b + 1) / 2;  // packed lower b(b+1)/2
  __shared__ double pivot;
  const int tid = threadIdx.x;
  for (int e = tid; e < b * (b + 1) / 2; e += blockDim.x) {
    int i = int((sqrt(8.0 * e + 1.0) - 1.0) / 2.0);
    while (pk(i, 0) > e) --i;
    while (pk(i + 1, 0) <= e) ++i;
    const int j = e - pk(i, 0);
    L[e] = s[i + i64(j) * b];
  }
  __syncthreads();
  // Right-looking Cholesky.
  for (int j = 0; j < b; ++j) {
    if (tid == 0) {
      double d = L[pk(j, j)].x;
      if (!(d > 0.0)) {
        atomicOr(flag, 1);
        d = 1.0;
      }
      pivot = sqrt(d);
      L[pk(j, j)] = make_double2(pivot, 0.0);
    }
    __syncthreads();
    const double inv = 1.0 / pivot;
    for (int i = j + 1 + tid; i < b; i += blockDim.x) {
      double2 v = L[pk(i, j)];
      L[pk(i, j)] = make_double2(v.x * inv, v.y * inv);
    }
    __syncthreads();
    // trailing update: A[i][k] -= L[i][j] * conj(L[k][j]) for j < k <= i
    const int m = b - j - 1;
    const int cnt = m * (m + 1) / 2;
    for (int e = tid; e < cnt; e += blockDim.x) {
      int ii = int((sqrt(8.0 * e + 1.0) - 1.0) / 2.0);
      while (ii * (ii + 1) / 2 > e) --ii;
      while ((ii + 1) * (ii + 2) / 2 <= e) ++ii;
      const int kk = e - ii * (ii + 1) / 2;
      const int i = j + 1 + ii, k = j + 1 + kk;
      const double2 lij = L[pk(i, j)], lkj = L[pk(k, j)];
      double2 a = L[pk(i, k)];
      // a -= lij * conj(lkj)
      a.x -= lij.x * lkj.x + lij.y * lkj.y;
      a.y -= lij.y * lkj.x - lij.x * lkj.y;
      L[pk(i, k)] = a;
    }
    __syncthreads();
  }
  // M = L^{-1}: columns are independent forward substitutions.
  for (int j = tid; j < b; j += blockDim.x) {
    M[pk(j, j)] = make_double2(1.0 / L[pk(j, j)].x, 0.0);
    for (int i = j + 1; i < b; ++i) {
      double2 acc = make_double2(0.0, 0.0);
      for (int k = j; k < i; ++k) acc = cfma(acc, L[pk(i, k)], M[pk(k, j)]);
      const double inv = 1.0 / L[pk(i, i)].x;
      M[pk(i, j)] = make_double2(-acc.x * inv, -acc.y * inv);
    }
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int j = e / b, i = e % b;
    minv[e] = i >= j ? M[pk(i, j)] : make_double2(0.0, 0.0);
  }
}

// One CTA of 32 x 32 threads: in-place right-looking Cholesky S = L L^H of a
// b x b Hermitian matrix held whole in shared memory (b <= 112).  Writes L
// (lower, column-major, leading dimension b) for a following TRSM.
__global__ void __launch_bounds__(1024) chol_kernel(const double2* __restrict__ s, int b, double2* __restrict__ l,
                                                    int* __restrict__ flag) {
  extern __shared__ double2 sm[];
  const int ld = b + 1;  // row-major A[i][k] at i*ld + k
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  __shared__ double piv;
  for (int e = tid; e < b * b; e += 1024) {
    const int k = e / b, i = e % b;  // coalesced read of column-major S(i,k)
    sm[i * ld + k] = s[e];
  }
  __syncthreads();
  (void)piv;
  constexpr int NB = 16;  // blocked right-looking: 16-wide panels
  for (int kb = 0; kb < b; kb += NB) {
    const int ke = min(b, kb + NB);
    // 1. unblocked factor of the diagonal block by warp 0
    if (tid < 32) {
      for (int j = kb; j < ke; ++j) {
        double d = sm[j * ld + j].x;
        if (!(d > 0.0)) {
          if (tid == 0) atomicOr(flag, 1);
          d = 1.0;
        }
        const double p = sqrt(d), inv = 1.0 / p;
        __syncwarp();
        if (tid == 0) sm[j * ld + j] = make_double2(p, 0.0);
        const int i = j + 1 + tid;
        if (i < ke) {
          const double2 v = sm[i * ld + j];
          sm[i * ld + j] = make_double2(v.x * inv, v.y * inv);
        }
        __syncwarp();
        if (i < ke) {
          const double2 lij = sm[i * ld + j];
          for (int k = j + 1; k <= i; ++k) {
            const double2 lkj = sm[k * ld + j];
            double2 a = sm[i * ld + k];
            a.x -= lij.x * lkj.x + lij.y * lkj.y;
            a.y -= lij.y * lkj.x - lij.x * lkj.y;
            sm[i * ld + k] = a;
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // 2. panel: rows below solve x L_blk^H = a (forward substitution per row)
    for (int i = ke + tid; i < b; i += 1024) {
      for (int j = kb; j < ke; ++j) {
        double2 a = sm[i * ld + j];
        for (int t = kb; t < j; ++t) {
          const double2 x = sm[i * ld + t], l = sm[j * ld + t];
          a.x -= x.x * l.x + x.y * l.y;  // a -= x * conj(l)
          a.y -= x.y * l.x - x.x * l.y;
        }
        const double inv = 1.0 / sm[j * ld + j].x;
        sm[i * ld + j] = make_double2(a.x * inv, a.y * inv);
      }
    }
    __syncthreads();
    // 3. trailing update A[i][k] -= sum_t L[i][t] conj(L[k][t]), ke <= k <= i
    for (int i = ke + ty; i < b; i += 32) {
      for (int k = ke + tx; k <= i; k += 32) {
        double2 a = sm[i * ld + k];
#pragma unroll 4
        for (int t = kb; t < ke; ++t) {
          const double2 x = sm[i * ld + t], y = sm[k * ld + t];
          a.x -= x.x * y.x + x.y * y.y;
          a.y -= x.y * y.x - x.x * y.y;
        }
        sm[i * ld + k] = a;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += 1024) {
    const int k = e / b, i = e % b;
    l[e] = i >= k ? sm[i * ld + k] : make_double2(0.0, 0.0);
  }
}

// One CTA, 128 threads, one barrier per step: "lazy" right-looking Cholesky
// of the b x b Hermitian S (b <= 118) held in shared memory.  Column j is
// left unscaled during the sweep (updates use A_ij conj(A_kj) / d_j); the
// final pass writes L (column-major, leading dimension b, zero upper part).
__global__ void __launch_bounds__(128) chol_lazy_kernel(const double2* __restrict__ s, int b,
                                                        double2* __restrict__ l, int* __restrict__ flag) {
  extern __shared__ double2 sm[];
  const int ld = b + 1;
  const int tid = threadIdx.x;
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int k = e / b, i = e % b;
    sm[i * ld + k] = s[e];
  }
  for (int j = 0; j < b; ++j) {
    __syncthreads();
    double d = sm[j * ld + j].x;
    if (!(d > 0.0)) {
      if (tid == 0) {
        atomicOr(flag, 1);
        sm[j * ld + j].x = 1.0;
      }
      d = 1.0;
    }
    const double inv_d = 1.0 / d;
    // trailing update, two threads per row (even/odd columns)
    for (int r = tid >> 1; j + 1 + r < b; r += (blockDim.x >> 1)) {
      const int i = j + 1 + r;
      const double2 aij = sm[i * ld + j];
      const double2 sij = make_double2(aij.x * inv_d, aij.y * inv_d);
      for (int k = j + 1 + (tid & 1); k <= i; k += 2) {
        const double2 akj = sm[k * ld + j];
        double2 a = sm[i * ld + k];
        a.x -= sij.x * akj.x + sij.y * akj.y;  // a -= (A_ij / d) conj(A_kj)
        a.y -= sij.y * akj.x - sij.x * akj.y;
        sm[i * ld + k] = a;
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int k = e / b, i = e % b;
    double2 v = make_double2(0.0, 0.0);
    if (i >= k) {
      const double p = sqrt(sm[k * ld + k].x);
      v = sm[i * ld + k];
      if (i == k) {
        v = make_double2(p, 0.0);
      } else {
        v.x /= p;
        v.y /= p;
      }
    }
    l[e] = v;
  }
}

// V = X L^{-H} row by row (X, V: n x b column-major; L lower, column-major):
// v_c = (x_c - sum_{t<c} v_t conj(L_ct)) / L_cc.  A warp owns a row; lanes
// hold v_t for t = lane + 32u; L is staged once per CTA in shared memory.
__global__ void __launch_bounds__(256) trsm_rows_kernel(double2* __restrict__ x, i64 n, int b,
                                                        const double2* __restrict__ l) {
  extern __shared__ double2 sl[];  // L row-major [c][t], ld = b
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int t = e / b, c = e % b;  // coalesced read of column-major L(c, t)
    sl[c * b + t] = l[e];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  constexpr int kU = 4;  // b <= 128
  for (i64 r = i64(blockIdx.x) * nw + warp; r < n; r += i64(gridDim.x) * nw) {
    double2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = make_double2(0.0, 0.0);
    for (int c = 0; c < b; ++c) {
      double sx = 0.0, sy = 0.0;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = lane + 32 * u;
        if (t < c) {
          const double2 lct = sl[c * b + t];
          sx += v[u].x * lct.x + v[u].y * lct.y;  // v_t * conj(L_ct)
          sy += v[u].y * lct.x - v[u].x * lct.y;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
      }
      if (lane == (c & 31)) {
        const double2 xc = x[r + i64(c) * n];
        const double inv = 1.0 / sl[c * b + c].x;
        v[c >> 5] = make_double2((xc.x - sx) * inv, (xc.y - sy) * inv);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int t = lane + 32 * u;
      if (t < b) x[r + i64(t) * n] = v[u];
    }
  }
}


// ---- CholQR for b <= 64 without library calls (cholqr_pass):
// one CTA factors S = L L^H (right-looking, one barrier per pivot; L is kept
// implicitly as S[i][k] * rs[k]) and forms M = L^{-1} (eight lanes per
// column, forward substitution), then a row-tiled kernel applies X <- X M^H.
constexpr int kCholThreads = 512;
constexpr int kCholMax = 64;

__global__ void __launch_bounds__(kCholThreads) chol_inv64_kernel(const double2* __restrict__ s, int b,
                                                                   double2* __restrict__ m_out, int* flag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ld = b + 1;
  double2* S = reinterpret_cast<double2*>(smem_raw);  // [b][ld], lower triangle; column k scaled lazily
  double2* M = S + b * ld;                             // [b][ld], rows of L^{-1}
  double* rs = reinterpret_cast<double*>(M + b * ld);  // 1 / L[k][k]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    constexpr int kPer = kCholMax * kCholMax / kCholThreads;  // 8
    double2 v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + kCholThreads * u;
      v[u] = e < b * b ? s[e] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + kCholThreads * u;
      const int i = e % b, j = e / b;  // column-major source
      if (e < b * b) {
        if (i >= j) S[i * ld + j] = v[u];
        M[i * ld + j] = make_double2(0.0, 0.0);
      }
    }
  }
  __syncthreads();
  // Pivot k (one barrier): rs[k]; row k of M from the final rows < k,
  //   M[k][c] = rs[k] (delta_kc - sum_{j=c}^{k-1} L[k][j] M[j][c]),  L[k][j] = S[k][j] rs[j];
  // and the trailing update S[i][j] -= S[i][k] conj(S[j][k]) rs[k]^2.
  const int c = tid >> 3, h = tid & 7;  // eight lanes per column of M
  for (int k = 0; k < b; ++k) {
    double dkk = S[k * ld + k].x;
    if (!(dkk > 0.0)) {
      if (tid == 0) atomicExch(flag, 1);
      dkk = 1e-300;
    }
    const double r = rsqrt(dkk), r2 = r * r;
    double2 acc = make_double2(0.0, 0.0);
    if (c < k) {
#pragma unroll 4
      for (int j = c + h; j < k; j += 8) {
        const double2 skj = S[k * ld + j], mjc = M[j * ld + c];
        const double rj = rs[j];
        acc.x += (skj.x * mjc.x - skj.y * mjc.y) * rj;
        acc.y += (skj.x * mjc.y + skj.y * mjc.x) * rj;
      }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (h == 0 && c <= k) M[k * ld + c] = c == k ? make_double2(r, 0.0) : make_double2(-acc.x * r, -acc.y * r);
    if (tid == 0) rs[k] = r;
    for (int i = k + 1 + warp; i < b; i += kCholThreads / 32) {
      const double2 sik = S[i * ld + k];
      for (int j = k + 1 + lane; j <= i; j += 32) {
        const double2 sjk = S[j * ld + k];
        double2 a = S[i * ld + j];
        a.x -= (sik.x * sjk.x + sik.y * sjk.y) * r2;
        a.y -= (sik.y * sjk.x - sik.x * sjk.y) * r2;
        S[i * ld + j] = a;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += kCholThreads) m_out[e] = M[(e / b) * ld + e % b];  // row-major
}

// Blocked one-CTA Cholesky S = L L^H for b <= 64 (lower, column-major in and
// out, like cusolverDnXpotrf): 16-column block steps; the diagonal block is
// factored by one warp (warp-synchronous), the panel below by row-parallel
// forward substitution, the trailing lower triangle by all threads.  A
// non-positive pivot raises *flag (POTRF's info).
constexpr int kBlkNB = 16;
__global__ void __launch_bounds__(256) chol_blocked_kernel(const double2* __restrict__ s, int b,
                                                           double2* __restrict__ l_out, int* flag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Am = reinterpret_cast<double2*>(smem_raw);  // [64][65]
  double* rd = reinterpret_cast<double*>(Am + 64 * 65);  // 1 / L[j][j]
#define A(i, c) Am[(i) * 65 + (c)]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    double2 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = tid + 256 * u;
      v[u] = e < b * b ? s[e] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = tid + 256 * u;
      if (e < b * b) A(e % b, e / b) = v[u];  // column-major source
    }
  }
  __syncthreads();
  for (int k0 = 0; k0 < b; k0 += kBlkNB) {
    const int m = min(kBlkNB, b - k0);
    // (1) diagonal block, warp 0
    if (warp == 0) {
      for (int j = 0; j < m; ++j) {
        const int jj = k0 + j;
        double d = A(jj, jj).x;
        if (!(d > 0.0)) {
          if (lane == 0) atomicExch(flag, 1);
          d = 1e-300;
        }
        const double r = rsqrt(d);
        __syncwarp();
        if (lane == 0) {
          A(jj, jj) = make_double2(d * r, 0.0);  // sqrt(d)
          rd[jj] = r;
        }
        for (int i = j + 1 + lane; i < m; i += 32) {
          const double2 a = A(k0 + i, jj);
          A(k0 + i, jj) = make_double2(a.x * r, a.y * r);
        }
        __syncwarp();
        // trailing update inside the block: A(i, c) -= L[i][j] conj(L[c][j]), j < c <= i < m
        for (int e = lane; e < (m - j - 1) * (m - j - 1); e += 32) {
          const int i = j + 1 + e / (m - j - 1), c = j + 1 + e % (m - j - 1);
          if (c <= i) {
            const double2 li = A(k0 + i, jj), lc = A(k0 + c, jj);
            double2 a = A(k0 + i, k0 + c);
            a.x -= li.x * lc.x + li.y * lc.y;
            a.y -= li.y * lc.x - li.x * lc.y;
            A(k0 + i, k0 + c) = a;
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // (2) panel: rows i >= k0 + m solve A(i, k0:k0+m) <- A(i, k0:k0+m) L_kk^{-H}
    for (int i = k0 + m + tid; i < b; i += 256) {
      for (int j = 0; j < m; ++j) {
        double2 a = A(i, k0 + j);
        for (int c = 0; c < j; ++c) {  // a -= A(i, k0+c) conj(L[k0+j][k0+c])
          const double2 x = A(i, k0 + c), lj = A(k0 + j, k0 + c);
          a.x -= x.x * lj.x + x.y * lj.y;
          a.y -= x.y * lj.x - x.x * lj.y;
        }
        const double r = rd[k0 + j];
        A(i, k0 + j) = make_double2(a.x * r, a.y * r);
      }
    }
    __syncthreads();
    // (3) trailing lower triangle: A(i, c) -= sum_{j<m} L[i][k0+j] conj(L[c][k0+j]), k0+m <= c <= i < b
    const int t0 = k0 + m, tn = b - t0;
    for (int e = tid; e < tn * tn; e += 256) {
      const int i = t0 + e / tn, c = t0 + e % tn;
      if (c > i) continue;
      double ax = 0.0, ay = 0.0;
#pragma unroll 4
      for (int j = 0; j < m; ++j) {
        const double2 li = A(i, k0 + j), lc = A(c, k0 + j);
        ax += li.x * lc.x + li.y * lc.y;
        ay += li.y * lc.x - li.x * lc.y;
      }
      double2 a = A(i, c);
      a.x -= ax;
      a.y -= ay;
      A(i, c) = a;
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += 256) {
    const int i = e % b, c = e / b;
    l_out[e] = c <= i ? A(i, c) : make_double2(0.0, 0.0);
  }
}
#undef A

// X (n x b, column-major) <- X L^{-H}, L lower triangular column-major b x b
// (cuSOLVER POTRF output), by forward substitution on each row:
//   y_j = (x_j - sum_{k<j} y_k conj(L[j][k])) / L[j][j].
// A lane pair owns a row (lane h keeps the columns k = h mod 2 in registers);
// every step the pair combines its partial sums with one shuffle.  conj(L)
// is staged in shared memory (broadcast reads).
constexpr int kTrsmThreads = 128;
template <int B>
__global__ void __launch_bounds__(kTrsmThreads) trsm_pairs_kernel(double2* __restrict__ x, i64 n,
                                                                  const double2* __restrict__ l) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Lc = reinterpret_cast<double2*>(smem_raw);  // Lc[j * B + k] = conj(L[j][k]), k <= j
  double* dinv = reinterpret_cast<double*>(Lc + B * B);
  for (int e = threadIdx.x; e < B * B; e += kTrsmThreads) {
    const int j = e % B, k = e / B;  // column-major source: e = j + k B
    const double2 v = l[e];
    Lc[j * B + k] = make_double2(v.x, -v.y);
    if (j == k) dinv[j] = 1.0 / v.x;
  }
  __syncthreads();
  const int h = threadIdx.x & 1;
  const i64 r = (i64(blockIdx.x) * kTrsmThreads + threadIdx.x) >> 1;
  const bool live = r < n;
  constexpr int H = B / 2;
  double2 y[H];
#pragma unroll
  for (int u = 0; u < H; ++u) y[u] = live ? x[r + i64(2 * u + h) * n] : make_double2(0.0, 0.0);
#pragma unroll
  for (int j = 0; j < B; ++j) {
    double2 p0 = make_double2(0.0, 0.0), p1 = p0;
#pragma unroll
    for (int u = 0; 2 * u < j; ++u) {
      const int k = 2 * u + h;  // runtime parity: guard k < j
      if (k < j) {
        const double2 lc = Lc[j * B + k];
        double2& p = (u & 1) ? p1 : p0;
        p.x += y[u].x * lc.x - y[u].y * lc.y;
        p.y += y[u].x * lc.y + y[u].y * lc.x;
      }
    }
    double2 p = make_double2(p0.x + p1.x, p0.y + p1.y);
    p.x += __shfl_xor_sync(0xffffffffu, p.x, 1);
    p.y += __shfl_xor_sync(0xffffffffu, p.y, 1);
    if ((j & 1) == h) {
      const double di = dinv[j];
      y[j >> 1] = make_double2((y[j >> 1].x - p.x) * di, (y[j >> 1].y - p.y) * di);
    }
  }
  if (live)
#pragma unroll
    for (int u = 0; u < H; ++u) x[r + i64(2 * u + h) * n] = y[u];
}

// X (n x b, column-major) <- X M^H, M lower triangular (row-major b x b).
constexpr int kApplyRows = 16;
__global__ void __launch_bounds__(256) apply_minvh_kernel(double2* __restrict__ x, i64 n, int b,
                                                          const double2* __restrict__ m) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ld = b + 1;
  double2* Ms = reinterpret_cast<double2*>(smem_raw);  // [b][ld]
  double2* Xs = Ms + b * ld;                           // [kApplyRows][ld]
  const i64 r0 = i64(blockIdx.x) * kApplyRows;
  {
    constexpr int kM = kCholMax * kCholMax / 256, kX = kApplyRows * kCholMax / 256;  // 16, 4
    double2 mv[kM], xv[kX];
#pragma unroll
    for (int u = 0; u < kM; ++u) {
      const int e = threadIdx.x + 256 * u;
      mv[u] = e < b * b ? m[e] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < kX; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int rr = e % kApplyRows, c = e / kApplyRows;
      const i64 r = r0 + rr;
      xv[u] = (c < b && r < n) ? x[r + i64(c) * n] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < kM; ++u) {
      const int e = threadIdx.x + 256 * u;
      if (e < b * b) Ms[(e / b) * ld + e % b] = mv[u];
    }
#pragma unroll
    for (int u = 0; u < kX; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int rr = e % kApplyRows, c = e / kApplyRows;
      if (c < b) Xs[rr * ld + c] = xv[u];
    }
  }
  __syncthreads();
  const int rr = threadIdx.x % kApplyRows, jg = threadIdx.x / kApplyRows;  // 16 column groups
  constexpr int kPer = kCholMax / 16;
  double2 acc[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) acc[u] = make_double2(0.0, 0.0);
  for (int k = 0; k < b; ++k) {
    const double2 xv = Xs[rr * ld + k];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int j = jg + 16 * u;
      if (j < b) acc[u] = cfma_conj_rev(acc[u], xv, Ms[j * ld + k]);
    }
  }
  const i64 r = r0 + rr;
  if (r < n)
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int j = jg + 16 * u;
      if (j < b) x[r + i64(j) * n] = acc[u];
    }
}
}  // namespace

void cholqr_fast(sk_ctx* ctx, double2* x, i64 n, int b, double2* s, double2* l, int* flag) {
  if (b > 118) fail(SK_ERR_UNSUPPORTED, "cholqr_fast: block too large");
  cross_gram(ctx, x, x, n, b, s);
  const size_t smem = size_t(b) * (b + 1) * sizeof(double2);
  set_smem_limit(reinterpret_cast<const void*>(chol_lazy_kernel), smem);
  chol_lazy_kernel<<<1, 128, smem, ctx->stream>>>(s, b, l, flag);
  ++ctx->launches;
  SKB_LAUNCH("chol_lazy_kernel");
  const size_t smem2 = size_t(b) * b * sizeof(double2);
  set_smem_limit(reinterpret_cast<const void*>(trsm_rows_kernel), smem2);
  const i64 blocks = std::min<i64>((n + 7) / 8, ctx->sm_count);
  trsm_rows_kernel<<<unsigned(blocks), 256, smem2, ctx->stream>>>(x, n, b, l);
  ++ctx->launches;
  SKB_LAUNCH("trsm_rows_kernel");
}

void cholesky_small(sk_ctx* ctx, const double2* s, int b, double2* l, int* flag) {
  const size_t smem = size_t(b) * (b + 1) * sizeof(double2);
  if (smem > 227 * 1024) fail(SK_ERR_UNSUPPORTED, "cholesky_small: block too large");
  set_smem_limit(reinterpret_cast<const void*>(chol_kernel), smem);
  chol_kernel<<<1, dim3(32, 32), smem, ctx->stream>>>(s, b, l, flag);
  ++ctx->launches;
  SKB_LAUNCH("chol_kernel");
}

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

void chol_inv(sk_ctx* ctx, const double2* s, int b, double2* minv, int* flag) {
  const size_t smem = size_t(b) * (b + 1) * sizeof(double2);
  if (smem > 227 * 1024) fail(SK_ERR_UNSUPPORTED, "chol_inv: block too large");
  set_smem_limit(reinterpret_cast<const void*>(chol_inv_kernel), smem);
  chol_inv_kernel<<<1, 256, smem, ctx->stream>>>(s, b, minv, flag);
  ++ctx->launches;
  SKB_LAUNCH("chol_inv");
}

bool cholqr_pass(sk_ctx* ctx, double2* x, i64 n, int b, double2* s, double2* m, int* flag) {
  if (b < 1 || b > kCholMax) return false;
  static const bool prof = std::getenv("SKB_PROFILE_NS") != nullptr;
  cudaEvent_t pe[4];
  if (prof)
    for (auto& e : pe) {
      SKB_CUDA(cudaEventCreate(&e));
    }
  if (prof) SKB_CUDA(cudaEventRecord(pe[0], ctx->stream));
  cross_gram(ctx, x, x, n, b, s);
  if (prof) SKB_CUDA(cudaEventRecord(pe[1], ctx->stream));
  const size_t smem = size_t(2 * b * (b + 1)) * sizeof(double2) + size_t(b) * sizeof(double);
  set_smem_limit(reinterpret_cast<const void*>(chol_inv64_kernel), smem);
  chol_inv64_kernel<<<1, kCholThreads, smem, ctx->stream>>>(s, b, m, flag);
  ++ctx->launches;
  SKB_LAUNCH("chol_inv64_kernel");
  if (prof) SKB_CUDA(cudaEventRecord(pe[2], ctx->stream));
  const size_t smem2 = size_t((b + kApplyRows) * (b + 1)) * sizeof(double2);
  set_smem_limit(reinterpret_cast<const void*>(apply_minvh_kernel), smem2);
  apply_minvh_kernel<<<unsigned((n + kApplyRows - 1) / kApplyRows), 256, smem2, ctx->stream>>>(x, n, b, m);
  ++ctx->launches;
  SKB_LAUNCH("apply_minvh_kernel");
  if (prof) {
    SKB_CUDA(cudaEventRecord(pe[3], ctx->stream));
    SKB_CUDA(cudaEventSynchronize(pe[3]));
    float t0 = 0.f, t1 = 0.f, t2 = 0.f;
    cudaEventElapsedTime(&t0, pe[0], pe[1]);
    cudaEventElapsedTime(&t1, pe[1], pe[2]);
    cudaEventElapsedTime(&t2, pe[2], pe[3]);
    std::fprintf(stderr, "[cholqr b=%d] gram %.1f us  chol_inv %.1f us  apply %.1f us\n", b, t0 * 1e3, t1 * 1e3,
                 t2 * 1e3);
    for (auto& e : pe) cudaEventDestroy(e);
  }
  return true;
}

template <int B>
void launch_trsm_rows(sk_ctx* ctx, double2* x, i64 n, const double2* l) {
  const unsigned blocks = unsigned((2 * n + kTrsmThreads - 1) / kTrsmThreads);
  const size_t smem = size_t(B) * B * sizeof(double2) + size_t(B) * sizeof(double);
  set_smem_limit(reinterpret_cast<const void*>(trsm_pairs_kernel<B>), smem);
  trsm_pairs_kernel<B><<<blocks, kTrsmThreads, smem, ctx->stream>>>(x, n, l);
}

bool trsm_rows_lower(sk_ctx* ctx, double2* x, i64 n, int b, const double2* l) {
  if (b == 64)
    launch_trsm_rows<64>(ctx, x, n, l);
  else if (b == 48)
    launch_trsm_rows<48>(ctx, x, n, l);
  else if (b == 32)
    launch_trsm_rows<32>(ctx, x, n, l);
  else
    return false;
  ++ctx->launches;
  SKB_LAUNCH("trsm_pairs_kernel");
  return true;
}

void cholesky_blocked(sk_ctx* ctx, const double2* s, int b, double2* l, int* flag) {
  if (b < 1 || b > 64) fail(SK_ERR_UNSUPPORTED, "cholesky_blocked: b must be in [1, 64]");
  const size_t smem = 64 * 65 * sizeof(double2) + 64 * sizeof(double);
  set_smem_limit(reinterpret_cast<const void*>(chol_blocked_kernel), smem);
  chol_blocked_kernel<<<1, 256, smem, ctx->stream>>>(s, b, l, flag);
  ++ctx->launches;
  SKB_LAUNCH("chol_blocked_kernel");
}

}  // namespace skb
