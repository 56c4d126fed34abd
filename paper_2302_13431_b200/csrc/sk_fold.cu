// Fold of the aggregate W into per-channel-pair lag kernels on the
// (4 tau + 1)^D lag box (spatial_gram.cpp:108-131):
//
//   k_pq[l] = sum_{(s,t): n_t - n_s = l} W[q|L| + s, p|L| + t]      (p <= q)
//
// The (s,t) lists per lag are a CSR table built once per support on the host,
// so every output is a fixed-order sum (deterministic, no atomics).  Lag
// kernels are kept in FP64: the G(x) expansion that follows runs in FP64 and
// only its output is rounded (to an fp32 hi/lo pair).
//
// On the pipeline path W is never formed from the R ~ n nullspace filters:
// with a complete orthonormal eigenbasis W = F F^H = I - U_sig U_sig^H, where
// U_sig holds the n - R ~ 17-48 signal eigenvectors.  The
// caller passes Ws = U_sig U_sig^H (lower triangle, FP64, from cuBLAS ZHERK)
// and the identity is folded in analytically.
#include "sk_internal.h"

namespace skb {

namespace {

template <bool kSignal>
__global__ void __launch_bounds__(256) fold_f64_kernel(const double2* __restrict__ w, i64 n, int lam, int nbox,
                                                       const int2* __restrict__ pairs, const int* __restrict__ ptr,
                                                       const int* __restrict__ st, double2* __restrict__ lags) {
  const int2 pq = pairs[blockIdx.x];
  const int p = pq.x, q = pq.y;
  const i64 row0 = i64(q) * lam, col0 = i64(p) * lam;
  for (int l = threadIdx.x; l < nbox; l += blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int e = ptr[l]; e < ptr[l + 1]; ++e) {
      const int s = st[e] & 0xffff, t = st[e] >> 16;
      const i64 r = row0 + s, c = col0 + t;
      double2 v;
      if (kSignal) {
        if (r >= c) {
          v = w[r + c * n];
        } else {
          v = w[c + r * n];
          v.y = -v.y;
        }
        v.x = -v.x;
        v.y = -v.y;
        if (r == c) v.x += 1.0;
      } else {
        v = w[r + c * n];
      }
      re += v.x;
      im += v.y;
    }
    lags[i64(blockIdx.x) * nbox + l] = make_double2(re, im);
  }
}

__global__ void __launch_bounds__(256) fold_f32_kernel(const float2* __restrict__ w, i64 n, int lam, int nbox,
                                                       const int2* __restrict__ pairs, const int* __restrict__ ptr,
                                                       const int* __restrict__ st, double2* __restrict__ lags) {
  const int2 pq = pairs[blockIdx.x];
  const i64 row0 = i64(pq.y) * lam, col0 = i64(pq.x) * lam;
  for (int l = threadIdx.x; l < nbox; l += blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int e = ptr[l]; e < ptr[l + 1]; ++e) {
      const int s = st[e] & 0xffff, t = st[e] >> 16;
      const float2 v = w[(row0 + s) + (col0 + t) * n];
      re += v.x;
      im += v.y;
    }
    lags[i64(blockIdx.x) * nbox + l] = make_double2(re, im);
  }
}

// Fold straight from the signal basis (no n x n Ws): per pair (p, q) the
// block M[s][t] = sum_k U[q|L|+s, k] conj(U[p|L|+t, k]) is formed in shared
// memory by 4 x 4 register tiles (FP64, U read through L1), then every lag
// sums its (s, t) list from M in list order (deterministic, like the Ws path):
//   k_pq[l] = sum_{(s,t) in L(l)} (delta_{(q,s),(p,t)} - M[s][t]).
constexpr int kFoldT = 4;  // tile edge
__global__ void __launch_bounds__(256) fold_from_u_kernel(const double2* __restrict__ u, i64 n, int k, int lam,
                                                          int nbox, const int2* __restrict__ pairs,
                                                          const int* __restrict__ ptr, const int* __restrict__ st,
                                                          double2* __restrict__ lags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* M = reinterpret_cast<double2*>(smem_raw);  // [lam][lam + 1]
  const int ldm = lam + 1;
  const int2 pq = pairs[blockIdx.x];
  const int p = pq.x, q = pq.y;
  const double2* uq = u + i64(q) * lam;
  const double2* up = u + i64(p) * lam;
  const int nt = (lam + kFoldT - 1) / kFoldT;
  for (int tile = threadIdx.x; tile < nt * nt; tile += blockDim.x) {
    const int s0 = (tile / nt) * kFoldT, t0 = (tile % nt) * kFoldT;
    double2 acc[kFoldT][kFoldT];
#pragma unroll
    for (int a = 0; a < kFoldT; ++a)
#pragma unroll
      for (int b = 0; b < kFoldT; ++b) acc[a][b] = make_double2(0.0, 0.0);
    for (int kk = 0; kk < k; ++kk) {
      double2 x[kFoldT], y[kFoldT];
#pragma unroll
      for (int a = 0; a < kFoldT; ++a) {
        x[a] = s0 + a < lam ? uq[s0 + a + i64(kk) * n] : make_double2(0.0, 0.0);
        y[a] = t0 + a < lam ? up[t0 + a + i64(kk) * n] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int a = 0; a < kFoldT; ++a)
#pragma unroll
        for (int b = 0; b < kFoldT; ++b) {  // acc += x conj(y)
          acc[a][b].x = fma(x[a].x, y[b].x, fma(x[a].y, y[b].y, acc[a][b].x));
          acc[a][b].y = fma(x[a].y, y[b].x, fma(-x[a].x, y[b].y, acc[a][b].y));
        }
    }
#pragma unroll
    for (int a = 0; a < kFoldT; ++a)
#pragma unroll
      for (int b = 0; b < kFoldT; ++b)
        if (s0 + a < lam && t0 + b < lam) M[(s0 + a) * ldm + t0 + b] = acc[a][b];
  }
  __syncthreads();
  for (int l = threadIdx.x; l < nbox; l += blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int e = ptr[l]; e < ptr[l + 1]; ++e) {
      const int s = st[e] & 0xffff, t = st[e] >> 16;
      const double2 v = M[s * ldm + t];
      re -= v.x;
      im -= v.y;
      if (p == q && s == t) re += 1.0;
    }
    lags[i64(blockIdx.x) * nbox + l] = make_double2(re, im);
  }
}

}  // namespace

size_t fold_from_u_smem(int lam) { return size_t(lam) * (lam + 1) * sizeof(double2); }

void fold_lags_from_u(sk_ctx* ctx, const double2* u, i64 n, int k, int npairs, int lam, int nbox,
                      const int2* d_pairs, const int* d_lag_ptr, const int* d_lag_st, double2* lags) {
  const size_t smem = fold_from_u_smem(lam);
  set_smem_limit(reinterpret_cast<const void*>(fold_from_u_kernel), smem);
  fold_from_u_kernel<<<npairs, 256, smem, ctx->stream>>>(u, n, k, lam, nbox, d_pairs, d_lag_ptr, d_lag_st, lags);
  ++ctx->launches;
  SKB_LAUNCH("fold_from_u_kernel");
}

void fold_lags_f64(sk_ctx* ctx, const double2* w, i64 n, int npairs, int lam, int nbox, const int2* d_pairs,
                   const int* d_lag_ptr, const int* d_lag_st, bool w_is_signal, double2* lags) {
  if (w_is_signal)
    fold_f64_kernel<true><<<npairs, 256, 0, ctx->stream>>>(w, n, lam, nbox, d_pairs, d_lag_ptr, d_lag_st, lags);
  else
    fold_f64_kernel<false><<<npairs, 256, 0, ctx->stream>>>(w, n, lam, nbox, d_pairs, d_lag_ptr, d_lag_st, lags);
  ++ctx->launches;
  SKB_LAUNCH("fold_f64_kernel");
}

void fold_lags_f32(sk_ctx* ctx, const float2* w, i64 n, int npairs, int lam, int nbox, const int2* d_pairs,
                   const int* d_lag_ptr, const int* d_lag_st, double2* lags) {
  fold_f32_kernel<<<npairs, 256, 0, ctx->stream>>>(w, n, lam, nbox, d_pairs, d_lag_ptr, d_lag_st, lags);
  ++ctx->launches;
  SKB_LAUNCH("fold_f32_kernel");
}

}  // namespace skb
