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

}  // namespace

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
