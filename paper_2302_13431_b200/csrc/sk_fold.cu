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
// U_sig holds the n - R ~ 17-59 signal eigenvectors, folded
// by the correlation theorem below (fold_lags_spectral).  The CSR kernels
// serve the standalone gram_field_fast (caller-supplied W) and the fallback
// for lag boxes whose spectral buffers exceed shared memory (Ws = U U^H).
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

// ---------------------------------------------------------------- spectral fold
// The signal part of the fold is a sum of cross-correlations on the support
// lattice: with W = I - U U^H (U = U_sig, n x k),
//   k_pq[d] = |L| delta_pq [d = 0] - sum_kk sum_{(s,t): n_t - n_s = d} U_q[s,kk] conj(U_p[t,kk]).
// On the lag box (P = 4 tau + 1 per axis, so every lag d in [-2tau, 2tau]^D
// has a unique residue mod P) the correlation theorem gives
//   c_pq(d) = P^-D sum_f S_pq(f) e^{-2 pi i f.d / P},
//   S_pq(f) = sum_kk a_q^kk(f) conj(a_p^kk(f)),  a_q^kk(f) = sum_s U_q[s,kk] e^{-2 pi i f.n_s / P}.
// Three FP64 kernels: (A) per (kk, q) the separable DFT of u_q^kk from its
// (2 tau + 1)^D box to the P^D frequencies; (B) per frequency the Q x Q
// Hermitian product over the k signal vectors (p <= q pairs only); (C) per
// pair the separable inverse DFT back onto the lag box.  O(P^D (Q k (2tau+1) +
// h k) + h P^{D+1}) flops instead of the n x n x k ZHERK + n^2 fold, no n x n
// buffer, fixed-order sums (deterministic).
namespace {

// One axis of a separable DFT in shared memory: in has extents ext (nd <= 3,
// row-major), out replaces axis `ax` (extent Lin) by Lout outputs:
//   out[.., f, ..] = scale * sum_j in[.., j, ..] tw[((f * (j - j0)) mod P)]   (tw[m] = e^{sign 2 pi i m/P})
__device__ void dft_axis(const double2* in, double2* out, const int* ext, int nd, int ax, int Lout, int j0,
                         const double2* tw, int P, double scale) {
  int outer = 1, inner = 1;
  for (int a = 0; a < ax; ++a) outer *= ext[a];
  for (int a = ax + 1; a < nd; ++a) inner *= ext[a];
  const int Lin = ext[ax];
  const int total = outer * Lout * inner;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int i = e % inner;
    const int f = (e / inner) % Lout;
    const int o = e / (inner * Lout);
    const double2* src = in + i64(o) * Lin * inner + i;
    double re = 0.0, im = 0.0;
    for (int j = 0; j < Lin; ++j) {
      int m = (f * (j - j0)) % P;
      if (m < 0) m += P;
      const double2 v = src[i64(j) * inner];
      const double2 w = tw[m];
      re += v.x * w.x - v.y * w.y;
      im += v.x * w.y + v.y * w.x;
    }
    out[e] = make_double2(re * scale, im * scale);
  }
}

__device__ void make_twiddles(double2* tw, int P, double sign) {
  for (int m = threadIdx.x; m < P; m += blockDim.x) {
    double sn, cs;
    sincospi(sign * 2.0 * double(m) / double(P), &sn, &cs);
    tw[m] = make_double2(cs, sn);
  }
}

// (A) a[f][kk][q] = sum_s U[q lam + s, kk] e^{-2 pi i f.n_s / P}; block = (kk, q).
// blockIdx.y: slice of a multislice group (its own basis and column count).
__global__ void __launch_bounds__(256) spec_u_kernel(const FoldBatch fb, i64 n, i64 a_stride, int q, int lam,
                                                     const int* __restrict__ offs, int nd, int tau,
                                                     double2* __restrict__ a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int k = fb.k[blockIdx.y];
  if (int(blockIdx.x) >= k * q) return;
  const double2* __restrict__ u = fb.u[blockIdx.y];
  a += i64(blockIdx.y) * a_stride;
  const int P = 4 * tau + 1, B = 2 * tau + 1;
  int nbox = 1, bbox = 1;
  for (int d = 0; d < nd; ++d) {
    nbox *= P;
    bbox *= B;
  }
  double2* tw = reinterpret_cast<double2*>(smem_raw);
  double2* buf0 = tw + P;
  double2* buf1 = buf0 + nbox;
  const int kk = blockIdx.x / q, ch = blockIdx.x % q;
  make_twiddles(tw, P, -1.0);
  for (int e = threadIdx.x; e < bbox; e += blockDim.x) buf0[e] = make_double2(0.0, 0.0);
  __syncthreads();
  const double2* col = u + i64(kk) * n + i64(ch) * lam;
  for (int sidx = threadIdx.x; sidx < lam; sidx += blockDim.x) {
    int at = 0;
    for (int d = 0; d < nd; ++d) at = at * B + (offs[sidx * nd + d] + tau);
    buf0[at] = col[sidx];
  }
  __syncthreads();
  int ext[3] = {B, B, B};
  double2* src = buf0;
  double2* dst = buf1;
  for (int ax = 0; ax < nd; ++ax) {
    dft_axis(src, dst, ext, nd, ax, P, tau, tw, P, 1.0);  // box index j <-> n = j - tau
    ext[ax] = P;
    __syncthreads();
    double2* t = src;
    src = dst;
    dst = t;
  }
  for (int f = threadIdx.x; f < nbox; f += blockDim.x) a[(i64(f) * k + kk) * q + ch] = src[f];
}

// (B) S[pair][f] = sum_kk a[f][kk][c] conj(a[f][kk][p]) for pair (p <= c); block = (f, slice)
__global__ void __launch_bounds__(256) spec_pairs_kernel(const double2* __restrict__ a, const FoldBatch fb,
                                                         i64 a_stride, int q, int nbox, double2* __restrict__ S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* af = reinterpret_cast<double2*>(smem_raw);  // [k][q]
  const int f = blockIdx.x;
  const int k = fb.k[blockIdx.y];
  a += i64(blockIdx.y) * a_stride;
  S += i64(blockIdx.y) * (i64(q) * (q + 1) / 2) * nbox;
  for (int e = threadIdx.x; e < k * q; e += blockDim.x) af[e] = a[i64(f) * k * q + e];
  __syncthreads();
  const int h = q * (q + 1) / 2;
  for (int pr = threadIdx.x; pr < h; pr += blockDim.x) {
    int p = 0, rem = pr;
    while (rem >= q - p) {
      rem -= q - p;
      ++p;
    }
    const int c = p + rem;
    double re = 0.0, im = 0.0;
    for (int kk = 0; kk < k; ++kk) {
      const double2 x = af[kk * q + c], y = af[kk * q + p];  // x conj(y)
      re += x.x * y.x + x.y * y.y;
      im += x.y * y.x - x.x * y.y;
    }
    S[i64(pr) * nbox + f] = make_double2(re, im);
  }
}

// (C) lags[pair][l] = |L| delta_pc [l = centre] - P^-D sum_f S[pair][f] e^{-2 pi i f.d / P}; block = pair
__global__ void __launch_bounds__(256) spec_lags_kernel(const double2* __restrict__ S, int q, int nd, int tau, int lam,
                                                        double2* __restrict__ lags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P = 4 * tau + 1;
  int nbox = 1;
  for (int d = 0; d < nd; ++d) nbox *= P;
  double2* tw = reinterpret_cast<double2*>(smem_raw);
  double2* buf0 = tw + P;
  double2* buf1 = buf0 + nbox;
  const int pr = blockIdx.x;
  S += i64(blockIdx.y) * (i64(q) * (q + 1) / 2) * nbox;     // blockIdx.y: slice of a multislice group
  lags += i64(blockIdx.y) * (i64(q) * (q + 1) / 2) * nbox;
  make_twiddles(tw, P, -1.0);
  for (int e = threadIdx.x; e < nbox; e += blockDim.x) buf0[e] = S[i64(pr) * nbox + e];
  __syncthreads();
  int ext[3] = {P, P, P};
  double2* src = buf0;
  double2* dst = buf1;
  // frequency f = 0..P-1 in, lag index j = 0..P-1 out with d = j - 2 tau:
  // e^{-2 pi i f d / P}; dft_axis evaluates tw[(f' (j' - j0))] with the roles
  // of input / output index swapped, so pass j0 = 0 and fold the shift into
  // the output index through (j - 2tau) * f = f * j - f * 2tau (mod P).
  for (int ax = 0; ax < nd; ++ax) {
    int outer = 1, inner = 1;
    for (int a = 0; a < ax; ++a) outer *= ext[a];
    for (int a = ax + 1; a < nd; ++a) inner *= ext[a];
    const int total = outer * P * inner;
    const double scale = 1.0 / double(P);
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int i = e % inner;
      const int j = (e / inner) % P;
      const int o = e / (inner * P);
      const double2* sp = src + i64(o) * P * inner + i;
      const int d = j - 2 * tau;
      double re = 0.0, im = 0.0;
      for (int ff = 0; ff < P; ++ff) {
        int m = (ff * d) % P;
        if (m < 0) m += P;
        const double2 v = sp[i64(ff) * inner];
        const double2 w = tw[m];
        re += v.x * w.x - v.y * w.y;
        im += v.x * w.y + v.y * w.x;
      }
      dst[e] = make_double2(re * scale, im * scale);
    }
    __syncthreads();
    double2* t = src;
    src = dst;
    dst = t;
  }
  int p = 0, rem = pr;
  while (rem >= q - p) {
    rem -= q - p;
    ++p;
  }
  const bool diag = rem == 0;
  const int centre = (nbox - 1) / 2;
  for (int l = threadIdx.x; l < nbox; l += blockDim.x) {
    double2 v = src[l];
    v.x = -v.x;
    v.y = -v.y;
    if (diag && l == centre) v.x += double(lam);
    lags[i64(pr) * nbox + l] = v;
  }
}

}  // namespace

size_t spectral_fold_smem(int nd, int tau, int k, int q) {
  const int P = 4 * tau + 1;
  size_t nbox = 1;
  for (int d = 0; d < nd; ++d) nbox *= size_t(P);
  const size_t box = (size_t(P) + 2 * nbox) * sizeof(double2);
  return std::max(box, size_t(k) * size_t(q) * sizeof(double2));
}

void fold_lags_spectral(sk_ctx* ctx, const double2* u, i64 n, int k, int q, int lam, int nd, int tau,
                        const int* d_offs, double2* lags) {
  FoldBatch fb{};
  fb.u[0] = u;
  fb.k[0] = k;
  fold_lags_spectral_batched(ctx, fb, 1, n, q, lam, nd, tau, d_offs, lags);
}

// The same for a group of slices (one launch per stage, the slice on grid.y):
// lags [slices][h][nbox].
void fold_lags_spectral_batched(sk_ctx* ctx, const FoldBatch& fb, int slices, i64 n, int q, int lam, int nd, int tau,
                                const int* d_offs, double2* lags) {
  const int P = 4 * tau + 1;
  int nbox = 1;
  for (int d = 0; d < nd; ++d) nbox *= P;
  const int h = q * (q + 1) / 2;
  int kmax = 0;
  for (int i = 0; i < slices; ++i) kmax = std::max(kmax, fb.k[i]);
  const size_t box_smem = (size_t(P) + 2 * size_t(nbox)) * sizeof(double2);
  double2* S = ctx->arena.get<double2>("field:spec_S", i64(slices) * h * nbox);
  const i64 a_stride = i64(nbox) * kmax * q;
  double2* a = ctx->arena.get<double2>("field:spec_a", std::max<i64>(1, i64(slices) * a_stride));
  if (kmax > 0) {
    set_smem_limit(reinterpret_cast<const void*>(spec_u_kernel), box_smem);
    spec_u_kernel<<<dim3(unsigned(kmax * q), unsigned(slices)), 256, box_smem, ctx->stream>>>(fb, n, a_stride, q, lam,
                                                                                             d_offs, nd, tau, a);
    SKB_LAUNCH("spec_u_kernel");
    ++ctx->launches;
  }
  // (a slice without signal columns sums nothing: S = 0)
  const size_t ps = std::max<size_t>(16, size_t(kmax) * q * sizeof(double2));
  set_smem_limit(reinterpret_cast<const void*>(spec_pairs_kernel), ps);
  spec_pairs_kernel<<<dim3(unsigned(nbox), unsigned(slices)), 256, ps, ctx->stream>>>(a, fb, a_stride, q, nbox, S);
  SKB_LAUNCH("spec_pairs_kernel");
  set_smem_limit(reinterpret_cast<const void*>(spec_lags_kernel), box_smem);
  spec_lags_kernel<<<dim3(unsigned(h), unsigned(slices)), 256, box_smem, ctx->stream>>>(S, q, nd, tau, lam, lags);
  SKB_LAUNCH("spec_lags_kernel");
  ctx->launches += 2;
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

namespace skb {

// ---------------------------------------------------------------- aggregate_w
// Standalone aggregate_w (spatial_gram.cpp:87-94): W = F F^H for the n x r
// nullspace filters F (c64, column-major).  W is Hermitian: only tiles on or
// below the diagonal are computed (64 x 64 per CTA, 4 x 4 complex outputs per
// thread, FP32 accumulation over r in 16-column slabs staged in shared
// memory); each tile is stored with its conjugate mirror.
namespace {
constexpr int kHT = 64;  // output tile edge
constexpr int kHK = 16;  // r slab
__global__ void __launch_bounds__(256) herk_tiles_kernel(const float2* __restrict__ f, i64 n, i64 r,
                                                         float2* __restrict__ w) {
  // blockIdx.x enumerates lower-triangular tiles (bi >= bj)
  int bi = 0, rem = int(blockIdx.x);
  while (rem > bi) {
    rem -= bi + 1;
    ++bi;
  }
  const int bj = rem;
  __shared__ float2 As[kHK][kHT + 1];
  __shared__ float2 Bs[kHK][kHT + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const i64 i0 = i64(bi) * kHT, j0 = i64(bj) * kHT;
  float2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = make_float2(0.f, 0.f);
  for (i64 k0 = 0; k0 < r; k0 += kHK) {
    for (int e = threadIdx.x; e < kHT * kHK; e += blockDim.x) {
      const int row = e % kHT, kk = e / kHT;
      const i64 kc = k0 + kk;
      As[kk][row] = (i0 + row < n && kc < r) ? f[(i0 + row) + kc * n] : make_float2(0.f, 0.f);
      Bs[kk][row] = (j0 + row < n && kc < r) ? f[(j0 + row) + kc * n] : make_float2(0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kHK; ++kk) {
      float2 x[4], y[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        x[a] = As[kk][ty + 16 * a];
        y[a] = Bs[kk][tx + 16 * a];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {  // acc += x conj(y)
          acc[a][b].x = fmaf(x[a].x, y[b].x, fmaf(x[a].y, y[b].y, acc[a][b].x));
          acc[a][b].y = fmaf(x[a].y, y[b].x, fmaf(-x[a].x, y[b].y, acc[a][b].y));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const i64 i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      if (i >= n || j >= n || i < j) continue;
      w[i + j * n] = i == j ? make_float2(acc[a][b].x, 0.f) : acc[a][b];  // Hermitian: real diagonal
      if (i != j) w[j + i * n] = make_float2(acc[a][b].x, -acc[a][b].y);
    }
}
}  // namespace

void herk_full(sk_ctx* ctx, const float2* f, i64 n, i64 r, float2* w) {
  const i64 nt = (n + kHT - 1) / kHT;
  herk_tiles_kernel<<<unsigned(nt * (nt + 1) / 2), 256, 0, ctx->stream>>>(f, n, r, w);
  ++ctx->launches;
  SKB_LAUNCH("herk_tiles_kernel");
}

}  // namespace skb
