// K5 — periodic-sinc interpolation (maps.cpp:54-99) by radix-2 FFTs in
// shared memory, one axis at a time.
//
// The reference does image_to_kspace on the low grid (x 1/n), places the
// centred spectrum into a zero grid of the full size and runs
// kspace_to_image.  Per axis that is, for a line x[0..n) -> out[0..N):
//   Y = FFT_n(ifftshift(x)),  z[a] = Y[f mod n] / n  for the signed frequency
//   f = ((a + C) mod N) - C in [-c, n - c)  (zero otherwise),
//   out = fftshift(IFFT_N(z))   (c = n/2, C = N/2).
// One CTA transforms T lines: it gathers them (shift and bit reversal folded
// into the load), runs the n-point forward FFT and the N-point inverse FFT
// in place in shared memory, and scatters the shifted result.  Lines are
// columns of a row-major volume (stride `inner`); loads/stores are coalesced
// across lines when inner >= T, along the line otherwise.
//
// Maps use FP32, the eigenvalue map FP64 (its in-support values ~1e-4 sit
// next to ~1 outside, and the per-voxel tolerance is relative).
#include "sk_internal.h"

#include <cstdlib>

namespace skb {

namespace {

template <typename R>
struct Cplx;
template <>
struct Cplx<float> {
  using T = float2;
};
template <>
struct Cplx<double> {
  using T = double2;
};

__device__ __forceinline__ int bitrev(int x, int bits) { return int(__brev(unsigned(x)) >> (32 - bits)); }

template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
  C r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}

// Padded position of element i in a line: one slot every 16 elements keeps
// the strided radix-16 accesses off a single bank.
__device__ __forceinline__ int pz(int i) { return i + (i >> 4); }

// In-place DIT FFT over 2^log_lines lines of length 2^log2len (bit-reversed
// input, padded positions, row stride ld), up to four radix-2 stages per pass
// done in registers (a thread owns 2^r elements spaced by the first stage's
// half distance); twiddles tw[k << log_tw_stride] = exp(-i 2 pi k / (len << log_tw_stride)),
// conjugated for the inverse.  All index math is shifts/masks.
template <typename C>
__device__ __forceinline__ void fft_lines(C* buf, int log_lines, int ld, int log2len, const C* tw, int log_tw_stride,
                                          bool inverse) {
  constexpr int RM = 4;
  // unrolled: with log2len known at compile time (the templated kernels) every
  // pass's radix r and index masks fold (the rolled loop stalled on branch
  // resolution: 12% of the C4 interpolation's samples)
#pragma unroll
  for (int s0 = 1; s0 <= log2len; s0 += RM) {
    const int r = min(RM, log2len - s0 + 1);
    const int hl0 = s0 - 1;
    const int glog = log2len - r;  // items per line
    const int total = 1 << (log_lines + glog);
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int line = e >> glog, it = e & ((1 << glog) - 1);
      const int j = it & ((1 << hl0) - 1), g = it >> hl0;
      const int base = (g << (hl0 + r)) + j;
      C* b = buf + line * ld;
      C x[1 << RM];
#pragma unroll
      for (int m = 0; m < (1 << RM); ++m)
        if (m < (1 << r)) x[m] = b[pz(base + (m << hl0))];
#pragma unroll
      for (int q = 0; q < RM; ++q) {
        if (q < r) {
          const int sh = log2len - (s0 + q) + log_tw_stride;
#pragma unroll
          for (int m = 0; m < (1 << RM); ++m) {
            if (m < (1 << r) && !(m & (1 << q))) {
              C w = tw[(j + ((m & ((1 << q) - 1)) << hl0)) << sh];
              if (inverse) w.y = -w.y;
              const C t = cmul(w, x[m + (1 << q)]);
              const C u = x[m];
              x[m].x = u.x + t.x;
              x[m].y = u.y + t.y;
              x[m + (1 << q)].x = u.x - t.x;
              x[m + (1 << q)].y = u.y - t.y;
            }
          }
        }
      }
#pragma unroll
      for (int m = 0; m < (1 << RM); ++m)
        if (m < (1 << r)) b[pz(base + (m << hl0))] = x[m];
    }
    __syncthreads();
  }
}

// Lines are (b, i) pairs of a [batch][len][inner] volume; inner = 2^log_inner.
// LOGN_ / LOGNN_ / LOGT_ >= 0 fix log2(n), log2(N), log2(T) at compile time
// (all index math then folds to constants); -1 = runtime sizes.
template <typename R, int LOGN_ = -1, int LOGNN_ = -1, int LOGT_ = -1>
__global__ void __launch_bounds__(256) interp_fft_kernel(const typename Cplx<R>::T* __restrict__ in,
                                                         typename Cplx<R>::T* __restrict__ out, unsigned lines_total,
                                                         int log_inner, int logT_arg, int logn_arg, int logN_arg) {
  using C = typename Cplx<R>::T;
  const int logn = LOGN_ >= 0 ? LOGN_ : logn_arg;
  const int logN = LOGNN_ >= 0 ? LOGNN_ : logN_arg;
  const int logT = LOGT_ >= 0 ? LOGT_ : logT_arg;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = 1 << logn, N = 1 << logN, T = 1 << logT;
  C* tw = reinterpret_cast<C*>(smem_raw);  // N/2 forward twiddles exp(-i 2 pi k / N)
  C* buf = tw + N / 2;                     // [T][ld], padded lines
  const int ld = N + N / 16 + 1;
  for (int k = threadIdx.x; k < N / 2; k += blockDim.x) {
    R s, c;
    if constexpr (sizeof(R) == 8) {
      sincospi(-2.0 * double(k) / double(N), &s, &c);
    } else {
      sincospif(-2.0f * float(k) / float(N), &s, &c);
    }
    tw[k].x = c;
    tw[k].y = s;
  }
  const unsigned l0 = blockIdx.x << logT;
  const int cl = n / 2, CL = N / 2;
  const bool across = log_inner >= logT;  // coalesce across lines (columns) or along the line
  const unsigned imask = (1u << log_inner) - 1u;
  auto src_index = [&](unsigned line, int a) -> size_t {  // element a of line (b, i)
    const unsigned b = line >> log_inner, i = line & imask;
    return ((size_t(b) << logn) + a) * (size_t(1) << log_inner) + i;
  };
  for (int e = threadIdx.x; e < (T << logn); e += blockDim.x) {
    const int t = across ? (e & (T - 1)) : (e >> logn);
    const int a = across ? (e >> logT) : (e & (n - 1));
    const unsigned line = l0 + t;
    C v;
    v.x = R(0);
    v.y = R(0);
    if (line < lines_total) v = in[src_index(line, (a + cl) & (n - 1))];  // ifftshift
    buf[t * ld + pz(bitrev(a, logn))] = v;
  }
  __syncthreads();
  fft_lines(buf, logT, ld, logn, tw, logN - logn, false);  // Y = FFT_n
  // Re-place Y into the zero-padded N line in bit-reversed order for the inverse.
  // Every thread reads its Y entries into registers first (in-place overlap).
  constexpr int kMaxPer = 16;  // T * n <= 16 * 256 (launcher)
  C keep[kMaxPer];
  int dst[kMaxPer];
  const R inv_n = R(1) / R(n);
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int e = threadIdx.x + u * 256;
    dst[u] = -1;
    if (e < (T << logn)) {
      const int t = e >> logn, k = e & (n - 1);
      const int f = k < n - cl ? k : k - n;  // signed frequency of Y[k] (f in [-c, n - c))
      const int a = (f + N) & (N - 1);       // its slot in the unshifted N-point spectrum
      C v = buf[t * ld + pz(k)];
      v.x *= inv_n;
      v.y *= inv_n;
      keep[u] = v;
      dst[u] = t * ld + pz(bitrev(a, logN));
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < T * ld; e += blockDim.x) {
    C z;
    z.x = R(0);
    z.y = R(0);
    buf[e] = z;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u)
    if (dst[u] >= 0) buf[dst[u]] = keep[u];
  __syncthreads();
  fft_lines(buf, logT, ld, logN, tw, 0, true);  // IFFT_N (unscaled, kspace_to_image)
  auto dst_index = [&](unsigned line, int jj) -> size_t {
    const unsigned b = line >> log_inner, i = line & imask;
    return ((size_t(b) << logN) + jj) * (size_t(1) << log_inner) + i;
  };
  for (int e = threadIdx.x; e < (T << logN); e += blockDim.x) {
    const int t = across ? (e & (T - 1)) : (e >> logN);
    const int jj = across ? (e >> logT) : (e & (N - 1));
    const unsigned line = l0 + t;
    if (line < lines_total) out[dst_index(line, jj)] = buf[t * ld + pz((jj - CL) & (N - 1))];  // fftshift
  }
}

// Factor-2 interpolation (N = 2n), the BASELINE grids' case.  With the
// reference's placement (signed frequencies f in [-c, n - c), c = n / 2) the
// unshifted N-point output w = IFFT_N(z) splits into
//   w[2k]     = y[k]                                (y = ifftshift(x): the input),
//   w[2k + 1] = (1/n) IFFT_n(Y[k] e^{i pi f(k) / n})[k]   (Y = FFT_n(y)),
// so a line costs FFT_n + IFFT_n on n-point buffers instead of FFT_n +
// IFFT_{2n} on a zero-padded 2n-point line (~40% fewer butterflies, half the
// shared memory per line, no zero fill).  out[jj] = w[(jj - n) mod 2n].
template <typename R, int LOGN_ = -1, int LOGT_ = -1>
__global__ void __launch_bounds__(256) interp2_fft_kernel(const typename Cplx<R>::T* __restrict__ in,
                                                          typename Cplx<R>::T* __restrict__ out, unsigned lines_total,
                                                          int log_inner, int logT_arg, int logn_arg) {
  using C = typename Cplx<R>::T;
  const int logn = LOGN_ >= 0 ? LOGN_ : logn_arg;
  const int logT = LOGT_ >= 0 ? LOGT_ : logT_arg;
  const int logN = logn + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = 1 << logn, N = 2 << logn, T = 1 << logT;
  C* tw = reinterpret_cast<C*>(smem_raw);  // n twiddles exp(-i 2 pi k / N)
  const int ld = n + n / 16 + 1;
  C* buf = tw + n;      // [T][ld] transform line
  C* ybuf = buf + T * ld;  // [T][ld] y = ifftshift(x), natural order (the even outputs)
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    R s, c;
    if constexpr (sizeof(R) == 8) {
      sincospi(-2.0 * double(k) / double(N), &s, &c);
    } else {
      sincospif(-2.0f * float(k) / float(N), &s, &c);
    }
    tw[k].x = c;
    tw[k].y = s;
  }
  const unsigned l0 = blockIdx.x << logT;
  const int cl = n / 2;
  const bool across = log_inner >= logT;
  const unsigned imask = (1u << log_inner) - 1u;
  const size_t stride = size_t(1) << log_inner;
  // loads: a thread's elements all in flight before the shared-memory
  // stores (one load-store pair per iteration kept one global load in flight:
  // the dominant long-scoreboard stall of the pass)
  constexpr int kLd = 16;  // T * n <= 16 * 256 (launcher)
  {
    C v[kLd];
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int e = threadIdx.x + u * 256;
      v[u].x = R(0);
      v[u].y = R(0);
      if (e < (T << logn)) {
        const int t = across ? (e & (T - 1)) : (e >> logn);
        const int a = across ? (e >> logT) : (e & (n - 1));
        const unsigned line = l0 + t;
        if (line < lines_total) {
          const unsigned b = line >> log_inner, i = line & imask;
          v[u] = in[((size_t(b) << logn) + ((a + cl) & (n - 1))) * stride + i];  // ifftshift
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int e = threadIdx.x + u * 256;
      if (e < (T << logn)) {
        const int t = across ? (e & (T - 1)) : (e >> logn);
        const int a = across ? (e >> logT) : (e & (n - 1));
        buf[t * ld + pz(bitrev(a, logn))] = v[u];
        ybuf[t * ld + pz(a)] = v[u];
      }
    }
  }
  __syncthreads();
  fft_lines(buf, logT, ld, logn, tw, 1, false);  // Y = FFT_n (twiddles tw[2k])
  // Y'[k] = Y[k] e^{2 pi i f / N} / n into bit-reversed order for the inverse
  constexpr int kMaxPer = 16;  // T * n <= 16 * 256 (launcher)
  C keep[kMaxPer];
  const R inv_n = R(1) / R(n);
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int e = threadIdx.x + u * 256;
    if (e < (T << logn)) {
      const int t = e >> logn, k = e & (n - 1);
      const int f = k < n - cl ? k : k - n;
      C w = tw[f >= 0 ? f : -f];
      if (f >= 0) w.y = -w.y;  // e^{+2 pi i f / N}
      const C y = buf[t * ld + pz(k)];
      C v = cmul(y, w);
      v.x *= inv_n;
      v.y *= inv_n;
      keep[u] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int e = threadIdx.x + u * 256;
    if (e < (T << logn)) {
      const int t = e >> logn, k = e & (n - 1);
      buf[t * ld + pz(bitrev(k, logn))] = keep[u];
    }
  }
  __syncthreads();
  fft_lines(buf, logT, ld, logn, tw, 1, true);  // odd outputs w[2k + 1]
  for (int e = threadIdx.x; e < (T << logN); e += blockDim.x) {
    const int t = across ? (e & (T - 1)) : (e >> logN);
    const int jj = across ? (e >> logT) : (e & (N - 1));
    const unsigned line = l0 + t;
    if (line < lines_total) {
      const int m = (jj - n) & (N - 1);  // fftshift
      const C v = (m & 1) ? buf[t * ld + pz(m >> 1)] : ybuf[t * ld + pz(m >> 1)];
      const unsigned b = line >> log_inner, i = line & imask;
      out[((size_t(b) << logN) + jj) * (size_t(1) << log_inner) + i] = v;
    }
  }
}

// Last interpolation pass fused with the sum-of-squares renormalisation of
// finalize (maps.cpp:240-250): the innermost (contiguous) axis, factor 2, one
// CTA per outer position with all Q channel lines (T = Q), so each output
// voxel's channels meet in shared memory: sos = sum_c |out_c|^2, then
// out_c / sqrt(sos) where sos > 0.  Saves the separate renormalisation pass
// (which reads the full-resolution maps twice and writes them once).
// in [Q][P][n] -> out [Q][P][2n]; blockIdx.y: slice of a stack [slices][Q][P][.].
template <int LOGN_, int LOGQ_>
__global__ void __launch_bounds__(256) interp2_sos_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                          unsigned positions, int logn_arg, int logq_arg) {
  using C = float2;
  using R = float;
  const int logn = LOGN_ >= 0 ? LOGN_ : logn_arg;
  const int logT = LOGQ_ >= 0 ? LOGQ_ : logq_arg;
  const int logN = logn + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = 1 << logn, N = 2 << logn, T = 1 << logT;
  SKB_DCHECK(blockDim.x == 256 && (T << logn) <= 16 * 256);  // keep[] below holds 16 values per thread
  C* tw = reinterpret_cast<C*>(smem_raw);
  const int ld = n + n / 16 + 1;
  C* buf = tw + n;
  C* ybuf = buf + T * ld;
  float* inv = reinterpret_cast<float*>(ybuf + T * ld);  // [N]
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    R sn, cs;
    sincospif(-2.0f * float(k) / float(N), &sn, &cs);
    tw[k].x = cs;
    tw[k].y = sn;
  }
  const unsigned p = blockIdx.x;
  in += (size_t(blockIdx.y) * T * positions) << logn;
  out += (size_t(blockIdx.y) * T * positions) << logN;
  const int cl = n / 2;
  {  // all of a thread's loads in flight before the shared-memory stores (as interp2_fft_kernel)
    constexpr int kLd = 16;
    C v[kLd];
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int e = threadIdx.x + u * 256;
      if (e < (T << logn)) {
        const int t = e >> logn, a = e & (n - 1);
        v[u] = in[((size_t(t) * positions + p) << logn) + ((a + cl) & (n - 1))];  // ifftshift
      }
    }
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int e = threadIdx.x + u * 256;
      if (e < (T << logn)) {
        const int t = e >> logn, a = e & (n - 1);
        buf[t * ld + pz(bitrev(a, logn))] = v[u];
        ybuf[t * ld + pz(a)] = v[u];
      }
    }
  }
  __syncthreads();
  fft_lines(buf, logT, ld, logn, tw, 1, false);
  constexpr int kMaxPer = 16;
  C keep[kMaxPer];
  const R inv_n = R(1) / R(n);
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int e = threadIdx.x + u * 256;
    if (e < (T << logn)) {
      const int t = e >> logn, k = e & (n - 1);
      const int f = k < n - cl ? k : k - n;
      C w = tw[f >= 0 ? f : -f];
      if (f >= 0) w.y = -w.y;
      const C y = buf[t * ld + pz(k)];
      C v = cmul(y, w);
      v.x *= inv_n;
      v.y *= inv_n;
      keep[u] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int e = threadIdx.x + u * 256;
    if (e < (T << logn)) {
      const int t = e >> logn, k = e & (n - 1);
      buf[t * ld + pz(bitrev(k, logn))] = keep[u];
    }
  }
  __syncthreads();
  fft_lines(buf, logT, ld, logn, tw, 1, true);
  // per output sample m (pre-fftshift index): sum over the Q channels
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    const C* src = (m & 1) ? buf : ybuf;
    float sos = 0.f;
    for (int t = 0; t < T; ++t) {
      const C v = src[t * ld + pz(m >> 1)];
      sos += v.x * v.x + v.y * v.y;
    }
    inv[m] = sos > 0.f ? 1.0f / sqrtf(sos) : 1.0f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < (T << logN); e += blockDim.x) {
    const int t = e >> logN, jj = e & (N - 1);
    const int m = (jj - n) & (N - 1);  // fftshift
    C v = (m & 1) ? buf[t * ld + pz(m >> 1)] : ybuf[t * ld + pz(m >> 1)];
    const float s = inv[m];
    v.x *= s;
    v.y *= s;
    out[((size_t(t) * positions + p) << logN) + jj] = v;
  }
}

// Centred transform along one axis (fft.cpp:71-112 kspace_to_image /
// image_to_kspace): out = fftshift(DFT_sign(ifftshift(x))) * scale, one CTA
// per T lines, same shared-memory FFT as the interpolation.
template <typename R>
__global__ void __launch_bounds__(256) centered_fft_kernel(const typename Cplx<R>::T* __restrict__ in,
                                                           typename Cplx<R>::T* __restrict__ out, unsigned lines_total,
                                                           int log_inner, int logT, int logN, bool inverse, R scale) {
  using C = typename Cplx<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = 1 << logN, T = 1 << logT;
  C* tw = reinterpret_cast<C*>(smem_raw);
  C* buf = tw + N / 2;
  const int ld = N + N / 16 + 1;
  for (int k = threadIdx.x; k < N / 2; k += blockDim.x) {
    R s, c;
    if constexpr (sizeof(R) == 8) {
      sincospi(-2.0 * double(k) / double(N), &s, &c);
    } else {
      sincospif(-2.0f * float(k) / float(N), &s, &c);
    }
    tw[k].x = c;
    tw[k].y = s;
  }
  const unsigned l0 = blockIdx.x << logT;
  const int CL = N / 2;
  const bool across = log_inner >= logT;
  const unsigned imask = (1u << log_inner) - 1u;
  auto index = [&](unsigned line, int a) -> size_t {
    const unsigned b = line >> log_inner, i = line & imask;
    return ((size_t(b) << logN) + a) * (size_t(1) << log_inner) + i;
  };
  for (int e = threadIdx.x; e < (T << logN); e += blockDim.x) {
    const int t = across ? (e & (T - 1)) : (e >> logN);
    const int a = across ? (e >> logT) : (e & (N - 1));
    const unsigned line = l0 + t;
    C v;
    v.x = R(0);
    v.y = R(0);
    if (line < lines_total) v = in[index(line, (a + CL) & (N - 1))];  // ifftshift
    buf[t * ld + pz(bitrev(a, logN))] = v;
  }
  __syncthreads();
  fft_lines(buf, logT, ld, logN, tw, 0, inverse);
  for (int e = threadIdx.x; e < (T << logN); e += blockDim.x) {
    const int t = across ? (e & (T - 1)) : (e >> logN);
    const int jj = across ? (e >> logT) : (e & (N - 1));
    const unsigned line = l0 + t;
    if (line < lines_total) {
      C v = buf[t * ld + pz((jj - CL) & (N - 1))];  // fftshift
      v.x *= scale;
      v.y *= scale;
      out[index(line, jj)] = v;
    }
  }
}

template <typename R, int LN, int LNN, int LT>
void launch_interp_k(sk_ctx* ctx, const void* in, void* out, unsigned lines, int log_inner, int logT, int logn,
                     int logN, size_t smem, unsigned blocks) {
  using C = typename Cplx<R>::T;
  set_smem_limit(reinterpret_cast<const void*>(interp_fft_kernel<R, LN, LNN, LT>), smem);
  interp_fft_kernel<R, LN, LNN, LT><<<blocks, 256, smem, ctx->stream>>>(static_cast<const C*>(in), static_cast<C*>(out),
                                                                        lines, log_inner, logT, logn, logN);
}

template <typename R, int LN, int LT>
void launch_interp2_k(sk_ctx* ctx, const void* in, void* out, unsigned lines, int log_inner, int logT, int logn,
                      size_t smem, unsigned blocks) {
  using C = typename Cplx<R>::T;
  set_smem_limit(reinterpret_cast<const void*>(interp2_fft_kernel<R, LN, LT>), smem);
  interp2_fft_kernel<R, LN, LT><<<blocks, 256, smem, ctx->stream>>>(static_cast<const C*>(in), static_cast<C*>(out),
                                                                    lines, log_inner, logT, logn);
}

template <typename R>
void launch_interp(sk_ctx* ctx, const void* in, void* out, i64 batch, int n, int N, i64 inner) {
  using C = typename Cplx<R>::T;
  const int logn = __builtin_ctz(unsigned(n)), logN = __builtin_ctz(unsigned(N));
  if (N == 2 * n) {  // factor 2: FFT_n + IFFT_n (the even outputs are the samples), C4 K5 4.26 -> 4.09 ms
    const int ldn = n + n / 16 + 1;
    int T = 32;
    while (T > 1 && (size_t(T) * ldn * 2 * sizeof(C) + size_t(n) * sizeof(C) > 110 * 1024 || T * n > 16 * 256)) T /= 2;
    const int logT = __builtin_ctz(unsigned(T));
    const size_t smem = size_t(T) * ldn * 2 * sizeof(C) + size_t(n) * sizeof(C);
    const i64 lines = batch * inner;
    const unsigned blocks = unsigned((lines + T - 1) / T);
    const int li = __builtin_ctzll(static_cast<unsigned long long>(inner));
    if (sizeof(R) == 4 && logn == 6 && logT == 5)
      launch_interp2_k<R, 6, 5>(ctx, in, out, unsigned(lines), li, logT, logn, smem, blocks);
    else if (sizeof(R) == 4 && logn == 7 && logT == 5)
      launch_interp2_k<R, 7, 5>(ctx, in, out, unsigned(lines), li, logT, logn, smem, blocks);
    else
      launch_interp2_k<R, -1, -1>(ctx, in, out, unsigned(lines), li, logT, logn, smem, blocks);
    ++ctx->launches;
    SKB_LAUNCH("interp2_fft_kernel");
    return;
  }
  // lines per block: keep T*n <= 16*256 (register staging) and smem <= ~110 KB
  const int ld = N + N / 16 + 1;
  int T = 32;
  while (T > 1 && (size_t(T) * ld * sizeof(C) + size_t(N / 2) * sizeof(C) > 110 * 1024 || T * n > 16 * 256)) T /= 2;
  const int logT = __builtin_ctz(unsigned(T));
  const size_t smem = size_t(T) * ld * sizeof(C) + size_t(N / 2) * sizeof(C);
  const i64 lines = batch * inner;
  const unsigned blocks = unsigned((lines + T - 1) / T);
  const int li = __builtin_ctzll(static_cast<unsigned long long>(inner));
  // compile-time sizes for the BASELINE grids (64 -> 128/256, 128 -> 256), runtime otherwise
  const int key = logn * 100 + logN * 10 + logT;
  if constexpr (sizeof(R) == 4) {
    switch (key) {
      case 6 * 100 + 7 * 10 + 5: launch_interp_k<R, 6, 7, 5>(ctx, in, out, unsigned(lines), li, logT, logn, logN, smem, blocks); break;
      case 6 * 100 + 8 * 10 + 5: launch_interp_k<R, 6, 8, 5>(ctx, in, out, unsigned(lines), li, logT, logn, logN, smem, blocks); break;
      case 7 * 100 + 8 * 10 + 5: launch_interp_k<R, 7, 8, 5>(ctx, in, out, unsigned(lines), li, logT, logn, logN, smem, blocks); break;
      default: launch_interp_k<R, -1, -1, -1>(ctx, in, out, unsigned(lines), li, logT, logn, logN, smem, blocks);
    }
  } else {
    launch_interp_k<R, -1, -1, -1>(ctx, in, out, unsigned(lines), li, logT, logn, logN, smem, blocks);
  }
  ++ctx->launches;
  SKB_LAUNCH("interp_fft_kernel");
}

}  // namespace

bool centered_fft_axis(sk_ctx* ctx, const void* in, void* out, i64 batch, int N, i64 inner, bool inverse,
                       double scale) {
  const bool pow2 = N >= 2 && !(N & (N - 1)) && inner > 0 && !(inner & (inner - 1));
  if (!pow2 || N > 1024 || batch * inner >= (i64(1) << 31)) return false;
  using C = float2;
  const int logN = __builtin_ctz(unsigned(N));
  const int ld = N + N / 16 + 1;
  int T = 32;
  while (T > 1 && size_t(T) * ld * sizeof(C) + size_t(N / 2) * sizeof(C) > 110 * 1024) T /= 2;
  const int logT = __builtin_ctz(unsigned(T));
  const size_t smem = size_t(T) * ld * sizeof(C) + size_t(N / 2) * sizeof(C);
  set_smem_limit(reinterpret_cast<const void*>(centered_fft_kernel<float>), smem);
  const i64 lines = batch * inner;
  centered_fft_kernel<float><<<unsigned((lines + T - 1) / T), 256, smem, ctx->stream>>>(
      static_cast<const C*>(in), static_cast<C*>(out), unsigned(lines),
      __builtin_ctzll(static_cast<unsigned long long>(inner)), logT, logN, inverse, float(scale));
  ++ctx->launches;
  SKB_LAUNCH("centered_fft_kernel");
  return true;
}

bool interp_last_axis_sos(sk_ctx* ctx, const float2* in, float2* out, int q, i64 positions, int n, int N,
                          int slices) {
  const bool pow2 = n >= 2 && !(n & (n - 1)) && q >= 1 && !(q & (q - 1));
  if (!pow2 || N != 2 * n || q > 32 || i64(q) * n > 16 * 256 || positions < 1 || positions >= (i64(1) << 31) ||
      slices < 1 || slices > 65535)
    return false;
  const int logn = __builtin_ctz(unsigned(n)), logq = __builtin_ctz(unsigned(q));
  const int ld = n + n / 16 + 1;
  const size_t smem = size_t(n) * sizeof(float2) + 2 * size_t(q) * ld * sizeof(float2) + size_t(N) * sizeof(float);
  if (smem > 200 * 1024) return false;
  auto go = [&](auto kern) {
    set_smem_limit(reinterpret_cast<const void*>(kern), smem);
    kern<<<dim3(unsigned(positions), unsigned(slices)), 256, smem, ctx->stream>>>(in, out, unsigned(positions), logn,
                                                                                 logq);
  };
  if (logn == 6 && logq == 5)
    go(interp2_sos_kernel<6, 5>);
  else if (logn == 7 && logq == 5)
    go(interp2_sos_kernel<7, 5>);
  else
    go(interp2_sos_kernel<-1, -1>);
  ++ctx->launches;
  SKB_LAUNCH("interp2_sos_kernel");
  return true;
}

bool interp_axis_fft(sk_ctx* ctx, const void* in, void* out, i64 batch, int n, int N, i64 inner, bool fp64) {
  const bool pow2 = n > 0 && N > 0 && !(n & (n - 1)) && !(N & (N - 1)) && inner > 0 && !(inner & (inner - 1));
  if (!pow2 || n > N || N > 1024 || n < 2 || batch * inner >= (i64(1) << 31)) return false;
  if (fp64)
    launch_interp<double>(ctx, in, out, batch, n, N, inner);
  else
    launch_interp<float>(ctx, in, out, batch, n, N, inner);
  return true;
}

}  // namespace skb
