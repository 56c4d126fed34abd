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

// In-place radix-2 DIT over `lines` lines of length len (bit-reversed input),
// twiddles tw[k * step] = exp(sign i 2 pi k / (len*step))... sign via conj flag.
template <typename C>
__device__ void fft_lines(C* buf, int lines, int ld, int len, int log2len, const C* tw, int tw_stride, bool inverse) {
  for (int s = 1; s <= log2len; ++s) {
    const int m = 1 << s, half = m >> 1;
    const int per_line = len >> 1;
    for (int e = threadIdx.x; e < lines * per_line; e += blockDim.x) {
      const int line = e / per_line, k = e % per_line;
      const int grp = k / half, j = k % half;
      const int i0 = grp * m + j, i1 = i0 + half;
      C w = tw[j * (len / m) * tw_stride];
      if (inverse) w.y = -w.y;
      C* b = buf + line * ld;
      const C u = b[i0];
      const C t = cmul(w, b[i1]);
      b[i0].x = u.x + t.x;
      b[i0].y = u.y + t.y;
      b[i1].x = u.x - t.x;
      b[i1].y = u.y - t.y;
    }
    __syncthreads();
  }
}

template <typename R>
__global__ void __launch_bounds__(256) interp_fft_kernel(const typename Cplx<R>::T* __restrict__ in,
                                                         typename Cplx<R>::T* __restrict__ out, i64 batch, int n, int N,
                                                         i64 inner, int T, int logn, int logN) {
  using C = typename Cplx<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tw = reinterpret_cast<C*>(smem_raw);  // N/2 forward twiddles exp(-i 2 pi k / N)
  C* buf = tw + N / 2;                     // [T][N + 1]
  const int ld = N + 1;
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
  // lines handled by this block: line id = blockIdx.x * T + t, line -> (b, i)
  const i64 lines_total = batch * inner;
  const i64 l0 = i64(blockIdx.x) * T;
  const int cl = n / 2, CL = N / 2;
  const bool across = inner >= T;  // coalesce across lines (columns) or along the line
  for (int e = threadIdx.x; e < T * n; e += blockDim.x) {
    const int t = across ? e % T : e / n;
    const int a = across ? e / T : e % n;
    const i64 line = l0 + t;
    C v;
    v.x = R(0);
    v.y = R(0);
    if (line < lines_total) {
      const i64 b = line / inner, i = line % inner;
      v = in[(b * n + (a + cl) % n) * inner + i];  // ifftshift
    }
    buf[t * ld + bitrev(a, logn)] = v;
  }
  __syncthreads();
  fft_lines(buf, T, ld, n, logn, tw, N / n, false);  // Y = FFT_n
  // Re-place Y into the zero-padded N line in bit-reversed order for the inverse.
  // Every thread reads its Y entries into registers first (in-place overlap).
  constexpr int kMaxPer = 16;
  C keep[kMaxPer];
  int dst[kMaxPer];
  int cnt = 0;
  const R inv_n = R(1) / R(n);
  for (int e = threadIdx.x; e < T * n && cnt < kMaxPer; e += blockDim.x, ++cnt) {
    const int t = e / n, k = e % n;
    const int f = k < n - cl ? k : k - n;  // signed frequency of Y[k] (f in [-c, n - c))
    const int a = (f + N) % N;             // its slot in the unshifted N-point spectrum
    C v = buf[t * ld + k];
    v.x *= inv_n;
    v.y *= inv_n;
    keep[cnt] = v;
    dst[cnt] = t * ld + bitrev(a, logN);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < T * N; e += blockDim.x) {
    const int t = e / N, a = e % N;
    C z;
    z.x = R(0);
    z.y = R(0);
    buf[t * ld + a] = z;
  }
  __syncthreads();
  for (int k = 0; k < cnt; ++k) buf[dst[k]] = keep[k];
  __syncthreads();
  fft_lines(buf, T, ld, N, logN, tw, 1, true);  // IFFT_N (unscaled, kspace_to_image)
  for (int e = threadIdx.x; e < T * N; e += blockDim.x) {
    const int t = across ? e % T : e / N;
    const int j = across ? e / T : e % N;
    const i64 line = l0 + t;
    if (line < lines_total) {
      const i64 b = line / inner, i = line % inner;
      out[(b * N + j) * inner + i] = buf[t * ld + (j - CL + N) % N];  // fftshift
    }
  }
}

template <typename R>
void launch_interp(sk_ctx* ctx, const void* in, void* out, i64 batch, int n, int N, i64 inner) {
  using C = typename Cplx<R>::T;
  const int logn = __builtin_ctz(unsigned(n)), logN = __builtin_ctz(unsigned(N));
  // lines per block: keep T*n <= 16*256 (register staging) and smem <= ~110 KB
  int T = 32;
  while (T > 1 && (size_t(T) * (N + 1) * sizeof(C) + size_t(N / 2) * sizeof(C) > 110 * 1024 || T * n > 16 * 256)) T /= 2;
  const size_t smem = size_t(T) * (N + 1) * sizeof(C) + size_t(N / 2) * sizeof(C);
  set_smem_limit(reinterpret_cast<const void*>(interp_fft_kernel<R>), smem);
  const i64 lines = batch * inner;
  const i64 blocks = (lines + T - 1) / T;
  interp_fft_kernel<R><<<unsigned(blocks), 256, smem, ctx->stream>>>(static_cast<const C*>(in), static_cast<C*>(out),
                                                                    batch, n, N, inner, T, logn, logN);
  ++ctx->launches;
  SKB_LAUNCH("interp_fft_kernel");
}

}  // namespace

bool interp_axis_fft(sk_ctx* ctx, const void* in, void* out, i64 batch, int n, int N, i64 inner, bool fp64) {
  const bool pow2 = n > 0 && N > 0 && !(n & (n - 1)) && !(N & (N - 1));
  if (!pow2 || n > N || N > 1024 || n < 2) return false;
  if (fp64)
    launch_interp<double>(ctx, in, out, batch, n, N, inner);
  else
    launch_interp<float>(ctx, in, out, batch, n, N, inner);
  return true;
}

}  // namespace skb
