// K1 — FFT-way Gram C^H C on the ellipsoidal support (calibration.cpp:80-144).
//
// The reference forms, for every ordered channel pair, the full inverse
// transform of conj(S_p) * S_q on the zero-padded grid and then reads only
// the |Lambda - Lambda| lags n_s - n_t it needs.  Here one CTA per unordered
// pair p <= q (h = Q(Q+1)/2 CTAs) evaluates that inverse transform directly
// on the (4 tau + 1)^D lag box, axis by axis in shared memory (a pruned
// inverse DFT: the padded spectra never round-trip through a full grid), and
// writes block (p,q) and its Hermitian mirror (q,p) of the column-major Gram.
// Writing the mirror from the same pair makes the result exactly Hermitian,
// which is what the reference's final (G + G^H)/2 (calibration.cpp:142)
// enforces.
//
// Channel spectra S_q = F^-(calib_q placed at the pad-grid origin) are made
// beforehand by apply_axis (sk_axis.cu) with DFT matrices.
#include "sk_internal.h"

namespace skb {

namespace {

constexpr int kMaxLb = 29;  // 4*tau+1 for tau <= 7

__device__ __forceinline__ float2 cconj_mul(float2 a, float2 b) {  // conj(a) * b
  return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}

// e^{+i 2 pi m / P} for m in [0, P): twiddle tables for the three axes.  The
// pad extents are powers of two (calibration.cpp:89-93), so the phase index
// reduces with a mask (two's complement handles negative lags).
__device__ __forceinline__ float2 twiddle(const float2* tw, int k, int lag, int P) { return tw[(k * lag) & (P - 1)]; }

// LB > 0: the lag-box extent 4 tau + 1 fixed at compile time (register
// accumulators sized to it, the unstaged axis-0 contraction unrolled over four
// k0 with all their loads in flight); LB = 0: runtime extent (<= kMaxLb).
template <int LB>
__global__ void __launch_bounds__(512) gram_pairs_kernel(const float2* __restrict__ spectra, GramGeom g,
                                                         const int2* __restrict__ pairs,
                                                         const int* __restrict__ d_off,
                                                         const float2* __restrict__ tw_all,
                                                         float2* __restrict__ gram) {
  constexpr int kAcc = LB > 0 ? LB : kMaxLb;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int2 pq = pairs[blockIdx.x];
  const int p = pq.x, q = pq.y;
  const int P0 = g.pad[0], P1 = g.pad[1], P2 = g.pad[2];
  const int lb = LB > 0 ? LB : g.lb, t2 = 2 * g.tau;
  const i64 npad = i64(P0) * P1 * P2;
  // blockIdx.y: slice of a multislice group (its own spectra and Gram)
  spectra += i64(blockIdx.y) * g.q * npad;
  gram += i64(blockIdx.y) * (i64(g.q) * g.lam) * (i64(g.q) * g.lam);
  const int rest = P1 * P2;
  // twiddle tables (axis a at offset sum_{b<a} P_b)
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  for (int e = threadIdx.x; e < P0 + P1 + P2; e += blockDim.x) tw[e] = tw_all[e];
  float2* A = tw + (P0 + P1 + P2);            // [lb][P1][P2]
  float2* B = A + i64(lb) * rest;             // [lb][lb][P2]
  float2* box = B + i64(lb) * lb * P2;        // [lb]^D
  int* off = reinterpret_cast<int*>(box + (g.nd == 1 ? lb : (g.nd == 2 ? lb * lb : lb * lb * lb)));
  for (int e = threadIdx.x; e < g.lam; e += blockDim.x) off[e] = d_off[e];
  __syncthreads();

  const float2* Sp = spectra + i64(p) * npad;
  const float2* Sq = spectra + i64(q) * npad;
  const float2* tw0 = tw;
  const float2* tw1 = tw + P0;
  const float2* tw2 = tw + P0 + P1;

  // Stage A: contract axis 0 of conj(S_p) S_q onto the lb lags.
  float2* stageA_out = (g.nd == 1) ? box : A;
  float2* prod = reinterpret_cast<float2*>(off + ((g.lam + 3) & ~3));
  if (g.stage_prod) {
    // Small pad grid: stage the pair product once, then spread (lag, column)
    // items over all threads (a warp shares one lag -> broadcast twiddles).
    for (int e = threadIdx.x; e < npad; e += blockDim.x) prod[e] = cconj_mul(Sp[e], Sq[e]);
    __syncthreads();
    for (int item = threadIdx.x; item < lb * rest; item += blockDim.x) {
      const int l = item / rest, r = item % rest;
      float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
      int k0 = 0;
      for (; k0 + 1 < P0; k0 += 2) {
        cmac(acc0, prod[k0 * rest + r], twiddle(tw0, k0, l - t2, P0));
        cmac(acc1, prod[(k0 + 1) * rest + r], twiddle(tw0, k0 + 1, l - t2, P0));
      }
      if (k0 < P0) cmac(acc0, prod[k0 * rest + r], twiddle(tw0, k0, l - t2, P0));
      stageA_out[i64(l) * rest + r] = make_float2(acc0.x + acc1.x, acc0.y + acc1.y);
    }
  }
  for (int r = threadIdx.x; !g.stage_prod && r < rest; r += blockDim.x) {
    float2 acc[kAcc];
#pragma unroll
    for (int l = 0; l < kAcc; ++l) acc[l] = make_float2(0.f, 0.f);
    int k0 = 0;
    if (LB > 0) {
      constexpr int U = 4;  // P0 is a power of two >= 4 on this path (3-D pads)
      for (; k0 + U <= P0; k0 += U) {
        float2 sp[U], sq[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          sp[u] = Sp[i64(k0 + u) * rest + r];
          sq[u] = Sq[i64(k0 + u) * rest + r];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float2 prod = cconj_mul(sp[u], sq[u]);
#pragma unroll
          for (int l = 0; l < kAcc; ++l) cmac(acc[l], prod, twiddle(tw0, k0 + u, l - t2, P0));
        }
      }
    }
    for (; k0 < P0; ++k0) {
      const float2 prod = cconj_mul(Sp[i64(k0) * rest + r], Sq[i64(k0) * rest + r]);
#pragma unroll
      for (int l = 0; l < kAcc; ++l)
        if (l < lb) cmac(acc[l], prod, twiddle(tw0, k0, l - t2, P0));
    }
#pragma unroll
    for (int l = 0; l < kAcc; ++l)
      if (l < lb) stageA_out[i64(l) * rest + r] = acc[l];
  }
  __syncthreads();
  if (g.nd >= 2) {
    // Stage B: contract axis 1.  A[l0][k1][k2] -> B[l0][l1][k2]
    float2* stageB_out = (g.nd == 2) ? box : B;
    const int outs = lb * lb * P2;
    for (int e = threadIdx.x; e < outs; e += blockDim.x) {
      const int k2 = e % P2, l1 = (e / P2) % lb, l0 = e / (P2 * lb);
      float2 acc = make_float2(0.f, 0.f);
      const float2* src = A + (i64(l0) * P1) * P2 + k2;
      for (int k1 = 0; k1 < P1; ++k1) cmac(acc, src[i64(k1) * P2], twiddle(tw1, k1, l1 - t2, P1));
      stageB_out[e] = acc;
    }
    __syncthreads();
    if (g.nd == 3) {
      const int outs3 = lb * lb * lb;
      for (int e = threadIdx.x; e < outs3; e += blockDim.x) {
        const int l2 = e % lb, l01 = e / lb;
        float2 acc = make_float2(0.f, 0.f);
        const float2* src = B + i64(l01) * P2;
        for (int k2 = 0; k2 < P2; ++k2) cmac(acc, src[k2], twiddle(tw2, k2, l2 - t2, P2));
        box[e] = acc;
      }
      __syncthreads();
    }
  }
  // Scale by 1/N_pad (calibration.cpp:136); diagonal pairs made exactly Hermitian.
  const int nbox = g.nd == 1 ? lb : (g.nd == 2 ? lb * lb : lb * lb * lb);
  const int ctr = (nbox - 1) / 2;  // index of lag 0 (box is symmetric about its centre)
  const float inv = 1.0f / float(npad);
  for (int e = threadIdx.x; e <= ctr; e += blockDim.x) {
    const int m = 2 * ctr - e;
    float2 a = box[e], b = box[m];
    a.x *= inv; a.y *= inv; b.x *= inv; b.y *= inv;
    if (p == q) {
      const float2 s = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));
      a = s;
      b = make_float2(s.x, -s.y);
    }
    box[e] = a;
    box[m] = b;
  }
  __syncthreads();
  // Gram blocks (column-major, n x n): G[(p,s),(q,t)] = corr_pq[n_s - n_t].
  const i64 n = i64(g.q) * g.lam;
  const int lam = g.lam;
  for (int e = threadIdx.x; e < lam * lam; e += blockDim.x) {
    const int t = e / lam, s = e % lam;
    gram[(i64(p) * lam + s) + (i64(q) * lam + t) * n] = box[off[s] - off[t] + ctr];
  }
  if (p != q) {
    for (int e = threadIdx.x; e < lam * lam; e += blockDim.x) {
      const int s = e / lam, t = e % lam;
      const float2 v = box[off[s] - off[t] + ctr];
      gram[(i64(q) * lam + t) + (i64(p) * lam + s) * n] = make_float2(v.x, -v.y);
    }
  }
}

}  // namespace

size_t gram_pairs_smem(const GramGeom& g) {
  const int P0 = g.pad[0], P1 = g.pad[1], P2 = g.pad[2];
  const size_t lb = size_t(g.lb);
  const size_t nbox = g.nd == 1 ? lb : (g.nd == 2 ? lb * lb : lb * lb * lb);
  const size_t prod = g.stage_prod ? size_t(P0) * P1 * P2 : 0;
  return (size_t(P0 + P1 + P2) + lb * P1 * P2 + lb * lb * P2 + nbox + prod) * sizeof(float2) +
         size_t((g.lam + 3) & ~3) * sizeof(int);
}

void gram_pairs_launch(sk_ctx* ctx, const float2* spectra, const GramGeom& g_in, const int2* d_pairs, int npairs,
                       const int* d_off, const float2* d_tw, float2* gram, int slices) {
  GramGeom g = g_in;
  if (g.lb > kMaxLb) fail(9, "gram_fft: kernel radius > 7 is outside the B200 path");
  for (int a = 0; a < 3; ++a)
    if (g.pad[a] & (g.pad[a] - 1)) fail(9, "gram_fft: pad extents must be powers of two");
  g.stage_prod = 0;
  {
    GramGeom t = g;
    t.stage_prod = 1;
    if (gram_pairs_smem(t) <= 160 * 1024) g.stage_prod = 1;
  }
  const size_t smem = gram_pairs_smem(g);
  if (smem > 227 * 1024) fail(9, "gram_fft: padded calibration too large for the on-chip lag contraction");
  // 512 threads when the axis-0 contraction is unstaged (3-D pads: one CTA per
  // SM by shared memory, the column loop needs the warps), 256 otherwise
  // (2-D: 128 / 256 / 512 measured equal).
  const int threads = g.stage_prod ? 256 : 512;
  auto go = [&](auto kern) {
    set_smem_limit(reinterpret_cast<const void*>(kern), smem);
    kern<<<dim3(unsigned(npairs), unsigned(slices)), threads, smem, ctx->stream>>>(spectra, g, d_pairs, d_off, d_tw,
                                                                                   gram);
  };
  switch (g.lb) {  // lag-box extent fixed at compile time for the BASELINE radii, else run time
    case 9: go(gram_pairs_kernel<9>); break;
    case 13: go(gram_pairs_kernel<13>); break;
    case 17: go(gram_pairs_kernel<17>); break;
    case 21: go(gram_pairs_kernel<21>); break;
    case 25: go(gram_pairs_kernel<25>); break;
    default: go(gram_pairs_kernel<0>); break;
  }
  ++ctx->launches;
  SKB_LAUNCH("gram_pairs_kernel");
}

}  // namespace skb
