// K4 for more than 64 channels (eigensolve.cpp:40-74 is generic in Q): the
// register-resident kernel of sk_power.cu holds one matrix row per thread and
// stops at Q = 64.  Here one CTA owns one voxel: the packed hi triangle
// (h = Q(Q+1)/2 entries) sits in shared memory, thread p forms row p of M v
// from it (upper part of the row contiguous, lower part read transposed with
// a conjugate), and the norms go through a block reduction.  Same arguments,
// control flow (fixed count, e_0 restart at it == 0, freeze below 1e-14) and
// epilogue (FP64 Rayleigh quotient on hi + lo, SoS + phase reference, mask)
// as power_kernel.  No BASELINE config takes this path; it is sized for
// correctness at any Q the shared memory holds (Q <= kWideMaxQ), not tuned.
#include "sk_internal.h"

namespace skb {

namespace {

constexpr int kWideThreads = 256;

template <typename T>
__device__ __forceinline__ T block_sum(T x, T* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();  // red is free again (previous readers are past their loop)
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  T s = T(0);
#pragma unroll
  for (int k = 0; k < kWideThreads / 32; ++k) s += red[k];
  return s;
}

__global__ void __launch_bounds__(kWideThreads) power_wide_kernel(PowerArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Q = a.q;
  const int h = Q * (Q + 1) / 2;
  float2* P = reinterpret_cast<float2*>(smem_raw);                 // [h] packed hi triangle
  float2* vs = P + ((h + 1) & ~1);                                // [Q] current iterate (16-byte aligned)
  double2* vd = reinterpret_cast<double2*>(vs + ((Q + 1) & ~1));  // [Q] final v in FP64
  double* redd = reinterpret_cast<double*>(vd + Q);               // [8]
  float* red = reinterpret_cast<float*>(redd + kWideThreads / 32);  // [8]
  const i64 ld = a.ld > 0 ? a.ld : a.n;
  const int p = threadIdx.x;
  const bool row = p < Q;
  const int base_p = row ? p * Q - p * (p - 1) / 2 : 0;  // packed index of (p, p)

  // row p of M times the vector in vs (M Hermitian, real diagonal: spatial_gram.cpp:140-146)
  auto matvec = [&]() -> float2 {
    float2 s = make_float2(0.f, 0.f);
    if (row) {
      int idx = p;  // packed (0, p)
      for (int c = 0; c < p; ++c) {  // M(p, c) = conj(P(c, p))
        const float2 m = P[idx], v = vs[c];
        s.x = fmaf(m.x, v.x, fmaf(m.y, v.y, s.x));
        s.y = fmaf(m.x, v.y, fmaf(-m.y, v.x, s.y));
        idx += Q - c - 1;
      }
      {
        const float2 v = vs[p];
        const float d = P[base_p].x;
        s.x = fmaf(d, v.x, s.x);
        s.y = fmaf(d, v.y, s.y);
      }
      for (int c = p + 1; c < Q; ++c) {
        const float2 m = P[base_p + (c - p)], v = vs[c];
        s.x = fmaf(m.x, v.x, fmaf(-m.y, v.y, s.x));
        s.y = fmaf(m.x, v.y, fmaf(m.y, v.x, s.y));
      }
    }
    return s;
  };

  for (i64 j = blockIdx.x; j < a.n; j += gridDim.x) {
    __syncthreads();  // the previous voxel's readers of P / vs / vd are done
    for (int e = threadIdx.x; e < h; e += kWideThreads) P[e] = a.planes[i64(e) * ld + j];
    const float init = rsqrtf(float(Q));
    float2 vp = row ? make_float2(init, 0.f) : make_float2(0.f, 0.f);
    if (row) vs[p] = vp;
    const float2 rc = (a.recon != nullptr && row) ? a.recon[i64(p) * ld + j] : make_float2(0.f, 0.f);
    __syncthreads();

    bool done = false;
    for (int it = 0; it < a.iters && !done; ++it) {
      const float2 mv = matvec();
      float2 w = make_float2(a.alpha * vp.x + a.beta * mv.x, a.alpha * vp.y + a.beta * mv.y);
      float n2 = block_sum(row ? w.x * w.x + w.y * w.y : 0.f, red);
      if (n2 < 1e-28f && it == 0) {  // annihilated all-ones start: restart from e_0 (eigensolve.cpp:56-63)
        vp = (p == 0) ? make_float2(1.f, 0.f) : make_float2(0.f, 0.f);
        // (B e_0)[p] = alpha e_0[p] + beta M[p][0], M[p][0] = conj(P(0, p))
        float2 m0 = make_float2(0.f, 0.f);
        if (row) m0 = p == 0 ? make_float2(P[0].x, 0.f) : make_float2(P[p].x, -P[p].y);
        w = make_float2(a.alpha * vp.x + a.beta * m0.x, a.alpha * vp.y + a.beta * m0.y);
        n2 = block_sum(row ? w.x * w.x + w.y * w.y : 0.f, red);
      }
      if (n2 < 1e-28f) {  // ||B v|| < 1e-14: keep the current v
        done = true;
      } else {
        const float inv = rsqrtf(n2);
        vp = make_float2(w.x * inv, w.y * inv);
      }
      __syncthreads();  // every read of vs by this iteration's products is done
      if (row) vs[p] = vp;
      __syncthreads();
    }

    // Rayleigh quotient in FP64 on hi + lo over the packed triangle (as power_kernel)
    if (row) vd[p] = make_double2(double(vp.x), double(vp.y));
    __syncthreads();
    double xd = 0.0;
    {
      int pp = 0, rowbase = 0;  // rowbase: packed index of (pp, pp)
      for (int e = threadIdx.x; e < h; e += kWideThreads) {
        while (e >= rowbase + Q - pp) rowbase += Q - pp++;
        const int cc = pp + (e - rowbase);
        const float2 hv = P[e];
        double mx = double(hv.x), my = double(hv.y);
        if (a.planes_lo != nullptr) {
          const float2 lv = lo_unpack(a.planes_lo[i64(e) * ld + j]);
          mx += double(lv.x);
          my += double(lv.y);
        }
        const double2 vpp = vd[pp], vc = vd[cc];
        if (pp == cc) {
          xd = fma(mx, vpp.x * vpp.x + vpp.y * vpp.y, xd);
        } else {
          const double tx = mx * vc.x - my * vc.y, ty = mx * vc.y + my * vc.x;
          xd = fma(2.0, vpp.x * tx + vpp.y * ty, xd);
        }
      }
    }
    const double mv64 = block_sum(xd, redd);
    const float vn2 = block_sum(row ? vp.x * vp.x + vp.y * vp.y : 0.f, red);
    if (a.recon != nullptr) {
      const float ux = block_sum(vp.x * rc.x + vp.y * rc.y, red);  // conj(v) . recon
      const float uy = block_sum(vp.x * rc.y - vp.y * rc.x, red);
      if (vn2 > 0.f) {
        const float inv = 1.0f / sqrtf(vn2);
        vp = make_float2(vp.x * inv, vp.y * inv);
      } else if (p == 0 && a.zeroed) {
        atomicAdd(a.zeroed, 1ull);
      }
      const float mag = sqrtf(ux * ux + uy * uy);
      if (mag > 0.f) {
        const float cx = ux / mag, cy = uy / mag;
        vp = make_float2(vp.x * cx - vp.y * cy, vp.x * cy + vp.y * cx);
      }
    }
    if (row) a.maps[i64(p) * ld + j] = vp;
    if (p == 0) {
      const float lam = float(mv64 * double(a.lam_scale));
      if (a.lambda) a.lambda[j] = lam;
      if (a.value) a.value[j] = float(double(a.alpha) * vn2 + double(a.beta) * mv64);
      if (a.mask) a.mask[j] = lam < a.mask_threshold ? 1 : 0;
    }
  }
}

size_t wide_smem(int q) {
  const size_t h = size_t(q) * (q + 1) / 2;
  return ((h + 1) & ~size_t(1)) * sizeof(float2) + size_t((q + 1) & ~1) * sizeof(float2) + size_t(q) * sizeof(double2) +
         (kWideThreads / 32) * (sizeof(double) + sizeof(float)) + 16;
}

}  // namespace

int power_wide_max_q() {
  int q = kWideThreads;
  while (q > 64 && wide_smem(q) > 220 * 1024) --q;
  return q;
}

void power_iteration_wide(sk_ctx* ctx, const PowerArgs& a) {
  if (a.n <= 0) return;
  if (a.q > power_wide_max_q())
    fail(SK_ERR_UNSUPPORTED, "eig_power_field: more than " + std::to_string(power_wide_max_q()) +
                                 " channels does not fit the shared-memory K4 path");
  const size_t smem = wide_smem(a.q);
  set_smem_limit(reinterpret_cast<const void*>(power_wide_kernel), smem);
  const i64 blocks = std::min<i64>(a.n, 8 * i64(ctx->sm_count));
  power_wide_kernel<<<unsigned(blocks), kWideThreads, smem, ctx->stream>>>(a);
  ++ctx->launches;
  SKB_LAUNCH("power_wide_kernel");
}

}  // namespace skb
