// Elementwise / layout kernels around the hot path: precision conversion for
// the FP64 eigensolve, GramField <-> packed-plane repacking for the
// reference-layout entry points, espirit_inplace (spatial_gram.cpp:156-164),
// the post-interpolation SoS renormalisation + support mask
// (maps.cpp:242-258), and the standalone normalize_maps epilogue.
#include "sk_internal.h"

#include <cmath>
#include <vector>

namespace skb {

namespace {

constexpr int kT = 256;
inline unsigned blocks_for(i64 n) { return unsigned(std::min<i64>((n + kT - 1) / kT, i64(1) << 30)); }

__global__ void c64_to_c128_kernel(const float2* __restrict__ in, double2* __restrict__ out, i64 n) {
  for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
    out[i] = make_double2(in[i].x, in[i].y);
}

__global__ void c128_to_c64_kernel(const double2* __restrict__ in, float2* __restrict__ out, i64 n) {
  for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
    out[i] = make_float2(float(in[i].x), float(in[i].y));
}

// GramField (voxel-major, col-major Q x Q) -> planes [h][N] (upper, p <= q).
__global__ void full_to_planes_kernel(const float2* __restrict__ field, i64 n, int q, float2* __restrict__ planes) {
  const int h = q * (q + 1) / 2;
  const i64 total = i64(h) * n;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const i64 j = e % n;
    int pair = int(e / n), p = 0;
    while (pair >= q - p) {
      pair -= q - p;
      ++p;
    }
    const int c = p + pair;
    planes[e] = field[j * q * q + i64(c) * q + p];  // (row p, col c)
  }
}

// planes -> GramField with the conjugate mirror and real diagonal
// (spatial_gram.cpp:133-146).
__global__ void planes_to_full_kernel(const float2* __restrict__ planes, const lo2* __restrict__ planes_lo, i64 n,
                                      int q, float2* __restrict__ field) {
  const i64 total = n * q * q;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const i64 j = e / (i64(q) * q);
    const int rc = int(e % (i64(q) * q));
    const int col = rc / q, row = rc % q;
    const int p = min(row, col), c = max(row, col);
    const int pair = p * q - p * (p - 1) / 2 + (c - p);
    float2 v = planes[i64(pair) * n + j];
    if (planes_lo) {
      const float2 l = lo_unpack(planes_lo[i64(pair) * n + j]);
      v = make_float2(float(double(v.x) + double(l.x)), float(double(v.y) + double(l.y)));
    }
    if (row > col) v.y = -v.y;
    if (row == col) v.y = 0.f;
    field[e] = v;
  }
}

__global__ void espirit_kernel(float2* __restrict__ field, i64 n, int q, float inv_lam) {
  const i64 total = n * q * q;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const int rc = int(e % (i64(q) * q));
    float2 v = field[e];
    v.x *= -inv_lam;
    v.y *= -inv_lam;
    if (rc / q == rc % q) v.x += 1.f;
    field[e] = v;
  }
}

// One thread per voxel: SoS renormalisation of the interpolated maps, lambda
// real part, support mask.
__global__ void renorm_mask_kernel(float2* __restrict__ maps, i64 n, int q, const float2* __restrict__ lam_c,
                                   float* __restrict__ lam, uint8_t* __restrict__ mask, float thr) {
  for (i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += i64(gridDim.x) * blockDim.x) {
    if (maps != nullptr) {
      float sos = 0.f;
      for (int c = 0; c < q; ++c) {
        const float2 v = maps[i64(c) * n + j];
        sos += v.x * v.x + v.y * v.y;
      }
      if (sos > 0.f) {
        const float inv = 1.0f / sqrtf(sos);
        for (int c = 0; c < q; ++c) {
          float2 v = maps[i64(c) * n + j];
          v.x *= inv;
          v.y *= inv;
          maps[i64(c) * n + j] = v;
        }
      }
    }
    if (lam_c != nullptr) {
      const float l = lam_c[j].x;
      if (lam) lam[j] = l;
      if (mask) mask[j] = l < thr ? 1 : 0;
    }
  }
}

// Channel-split renormalisation (z-slab sharding, maps.cpp:236-258): partial
// sum of squares over a channel subset, then division by the all-reduced sum.
__global__ void sos_accumulate_kernel(const float2* __restrict__ maps, i64 n, int q, float* __restrict__ sos) {
  for (i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += i64(gridDim.x) * blockDim.x) {
    float acc = sos[j];
    for (int c = 0; c < q; ++c) {
      const float2 v = maps[i64(c) * n + j];
      acc += v.x * v.x + v.y * v.y;
    }
    sos[j] = acc;
  }
}
__global__ void renorm_sos_kernel(float2* __restrict__ maps, i64 n, int q, const float* __restrict__ sos) {
  for (i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += i64(gridDim.x) * blockDim.x) {
    const float s = sos[j];
    if (s > 0.f) {
      const float inv = 1.0f / sqrtf(s);
      for (int c = 0; c < q; ++c) {
        float2 v = maps[i64(c) * n + j];
        v.x *= inv;
        v.y *= inv;
        maps[i64(c) * n + j] = v;
      }
    }
  }
}

__global__ void mask_only_kernel(const float* __restrict__ lam, i64 n, float thr, uint8_t* __restrict__ mask) {
  for (i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += i64(gridDim.x) * blockDim.x)
    mask[j] = lam[j] < thr ? 1 : 0;
}

__global__ void real_to_c128_kernel(const float* __restrict__ in, double2* __restrict__ out, i64 n) {
  for (i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += i64(gridDim.x) * blockDim.x)
    out[j] = make_double2(double(in[j]), 0.0);
}

__global__ void lam64_mask_kernel(const double2* __restrict__ lam_c, i64 n, float* __restrict__ lam,
                                  uint8_t* __restrict__ mask, float thr) {
  for (i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += i64(gridDim.x) * blockDim.x) {
    const double l = lam_c[j].x;  // interpolate_real keeps the real part (maps.cpp:92-99)
    if (lam) lam[j] = float(l);
    if (mask) mask[j] = l < double(thr) ? 1 : 0;
  }
}

__global__ void real_to_c64_kernel(const float* __restrict__ in, float2* __restrict__ out, i64 n) {
  for (i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += i64(gridDim.x) * blockDim.x)
    out[j] = make_float2(in[j], 0.f);
}

__global__ void copy_strided_kernel(const float2* __restrict__ src, i64 src_rs, i64 src_cs, float2* __restrict__ dst,
                                    i64 dst_rs, i64 dst_cs, i64 rows, i64 cols) {
  const i64 total = rows * cols;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const i64 c = e / rows, r = e % rows;
    dst[r * dst_rs + c * dst_cs] = src[r * src_rs + c * src_cs];
  }
}

// normalize_maps on channel-major maps (maps.cpp:117-172), one thread per voxel.
__global__ void normalize_kernel(float2* __restrict__ maps, i64 n, int q, const float2* __restrict__ recon,
                                 unsigned long long* zeroed) {
  for (i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += i64(gridDim.x) * blockDim.x) {
    float sos = 0.f;
    for (int c = 0; c < q; ++c) {
      const float2 v = maps[i64(c) * n + j];
      sos += v.x * v.x + v.y * v.y;
    }
    float inv = 1.f;
    if (sos > 0.f)
      inv = 1.0f / sqrtf(sos);
    else
      atomicAdd(zeroed, 1ull);
    float ux = 0.f, uy = 0.f;
    for (int c = 0; c < q; ++c) {
      const float2 v = maps[i64(c) * n + j];
      const float2 r = recon[i64(c) * n + j];
      const float vx = v.x * inv, vy = v.y * inv;
      ux += vx * r.x + vy * r.y;
      uy += vx * r.y - vy * r.x;
    }
    const float mag = sqrtf(ux * ux + uy * uy);
    float cx = 1.f, cy = 0.f;
    if (mag > 0.f) {
      cx = ux / mag;
      cy = uy / mag;
    }
    for (int c = 0; c < q; ++c) {
      const float2 v = maps[i64(c) * n + j];
      const float vx = v.x * inv, vy = v.y * inv;
      maps[i64(c) * n + j] = make_float2(vx * cx - vy * cy, vx * cy + vy * cx);
    }
  }
}

// Deterministic Gaussian-ish start block for the subspace eigensolver
// (hash-based, reproducible across runs and GPUs).
__device__ __forceinline__ unsigned int mix32(unsigned int x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
__global__ void random_block_kernel(double2* __restrict__ v, i64 n, i64 cols, i64 col0, unsigned int seed, i64 sv) {
  v += i64(blockIdx.y) * sv;  // batch: the same start block in every slice
  const i64 total = n * cols;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const i64 c = e / n + col0, r = e % n;
    const unsigned int h1 = mix32(unsigned(r) * 2654435761u ^ mix32(unsigned(c) + seed));
    const unsigned int h2 = mix32(h1 ^ 0x9e3779b9u);
    // sum of uniforms: cheap, symmetric, full-rank with probability 1
    const double u1 = (double(h1) + 0.5) / 4294967296.0 - 0.5;
    const double u2 = (double(h2) + 0.5) / 4294967296.0 - 0.5;
    v[r + c * n] = make_double2(u1, u2);
  }
}

// res[c] = || Y[:,c] - theta[c] V[:,c] ||^2  (one block per column)
__global__ void ritz_residual_kernel(const double2* __restrict__ y, const double2* __restrict__ v,
                                     const double* __restrict__ theta, i64 n, double* __restrict__ res, i64 sb,
                                     i64 sw) {
  y += i64(blockIdx.y) * sb;
  v += i64(blockIdx.y) * sb;
  theta += i64(blockIdx.y) * sw;
  res += i64(blockIdx.y) * sw;
  const i64 c = blockIdx.x;
  const double t = theta[c];
  double acc = 0.0;
  for (i64 r = threadIdx.x; r < n; r += blockDim.x) {
    const double2 a = y[r + c * n], b = v[r + c * n];
    const double dx = a.x - t * b.x, dy = a.y - t * b.y;
    acc += dx * dx + dy * dy;
  }
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (int(threadIdx.x) < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) res[c] = red[0];
}

// M = shift*I - A + alpha * U U^H is formed by the caller with ZHERK; this adds
// the diagonal shift and negates A in one pass (lower triangle only).
__global__ void shift_negate_kernel(const double2* __restrict__ a, double2* __restrict__ m, i64 n, double shift) {
  const i64 total = n * n;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const i64 c = e / n, r = e % n;
    if (r < c) continue;
    double2 v = a[e];
    v.x = -v.x;
    v.y = -v.y;
    if (r == c) v.x += shift;
    m[e] = v;
  }
}

}  // namespace

#define SKB_GRID(n) blocks_for(n), kT, 0, ctx->stream

// 2-D grid for `batch` slices: x covers one slice's elements, y the slices.
inline dim3 batch_grid(i64 per_slice, i64 batch) {
  return dim3(std::max(1u, std::min(blocks_for(per_slice), unsigned(std::max<i64>(1, 4096 / std::max<i64>(batch, 1))))),
              unsigned(batch));
}

void random_block(sk_ctx* ctx, double2* v, i64 n, i64 cols, i64 col0, unsigned int seed, i64 batch, i64 sv) {
  random_block_kernel<<<batch_grid(n * cols, batch), kT, 0, ctx->stream>>>(v, n, cols, col0, seed, sv);
  ++ctx->launches;
  SKB_LAUNCH("random_block");
}
void ritz_residuals(sk_ctx* ctx, const double2* y, const double2* v, const double* theta, i64 n, i64 cols,
                    double* res, i64 batch, i64 sb, i64 sw) {
  ritz_residual_kernel<<<dim3(unsigned(cols), unsigned(batch)), 256, 0, ctx->stream>>>(y, v, theta, n, res, sb, sw);
  ++ctx->launches;
  SKB_LAUNCH("ritz_residual");
}
void shift_negate(sk_ctx* ctx, const double2* a, double2* m, i64 n, double shift) {
  shift_negate_kernel<<<SKB_GRID(n * n)>>>(a, m, n, shift);
  ++ctx->launches;
  SKB_LAUNCH("shift_negate");
}

void c64_to_c128(sk_ctx* ctx, const float2* in, double2* out, i64 n) {
  c64_to_c128_kernel<<<SKB_GRID(n)>>>(in, out, n);
  ++ctx->launches;
  SKB_LAUNCH("c64_to_c128");
}
void c128_to_c64(sk_ctx* ctx, const double2* in, float2* out, i64 n) {
  c128_to_c64_kernel<<<SKB_GRID(n)>>>(in, out, n);
  ++ctx->launches;
  SKB_LAUNCH("c128_to_c64");
}
void field_full_to_planes(sk_ctx* ctx, const float2* field, i64 n, int q, float2* planes) {
  full_to_planes_kernel<<<SKB_GRID(n * q * (q + 1) / 2)>>>(field, n, q, planes);
  ++ctx->launches;
  SKB_LAUNCH("full_to_planes");
}
void planes_to_field_full(sk_ctx* ctx, const float2* planes, const lo2* planes_lo, i64 n, int q, float2* field) {
  planes_to_full_kernel<<<SKB_GRID(n * q * q)>>>(planes, planes_lo, n, q, field);
  ++ctx->launches;
  SKB_LAUNCH("planes_to_full");
}
void espirit_field(sk_ctx* ctx, float2* field, i64 n, int q, float inv_lam) {
  espirit_kernel<<<SKB_GRID(n * q * q)>>>(field, n, q, inv_lam);
  ++ctx->launches;
  SKB_LAUNCH("espirit");
}
void renormalize_and_mask(sk_ctx* ctx, float2* maps, i64 n, int q, const float2* lambda_c, float* lambda,
                          uint8_t* mask, float thr) {
  renorm_mask_kernel<<<SKB_GRID(n)>>>(maps, n, q, lambda_c, lambda, mask, thr);
  ++ctx->launches;
  SKB_LAUNCH("renorm_mask");
}
void sos_accumulate(sk_ctx* ctx, const float2* maps, i64 n, int q, float* sos) {
  sos_accumulate_kernel<<<SKB_GRID(n)>>>(maps, n, q, sos);
  ++ctx->launches;
  SKB_LAUNCH("sos_accumulate");
}
void renorm_with_sos(sk_ctx* ctx, float2* maps, i64 n, int q, const float* sos) {
  renorm_sos_kernel<<<SKB_GRID(n)>>>(maps, n, q, sos);
  ++ctx->launches;
  SKB_LAUNCH("renorm_sos");
}
// projection_residual (metrics.cpp:11-49), per block: sum_j ||rho_j||^2 and
// sum_j ||rho_j - c_j (c_j^H rho_j / ||c_j||^2)||^2 in FP64 (rho = unitary
// image of the k-space data, c = maps, voxel-major over channels).
__global__ void __launch_bounds__(256) residual_partial_kernel(const float2* __restrict__ img,
                                                               const float2* __restrict__ maps, i64 n, int q,
                                                               double2* __restrict__ partial) {
  double num = 0.0, den = 0.0;
  for (i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += i64(gridDim.x) * blockDim.x) {
    double rr = 0.0, cn = 0.0, dx = 0.0, dy = 0.0;
    for (int c = 0; c < q; ++c) {
      const float2 r = img[i64(c) * n + j], m = maps[i64(c) * n + j];
      rr += double(r.x) * r.x + double(r.y) * r.y;
      cn += double(m.x) * m.x + double(m.y) * m.y;
      dx += double(m.x) * r.x + double(m.y) * r.y;  // conj(c) . rho
      dy += double(m.x) * r.y - double(m.y) * r.x;
    }
    den += rr;
    if (cn > 0.0) {
      const double kx = dx / cn, ky = dy / cn;
      double s = 0.0;
      for (int c = 0; c < q; ++c) {
        const float2 r = img[i64(c) * n + j], m = maps[i64(c) * n + j];
        const double ex = double(r.x) - (double(m.x) * kx - double(m.y) * ky);
        const double ey = double(r.y) - (double(m.x) * ky + double(m.y) * kx);
        s += ex * ex + ey * ey;
      }
      num += s;
    } else {
      num += rr;
    }
  }
  __shared__ double sn[256], sd[256];
  sn[threadIdx.x] = num;
  sd[threadIdx.x] = den;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (int(threadIdx.x) < o) {
      sn[threadIdx.x] += sn[threadIdx.x + o];
      sd[threadIdx.x] += sd[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = make_double2(sn[0], sd[0]);
}

double projection_residual_value(sk_ctx* ctx, const float2* img, const float2* maps, i64 n, int q) {
  const int blocks = int(std::min<i64>((n + 255) / 256, 4 * i64(ctx->sm_count)));
  double2* partial = ctx->arena.get<double2>("res:partial", std::max(blocks, 1));
  residual_partial_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(img, maps, n, q, partial);
  ++ctx->launches;
  SKB_LAUNCH("residual_partial");
  std::vector<double2> h(size_t(std::max(blocks, 1)));
  SKB_CUDA(cudaMemcpyAsync(h.data(), partial, h.size() * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
  SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  double num = 0.0, den = 0.0;
  for (const double2& v : h) {  // fixed order: deterministic
    num += v.x;
    den += v.y;
  }
  return den > 0.0 ? std::sqrt(num / den) : 0.0;
}

// 3xTF32 split of complex operands for the K2 FP32 products (tensor cores):
// x = hi + lo with hi = tf32(x), lo = tf32(x - hi); complex n x m (column-major)
// becomes real [Re; Im] (2n x m) for the Gram and [Re, Im] (n x 2m) for the block.
// K-concatenated 3xTF32 operand: V' (2n x 4m, column-major) = [[V_hi, V_lo]; [0, V_hi]]
// so that [A_hi | A_lo] V' = [A_hi V_hi, A_hi V_lo + A_lo V_hi] in ONE GEMM that
// reads the split Gram once ([Re, Im] column blocks of width m inside each half).
__global__ void split_block_cat_kernel(const double2* __restrict__ v, i64 n, i64 m, float* __restrict__ vc, i64 sv,
                                       i64 svc) {
  v += i64(blockIdx.y) * sv;
  vc += i64(blockIdx.y) * svc;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < n * m; e += i64(gridDim.x) * blockDim.x) {
    const i64 r = e % n, c = e / n;
    const double2 x = v[e];
    const i64 ld = 2 * n;
    float h, l;
    tf32_split(float(x.x), h, l);
    vc[r + c * ld] = h;                    // [V_hi; 0], Re columns
    vc[n + r + c * ld] = 0.f;
    vc[r + (2 * m + c) * ld] = l;          // [V_lo; V_hi], Re columns
    vc[n + r + (2 * m + c) * ld] = h;
    tf32_split(float(x.y), h, l);
    vc[r + (m + c) * ld] = h;              // Im columns
    vc[n + r + (m + c) * ld] = 0.f;
    vc[r + (3 * m + c) * ld] = l;
    vc[n + r + (3 * m + c) * ld] = h;
  }
}
// Y from C' = [A_hi | A_lo] V' (2n x 4m): C = C'[:, :2m] + C'[:, 2m:], then as combine_block.
__global__ void combine_block_cat_kernel(const float* __restrict__ c, i64 n, i64 m, double2* __restrict__ y, i64 sc,
                                         i64 sy) {
  c += i64(blockIdx.y) * sc;
  y += i64(blockIdx.y) * sy;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < n * m; e += i64(gridDim.x) * blockDim.x) {
    const i64 r = e % n, k = e / n, ld = 2 * n, h = 2 * m * ld;
    const double c11 = double(c[r + k * ld]) + double(c[h + r + k * ld]);
    const double c21 = double(c[n + r + k * ld]) + double(c[h + n + r + k * ld]);
    const double c12 = double(c[r + (k + m) * ld]) + double(c[h + r + (k + m) * ld]);
    const double c22 = double(c[n + r + (k + m) * ld]) + double(c[h + n + r + (k + m) * ld]);
    y[e] = make_double2(c11 - c22, c12 + c21);
  }
}
void split_block_cat_tf32(sk_ctx* ctx, const double2* v, i64 n, i64 m, float* vc, i64 batch, i64 sv, i64 svc) {
  split_block_cat_kernel<<<batch_grid(n * m, batch), kT, 0, ctx->stream>>>(v, n, m, vc, sv, svc);
  ++ctx->launches;
  SKB_LAUNCH("split_block_cat");
}
void combine_block_cat(sk_ctx* ctx, const float* c, i64 n, i64 m, double2* y, i64 batch, i64 sc, i64 sy) {
  combine_block_cat_kernel<<<batch_grid(n * m, batch), kT, 0, ctx->stream>>>(c, n, m, y, sc, sy);
  ++ctx->launches;
  SKB_LAUNCH("combine_block_cat");
}

// One pass over the c64 Gram: the FP64 copy for the ZGEMM steps and the
// [Re; Im] TF32 hi/lo split for the 3xTF32 steps ([Re A; Im A] column blocks, hi then lo).
__global__ void promote_split_kernel(const float2* __restrict__ a, i64 n, double2* __restrict__ a64,
                                     float* __restrict__ hi, float* __restrict__ lo, i64 sa, i64 sh) {
  a += i64(blockIdx.y) * sa;
  a64 += i64(blockIdx.y) * sa;
  hi += i64(blockIdx.y) * sh;
  lo += i64(blockIdx.y) * sh;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < n * n; e += i64(gridDim.x) * blockDim.x) {
    const i64 r = e % n, c = e / n;
    const float2 v = a[e];
    a64[e] = make_double2(double(v.x), double(v.y));
    float h, l;
    tf32_split(v.x, h, l);
    hi[r + c * 2 * n] = h;
    lo[r + c * 2 * n] = l;
    tf32_split(v.y, h, l);
    hi[n + r + c * 2 * n] = h;
    lo[n + r + c * 2 * n] = l;
  }
}
void promote_split_gram(sk_ctx* ctx, const float2* a, i64 n, double2* a64, float* hi, float* lo, i64 batch, i64 sa,
                        i64 sh) {
  promote_split_kernel<<<batch_grid(n * n, batch), kT, 0, ctx->stream>>>(a, n, a64, hi, lo, sa, sh);
  ++ctx->launches;
  SKB_LAUNCH("promote_split");
}


// Batched FP64 products in the Gauss 3M form on real planes (the batched
// solver: three real DGEMMs per complex product instead of four; cuBLAS has
// no strided-batched ZGEMM-3M).  promote_split3: the c64 Gram -> planes
// [Re A][Im A][Re A + Im A] (n x n doubles each) and the TF32 split of
// promote_split; split3: V -> [Re V][Im V][Re V + Im V]; combine3: the three
// products T1 = Re A Re V, T2 = Im A Im V, T3 = (Re A + Im A)(Re V + Im V)
// -> Y = (T1 - T2) + i (T3 - T1 - T2).
__global__ void promote_split3_kernel(const float2* __restrict__ a, i64 n, double* __restrict__ a3,
                                      float* __restrict__ hi, float* __restrict__ lo, i64 sa, i64 sh) {
  a += i64(blockIdx.y) * sa;
  a3 += i64(blockIdx.y) * 3 * sa;
  hi += i64(blockIdx.y) * sh;
  lo += i64(blockIdx.y) * sh;
  const i64 nn = n * n;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < nn; e += i64(gridDim.x) * blockDim.x) {
    const i64 r = e % n, c = e / n;
    const float2 v = a[e];
    a3[e] = double(v.x);
    a3[nn + e] = double(v.y);
    a3[2 * nn + e] = double(v.x) + double(v.y);
    float h, l;
    tf32_split(v.x, h, l);
    hi[r + c * 2 * n] = h;
    lo[r + c * 2 * n] = l;
    tf32_split(v.y, h, l);
    hi[n + r + c * 2 * n] = h;
    lo[n + r + c * 2 * n] = l;
  }
}
__global__ void split3_kernel(const double2* __restrict__ v, i64 len, double* __restrict__ v3, i64 sv) {
  v += i64(blockIdx.y) * sv;
  v3 += i64(blockIdx.y) * 3 * len;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < len; e += i64(gridDim.x) * blockDim.x) {
    const double2 x = v[e];
    v3[e] = x.x;
    v3[len + e] = x.y;
    v3[2 * len + e] = x.x + x.y;
  }
}
__global__ void combine3_kernel(const double* __restrict__ t3, i64 len, double2* __restrict__ y, i64 sy) {
  t3 += i64(blockIdx.y) * 3 * len;
  y += i64(blockIdx.y) * sy;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < len; e += i64(gridDim.x) * blockDim.x) {
    const double t1 = t3[e], t2 = t3[len + e], t = t3[2 * len + e];
    y[e] = make_double2(t1 - t2, (t - t1) - t2);
  }
}
void promote_split3_gram(sk_ctx* ctx, const float2* a, i64 n, double* a3, float* hi, float* lo, i64 batch, i64 sa,
                         i64 sh) {
  promote_split3_kernel<<<batch_grid(n * n, batch), kT, 0, ctx->stream>>>(a, n, a3, hi, lo, sa, sh);
  ++ctx->launches;
  SKB_LAUNCH("promote_split3");
}
void split3_block(sk_ctx* ctx, const double2* v, i64 len, double* v3, i64 batch, i64 sv) {
  split3_kernel<<<batch_grid(len, batch), kT, 0, ctx->stream>>>(v, len, v3, sv);
  ++ctx->launches;
  SKB_LAUNCH("split3");
}
void combine3_block(sk_ctx* ctx, const double* t3, i64 len, double2* y, i64 batch, i64 sy) {
  combine3_kernel<<<batch_grid(len, batch), kT, 0, ctx->stream>>>(t3, len, y, sy);
  ++ctx->launches;
  SKB_LAUNCH("combine3");
}

void mask_kernel(sk_ctx* ctx, const float* lambda, i64 n, float thr, uint8_t* mask) {
  mask_only_kernel<<<SKB_GRID(n)>>>(lambda, n, thr, mask);
  ++ctx->launches;
  SKB_LAUNCH("mask");
}
void real_to_c128(sk_ctx* ctx, const float* in, double2* out, i64 n) {
  real_to_c128_kernel<<<SKB_GRID(n)>>>(in, out, n);
  ++ctx->launches;
  SKB_LAUNCH("real_to_c128");
}
void lam64_to_f32_mask(sk_ctx* ctx, const double2* lam_c, i64 n, float* lam, uint8_t* mask, float thr) {
  lam64_mask_kernel<<<SKB_GRID(n)>>>(lam_c, n, lam, mask, thr);
  ++ctx->launches;
  SKB_LAUNCH("lam64_mask");
}
void real_to_c64(sk_ctx* ctx, const float* in, float2* out, i64 n) {
  real_to_c64_kernel<<<SKB_GRID(n)>>>(in, out, n);
  ++ctx->launches;
  SKB_LAUNCH("real_to_c64");
}
void copy_strided(sk_ctx* ctx, const float2* src, i64 src_rs, i64 src_cs, float2* dst, i64 dst_rs, i64 dst_cs, i64 rows,
                  i64 cols) {
  copy_strided_kernel<<<SKB_GRID(rows * cols)>>>(src, src_rs, src_cs, dst, dst_rs, dst_cs, rows, cols);
  ++ctx->launches;
  SKB_LAUNCH("copy_strided");
}
void normalize_standalone(sk_ctx* ctx, float2* maps, i64 n, int q, const float2* recon, unsigned long long* zeroed) {
  normalize_kernel<<<SKB_GRID(n)>>>(maps, n, q, recon, zeroed);
  ++ctx->launches;
  SKB_LAUNCH("normalize");
}

}  // namespace skb

namespace skb {

// ---------------------------------------------------------------- parity probe
// Test hook behind sk_estimate_maps_probe: gathers of the Gram and of G(x)
// (hi + lo planes, FP64) at caller-chosen entries, and Frobenius norms with a
// fixed-order reduction.  Reads only; the pipeline's own buffers are untouched.
namespace {
__device__ __forceinline__ int pair_row(int pair, int q) {
  // pair index of (p, c), p <= c, is p*q - p*(p-1)/2 + (c - p): invert for p
  const double b = 2.0 * q + 1.0;
  int p = int((b - sqrt(b * b - 8.0 * pair)) * 0.5);
  while (p > 0 && p * q - p * (p - 1) / 2 > pair) --p;
  while ((p + 1) * q - (p + 1) * p / 2 <= pair) ++p;
  return p;
}

__global__ void probe_gram_kernel(const float2* __restrict__ g, i64 n, const long long* __restrict__ idx, i64 k,
                                  double2* __restrict__ out) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const float2 v = g[idx[2 * t] + idx[2 * t + 1] * n];
  out[t] = make_double2(v.x, v.y);
}

__global__ void probe_field_kernel(const float2* __restrict__ hi, const lo2* __restrict__ lo, i64 nvox, int q,
                                   const long long* __restrict__ idx, i64 k, double2* __restrict__ out) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const i64 j = idx[3 * t];
  const int row = int(idx[3 * t + 1]), col = int(idx[3 * t + 2]);
  const int p = min(row, col), c = max(row, col);
  const i64 pair = i64(p) * q - i64(p) * (p - 1) / 2 + (c - p);
  const float2 h = hi[pair * nvox + j];
  double re = h.x, im = h.y;
  if (lo) {
    const float2 l = lo_unpack(lo[pair * nvox + j]);
    re += double(l.x);
    im += double(l.y);
  }
  if (row > col) im = -im;   // G(q,p) = conj G(p,q)
  if (row == col) im = 0.0;  // spatial_gram.cpp:140-146
  out[t] = make_double2(re, im);
}

// sum |a (+ lo)|^2; planes mode (q > 0): element e lies in plane e / plane_len,
// off-diagonal planes count twice (their mirrored half of the full matrix).
__global__ void __launch_bounds__(256) sumsq_partial_kernel(const float2* __restrict__ a,
                                                            const lo2* __restrict__ lo, i64 total,
                                                            i64 plane_len, int q, double* __restrict__ partial) {
  __shared__ double s[256];
  double acc = 0.0;
  for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const float2 v = a[e];
    double re = v.x, im = v.y;
    if (lo) {
      const float2 l = lo_unpack(lo[e]);
      re += double(l.x);
      im += double(l.y);
    }
    double w = 1.0;
    if (q > 0) {
      const int pair = int(e / plane_len);
      const int p = pair_row(pair, q);
      const bool diag = pair == p * q - p * (p - 1) / 2;
      w = diag ? 1.0 : 2.0;
      if (diag) im = 0.0;
    }
    acc += w * (re * re + im * im);
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (int(threadIdx.x) < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = s[0];
}
}  // namespace

void probe_gather_gram(sk_ctx* ctx, const float2* gram, i64 n, const long long* idx, i64 k, double2* out) {
  if (k <= 0) return;
  probe_gram_kernel<<<unsigned((k + 255) / 256), 256, 0, ctx->stream>>>(gram, n, idx, k, out);
  ++ctx->launches;
  SKB_LAUNCH("probe_gram");
}

void probe_gather_field(sk_ctx* ctx, const float2* hi, const lo2* lo, i64 nvox, int q, const long long* idx,
                        i64 k, double2* out) {
  if (k <= 0) return;
  probe_field_kernel<<<unsigned((k + 255) / 256), 256, 0, ctx->stream>>>(hi, lo, nvox, q, idx, k, out);
  ++ctx->launches;
  SKB_LAUNCH("probe_field");
}

double probe_sumsq(sk_ctx* ctx, const float2* a, const lo2* lo, i64 total, i64 plane_len, int q) {
  const int blocks = int(std::max<i64>(1, std::min<i64>((total + 255) / 256, 4 * i64(ctx->sm_count))));
  double* partial = ctx->arena.get<double>("probe:partial", blocks);
  sumsq_partial_kernel<<<blocks, 256, 0, ctx->stream>>>(a, lo, total, plane_len, q, partial);
  ++ctx->launches;
  SKB_LAUNCH("probe_sumsq");
  std::vector<double> h(static_cast<size_t>(blocks));
  SKB_CUDA(cudaMemcpyAsync(h.data(), partial, h.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  double s = 0.0;
  for (double v : h) s += v;
  return s;
}

}  // namespace skb
