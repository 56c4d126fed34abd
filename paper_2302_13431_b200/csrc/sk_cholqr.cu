// CholQR for the K2 subspace block at b = 64, three lean kernels per pass
// (replaces cross_gram + cuSOLVER POTRF + cuBLAS TRSM, ~90 us per pass at
// n ~ 2.6k, whose cost is launch/latency, not arithmetic):
//
//  * gram64_kernel<HERM>: S = X^H X (HERM: ten lower 16x16 tiles) or
//    H = X^H Y (sixteen tiles).  ~n/144 rows per CTA; partials are summed
//    inside each 8-CTA cluster over DSMEM, and the last cluster to arrive
//    (one atomic ticket) sums the cluster partials in cluster order, so the
//    result is deterministic.  Output: full 64 x 64 column-major.
//  * chol64_kernel: one CTA, S = L L^H right-looking with the matrix in
//    registers (warp w owns rows w, 31-w, 32+w, 63-w: 130 lower entries per
//    warp), one barrier per pivot; then the inverses of the four 16 x 16
//    diagonal blocks of L.  A non-positive pivot raises *flag (POTRF info).
//  * trsm64_kernel: X <- X L^{-H} by 16-column blocks,
//    Y_b = (X_b - sum_{a<b} Y_a L_ba^H) Dinv_b^H; each row is owned by one
//    half-warp, so the solve needs no CTA barrier.
//
// The FP64 work is n*64^2*2 (gram) + 64^3/3 (Cholesky) + n*64^2*2 (solve)
// complex multiply-adds; the one-CTA Cholesky (~350k DFMA on one SM) is the
// latency floor of a pass.
#include "sk_internal.h"

#include <cooperative_groups.h>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace skb {

namespace {

// Block width B in {32, 64} (template parameter); rows of staged blocks are
// padded to B + 1 (conflict-free 16-byte columns).
constexpr int kQCluster = 8;     // CTAs per gram cluster
constexpr int kQStage = 32;      // rows staged per gram pass
constexpr int kQGramThreads = 256;
template <int B>
constexpr int chol_threads() { return 8 * B; }  // B / 4 warps: warp w owns columns 4w..4w+3

__device__ __forceinline__ double2 cfma_conj(double2 acc, double2 a, double2 b) {  // acc + conj(a) * b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cfms_conj_rev(double2 acc, double2 a, double2 b) {  // acc - a * conj(b)
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(-a.y, b.x, acc.y);
  acc.y = fma(a.x, b.y, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cfma_conj_rev(double2 acc, double2 a, double2 b) {  // acc + a * conj(b)
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y);
  acc.y = fma(-a.x, b.y, acc.y);
  return acc;
}

// Element (rr, col) of the n x m block Y held as the K-concatenated 3xTF32
// GEMM result C' (2n x 4m floats): C = C'[:, :2m] + C'[:, 2m:], Y = (C11 -
// C22) + i (C12 + C21) (as combine_block_cat, sk_misc.cu).
__device__ __forceinline__ double2 cat_load(const float* __restrict__ c, i64 n, int m, i64 rr, int col) {
  const i64 ld = 2 * n, h = 2 * i64(m) * ld;
  const float* p = c + rr + i64(col) * ld;
  const float* q = p + i64(m) * ld;
  const double c11 = double(p[0]) + double(p[h]);
  const double c21 = double(p[n]) + double(p[h + n]);
  const double c12 = double(q[0]) + double(q[h]);
  const double c22 = double(q[n]) + double(q[h + n]);
  return make_double2(c11 - c22, c12 + c21);
}
// The 3xTF32 operand V' = [[V_hi, V_lo]; [0, V_hi]] entries of element (rr, col) (as split_block_cat).
__device__ __forceinline__ void cat_store(float* __restrict__ vc, i64 n, int m, i64 rr, int col, double2 x) {
  const i64 ld = 2 * n;
  float h, l;
  tf32_split(float(x.x), h, l);
  vc[rr + i64(col) * ld] = h;
  vc[n + rr + i64(col) * ld] = 0.f;
  vc[rr + (2 * i64(m) + col) * ld] = l;
  vc[n + rr + (2 * i64(m) + col) * ld] = h;
  tf32_split(float(x.y), h, l);
  vc[rr + (i64(m) + col) * ld] = h;
  vc[n + rr + (i64(m) + col) * ld] = 0.f;
  vc[rr + (3 * i64(m) + col) * ld] = l;
  vc[n + rr + (3 * i64(m) + col) * ld] = h;
}

// 16 x 16 tiles of the B x B result, T = B / 16 per side: tile t -> (ti, tj);
// HERM lists the lower tiles row by row, else all T^2.
template <int B, bool HERM>
__host__ __device__ constexpr int tile_i(int t) {
  if (HERM) {
    int i = 0;
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    return i;
  }
  return t / (B / 16);
}
template <int B, bool HERM>
__host__ __device__ constexpr int tile_j(int t) {
  return HERM ? t - tile_i<B, HERM>(t) * (tile_i<B, HERM>(t) + 1) / 2 : t % (B / 16);
}
template <int B, bool HERM>
constexpr int n_tiles() { return HERM ? (B / 16) * (B / 16 + 1) / 2 : (B / 16) * (B / 16); }

template <int B, bool HERM>
__global__ void __cluster_dims__(kQCluster, 1, 1) __launch_bounds__(kQGramThreads)
    gram64_kernel(const double2* __restrict__ x, const double2* __restrict__ y, i64 n, int rows,
                  double2* __restrict__ cpart, unsigned* __restrict__ counter, double2* __restrict__ out, i64 sx,
                  const float* __restrict__ ccat, i64 sc) {
  constexpr int NT = n_tiles<B, HERM>();
  constexpr int kQ = B, kQLd = B + 1;
  // batch (multislice K2): slice blockIdx.y, its own partials, ticket and output
  x += i64(blockIdx.y) * sx;
  y += i64(blockIdx.y) * sx;
  if (ccat) ccat += i64(blockIdx.y) * sc;  // HERM only: X taken from the concatenated GEMM result
  out += i64(blockIdx.y) * kQ * kQ;
  cpart += i64(blockIdx.y) * (gridDim.x / kQCluster) * NT * kQGramThreads;
  counter += blockIdx.y;
  constexpr int PER = NT * kQGramThreads / kQCluster;  // elements each cluster rank reduces
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* xs = reinterpret_cast<double2*>(smem_raw);  // [kQStage][kQLd]
  double2* ys = HERM ? xs : xs + kQStage * kQLd;
  double2* part = xs + (HERM ? 1 : 2) * kQStage * kQLd;  // [NT][256]
  __shared__ int last_flag;
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x;
  SKB_DCHECK(blockDim.x == kQGramThreads && gridDim.x % kQCluster == 0);
  const int r = tid >> 4, c = tid & 15;
  const i64 row0 = i64(blockIdx.x) * rows, row1 = min(n, row0 + rows);
  double2 acc[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t] = make_double2(0.0, 0.0);
  for (i64 rs = row0; rs < row1; rs += kQStage) {
    constexpr int kPer = kQStage * kQ / kQGramThreads;  // 8 (B = 64), 4 (B = 32)
    double2 v[kPer], w[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + kQGramThreads * u;
      const int k = e % kQStage, col = e / kQStage;  // lanes along rows: column-major X (coalesced)
      const i64 rr = rs + k;
      v[u] = rr < row1 ? (HERM && ccat ? cat_load(ccat, n, kQ, rr, col) : x[rr + i64(col) * n])
                       : make_double2(0.0, 0.0);
      if (!HERM) w[u] = rr < row1 ? y[rr + i64(col) * n] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + kQGramThreads * u;
      const int k = e % kQStage, col = e / kQStage;
      xs[k * kQLd + col] = v[u];
      if (!HERM) ys[k * kQLd + col] = w[u];
    }
    __syncthreads();
    const int kn = int(min(i64(kQStage), row1 - rs));
#pragma unroll 2
    for (int k = 0; k < kn; ++k) {
      double2 xi[B / 16], yj[B / 16];
#pragma unroll
      for (int a = 0; a < B / 16; ++a) {
        xi[a] = xs[k * kQLd + 16 * a + r];
        yj[a] = ys[k * kQLd + 16 * a + c];
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) acc[t] = cfma_conj(acc[t], xi[tile_i<B, HERM>(t)], yj[tile_j<B, HERM>(t)]);
    }
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) part[t * kQGramThreads + tid] = acc[t];
  cluster.sync();
  const int rank = int(cluster.block_rank());
  const int cid = blockIdx.x / kQCluster, ncl = gridDim.x / kQCluster;
  for (int e = tid; e < PER; e += kQGramThreads) {
    const int g = rank * PER + e;
    double2 s = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < kQCluster; ++q) {
      const double2 p = cluster.map_shared_rank(part, q)[g];
      s.x += p.x;
      s.y += p.y;
    }
    cpart[i64(cid) * NT * kQGramThreads + g] = s;
  }
  __threadfence();
  cluster.sync();
  if (rank == 0 && tid == 0) last_flag = atomicAdd(counter, 1u) == unsigned(ncl - 1);
  cluster.sync();
  const bool last = *cluster.map_shared_rank(&last_flag, 0) != 0;
  if (last) {
    __threadfence();
    for (int e = tid; e < PER; e += kQGramThreads) {
      const int g = rank * PER + e;
      double2 s = make_double2(0.0, 0.0);
      int q = 0;
      for (; q + 8 <= ncl; q += 8) {  // cluster order (deterministic), eight loads in flight
        double2 p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = __ldcg(&cpart[i64(q + u) * NT * kQGramThreads + g]);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          s.x += p[u].x;
          s.y += p[u].y;
        }
      }
      for (; q < ncl; ++q) {
        const double2 p = __ldcg(&cpart[i64(q) * NT * kQGramThreads + g]);
        s.x += p.x;
        s.y += p.y;
      }
      const int t = g / kQGramThreads, tt = g % kQGramThreads;
      const int ti = tile_i<B, HERM>(t), tj = tile_j<B, HERM>(t);
      const int i = 16 * ti + (tt >> 4), j = 16 * tj + (tt & 15);
      if (!HERM) {
        out[i + kQ * j] = s;
      } else if (i > j) {  // exactly Hermitian: the lower entry and its mirror
        out[i + kQ * j] = s;
        out[j + kQ * i] = make_double2(s.x, -s.y);
      } else if (i == j) {
        out[i + kQ * i] = make_double2(s.x, 0.0);
      }
    }
    if (rank == 0 && tid == 0) *counter = 0u;  // ready for the next launch (stream order)
  }
  cluster.sync();  // rank 0's last_flag stays readable until every rank has read it
}

// Warp w owns the four columns 4w..4w+3 (slot c), lane l the rows l and
// l + 32 (slot h).  Step s (one barrier): block s of L (columns 4s..4s+3) is
// published in colb; every warp w > s applies the rank-4 update to its
// columns, and warp s + 1 then factors its own 4 x 4 diagonal block inside
// the warp (shuffles only: diagonal and the three sub-diagonal entries of
// the pivot column, 1/sqrt(d), scale, update the remaining columns) and
// publishes block s + 1.  The pivot chain therefore crosses a CTA barrier
// once per four pivots; the rank-4 updates of the other warps overlap it.
template <int B>
__device__ __forceinline__ void chol64_factor4(double2 (&a)[4][B / 32], double2 (*pub)[B], double2* Ls, double* rsv,
                                               int w, int lane, int* flag) {
  constexpr int H = B / 32, kQLd = B + 1;
  const int j0 = 4 * w, hj = j0 >> 5;  // the block's rows j0..j0+3 lie in row slot hj
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = j0 + q;
    const double2 cj = a[q][H > 1 ? hj : 0];
    const double d = __shfl_sync(0xffffffffu, cj.x, j & 31);
    double2 cq[4];
#pragma unroll
    for (int t = q + 1; t < 4; ++t) {  // unscaled entries (j0 + t, j)
      cq[t].x = __shfl_sync(0xffffffffu, cj.x, (j0 + t) & 31);
      cq[t].y = __shfl_sync(0xffffffffu, cj.y, (j0 + t) & 31);
    }
    const bool ok = d > 0.0;
    const double r = rsqrt(ok ? d : 1e-300), r2 = r * r;  // library rsqrt: ~75 cycles (a float seed + Newton is slower)
    if (lane == 0) {
      if (!ok) atomicExch(flag, 1);
      rsv[j] = r;
    }
#pragma unroll
    for (int t = q + 1; t < 4; ++t)
#pragma unroll
      for (int h = 0; h < H; ++h) {  // a(i, j0+t) -= c(i) conj(c(j0+t)) / d
        const double2 ci = a[q][h];
        const double tr = ci.x * cq[t].x + ci.y * cq[t].y, tim = ci.y * cq[t].x - ci.x * cq[t].y;
        a[t][h].x = fma(-tr, r2, a[t][h].x);
        a[t][h].y = fma(-tim, r2, a[t][h].y);
      }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      a[q][h].x *= r;
      a[q][h].y = (lane + 32 * h == j) ? 0.0 : a[q][h].y * r;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int i = lane + 32 * h;
      if (i >= j0 + q) {
        pub[q][i] = a[q][h];
        Ls[i * kQLd + j0 + q] = a[q][h];
      }
    }
}

template <int B>
__global__ void __launch_bounds__(chol_threads<B>()) chol64_kernel(const double2* __restrict__ s_in,
                                                                  double2* __restrict__ l_out,
                                                                  double2* __restrict__ dinv_out, int* flag) {
  constexpr int kQ = B, kQLd = B + 1, H = B / 32, NB = B / 16;
  SKB_DCHECK(blockDim.x == chol_threads<B>());  // warp w owns columns 4w..4w+3
  // batch (multislice K2): one CTA per slice
  s_in += i64(blockIdx.x) * kQ * kQ;
  l_out += i64(blockIdx.x) * kQ * kQ;
  dinv_out += i64(blockIdx.x) * NB * 256;
  flag += 3 * blockIdx.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ls = reinterpret_cast<double2*>(smem_raw);  // [B][B + 1], L (lower)
  __shared__ double2 colb[2][4][kQ];                    // block s of L (four columns), double-buffered
  __shared__ double rsv[kQ];                            // 1/L[k][k]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int j0 = 4 * w;
  double2 a[4][H];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int h = 0; h < H; ++h) a[c][h] = s_in[(lane + 32 * h) + kQ * (j0 + c)];  // S[i][j], coalesced in i
  {
    if (w == 0) chol64_factor4<B>(a, colb[0], Ls, rsv, w, lane, flag);
#pragma unroll 1
    for (int s = 0; s < B / 4 - 1; ++s) {
      __syncthreads();
      if (w > s) {
        const double2 (*cb)[kQ] = colb[s & 1];
        double2 li[4][H];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < H; ++h) li[q][h] = cb[q][lane + 32 * h];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double2 lj[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) lj[q] = cb[q][j0 + c];
#pragma unroll
          for (int h = 0; h < H; ++h) {
            if (H == 2 && h == 0 && w >= 8) continue;  // columns >= 32 have no entries in rows < 32
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // a -= l(i, q) conj(l(j, q))
              a[c][h].x = fma(-li[q][h].x, lj[q].x, a[c][h].x);
              a[c][h].x = fma(-li[q][h].y, lj[q].y, a[c][h].x);
              a[c][h].y = fma(-li[q][h].y, lj[q].x, a[c][h].y);
              a[c][h].y = fma(li[q][h].x, lj[q].y, a[c][h].y);
            }
          }
        }
      }
      if (w == s + 1) chol64_factor4<B>(a, colb[(s + 1) & 1], Ls, rsv, w, lane, flag);
    }
  }
  __syncthreads();
  for (int e = tid; e < kQ * kQ; e += chol_threads<B>()) {
    const int i = e % kQ, j = e / kQ;
    l_out[e] = i >= j ? Ls[i * kQLd + j] : make_double2(0.0, 0.0);
  }
  // Dinv_b = L_bb^{-1}: warp b, lane c < 16 forms column c by forward
  // substitution with the column in registers (x_m = 0 for m < c, so the
  // sums need no bounds; the newest term enters last: short chain).
  if (w < NB && lane < 16) {
    const int b = w, c = lane, o = 16 * b;
    double2 xv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < c) {
        xv[i] = make_double2(0.0, 0.0);
      } else if (i == c) {
        xv[i] = make_double2(rsv[o + i], 0.0);
      } else {
        double2 sum = make_double2(0.0, 0.0);
#pragma unroll
        for (int m = 0; m < i; ++m) {
          const double2 l = Ls[(o + i) * kQLd + o + m];
          sum.x = fma(l.x, xv[m].x, fma(-l.y, xv[m].y, sum.x));
          sum.y = fma(l.x, xv[m].y, fma(l.y, xv[m].x, sum.y));
        }
        const double ri = rsv[o + i];
        xv[i] = make_double2(-sum.x * ri, -sum.y * ri);
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) dinv_out[b * 256 + i * 16 + c] = xv[i];
  }
}

// X (n x B column-major) <- X L^{-H}; `rows` rows per CTA, 16 threads per row.
template <int B>
__global__ void __launch_bounds__(1024) trsm64_kernel(double2* __restrict__ x, i64 n, int rows,
                                                      const double2* __restrict__ l,
                                                      const double2* __restrict__ dinv, i64 sx,
                                                      const float* __restrict__ ccat, i64 sc,
                                                      float* __restrict__ vcat, i64 svc) {
  constexpr int kQ = B, kQLd = B + 1, NB = B / 16;
  x += i64(blockIdx.y) * sx;  // batch: slice blockIdx.y
  if (ccat) ccat += i64(blockIdx.y) * sc;
  if (vcat) vcat += i64(blockIdx.y) * svc;
  l += i64(blockIdx.y) * kQ * kQ;
  dinv += i64(blockIdx.y) * NB * 256;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ls = reinterpret_cast<double2*>(smem_raw);  // [B][B + 1]
  double2* Ds = Ls + kQ * kQLd;                         // [NB][16][17]
  double2* Xs = Ds + NB * 16 * 17;                      // [rows][B + 1]
  const int tid = threadIdx.x, nt = blockDim.x;
  SKB_DCHECK(rows >= 1 && rows <= 64 && rows * 16 <= nt + 15);  // one half-warp per staged row
  const i64 row0 = i64(blockIdx.x) * rows;
  const int nr = int(min(i64(rows), n - row0));
  // all loads of a thread in flight together (one L2 round trip, not one per element)
  for (int e0 = 0; e0 < kQ * kQ; e0 += 8 * nt) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * nt;
      v[u] = e < kQ * kQ ? l[e] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * nt;
      if (e < kQ * kQ) Ls[(e % kQ) * kQLd + (e / kQ)] = v[u];
    }
  }
  for (int e0 = 0; e0 < NB * 256; e0 += 4 * nt) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + tid + u * nt;
      v[u] = e < NB * 256 ? dinv[e] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + tid + u * nt;
      if (e < NB * 256) Ds[(e >> 8) * 272 + ((e >> 4) & 15) * 17 + (e & 15)] = v[u];
    }
  }
  for (int e0 = 0; e0 < rows * kQ; e0 += 4 * nt) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + tid + u * nt;
      const int rr = e % rows, col = e / rows;
      v[u] = (e < rows * kQ && rr < nr)
                 ? (ccat ? cat_load(ccat, n, kQ, row0 + rr, col) : x[row0 + rr + i64(col) * n])
                 : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + tid + u * nt;
      if (e < rows * kQ) Xs[(e % rows) * kQLd + e / rows] = v[u];
    }
  }
  __syncthreads();
  const int r = tid >> 4, c = tid & 15;
  if (r < rows) {  // the 16 threads of row r are one half-warp
    const unsigned hmask = 0xffffu << (tid & 16);
    double2* xr = Xs + r * kQLd;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = 16 * b + c;
      double2 t0 = xr[j], t1 = make_double2(0.0, 0.0);
      const double2* lj = Ls + j * kQLd;
#pragma unroll
      for (int m = 0; m < 16 * b; m += 2) {
        t0 = cfms_conj_rev(t0, xr[m], lj[m]);
        t1 = cfms_conj_rev(t1, xr[m + 1], lj[m + 1]);
      }
      t0.x += t1.x;
      t0.y += t1.y;
      __syncwarp(hmask);
      xr[j] = t0;  // T_b
      __syncwarp(hmask);
      const double2* dc = Ds + b * 272 + c * 17;
      double2 y0 = make_double2(0.0, 0.0), y1 = y0;
#pragma unroll
      for (int m = 0; m < 16; m += 2) {  // Dinv_b upper part is zero
        y0 = cfma_conj_rev(y0, xr[16 * b + m], dc[m]);
        y1 = cfma_conj_rev(y1, xr[16 * b + m + 1], dc[m + 1]);
      }
      __syncwarp(hmask);
      xr[j] = make_double2(y0.x + y1.x, y0.y + y1.y);
      __syncwarp(hmask);
    }
  }
  __syncthreads();
  for (int e = tid; e < nr * kQ; e += nt) {
    const int rr = e % nr, col = e / nr;
    const double2 v = Xs[rr * kQLd + col];
    x[row0 + rr + i64(col) * n] = v;
    if (vcat) cat_store(vcat, n, kQ, row0 + rr, col, v);
  }
}

// Ticket counters of the gram64 reductions, one per slice of a batch (each
// launch leaves its counter at zero again).
constexpr i64 kMaxBatch = 4096;
unsigned* gram_counter(sk_ctx* ctx) {
  static const char* kName = "cq:counter";
  auto it = ctx->arena_zeroed.find(kName);
  if (it != ctx->arena_zeroed.end()) return static_cast<unsigned*>(it->second);
  unsigned* p = ctx->arena.get<unsigned>(kName, kMaxBatch);
  SKB_CUDA(cudaMemsetAsync(p, 0, kMaxBatch * sizeof(unsigned), ctx->stream));
  ctx->arena_zeroed[kName] = p;
  return p;
}

template <int B, bool HERM>
void launch_gram64(sk_ctx* ctx, const double2* x, const double2* y, i64 n, double2* out, i64 batch = 1, i64 sx = 0,
                   const float* ccat = nullptr, i64 sc = 0) {
  if (batch > kMaxBatch) fail(SK_ERR_DIM, "gram64: batch too large");
  constexpr int NT = n_tiles<B, HERM>();
  // one wave of CTAs over the whole batch: ~sm_count CTAs per slice alone,
  // fewer (more rows each) when many slices share the launch; at least 16
  // rows per CTA (small blocks: the cluster reduction outweighs the rows)
  const i64 per_slice = std::max<i64>(1, 2 * i64(ctx->sm_count) / std::max<i64>(batch, 1));
  const int target = int(std::max<i64>(kQCluster, std::min<i64>(ctx->sm_count, per_slice) / kQCluster * kQCluster));
  const int rows = int(std::max<i64>(16, (n + target - 1) / target));
  i64 ctas = (n + rows - 1) / rows;
  ctas = ((ctas + kQCluster - 1) / kQCluster) * kQCluster;
  const i64 ncl = ctas / kQCluster;
  double2* cpart = ctx->arena.get<double2>(HERM ? "cq:part_h" : "cq:part_x", batch * ncl * NT * kQGramThreads);
  const size_t smem = size_t((HERM ? 1 : 2) * kQStage * (B + 1) + NT * kQGramThreads) * sizeof(double2);
  set_smem_limit(reinterpret_cast<const void*>(gram64_kernel<B, HERM>), smem);
  gram64_kernel<B, HERM><<<dim3(unsigned(ctas), unsigned(batch)), kQGramThreads, smem, ctx->stream>>>(
      x, y, n, rows, cpart, gram_counter(ctx), out, sx, ccat, sc);
  ++ctx->launches;
  SKB_LAUNCH("gram64_kernel");
}

template <int B>
void cholqr_blk(sk_ctx* ctx, double2* x, i64 n, int passes, int* flag, i64 batch, i64 sx, const CatIO& io) {
  constexpr int NB = B / 16;
  double2* S = ctx->arena.get<double2>("cq:S", batch * B * B);
  double2* L = ctx->arena.get<double2>("cq:L", batch * B * B);
  double2* D = ctx->arena.get<double2>("cq:D", batch * NB * 256);
  const size_t smem_c = size_t(B * (B + 1)) * sizeof(double2);
  set_smem_limit(reinterpret_cast<const void*>(chol64_kernel<B>), smem_c);
  // rows per trsm CTA: every CTA stages L and the diagonal inverses (80 KB at
  // B = 64), so a batch takes the 64-row maximum (a single slice spreads over
  // the SMs, at least 16 rows per CTA)
  const i64 cta_target = std::max<i64>(1, i64(ctx->sm_count) / std::max<i64>(batch, 1));
  const int rows = int(std::min<i64>(64, std::max<i64>(16, (n + cta_target - 1) / cta_target)));
  const unsigned threads = unsigned(((rows * 16 + 31) / 32) * 32);
  const size_t smem_t = size_t(B * (B + 1) + NB * 16 * 17 + rows * (B + 1)) * sizeof(double2);
  set_smem_limit(reinterpret_cast<const void*>(trsm64_kernel<B>), smem_t);
  for (int p = 0; p < passes; ++p) {
    const float* cc = p == 0 ? io.ccat : nullptr;           // the first pass reads the concatenated product
    float* vc = p + 1 == passes ? io.vcat : nullptr;        // the last pass also writes the next split operand
    launch_gram64<B, true>(ctx, x, x, n, S, batch, sx, cc, io.sc);
    chol64_kernel<B><<<unsigned(batch), chol_threads<B>(), smem_c, ctx->stream>>>(S, L, D, flag);
    ++ctx->launches;
    SKB_LAUNCH("chol64_kernel");
    trsm64_kernel<B><<<dim3(unsigned((n + rows - 1) / rows), unsigned(batch)), threads, smem_t, ctx->stream>>>(
        x, n, rows, L, D, sx, cc, io.sc, vc, io.svc);
    ++ctx->launches;
    SKB_LAUNCH("trsm64_kernel");
  }
}

}  // namespace

void gram64(sk_ctx* ctx, const double2* x, const double2* y, i64 n, double2* out, i64 batch, i64 sx) {
  if (x == y)
    launch_gram64<64, true>(ctx, x, x, n, out, batch, sx);
  else
    launch_gram64<64, false>(ctx, x, y, n, out, batch, sx);
}

void gram_blk(sk_ctx* ctx, int b, const double2* x, const double2* y, i64 n, double2* out) {
  if (b == 64) return gram64(ctx, x, y, n, out);
  if (b != 32) fail(SK_ERR_UNSUPPORTED, "gram_blk: block width must be 32 or 64");
  if (x == y)
    launch_gram64<32, true>(ctx, x, x, n, out);
  else
    launch_gram64<32, false>(ctx, x, y, n, out);
}

void cholqr64(sk_ctx* ctx, double2* x, i64 n, int passes, int* flag, i64 batch, i64 sx, const CatIO& io) {
  cholqr_blk<64>(ctx, x, n, passes, flag, batch, sx, io);
}

void cholqr_b(sk_ctx* ctx, int b, double2* x, i64 n, int passes, int* flag, const CatIO& io) {
  if (b == 64) return cholqr_blk<64>(ctx, x, n, passes, flag, 1, 0, io);
  if (b != 32) fail(SK_ERR_UNSUPPORTED, "cholqr_b: block width must be 32 or 64");
  cholqr_blk<32>(ctx, x, n, passes, flag, 1, 0, io);
}

}  // namespace skb
