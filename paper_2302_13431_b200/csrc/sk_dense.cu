// The reference's `baseline` preset on the GPU:
//
//   build_calib_matrix (calibration.cpp:30-68)  gather of the P x Q|Lambda|
//       calibration matrix, one thread per entry (row = valid shift in
//       row-major order, next_index of types.cpp:19-25; column q*|Lambda|+i).
//   gram_explicit      (calibration.cpp:70-78)  C^H C as one FP64 Hermitian
//       rank-P update (cuBLAS ZHERK on the promoted matrix — a plain library
//       product), mirrored into the full exactly-Hermitian n x n Gram.
//   eig_dense_field    (eigensolve.cpp:9-38)    every voxel's Q x Q Hermitian
//       matrix diagonalised to FP64 accuracy by cyclic Jacobi, one warp per
//       voxel: the parallel (round-robin) ordering rotates Q/2 disjoint
//       (p, q) planes per step, all rotation parameters are computed from the
//       same matrix, then the column and the row updates are applied by the
//       whole warp (A <- U^H A U, V <- V U), sweeps until the off-diagonal
//       Frobenius norm is below 1e-15 of the matrix norm.  The extremal
//       eigenpair (smallest for the nullspace method, largest for ESPIRiT) and
//       the runner-up eigenvalue are returned, as the reference's
//       SelfAdjointEigenSolver columns 0 / Q-1.
//
// The matrices arrive as packed Hermitian planes [h][N] (the K3 layout) with
// an optional fp32 residual plane set (lo): the solver works on hi + lo in
// FP64.  B = alpha I + beta G is applied on load (espirit_inplace).
#include "sk_internal.h"

namespace skb {

namespace {

// ------------------------------------------------------------ calib matrix
struct CalibGeom {
  int nd;
  int ext[3];      // calibration extents (row-major, last axis fastest)
  int shift[3];    // ext - 2 tau
  int tau, lam, q;
  i64 rows;        // P
};

__global__ void calib_matrix_kernel(const float2* __restrict__ calib, const int* __restrict__ off, CalibGeom g,
                                    double2* __restrict__ c) {
  const i64 n = i64(g.q) * g.lam;
  const i64 total = g.rows * n;
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const i64 row = e % g.rows, col = e / g.rows;  // column-major P x n
    const int qq = int(col / g.lam), i = int(col % g.lam);
    // shift index of `row` (row-major over shift extents), then the sample
    // at (idx + tau - offset_i) (calibration.cpp:55-62)
    i64 r = row, at = 0, stride = 1;
    for (int a = g.nd - 1; a >= 0; --a) {
      const int idx = int(r % g.shift[a]);
      r /= g.shift[a];
      at += i64(idx + g.tau - off[i * g.nd + a]) * stride;
      stride *= g.ext[a];
    }
    const float2 v = calib[i64(qq) * stride + at];
    c[e] = make_double2(double(v.x), double(v.y));
  }
}

// Full Hermitian n x n (c64) from the lower triangle of an FP64 HERK result.
__global__ void herk_mirror_kernel(const double2* __restrict__ lower, i64 n, float2* __restrict__ g) {
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < n * n; e += i64(gridDim.x) * blockDim.x) {
    const i64 r = e % n, c = e / n;
    double2 v;
    if (r > c) {
      v = lower[e];
    } else if (r < c) {
      const double2 t = lower[c + r * n];
      v = make_double2(t.x, -t.y);
    } else {
      v = make_double2(lower[e].x, 0.0);
    }
    g[e] = make_float2(float(v.x), float(v.y));
  }
}

// ------------------------------------------------------------ dense Jacobi
__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmconj(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// Round-robin pairing (circle method) on m = even(Q) indices: pair k of
// round r; indices >= Q are the padding slot of an odd Q (no rotation).
__device__ __forceinline__ void rr_pair(int r, int k, int m, int& p, int& q) {
  int a, b;
  if (k == 0) {
    a = r;
    b = m - 1;
  } else {
    a = (r + k) % (m - 1);
    b = (r - k + (m - 1)) % (m - 1);
  }
  p = min(a, b);
  q = max(a, b);
}

struct Rot {
  double c, s;
  double2 ph;  // e^{-i phi}, a_pq = |a_pq| e^{i phi}
  int p, q;
  double dp, dq;  // new diagonal entries
};

__global__ void __launch_bounds__(256) dense_eig_kernel(DenseEigArgs a, int warps_per_block) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Q = a.q, ld = Q + 1, m = Q + (Q & 1), half = m / 2;
  const int h = Q * (Q + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* pct = reinterpret_cast<int*>(smem_raw);  // [h] packed index -> (p << 8) | c
  const size_t pct_bytes = (size_t(h) * sizeof(int) + 15) & ~size_t(15);
  const size_t per_warp = 2 * size_t(Q) * ld * sizeof(double2) + size_t(half) * sizeof(Rot);
  unsigned char* mine = smem_raw + pct_bytes + size_t(warp) * ((per_warp + 15) & ~size_t(15));
  double2* A = reinterpret_cast<double2*>(mine);  // [Q][ld] row-major
  double2* V = A + Q * ld;                        // [Q][ld] row-major, eigenvectors in columns
  Rot* rot = reinterpret_cast<Rot*>(V + Q * ld);
  for (int e = threadIdx.x; e < h; e += blockDim.x) {
    int pp = 0, base = 0;
    while (e >= base + Q - pp) base += Q - pp++;
    pct[e] = (pp << 8) | (pp + e - base);
  }
  __syncthreads();

  const i64 nwarps = i64(gridDim.x) * warps_per_block;
  for (i64 j = blockIdx.x * i64(warps_per_block) + warp; j < a.n; j += nwarps) {
    // load B = alpha I + beta (hi + lo) in FP64; V = I
    for (int e = lane; e < h; e += 32) {
      const int pc = pct[e], p = pc >> 8, c = pc & 0xff;
      const float2 hv = a.planes[i64(e) * a.n + j];
      double2 g = make_double2(double(hv.x), double(hv.y));
      if (a.planes_lo) {
        const float2 lv = lo_unpack(a.planes_lo[i64(e) * a.n + j]);
        g.x += double(lv.x);
        g.y += double(lv.y);
      }
      g = make_double2(a.beta * g.x, a.beta * g.y);
      if (p == c) g = make_double2(g.x + a.alpha, 0.0);  // spatial_gram.cpp:140-146 (real diagonal)
      A[p * ld + c] = g;
      A[c * ld + p] = make_double2(g.x, -g.y);
    }
    for (int e = lane; e < Q * Q; e += 32) V[(e / Q) * ld + e % Q] = make_double2(e / Q == e % Q ? 1.0 : 0.0, 0.0);
    __syncwarp();

    for (int sweep = 0; sweep < 40; ++sweep) {
      // convergence: off-diagonal Frobenius norm against the whole matrix
      double off = 0.0, tot = 0.0;
      for (int e = lane; e < Q * Q; e += 32) {
        const int r = e / Q, c = e % Q;
        const double2 v = A[r * ld + c];
        const double x = v.x * v.x + v.y * v.y;
        tot += x;
        if (r != c) off += x;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        off += __shfl_xor_sync(0xffffffffu, off, o);
        tot += __shfl_xor_sync(0xffffffffu, tot, o);
      }
      if (!(off > 1e-30 * tot) || tot == 0.0) break;  // also leaves on NaN
      for (int r = 0; r < m - 1; ++r) {
        // 1. rotation parameters of the Q/2 disjoint planes, from the same A
        for (int k = lane; k < half; k += 32) {
          int p, q;
          rr_pair(r, k, m, p, q);
          Rot t{1.0, 0.0, make_double2(1.0, 0.0), p, q, 0.0, 0.0};
          if (q < Q) {
            const double app = A[p * ld + p].x, aqq = A[q * ld + q].x;
            const double2 apq = A[p * ld + q];
            const double rr = hypot(apq.x, apq.y);
            t.dp = app;
            t.dq = aqq;
            if (rr > 1e-300 && rr > 1e-18 * fmax(fabs(app), fabs(aqq))) {
              t.ph = make_double2(apq.x / rr, -apq.y / rr);
              const double zeta = (aqq - app) / (2.0 * rr);
              const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
              t.c = 1.0 / sqrt(1.0 + tt * tt);
              t.s = tt * t.c;
              t.dp = app - tt * rr;
              t.dq = aqq + tt * rr;
            } else {
              t.q = Q;  // nothing to rotate
            }
          }
          rot[k] = t;
        }
        __syncwarp();
        // 2. columns: A <- A U, V <- V U (col p: c a_p - s ph a_q; col q: s a_p + c ph a_q)
        for (int e = lane; e < 2 * half * Q; e += 32) {
          const int mat = e / (half * Q), rem = e % (half * Q), k = rem / Q, row = rem % Q;
          const Rot t = rot[k];
          if (t.q >= Q) continue;
          double2* X = mat ? V : A;
          const double2 xp = X[row * ld + t.p], xq = cm(X[row * ld + t.q], t.ph);
          X[row * ld + t.p] = make_double2(t.c * xp.x - t.s * xq.x, t.c * xp.y - t.s * xq.y);
          X[row * ld + t.q] = make_double2(t.s * xp.x + t.c * xq.x, t.s * xp.y + t.c * xq.y);
        }
        __syncwarp();
        // 3. rows: A <- U^H A (row p: c a_p - s conj(ph) a_q; row q: s a_p + c conj(ph) a_q)
        for (int e = lane; e < half * Q; e += 32) {
          const int k = e / Q, col = e % Q;
          const Rot t = rot[k];
          if (t.q >= Q) continue;
          const double2 xp = A[t.p * ld + col], xq = cmconj(A[t.q * ld + col], t.ph);
          A[t.p * ld + col] = make_double2(t.c * xp.x - t.s * xq.x, t.c * xp.y - t.s * xq.y);
          A[t.q * ld + col] = make_double2(t.s * xp.x + t.c * xq.x, t.s * xp.y + t.c * xq.y);
        }
        __syncwarp();
        // the rotated pair is diagonal by construction
        for (int k = lane; k < half; k += 32) {
          const Rot t = rot[k];
          if (t.q >= Q) continue;
          A[t.p * ld + t.q] = A[t.q * ld + t.p] = make_double2(0.0, 0.0);
          A[t.p * ld + t.p] = make_double2(t.dp, 0.0);
          A[t.q * ld + t.q] = make_double2(t.dq, 0.0);
        }
        __syncwarp();
      }
    }
    // extremal eigenvalue (ties: lowest index, as an ascending sort keeps order)
    // and the runner-up
    int best = 0;
    double bv = A[0].x;
    for (int i = 1; i < Q; ++i) {
      const double d = A[i * ld + i].x;
      if (a.largest ? d > bv : d < bv) {
        bv = d;
        best = i;
      }
    }
    double sv = bv;
    bool have = false;
    for (int i = 0; i < Q; ++i) {
      if (i == best) continue;
      const double d = A[i * ld + i].x;
      if (!have || (a.largest ? d > sv : d < sv)) {
        sv = d;
        have = true;
      }
    }
    // unit eigenvector = column `best` of V (Jacobi keeps V unitary)
    for (int c = lane; c < Q; c += 32) {
      const double2 v = V[c * ld + best];
      a.vec[i64(c) * a.n + j] = make_float2(float(v.x), float(v.y));
    }
    if (lane == 0) {
      if (a.value) a.value[j] = float(bv);
      if (a.second) a.second[j] = float(sv);
      if (a.lambda) a.lambda[j] = float(a.lam_add + a.lam_mul * bv);
      if (a.mask) a.mask[j] = float(a.lam_add + a.lam_mul * bv) < a.mask_threshold ? 1 : 0;
    }
    __syncwarp();
  }
}

}  // namespace

void calib_matrix(sk_ctx* ctx, const float2* calib, const Dims& cdims, int q, const Support& s, const int* d_off,
                  double2* c) {
  CalibGeom g{};
  g.nd = int(cdims.size());
  g.rows = 1;
  for (int a = 0; a < g.nd; ++a) {
    g.ext[a] = int(cdims[size_t(a)]);
    g.shift[a] = int(cdims[size_t(a)]) - 2 * s.tau;
    g.rows *= g.shift[a];
  }
  g.tau = s.tau;
  g.lam = int(s.count);
  g.q = q;
  const i64 total = g.rows * i64(q) * s.count;
  if (total <= 0) return;
  const int threads = 256;
  const i64 blocks = std::min<i64>((total + threads - 1) / threads, i64(ctx->sm_count) * 8);
  calib_matrix_kernel<<<unsigned(blocks), threads, 0, ctx->stream>>>(calib, d_off, g, c);
  ++ctx->launches;
  SKB_LAUNCH("calib_matrix_kernel");
}

void gram_explicit_dev(sk_ctx* ctx, const double2* c, i64 rows, i64 n, double2* lower, float2* gram) {
  const double one = 1.0, zero = 0.0;
  check_cublas(cublasZherk(ctx->cublas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, int(n), int(rows), &one,
                           reinterpret_cast<const cuDoubleComplex*>(c), int(std::max<i64>(rows, 1)), &zero,
                           reinterpret_cast<cuDoubleComplex*>(lower), int(n)),
               "cublasZherk (gram_explicit)");
  ++ctx->lib_calls;
  const i64 total = n * n;
  const i64 blocks = std::min<i64>((total + 255) / 256, i64(ctx->sm_count) * 8);
  herk_mirror_kernel<<<unsigned(blocks), 256, 0, ctx->stream>>>(lower, n, gram);
  ++ctx->launches;
  SKB_LAUNCH("herk_mirror_kernel");
}

void dense_eig(sk_ctx* ctx, const DenseEigArgs& a) {
  if (a.n <= 0) return;
  const int Q = a.q, ld = Q + 1, half = (Q + (Q & 1)) / 2, h = Q * (Q + 1) / 2;
  const size_t pct_bytes = (size_t(h) * sizeof(int) + 15) & ~size_t(15);
  const size_t per_warp = ((2 * size_t(Q) * ld * sizeof(double2) + size_t(half) * sizeof(Rot)) + 15) & ~size_t(15);
  int wpb = int(std::min<size_t>(8, (200 * 1024 - pct_bytes) / per_warp));
  if (wpb < 1) fail(SK_ERR_UNSUPPORTED, "eig_dense_field: channel count too large for the shared-memory Jacobi");
  const size_t smem = pct_bytes + size_t(wpb) * per_warp;
  set_smem_limit(reinterpret_cast<const void*>(dense_eig_kernel), smem);
  int per_sm = 0;
  SKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dense_eig_kernel, 32 * wpb, smem));
  const i64 blocks = std::min<i64>((a.n + wpb - 1) / wpb, i64(std::max(per_sm, 1)) * ctx->sm_count);
  dense_eig_kernel<<<unsigned(blocks), 32 * wpb, smem, ctx->stream>>>(a, wpb);
  ++ctx->launches;
  SKB_LAUNCH("dense_eig_kernel");
}

}  // namespace skb
