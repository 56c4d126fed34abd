// One-CTA FP64 Hermitian eigensolver for the Rayleigh-Ritz matrix of the K2
// subspace solver (b <= 64, everything resident in shared memory).
//
// The reference solves the full Gram eigenproblem with Eigen's
// SelfAdjointEigenSolver (nullspace.cpp:13); the B200 path projects onto a
// b-column block (run_eigh_subspace) and only needs the b x b projection
// H = V^H A V diagonalised.  cuSOLVER's dense solvers spend ~1 ms of small
// launches on b = 64 (measured: Zheevj, Xsyevd and XsyevBatched alike), so
// this kernel does the whole decomposition in one CTA.  It is latency-bound
// (one SM, dependent FP64 chains), so every phase is organised around few
// block barriers and no FP64 divisions on the critical chains (reciprocal
// approximation + Newton steps instead):
//
//   1. Householder tridiagonalisation H = Q T Q^H (the zhetd2 / zlarfg
//      convention: H_k = I - tau v v^H, v_0 = 1, real off-diagonal beta);
//      H is kept as a full Hermitian matrix (padded rows) in shared memory so
//      that rows are read contiguously without conjugation branches.  Two
//      barriers per column: norms and p^H v are reduced redundantly by every
//      warp, v and w = p - tau/2 (p^H v) v are formed on the fly.
//   2. Eigenvalues of T by multisection (Sturm counts from the scaled
//      leading-minor recurrence, zero minors by the dlaebz rule): every
//      eigenvalue is bracketed by TPE threads that evaluate two interior
//      points each per step, to 1e-10 ||T||.
//   3. Eigenvectors of T by inverse iteration (dstein): two solves of
//      (T - lambda I) z = r with partial pivoting from a pseudo-random start
//      (factors in shared memory), a Rayleigh-quotient refinement of lambda
//      (to ~eps ||T||), and Gram-Schmidt plus shifted re-solves inside
//      clusters of close eigenvalues.
//   4. Back-transformation X = Q Z, one column per 8 lanes with the column
//      in registers (no block barriers, no shared-memory traffic for X).
//
// Output matches cusolverDnZheevj: eigenvalues ascending in w, eigenvectors
// overwrite H column-major.  A non-finite intermediate raises info[0] (the
// caller then takes the full-matrix path, as for any solver failure).
#include "sk_internal.h"

#include <cfloat>
#include <cstdio>
#include <cstdlib>

namespace skb {

namespace {

constexpr int kThreads = 512;
constexpr int kMaxN = 64;

__device__ long long g_phase_clock[8];  // development aid: clock64 at phase boundaries (thread 0)
#define SKB_EIG_STAMP(i) \
  if (threadIdx.x == 0) g_phase_clock[i] = clock64();

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {  // acc + a b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cfma_conj(double2 acc, double2 a, double2 b) {  // acc + conj(a) b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}

// 1/x from the hardware approximation plus Newton steps (1: ~2^-46, 2: ~ulp).
template <int kNewton>
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#pragma unroll
  for (int i = 0; i < kNewton; ++i) r = fma(r, fma(-x, r, 1.0), r);
  return r;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Block-wide sum; every thread receives the total.
__device__ __forceinline__ double block_sum(double x, double* red) {
  x = warp_sum(x);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kThreads / 32; ++k) s += red[k];
  __syncthreads();
  return s;
}

// Number of eigenvalues of the symmetric tridiagonal (ds = s d, e2s = (s e)^2) not
// above x0 and x1 (two independent chains for ILP), from the signs of the
// leading principal minors P_k = det(s (T_k - x I)) (Sturm sequence):
//   P_k = (s d_k - s x) P_{k-1} - e2s_{k-1} P_{k-2},
// one FMA on the dependent chain per step instead of the LDL pivot's
// reciprocal (bisection phase 90 k -> 20 k cycles at n = 64).  A zero minor
// counts as a sign change and takes the sign opposite to its predecessor,
// which is the LDL rule's "zero pivot -> -pivmin" (dlaebz); s is a power of
// two with s ||T|| < 1, so |P_k| grows at most ~3^8 per eight steps and the
// pair is rescaled by 2^-+400 every eight steps.
__device__ __forceinline__ void sturm_count2(const double* ds, const double* e2s, int n, double x0, double x1,
                                             double s, int& c0, int& c1) {
  const double y0 = x0 * s, y1 = x1 * s;
  double a1 = 1.0, a2 = 0.0, b1 = 1.0, b2 = 0.0;  // P_{k-1}, P_{k-2} of the two chains
  unsigned sa = 0u, sb = 0u;                       // sign taken for P_{k-1}
  int na = 0, nb = 0;
  for (int k0 = 0; k0 < n; k0 += 8) {
    // eight steps per block: the shared loads of a block issue ahead of its chain
    double dk[8], ek[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = k0 + j;
      dk[j] = k < n ? ds[k] : 0.0;
      ek[j] = (k > 0 && k < n) ? e2s[k - 1] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (k0 + j < n) {
        const double pa = fma(dk[j] - y0, a1, -ek[j] * a2);
        const double pb = fma(dk[j] - y1, b1, -ek[j] * b2);
        const unsigned ta = pa == 0.0 ? sa ^ 1u : unsigned(__double2hiint(pa)) >> 31;
        const unsigned tb = pb == 0.0 ? sb ^ 1u : unsigned(__double2hiint(pb)) >> 31;
        na += int(ta != sa);
        nb += int(tb != sb);
        sa = ta;
        sb = tb;
        a2 = a1;
        a1 = pa;
        b2 = b1;
        b1 = pb;
      }
    }
    const double ma = fmax(fabs(a1), fabs(a2)), mb = fmax(fabs(b1), fabs(b2));
    const double fa = ma < 0x1p-400 ? 0x1p400 : ma > 0x1p400 ? 0x1p-400 : 1.0;
    const double fb = mb < 0x1p-400 ? 0x1p400 : mb > 0x1p400 ? 0x1p-400 : 1.0;
    a1 *= fa;
    a2 *= fa;
    b1 *= fb;
    b2 *= fb;
  }
  c0 = na;
  c1 = nb;
}

__device__ __forceinline__ double hash_unit(unsigned a, unsigned b) {  // deterministic value in (-1, 1)
  unsigned h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  return (double(h) + 0.5) * (2.0 / 4294967296.0) - 1.0;
}

// Solve (T - s I) z = r in place (z holds r on entry, stride zs) by Gaussian
// elimination with partial pivoting (dgtsv / dlagtf style); zero pivots are
// perturbed to `tiny`.  Factor rows (1/u0, u1, u2) go to shared memory
// u[(i * 3 + f) * stride + t] (conflict-free across t); the eliminated
// right-hand side is kept in z.
__device__ void tri_solve(const double* d, const double* e, int n, double s, double tiny, double* z, int zs,
                          double* u, int stride, int t) {
  auto U = [&](int i, int f) -> double& { return u[(i * 3 + f) * stride + t]; };
  double p0 = d[0] - s, p1 = n > 1 ? e[0] : 0.0, p2 = 0.0, r0 = z[0];
  for (int i = 0; i + 1 < n; ++i) {
    const double sub = e[i], dg = d[i + 1] - s, sup = (i + 2 < n) ? e[i + 1] : 0.0, rr = z[(i + 1) * zs];
    if (fabs(p0) >= fabs(sub)) {
      if (p0 == 0.0) p0 = tiny;
      const double inv = frcp<2>(p0), l = sub * inv;
      U(i, 0) = inv;
      U(i, 1) = p1;
      U(i, 2) = p2;
      z[i * zs] = r0;
      p0 = dg - l * p1;
      p1 = sup - l * p2;
      r0 = rr - l * r0;
    } else {
      const double inv = frcp<2>(sub), l = p0 * inv;
      U(i, 0) = inv;
      U(i, 1) = dg;
      U(i, 2) = sup;
      z[i * zs] = rr;
      const double n0 = p1 - l * dg, n1 = p2 - l * sup, nr = r0 - l * rr;
      p0 = n0;
      p1 = n1;
      r0 = nr;
    }
    p2 = 0.0;
  }
  if (p0 == 0.0) p0 = tiny;
  double z1 = r0 * frcp<2>(p0), z2 = 0.0;  // z_{i+1}, z_{i+2}
  z[(n - 1) * zs] = z1;
  for (int i = n - 2; i >= 0; --i) {
    const double zi = (z[i * zs] - U(i, 1) * z1 - U(i, 2) * z2) * U(i, 0);
    z[i * zs] = zi;
    z2 = z1;
    z1 = zi;
  }
}

// NF > 0: the order is fixed at compile time (n == NF; loop bounds and
// strides fold); 0: runtime n.
template <int NF>
__global__ void __launch_bounds__(kThreads) herm_eig_kernel(double2* __restrict__ H, int n_arg, double* __restrict__ w,
                                                             double floor_rel, int* __restrict__ info) {
  const int n = NF > 0 ? NF : n_arg;
  SKB_DCHECK(n >= 1 && n <= kMaxN && blockDim.x == kThreads);
  // batch (multislice K2): one CTA per slice
  H += size_t(blockIdx.x) * n * n;
  w += size_t(blockIdx.x) * n;
  info += 3 * blockIdx.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ld = n + 1;  // padded row stride (double2) of the full Hermitian A (bank skew)
  const int zs = n + 1;  // padded row stride of zr
  const int uwords = (max(2 * n * (n + 1), 3 * n * n) + 1) & ~1;  // the LU factors (step 3); even
  double2* A = reinterpret_cast<double2*>(smem_raw);  // full Hermitian matrix; row k holds v_k after step k
  double* un = reinterpret_cast<double*>(A + n * ld);  // LU factors (step 3)
  double2* pv = reinterpret_cast<double2*>(un + uwords);  // [n]
  double2* vv = pv + n;                                    // [n]
  double2* tau = vv + n;                                   // [n]
  double* d = reinterpret_cast<double*>(tau + n);
  double* e = d + n;
  double* e2 = e + n;
  double* lam = e2 + n;
  double* dsc = lam + n;  // s d (the Sturm recurrence's scaled diagonal)
  double* red = dsc + n;  // [kThreads / 32]
  double* zr = red + kThreads / 32;                // [n][zs] real eigenvectors of T, row-major [i][t]
  int* cl = reinterpret_cast<int*>(zr + n * zs);  // [2n + 1] cluster table

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  SKB_EIG_STAMP(0);

  // lower triangle of H (column-major) -> full Hermitian A (row-major)
  for (int e0 = tid; e0 < n * n; e0 += kThreads) {
    const int i = e0 % n, j = e0 / n;
    if (i >= j) {
      double2 a = H[i + size_t(j) * n];
      if (i == j) a.y = 0.0;
      A[i * ld + j] = a;
      A[j * ld + i] = cconj(a);
    }
  }
  __syncthreads();

  // ---- 1. tridiagonalisation (zhetd2, lower): x = A(k+1:, k) = conj(A(k, k+1:))
  // Three block barriers per column: v published, p published, A22 updated.
  // Row i of the trailing matrix belongs to the 8 lanes tid >> 3 == i (lane h
  // takes columns h, h + 8, ...) in both the product and the update, so every
  // chain is short and the loads of a thread are independent.
  for (int k = 0; k + 1 < n; ++k) {
    const int m = n - k - 1;
    const double2* rowk = A + k * ld + k + 1;  // conj(x)
    // ||x[1:]||^2, redundantly per warp (m <= 63)
    double part = 0.0;
    for (int i = 1 + lane; i < m; i += 32) {
      const double2 a = rowk[i];
      part += a.x * a.x + a.y * a.y;
    }
    const double xnorm2 = warp_sum(part);
    const double2 alpha = cconj(rowk[0]);
    double2 t = make_double2(0.0, 0.0), scale = make_double2(0.0, 0.0);
    double beta = alpha.x;
    if (xnorm2 > 0.0 || alpha.y != 0.0) {  // zlarfg
      beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xnorm2), alpha.x);
      const double ib = frcp<2>(beta);
      t = make_double2((beta - alpha.x) * ib, -alpha.y * ib);
      const double2 den = make_double2(alpha.x - beta, alpha.y);
      const double inv = frcp<2>(den.x * den.x + den.y * den.y);
      scale = make_double2(den.x * inv, -den.y * inv);
    }
    if (tid == 0) {
      e[k] = beta;
      d[k] = A[k * ld + k].x;
      tau[k] = t;
    }
    if (t.x == 0.0 && t.y == 0.0) continue;  // H_k = I (uniform across the block; A unchanged)
    if (tid < m) vv[tid] = tid == 0 ? make_double2(1.0, 0.0) : cmul(cconj(rowk[tid]), scale);
    __syncthreads();
    const int ri = tid >> 3, rh = tid & 7;
    const bool row_live = ri < m;
    double2* ar = A + (k + 1 + ri) * ld + k + 1;
    {  // p = tau * A22 v
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
      if (row_live) {
#pragma unroll 4
        for (int j = rh; j < m; j += 16) {
          acc0 = cfma(acc0, ar[j], vv[j]);
          if (j + 8 < m) acc1 = cfma(acc1, ar[j + 8], vv[j + 8]);
        }
      }
      double2 acc = cadd(acc0, acc1);
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (row_live && rh == 0) pv[ri] = cmul(t, acc);
    }
    __syncthreads();
    // a2 = -tau/2 (p^H v), redundantly per warp; w = p + a2 v
    double2 dp = make_double2(0.0, 0.0);
    for (int i = lane; i < m; i += 32) dp = cfma_conj(dp, pv[i], vv[i]);
    dp.x = warp_sum(dp.x);
    dp.y = warp_sum(dp.y);
    const double2 a2 = cmul(make_double2(-0.5 * t.x, -0.5 * t.y), dp);
    if (tid < m) A[k * ld + k + 1 + tid] = vv[tid];  // v_k into row k (dead after this step)
    if (row_live) {  // A22 -= v w^H + w v^H (both triangles)
      const double2 vi = vv[ri], wi = cfma(pv[ri], a2, vi);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = rh + 8 * u;
        if (j < m) {
          const double2 vj = vv[j], wj = cfma(pv[j], a2, vj);
          const double2 sub = cadd(cmul(vi, cconj(wj)), cmul(wi, cconj(vj)));
          double2 a = ar[j];
          a.x -= sub.x;
          a.y = (ri == j) ? 0.0 : a.y - sub.y;
          ar[j] = a;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    d[n - 1] = A[(n - 1) * ld + n - 1].x;
    tau[n - 1] = make_double2(0.0, 0.0);
  }
  __syncthreads();

  SKB_EIG_STAMP(1);
  // ---- 2. eigenvalues by multisection
  double lo = 0.0, hi = 0.0, emax2 = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
    lo = i == 0 ? d[i] - r : fmin(lo, d[i] - r);
    hi = i == 0 ? d[i] + r : fmax(hi, d[i] + r);
    if (i + 1 < n) emax2 = fmax(emax2, e[i] * e[i]);
  }
  const double tnorm = fmax(fabs(lo), fabs(hi));
  const double sscale = tnorm > 0.0 ? ldexp(1.0, -(ilogb(tnorm) + 1)) : 1.0;  // sturm_count2's s
  if (tid < n - 1) e2[tid] = (e[tid] * sscale) * (e[tid] * sscale);
  if (tid < n) dsc[tid] = d[tid] * sscale;
  __syncthreads();
  const double pivmin = DBL_MIN * fmax(1.0, emax2);
  lo -= 2.0 * DBL_EPSILON * tnorm + pivmin;
  hi += 2.0 * DBL_EPSILON * tnorm + pivmin;
  int tpe = 1;
  while (tpe * 2 * n <= kThreads && tpe < 4) tpe *= 2;  // more points per step hit the MUFU/FP64 rate
  {
    const int t = tid / tpe, s = tid % tpe, base = lane & ~(tpe - 1);
    const int pts = 2 * tpe;  // interior points per eigenvalue per step
    const bool act = t < n;
    double a = lo, b = hi;
    // fixed step count (uniform control flow); to 1e-10 ||T||, the Rayleigh
    // quotient after inverse iteration supplies the rest
    const int steps = int(ceil(log((hi - lo) / (1e-10 * tnorm + pivmin)) / log(double(pts + 1)))) + 1;
    for (int it = 0; it < steps; ++it) {
      const double wdt = (b - a) / double(pts + 1);
      const double x0 = a + wdt * double(2 * s + 1), x1 = a + wdt * double(2 * s + 2);
      int k0 = 0, k1 = 0;
      if (act) sturm_count2(dsc, e2, n, x0, x1, sscale, k0, k1);
      double na = a, nb = b;
      for (int q = 0; q < tpe; ++q) {
        const double y0 = __shfl_sync(0xffffffffu, x0, base + q), y1 = __shfl_sync(0xffffffffu, x1, base + q);
        const int m0 = __shfl_sync(0xffffffffu, k0, base + q), m1 = __shfl_sync(0xffffffffu, k1, base + q);
        if (m0 <= t) na = fmax(na, y0);
        if (m0 > t) nb = fmin(nb, y0);
        if (m1 <= t) na = fmax(na, y1);
        if (m1 > t) nb = fmin(nb, y1);
      }
      a = na;
      b = nb;
    }
    if (act && s == 0) lam[t] = 0.5 * (a + b);
  }
  __syncthreads();

  SKB_EIG_STAMP(2);
  // ---- 3. eigenvectors of T by inverse iteration (one thread per eigenvalue)
  const double tiny = DBL_EPSILON * tnorm + pivmin;
  if (tid < n) {
    const int t = tid;
    double* z = zr + t;  // column t, row stride zs
    for (int i = 0; i < n; ++i) z[i * zs] = hash_unit(unsigned(t), unsigned(i));
    for (int pass = 0; pass < 2; ++pass) {
      tri_solve(d, e, n, lam[t], tiny, z, zs, un, n, t);
      double s2 = 0.0;
      for (int i = 0; i < n; ++i) s2 += z[i * zs] * z[i * zs];
      const double inv = rsqrt(s2);
      for (int i = 0; i < n; ++i) z[i * zs] *= inv;
    }
    double rq = 0.0;  // Rayleigh quotient refinement of lambda
    for (int i = 0; i < n; ++i) {
      const double zi = z[i * zs];
      rq += d[i] * zi * zi;
      if (i + 1 < n) rq += 2.0 * e[i] * zi * z[(i + 1) * zs];
    }
    lam[t] = rq;
  }
  __syncthreads();

  SKB_EIG_STAMP(3);
  // Clusters (dstein): consecutive eigenvalues closer than kClus ||T||.
  // Inverse-iteration vectors are orthogonal to ~eps ||T|| / gap, so cluster
  // members are orthonormalised (CGS2, in order) and - when the cluster
  // reaches above floor_rel ||T|| - re-solved with their own shifts and
  // re-orthonormalised twice, which converges to the individual eigenvectors.
  // Clusters below the floor (the noise tail of a Ritz spectrum, never used
  // individually by the caller) only get the orthonormalisation.
  constexpr double kClus = 1e-5;
  int* cs = cl;      // cluster start of j
  int* cf = cl + n;  // bit0: multi-member cluster, bit1: refine
  if (tid == 0) {
    int any = 0;
    for (int i = 0; i < n; ++i) {
      cs[i] = (i > 0 && fabs(lam[i] - lam[i - 1]) < kClus * tnorm) ? cs[i - 1] : i;
      cf[i] = 0;
    }
    for (int i = 0; i < n;) {
      int j = i;
      while (j + 1 < n && cs[j + 1] == i) ++j;
      if (j > i) {
        any = 1;
        const int fl = 1 | (lam[j] >= floor_rel * tnorm ? 2 : 0);
        for (int q = i; q <= j; ++q) cf[q] = fl;
      }
      i = j + 1;
    }
    cl[2 * n] = any;
  }
  __syncthreads();
  if (cl[2 * n]) {
    double* dots = reinterpret_cast<double*>(pv);  // free after step 1
    auto cgs2 = [&](int j) {  // z_j <- normalise((I - Z_c Z_c^T)^2 z_j), Z_c = members before j
      const int j0 = cs[j];
      for (int pass = 0; pass < 2 && j0 < j; ++pass) {
        for (int q = j0 + warp; q < j; q += kThreads / 32) {
          double sd = 0.0;
          for (int i = lane; i < n; i += 32) sd += zr[i * zs + q] * zr[i * zs + j];
          sd = warp_sum(sd);
          if (lane == 0) dots[q] = sd;
        }
        __syncthreads();
        for (int i = tid; i < n; i += kThreads) {
          double acc = zr[i * zs + j];
          for (int q = j0; q < j; ++q) acc -= dots[q] * zr[i * zs + q];
          zr[i * zs + j] = acc;
        }
        __syncthreads();
      }
      double part3 = 0.0;
      for (int i = tid; i < n; i += kThreads) part3 += zr[i * zs + j] * zr[i * zs + j];
      const double nn = block_sum(part3, red);
      const double inv = nn > 0.0 ? rsqrt(nn) : 0.0;
      for (int i = tid; i < n; i += kThreads) zr[i * zs + j] *= inv;
      __syncthreads();
    };
    for (int j = 0; j < n; ++j)
      if (cf[j] & 1) cgs2(j);
    for (int round = 0; round < 2; ++round) {
      if (tid < n && (cf[tid] & 2)) tri_solve(d, e, n, lam[tid], tiny, zr + tid, zs, un, n, tid);
      __syncthreads();
      for (int j = 0; j < n; ++j)
        if (cf[j] & 2) cgs2(j);
    }
    if (tid < n && (cf[tid] & 2)) {  // refresh lambda from the final vector
      double rq = 0.0;
      for (int i = 0; i < n; ++i) {
        const double zi = zr[i * zs + tid];
        rq += d[i] * zi * zi;
        if (i + 1 < n) rq += 2.0 * e[i] * zi * zr[(i + 1) * zs + tid];
      }
      lam[tid] = rq;
    }
    __syncthreads();
  }

  SKB_EIG_STAMP(4);
  // ---- 4. back-transformation X = Q Z (H_0 ... H_{n-2} applied right to left)
  // c01 = v0^H v1 of every reflector pair (column-independent), one warp per pair
  for (int k = n - 2 - 2 * warp; k >= 1; k -= 2 * (kThreads / 32)) {
    const double2* v1 = A + k * ld + k + 1;
    const double2* v0 = A + (k - 1) * ld + k;
    double2 c = make_double2(0.0, 0.0);
    for (int i = lane; i < n - k - 1; i += 32) c = cfma_conj(c, v0[i + 1], v1[i]);
    c.x = warp_sum(c.x);
    c.y = warp_sum(c.y);
    if (lane == 0) vv[k] = c;
  }
  __syncthreads();
  bool bad = false;
  {
    // Reflectors in pairs (k1 = k applied first, then k0 = k - 1):
    //   s1 = v1^H X,  s0 = v0^H X - tau1 (v0^H v1) s1,
    //   X -= tau1 v1 s1 + tau0 v0 s0      (v0 starts one row above v1).
    // Column c of X lives in the registers of its 8 lanes (lane rs holds rows
    // rs, rs + 8, ...); v_k's entry for row r is A[k][r] (zero above the
    // reflector), so a pair needs no shared-memory traffic for X and no
    // barrier (smem-resident X: 103 k cycles at n = 64).
    constexpr int RJ = kMaxN / 8;
    const int c = tid >> 3, rs = tid & 7;
    const bool act = c < n;
    double2 xr[RJ];
#pragma unroll
    for (int j = 0; j < RJ; ++j) {
      const int r = rs + 8 * j;
      xr[j] = make_double2((act && r < n) ? zr[r * zs + c] : 0.0, 0.0);
    }
    int k = n - 2;
    for (; k >= 1; k -= 2) {
      const double2 t1 = tau[k], t0 = tau[k - 1], c01 = vv[k];
      const double2* a1 = A + k * ld;        // v1[r] = A[k][r], r >= k + 1
      const double2* a0 = A + (k - 1) * ld;  // v0[r] = A[k-1][r], r >= k
      double2 s1 = make_double2(0.0, 0.0), s0 = s1;
#pragma unroll
      for (int j = 0; j < RJ; ++j) {
        const int r = rs + 8 * j;
        if (r < n && r >= k) {
          const double2 u1 = r > k ? a1[r] : make_double2(0.0, 0.0);
          s1 = cfma_conj(s1, u1, xr[j]);
          s0 = cfma_conj(s0, a0[r], xr[j]);
        }
      }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        s1.x += __shfl_xor_sync(0xffffffffu, s1.x, o);
        s1.y += __shfl_xor_sync(0xffffffffu, s1.y, o);
        s0.x += __shfl_xor_sync(0xffffffffu, s0.x, o);
        s0.y += __shfl_xor_sync(0xffffffffu, s0.y, o);
      }
      const double2 f1 = cmul(t1, s1);
      const double2 g = cmul(c01, f1);
      const double2 f0 = cmul(t0, make_double2(s0.x - g.x, s0.y - g.y));
#pragma unroll
      for (int j = 0; j < RJ; ++j) {
        const int r = rs + 8 * j;
        if (r < n && r >= k) {
          const double2 u1 = r > k ? a1[r] : make_double2(0.0, 0.0);
          const double2 u = cadd(cmul(u1, f1), cmul(a0[r], f0));
          xr[j].x -= u.x;
          xr[j].y -= u.y;
        }
      }
    }
    if (k == 0) {  // leftover single reflector: v[r] = A[0][r], r >= 1
      const double2 tk = tau[0];
      double2 sd = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < RJ; ++j) {
        const int r = rs + 8 * j;
        if (r < n && r >= 1) sd = cfma_conj(sd, A[r], xr[j]);
      }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        sd.x += __shfl_xor_sync(0xffffffffu, sd.x, o);
        sd.y += __shfl_xor_sync(0xffffffffu, sd.y, o);
      }
      const double2 f = cmul(tk, sd);
#pragma unroll
      for (int j = 0; j < RJ; ++j) {
        const int r = rs + 8 * j;
        if (r < n && r >= 1) {
          const double2 u = cmul(A[r], f);
          xr[j].x -= u.x;
          xr[j].y -= u.y;
        }
      }
    }
    if (act) {
#pragma unroll
      for (int j = 0; j < RJ; ++j) {
        const int r = rs + 8 * j;
        if (r < n) {
          bad |= !isfinite(xr[j].x) || !isfinite(xr[j].y);
          H[r + size_t(c) * n] = xr[j];
        }
      }
    }
  }
  if (tid < n) {
    w[tid] = lam[tid];
    bad |= !isfinite(lam[tid]);
  }
  if (bad) atomicExch(info, 1);
  SKB_EIG_STAMP(5);
}

size_t herm_eig_smem(int n) {
  const size_t np = size_t(n) * (n + 1);  // full matrix, padded rows
  const size_t uwords = (std::max<size_t>(2 * size_t(n) * (n + 1), 3 * size_t(n) * n) + 1) & ~size_t(1);
  return np * sizeof(double2) + uwords * sizeof(double) + 3 * size_t(n) * sizeof(double2) +
         (5 * size_t(n) + kThreads / 32 + size_t(n) * (n + 1)) * sizeof(double) + (2 * size_t(n) + 1) * sizeof(int);
}

}  // namespace

bool herm_eig_small(sk_ctx* ctx, double2* H, int n, double* w, int* info, double floor_rel, int batch) {
  if (n < 1 || n > kMaxN) return false;
  const size_t smem = herm_eig_smem(n);
  if (n == 64) {
    set_smem_limit(reinterpret_cast<const void*>(herm_eig_kernel<64>), smem);
    herm_eig_kernel<64><<<unsigned(batch), kThreads, smem, ctx->stream>>>(H, n, w, floor_rel, info);
  } else if (n == 32) {  // the 32-column block of small Grams (C1)
    set_smem_limit(reinterpret_cast<const void*>(herm_eig_kernel<32>), smem);
    herm_eig_kernel<32><<<unsigned(batch), kThreads, smem, ctx->stream>>>(H, n, w, floor_rel, info);
  } else {
    set_smem_limit(reinterpret_cast<const void*>(herm_eig_kernel<0>), smem);
    herm_eig_kernel<0><<<unsigned(batch), kThreads, smem, ctx->stream>>>(H, n, w, floor_rel, info);
  }
  ++ctx->launches;
  SKB_LAUNCH("herm_eig_kernel");
  if (std::getenv("SKB_PROFILE_NS")) {
    long long c[8];
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
    SKB_CUDA(cudaMemcpyFromSymbol(c, g_phase_clock, sizeof c));
    std::fprintf(stderr, "[eig n=%d] kcycles tridiag %.1f bisect %.1f invit %.1f clusters %.1f back %.1f\n", n,
                 (c[1] - c[0]) / 1e3, (c[2] - c[1]) / 1e3, (c[3] - c[2]) / 1e3, (c[4] - c[3]) / 1e3,
                 (c[5] - c[4]) / 1e3);
  }
  return true;
}

}  // namespace skb
