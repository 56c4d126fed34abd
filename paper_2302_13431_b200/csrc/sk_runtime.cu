// Host runtime: context, workspace, transform matrices, stage orchestration
// and the C-ABI (include/senskit_b200.h).  One sk_ctx per GPU; every entry
// point validates like the reference, runs on the context stream, and
// synchronises before returning.
//
// Pipeline (maps.cpp:265-330) as run here:
//   gram       K1: channel spectra (apply_axis DFT) + pair lag contraction
//                  (baseline preset: calibration-matrix gather + FP64 ZHERK)
//   nullspace  K2: FP64 block subspace iteration on the signal subspace
//                  (3xTF32 / ZGEMM-3M products, own CholQR and Ritz kernels,
//                  CUDA-graph replay), or cuSOLVER Xsyevd for the full spectrum
//   field      fold W = I - U_sig U_sig^H into lag kernels (ZHERK or straight
//                  from U_sig), K3 lag expansion -> packed G hi/lo planes
//   eigensolve K4: power iteration (+ fused normalize epilogue), or the
//                  warp-per-voxel Jacobi of the baseline preset
//   post       K5: apodised recon (before K4, timed here), interpolation with
//                  the fused SoS renormalisation, support mask
#include <algorithm>
#include <chrono>
#include <functional>
#include <cmath>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <thread>

#include "../../include/senskit_b200.h"
#include "sk_internal.h"
#include <complex>

using namespace skb;

namespace {
thread_local std::string g_last_error;
}

// ================================================================ errors
namespace skb {
[[noreturn]] void fail(int code, const std::string& msg) { throw Error(code, msg); }
void set_smem_limit(const void* func, size_t bytes) {
  // cudaFuncAttributeMaxDynamicSharedMemorySize is per device: key on both
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  size_t& g = granted[{dev, func}];
  if (bytes <= g) return;
  check_cuda(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)),
             "cudaFuncSetAttribute(max dynamic smem)");
  g = bytes;
}

void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) fail(SK_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
  fail(SK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void check_cublas(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) fail(SK_ERR_CUDA, std::string(what) + ": cuBLAS status " + std::to_string(int(s)));
}
void check_cusolver(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS)
    fail(SK_ERR_CUDA, std::string(what) + ": cuSOLVER status " + std::to_string(int(s)));
}

// ================================================================ arena
Arena::~Arena() { release_all(); }
void* Arena::get(const std::string& name, size_t bytes) {
  if (bytes == 0) bytes = 16;
  Slot& s = slots_[name];
  if (s.bytes < bytes) {
    if (s.ptr) {
      cudaFree(s.ptr);
      ++generation_;
    }
    s.ptr = nullptr;
    s.bytes = 0;
    const size_t want = (bytes + 255) & ~size_t(255);
    check_cuda(cudaMalloc(&s.ptr, want), ("cudaMalloc(" + name + ")").c_str());
    s.bytes = want;
  }
  return s.ptr;
}
void Arena::release_all() {
  for (auto& kv : slots_)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  slots_.clear();
  ++generation_;
}
MatrixCache::~MatrixCache() {
  for (auto& kv : mats) cudaFree(kv.second);
}

// ================================================================ support
Support make_support(int shape, int tau, int ndim) {  // kernels.cpp:7-35
  if (tau < 0) fail(SK_ERR_DIM, "kernel radius must be >= 0");
  if (ndim < 1) fail(SK_ERR_DIM, "kernel dimension must be >= 1");
  Support s;
  s.shape = shape;
  s.tau = tau;
  s.nd = ndim;
  const int side = 2 * tau + 1;
  std::vector<int> idx(size_t(ndim), 0);
  while (true) {
    long r2 = 0;
    for (int a = 0; a < ndim; ++a) {
      const long v = long(idx[size_t(a)]) - tau;
      r2 += v * v;
    }
    if (!(shape == 1 && r2 > long(tau) * tau))
      for (int a = 0; a < ndim; ++a) s.offsets.push_back(idx[size_t(a)] - tau);
    int a = ndim - 1;
    for (; a >= 0; --a) {
      if (++idx[size_t(a)] < side) break;
      idx[size_t(a)] = 0;
    }
    if (a < 0) break;
  }
  s.count = i64(s.offsets.size()) / ndim;
  return s;
}
}  // namespace skb

// ================================================================ helpers
namespace {

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes attr{};
  const cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// Device alias of caller-pinned host memory (cudaHostAlloc / registered), or
// nullptr (pageable host or device memory).
void* pinned_alias(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return attr.type == cudaMemoryTypeHost ? attr.devicePointer : nullptr;
}

// Device view of a caller input: the pointer itself, or an arena upload.
template <typename T>
const T* device_in(sk_ctx* ctx, const T* p, i64 count, const std::string& slot) {
  if (!p) return nullptr;
  if (is_device_ptr(p)) return p;
  T* d = ctx->arena.get<T>(slot, count);
  SKB_CUDA(cudaMemcpyAsync(d, p, size_t(count) * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return d;
}

// Device destination for a caller output (direct, or arena + copy-back).
template <typename T>
struct Out {
  T* user = nullptr;
  T* dev = nullptr;
  i64 count = 0;
  bool host = false;
  Out(sk_ctx* ctx, T* p, i64 n, const std::string& slot) : user(p), count(n) {
    if (!p) {
      dev = nullptr;
    } else if (is_device_ptr(p)) {
      dev = p;
    } else {
      host = true;
      dev = ctx->arena.get<T>(slot, n);
    }
  }
  void finish(sk_ctx* ctx) { finish_on(ctx->stream); }
  void finish_on(cudaStream_t st) {
    if (host && user) SKB_CUDA(cudaMemcpyAsync(user, dev, size_t(count) * sizeof(T), cudaMemcpyDeviceToHost, st));
  }
};

Dims dims_of(int nd, const int64_t* d) { return Dims(d, d + nd); }

// Host table -> device, ordered on the context's stream.  A synchronous
// cudaMemcpy from pageable memory may return before the DMA has landed and
// orders only the legacy default stream behind it; the kernels that read the
// table run on the context's non-blocking stream, so the copy goes onto that
// stream (found as a rare wrong-phase slice on a lane's first call:
// normalize_maps read a recon built from a partly uploaded DFT matrix).
void upload_table(sk_ctx* ctx, void* d, const void* h, size_t bytes) {
  SKB_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
  SKB_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Upload an N x L matrix (row-major) followed by its transpose (L x N).
float2* upload_matrix(sk_ctx* ctx, const std::string& key, int N, int L, const std::vector<std::complex<double>>& m) {
  auto it = ctx->matrices.mats.find(key);
  if (it != ctx->matrices.mats.end()) return it->second;
  std::vector<float2> h(size_t(2) * N * L);
  for (int j = 0; j < N; ++j)
    for (int a = 0; a < L; ++a) {
      const auto v = m[size_t(j) * L + a];
      h[size_t(j) * L + a] = make_float2(float(v.real()), float(v.imag()));
      h[size_t(N) * L + size_t(a) * N + j] = make_float2(float(v.real()), float(v.imag()));
    }
  float2* d = nullptr;
  SKB_CUDA(cudaMalloc(&d, h.size() * sizeof(float2)));
  upload_table(ctx, d, h.data(), h.size() * sizeof(float2));
  ctx->matrices.mats[key] = d;
  return d;
}

// exp(sign * i 2 pi m / n) with m reduced exactly in integers.
std::complex<double> cis(int sign, i64 m, i64 n) {
  m %= n;
  if (m < 0) m += n;
  const double ang = double(sign) * 2.0 * M_PI * double(m) / double(n);
  return {std::cos(ang), std::sin(ang)};
}

// Centred DFT taps: M[j][a] = w(a) exp(sign i 2 pi (a - a0)(j - j0) / N).
float2* dft_matrix(sk_ctx* ctx, int N, int L, i64 a0, i64 j0, int sign, double sigma) {
  const std::string key = "dft:" + std::to_string(N) + ":" + std::to_string(L) + ":" + std::to_string(a0) + ":" +
                          std::to_string(j0) + ":" + std::to_string(sign) + ":" + std::to_string(sigma);
  auto it = ctx->matrices.mats.find(key);
  if (it != ctx->matrices.mats.end()) return it->second;
  std::vector<std::complex<double>> m(size_t(N) * L);
  for (int j = 0; j < N; ++j)
    for (int a = 0; a < L; ++a) {
      double w = 1.0;
      if (sigma > 0) {
        const double f = double(a - a0);
        w = std::exp(-f * f / (2.0 * sigma * sigma));
      }
      m[size_t(j) * L + a] = w * cis(sign, (a - a0) * (j - j0), N);
    }
  return upload_matrix(ctx, key, N, L, m);
}

// Periodic-sinc interpolation along one axis (maps.cpp:54-90):
// image_to_kspace on n_low (x 1/n_low), centred zero-pad into N, kspace_to_image.
float2* sinc_matrix(sk_ctx* ctx, int N, int nl) {
  const std::string key = "sinc:" + std::to_string(N) + ":" + std::to_string(nl);
  auto it = ctx->matrices.mats.find(key);
  if (it != ctx->matrices.mats.end()) return it->second;
  const i64 cl = nl / 2, cf = N / 2;
  std::vector<std::complex<double>> m(size_t(N) * nl);
  for (int j = 0; j < N; ++j)
    for (int b = 0; b < nl; ++b) {
      std::complex<double> acc = 0;
      for (i64 f = -cl; f < nl - cl; ++f) acc += cis(+1, f * (j - cf), N) * cis(-1, f * (b - cl), nl);
      m[size_t(j) * nl + b] = acc / double(nl);
    }
  return upload_matrix(ctx, key, N, nl, m);
}

// Apply per-axis matrices last axis first: in [batch][in_ext...] -> out [batch][out_ext...].
void separable(sk_ctx* ctx, const float2* in, float2* out, i64 batch, const Dims& in_ext, const Dims& out_ext,
               const std::vector<float2*>& mats, const std::string& tag) {
  const int nd = int(in_ext.size());
  Dims cur = in_ext;
  const float2* src = in;
  for (int a = nd - 1; a >= 0; --a) {
    float2* dst;
    if (a == 0) {
      dst = out;
    } else {
      Dims next = cur;
      next[size_t(a)] = out_ext[size_t(a)];
      dst = ctx->arena.get<float2>(tag + (a % 2 ? ":a" : ":b"), batch * numel(next));
    }
    i64 b = batch, inner = 1;
    for (int k = 0; k < a; ++k) b *= cur[size_t(k)];
    for (int k = a + 1; k < nd; ++k) inner *= cur[size_t(k)];
    apply_axis(ctx, src, dst, mats[size_t(a)], b, int(in_ext[size_t(a)]), int(out_ext[size_t(a)]), inner);
    cur[size_t(a)] = out_ext[size_t(a)];
    src = dst;
  }
}

// FP64 (cos, sign*sin)(2 pi l (j - j0) / N) for j < N, l = 1..H ([j][l-1]).
double2* symdft_table64(sk_ctx* ctx, int N, int H, i64 j0, int sign) {
  const std::string key = "symcs64:" + std::to_string(N) + ":" + std::to_string(H) + ":" + std::to_string(j0) + ":" +
                          std::to_string(sign);
  auto it = ctx->matrices.mats.find(key);
  if (it != ctx->matrices.mats.end()) return reinterpret_cast<double2*>(it->second);
  std::vector<double2> h(size_t(N) * std::max(H, 1));
  for (int j = 0; j < N; ++j)
    for (int l = 1; l <= H; ++l) {
      const std::complex<double> z = cis(+1, i64(l) * (j - j0), N);
      h[size_t(j) * H + (l - 1)] = make_double2(z.real(), sign * z.imag());
    }
  double2* d = nullptr;
  SKB_CUDA(cudaMalloc(&d, h.size() * sizeof(double2)));
  upload_table(ctx, d, h.data(), h.size() * sizeof(double2));
  ctx->matrices.mats[key] = reinterpret_cast<float2*>(d);
  return d;
}

// G(x) lag expansion (spatial_gram.cpp:125-138): FP64 lag box [h][lb]^D ->
// fp32 hi/lo planes [h][grid] (sk_expand.cu).  Axes are transformed last to
// first; intermediates stay FP64.
// slab0/slab1: optional axis-0 row range [slab0, slab1) of the grid (z-slab
// sharding); the outputs then cover only those rows.
void expand_lags(sk_ctx* ctx, const double2* lags, float2* hi, lo2* lo, i64 h, int tau, const Dims& grid,
                 i64 slab0 = 0, i64 slab1 = -1) {
  const int nd = int(grid.size()), lb = 4 * tau + 1, H = 2 * tau;
  Dims cur(static_cast<size_t>(nd), lb);
  const double2* src = lags;
  for (int a = nd - 1; a >= 0; --a) {
    double2* dst = nullptr;
    if (a > 0) {
      Dims next = cur;
      next[size_t(a)] = grid[size_t(a)];
      dst = ctx->arena.get<double2>(std::string("field:tmp64") + (a % 2 ? ":a" : ":b"), h * numel(next));
    }
    i64 b = h, inner = 1;
    for (int k = 0; k < a; ++k) b *= cur[size_t(k)];
    for (int k = a + 1; k < nd; ++k) inner *= cur[size_t(k)];
    const int N = int(grid[size_t(a)]);
    const double2* cs = symdft_table64(ctx, N, H, center_index(N), -1);
    int Nout = N;
    int jc = int(center_index(N));  // centre row relative to the first output row
    if (a == 0 && slab1 >= 0) {  // rows [slab0, slab1) of the last (axis-0) stage only
      cs += slab0 * std::max(H, 1);
      Nout = int(slab1 - slab0);
      jc -= int(slab0);
    }
    expand_stage_f64(ctx, src, b, inner, H, Nout, jc, cs, dst, a == 0 ? hi : nullptr, a == 0 ? lo : nullptr);
    cur[size_t(a)] = grid[size_t(a)];
    src = dst;
  }
}

struct Planes {
  float2* hi = nullptr;
  lo2* lo = nullptr;
};

// Device index tables per (support, q), cached in the context (freed by sk_destroy).
SupportTables& tables_for(sk_ctx* ctx, const Support& s, int q) {
  const std::string key = std::to_string(s.shape) + ":" + std::to_string(s.tau) + ":" + std::to_string(s.nd) + ":" +
                          std::to_string(q);
  auto it = ctx->support_tables.find(key);
  if (it != ctx->support_tables.end()) return it->second;
  SupportTables t;
  t.lb = 4 * s.tau + 1;
  t.nbox = 1;
  std::vector<int> bs(size_t(s.nd), 1);
  for (int a = s.nd - 1; a >= 0; --a) {
    bs[size_t(a)] = t.nbox;
    t.nbox *= t.lb;
  }
  std::vector<int> off(static_cast<size_t>(s.count));
  for (i64 i = 0; i < s.count; ++i) {
    int o = 0;
    for (int a = 0; a < s.nd; ++a) o += s.off(i, a) * bs[size_t(a)];
    off[size_t(i)] = o;
  }
  const int ctr = (t.nbox - 1) / 2;
  std::vector<std::vector<int>> lists(static_cast<size_t>(t.nbox));
  for (i64 si = 0; si < s.count; ++si)
    for (i64 ti = 0; ti < s.count; ++ti)
      lists[size_t(off[size_t(ti)] - off[size_t(si)] + ctr)].push_back(int(si) | (int(ti) << 16));
  std::vector<int> ptr(size_t(t.nbox) + 1, 0), st;
  for (int l = 0; l < t.nbox; ++l) {
    ptr[size_t(l) + 1] = ptr[size_t(l)] + int(lists[size_t(l)].size());
    st.insert(st.end(), lists[size_t(l)].begin(), lists[size_t(l)].end());
  }
  std::vector<int2> pairs;
  for (int p = 0; p < q; ++p)
    for (int c = p; c < q; ++c) pairs.push_back(make_int2(p, c));
  auto up = [ctx](const void* h, size_t bytes) {
    void* d = nullptr;
    check_cuda(cudaMalloc(&d, std::max<size_t>(bytes, 16)), "cudaMalloc(table)");
    upload_table(ctx, d, h, bytes);
    return d;
  };
  t.pairs = static_cast<int2*>(up(pairs.data(), pairs.size() * sizeof(int2)));
  t.off = static_cast<int*>(up(off.data(), off.size() * sizeof(int)));
  t.lag_ptr = static_cast<int*>(up(ptr.data(), ptr.size() * sizeof(int)));
  t.lag_st = static_cast<int*>(up(st.data(), std::max<size_t>(st.size(), 1) * sizeof(int)));
  return ctx->support_tables.emplace(key, t).first->second;
}

i64 next_pow2(i64 n) {
  i64 p = 1;
  while (p < n) p <<= 1;
  return p;
}

void check_calib(const Dims& cdims, i64 q, const Support& s) {  // calibration.cpp:12-20
  if (cdims.empty()) fail(SK_ERR_DIM, "stack needs at least one axis");
  for (i64 d : cdims)
    if (d < 1) fail(SK_ERR_DIM, "stack axis extents must be >= 1");
  if (q < 1) fail(SK_ERR_DIM, "stack needs at least one channel");
  if (i64(cdims.size()) != s.nd) fail(SK_ERR_DIM, "support dimension does not match calibration region");
  for (i64 d : cdims)
    if (d <= 2 * s.tau) fail(SK_ERR_DIM, "calibration region too small for kernel radius " + std::to_string(s.tau));
  if (cdims.size() > 3) fail(SK_ERR_UNSUPPORTED, "more than 3 dimensions is outside the B200 path");
}

// ---------------------------------------------------------------- K1
// slices > 1: calib [slices][Q][E..] -> gram_dst [slices][n][n] (multislice groups: the channel
// spectra over slices x channels, the pair kernel with the slice on grid.y).
float2* run_gram(sk_ctx* ctx, const Dims& cdims, i64 q, const float2* calib, const Support& s, float2* gram_dst,
                 i64 slices = 1) {
  const int nd = int(cdims.size());
  const i64 lam = s.count, n = q * lam;
  Dims pad(cdims.size());
  for (size_t a = 0; a < cdims.size(); ++a) pad[a] = next_pow2(cdims[a] + 2 * s.tau);  // calibration.cpp:89-93
  std::vector<float2*> mats(static_cast<size_t>(nd));
  for (int a = 0; a < nd; ++a) mats[size_t(a)] = dft_matrix(ctx, int(pad[size_t(a)]), int(cdims[size_t(a)]), 0, 0, -1, 0.0);
  float2* spectra = ctx->arena.get<float2>("gram:spectra", slices * q * numel(pad));
  if (nd == 2 && sep2d_smem(int(cdims[0]), int(cdims[1]), int(pad[0]), int(pad[1])) <= 160 * 1024)
    sep2d(ctx, calib, spectra, slices * q, int(cdims[0]), int(cdims[1]), int(pad[0]), int(pad[1]), mats[0], mats[1]);
  else
    separable(ctx, calib, spectra, slices * q, cdims, pad, mats, "gram:tmp");
  SupportTables& t = tables_for(ctx, s, int(q));
  GramGeom g{};
  g.nd = nd;
  g.pad[0] = g.pad[1] = g.pad[2] = 1;
  for (int a = 0; a < nd; ++a) g.pad[a] = int(pad[size_t(a)]);
  g.lb = 4 * s.tau + 1;
  g.tau = s.tau;
  g.q = int(q);
  g.lam = int(lam);
  // twiddles e^{+i 2 pi m / P_a}
  std::vector<std::complex<double>> tw;
  for (int a = 0; a < 3; ++a)
    for (int m = 0; m < g.pad[a]; ++m) tw.push_back(cis(+1, m, g.pad[a]));
  const std::string key = "gramtw:" + std::to_string(g.pad[0]) + ":" + std::to_string(g.pad[1]) + ":" +
                          std::to_string(g.pad[2]);
  float2* d_tw = upload_matrix(ctx, key, int(tw.size()), 1, tw);
  float2* gram = gram_dst ? gram_dst : ctx->arena.get<float2>("gram:G", slices * n * n);
  gram_pairs_launch(ctx, spectra, g, t.pairs, int(q * (q + 1) / 2), t.off, d_tw, gram, int(slices));
  return gram;
}

// Support offsets (|Lambda| x nd, kernels.cpp:7-35) on the device, cached per context.
const int* support_offsets_dev(sk_ctx* ctx, const Support& s) {
  const std::string key = "suppoff:" + std::to_string(s.shape) + ":" + std::to_string(s.tau) + ":" + std::to_string(s.nd);
  auto it = ctx->tables.find(key);
  if (it != ctx->tables.end()) return static_cast<const int*>(it->second);
  void* d = nullptr;
  SKB_CUDA(cudaMalloc(&d, std::max<size_t>(1, s.offsets.size()) * sizeof(int)));
  upload_table(ctx, d, s.offsets.data(), s.offsets.size() * sizeof(int));
  ctx->tables[key] = d;
  return static_cast<const int*>(d);
}

i64 valid_shift_rows(const Dims& cdims, int tau) {
  i64 p = 1;
  for (i64 d : cdims) p *= std::max<i64>(0, d - 2 * tau);
  return p;
}

// Baseline Gram (calibration.cpp:30-78): C gathered in FP64, C^H C by one
// ZHERK, mirrored into the full Hermitian c64 matrix.
float2* run_gram_explicit(sk_ctx* ctx, const Dims& cdims, i64 q, const float2* calib, const Support& s,
                          float2* gram_dst) {
  const i64 n = q * s.count, rows = valid_shift_rows(cdims, s.tau);
  double2* c = ctx->arena.get<double2>("gramx:C", std::max<i64>(1, rows * n));
  double2* lower = ctx->arena.get<double2>("gramx:lower", n * n);
  calib_matrix(ctx, calib, cdims, int(q), s, support_offsets_dev(ctx, s), c);
  float2* gram = gram_dst ? gram_dst : ctx->arena.get<float2>("gram:G", n * n);
  gram_explicit_dev(ctx, c, rows, n, lower, gram);
  return gram;
}

// ---------------------------------------------------------------- K2
struct Eig {
  std::vector<double> evals;  // ascending
  double2* evecs = nullptr;   // n x n column-major, device (full solver only)
  const double2* usig = nullptr;  // n x k signal eigenvectors (lambda >= cut^2), device
  i64 n = 0, rank = 0, k = 0;
  double sigma1 = 0, cut = 0, margin = 0;
  std::vector<double> spectrum;  // descending sigma (subspace solver: top block only, rest 0)
  bool full = true, certified = false;
  int iterations = 0, block = 0;
};

Eig run_eigh(sk_ctx* ctx, const float2* gram, i64 n, double ratio) {  // nullspace.cpp:7-35
  if (!(ratio > 0.0 && ratio < 1.0)) fail(SK_ERR_DIM, "nullspace threshold ratio must lie in (0,1)");
  if (n <= 0) fail(SK_ERR_DIM, "Gram matrix must be square");
  Eig e;
  e.n = n;
  e.evecs = ctx->arena.get<double2>("eig:A", n * n);
  c64_to_c128(ctx, gram, e.evecs, n * n);
  double* d_w = ctx->arena.get<double>("eig:w", n);
  size_t dev_bytes = 0, host_bytes = 0;
  check_cusolver(cusolverDnXsyevd_bufferSize(ctx->cusolver, ctx->cusolver_params, CUSOLVER_EIG_MODE_VECTOR,
                                             CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, e.evecs, n, CUDA_R_64F, d_w,
                                             CUDA_C_64F, &dev_bytes, &host_bytes),
                 "Xsyevd_bufferSize");
  void* d_work = ctx->arena.get("eig:work", dev_bytes);
  static thread_local std::vector<unsigned char> h_work;
  h_work.resize(std::max<size_t>(host_bytes, 1));
  int* d_info = ctx->arena.get<int>("eig:info", 1);
  check_cusolver(cusolverDnXsyevd(ctx->cusolver, ctx->cusolver_params, CUSOLVER_EIG_MODE_VECTOR,
                                  CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, e.evecs, n, CUDA_R_64F, d_w, CUDA_C_64F,
                                  d_work, dev_bytes, h_work.data(), host_bytes, d_info),
                 "Xsyevd");
  ++ctx->lib_calls;
  e.evals.resize(size_t(n));
  int info = 0;
  SKB_CUDA(cudaMemcpyAsync(e.evals.data(), d_w, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SKB_CUDA(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (info != 0) fail(SK_ERR_OTHER, "Gram eigendecomposition failed");
  std::vector<double> sig(static_cast<size_t>(n));
  for (i64 i = 0; i < n; ++i) sig[size_t(i)] = std::sqrt(std::max(0.0, e.evals[size_t(i)]));
  e.spectrum.assign(sig.rbegin(), sig.rend());
  e.sigma1 = e.spectrum[0];
  e.cut = ratio * e.sigma1;
  i64 r = 0;
  while (r < n && sig[size_t(r)] < e.cut) ++r;
  e.rank = r;
  double margin = 1e300;
  for (double sv : sig)
    if (e.cut > 0) margin = std::min(margin, std::fabs(sv / e.cut - 1.0));
  e.margin = margin;
  if (r == 0) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "%f", ratio);
    fail(SK_ERR_NULLSPACE_EMPTY, std::string("calibration matrix has no approximate nullspace at ratio ") + buf);
  }
  e.k = n - r;
  e.usig = e.evecs + r * n;
  e.full = true;
  return e;
}

// ---------------------------------------------------------------- K2 (subspace)
// The pipeline needs only the signal subspace {lambda >= (ratio*sigma_1)^2}
// (k = n - R ~ 20-50 vectors) and the count R.  Block subspace
// iteration with Rayleigh-Ritz on the FP64-promoted Gram (3xTF32 steering
// products, ZGEMM-3M for the last steps, CholQR orthonormalisation, the own
// one-CTA eigensolver for b <= 64 else cuSOLVER on the b x b projection)
// returns exactly that.  Convergence: every Ritz pair with theta >= cut^2/2 has
// ||A v - theta v|| <= tol*theta_max, and the block extends below cut^2/2 so
// no eigenvalue above the cut can hide outside it.  Optional certification:
// Cholesky of cut^2*I - A + 2 theta_max U U^H succeeds iff lambda_{k+1} < cut^2
// (with U the k Ritz vectors above the cut), i.e. R is exact.  Any failure
// falls back to the full eigensolver.
struct SubspaceStatus {
  bool ok = false;
};

void zgemm(sk_ctx* ctx, cublasOperation_t ta, cublasOperation_t tb, i64 m, i64 n, i64 k, const double2* a, i64 lda,
           const double2* b, i64 ldb, double2* c, i64 ldc) {
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  // Gauss 3M form (three real DGEMMs instead of four) for the large n x b x n
  // products (C2 K2 1.376 -> 1.342 ms, C5 9.08 -> 8.28 ms against ZGEMM).
  auto gemm = m * n * k >= (i64(1) << 26) ? cublasZgemm3m : cublasZgemm;
  check_cublas(gemm(ctx->cublas, ta, tb, int(m), int(n), int(k), &one,
                           reinterpret_cast<const cuDoubleComplex*>(a), int(lda),
                           reinterpret_cast<const cuDoubleComplex*>(b), int(ldb), &zero,
                           reinterpret_cast<cuDoubleComplex*>(c), int(ldc)),
               "Zgemm");
  ++ctx->lib_calls;
}

// In-place Cholesky-QR of X (n x b).  Returns false if X is numerically rank deficient.
bool cholqr(sk_ctx* ctx, double2* x, i64 n, i64 b) {
  double2* s = ctx->arena.get<double2>("ss:S", b * b);
  const double one = 1.0, zero = 0.0;
  check_cublas(cublasZherk(ctx->cublas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, int(b), int(n), &one,
                           reinterpret_cast<const cuDoubleComplex*>(x), int(n), &zero,
                           reinterpret_cast<cuDoubleComplex*>(s), int(b)),
               "Zherk(cholqr)");
  size_t dbytes = 0, hbytes = 0;
  check_cusolver(cusolverDnXpotrf_bufferSize(ctx->cusolver, ctx->cusolver_params, CUBLAS_FILL_MODE_LOWER, b,
                                             CUDA_C_64F, s, b, CUDA_C_64F, &dbytes, &hbytes),
                 "Xpotrf_bufferSize");
  void* dwork = ctx->arena.get("ss:potrf_work", dbytes);
  static thread_local std::vector<unsigned char> hwork;
  hwork.resize(std::max<size_t>(hbytes, 1));
  int* info = ctx->arena.get<int>("ss:info", 1);
  check_cusolver(cusolverDnXpotrf(ctx->cusolver, ctx->cusolver_params, CUBLAS_FILL_MODE_LOWER, b, CUDA_C_64F, s, b,
                                  CUDA_C_64F, dwork, dbytes, hwork.data(), hbytes, info),
                 "Xpotrf");
  const cuDoubleComplex onec = make_cuDoubleComplex(1.0, 0.0);
  check_cublas(cublasZtrsm(ctx->cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT,
                           int(n), int(b), &onec, reinterpret_cast<const cuDoubleComplex*>(s), int(b),
                           reinterpret_cast<cuDoubleComplex*>(x), int(n)),
               "Ztrsm");
  ctx->lib_calls += 3;
  int h_info = 0;
  SKB_CUDA(cudaMemcpyAsync(&h_info, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  return h_info == 0;
}

// Eigendecomposition of the b x b Rayleigh-Ritz matrix (lower triangle used),
// eigenvalues ascending into w, eigenvectors overwrite H: the own one-CTA
// solver for b <= 64 (sk_eig.cu; 0.27 ms at b = 64 against ~1 ms for
// cuSOLVER's Jacobi, divide-and-conquer or batched solvers, all measured),
// cuSOLVER Jacobi (ZHEEVJ, tol 1e-14) above.
void small_heev(sk_ctx* ctx, double2* H, i64 b, double* w, int* d_info, double floor_rel = 0.0) {
  if (herm_eig_small(ctx, H, int(b), w, d_info, floor_rel)) return;
  if (!ctx->syevj) {
    check_cusolver(cusolverDnCreateSyevjInfo(&ctx->syevj), "CreateSyevjInfo");
    check_cusolver(cusolverDnXsyevjSetTolerance(ctx->syevj, 1e-14), "syevjSetTolerance");
    check_cusolver(cusolverDnXsyevjSetMaxSweeps(ctx->syevj, 30), "syevjSetMaxSweeps");
  }
  syevjInfo_t params = ctx->syevj;
  int lwork = 0;
  check_cusolver(cusolverDnZheevj_bufferSize(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, int(b),
                                             reinterpret_cast<cuDoubleComplex*>(H), int(b), w, &lwork, params),
                 "Zheevj_bufferSize");
  auto* work = ctx->arena.get<cuDoubleComplex>("ss:syevj_work", std::max(lwork, 1));
  check_cusolver(cusolverDnZheevj(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, int(b),
                                  reinterpret_cast<cuDoubleComplex*>(H), int(b), w, work, lwork, d_info, params),
                 "Zheevj");
  ++ctx->lib_calls;
}

// Orthonormalise X (n x b) in place by `passes` CholQR passes.  b = 64 and
// n >= 1024, b = 32 and n >= 128: the own kernels of sk_cholqr.cu (gram,
// one-CTA Cholesky, row TRSM; at b = 32 they took C1's K2 0.56 -> 0.50 ms
// against the library pass).  b <= 256 otherwise: own cross_gram + cuSOLVER
// POTRF + cuBLAS TRSM (measured against own one-CTA Cholesky variants and a
// lane-pair TRSM: faster once graphs hide the library's host cost).  Larger
// blocks: cuBLAS HERK + POTRF + TRSM with a synchronous check.  Returns false
// only on a detected (synchronous path) failure; the other paths raise `flag`.
bool orth(sk_ctx* ctx, double2*& x, double2*& tmp, i64 n, i64 b, int* flag, int passes = 2,
          const CatIO& io = CatIO()) {
  (void)tmp;
  if ((b == 64 && n >= 1024) || (b == 32 && n >= 128)) {
    cholqr_b(ctx, int(b), x, n, passes, flag, io);
    return true;
  }
  if (b > 256) {
    for (int p = 0; p < passes; ++p)
      if (!cholqr(ctx, x, n, b)) return false;
    return true;
  }
  double2* S = ctx->arena.get<double2>("ss:S", b * b);
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
  for (int pass = 0; pass < passes; ++pass) {
    cross_gram(ctx, x, x, n, int(b), S);  // S = X^H X
    size_t dbytes = 0, hbytes = 0;
    check_cusolver(cusolverDnXpotrf_bufferSize(ctx->cusolver, ctx->cusolver_params, CUBLAS_FILL_MODE_LOWER, b,
                                               CUDA_C_64F, S, b, CUDA_C_64F, &dbytes, &hbytes),
                   "Xpotrf_bufferSize");
    void* dwork = ctx->arena.get("ss:potrf_work", dbytes);
    static thread_local std::vector<unsigned char> hwork;
    hwork.resize(std::max<size_t>(hbytes, 1));
    check_cusolver(cusolverDnXpotrf(ctx->cusolver, ctx->cusolver_params, CUBLAS_FILL_MODE_LOWER, b, CUDA_C_64F, S, b,
                                    CUDA_C_64F, dwork, dbytes, hwork.data(), hbytes, flag + 1),
                   "Xpotrf");
    check_cublas(cublasZtrsm(ctx->cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT,
                             int(n), int(b), &one, reinterpret_cast<const cuDoubleComplex*>(S), int(b),
                             reinterpret_cast<cuDoubleComplex*>(x), int(n)),
                 "Ztrsm(orth)");  // X <- X L^{-H}
    ctx->lib_calls += 2;
  }
  return true;
}

// Development aid (SKB_PROFILE_NS=1): event laps inside the subspace solver,
// summed per phase label and printed to stderr when the solver returns.
struct PhaseLaps {
  sk_ctx* ctx;
  bool on;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  std::vector<double> host_us;
  explicit PhaseLaps(sk_ctx* c) : ctx(c), on(std::getenv("SKB_PROFILE_NS") != nullptr) { lap("start"); }
  void lap(const char* label) {
    if (!on) return;
    cudaEvent_t e;
    SKB_CUDA(cudaEventCreate(&e));
    SKB_CUDA(cudaEventRecord(e, ctx->stream));
    ev.emplace_back(label, e);
    host_us.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch())
                          .count());
  }
  ~PhaseLaps() {
    if (!on) return;
    cudaEventSynchronize(ev.back().second);
    std::map<std::string, std::pair<double, int>> sum;
    std::map<std::string, double> hsum;
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      auto& s = sum[ev[i].first];
      s.first += ms;
      s.second += 1;
      hsum[ev[i].first] += (host_us[i] - host_us[i - 1]) * 1e-3;
    }
    for (auto& kv : sum)
      std::fprintf(stderr, "[ns] %-10s %8.3f ms  %3dx   host enqueue %8.3f ms\n", kv.first.c_str(), kv.second.first,
                   kv.second.second, hsum[kv.first]);
    for (auto& p : ev) cudaEventDestroy(p.second);
  }
};

// Replay of one subspace round as a CUDA graph.  The first call with a key
// runs eagerly (the arena grows to its final size), the second captures the
// launch sequence, later calls replay it and restore the V/Y/T rotation of
// the captured run.  A capture failure (a library call that cannot be
// captured) marks the key eager-only.  Graphs bake in arena pointers beyond
// the key (Cholesky / Ritz scratch slots), so every captured round is dropped
// as soon as the arena frees any slot (Arena::generation).
void drop_stale_rounds(sk_ctx* ctx) {
  if (ctx->rounds_generation == ctx->arena.generation()) return;
  for (auto& kv : ctx->rounds)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  ctx->rounds.clear();
  ctx->rounds_generation = ctx->arena.generation();
}

void run_graphed(sk_ctx* ctx, bool allowed, const RoundKey& key, double2*& V, double2*& Y, double2*& T,
                 const std::function<void()>& body) {
  static const bool disabled = std::getenv("SKB_NO_GRAPH") != nullptr;
  if (!allowed || disabled) {
    body();
    return;
  }
  drop_stale_rounds(ctx);
  auto& g = ctx->rounds[key];
  if (g.exec) {
    SKB_CUDA(cudaGraphLaunch(g.exec, ctx->stream));
    V = g.v;
    Y = g.y;
    T = g.t;
    ctx->launches += g.launches;
    ctx->lib_calls += g.lib_calls;
    return;
  }
  // First sight of a key runs eagerly (allocates the round's buffers) unless
  // this size already ran a round: then the new step plan is captured at once,
  // so a plan change costs one capture, not an extra eager call plus a capture.
  const std::pair<i64, i64> size{key.n, key.b};
  const bool warm = ctx->warm_rounds.count(size) != 0;
  if (g.bad || (g.seen++ == 0 && !warm)) {
    body();
    ctx->warm_rounds.insert(size);
    return;
  }
  const i64 l0 = ctx->launches, c0 = ctx->lib_calls;
  cudaGraph_t graph = nullptr;
  SKB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
  double2 *v0 = V, *y0 = Y, *t0 = T;
  try {
    body();
  } catch (...) {
    cudaStreamEndCapture(ctx->stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    g.bad = true;
    V = v0;
    Y = y0;
    T = t0;
    ctx->launches = l0;
    ctx->lib_calls = c0;
    body();  // eager
    return;
  }
  const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &graph);
  if (ec != cudaSuccess || !graph || cudaGraphInstantiate(&g.exec, graph, 0) != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    g.bad = true;
    g.exec = nullptr;
    V = v0;
    Y = y0;
    T = t0;
    ctx->launches = l0;
    ctx->lib_calls = c0;
    body();
    return;
  }
  cudaGraphDestroy(graph);
  g.v = V;
  g.y = Y;
  g.t = T;
  g.launches = ctx->launches - l0;
  g.lib_calls = ctx->lib_calls - c0;
  if (ctx->rounds_generation != ctx->arena.generation()) {
    // the capture itself grew a slot: older rounds are stale, this one is current
    for (auto& kv : ctx->rounds) {
      const bool same = !(kv.first < key) && !(key < kv.first);
      if (!same && kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    }
    RoundGraph keep = g;
    ctx->rounds.clear();
    ctx->rounds[key] = keep;
    ctx->rounds_generation = ctx->arena.generation();
  }
  SKB_CUDA(cudaGraphLaunch(ctx->rounds[key].exec, ctx->stream));  // capture recorded, not ran, the round
}

// FP64 steps at the end of a round, before the (FP64) projection product; the
// steps before them are 3xTF32 steering steps.  Two for the single solver at
// b = 64 / 96; one where an FP64 step costs much more than a steering step and
// the same step count still converges: the batched solver (C3: iterations
// unchanged at 6, worst residual 1.1e-11 against the 3e-10 tolerance, 50.3 ->
// 48.0 ms per 128 slices), the 32-column block of small Grams (C1 K2 0.45
// -> 0.41 ms) and the wide blocks of big Grams (C5, b = 96: K2 6.8 -> 6.5 ms).  Measured the other way on C2: one FP64 step needs a ninth
// iteration (two more steering steps for one FP64 step saved, K2 1.27 -> 1.30
// ms).  The convergence test is the same either way.
constexpr int kFp64StepsSingle = 2, kFp64StepsSmall = 1, kFp64StepsBatched = 1;

bool run_eigh_subspace(sk_ctx* ctx, const float2* gram, i64 n, double ratio, bool certify, Eig& e) {
  PhaseLaps laps(ctx);
  e = Eig();
  e.n = n;
  e.full = false;
  double2* A = ctx->arena.get<double2>("eig:A", n * n);
  // Steering products as 3xTF32 tensor-core GEMMs over the K-concatenated
  // split Gram [A_hi | A_lo] (measured: plain FP32 CGEMM slower; single TF32
  // or BF16 double the step count, the wanted subspace reaching down to
  // ratio^2 * lambda_1; three separate hi/lo GEMMs read the split Gram 3x).
  float* ghi = ctx->arena.get<float>("ss:gcat", 4 * n * n);
  float* glo = ghi + 2 * n * n;
  promote_split_gram(ctx, gram, n, A, ghi, glo);  // FP64 copy + split in one pass
  laps.lap("promote");
  // Per-size hints from the previous call: block size and the number of
  // orthogonalised iterations before the (single) Rayleigh-Ritz check.
  auto& hint = ctx->subspace_hint;
  // Block size: small-matrix latency dominates up to n ~ 4k (b = 64 measured
  // best for C2/C3/C4), the n^2 b GEMM beyond (b = 96 best for C5).
  const bool big = n > 4096;
  i64 b = big ? 96 : 64;
  int q_plan = 3;
  auto it_h = hint.find(n);
  if (it_h != hint.end()) {
    const i64 k_prev = it_h->second.m;
    // big Grams: k + 32 rounded to 32, at least 96 (C5, k = 59: K2 8.3 -> 7.0 ms
    // against 128 columns once the FP64 products moved to ZGEMM 3M)
    b = big ? std::max<i64>(96, ((k_prev + 32 + 31) / 32) * 32) : std::max<i64>(64, ((k_prev + 16 + 15) / 16) * 16);
    // small Grams (library CholQR path, n < 1024) with a small signal space:
    // a 32-column block (C1, k = 21: K2 0.65 -> 0.54 ms; 48 columns measured
    // in between, C3's n = 1568 slower with 48 than with 64)
    if (!big && n < 1024 && k_prev + 11 <= 32) b = 32;
    q_plan = it_h->second.plan;
  }
  const int first_plan = q_plan;
  int rounds = 0;
  b = std::min(b, n);
  const i64 bcap = std::min(n, std::max<i64>(4 * b, 256));
  double2* V = ctx->arena.get<double2>("ss:V", n * bcap);
  double2* Y = ctx->arena.get<double2>("ss:Y", n * bcap);
  double2* T = ctx->arena.get<double2>("ss:T", n * bcap);
  double2* H = ctx->arena.get<double2>("ss:H", bcap * bcap);
  // w, residuals and the info triple in one slot: [w: bcap][res: bcap][info: 4 ints]
  const size_t wri = size_t(2 * bcap + 2);
  double* w = ctx->arena.get<double>("ss:wri", i64(wri));
  double* res = w + bcap;
  int* d_info = reinterpret_cast<int*>(w + 2 * bcap);
  if (ctx->hpin_cap < wri) {
    if (ctx->hpin) SKB_CUDA(cudaFreeHost(ctx->hpin));
    SKB_CUDA(cudaMallocHost(&ctx->hpin, wri * sizeof(double)));
    ctx->hpin_cap = wri;
  }
  int* flag = d_info + 1;
  SKB_CUDA(cudaMemsetAsync(d_info, 0, 3 * sizeof(int), ctx->stream));
  // A Gaussian start block is well conditioned and only its span matters:
  // no orthonormalisation before the first product.
  random_block(ctx, V, n, b, 0, 0x5eed5u);
  laps.lap("misc");
  const double tol = 3e-10;
  const int maxit = 80;
  const i64 guard = 8;
  std::vector<double> hw(static_cast<size_t>(bcap)), hres(static_cast<size_t>(bcap));
  bool converged = false;
  double last_worst = 0.0, last_rate = 0.0;
  int iters = 0;
  i64 m = 0;
  double theta_max = 0.0, c = 0.0;
  while (iters < maxit) {
    // One round: q_plan (GEMM, CholQR) steps, the projection, the b x b
    // eigensolve, the Ritz rotation and residuals.  No host decisions inside,
    // so in steady state (per-size hint fixed) it is replayed as a CUDA graph.
    bool body_ok = true;
    auto body = [&]() {
      // With the own CholQR kernels a steering step is GEMM + CholQR only: the
      // kernels read the concatenated product directly and the solve writes
      // the next step's split operand (CatIO) -- no combine / split passes
      // between them (nine launches fewer per C2 call; K2 time C1 0.47 -> 0.45 ms,
      // C4 2.63 -> 2.61 ms, C2 unchanged: the small passes were not on the critical path).
      const bool cat_io = (b == 64 && n >= 1024) || (b == 32 && n >= 128);
      const int nf64 = b == 64 ? kFp64StepsSingle : kFp64StepsSmall;  // (b = 32, and b >= 96: see above)
      bool have_split = false;
      for (int i = 0; i < q_plan; ++i) {
        CatIO io;
        if (i + nf64 < q_plan) {
          // 3xTF32 on tensor cores: [A_hi | A_lo] (2n x 2n) [[V_hi, V_lo]; [0, V_hi]]
          // (2n x 4b), the split Gram read once per step.
          const float one = 1.f, zero = 0.f;
          float* vcat = ctx->arena.get<float>("ss:vcat", 2 * n * 4 * bcap);
          float* ccat = ctx->arena.get<float>("ss:ccat", 2 * n * 4 * bcap);
          if (!have_split) split_block_cat_tf32(ctx, V, n, b, vcat);
          check_cublas(cublasGemmEx(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, int(2 * n), int(4 * b), int(2 * n), &one,
                                    ghi, CUDA_R_32F, int(2 * n), vcat, CUDA_R_32F, int(2 * n), &zero, ccat,
                                    CUDA_R_32F, int(2 * n), CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT),
                       "GemmEx(3xTF32 cat)");
          ++ctx->lib_calls;
          have_split = false;
          if (cat_io) {
            io.ccat = ccat;
            if ((i + 1) + nf64 < q_plan) {  // the next step is a steering step too
              io.vcat = vcat;
              have_split = true;
            }
          } else {
            combine_block_cat(ctx, ccat, n, b, Y);
          }
          laps.lap("gemm32");
        } else {
          zgemm(ctx, CUBLAS_OP_N, CUBLAS_OP_N, n, b, n, A, n, V, n, Y, n);  // Y = A V
          laps.lap("gemm64");
        }
        std::swap(V, Y);
        // Only the span matters between Rayleigh-Ritz steps: one CholQR pass
        // (orthogonality ~ kappa^2 eps) except before the projection.
        if (!orth(ctx, V, T, n, b, flag, i + 1 == q_plan ? 2 : 1, io)) {
          body_ok = false;
          return;
        }
        laps.lap("orth");
      }
      zgemm(ctx, CUBLAS_OP_N, CUBLAS_OP_N, n, b, n, A, n, V, n, Y, n);
      laps.lap("gemm64");
      // Rayleigh-Ritz on span(V): H = V^H A V = S diag(w) S^H.
      if ((b == 64 && n >= 1024) || (b == 32 && n >= 128)) {
        gram_blk(ctx, int(b), V, Y, n, H);
      } else if (b <= 256) {
        cross_gram(ctx, V, Y, n, int(b), H);
      } else {
        zgemm(ctx, CUBLAS_OP_C, CUBLAS_OP_N, b, b, n, V, n, Y, n, H, b);
      }
      laps.lap("rr_gram");
      // Ritz pairs below cut^2 / 2 are never used individually (the residual
      // test and the split both start there): a floor of cut^2 / 4 is safe.
      small_heev(ctx, H, b, w, d_info, 0.25 * ratio * ratio);
      laps.lap("rr_heev");
      zgemm(ctx, CUBLAS_OP_N, CUBLAS_OP_N, n, b, b, V, n, H, b, T, n);  // V <- V S
      std::swap(V, T);
      zgemm(ctx, CUBLAS_OP_N, CUBLAS_OP_N, n, b, b, Y, n, H, b, T, n);  // Y <- Y S
      std::swap(Y, T);
      ritz_residuals(ctx, Y, V, w, n, b, res);
      laps.lap("rr_rotate");
    };
    run_graphed(ctx, !laps.on && b <= 256,
                RoundKey{n, b, q_plan, V, Y, T, H, w, res, d_info, A, gram, ratio}, V, Y, T, body);
    if (!body_ok) return false;
    iters += q_plan + 1;
    ++rounds;
    SKB_CUDA(cudaMemcpyAsync(ctx->hpin, w, wri * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
    std::copy(ctx->hpin, ctx->hpin + b, hw.begin());
    std::copy(ctx->hpin + bcap, ctx->hpin + bcap + b, hres.begin());
    int hinfo[3];
    std::memcpy(hinfo, ctx->hpin + 2 * bcap, sizeof hinfo);
    laps.lap("sync");
    if (hinfo[0] != 0 || hinfo[1] != 0 || hinfo[2] != 0) return false;  // syevd failure / rank-deficient block
    theta_max = hw[size_t(b - 1)];
    if (!(theta_max > 0.0)) return false;
    c = ratio * ratio * theta_max;
    m = 0;
    for (i64 i = 0; i < b; ++i) m += hw[size_t(i)] >= c ? 1 : 0;
    if (m > b - guard && b < n) {
      const i64 nb = std::min(n, std::min(bcap, 2 * b));
      if (nb <= b) return false;
      random_block(ctx, V, n, nb - b, b, 0x5eed5u + unsigned(iters));
      b = nb;
      if (!orth(ctx, V, T, n, b, flag)) return false;
      q_plan = 3;
      rounds = -1000;  // block grown: this call says nothing about the plan
      continue;
    }
    // Converged when every Ritz pair at or above cut^2/2 has a small residual and
    // the block reaches below cut^2/2.
    double worst = 0.0, rate = 0.0;
    bool reaches = hw[0] < 0.5 * c || b == n;
    for (i64 i = 0; i < b; ++i) {
      if (hw[size_t(i)] < 0.5 * c) continue;
      const double r = std::sqrt(std::max(hres[size_t(i)], 0.0)) / theta_max;
      worst = std::max(worst, r);
      rate = std::max(rate, std::max(hw[0], 0.0) / hw[size_t(i)]);
    }
    if (reaches && worst <= tol) {
      converged = true;
      last_worst = worst;
      last_rate = rate;
      break;
    }
    // Predict the remaining iterations from the observed Ritz-value ratios.
    int extra = 1;
    if (reaches && rate > 0.0 && rate < 1.0 && worst > 0.0)
      extra = int(std::ceil(std::log(tol / worst) / std::log(rate)));
    q_plan = std::max(1, std::min(extra, 20));
  }
  if (!converged) return false;
  if (m == 0 || m == n) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "%f", ratio);
    fail(SK_ERR_NULLSPACE_EMPTY, std::string("calibration matrix has no approximate nullspace at ratio ") + buf);
  }
  double2* U = V + (b - m) * n;  // the last m Ritz columns (ascending theta)
  if (certify) {
    double2* M = ctx->arena.get<double2>("ss:M", n * n);
    shift_negate(ctx, A, M, n, c);
    const double alpha = 2.0 * theta_max, one = 1.0;
    check_cublas(cublasZherk(ctx->cublas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, int(n), int(m), &alpha,
                             reinterpret_cast<const cuDoubleComplex*>(U), int(n), &one,
                             reinterpret_cast<cuDoubleComplex*>(M), int(n)),
                 "Zherk(certify)");
    size_t dbytes = 0, hbytes = 0;
    check_cusolver(cusolverDnXpotrf_bufferSize(ctx->cusolver, ctx->cusolver_params, CUBLAS_FILL_MODE_LOWER, n,
                                               CUDA_C_64F, M, n, CUDA_C_64F, &dbytes, &hbytes),
                   "Xpotrf_bufferSize(certify)");
    void* dwork = ctx->arena.get("ss:cert_work", dbytes);
    static thread_local std::vector<unsigned char> hwork2;
    hwork2.resize(std::max<size_t>(hbytes, 1));
    check_cusolver(cusolverDnXpotrf(ctx->cusolver, ctx->cusolver_params, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, M, n,
                                    CUDA_C_64F, dwork, dbytes, hwork2.data(), hbytes, d_info),
                   "Xpotrf(certify)");
    ctx->lib_calls += 2;
    int h_info = 0;
    SKB_CUDA(cudaMemcpyAsync(&h_info, d_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h_info != 0) return false;  // an eigenvalue >= cut^2 outside the Ritz set: use the full solver
    e.certified = true;
  }
  double2* keep = ctx->arena.get<double2>("ss:U", n * m);
  SKB_CUDA(cudaMemcpyAsync(keep, U, size_t(n * m) * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream));
  laps.lap("finish");
  e.usig = keep;
  e.k = m;
  e.rank = n - m;
  e.sigma1 = std::sqrt(theta_max);
  e.cut = ratio * e.sigma1;
  e.spectrum.assign(size_t(n), 0.0);
  for (i64 i = 0; i < b; ++i) e.spectrum[size_t(i)] = std::sqrt(std::max(0.0, hw[size_t(b - 1 - i)]));
  double margin = 1e300;
  for (i64 i = 0; i < b; ++i) margin = std::min(margin, std::fabs(e.spectrum[size_t(i)] / e.cut - 1.0));
  e.margin = margin;
  e.iterations = iters;
  e.block = int(b);
  // Step plan for the next call of this size: the steps this call used, one
  // fewer when the final residual shows that one step less would still have
  // converged (residual one step earlier ~ worst / rate, 0.8x margin) and
  // that plan never needed an extra round before.
  auto& h = hint[n];
  if (rounds > 1 && it_h != hint.end()) h.failed_plan = std::max(h.failed_plan, first_plan);
  int plan = std::max(1, iters - 1);
  if (last_rate > 0.0 && last_rate < 1.0 && last_worst <= 0.8 * tol * last_rate && plan > 3 &&
      plan - 1 > h.failed_plan)
    --plan;
  if (std::getenv("SKB_PROFILE_NS"))
    std::fprintf(stderr, "[ns] n=%lld iters=%d rounds=%d worst=%.3e rate=%.3e next_plan=%d failed=%d\n", (long long)n,
                 iters, rounds, last_worst, last_rate, plan, h.failed_plan);
  h.m = m;
  h.plan = plan;
  return true;
}

// Nullspace stage dispatcher: solver 0 = auto (subspace unless the full
// spectrum is requested or n is small), 1 = full cuSOLVER, 2 = subspace.
Eig run_nullspace(sk_ctx* ctx, const float2* gram, i64 n, double ratio, int solver, bool need_spectrum,
                  bool certify) {
  if (!(ratio > 0.0 && ratio < 1.0)) fail(SK_ERR_DIM, "nullspace threshold ratio must lie in (0,1)");
  const bool subspace = solver == 2 || (solver == 0 && !need_spectrum && n > 128);
  if (subspace) {
    Eig e;
    if (run_eigh_subspace(ctx, gram, n, ratio, certify, e)) return e;
  }
  return run_eigh(ctx, gram, n, ratio);
}

// ---------------------------------------------------------------- K2 batched
// Multislice (sk_estimate_maps_batched): the subspace solver of
// run_eigh_subspace run in lockstep over `batch` slices of one Gram size, so
// that its small latency-bound kernels (CholQR, Ritz eigensolver) run one CTA
// set per slice side by side instead of one slice at a time: strided-batched
// 3xTF32 / ZGEMM products, gram64 / chol64 / trsm64 and the Ritz eigensolver
// with the slice on the grid's batch axis.  Same start block, step plan and
// convergence test per slice as the single-slice solver (the plan is the
// shared per-size hint).  Slices that do not pass the test in the planned
// round are reported in ok[] = 0 for the caller's single-slice fallback.
// Buffers live in arena slots suffixed by `set` (two sets alternate, so a
// batch's signal bases stay valid while the next batch is solved).
void run_eigh_subspace_batched(sk_ctx* ctx, const float2* grams, i64 batch, i64 n, double ratio, int set,
                               std::vector<Eig>& eigs, std::vector<char>& ok) {
  PhaseLaps laps(ctx);
  const std::string sfx = ":" + std::to_string(set);
  constexpr i64 b = 64;  // the batched CholQR kernels (sk_cholqr.cu) are b = 64, n >= 1024
  const i64 nn = n * n, nb = n * b;
  auto& hint = ctx->subspace_hint;
  int q_plan = 3;
  auto it_h = hint.find(n);
  if (it_h != hint.end()) q_plan = it_h->second.plan;
  // FP64 products in the Gauss 3M form on real planes [Re A][Im A][Re A + Im A]
  // (one strided-batched DGEMM over 3 x batch matrices per product; the
  // strided-batched ZGEMM it replaces ran four real products' worth)
  double* A3 = ctx->arena.get<double>("bk:A3" + sfx, batch * 3 * nn);
  double* V3 = ctx->arena.get<double>("bk:V3" + sfx, batch * 3 * nb);
  double* T3 = ctx->arena.get<double>("bk:T3" + sfx, batch * 3 * nb);
  float* gcat = ctx->arena.get<float>("bk:gcat" + sfx, batch * 4 * nn);
  promote_split3_gram(ctx, grams, n, A3, gcat, gcat + 2 * nn, batch, nn, 4 * nn);
  laps.lap("promote");
  double2* V = ctx->arena.get<double2>("bk:V" + sfx, batch * nb);
  double2* Y = ctx->arena.get<double2>("bk:Y" + sfx, batch * nb);
  double2* T = ctx->arena.get<double2>("bk:T" + sfx, batch * nb);
  double2* H = ctx->arena.get<double2>("bk:H" + sfx, batch * b * b);
  double* w = ctx->arena.get<double>("bk:w" + sfx, batch * b);
  double* res = ctx->arena.get<double>("bk:res" + sfx, batch * b);
  int* info = ctx->arena.get<int>("bk:info" + sfx, batch * 3);
  float* vcat = ctx->arena.get<float>("bk:vcat" + sfx, batch * 8 * nb);
  float* ccat = ctx->arena.get<float>("bk:ccat" + sfx, batch * 8 * nb);
  SKB_CUDA(cudaMemsetAsync(info, 0, size_t(batch) * 3 * sizeof(int), ctx->stream));
  random_block(ctx, V, n, b, 0, 0x5eed5u, batch, nb);
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  auto zgemm_b = [&](i64 m, i64 nc, i64 k, const double2* a, i64 lda, i64 sa, const double2* bm, i64 ldb, i64 sbm,
                     double2* c, i64 ldc, i64 sc) {
    check_cublas(cublasZgemmStridedBatched(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, int(m), int(nc), int(k), &one,
                                           reinterpret_cast<const cuDoubleComplex*>(a), int(lda), sa,
                                           reinterpret_cast<const cuDoubleComplex*>(bm), int(ldb), sbm, &zero,
                                           reinterpret_cast<cuDoubleComplex*>(c), int(ldc), sc, int(batch)),
                 "ZgemmStridedBatched");
    ++ctx->lib_calls;
  };
  auto product64 = [&](const double2* v, double2* y) {  // y = A v for every slice
    const double d1 = 1.0, d0 = 0.0;
    split3_block(ctx, v, nb, V3, batch, nb);
    check_cublas(cublasDgemmStridedBatched(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, int(n), int(b), int(n), &d1, A3,
                                           int(n), nn, V3, int(n), nb, &d0, T3, int(n), nb, int(3 * batch)),
                 "DgemmStridedBatched(3M)");
    ++ctx->lib_calls;
    combine3_block(ctx, T3, nb, y, batch, nb);
  };
  bool have_split = false;
  for (int i = 0; i < q_plan; ++i) {
    CatIO io;
    if (i + kFp64StepsBatched < q_plan) {  // 3xTF32 steering step over the K-concatenated split Gram
      const float f1 = 1.f, f0 = 0.f;
      if (!have_split) split_block_cat_tf32(ctx, V, n, b, vcat, batch, nb, 8 * nb);
      check_cublas(cublasGemmStridedBatchedEx(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, int(2 * n), int(4 * b),
                                              int(2 * n), &f1, gcat, CUDA_R_32F, int(2 * n), 4 * nn, vcat, CUDA_R_32F,
                                              int(2 * n), 8 * nb, &f0, ccat, CUDA_R_32F, int(2 * n), 8 * nb,
                                              int(batch), CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT),
                   "GemmStridedBatchedEx(3xTF32 cat)");
      ++ctx->lib_calls;
      // the CholQR kernels read the concatenated product and write the next split operand (CatIO)
      io.ccat = ccat;
      io.sc = 8 * nb;
      have_split = (i + 1) + kFp64StepsBatched < q_plan;
      if (have_split) {
        io.vcat = vcat;
        io.svc = 8 * nb;
      }
      laps.lap("gemm32");
    } else {
      product64(V, Y);  // Y = A V (FP64)
      laps.lap("gemm64");
    }
    std::swap(V, Y);
    cholqr64(ctx, V, n, i + 1 == q_plan ? 2 : 1, info + 1, batch, nb, io);
    laps.lap("orth");
  }
  product64(V, Y);
  laps.lap("gemm64");
  gram64(ctx, V, Y, n, H, batch, nb);  // H = V^H A V
  laps.lap("rr_gram");
  herm_eig_small(ctx, H, int(b), w, info, 0.25 * ratio * ratio, int(batch));
  laps.lap("rr_heev");
  zgemm_b(n, b, b, V, n, nb, H, b, b * b, T, n, nb);  // V <- V S
  std::swap(V, T);
  zgemm_b(n, b, b, Y, n, nb, H, b, b * b, T, n, nb);  // Y <- Y S
  std::swap(Y, T);
  ritz_residuals(ctx, Y, V, w, n, b, res, batch, nb, b);
  laps.lap("rr_rotate");
  std::vector<double> hw(size_t(batch * b)), hres(size_t(batch * b));
  std::vector<int> hinfo(size_t(batch * 3));
  SKB_CUDA(cudaMemcpyAsync(hw.data(), w, hw.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SKB_CUDA(cudaMemcpyAsync(hres.data(), res, hres.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SKB_CUDA(cudaMemcpyAsync(hinfo.data(), info, hinfo.size() * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  const double tol = 3e-10;  // run_eigh_subspace's test
  const i64 guard = 8;
  eigs.assign(size_t(batch), Eig());
  ok.assign(size_t(batch), 0);
  int spare_min = 3, failed = 0;
  for (i64 sl = 0; sl < batch; ++sl) {
    const double* ws = hw.data() + sl * b;
    const double* rs = hres.data() + sl * b;
    if (hinfo[size_t(3 * sl)] || hinfo[size_t(3 * sl + 1)] || hinfo[size_t(3 * sl + 2)]) {
      ++failed;
      continue;
    }
    const double theta_max = ws[b - 1];
    if (!(theta_max > 0.0)) {
      ++failed;
      continue;
    }
    const double c = ratio * ratio * theta_max;
    i64 m = 0;
    for (i64 i = 0; i < b; ++i) m += ws[i] >= c ? 1 : 0;
    double worst = 0.0, rate = 0.0;
    const bool reaches = ws[0] < 0.5 * c;
    for (i64 i = 0; i < b; ++i) {
      if (ws[i] < 0.5 * c) continue;
      worst = std::max(worst, std::sqrt(std::max(rs[i], 0.0)) / theta_max);
      rate = std::max(rate, std::max(ws[0], 0.0) / ws[i]);
    }
    if (m > b - guard || !reaches || worst > tol || m == 0 || m == n) {
      ++failed;
      continue;
    }
    int spare = 0;
    if (rate > 0.0 && rate < 1.0 && worst > 0.0)
      spare = std::max(0, int(std::floor(std::log(0.8 * tol / worst) / std::log(1.0 / rate))));
    spare_min = std::min(spare_min, spare);
    Eig& e = eigs[size_t(sl)];
    e.n = n;
    e.full = false;
    e.k = m;
    e.rank = n - m;
    e.usig = V + sl * nb + (b - m) * n;  // the last m Ritz columns (ascending theta)
    e.sigma1 = std::sqrt(theta_max);
    e.cut = ratio * e.sigma1;
    e.iterations = q_plan + 1;
    e.block = int(b);
    e.spectrum.assign(size_t(n), 0.0);
    for (i64 i = 0; i < b; ++i) e.spectrum[size_t(i)] = std::sqrt(std::max(0.0, ws[b - 1 - i]));
    ok[size_t(sl)] = 1;
  }
  // plan for the next batch of this size: one step more after any failure
  // (never planned again at the failing size), else the spare steps every
  // slice showed, at most one per batch
  auto& h = hint[n];
  if (failed) {
    h.failed_plan = std::max(h.failed_plan, q_plan);
    h.plan = q_plan + 1;
  } else if (spare_min > 0 && q_plan > 3 && q_plan - 1 > h.failed_plan) {
    h.plan = q_plan - 1;
  } else {
    h.plan = q_plan;
  }
}

// ---------------------------------------------------------------- K3
// Lag kernels from the signal subspace, expanded onto the grid as packed planes.
Planes run_field(sk_ctx* ctx, const Eig& e, const Support& s, int q, const Dims& grid, i64 slab0 = 0,
                 i64 slab1 = -1) {
  const i64 n = e.n, k = e.k;
  const int lam = int(s.count);
  SupportTables& t = tables_for(ctx, s, q);
  const int h = q * (q + 1) / 2;
  double2* lags = ctx->arena.get<double2>("field:lags64", i64(h) * t.nbox);
  // aggregate_w + fold (spatial_gram.cpp:87-94, 108-131): W = I - U_sig U_sig^H
  // folded onto the lag box by the correlation theorem (sk_fold.cu), own FP64
  // kernels, no n x n buffer (C2 field 0.282 -> 0.239 ms against cuBLAS ZHERK +
  // CSR fold, C5 3.59 -> 3.20 ms).  Lag boxes too large for its shared-memory
  // buffers (3-D with tau > 4; no BASELINE config) keep the ZHERK path.
  auto planes_for = [&]() {
    Planes p;
    const i64 nvox = slab1 >= 0 ? numel(grid) / grid[0] * (slab1 - slab0) : numel(grid);
    p.hi = ctx->arena.get<float2>("field:planes", i64(h) * nvox);
    p.lo = ctx->arena.get<lo2>("field:planes_lo", i64(h) * nvox);
    expand_lags(ctx, lags, p.hi, p.lo, h, s.tau, grid, slab0, slab1);
    return p;
  };
  if (spectral_fold_smem(s.nd, s.tau, int(k), q) <= 200 * 1024) {
    fold_lags_spectral(ctx, e.usig, n, int(k), q, lam, s.nd, s.tau, support_offsets_dev(ctx, s), lags);
    return planes_for();
  }
  double2* ws = ctx->arena.get<double2>("field:Ws", n * n);
  if (k > 0) {
    const double one = 1.0, zero = 0.0;
    check_cublas(cublasZherk(ctx->cublas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, int(n), int(k), &one,
                             reinterpret_cast<const cuDoubleComplex*>(e.usig), int(n), &zero,
                             reinterpret_cast<cuDoubleComplex*>(ws), int(n)),
                 "Zherk");
    ++ctx->lib_calls;
  } else {
    SKB_CUDA(cudaMemsetAsync(ws, 0, size_t(n * n) * sizeof(double2), ctx->stream));
  }
  fold_lags_f64(ctx, ws, n, h, lam, t.nbox, t.pairs, t.lag_ptr, t.lag_st, true, lags);
  return planes_for();
}

// Lag kernels from a caller-supplied W (gram_field_fast entry point).
Planes run_field_from_w(sk_ctx* ctx, const float2* w, const Support& s, int q, const Dims& grid) {
  const i64 n = i64(q) * s.count;
  SupportTables& t = tables_for(ctx, s, q);
  const int h = q * (q + 1) / 2;
  double2* lags = ctx->arena.get<double2>("field:lags64", i64(h) * t.nbox);
  fold_lags_f32(ctx, w, n, h, int(s.count), t.nbox, t.pairs, t.lag_ptr, t.lag_st, lags);
  Planes p;
  p.hi = ctx->arena.get<float2>("field:planes", i64(h) * numel(grid));
  p.lo = ctx->arena.get<lo2>("field:planes_lo", i64(h) * numel(grid));
  expand_lags(ctx, lags, p.hi, p.lo, h, s.tau, grid);
  return p;
}

// ---------------------------------------------------------------- K5 pieces
float2* run_recon(sk_ctx* ctx, const Dims& cdims, const Dims& co, i64 q, const float2* calib, const Dims& grid,
                  double apod_width, i64 slab0 = 0, i64 slab1 = -1) {  // maps.cpp:130-160
  const int nd = int(cdims.size());
  std::vector<float2*> mats(static_cast<size_t>(nd));
  for (int a = 0; a < nd; ++a) {
    const double sigma = apod_width > 0 ? apod_width : double(cdims[size_t(a)]) / 4.0;
    mats[size_t(a)] = dft_matrix(ctx, int(grid[size_t(a)]), int(cdims[size_t(a)]), co[size_t(a)],
                                 center_index(grid[size_t(a)]), +1, sigma);
  }
  Dims out_grid = grid;
  if (slab1 >= 0) {  // axis-0 rows [slab0, slab1): the row-major N x L matrix offset by slab0 rows
    mats[0] += slab0 * cdims[0];
    out_grid[0] = slab1 - slab0;
  }
  float2* recon = ctx->arena.get<float2>("post:recon", q * numel(out_grid));
  separable(ctx, calib, recon, q, cdims, out_grid, mats, "post:tmp");
  return recon;
}

// Interpolation, one axis at a time (last first): radix-2 FFT kernel for
// power-of-two extents (sk_interp.cu), the exact per-axis sinc matrix
// otherwise.  fp64 selects double2 elements (FFT path only).
bool interp_fft_ok(const Dims& low, const Dims& full) {
  for (size_t a = 0; a < low.size(); ++a) {
    const i64 n = low[a], N = full[a];
    if (n < 2 || N > 1024 || (n & (n - 1)) || (N & (N - 1)) || n > N) return false;
  }
  return true;
}

// Maps interpolation followed by the SoS renormalisation of finalize
// (maps.cpp:236-250).  When the innermost axis doubles and Q fits the fused
// kernel, the outer axes run first and the innermost pass renormalises in
// the same kernel; returns false when the caller still has to renormalise.
// slices > 1: a stack [slices][Q][low] -> [slices][Q][full] (multislice groups).
bool run_interp_renorm(sk_ctx* ctx, const float2* low, float2* out, i64 q, const Dims& low_dims, const Dims& full,
                       i64 slices = 1) {
  const int nd = int(low_dims.size());
  const int n = int(low_dims[size_t(nd - 1)]), N = int(full[size_t(nd - 1)]);
  if (!interp_fft_ok(low_dims, full) || N != 2 * n || q > 32 || (q & (q - 1)) || q * n > 4096) return false;
  Dims cur = low_dims;
  const float2* src = low;
  int pass = 0;
  for (int a = 0; a < nd - 1; ++a) {
    if (low_dims[size_t(a)] == full[size_t(a)]) continue;
    Dims next = cur;
    next[size_t(a)] = full[size_t(a)];
    float2* dst = ctx->arena.get<float2>(std::string("interp:fft") + (pass++ % 2 ? ":b" : ":a"),
                                         slices * q * numel(next));
    i64 b = slices * q, inner = 1;
    for (int k = 0; k < a; ++k) b *= cur[size_t(k)];
    for (int k = a + 1; k < nd; ++k) inner *= cur[size_t(k)];
    if (!interp_axis_fft(ctx, src, dst, b, int(low_dims[size_t(a)]), int(full[size_t(a)]), inner, false))
      fail(SK_ERR_UNSUPPORTED, "interpolate_maps: FFT path refused a planned axis");
    cur[size_t(a)] = full[size_t(a)];
    src = dst;
  }
  const i64 positions = numel(cur) / cur[size_t(nd - 1)];
  if (!interp_last_axis_sos(ctx, src, out, int(q), positions, n, N, int(slices)))
    fail(SK_ERR_UNSUPPORTED, "interpolate_maps: fused last pass refused its shape");
  return true;
}

void run_interp(sk_ctx* ctx, const float2* low, float2* out, i64 batch, const Dims& low_dims, const Dims& full) {
  const int nd = int(low_dims.size());
  if (interp_fft_ok(low_dims, full)) {
    Dims cur = low_dims;
    const float2* src = low;
    for (int a = nd - 1; a >= 0; --a) {
      float2* dst = out;
      if (a > 0) {
        Dims next = cur;
        next[size_t(a)] = full[size_t(a)];
        dst = ctx->arena.get<float2>(std::string("interp:fft") + (a % 2 ? ":a" : ":b"), batch * numel(next));
      }
      i64 b = batch, inner = 1;
      for (int k = 0; k < a; ++k) b *= cur[size_t(k)];
      for (int k = a + 1; k < nd; ++k) inner *= cur[size_t(k)];
      if (!interp_axis_fft(ctx, src, dst, b, int(low_dims[size_t(a)]), int(full[size_t(a)]), inner, false))
        fail(SK_ERR_UNSUPPORTED, "interpolate_maps: FFT path refused a planned axis");
      cur[size_t(a)] = full[size_t(a)];
      src = dst;
    }
    return;
  }
  std::vector<float2*> mats(static_cast<size_t>(nd));
  for (int a = 0; a < nd; ++a) mats[size_t(a)] = sinc_matrix(ctx, int(full[size_t(a)]), int(low_dims[size_t(a)]));
  separable(ctx, low, out, batch, low_dims, full, mats, "interp:tmp");
}

// interpolate_real (maps.cpp:92-99) + support mask (maps.cpp:47-52): FP64
// FFT path for power-of-two extents, the FP32 sinc-matrix path otherwise.
// batch > 1 (FFT path only): a stack of [batch] maps.
void run_interp_lambda(sk_ctx* ctx, const float* low, const Dims& low_dims, const Dims& full, float* lam_out,
                       uint8_t* mask, float thr, i64 batch = 1) {
  const int nd = int(low_dims.size());
  const i64 nlow = numel(low_dims), nfull = numel(full);
  if (interp_fft_ok(low_dims, full)) {
    double2* src = ctx->arena.get<double2>("interp:lam64", batch * nlow);
    real_to_c128(ctx, low, src, batch * nlow);
    Dims cur = low_dims;
    for (int a = nd - 1; a >= 0; --a) {
      Dims next = cur;
      next[size_t(a)] = full[size_t(a)];
      double2* dst = ctx->arena.get<double2>(std::string("interp:lam64") + (a % 2 ? ":a" : ":b"),
                                             batch * numel(next));
      i64 b = batch, inner = 1;
      for (int k = 0; k < a; ++k) b *= cur[size_t(k)];
      for (int k = a + 1; k < nd; ++k) inner *= cur[size_t(k)];
      if (!interp_axis_fft(ctx, src, dst, b, int(low_dims[size_t(a)]), int(full[size_t(a)]), inner, true))
        fail(SK_ERR_UNSUPPORTED, "interpolate_real: FFT path refused a planned axis");
      cur = next;
      src = dst;
    }
    lam64_to_f32_mask(ctx, src, batch * nfull, lam_out, mask, thr);
    return;
  }
  if (batch != 1) fail(SK_ERR_UNSUPPORTED, "interpolate_real: stacks need the FFT path");
  float2* lam_c = ctx->arena.get<float2>("post:lam_c", nlow);
  real_to_c64(ctx, low, lam_c, nlow);
  float2* lam_full_c = ctx->arena.get<float2>("post:lam_full_c", nfull);
  run_interp(ctx, lam_c, lam_full_c, 1, low_dims, full);
  renormalize_and_mask(ctx, nullptr, nfull, 0, lam_full_c, lam_out, mask, thr);
}

// ---------------------------------------------------------------- pipeline
struct PipelineOut {
  float2* maps = nullptr;     // device [Q][N_full] (nullable)
  float* lambda = nullptr;    // device [N_full]
  uint8_t* mask = nullptr;    // device [N_full]
  float2* gram = nullptr;     // debug: device n x n
  float2* field = nullptr;    // debug: device GramField layout (grid)
  float2* raw_maps = nullptr; // debug: device [Q][N_grid]
  float* raw_lambda = nullptr;
  double* spectrum = nullptr; // host n
  // pinned host destination of `maps` (full-resolution power grid): K4 runs in
  // voxel chunks and each chunk's maps go to the host on a copy stream while
  // the next chunk computes
  float2* maps_host = nullptr;
  // z-slab mode (sk_estimate_raw_slab): axis-0 grid rows [slab0, slab1); the
  // normalised maps / raw lambda of those rows go to maps / lambda and the
  // interpolation stage is skipped.
  i64 slab0 = 0, slab1 = -1;
  // parity probe (sk_estimate_maps_probe): device index lists in, FP64 samples out
  struct Probe {
    i64 n_gram = 0, n_field = 0;
    const long long* gram_idx = nullptr;   // device, (row, col) pairs
    const long long* field_idx = nullptr;  // device, (voxel, row, col) triples
    double2* gram_vals = nullptr;          // device
    double2* field_vals = nullptr;         // device
    double gram_sumsq = 0.0, field_sumsq = 0.0;
    float* raw_lambda = nullptr;           // device, N_grid
  }* probe = nullptr;
  // Precomputed signal basis (z-slab ranks after the rank-0 broadcast,
  // sk_estimate_raw_slab_basis): K1 and K2 are skipped.
  struct Basis {
    const double2* usig = nullptr;  // device, n x k
    i64 k = 0;
    double sigma1 = 0.0;
  }* basis = nullptr;
  // K1 + K2 only (sk_signal_basis): stop after the nullspace, hand the Eig out.
  Eig* eig_out = nullptr;
};

// K4 epilogue: voxels with lambda >= this keep the FP32 Rayleigh quotient
// (||G/|Lambda| || <= 1 for W a projection, so FP32 rounding is ~1e-7 absolute,
// < 1e-5 relative above 0.25).  Used on full-resolution map grids only (see
// the pipeline).
constexpr float kRq32Min = 0.25f;

void validate_config(const sk_config* cfg) {
  if (!cfg) fail(SK_ERR_DIM, "null config");
  if (cfg->gram != 0 && cfg->gram != 1) fail(SK_ERR_DIM, "unknown gram method");
  if (cfg->eig != 0 && cfg->eig != 1) fail(SK_ERR_DIM, "unknown eig method");
  if (cfg->method != 0 && cfg->method != 1) fail(SK_ERR_DIM, "unknown map method");
  if (cfg->field != 0 && cfg->field != 1) fail(SK_ERR_DIM, "unknown field path");
  if (cfg->kernel != 0 && cfg->kernel != 1) fail(SK_ERR_DIM, "unknown kernel shape");
  if (cfg->power_iters < 0) fail(SK_ERR_DIM, "power_iters must be >= 0");
}

void pipeline(sk_ctx* ctx, const Dims& cdims, const Dims& co, i64 q, const float2* calib, const Dims& full,
              const sk_config* cfg, PipelineOut& out, sk_provenance* prov) {
  validate_config(cfg);
  const int nd = int(cdims.size());
  if (full.size() != cdims.size()) fail(SK_ERR_DIM, "full_dims rank mismatch");  // maps.cpp:267-271
  for (int a = 0; a < nd; ++a)
    if (full[size_t(a)] < cdims[size_t(a)]) fail(SK_ERR_DIM, "full_dims must be at least the calibration extent");
  const Support s = make_support(cfg->kernel, cfg->tau, nd);
  check_calib(cdims, q, s);
  if (q > power_wide_max_q())
    fail(SK_ERR_UNSUPPORTED, "more than " + std::to_string(power_wide_max_q()) + " channels is outside the B200 path");
  // grid_dims_for (maps.cpp:188-193) or the explicit grid.
  Dims grid(static_cast<size_t>(nd));
  bool explicit_grid = true;
  for (int a = 0; a < nd; ++a) explicit_grid = explicit_grid && cfg->grid_dims[a] > 0;
  for (int a = 0; a < nd; ++a) {
    if (explicit_grid)
      grid[size_t(a)] = cfg->grid_dims[a];
    else if (cfg->grid == 1)
      grid[size_t(a)] = std::min(cdims[size_t(a)] + cfg->grid_pad, full[size_t(a)]);
    else
      grid[size_t(a)] = full[size_t(a)];
  }
  for (int a = 0; a < nd; ++a) {
    if (grid[size_t(a)] < cdims[size_t(a)]) fail(SK_ERR_DIM, "map grid smaller than calibration region");
    if (full[size_t(a)] < grid[size_t(a)])
      fail(SK_ERR_DIM, "interpolation target smaller than source on axis " + std::to_string(a));
  }
  const bool slab = out.slab1 >= 0;
  if (slab && (out.slab0 < 0 || out.slab1 <= out.slab0 || out.slab1 > grid[0]))
    fail(SK_ERR_DIM, "slab rows must satisfy 0 <= begin < end <= grid_dims[0]");
  const i64 lam = s.count, n = q * lam, nfull = numel(full);
  const i64 ngrid = slab ? numel(grid) / grid[0] * (out.slab1 - out.slab0) : numel(grid);  // voxels computed here
  const bool interp = !slab && grid != full;

  cudaEvent_t* ev = ctx->ev;
  SKB_CUDA(cudaEventRecord(ev[0], ctx->stream));
  // gram
  // compute_gram (maps.cpp:180-186)
  Eig e;
  if (out.basis) {
    SKB_CUDA(cudaEventRecord(ev[1], ctx->stream));
    e.n = n;
    e.k = out.basis->k;
    e.rank = n - e.k;
    e.usig = out.basis->usig;
    e.sigma1 = out.basis->sigma1;
    e.cut = cfg->nullspace_threshold * e.sigma1;
    e.full = false;
  } else {
    float2* gram = cfg->gram == 0 ? run_gram_explicit(ctx, cdims, q, calib, s, out.gram)
                                  : run_gram(ctx, cdims, q, calib, s, out.gram);
    if (out.probe) {
      probe_gather_gram(ctx, gram, q * s.count, out.probe->gram_idx, out.probe->n_gram, out.probe->gram_vals);
      out.probe->gram_sumsq = probe_sumsq(ctx, gram, nullptr, q * s.count * q * s.count, 0, 0);
    }
    SKB_CUDA(cudaEventRecord(ev[1], ctx->stream));
    // nullspace
    e = run_nullspace(ctx, gram, n, cfg->nullspace_threshold, cfg->eig_solver, out.spectrum != nullptr,
                      cfg->certify != 0);
  }
  SKB_CUDA(cudaEventRecord(ev[2], ctx->stream));
  if (out.eig_out) {
    *out.eig_out = e;
    return;
  }
  // field.  compute_field (maps.cpp:195-205): the naive path materialises the
  // R x Q x N filter field H (spatial_gram.cpp:36-64) and sums H^H H per voxel;
  // that is the same G(x) as the lag expansion of W = F F^H, so both paths
  // run the expansion, with the naive path's byte-cap contract kept.
  if (cfg->field == 0) {
    const i64 cap = cfg->field_byte_cap > 0 ? cfg->field_byte_cap : (i64(1) << 30);
    const double need = double(e.rank) * double(q) * double(numel(grid)) * 16.0;  // spatial_gram.cpp:43
    if (need > double(cap))
      fail(SK_ERR_LENGTH, "filter field would need " + std::to_string(i64(need)) + " bytes (cap " +
                              std::to_string(cap) + ")");
  }
  const Planes pl = run_field(ctx, e, s, int(q), grid, out.slab0, out.slab1);
  float2* planes = pl.hi;
  if (out.field) planes_to_field_full(ctx, pl.hi, pl.lo, ngrid, int(q), out.field);
  if (out.probe) {
    probe_gather_field(ctx, pl.hi, pl.lo, ngrid, int(q), out.probe->field_idx, out.probe->n_field,
                       out.probe->field_vals);
    out.probe->field_sumsq = probe_sumsq(ctx, pl.hi, pl.lo, i64(q * (q + 1) / 2) * ngrid, ngrid, int(q));
  }
  SKB_CUDA(cudaEventRecord(ev[3], ctx->stream));
  // post (part 1): apodised recon on the map grid, consumed by K4's epilogue
  float2* recon = run_recon(ctx, cdims, co, q, calib, grid, cfg->apod_width, out.slab0, out.slab1);
  SKB_CUDA(cudaEventRecord(ev[4], ctx->stream));
  // eigensolve (+ fused normalisation)
  unsigned long long* zeroed = ctx->arena.get<unsigned long long>("post:zeroed", 1);
  SKB_CUDA(cudaMemsetAsync(zeroed, 0, sizeof(unsigned long long), ctx->stream));
  float2* maps_grid = (!interp && out.maps) ? out.maps : ctx->arena.get<float2>("post:maps_grid", q * ngrid);
  float* lam_grid = (!interp && out.lambda) ? out.lambda : ctx->arena.get<float>("post:lam_grid", ngrid);
  if (cfg->eig == 0) {
    // solve_field, dense arm (maps.cpp:207-218): nullspace method -> smallest
    // eigenpair of G, lambda = value / |Lambda|; ESPIRiT -> largest eigenpair
    // of B = I - G/|Lambda|, lambda = 1 - value.  Then normalize_maps.
    const bool nullspace = cfg->method == 0;
    DenseEigArgs d{};
    d.planes = planes;
    d.planes_lo = pl.lo;
    d.n = ngrid;
    d.q = int(q);
    d.largest = nullspace ? 0 : 1;
    d.alpha = nullspace ? 0.0 : 1.0;
    d.beta = nullspace ? 1.0 : -1.0 / double(lam);
    d.lam_add = nullspace ? 0.0 : 1.0;
    d.lam_mul = nullspace ? 1.0 / double(lam) : -1.0;
    d.vec = out.raw_maps ? out.raw_maps : maps_grid;
    d.lambda = lam_grid;
    d.mask = (!interp && !slab && out.mask) ? out.mask : nullptr;
    d.mask_threshold = float(cfg->mask_threshold);
    dense_eig(ctx, d);
    if (out.raw_maps) {
      if (out.raw_lambda)
        SKB_CUDA(cudaMemcpyAsync(out.raw_lambda, lam_grid, size_t(ngrid) * sizeof(float), cudaMemcpyDeviceToDevice,
                                 ctx->stream));
      SKB_CUDA(cudaMemcpyAsync(maps_grid, out.raw_maps, size_t(q * ngrid) * sizeof(float2), cudaMemcpyDeviceToDevice,
                               ctx->stream));
    }
    normalize_standalone(ctx, maps_grid, ngrid, int(q), recon, zeroed);
  } else {
  if (out.raw_maps) {
    // raw (pre-normalisation) eigenvectors for parity dumps: run K4 without the epilogue first
    PowerArgs r{};
    r.planes = planes; r.planes_lo = pl.lo; r.n = ngrid; r.q = int(q); r.iters = cfg->power_iters;
    r.alpha = 1.f; r.beta = -1.f / float(lam); r.lam_scale = 1.f / float(lam);
    r.maps = out.raw_maps; r.lambda = out.raw_lambda;
    r.rq32_min = grid != full ? 0.f : kRq32Min;
    power_iteration(ctx, r);
  }
  PowerArgs pa{};
  pa.planes = planes;
  pa.planes_lo = pl.lo;
  pa.n = ngrid;
  pa.q = int(q);
  pa.iters = cfg->power_iters;
  pa.alpha = 1.f;                    // B = I - G/|Lambda|
  pa.beta = -1.f / float(lam);
  pa.lam_scale = 1.f / float(lam);   // lambda = v^H G v / |Lambda| = 1 - v^H B v
  pa.recon = recon;
  pa.maps = maps_grid;
  pa.lambda = lam_grid;
  pa.mask = (!interp && !slab && out.mask) ? out.mask : nullptr;
  pa.mask_threshold = float(cfg->mask_threshold);
  pa.zeroed = zeroed;
  // Not when an interpolation follows: the periodic-sinc interpolation spreads
  // the FP32 path's ~1e-7 absolute error of large-lambda voxels into the small
  // in-support values (measured: C3 in-mask lambda 3.4e-5 -> 5.6e-5 relative).
  pa.rq32_min = grid != full ? 0.f : kRq32Min;  // slabs are interpolated by the caller
  if (out.maps_host && !interp && !slab && maps_grid == out.maps) {
    // K4 in voxel chunks (multiples of 8 voxels: 16-byte aligned TMA bases)
    // with the maps copied to the host behind each chunk on a second stream.
    static const int kChunks = [] {
      const char* v = std::getenv("SKB_K4_CHUNKS");
      return v ? std::max(1, std::min(8, std::atoi(v))) : 4;
    }();
    if (!ctx->copy_stream) {
      SKB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      for (auto& e : ctx->chunk_ev) SKB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // decreasing chunk sizes (weights k, k-1, .., 1): the copy of the last
    // chunk, which nothing overlaps, is the smallest
    const i64 wsum = i64(kChunks) * (kChunks + 1) / 2;
    int c = 0;
    for (i64 jb = 0; jb < ngrid; ++c) {
      const i64 want = c + 1 >= kChunks ? ngrid - jb : (ngrid * (kChunks - c) / wsum + 7) / 8 * 8;
      const i64 cnt = std::min(std::max<i64>(want, 8), ngrid - jb);
      PowerArgs ca = pa;
      ca.planes = pa.planes + jb;
      ca.planes_lo = pa.planes_lo ? pa.planes_lo + jb : nullptr;
      ca.recon = pa.recon ? pa.recon + jb : nullptr;
      ca.maps = pa.maps + jb;
      ca.lambda = pa.lambda ? pa.lambda + jb : nullptr;
      ca.mask = pa.mask ? pa.mask + jb : nullptr;
      ca.n = cnt;
      ca.ld = ngrid;
      power_iteration(ctx, ca);
      SKB_CUDA(cudaEventRecord(ctx->chunk_ev[c], ctx->stream));
      SKB_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->chunk_ev[c], 0));
      SKB_CUDA(cudaMemcpy2DAsync(out.maps_host + jb, size_t(ngrid) * sizeof(float2), maps_grid + jb,
                                 size_t(ngrid) * sizeof(float2), size_t(cnt) * sizeof(float2), size_t(q),
                                 cudaMemcpyDeviceToHost, ctx->copy_stream));
      jb += cnt;
    }
    SKB_CUDA(cudaEventRecord(ctx->chunk_ev[8], ctx->copy_stream));
    SKB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->chunk_ev[8], 0));
  } else {
    power_iteration(ctx, pa);
  }
  }
  if (out.probe && out.probe->raw_lambda)
    SKB_CUDA(cudaMemcpyAsync(out.probe->raw_lambda, lam_grid, size_t(ngrid) * sizeof(float), cudaMemcpyDeviceToDevice,
                             ctx->stream));
  SKB_CUDA(cudaEventRecord(ev[5], ctx->stream));
  // post (part 2): interpolation + renormalisation + mask (maps.cpp:236-258)
  if (interp) {
    float2* maps_full = out.maps ? out.maps : ctx->arena.get<float2>("post:maps_full", q * nfull);
    const bool renormed = run_interp_renorm(ctx, maps_grid, maps_full, q, grid, full);
    if (!renormed) run_interp(ctx, maps_grid, maps_full, q, grid, full);
    run_interp_lambda(ctx, lam_grid, grid, full, out.lambda, out.mask, float(cfg->mask_threshold));
    if (!renormed) renormalize_and_mask(ctx, maps_full, nfull, int(q), nullptr, nullptr, nullptr, 0.f);
  }
  SKB_CUDA(cudaEventRecord(ev[6], ctx->stream));
  // the zeroed-voxel count through the context's pinned staging (a pageable
  // destination makes the copy a slower synchronous one)
  if (ctx->hpin_cap < 1) {
    SKB_CUDA(cudaMallocHost(&ctx->hpin, 64 * sizeof(double)));
    ctx->hpin_cap = 64;
  }
  SKB_CUDA(cudaMemcpyAsync(ctx->hpin, zeroed, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  unsigned long long h_zeroed = 0;
  std::memcpy(&h_zeroed, ctx->hpin, sizeof h_zeroed);
  if (out.spectrum)
    for (i64 i = 0; i < n; ++i) out.spectrum[i] = e.sigma1 > 0 ? e.spectrum[size_t(i)] / e.sigma1 : 0.0;
  if (prov) {
    float ms[6];
    for (int i = 0; i < 6; ++i) SKB_CUDA(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
    std::memset(prov, 0, sizeof *prov);
    for (int a = 0; a < nd; ++a) prov->grid_dims[a] = grid[size_t(a)];
    prov->support_size = lam;
    prov->valid_shifts = 1;
    for (i64 d : cdims) prov->valid_shifts *= std::max<i64>(0, d - 2 * cfg->tau);
    prov->nullspace_rank = e.rank;
    prov->zeroed_voxels = i64(h_zeroed);
    prov->sigma1 = e.sigma1;
    prov->cut_margin = e.margin;
    prov->eig_solver_used = e.full ? 1 : 2;
    prov->certified = e.certified ? 1 : 0;
    prov->subspace_iterations = e.iterations;
    prov->subspace_block = e.block;
    prov->stage_ms[0] = ms[0];
    prov->stage_ms[1] = ms[1];
    prov->stage_ms[2] = ms[2];
    prov->stage_ms[3] = ms[4];
    prov->stage_ms[4] = ms[3] + ms[5];
    float total = 0;
    SKB_CUDA(cudaEventElapsedTime(&total, ev[0], ev[6]));
    prov->total_ms = total;
  }
}


// ---------------------------------------------------------------- multislice group tail
// K3-K5 of a whole group of slices in one pass (sk_estimate_maps_batched with
// the batched K2): the per-slice kernels of a 128 x 128 map grid are too small
// to fill the GPU (C3: 15-40 us each, launch- and tail-bound even with twelve
// concurrent lanes), so the group runs them with the slice as a batch axis:
// the spectral fold with the slice on grid.y, the lag expansion over
// slices x pairs, the recon over slices x channels, K4 over a stack of slices
// (PowerArgs::slices), the interpolation passes over slices x channels and
// the FP64 lambda interpolation over slices.  Arithmetic per slice is exactly
// the single-slice pipeline's (same kernels, same order).
// Eligible: power-iteration eigensolver, a reduced map grid whose
// interpolation takes the FFT path with the fused SoS pass, a lag box that
// fits the spectral fold.  grid: the map grid (out).
bool group_tail_eligible(const sk_config* cfg, const Dims& cd, const Dims& fd, i64 q, const Support& s, Dims& grid) {
  const int nd = int(cd.size());
  if (!cfg || cfg->eig != 1 || cfg->field != 1 || q > 32 || (q & (q - 1))) return false;
  grid.assign(size_t(nd), 0);
  bool ex = true;
  for (int a = 0; a < nd; ++a) ex = ex && cfg->grid_dims[a] > 0;
  for (int a = 0; a < nd; ++a) {
    grid[size_t(a)] = ex ? cfg->grid_dims[a]
                         : (cfg->grid == 1 ? std::min(cd[size_t(a)] + cfg->grid_pad, fd[size_t(a)]) : fd[size_t(a)]);
    if (grid[size_t(a)] < cd[size_t(a)] || fd[size_t(a)] < grid[size_t(a)]) return false;
  }
  if (grid == fd || !interp_fft_ok(grid, fd)) return false;
  const i64 nl = grid[size_t(nd - 1)];
  if (fd[size_t(nd - 1)] != 2 * nl || q * nl > 4096) return false;
  // a 32-slice group's planes (12 bytes per packed entry) stay within 16 GiB
  const double group_bytes = 32.0 * double(q * (q + 1) / 2) * double(numel(grid)) * 12.0;
  if (group_bytes > 16.0 * 1024 * 1024 * 1024) return false;
  return spectral_fold_smem(s.nd, s.tau, 64, int(q)) <= 200 * 1024;
}

void pipeline_group_tail(sk_ctx* ctx, const Dims& cdims, const Dims& co, i64 q, const float2* calib_dev, i64 gs,
                         const PipelineOut::Basis* bases, const Dims& full, const Dims& grid, const sk_config* cfg,
                         float2* maps, float* lambda, uint8_t* mask, sk_provenance* prov) {
  const int nd = int(cdims.size());
  const Support s = make_support(cfg->kernel, cfg->tau, nd);
  const i64 lam = s.count, n = q * lam, ngrid = numel(grid), nfull = numel(full);
  const int h = int(q * (q + 1) / 2);
  SupportTables& t = tables_for(ctx, s, int(q));
  cudaEvent_t* ev = ctx->ev;
  SKB_CUDA(cudaEventRecord(ev[0], ctx->stream));
  // K3: lags [gs][h][nbox] -> planes [gs][h][grid]
  double2* lags = ctx->arena.get<double2>("field:lags64", gs * h * t.nbox);
  const int* offs = support_offsets_dev(ctx, s);
  for (i64 c0 = 0; c0 < gs; c0 += kFoldBatchMax) {
    const int cnt = int(std::min<i64>(kFoldBatchMax, gs - c0));
    FoldBatch fb{};
    for (int i = 0; i < cnt; ++i) {
      fb.u[i] = bases[c0 + i].usig;
      fb.k[i] = int(bases[c0 + i].k);
    }
    fold_lags_spectral_batched(ctx, fb, cnt, n, int(q), int(lam), s.nd, s.tau, offs, lags + c0 * h * t.nbox);
  }
  Planes pl;
  pl.hi = ctx->arena.get<float2>("field:planes", gs * h * ngrid);
  pl.lo = ctx->arena.get<lo2>("field:planes_lo", gs * h * ngrid);
  expand_lags(ctx, lags, pl.hi, pl.lo, gs * h, s.tau, grid);
  SKB_CUDA(cudaEventRecord(ev[1], ctx->stream));
  // post (part 1): recon [gs][Q][grid]
  float2* recon = run_recon(ctx, cdims, co, gs * q, calib_dev, grid, cfg->apod_width);
  SKB_CUDA(cudaEventRecord(ev[2], ctx->stream));
  // K4 over the stack
  unsigned long long* zeroed = ctx->arena.get<unsigned long long>("post:zeroed", gs);
  SKB_CUDA(cudaMemsetAsync(zeroed, 0, size_t(gs) * sizeof(unsigned long long), ctx->stream));
  float2* maps_grid = ctx->arena.get<float2>("post:maps_grid", gs * q * ngrid);
  float* lam_grid = ctx->arena.get<float>("post:lam_grid", gs * ngrid);
  PowerArgs pa{};
  pa.planes = pl.hi;
  pa.planes_lo = pl.lo;
  pa.n = ngrid;
  pa.q = int(q);
  pa.iters = cfg->power_iters;
  pa.alpha = 1.f;
  pa.beta = -1.f / float(lam);
  pa.lam_scale = 1.f / float(lam);
  pa.recon = recon;
  pa.maps = maps_grid;
  pa.lambda = lam_grid;
  pa.mask_threshold = float(cfg->mask_threshold);
  pa.zeroed = zeroed;
  pa.rq32_min = 0.f;  // an interpolation follows (see pipeline)
  pa.slices = int(gs);
  power_iteration(ctx, pa);
  SKB_CUDA(cudaEventRecord(ev[3], ctx->stream));
  // post (part 2): interpolation + renormalisation + mask
  if (!run_interp_renorm(ctx, maps_grid, maps, q, grid, full, gs))
    fail(SK_ERR_UNSUPPORTED, "multislice group: fused interpolation refused an eligible shape");
  run_interp_lambda(ctx, lam_grid, grid, full, lambda, mask, float(cfg->mask_threshold), gs);
  SKB_CUDA(cudaEventRecord(ev[4], ctx->stream));
  const size_t need = size_t(gs) + 1;  // pinned staging in doubles (8 bytes each, as the counters)
  if (ctx->hpin_cap < need) {
    if (ctx->hpin) SKB_CUDA(cudaFreeHost(ctx->hpin));
    SKB_CUDA(cudaMallocHost(&ctx->hpin, std::max<size_t>(need, 64) * sizeof(double)));
    ctx->hpin_cap = std::max<size_t>(need, 64);
  }
  SKB_CUDA(cudaMemcpyAsync(ctx->hpin, zeroed, size_t(gs) * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (prov) {
    float ms[4], total = 0;
    for (int i = 0; i < 4; ++i) SKB_CUDA(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
    SKB_CUDA(cudaEventElapsedTime(&total, ev[0], ev[4]));
    for (i64 i = 0; i < gs; ++i) {
      sk_provenance* p = prov + i;
      std::memset(p, 0, sizeof *p);
      for (int a = 0; a < nd; ++a) p->grid_dims[a] = grid[size_t(a)];
      p->support_size = lam;
      p->valid_shifts = 1;
      for (i64 d : cdims) p->valid_shifts *= std::max<i64>(0, d - 2 * cfg->tau);
      p->nullspace_rank = n - bases[i].k;
      unsigned long long z = 0;
      std::memcpy(&z, reinterpret_cast<const unsigned char*>(ctx->hpin) + size_t(i) * sizeof z, sizeof z);
      p->zeroed_voxels = i64(z);
      p->sigma1 = bases[i].sigma1;
      p->eig_solver_used = 2;
      // the group's device time shared evenly over its slices (K1 + K2 ran batched on the producer)
      p->stage_ms[2] = ms[0] / double(gs);
      p->stage_ms[3] = ms[2] / double(gs);
      p->stage_ms[4] = (ms[1] + ms[3]) / double(gs);
      p->total_ms = total / double(gs);
    }
  }
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return SK_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SK_ERR_OTHER;
  }
}

void require_ctx(sk_ctx* ctx) {
  if (!ctx) fail(SK_ERR_DIM, "null context");
  SKB_CUDA(cudaSetDevice(ctx->device));
}

}  // namespace

// ================================================================ C-ABI
extern "C" {

const char* sk_last_error(void) { return g_last_error.c_str(); }

int sk_create(int device, sk_ctx** out) {
  return guarded([&] {
    if (!out) fail(SK_ERR_DIM, "null output");
    int count = 0;
    SKB_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) fail(SK_ERR_CUDA, "no such CUDA device " + std::to_string(device));
    SKB_CUDA(cudaSetDevice(device));
    auto* ctx = new sk_ctx();
    ctx->device = device;
    SKB_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
    SKB_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    check_cublas(cublasCreate(&ctx->cublas), "cublasCreate");
    check_cublas(cublasSetStream(ctx->cublas, ctx->stream), "cublasSetStream");
    check_cusolver(cusolverDnCreate(&ctx->cusolver), "cusolverDnCreate");
    check_cusolver(cusolverDnSetStream(ctx->cusolver, ctx->stream), "cusolverDnSetStream");
    check_cusolver(cusolverDnCreateParams(&ctx->cusolver_params), "cusolverDnCreateParams");
    for (auto& e : ctx->ev) SKB_CUDA(cudaEventCreate(&e));
    *out = ctx;
  });
}

int sk_destroy(sk_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    for (sk_ctx* sub : ctx->lanes) sk_destroy(sub);
    ctx->lanes.clear();
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->syevj) cusolverDnDestroySyevjInfo(ctx->syevj);
    if (ctx->hpin) cudaFreeHost(ctx->hpin);
    for (auto& kv : ctx->rounds)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    ctx->rounds.clear();
    ctx->arena.release_all();
    for (auto& kv : ctx->support_tables) {
      cudaFree(kv.second.pairs);
      cudaFree(kv.second.off);
      cudaFree(kv.second.lag_ptr);
      cudaFree(kv.second.lag_st);
    }
    ctx->support_tables.clear();
    for (auto& kv : ctx->tables) cudaFree(kv.second);
    ctx->tables.clear();
    for (auto& e : ctx->ev) cudaEventDestroy(e);
    for (auto& e : ctx->chunk_ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : ctx->d2h_done)
      if (e) cudaEventDestroy(e);
    if (ctx->d2h_ready) cudaEventDestroy(ctx->d2h_ready);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->hp_stream) cudaStreamDestroy(ctx->hp_stream);
    cusolverDnDestroyParams(ctx->cusolver_params);
    cusolverDnDestroy(ctx->cusolver);
    cublasDestroy(ctx->cublas);
    cudaStreamDestroy(ctx->own_stream);
    delete ctx;
  });
}

int sk_set_stream(sk_ctx* ctx, void* stream) {
  return guarded([&] {
    require_ctx(ctx);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    check_cublas(cublasSetStream(ctx->cublas, ctx->stream), "cublasSetStream");
    check_cusolver(cusolverDnSetStream(ctx->cusolver, ctx->stream), "cusolverDnSetStream");
  });
}

// Counters include the concurrent lanes (sub-contexts) of batched calls.
int64_t sk_kernel_launches(const sk_ctx* ctx) {
  if (!ctx) return 0;
  int64_t n = ctx->launches;
  for (const sk_ctx* l : ctx->lanes) n += sk_kernel_launches(l);
  return n;
}
int64_t sk_library_calls(const sk_ctx* ctx) {
  if (!ctx) return 0;
  int64_t n = ctx->lib_calls;
  for (const sk_ctx* l : ctx->lanes) n += sk_library_calls(l);
  return n;
}

int sk_make_support(int shape, int tau, int ndim, int32_t* offsets, int64_t* count) {
  return guarded([&] {
    const Support s = make_support(shape, tau, ndim);
    if (count) *count = s.count;
    if (offsets) std::copy(s.offsets.begin(), s.offsets.end(), offsets);
  });
}

int sk_reduced_grid_dims(int ndim, const int64_t* calib_dims, int64_t pad, const int64_t* full_dims, int64_t* out) {
  return guarded([&] {
    for (int a = 0; a < ndim; ++a) out[a] = std::min(calib_dims[a] + pad, full_dims[a]);
  });
}

int sk_gram_fft(sk_ctx* ctx, int ndim, const int64_t* calib_dims, int64_t channels, const sk_c64* calib, int shape,
                int tau, sk_c64* gram) {
  return guarded([&] {
    require_ctx(ctx);
    const Dims cd = dims_of(ndim, calib_dims);
    const Support s = make_support(shape, tau, ndim);
    check_calib(cd, channels, s);
    const i64 n = channels * s.count;
    const float2* d_cal = device_in(ctx, reinterpret_cast<const float2*>(calib), channels * numel(cd), "in:calib");
    Out<float2> g(ctx, reinterpret_cast<float2*>(gram), n * n, "out:gram");
    run_gram(ctx, cd, channels, d_cal, s, g.dev);
    g.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_build_calib_matrix(sk_ctx* ctx, int ndim, const int64_t* calib_dims, int64_t channels, const sk_c64* calib,
                          int shape, int tau, sk_c64* cmat, int64_t* rows) {
  return guarded([&] {
    require_ctx(ctx);
    const Dims cd = dims_of(ndim, calib_dims);
    const Support s = make_support(shape, tau, ndim);
    check_calib(cd, channels, s);
    const i64 n = channels * s.count, p = valid_shift_rows(cd, s.tau);
    if (rows) *rows = p;
    if (cmat == nullptr) return;
    const float2* d_cal = device_in(ctx, reinterpret_cast<const float2*>(calib), channels * numel(cd), "in:calib");
    double2* c = ctx->arena.get<double2>("gramx:C", std::max<i64>(1, p * n));
    calib_matrix(ctx, d_cal, cd, int(channels), s, support_offsets_dev(ctx, s), c);
    Out<float2> o(ctx, reinterpret_cast<float2*>(cmat), p * n, "out:cmat");
    c128_to_c64(ctx, c, o.dev, p * n);
    o.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_gram_explicit(sk_ctx* ctx, int64_t rows, int64_t n, const sk_c64* cmat, sk_c64* gram) {
  return guarded([&] {
    require_ctx(ctx);
    if (rows < 0 || n < 1) fail(SK_ERR_DIM, "gram_explicit: bad calibration matrix shape");
    const float2* d_c = device_in(ctx, reinterpret_cast<const float2*>(cmat), rows * n, "in:cmat");
    double2* c = ctx->arena.get<double2>("gramx:C", std::max<i64>(1, rows * n));
    c64_to_c128(ctx, d_c, c, rows * n);
    double2* lower = ctx->arena.get<double2>("gramx:lower", n * n);
    Out<float2> g(ctx, reinterpret_cast<float2*>(gram), n * n, "out:gram");
    gram_explicit_dev(ctx, c, rows, n, lower, g.dev);
    g.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_eig_dense_field(sk_ctx* ctx, int64_t voxels, int64_t q, const sk_c64* field, int largest, sk_c64* vectors,
                       float* values, float* second_values) {
  return guarded([&] {
    require_ctx(ctx);
    if (voxels < 0 || q < 1) fail(SK_ERR_DIM, "eig_dense_field: bad field shape");
    if (q > 64) fail(SK_ERR_UNSUPPORTED, "more than 64 channels is outside the B200 path");
    if (voxels == 0) return;
    const float2* d_f = device_in(ctx, reinterpret_cast<const float2*>(field), voxels * q * q, "in:field");
    float2* planes = ctx->arena.get<float2>("field:planes", voxels * q * (q + 1) / 2);
    field_full_to_planes(ctx, d_f, voxels, int(q), planes);
    float2* vec = ctx->arena.get<float2>("dense:vec", voxels * q);
    Out<float> val(ctx, values, voxels, "out:values");
    Out<float> sec(ctx, second_values, voxels, "out:second");
    DenseEigArgs d{};
    d.planes = planes;
    d.n = voxels;
    d.q = int(q);
    d.largest = largest ? 1 : 0;
    d.alpha = 0.0;
    d.beta = 1.0;
    d.vec = vec;
    d.value = val.dev;
    d.second = sec.dev;
    dense_eig(ctx, d);
    if (vectors) {  // [Q][N] -> Q x N column per voxel (eigensolve.hpp:13)
      Out<float2> v(ctx, reinterpret_cast<float2*>(vectors), voxels * q, "out:vectors");
      copy_strided(ctx, vec, 1, voxels, v.dev, q, 1, voxels, q);
      v.finish(ctx);
    }
    val.finish(ctx);
    sec.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_extract_nullspace(sk_ctx* ctx, int64_t n, const sk_c64* gram, double ratio, int64_t* rank, double* spectrum,
                         sk_c64* filters, int64_t filters_capacity) {
  return guarded([&] {
    require_ctx(ctx);
    const float2* d_g = device_in(ctx, reinterpret_cast<const float2*>(gram), n * n, "in:gram");
    Eig e = run_eigh(ctx, d_g, n, ratio);
    if (rank) *rank = e.rank;
    if (spectrum) std::copy(e.spectrum.begin(), e.spectrum.end(), spectrum);
    if (filters) {
      if (filters_capacity < e.rank) fail(SK_ERR_DIM, "filters buffer has fewer columns than the nullspace rank");
      Out<float2> f(ctx, reinterpret_cast<float2*>(filters), n * e.rank, "out:filters");
      c128_to_c64(ctx, e.evecs, f.dev, n * e.rank);
      f.finish(ctx);
    }
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_aggregate_w(sk_ctx* ctx, int64_t n, int64_t r, const sk_c64* filters, sk_c64* w) {
  return guarded([&] {
    require_ctx(ctx);
    if (r < 1) fail(SK_ERR_NULLSPACE_EMPTY, "aggregate requires at least one filter");  // spatial_gram.cpp:88
    const float2* d_f = device_in(ctx, reinterpret_cast<const float2*>(filters), n * r, "in:filters");
    Out<float2> o(ctx, reinterpret_cast<float2*>(w), n * n, "out:w");
    herk_full(ctx, d_f, n, r, o.dev);  // own tiled Hermitian product (sk_fold.cu)
    o.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_gram_field_fast(sk_ctx* ctx, int64_t q, const sk_c64* w, int shape, int tau, int ndim, const int64_t* dims,
                       sk_c64* field) {
  return guarded([&] {
    require_ctx(ctx);
    const Dims grid = dims_of(ndim, dims);
    const Support s = make_support(shape, tau, ndim);
    if (i64(grid.size()) != s.nd) fail(SK_ERR_DIM, "voxel grid rank does not match support dimension");
    for (i64 d : grid)
      if (d < 1) fail(SK_ERR_DIM, "voxel grid extents must be >= 1");
    if (4 * tau + 1 > 29) fail(SK_ERR_UNSUPPORTED, "kernel radius > 7 is outside the B200 path");
    const i64 n = q * s.count, ng = numel(grid);
    const float2* d_w = device_in(ctx, reinterpret_cast<const float2*>(w), n * n, "in:w");
    const Planes pl = run_field_from_w(ctx, d_w, s, int(q), grid);
    Out<float2> f(ctx, reinterpret_cast<float2*>(field), ng * q * q, "out:field");
    planes_to_field_full(ctx, pl.hi, pl.lo, ng, int(q), f.dev);
    f.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_espirit_inplace(sk_ctx* ctx, int64_t voxels, int64_t q, sk_c64* field, int64_t support_size) {
  return guarded([&] {
    require_ctx(ctx);
    const i64 cnt = voxels * q * q;
    const bool dev = is_device_ptr(field);
    float2* d = dev ? reinterpret_cast<float2*>(field) : ctx->arena.get<float2>("io:field", cnt);
    if (!dev) SKB_CUDA(cudaMemcpyAsync(d, field, size_t(cnt) * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
    espirit_field(ctx, d, voxels, int(q), float(1.0 / double(support_size)));
    if (!dev) SKB_CUDA(cudaMemcpyAsync(field, d, size_t(cnt) * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_eig_power_field(sk_ctx* ctx, int64_t voxels, int64_t q, const sk_c64* b_field, int iters, sk_c64* vectors,
                       float* values) {
  return guarded([&] {
    require_ctx(ctx);
    if (q > power_wide_max_q())
      fail(SK_ERR_UNSUPPORTED, "more than " + std::to_string(power_wide_max_q()) + " channels is outside the B200 path");
    const float2* d_b = device_in(ctx, reinterpret_cast<const float2*>(b_field), voxels * q * q, "in:field");
    float2* planes = ctx->arena.get<float2>("field:planes", voxels * q * (q + 1) / 2);
    field_full_to_planes(ctx, d_b, voxels, int(q), planes);
    float2* maps = ctx->arena.get<float2>("power:maps", voxels * q);
    Out<float> val(ctx, values, voxels, "out:values");
    PowerArgs a{};
    a.planes = planes;
    a.n = voxels;
    a.q = int(q);
    a.iters = iters;
    a.alpha = 0.f;  // B given directly
    a.beta = 1.f;
    a.lam_scale = 1.f;
    a.maps = maps;
    a.value = val.dev;
    power_iteration(ctx, a);
    // [Q][N] -> Q x N column per voxel (eigensolve.hpp:13): element (c, j) at c + j*Q
    if (vectors) {
      Out<float2> vec(ctx, reinterpret_cast<float2*>(vectors), voxels * q, "out:vectors");
      // rows = voxels j, cols = channels c: src maps[c*N + j], dst vectors[c + j*Q]
      copy_strided(ctx, maps, 1, voxels, vec.dev, q, 1, voxels, q);
      vec.finish(ctx);
    }
    val.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_normalize_maps(sk_ctx* ctx, int ndim, const int64_t* dims, int64_t q, const sk_c64* raw,
                      const int64_t* calib_dims, const int64_t* center_offset, const sk_c64* calib, double apod_width,
                      sk_c64* out, int64_t* zeroed_voxels) {
  return guarded([&] {
    require_ctx(ctx);
    const Dims grid = dims_of(ndim, dims), cd = dims_of(ndim, calib_dims), co = dims_of(ndim, center_offset);
    for (int a = 0; a < ndim; ++a)
      if (grid[size_t(a)] < cd[size_t(a)]) fail(SK_ERR_DIM, "map grid smaller than calibration region");
    const i64 ng = numel(grid);
    const float2* d_raw = device_in(ctx, reinterpret_cast<const float2*>(raw), q * ng, "in:raw");
    const float2* d_cal = device_in(ctx, reinterpret_cast<const float2*>(calib), q * numel(cd), "in:calib");
    float2* recon = run_recon(ctx, cd, co, q, d_cal, grid, apod_width);
    Out<float2> o(ctx, reinterpret_cast<float2*>(out), q * ng, "out:maps");
    SKB_CUDA(cudaMemcpyAsync(o.dev, d_raw, size_t(q * ng) * sizeof(float2), cudaMemcpyDeviceToDevice, ctx->stream));
    unsigned long long* z = ctx->arena.get<unsigned long long>("post:zeroed", 1);
    SKB_CUDA(cudaMemsetAsync(z, 0, sizeof(unsigned long long), ctx->stream));
    normalize_standalone(ctx, o.dev, ng, int(q), recon, z);
    o.finish(ctx);
    unsigned long long hz = 0;
    SKB_CUDA(cudaMemcpyAsync(&hz, z, sizeof hz, cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (zeroed_voxels) *zeroed_voxels = i64(hz);
  });
}

int sk_interpolate_maps(sk_ctx* ctx, int ndim, const int64_t* low_dims, int64_t q, const sk_c64* low,
                        const int64_t* full_dims, sk_c64* out) {
  return guarded([&] {
    require_ctx(ctx);
    const Dims ld = dims_of(ndim, low_dims), fd = dims_of(ndim, full_dims);
    for (int a = 0; a < ndim; ++a)
      if (fd[size_t(a)] < ld[size_t(a)])
        fail(SK_ERR_DIM, "interpolation target smaller than source on axis " + std::to_string(a));
    const float2* d_low = device_in(ctx, reinterpret_cast<const float2*>(low), q * numel(ld), "in:low");
    Out<float2> o(ctx, reinterpret_cast<float2*>(out), q * numel(fd), "out:interp");
    run_interp(ctx, d_low, o.dev, q, ld, fd);
    o.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_interpolate_real(sk_ctx* ctx, int ndim, const int64_t* low_dims, const float* low, const int64_t* full_dims,
                        float* out) {
  return guarded([&] {
    require_ctx(ctx);
    const Dims ld = dims_of(ndim, low_dims), fd = dims_of(ndim, full_dims);
    for (int a = 0; a < ndim; ++a)
      if (fd[size_t(a)] < ld[size_t(a)])
        fail(SK_ERR_DIM, "interpolation target smaller than source on axis " + std::to_string(a));
    const float* d_low = device_in(ctx, low, numel(ld), "in:lowr");
    Out<float> o(ctx, out, numel(fd), "out:interpr");
    run_interp_lambda(ctx, d_low, ld, fd, o.dev, nullptr, 0.f);
    o.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_support_mask(sk_ctx* ctx, int64_t voxels, const float* lambda, double thr, uint8_t* mask) {
  return guarded([&] {
    require_ctx(ctx);
    const float* d_l = device_in(ctx, lambda, voxels, "in:lambda");
    Out<uint8_t> o(ctx, mask, voxels, "out:mask");
    mask_kernel(ctx, d_l, voxels, float(thr), o.dev);
    o.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_debug_small_eigh(sk_ctx* ctx, int64_t n, double* h, double* w) {
  return guarded([&] {
    require_ctx(ctx);
    if (n < 1 || n > 4096 || h == nullptr || w == nullptr) fail(SK_ERR_DIM, "sk_debug_small_eigh: bad arguments");
    double2* dh = ctx->arena.get<double2>("dbg:h", n * n);
    double* dw = ctx->arena.get<double>("dbg:w", n);
    int* info = ctx->arena.get<int>("dbg:info", 1);
    SKB_CUDA(cudaMemsetAsync(info, 0, sizeof(int), ctx->stream));
    SKB_CUDA(cudaMemcpyAsync(dh, h, size_t(n * n) * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    small_heev(ctx, dh, n, dw, info);
    int hinfo = 0;
    SKB_CUDA(cudaMemcpyAsync(h, dh, size_t(n * n) * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaMemcpyAsync(w, dw, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hinfo != 0) fail(SK_ERR_OTHER, "sk_debug_small_eigh: solver reported failure");
  });
}

int sk_debug_cholqr(sk_ctx* ctx, int64_t n, int64_t b, double* x, int passes) {
  return guarded([&] {
    require_ctx(ctx);
    if (n < 1 || b < 1 || b > n || b > 256 || passes < 1 || passes > 4 || x == nullptr)
      fail(SK_ERR_DIM, "sk_debug_cholqr: bad arguments");
    double2* dx = ctx->arena.get<double2>("dbg:x", n * b);
    double2* dt = ctx->arena.get<double2>("dbg:t", n * b);
    int* info = ctx->arena.get<int>("dbg:qinfo", 3);
    SKB_CUDA(cudaMemsetAsync(info, 0, 3 * sizeof(int), ctx->stream));
    SKB_CUDA(cudaMemcpyAsync(dx, x, size_t(n * b) * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    double2* px = dx;
    double2* pt = dt;
    if (!orth(ctx, px, pt, n, b, info + 1, passes)) fail(SK_ERR_OTHER, "sk_debug_cholqr: orthonormalisation failed");
    int hinfo[3] = {0, 0, 0};
    SKB_CUDA(cudaMemcpyAsync(x, px, size_t(n * b) * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaMemcpyAsync(hinfo, info, 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hinfo[1] != 0 || hinfo[2] != 0) fail(SK_ERR_OTHER, "sk_debug_cholqr: non-positive pivot");
  });
}

int sk_debug_cross_gram(sk_ctx* ctx, int64_t n, int64_t b, const double* x, const double* y, double* out) {
  return guarded([&] {
    require_ctx(ctx);
    if (n < 1 || b < 1 || b > 256 || x == nullptr || out == nullptr)
      fail(SK_ERR_DIM, "sk_debug_cross_gram: bad arguments");
    double2* dx = ctx->arena.get<double2>("dbg:x", n * b);
    double2* dy = y ? ctx->arena.get<double2>("dbg:y", n * b) : dx;
    double2* dh = ctx->arena.get<double2>("dbg:h", b * b);
    SKB_CUDA(cudaMemcpyAsync(dx, x, size_t(n * b) * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    if (y) SKB_CUDA(cudaMemcpyAsync(dy, y, size_t(n * b) * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    if (b == 64)
      gram64(ctx, dx, dy, n, dh);
    else
      cross_gram(ctx, dx, dy, n, int(b), dh);
    SKB_CUDA(cudaMemcpyAsync(out, dh, size_t(b * b) * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"

namespace {
struct ProbeIn {
  int64_t n_gram = 0, n_field = 0;
  const int64_t* gram_idx = nullptr;
  const int64_t* field_idx = nullptr;
  double* gram_vals = nullptr;
  double* field_vals = nullptr;
  double* gram_fro = nullptr;
  double* field_fro = nullptr;
  float* raw_lambda = nullptr;  // host, N_grid
};

int estimate_impl(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset, int64_t q,
                  const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg, sk_c64* maps, float* lambda,
                  uint8_t* mask, double* spectrum, sk_provenance* prov, sk_c64* gram_out, sk_c64* field_out,
                  sk_c64* raw_maps_out, float* raw_lambda_out, const ProbeIn* pin,
                  const PipelineOut::Basis* basis_in = nullptr) {
  return guarded([&] {
    require_ctx(ctx);
    if (ndim < 1) fail(SK_ERR_DIM, "stack needs at least one axis");
    const Dims cd = dims_of(ndim, calib_dims), co = dims_of(ndim, center_offset), fd = dims_of(ndim, full_dims);
    for (i64 d : cd)
      if (d < 1) fail(SK_ERR_DIM, "stack axis extents must be >= 1");
    if (q < 1) fail(SK_ERR_DIM, "stack needs at least one channel");
    const i64 nfull = numel(fd);
    const float2* d_cal = device_in(ctx, reinterpret_cast<const float2*>(calib), q * numel(cd), "in:calib");
    // Batched lanes (defer_d2h): the host outputs' staging alternates between
    // two slots and is copied out on the copy stream while the lane's next
    // slice computes; a slot is reused only after its copy completed.
    const bool defer = ctx->defer_d2h != 0;
    const std::string sfx = defer ? ":" + std::to_string(ctx->d2h_slot) : "";
    Out<float2> om(ctx, reinterpret_cast<float2*>(maps), q * nfull, "out:maps" + sfx);
    Out<float> ol(ctx, lambda, nfull, "out:lambda" + sfx);
    Out<uint8_t> ok(ctx, mask, nfull, "out:mask" + sfx);
    if (defer) {
      if (!ctx->copy_stream) {
        SKB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (auto& e : ctx->chunk_ev) SKB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      if (!ctx->d2h_ready) {
        SKB_CUDA(cudaEventCreateWithFlags(&ctx->d2h_ready, cudaEventDisableTiming));
        for (auto& e : ctx->d2h_done) SKB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : ctx->d2h_done) SKB_CUDA(cudaEventRecord(e, ctx->copy_stream));
      }
      SKB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->d2h_done[ctx->d2h_slot], 0));  // slot's last copy drained
    }
    // debug dumps need sizes: derive them the same way the pipeline does
    const Support s = make_support(cfg ? cfg->kernel : 0, cfg ? cfg->tau : 0, ndim);
    const i64 n = q * s.count;
    Dims grid(static_cast<size_t>(ndim));
    if (cfg) {
      bool ex = true;
      for (int a = 0; a < ndim; ++a) ex = ex && cfg->grid_dims[a] > 0;
      for (int a = 0; a < ndim; ++a)
        grid[size_t(a)] = ex ? cfg->grid_dims[a]
                             : (cfg->grid == 1 ? std::min(cd[size_t(a)] + cfg->grid_pad, fd[size_t(a)]) : fd[size_t(a)]);
    }
    const i64 ng = numel(grid);
    // Pinned host maps on a full-resolution power-iteration grid: K4 is the
    // only writer of the maps (coalesced channel-major stores of 32-64 B per
    // tile row), so it can write them straight into the caller's pinned
    // buffer over the host link while it computes, instead of a device
    // staging buffer and a D2H copy after the pipeline.  Worth it only when
    // K4 runs long enough per map byte (rate ~ FP32 rate / (iters * Q)):
    // measured C5 (iters*Q = 5120) e2e 7.2 -> 7.8 M voxels/s, C2 (1600)
    // 20.6 -> 16.6 (the short, write-rate-bound K4 slows down).
    // SKB_ZERO_COPY=0 disables, =2 forces.
    static const int zero_copy = [] {
      const char* v = std::getenv("SKB_ZERO_COPY");
      return v ? std::atoi(v) : 1;
    }();
    float2* maps_alias = nullptr;
    if (!defer && zero_copy && maps && cfg && cfg->eig == 1 && grid == fd &&
        (zero_copy == 2 || i64(cfg->power_iters) * q >= 4096))
      maps_alias = static_cast<float2*>(pinned_alias(maps));
    if (maps_alias) om = Out<float2>(ctx, nullptr, 0, "out:maps");
    // otherwise pinned host maps on a full-resolution power grid are copied
    // out chunk by chunk behind K4 (PipelineOut::maps_host)
    float2* maps_host = nullptr;
    if (!defer && !maps_alias && zero_copy && maps && om.host && cfg && cfg->eig == 1 && grid == fd &&
        pinned_alias(maps))
      maps_host = reinterpret_cast<float2*>(maps);
    Out<float2> og(ctx, reinterpret_cast<float2*>(gram_out), n * n, "dbg:gram");
    Out<float2> of(ctx, reinterpret_cast<float2*>(field_out), ng * q * q, "dbg:field");
    Out<float2> orm(ctx, reinterpret_cast<float2*>(raw_maps_out), q * ng, "dbg:raw");
    Out<float> orl(ctx, raw_lambda_out, ng, "dbg:rawl");
    std::vector<double> spec(size_t(std::max<i64>(n, 1)));
    PipelineOut po;
    po.maps = maps_alias ? maps_alias : om.dev;
    po.maps_host = maps_host;
    po.lambda = ol.dev;
    po.mask = ok.dev;
    po.gram = og.dev;
    po.field = of.dev;
    po.raw_maps = orm.dev;
    po.raw_lambda = orl.dev;
    po.spectrum = spectrum ? spec.data() : nullptr;
    PipelineOut::Probe probe;
    Out<float> opl(ctx, pin ? pin->raw_lambda : nullptr, ng, "probe:rawl");
    if (pin) {
      const i64 ng_idx = std::max<int64_t>(pin->n_gram, 0), nf_idx = std::max<int64_t>(pin->n_field, 0);
      long long* gi = ctx->arena.get<long long>("probe:gram_idx", std::max<i64>(1, 2 * ng_idx));
      long long* fi = ctx->arena.get<long long>("probe:field_idx", std::max<i64>(1, 3 * nf_idx));
      if (ng_idx)
        SKB_CUDA(cudaMemcpyAsync(gi, pin->gram_idx, size_t(2 * ng_idx) * 8, cudaMemcpyHostToDevice, ctx->stream));
      if (nf_idx)
        SKB_CUDA(cudaMemcpyAsync(fi, pin->field_idx, size_t(3 * nf_idx) * 8, cudaMemcpyHostToDevice, ctx->stream));
      for (i64 k = 0; k < 2 * ng_idx; ++k)
        if (pin->gram_idx[k] < 0 || pin->gram_idx[k] >= n) fail(SK_ERR_DIM, "probe gram index out of range");
      for (i64 k = 0; k < nf_idx; ++k)
        if (pin->field_idx[3 * k] < 0 || pin->field_idx[3 * k] >= ng || pin->field_idx[3 * k + 1] < 0 ||
            pin->field_idx[3 * k + 1] >= q || pin->field_idx[3 * k + 2] < 0 || pin->field_idx[3 * k + 2] >= q)
          fail(SK_ERR_DIM, "probe field index out of range");
      probe.n_gram = ng_idx;
      probe.n_field = nf_idx;
      probe.gram_idx = gi;
      probe.field_idx = fi;
      probe.gram_vals = ctx->arena.get<double2>("probe:gram_vals", std::max<i64>(1, ng_idx));
      probe.field_vals = ctx->arena.get<double2>("probe:field_vals", std::max<i64>(1, nf_idx));
      probe.raw_lambda = opl.dev;
      po.probe = &probe;
    }
    PipelineOut::Basis basis_copy;
    if (basis_in) {  // multislice: the slice's signal basis from the batched K2
      basis_copy = *basis_in;
      po.basis = &basis_copy;
    }
    pipeline(ctx, cd, co, q, d_cal, fd, cfg, po, prov);
    if (pin) {
      if (pin->n_gram > 0)
        SKB_CUDA(cudaMemcpyAsync(pin->gram_vals, probe.gram_vals, size_t(pin->n_gram) * 16, cudaMemcpyDeviceToHost,
                                 ctx->stream));
      if (pin->n_field > 0)
        SKB_CUDA(cudaMemcpyAsync(pin->field_vals, probe.field_vals, size_t(pin->n_field) * 16,
                                 cudaMemcpyDeviceToHost, ctx->stream));
      if (pin->gram_fro) *pin->gram_fro = std::sqrt(probe.gram_sumsq);
      if (pin->field_fro) *pin->field_fro = std::sqrt(probe.field_sumsq);
      opl.finish(ctx);
    }
    if (defer) {
      SKB_CUDA(cudaEventRecord(ctx->d2h_ready, ctx->stream));
      SKB_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->d2h_ready, 0));
      om.finish_on(ctx->copy_stream);
      ol.finish_on(ctx->copy_stream);
      ok.finish_on(ctx->copy_stream);
      SKB_CUDA(cudaEventRecord(ctx->d2h_done[ctx->d2h_slot], ctx->copy_stream));
      ctx->d2h_slot ^= 1;
    } else {
      if (!maps_host) om.finish(ctx);
      ol.finish(ctx);
      ok.finish(ctx);
    }
    og.finish(ctx);
    of.finish(ctx);
    orm.finish(ctx);
    orl.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (spectrum) std::copy(spec.begin(), spec.begin() + n, spectrum);
  });
}
}  // namespace

extern "C" {

int sk_estimate_maps_debug(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                           int64_t q, const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg,
                           sk_c64* maps, float* lambda, uint8_t* mask, double* spectrum, sk_provenance* prov,
                           sk_c64* gram_out, sk_c64* field_out, sk_c64* raw_maps_out, float* raw_lambda_out) {
  return estimate_impl(ctx, ndim, calib_dims, center_offset, q, calib, full_dims, cfg, maps, lambda, mask, spectrum,
                       prov, gram_out, field_out, raw_maps_out, raw_lambda_out, nullptr);
}

int sk_estimate_maps_probe(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                           int64_t q, const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg,
                           sk_c64* maps, float* lambda, uint8_t* mask, sk_provenance* prov, int64_t n_gram,
                           const int64_t* gram_idx, double* gram_vals, double* gram_fro, int64_t n_field,
                           const int64_t* field_idx, double* field_vals, double* field_fro, float* raw_lambda) {
  ProbeIn pin;
  pin.n_gram = n_gram;
  pin.n_field = n_field;
  pin.gram_idx = gram_idx;
  pin.field_idx = field_idx;
  pin.gram_vals = gram_vals;
  pin.field_vals = field_vals;
  pin.gram_fro = gram_fro;
  pin.field_fro = field_fro;
  pin.raw_lambda = raw_lambda;
  return estimate_impl(ctx, ndim, calib_dims, center_offset, q, calib, full_dims, cfg, maps, lambda, mask, nullptr,
                       prov, nullptr, nullptr, nullptr, nullptr, &pin);
}

int sk_projection_residual(sk_ctx* ctx, int ndim, const int64_t* dims, int64_t channels, const sk_c64* kspace,
                           const sk_c64* maps, double* value) {
  return guarded([&] {
    require_ctx(ctx);
    if (ndim < 1 || channels < 1 || !value) fail(SK_ERR_DIM, "bad arguments");
    const Dims d = dims_of(ndim, dims);
    for (i64 e : d)
      if (e < 1) fail(SK_ERR_DIM, "stack axis extents must be >= 1");
    const i64 n = numel(d), cnt = channels * n;
    const float2* d_k = device_in(ctx, reinterpret_cast<const float2*>(kspace), cnt, "in:res_kspace");
    const float2* d_m = device_in(ctx, reinterpret_cast<const float2*>(maps), cnt, "in:res_maps");
    // image = kspace_to_image_unitary per channel (metrics.cpp:21-27, fft.cpp:105-112)
    float2* bufs[2] = {ctx->arena.get<float2>("res:img_a", cnt), ctx->arena.get<float2>("res:img_b", cnt)};
    const float2* src = d_k;
    int which = 0;
    for (int a = ndim - 1; a >= 0; --a) {
      const int N = int(d[size_t(a)]);
      if (N == 1) continue;
      i64 b = channels, inner = 1;
      for (int k = 0; k < a; ++k) b *= d[size_t(k)];
      for (int k = a + 1; k < ndim; ++k) inner *= d[size_t(k)];
      float2* dst = bufs[which];
      if (!centered_fft_axis(ctx, src, dst, b, N, inner, true, 1.0))
        apply_axis(ctx, src, dst, dft_matrix(ctx, N, N, center_index(N), center_index(N), +1, 0.0), b, N, N, inner);
      src = dst;
      which ^= 1;
    }
    float2* img = const_cast<float2*>(src);
    if (src == d_k) {  // every extent is 1
      img = bufs[0];
      SKB_CUDA(cudaMemcpyAsync(img, d_k, size_t(cnt) * sizeof(float2), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    // the unitary scale 1/sqrt(N) cancels in sqrt(num / den): both sums scale by 1/N
    *value = projection_residual_value(ctx, img, d_m, n, int(channels));
  });
}

int sk_estimate_raw_slab(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                         int64_t q, const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg,
                         int64_t slab_begin, int64_t slab_end, sk_c64* maps, float* lambda, sk_provenance* prov) {
  return guarded([&] {
    require_ctx(ctx);
    if (ndim < 1 || !cfg) fail(SK_ERR_DIM, "bad arguments");
    const Dims cd = dims_of(ndim, calib_dims), co = dims_of(ndim, center_offset), fd = dims_of(ndim, full_dims);
    for (i64 d : cd)
      if (d < 1) fail(SK_ERR_DIM, "stack axis extents must be >= 1");
    if (q < 1) fail(SK_ERR_DIM, "stack needs at least one channel");
    Dims grid(static_cast<size_t>(ndim));
    bool ex = true;
    for (int a = 0; a < ndim; ++a) ex = ex && cfg->grid_dims[a] > 0;
    for (int a = 0; a < ndim; ++a)
      grid[size_t(a)] = ex ? cfg->grid_dims[a]
                           : (cfg->grid == 1 ? std::min(cd[size_t(a)] + cfg->grid_pad, fd[size_t(a)]) : fd[size_t(a)]);
    if (slab_begin < 0 || slab_end <= slab_begin || slab_end > grid[0])
      fail(SK_ERR_DIM, "slab rows must satisfy 0 <= begin < end <= grid_dims[0]");
    const i64 nvox = numel(grid) / grid[0] * (slab_end - slab_begin);
    const float2* d_cal = device_in(ctx, reinterpret_cast<const float2*>(calib), q * numel(cd), "in:calib");
    Out<float2> om(ctx, reinterpret_cast<float2*>(maps), q * nvox, "out:slab_maps");
    Out<float> ol(ctx, lambda, nvox, "out:slab_lambda");
    PipelineOut po;
    po.maps = om.dev ? om.dev : ctx->arena.get<float2>("out:slab_maps", q * nvox);
    po.lambda = ol.dev ? ol.dev : ctx->arena.get<float>("out:slab_lambda", nvox);
    po.slab0 = slab_begin;
    po.slab1 = slab_end;
    pipeline(ctx, cd, co, q, d_cal, fd, cfg, po, prov);
    om.finish(ctx);
    ol.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_signal_basis(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset, int64_t q,
                    const sk_c64* calib, const sk_config* cfg, int64_t kmax, double* u_sig, int64_t* k,
                    int64_t* rank, double* sigma1, double* cut_margin) {
  return guarded([&] {
    require_ctx(ctx);
    if (ndim < 1 || !cfg) fail(SK_ERR_DIM, "bad arguments");
    const Dims cd = dims_of(ndim, calib_dims), co = dims_of(ndim, center_offset);
    for (i64 d : cd)
      if (d < 1) fail(SK_ERR_DIM, "stack axis extents must be >= 1");
    if (q < 1) fail(SK_ERR_DIM, "stack needs at least one channel");
    const float2* d_cal = device_in(ctx, reinterpret_cast<const float2*>(calib), q * numel(cd), "in:calib");
    PipelineOut po;
    Eig e;
    po.eig_out = &e;
    sk_config c = *cfg;  // only K1 + K2 run: the map grid is irrelevant (full = calib dims)
    c.grid = 0;
    for (auto& g : c.grid_dims) g = 0;
    pipeline(ctx, cd, co, q, d_cal, cd, &c, po, nullptr);
    if (k) *k = e.k;
    if (rank) *rank = e.rank;
    if (sigma1) *sigma1 = e.sigma1;
    if (cut_margin) *cut_margin = e.margin;
    if (e.k > kmax) fail(SK_ERR_DIM, "signal basis has " + std::to_string(e.k) + " columns, capacity " +
                                         std::to_string(kmax));
    if (u_sig && e.k > 0)
      SKB_CUDA(cudaMemcpyAsync(u_sig, e.usig, size_t(e.n * e.k) * sizeof(double2), cudaMemcpyDefault, ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_estimate_raw_slab_basis(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                               int64_t q, const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg,
                               const double* u_sig, int64_t k, double sigma1, int64_t slab_begin, int64_t slab_end,
                               sk_c64* maps, float* lambda, sk_provenance* prov) {
  return guarded([&] {
    require_ctx(ctx);
    if (ndim < 1 || !cfg) fail(SK_ERR_DIM, "bad arguments");
    const Dims cd = dims_of(ndim, calib_dims), co = dims_of(ndim, center_offset), fd = dims_of(ndim, full_dims);
    for (i64 d : cd)
      if (d < 1) fail(SK_ERR_DIM, "stack axis extents must be >= 1");
    if (q < 1) fail(SK_ERR_DIM, "stack needs at least one channel");
    const Support s = make_support(cfg->kernel, cfg->tau, ndim);
    const i64 n = q * s.count;
    if (k < 0 || k > n) fail(SK_ERR_DIM, "signal basis column count out of range");
    Dims grid(static_cast<size_t>(ndim));
    bool ex = true;
    for (int a = 0; a < ndim; ++a) ex = ex && cfg->grid_dims[a] > 0;
    for (int a = 0; a < ndim; ++a)
      grid[size_t(a)] = ex ? cfg->grid_dims[a]
                           : (cfg->grid == 1 ? std::min(cd[size_t(a)] + cfg->grid_pad, fd[size_t(a)]) : fd[size_t(a)]);
    if (slab_begin < 0 || slab_end <= slab_begin || slab_end > grid[0])
      fail(SK_ERR_DIM, "slab rows must satisfy 0 <= begin < end <= grid_dims[0]");
    const i64 nvox = numel(grid) / grid[0] * (slab_end - slab_begin);
    const float2* d_cal = device_in(ctx, reinterpret_cast<const float2*>(calib), q * numel(cd), "in:calib");
    const double2* d_u = device_in(ctx, reinterpret_cast<const double2*>(u_sig), n * std::max<i64>(k, 1), "in:usig");
    Out<float2> om(ctx, reinterpret_cast<float2*>(maps), q * nvox, "out:slab_maps");
    Out<float> ol(ctx, lambda, nvox, "out:slab_lambda");
    PipelineOut po;
    PipelineOut::Basis basis;
    basis.usig = d_u;
    basis.k = k;
    basis.sigma1 = sigma1;
    po.basis = &basis;
    po.maps = om.dev ? om.dev : ctx->arena.get<float2>("out:slab_maps", q * nvox);
    po.lambda = ol.dev ? ol.dev : ctx->arena.get<float>("out:slab_lambda", nvox);
    po.slab0 = slab_begin;
    po.slab1 = slab_end;
    pipeline(ctx, cd, co, q, d_cal, fd, cfg, po, prov);
    om.finish(ctx);
    ol.finish(ctx);
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_sos_accumulate(sk_ctx* ctx, int64_t voxels, int64_t channels, const sk_c64* maps, float* sos) {
  return guarded([&] {
    require_ctx(ctx);
    if (voxels < 0 || channels < 0) fail(SK_ERR_DIM, "bad arguments");
    const float2* d_m = device_in(ctx, reinterpret_cast<const float2*>(maps), channels * voxels, "in:maps");
    const bool host = sos && !is_device_ptr(sos);
    float* d_s = host ? ctx->arena.get<float>("io:sos", voxels) : sos;
    if (host) SKB_CUDA(cudaMemcpyAsync(d_s, sos, size_t(voxels) * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    sos_accumulate(ctx, d_m, voxels, int(channels), d_s);
    if (host) SKB_CUDA(cudaMemcpyAsync(sos, d_s, size_t(voxels) * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_renormalize_sos(sk_ctx* ctx, int64_t voxels, int64_t channels, sk_c64* maps, const float* sos) {
  return guarded([&] {
    require_ctx(ctx);
    if (voxels < 0 || channels < 0) fail(SK_ERR_DIM, "bad arguments");
    const float* d_s = device_in(ctx, sos, voxels, "in:sos");
    const bool host = maps && !is_device_ptr(maps);
    float2* d_m = host ? ctx->arena.get<float2>("io:renorm_maps", channels * voxels) : reinterpret_cast<float2*>(maps);
    if (host)
      SKB_CUDA(cudaMemcpyAsync(d_m, maps, size_t(channels * voxels) * sizeof(float2), cudaMemcpyHostToDevice,
                               ctx->stream));
    renorm_with_sos(ctx, d_m, voxels, int(channels), d_s);
    if (host)
      SKB_CUDA(cudaMemcpyAsync(maps, d_m, size_t(channels * voxels) * sizeof(float2), cudaMemcpyDeviceToHost,
                               ctx->stream));
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int sk_estimate_maps(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset, int64_t q,
                     const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg, sk_c64* maps, float* lambda,
                     uint8_t* mask, double* spectrum, sk_provenance* prov) {
  return sk_estimate_maps_debug(ctx, ndim, calib_dims, center_offset, q, calib, full_dims, cfg, maps, lambda, mask,
                                spectrum, prov, nullptr, nullptr, nullptr, nullptr);
}

int sk_estimate_maps_batched(sk_ctx* ctx, int64_t slices, int ndim, const int64_t* calib_dims,
                             const int64_t* center_offset, int64_t q, const sk_c64* calib, const int64_t* full_dims,
                             const sk_config* cfg, sk_c64* maps, float* lambda, uint8_t* mask, sk_provenance* prov) {
  if (!ctx || slices < 0 || ndim < 1) {
    g_last_error = "bad arguments";
    return SK_ERR_DIM;
  }
  const Dims cd = dims_of(ndim, calib_dims), fd = dims_of(ndim, full_dims);
  const i64 ncal = q * numel(cd), nfull = numel(fd);
  // Slices are independent pipelines whose small dense stages are latency
  // bound: run them on `lanes` sub-contexts (own stream, cuBLAS/cuSOLVER
  // handles and workspace) driven by host threads, so the GPU overlaps them.
  int lanes = 12;  // measured best for C3 (8: 81, 12: 92, 16: 91 M voxels/s)
  if (const char* v = std::getenv("SKB_LANES")) lanes = std::max(1, std::atoi(v));
  lanes = int(std::min<i64>(lanes, std::max<i64>(slices, 1)));
  int rc0 = guarded([&] {
    require_ctx(ctx);
    while (int(ctx->lanes.size()) < lanes) {
      sk_ctx* sub = nullptr;
      const int rc = sk_create(ctx->device, &sub);
      if (rc != SK_OK) fail(rc, g_last_error);
      ctx->lanes.push_back(sub);
    }
    SKB_CUDA(cudaStreamSynchronize(ctx->stream));  // inputs written on the caller's stream are visible
  });
  if (rc0 != SK_OK) return rc0;
  std::vector<int> rcs(size_t(lanes), SK_OK);
  std::vector<std::string> errs(static_cast<size_t>(lanes));
  // Pinned host outputs: each lane copies a slice's outputs on its copy stream
  // while it computes the next slice (SKB_DEFER_D2H=0 keeps the copy inline).
  static const bool defer_env = [] {
    const char* v = std::getenv("SKB_DEFER_D2H");
    return !v || std::atoi(v) != 0;
  }();
  const bool defer = defer_env && maps && pinned_alias(maps) != nullptr;
  // Batched K2 (run_eigh_subspace_batched): the calling thread computes the
  // Grams and signal bases of groups of G slices on the main context while
  // the lanes run K3-K5 of the previous group with those bases.  Eligible:
  // FFT Gram, subspace nullspace solver without certificate, n >= 1024 (the
  // b = 64 batched CholQR), a signal space that fits the 64-column block.
  i64 n_gram = 0;
  Support sup{};
  bool bk2 = false;
  if (cfg && lanes >= 2 && slices >= 2) {
    const int rc = guarded([&] {
      sup = make_support(cfg->kernel, cfg->tau, ndim);
      n_gram = q * sup.count;
    });
    const auto it = ctx->subspace_hint.find(n_gram);
    static const bool bk2_env = [] {
      const char* v = std::getenv("SKB_BATCHED_K2");
      return !v || std::atoi(v) != 0;
    }();
    // Not with pinned host outputs (defer): the host link bounds those calls and
    // the lanes' own K2 measured faster there (C3 e2e 121 vs 100 M voxels/s).
    bk2 = bk2_env && !defer && rc == SK_OK && cfg->gram == 1 && (cfg->eig_solver == 0 || cfg->eig_solver == 2) &&
          !cfg->certify && n_gram >= 1024 && n_gram <= 8192 &&
          (it == ctx->subspace_hint.end() || it->second.m + 16 <= 64);
  }
  // Groups: a small first group (the lanes start after it, not after a full
  // one), then G slices each.  Uniform G on C3 (128 slices): 8: 71, 16: 62.7,
  // 32: 60.3, 64: 59.9 ms per call; G = 32 keeps the two buffer sets at
  // ~3.5 GB each.
  const i64 G = bk2 ? std::min<i64>(slices, 32) : slices;
  std::vector<i64> gstart;  // group g = slices [gstart[g], gstart[g + 1])
  if (bk2) {
    const i64 first = std::min<i64>(slices, std::max<i64>(2, G / 4));
    gstart.push_back(0);
    for (i64 s0 = first; s0 < slices; s0 += G) gstart.push_back(s0);
    // (a small last group, whose K3-K5 nothing overlaps, measured no gain: 52.9 against 52.2 ms on C3)
    gstart.push_back(slices);
  }
  const i64 groups = bk2 ? i64(gstart.size()) - 1 : 0;
  // K3-K5 of each group in one batched pass on one consumer context
  // (pipeline_group_tail) instead of slice by slice on the lanes: device
  // outputs and an eligible configuration; SKB_GROUP_TAIL=0 keeps the lanes.
  Dims grid_t;
  static const bool tail_env = [] {
    const char* v = std::getenv("SKB_GROUP_TAIL");
    return !v || std::atoi(v) != 0;
  }();
  const bool tail = bk2 && tail_env && maps && lambda && mask && is_device_ptr(maps) && is_device_ptr(lambda) &&
                    is_device_ptr(mask) && group_tail_eligible(cfg, cd, fd, q, sup, grid_t);
  std::vector<const float2*> gcal(size_t(groups), nullptr);  // device calibration block of each group
  std::vector<PipelineOut::Basis> bases(size_t(bk2 ? slices : 0));
  std::vector<char> has_basis(size_t(bk2 ? slices : 0), 0);
  std::vector<cudaEvent_t> gev(size_t(groups), nullptr);
  std::mutex mu;
  std::condition_variable cv;
  i64 groups_ready = 0;
  bool abort_k2 = false;
  // a lane or the group consumer stopped on an error: nobody may wait for its
  // share of a group any more (the producer returns, the other workers stop)
  bool worker_failed = false;
  std::vector<i64> done(size_t(groups), 0);
  auto group_size = [&](i64 g) { return gstart[size_t(g + 1)] - gstart[size_t(g)]; };
  auto group_of = [&](i64 s) { return i64(std::upper_bound(gstart.begin(), gstart.end(), s) - gstart.begin()) - 1; };
  auto work = [&](int lane) {
    sk_ctx* sub = lanes == 1 ? ctx : ctx->lanes[size_t(lane)];
    cudaSetDevice(ctx->device);
    sub->defer_d2h = defer ? 1 : 0;
    for (i64 s = lane; s < slices; s += lanes) {
      const PipelineOut::Basis* basis = nullptr;
      i64 g = -1;
      if (bk2) {
        g = group_of(s);
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return groups_ready > g || abort_k2 || worker_failed; });
        if (abort_k2 || worker_failed) break;
        lk.unlock();
        if (cudaStreamWaitEvent(sub->stream, gev[size_t(g)], 0) != cudaSuccess) {
          rcs[size_t(lane)] = SK_ERR_CUDA;
          errs[size_t(lane)] = "multislice: waiting on the batched nullspace failed";
          std::lock_guard<std::mutex> lk2(mu);
          worker_failed = true;
          cv.notify_all();
          break;
        }
        if (has_basis[size_t(s)]) basis = &bases[size_t(s)];
      }
      const int rc = estimate_impl(sub, ndim, calib_dims, center_offset, q, calib + s * ncal, full_dims, cfg,
                                   maps ? maps + s * q * nfull : nullptr, lambda ? lambda + s * nfull : nullptr,
                                   mask ? mask + s * nfull : nullptr, nullptr, prov ? prov + s : nullptr, nullptr,
                                   nullptr, nullptr, nullptr, nullptr, basis);
      if (bk2) {
        std::lock_guard<std::mutex> lk(mu);
        ++done[size_t(g)];
        cv.notify_all();
      }
      if (rc != SK_OK) {
        rcs[size_t(lane)] = rc;
        errs[size_t(lane)] = sk_last_error();
        if (bk2) {
          std::lock_guard<std::mutex> lk(mu);
          worker_failed = true;
          cv.notify_all();
        }
        break;
      }
    }
    sub->defer_d2h = 0;
    if (defer && sub->copy_stream && cudaStreamSynchronize(sub->copy_stream) != cudaSuccess &&
        rcs[size_t(lane)] == SK_OK) {
      rcs[size_t(lane)] = SK_ERR_CUDA;
      errs[size_t(lane)] = "multislice: deferred device-to-host copy failed";
    }
  };
  const auto t_start = std::chrono::steady_clock::now();
  // Group consumer (tail): one thread, one context, a whole group per pass.
  auto consume = [&]() {
    sk_ctx* sub = ctx->lanes[0];
    cudaSetDevice(ctx->device);
    sub->defer_d2h = 0;
    const Dims cod = dims_of(ndim, center_offset);
    for (i64 g = 0; g < groups; ++g) {
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return groups_ready > g || abort_k2 || worker_failed; });
        if (abort_k2 || worker_failed) break;
      }
      if (cudaStreamWaitEvent(sub->stream, gev[size_t(g)], 0) != cudaSuccess) {
        rcs[0] = SK_ERR_CUDA;
        errs[0] = "multislice: waiting on the batched nullspace failed";
        std::lock_guard<std::mutex> lk2(mu);
        worker_failed = true;
        cv.notify_all();
        break;
      }
      const i64 s0 = gstart[size_t(g)], gs = group_size(g);
      bool all = true;
      for (i64 i = 0; i < gs; ++i) all = all && has_basis[size_t(s0 + i)];
      int rc = SK_OK;
      if (all) {
        rc = guarded([&] {
          pipeline_group_tail(sub, cd, cod, q, gcal[size_t(g)], gs, &bases[size_t(s0)], fd, grid_t, cfg,
                              reinterpret_cast<float2*>(maps) + s0 * q * nfull, lambda + s0 * nfull, mask + s0 * nfull,
                              prov ? prov + s0 : nullptr);
        });
      } else {  // a slice missed the batched convergence test: this group slice by slice
        for (i64 i = 0; i < gs && rc == SK_OK; ++i) {
          const i64 sl = s0 + i;
          rc = estimate_impl(sub, ndim, calib_dims, center_offset, q, calib + sl * ncal, full_dims, cfg,
                             maps + sl * q * nfull, lambda + sl * nfull, mask + sl * nfull, nullptr,
                             prov ? prov + sl : nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                             has_basis[size_t(sl)] ? &bases[size_t(sl)] : nullptr);
        }
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        done[size_t(g)] = gs;
        cv.notify_all();
      }
      if (std::getenv("SKB_PROFILE_NS")) {
        float tail_ms = 0.f;
        cudaEventElapsedTime(&tail_ms, sub->ev[0], sub->ev[4]);
        std::fprintf(stderr, "[bk2] group %lld tail done at %.3f ms (device %.3f ms, %s)\n", (long long)g,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(),
                     tail_ms, all ? "batched" : "per slice");
      }
      if (rc != SK_OK) {
        rcs[0] = rc;
        errs[0] = sk_last_error();
        std::lock_guard<std::mutex> lk(mu);
        worker_failed = true;
        cv.notify_all();
        break;
      }
    }
  };
  // The batched K2 producer (calling thread): group g's Grams + bases into
  // buffer set g % 2, after the lanes finished group g - 2 with that set.
  std::string k2_err;
  auto produce = [&]() -> int {
    return guarded([&] {
      const Dims cdl = cd;
      const i64 nn = n_gram * n_gram;
      const double ratio = cfg->nullspace_threshold;
      for (i64 g = 0; g < groups; ++g) {
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return g < 2 || done[size_t(g - 2)] == group_size(g - 2) || worker_failed; });
          if (worker_failed) return;  // its error is reported below
        }
        const int set = int(g % 2);
        const i64 gs = group_size(g), s0 = gstart[size_t(g)];
        float2* grams = ctx->arena.get<float2>("bk:grams:" + std::to_string(set), G * nn);
        float2* cal_dev = nullptr;
        const bool cal_on_dev = is_device_ptr(calib);
        if (!cal_on_dev) {
          cal_dev = ctx->arena.get<float2>("bk:cal:" + std::to_string(set), G * ncal);
          SKB_CUDA(cudaMemcpyAsync(cal_dev, calib + s0 * ncal, size_t(gs * ncal) * sizeof(float2),
                                   cudaMemcpyHostToDevice, ctx->stream));
        }
        gcal[size_t(g)] = cal_on_dev ? reinterpret_cast<const float2*>(calib) + s0 * ncal : cal_dev;
        check_calib(cdl, q, sup);
        run_gram(ctx, cdl, q, gcal[size_t(g)], sup, grams, gs);  // K1 of the whole group: two launches
        if (std::getenv("SKB_PROFILE_NS")) {
          SKB_CUDA(cudaStreamSynchronize(ctx->stream));
          std::fprintf(stderr, "[bk2] group %lld Grams done at %.3f ms\n", (long long)g,
                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
        }
        // first batch of this size: one single-slice solve settles the step plan
        if (ctx->subspace_hint.find(n_gram) == ctx->subspace_hint.end())
          (void)run_nullspace(ctx, grams, n_gram, ratio, 2, false, false);
        std::vector<Eig> eg;
        std::vector<char> okv;
        run_eigh_subspace_batched(ctx, grams, gs, n_gram, ratio, set, eg, okv);
        for (i64 i = 0; i < gs; ++i) {
          if (!okv[size_t(i)]) continue;  // the lane runs this slice's own K1 + K2
          bases[size_t(s0 + i)].usig = eg[size_t(i)].usig;
          bases[size_t(s0 + i)].k = eg[size_t(i)].k;
          bases[size_t(s0 + i)].sigma1 = eg[size_t(i)].sigma1;
          has_basis[size_t(s0 + i)] = 1;
        }
        SKB_CUDA(cudaEventCreateWithFlags(&gev[size_t(g)], cudaEventDisableTiming));
        SKB_CUDA(cudaEventRecord(gev[size_t(g)], ctx->stream));
        if (std::getenv("SKB_PROFILE_NS")) {
          SKB_CUDA(cudaStreamSynchronize(ctx->stream));
          int nok = 0;
          for (char c : okv) nok += c;
          std::fprintf(stderr, "[bk2] group %lld ready at %.3f ms, %d/%lld batched\n", (long long)g,
                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(),
                       nok, (long long)gs);
        }
        {
          std::lock_guard<std::mutex> lk(mu);
          groups_ready = g + 1;
        }
        cv.notify_all();
      }
    });
  };
  int rc_k2 = SK_OK;
  if (lanes == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    cudaStream_t saved = nullptr;
    if (tail) {
      // the producer on a highest-priority stream for the duration of the call
      // (the caller's stream was synchronised above and is waited for below):
      // C3 54.3 -> 52.0 ms per call against the default priority
      const int rcp = guarded([&] {
        if (!ctx->hp_stream) {
          int least = 0, greatest = 0;
          SKB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
          SKB_CUDA(cudaStreamCreateWithPriority(&ctx->hp_stream, cudaStreamNonBlocking, greatest));
        }
        saved = ctx->stream;
        ctx->stream = ctx->hp_stream;
        check_cublas(cublasSetStream(ctx->cublas, ctx->stream), "cublasSetStream");
        check_cusolver(cusolverDnSetStream(ctx->cusolver, ctx->stream), "cusolverDnSetStream");
      });
      if (rcp != SK_OK) return rcp;
    }
    if (tail)
      pool.emplace_back(consume);
    else
      for (int l = 0; l < lanes; ++l) pool.emplace_back(work, l);
    if (bk2) {
      rc_k2 = produce();
      if (rc_k2 != SK_OK) {
        k2_err = g_last_error;
        std::lock_guard<std::mutex> lk(mu);
        abort_k2 = true;
        cv.notify_all();
      }
    }
    for (auto& t : pool) t.join();
    if (saved) {
      cudaStreamSynchronize(ctx->stream);
      ctx->stream = saved;
      cublasSetStream(ctx->cublas, ctx->stream);
      cusolverDnSetStream(ctx->cusolver, ctx->stream);
    }
  }
  for (auto& e : gev)
    if (e) cudaEventDestroy(e);
  if (bk2 && std::getenv("SKB_PROFILE_NS"))
    std::fprintf(stderr, "[bk2] all slices done at %.3f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  if (rc_k2 != SK_OK) {
    g_last_error = k2_err;
    return rc_k2;
  }
  for (int l = 0; l < lanes; ++l)
    if (rcs[size_t(l)] != SK_OK) {
      g_last_error = errs[size_t(l)];
      return rcs[size_t(l)];
    }
  return SK_OK;
}

}  // extern "C"
