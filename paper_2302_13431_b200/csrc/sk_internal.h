// Internal declarations shared by the host runtime (sk_runtime.cu) and the
// kernels.  Nothing here crosses the C-ABI boundary (include/senskit_b200.h).
#pragma once

#include <cuComplex.h>
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/senskit_b200.h"

// Device-side bounds/invariant checks: compiled in with -DSKB_CHECKED (a
// debug build of the library; the sanitizer is not available on the GPU pool).
#ifdef SKB_CHECKED
#include <cassert>
#define SKB_DCHECK(x) assert(x)
#else
#define SKB_DCHECK(x) ((void)0)
#endif

namespace skb {

// 3xTF32 split: x = hi + lo with hi = tf32(x), lo = tf32(x - hi).
#ifdef __CUDACC__
__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
  unsigned h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  unsigned l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - hi));
  lo = __uint_as_float(l);
}
#endif

using i64 = std::int64_t;
using Dims = std::vector<i64>;

// The residual planes of G(x) (lo = G - fl32(G), |lo| <= 2^-24 |G|) are kept
// as bf16 pairs: 8 significant bits of the residual leave G known to
// 2^-33 |G| per entry, far below the FP32 Gram's own ~1e-7, at half the
// bytes of an fp32 residual (K3 writes and K4 reads 12 instead of 16 bytes
// per packed entry).
using lo2 = __nv_bfloat162;
__host__ __device__ __forceinline__ lo2 lo_pack(double x, double y) {
  return __floats2bfloat162_rn(float(x), float(y));
}
__host__ __device__ __forceinline__ float2 lo_unpack(lo2 v) { return __bfloat1622float2(v); }

// Error classes mirror the reference's exceptions (types.hpp:22-32).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
void check_cublas(cublasStatus_t s, const char* what);
void check_cusolver(cusolverStatus_t s, const char* what);
#define SKB_CUDA(x) ::skb::check_cuda((x), #x)
#define SKB_LAUNCH(what) ::skb::check_cuda(cudaGetLastError(), what)
// Raise a kernel's dynamic shared-memory limit only when the request grows
// (cudaFuncSetAttribute is host work on every launch otherwise).
void set_smem_limit(const void* func, size_t bytes);

inline i64 numel(const Dims& d) {
  i64 n = 1;
  for (i64 e : d) n *= e;
  return n;
}
inline i64 center_index(i64 n) { return n / 2; }  // types.hpp:45

// ------------------------------------------------------------- kernel support
struct Support {
  int shape = 0, tau = 0, nd = 0;
  i64 count = 0;
  std::vector<int> offsets;  // count x nd
  int off(i64 i, int a) const { return offsets[size_t(i * nd + a)]; }
};
Support make_support(int shape, int tau, int ndim);  // kernels.cpp:7-35

// ---------------------------------------------------------------- workspace
// Grow-only device buffers keyed by name; a context owns one arena.
class Arena {
 public:
  ~Arena();
  void* get(const std::string& name, size_t bytes);
  template <typename T>
  T* get(const std::string& name, i64 count) {
    return static_cast<T*>(get(name, size_t(count) * sizeof(T)));
  }
  void release_all();
  // Bumped whenever an existing slot is freed (grown or released): captured
  // CUDA graphs that baked in arena pointers are stale after a bump.
  uint64_t generation() const { return generation_; }

 private:
  uint64_t generation_ = 0;
  struct Slot {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Slot> slots_;
};

// Small complex matrices (DFT / sinc / apodised DFT) for the separable
// transforms, built in FP64 on the host and cached on the device.
struct MatrixCache {
  std::map<std::string, float2*> mats;
  ~MatrixCache();
};

// Key of a captured subspace round (run_eigh_subspace): sizes, plan, the
// arena pointers it touches and the threshold it bakes in.
struct RoundKey {
  i64 n, b;
  int q;
  const void *v, *y, *t, *h, *w, *res, *info, *a, *gram;
  double ratio;
  bool operator<(const RoundKey& o) const {
    return std::tie(n, b, q, v, y, t, h, w, res, info, a, gram, ratio) <
           std::tie(o.n, o.b, o.q, o.v, o.y, o.t, o.h, o.w, o.res, o.info, o.a, o.gram, o.ratio);
  }
};
// Cached device index tables per (support, q), owned by the context.
struct SupportTables {
  int2* pairs = nullptr;  // h entries (p <= q)
  int* off = nullptr;     // lam: box index of n_s relative to lag 0
  int* lag_ptr = nullptr; // nbox + 1
  int* lag_st = nullptr;  // lam^2 packed (s | t << 16), grouped by lag n_t - n_s
  int nbox = 0, lb = 0;
};

struct RoundGraph {
  cudaGraphExec_t exec = nullptr;
  int seen = 0;
  bool bad = false;
  double2 *v = nullptr, *y = nullptr, *t = nullptr;  // V / Y / T after the round
  int64_t launches = 0, lib_calls = 0;
};

}  // namespace skb

struct sk_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cublasHandle_t cublas = nullptr;
  cusolverDnHandle_t cusolver = nullptr;
  cusolverDnParams_t cusolver_params = nullptr;
  skb::Arena arena;
  skb::MatrixCache matrices;
  std::map<std::string, void*> tables;  // cached index tables (device)
  std::map<std::string, skb::SupportTables> support_tables;  // per (support, q)
  uint64_t rounds_generation = 0;       // arena generation the captured rounds were built against
  int64_t launches = 0;   // our kernels
  int64_t lib_calls = 0;  // cuSOLVER / cuBLAS calls
  cudaEvent_t ev[8] = {};
  // subspace solver hints per Gram size: signal count, orthogonalised steps
  // planned before the first Rayleigh-Ritz check, and the largest plan that
  // once needed an extra round (never planned again)
  struct SubspaceHint {
    int64_t m = 0;
    int plan = 3;
    int failed_plan = 0;
  };
  std::map<int64_t, SubspaceHint> subspace_hint;
  syevjInfo_t syevj = nullptr;
  // pinned host staging for the subspace solver's per-round convergence data
  // (one device-to-host copy of w, residuals and info instead of three)
  double* hpin = nullptr;
  size_t hpin_cap = 0;
  // concurrent lanes for multislice batches (sub-contexts on the same device)
  std::vector<sk_ctx*> lanes;
  // arena slots zeroed once at allocation (kernel-maintained counters)
  std::map<std::string, void*> arena_zeroed;
  // (n, b) sizes whose round already ran eagerly (buffers allocated): a new
  // step plan for such a size is captured on first sight
  std::set<std::pair<int64_t, int64_t>> warm_rounds;
  // captured subspace rounds (CUDA graphs), see run_graphed
  std::map<skb::RoundKey, skb::RoundGraph> rounds;
  // chunked K4 + overlapped device->host copies of the maps (pinned host outputs)
  cudaStream_t copy_stream = nullptr;
  // multislice with the grouped tail: the batched K1 + K2 producer runs on a
  // highest-priority stream so its short latency-bound kernels are scheduled
  // ahead of the consumer's large K3-K5 launches
  cudaStream_t hp_stream = nullptr;
  cudaEvent_t chunk_ev[9] = {};
  // multislice lanes: host outputs copied on copy_stream behind the pipeline
  // (double-buffered staging), drained by the batched driver
  int defer_d2h = 0;
  int d2h_slot = 0;
  cudaEvent_t d2h_done[2] = {};
  cudaEvent_t d2h_ready = nullptr;
};

namespace skb {

// ----------------------------------------------------------- kernel wrappers
// Separable "apply a small matrix along one axis":
//   out[b][j][i] = sum_a M[j][a] * in[b][a][i],  M is N x L (row-major, c64).
void apply_axis(sk_ctx* ctx, const float2* in, float2* out, const float2* M, i64 batch, int L, int N, i64 inner);
// Both axes of a 2-D separable transform in one CTA per batch item (M0: P0 x E0,
// M1: P1 x E1, row-major); for shared-memory-sized problems (sep2d_smem).
size_t sep2d_smem(int E0, int E1, int P0, int P1);
void sep2d(sk_ctx* ctx, const float2* in, float2* out, i64 batch, int E0, int E1, int P0, int P1, const float2* M0,
           const float2* M1);
// Symmetric-tap centred DFT (taps l = -H..H): cs[j][l-1] = (cos, sign*sin)(2 pi l (j - j0)/N).
void apply_axis_symdft(sk_ctx* ctx, const float2* in, float2* out, const float2* cs, i64 batch, int H, int N,
                       i64 inner);

// K1: pairwise correlation on the lag box + Gram assembly (calibration.cpp:111-142).
struct GramGeom {
  int nd;
  int pad[3];      // pad grid extents
  int lb;          // lag box extent per axis (4*tau + 1)
  int tau;
  int q;           // channels
  int lam;         // |Lambda|
  int stage_prod;  // set by the launcher: stage conj(S_p) S_q in shared memory
};
size_t gram_pairs_smem(const GramGeom& g);
void gram_pairs_launch(sk_ctx* ctx, const float2* spectra, const GramGeom& g, const int2* d_pairs, int npairs,
                       const int* d_off, const float2* d_tw, float2* gram, int slices = 1);

// Fold W (or I - U U^H) into per-pair lag kernels on the lag box
// (spatial_gram.cpp:108-131).  w_is_signal: W = I - w (w = U_sig U_sig^H,
// lower triangle valid) else W = w (full matrix).
void fold_lags_f64(sk_ctx* ctx, const double2* w, i64 n, int npairs, int lam, int nbox, const int2* d_pairs,
                   const int* d_lag_ptr, const int* d_lag_st, bool w_is_signal, double2* lags);
// Same fold for W = I - U U^H straight from the n x k signal basis U (no n x n
// product); shared memory lam * (lam + 1) * 16 bytes per pair.
// W = F F^H (c64, n x r filters, both triangles written; standalone aggregate_w)
void herk_full(sk_ctx* ctx, const float2* f, i64 n, i64 r, float2* w);
// signal-space fold by the correlation theorem on the lag box (no n x n W, no library call)
size_t spectral_fold_smem(int nd, int tau, int k, int q);
// A group of slices for the spectral fold (passed by value as a kernel parameter).
constexpr int kFoldBatchMax = 32;
struct FoldBatch {
  const double2* u[kFoldBatchMax];  // device, n x k_i signal bases
  int k[kFoldBatchMax];
};
void fold_lags_spectral_batched(sk_ctx* ctx, const FoldBatch& fb, int slices, i64 n, int q, int lam, int nd, int tau,
                                const int* d_offs, double2* lags);
void fold_lags_spectral(sk_ctx* ctx, const double2* u, i64 n, int k, int q, int lam, int nd, int tau,
                        const int* d_offs, double2* lags);
void fold_lags_f32(sk_ctx* ctx, const float2* w, i64 n, int npairs, int lam, int nbox, const int2* d_pairs,
                   const int* d_lag_ptr, const int* d_lag_st, double2* lags);
// One FP64 stage of the G(x) lag expansion (sk_expand.cu): in [batch][2H+1][inner]
// -> out [batch][N][inner]; final stage writes the fp32 hi/lo pair (out64 == nullptr).
// jc: row of the grid centre relative to the first output row (the table
// cs starts at that row; used to pair mirrored rows).
void expand_stage_f64(sk_ctx* ctx, const double2* in, i64 batch, i64 inner, int H, int N, int jc, const double2* cs,
                      double2* out64, float2* hi, lo2* lo);

// K4: batched per-voxel power iteration over packed Hermitian planes
// [h][N] (h = Q(Q+1)/2, plane (p<=q) holds M(row p, col q)).
// Iterates v <- (alpha v + beta M v) / ||.||; reports mv = Re(v^H M v).
// Optional epilogue (recon != nullptr): SoS normalisation + phase reference
// against recon [Q][N] (maps.cpp:117-172), zeroed voxel count, mask.
struct PowerArgs {
  const float2* planes;
  const lo2* planes_lo;     // nullable: bf16 residual G - hi, used only in the final Rayleigh quotient
  i64 n;            // voxels
  int q;            // channels
  int iters;
  float alpha, beta;
  float lam_scale;  // lambda = mv * lam_scale
  const float2* recon;   // nullable
  float2* maps;          // [Q][N]
  float* lambda;         // [N] (lambda = mv*lam_scale) nullable
  float* value;          // [N] alpha + beta*mv (B-form Rayleigh) nullable
  uint8_t* mask;         // nullable
  float mask_threshold;
  unsigned long long* zeroed;  // nullable
  // > 0: a voxel whose FP32 Rayleigh quotient on hi gives mv * lam_scale >= rq32_min
  // keeps it and skips the FP64 (hi + lo) evaluation (pipeline: ||G/|Lambda| || <= 1,
  // so FP32 rounding is ~1e-7 absolute; the FP64 pass is for small lambda)
  float rq32_min;
  // > 0: stride of planes / recon / maps (the pointers address voxel n0 of a
  // larger grid of ld voxels; n voxels are processed).  0: ld = n.
  i64 ld;
  // > 1: a stack of independent slices in one launch (multislice groups):
  // planes [slices][h][ld], recon / maps [slices][Q][ld], lambda / value / mask
  // [slices][ld], zeroed [slices]; n voxels per slice.  0 / 1: one slice.
  int slices;
};
void power_iteration(sk_ctx* ctx, const PowerArgs& a);
// More than 64 channels (sk_power_wide.cu): one CTA per voxel, the packed
// triangle in shared memory; power_iteration dispatches to it.
void power_iteration_wide(sk_ctx* ctx, const PowerArgs& a);
int power_wide_max_q();

// Baseline preset (sk_dense.cu).
// build_calib_matrix (calibration.cpp:30-68): P x Q|Lambda| column-major, FP64.
void calib_matrix(sk_ctx* ctx, const float2* calib, const Dims& cdims, int q, const Support& s, const int* d_off,
                  double2* c);
// gram_explicit (calibration.cpp:70-78): lower <- C^H C (ZHERK), gram <- full Hermitian c64.
void gram_explicit_dev(sk_ctx* ctx, const double2* c, i64 rows, i64 n, double2* lower, float2* gram);
// eig_dense_field (eigensolve.cpp:9-38) on packed planes: per voxel the extremal
// eigenpair of B = alpha I + beta (hi + lo) by FP64 cyclic Jacobi.
struct DenseEigArgs {
  const float2* planes;
  const lo2* planes_lo;     // nullable
  i64 n;
  int q;
  int largest;              // 1: largest (ESPIRiT), 0: smallest (nullspace method)
  double alpha, beta;
  float2* vec;              // [Q][N] unit eigenvectors
  float* value;             // [N] nullable
  float* second;            // [N] runner-up eigenvalue, nullable
  float* lambda;            // [N] lam_add + lam_mul * value, nullable
  uint8_t* mask;            // [N] lambda < mask_threshold, nullable
  double lam_add, lam_mul;
  float mask_threshold;
};
void dense_eig(sk_ctx* ctx, const DenseEigArgs& a);

// Conversions / small elementwise kernels.
void c64_to_c128(sk_ctx* ctx, const float2* in, double2* out, i64 n);
void c128_to_c64(sk_ctx* ctx, const double2* in, float2* out, i64 n);
void field_full_to_planes(sk_ctx* ctx, const float2* field, i64 n, int q, float2* planes);
void planes_to_field_full(sk_ctx* ctx, const float2* planes, const lo2* planes_lo, i64 n, int q, float2* field);
void espirit_field(sk_ctx* ctx, float2* field, i64 n, int q, float inv_lam);
void renormalize_and_mask(sk_ctx* ctx, float2* maps, i64 n, int q, const float2* lambda_c, float* lambda,
                          uint8_t* mask, float thr);
void mask_kernel(sk_ctx* ctx, const float* lambda, i64 n, float thr, uint8_t* mask);
void sos_accumulate(sk_ctx* ctx, const float2* maps, i64 n, int q, float* sos);   // sos += sum_c |maps_c|^2
// projection_residual value (metrics.cpp:11-49) from the unitary image and the maps (synchronous).
double projection_residual_value(sk_ctx* ctx, const float2* img, const float2* maps, i64 n, int q);
// parity probe (sk_estimate_maps_probe): gathers + Frobenius sums, FP64
void probe_gather_gram(sk_ctx* ctx, const float2* gram, i64 n, const long long* idx, i64 k, double2* out);
void probe_gather_field(sk_ctx* ctx, const float2* hi, const lo2* lo, i64 nvox, int q, const long long* idx,
                        i64 k, double2* out);
double probe_sumsq(sk_ctx* ctx, const float2* a, const lo2* lo, i64 total, i64 plane_len, int q);
// Centred transform along one axis (fft.cpp kspace_to_image / image_to_kspace):
// out = fftshift(DFT(ifftshift(in))) * scale, inverse = conjugate kernel.
// Returns false (nothing launched) unless N and inner are powers of two.
bool centered_fft_axis(sk_ctx* ctx, const void* in, void* out, i64 batch, int N, i64 inner, bool inverse,
                       double scale);
void renorm_with_sos(sk_ctx* ctx, float2* maps, i64 n, int q, const float* sos);  // maps /= sqrt(sos) where > 0
void real_to_c64(sk_ctx* ctx, const float* in, float2* out, i64 n);
void real_to_c128(sk_ctx* ctx, const float* in, double2* out, i64 n);
void lam64_to_f32_mask(sk_ctx* ctx, const double2* lam_c, i64 n, float* lam, uint8_t* mask, float thr);
// Periodic-sinc interpolation along one axis by shared-memory radix-2 FFTs
// (sk_interp.cu): in [batch][n][inner] -> out [batch][N][inner], float2 or
// double2 elements.  Returns false (nothing launched) unless n, N are powers
// of two with 2 <= n <= N <= 1024.
bool interp_axis_fft(sk_ctx* ctx, const void* in, void* out, i64 batch, int n, int N, i64 inner, bool fp64);
// Last (innermost, factor-2) interpolation pass of a [Q][P][n] stack fused with
// the per-voxel sum-of-squares renormalisation; false (nothing launched) when
// the shape is outside the kernel (Q a power of two <= 32, Q*n <= 4096).
bool interp_last_axis_sos(sk_ctx* ctx, const float2* in, float2* out, int q, i64 positions, int n, int N, int slices = 1);
void copy_strided(sk_ctx* ctx, const float2* src, i64 src_rs, i64 src_cs, float2* dst, i64 dst_rs, i64 dst_cs, i64 rows,
                  i64 cols);
void normalize_standalone(sk_ctx* ctx, float2* maps, i64 n, int q, const float2* recon, unsigned long long* zeroed);

// Subspace eigensolver helpers (FP64).
// 3xTF32 tensor-core products for K2's steering steps (sk_misc.cu): the complex
// Gram as real [Re; Im] hi/lo (2n x n), the block as [Re, Im] hi/lo (n x 2m),
// and the recombination of C = [Re; Im] [Re, Im] into the complex product.
// Batched forms (multislice K2): `batch` slices at strides s* (elements) in one launch.
void promote_split_gram(sk_ctx* ctx, const float2* a, i64 n, double2* a64, float* hi, float* lo, i64 batch = 1,
                        i64 sa = 0, i64 sh = 0);
// Batched Gauss-3M FP64 products on real planes (sk_misc.cu).
void promote_split3_gram(sk_ctx* ctx, const float2* a, i64 n, double* a3, float* hi, float* lo, i64 batch, i64 sa,
                         i64 sh);
void split3_block(sk_ctx* ctx, const double2* v, i64 len, double* v3, i64 batch, i64 sv);
void combine3_block(sk_ctx* ctx, const double* t3, i64 len, double2* y, i64 batch, i64 sy);
void split_block_cat_tf32(sk_ctx* ctx, const double2* v, i64 n, i64 m, float* vc, i64 batch = 1, i64 sv = 0,
                          i64 svc = 0);
void combine_block_cat(sk_ctx* ctx, const float* c, i64 n, i64 m, double2* y, i64 batch = 1, i64 sc = 0, i64 sy = 0);
void random_block(sk_ctx* ctx, double2* v, i64 n, i64 cols, i64 col0, unsigned int seed, i64 batch = 1, i64 sv = 0);
void ritz_residuals(sk_ctx* ctx, const double2* y, const double2* v, const double* theta, i64 n, i64 cols,
                    double* res, i64 batch = 1, i64 sb = 0, i64 sw = 0);
void shift_negate(sk_ctx* ctx, const double2* a, double2* m, i64 n, double shift);
void cross_gram(sk_ctx* ctx, const double2* x, const double2* y, i64 n, int b, double2* out);
// b = 64 block kernels (sk_cholqr.cu): X^H Y (X^H X when y == x) into a
// 64 x 64 column-major matrix, and `passes` CholQR passes X <- X L^{-H}
// (one-CTA Cholesky; a non-positive pivot raises *flag).
void gram64(sk_ctx* ctx, const double2* x, const double2* y, i64 n, double2* out, i64 batch = 1, i64 sx = 0);
// flag: per-slice int at flag[3 * slice] (the nullspace info triple's flag slot)
// CatIO (3xTF32 steering steps): the CholQR kernels can take their input block
// straight from the K-concatenated GEMM result C' (ccat, 2n x 4b floats per
// slice: Y = C'[:, :2b] + C'[:, 2b:] combined on load) instead of a formed
// c128 block, and the solve can write, beside the c128 result, its 3xTF32
// split operand V' for the next step's GEMM (vcat) -- the separate combine
// and split passes of a steering step disappear.
struct CatIO {
  const float* ccat = nullptr;  // first pass loads from it (x is then output only)
  i64 sc = 0;                   // slice stride of ccat (floats)
  float* vcat = nullptr;        // last pass also writes the split block here
  i64 svc = 0;                  // slice stride of vcat (floats)
};
void cholqr64(sk_ctx* ctx, double2* x, i64 n, int passes, int* flag, i64 batch = 1, i64 sx = 0,
              const CatIO& io = CatIO());
// the same kernels at block width b in {32, 64} (single slice)
void gram_blk(sk_ctx* ctx, int b, const double2* x, const double2* y, i64 n, double2* out);
void cholqr_b(sk_ctx* ctx, int b, double2* x, i64 n, int passes, int* flag, const CatIO& io = CatIO());
// One-CTA Hermitian eigensolver (sk_eig.cu) for b <= 64: eigenvalues ascending
// into w, eigenvectors overwrite H (column-major); info[0] = 1 on a
// non-finite result.  Returns false (nothing launched) for larger b.
// Clusters of close eigenvalues lying entirely below floor_rel * ||H|| are
// only orthonormalised, not refined to individual eigenvectors.
// batch: H [batch][n][n], w [batch][n], info[3 * slice]
bool herm_eig_small(sk_ctx* ctx, double2* H, int n, double* w, int* info, double floor_rel = 0.0, int batch = 1);

}  // namespace skb
