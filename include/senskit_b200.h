/* senskit_b200 — C-ABI drop-in for the reference `senskit` PISCO hot path.
 *
 * Every entry point replaces one reference C++ function (cited per
 * declaration, paths relative to the reference's proj/).  Plain pointers and
 * sizes only; no torch or CUDA types cross this boundary.
 *
 * Buffers: every array argument may be a HOST pointer (pageable or pinned) or
 * a DEVICE pointer on the context's GPU; the library detects which with
 * cudaPointerGetAttributes and copies as needed.  Complex arrays are
 * interleaved float32 (sk_c64), matching the reference's CStack v1 on-disk
 * format (io.hpp:9-16); layouts are the reference's:
 *   stacks      channel-major, row-major voxels:   data[q*N + j]   (types.hpp:58-74)
 *   matrices    column-major (Eigen default):      m[r + c*rows]
 *   GramField   voxel-major, column-major Q x Q:   v[j*Q*Q + c*Q + r] (spatial_gram.hpp:36-51)
 *
 * Every call is synchronous at return (the reference's calls block).  One
 * context per GPU; a context is not re-entrant.
 *
 * Return codes mirror the reference CLI contract (tools/senskit_main.cpp:23-27)
 * for the error classes the reference throws (types.hpp:22-32):
 */
#ifndef SENSKIT_B200_H
#define SENSKIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SK_OK = 0,
  SK_ERR_OTHER = 1,           /* std::runtime_error                                */
  SK_ERR_IO = 3,              /* IoError                                           */
  SK_ERR_NULLSPACE_EMPTY = 4, /* NullspaceEmptyError (nullspace.cpp:29-31)          */
  SK_ERR_DIM = 5,             /* DimError                                          */
  SK_ERR_LENGTH = 6,          /* std::length_error (field byte cap)                */
  SK_ERR_CUDA = 7,            /* CUDA / cuSOLVER / cuBLAS failure                  */
  SK_ERR_OOM = 8,             /* device allocation failed                          */
  SK_ERR_UNSUPPORTED = 9      /* configuration outside the B200 path */
};

typedef struct { float re, im; } sk_c64;
typedef struct sk_ctx sk_ctx;

/* PipelineConfig (maps.hpp:23-45).  Both presets run on the GPU: `pisco`
 * (gram = fft, eig = power) and `baseline` (gram = explicit, eig = dense,
 * method nullspace or espirit).  field = naive keeps the reference's contract
 * (SK_ERR_LENGTH when the R x Q x N filter field would exceed field_byte_cap)
 * and evaluates the same G(x) = sum_r H_r(x)^H H_r(x) through the lag
 * expansion of W = F F^H.
 * grid_dims: explicit map grid (all > 0) overrides grid/grid_pad, which is
 * how the reference drives anisotropic grids (pipeline::compute_field /
 * finalize with explicit dims, maps.hpp:115-123). */
typedef struct {
  int32_t kernel;             /* 0 rect, 1 ellipsoid        maps.hpp:24 */
  int32_t tau;                /*                            maps.hpp:25 */
  int32_t gram;               /* 0 explicit, 1 fft          maps.hpp:26 */
  double nullspace_threshold; /*                            maps.hpp:27 */
  int32_t grid;               /* 0 full, 1 reduced          maps.hpp:28 */
  int64_t grid_pad;           /*                            maps.hpp:29 */
  int32_t eig;                /* 0 dense, 1 power           maps.hpp:30 */
  int32_t power_iters;        /*                            maps.hpp:31 */
  int32_t method;             /* 0 nullspace, 1 espirit     maps.hpp:32 */
  int32_t field;              /* 0 naive, 1 fast            maps.hpp:33 */
  double mask_threshold;      /*                            maps.hpp:37 */
  double apod_width;          /*                            maps.hpp:40 */
  int64_t grid_dims[3];       /* explicit map grid or zeros */
  /* B200 extensions (zero = default):
   * eig_solver  nullspace eigensolve: 0 auto (block subspace iteration on the
   *             signal subspace unless spectrum_normalized is requested or
   *             n <= 512), 1 full cuSOLVER Xsyevd, 2 subspace.
   * certify     subspace solver only: prove R exact with one Cholesky of
   *             cut^2 I - G + 2 sigma_1^2 U U^H (falls back to the full solver
   *             if it fails). */
  int32_t eig_solver;
  int32_t certify;
  /* field_byte_cap (maps.hpp:41; 0 = kDefaultFieldByteCap = 1 GiB): the
   * naive path's R*Q*N*16-byte filter-field budget (spatial_gram.cpp:43-47). */
  int64_t field_byte_cap;
} sk_config;

/* Provenance (maps.hpp:55-73) with device-timed stages. */
typedef struct {
  int64_t grid_dims[3];
  int64_t support_size;
  int64_t valid_shifts;
  int64_t nullspace_rank;
  int64_t zeroed_voxels;
  double sigma1;
  double cut_margin;   /* min over sigma of |sigma/cut - 1|: how far R is from flipping */
  int32_t eig_solver_used; /* 1 full, 2 subspace */
  int32_t certified;       /* subspace: R proven exact by the Cholesky test */
  int32_t subspace_iterations;
  int32_t subspace_block;
  double stage_ms[5];  /* gram, nullspace, field, eigensolve, post (CUDA events) */
  double total_ms;     /* device time of the whole call */
} sk_provenance;

/* ------------------------------------------------------------- context */
int sk_create(int device, sk_ctx** out);
int sk_destroy(sk_ctx* ctx);
/* Use a caller-owned cudaStream_t (passed as void*); NULL restores the
 * context's own stream. */
int sk_set_stream(sk_ctx* ctx, void* stream);
const char* sk_last_error(void);
/* Kernels launched by this context since creation (our sm_100a kernels), and
 * cuSOLVER / cuBLAS calls made (the eigensolve and Hermitian rank-k update). */
int64_t sk_kernel_launches(const sk_ctx* ctx);
int64_t sk_library_calls(const sk_ctx* ctx);

/* ------------------------------------------------------ host utilities */
/* make_support (kernels.hpp:24, kernels.cpp:7-35): |Lambda| x ndim offsets,
 * row-major, lexicographic.  offsets may be NULL to query the count. */
int sk_make_support(int shape, int tau, int ndim, int32_t* offsets, int64_t* count);
/* reduced_grid_dims (maps.hpp:102, maps.cpp:39-45) */
int sk_reduced_grid_dims(int ndim, const int64_t* calib_dims, int64_t pad, const int64_t* full_dims,
                         int64_t* out);

/* ------------------------------------------------------- stage entry points */
/* gram_fft (calibration.hpp:42, calibration.cpp:80-144): calib Q x E^D
 * (channel-major; the pad grid origin holds sample 0 as in the reference);
 * gram: n x n column-major, n = Q*|Lambda|. */
int sk_gram_fft(sk_ctx* ctx, int ndim, const int64_t* calib_dims, int64_t channels, const sk_c64* calib,
                int shape, int tau, sk_c64* gram);

/* build_calib_matrix (calibration.hpp:32, calibration.cpp:30-68): cmat is
 * P x n column-major (P = prod(E - 2 tau) valid shifts, row-major shift
 * order; column q*|Lambda| + i); *rows = P.  cmat == NULL only reports P. */
int sk_build_calib_matrix(sk_ctx* ctx, int ndim, const int64_t* calib_dims, int64_t channels, const sk_c64* calib,
                          int shape, int tau, sk_c64* cmat, int64_t* rows);

/* gram_explicit (calibration.hpp:35, calibration.cpp:70-78): gram = C^H C
 * (n x n column-major, exactly Hermitian), accumulated in FP64. */
int sk_gram_explicit(sk_ctx* ctx, int64_t rows, int64_t n, const sk_c64* cmat, sk_c64* gram);

/* extract_nullspace (nullspace.hpp:24, nullspace.cpp:7-35): spectrum = all n
 * singular values, descending; filters (may be NULL) n x R column-major.
 * filters_capacity: number of columns the caller allocated (>= R or error). */
int sk_extract_nullspace(sk_ctx* ctx, int64_t n, const sk_c64* gram, double threshold_ratio, int64_t* rank,
                         double* spectrum, sk_c64* filters, int64_t filters_capacity);

/* aggregate_w (spatial_gram.hpp:61, spatial_gram.cpp:87-94): W = F F^H. */
int sk_aggregate_w(sk_ctx* ctx, int64_t n, int64_t rank, const sk_c64* filters, sk_c64* w);

/* gram_field_fast (spatial_gram.hpp:67, spatial_gram.cpp:96-148):
 * field: N x Q x Q GramField layout. */
int sk_gram_field_fast(sk_ctx* ctx, int64_t channels, const sk_c64* w, int shape, int tau, int ndim,
                       const int64_t* dims, sk_c64* field);

/* espirit_inplace (spatial_gram.hpp:73, spatial_gram.cpp:156-164). */
int sk_espirit_inplace(sk_ctx* ctx, int64_t voxels, int64_t channels, sk_c64* field, int64_t support_size);

/* eig_power_field (eigensolve.hpp:27, eigensolve.cpp:40-74): b_field in the
 * GramField layout; vectors Q x N (column per voxel); values = Re(v^H B v). */
int sk_eig_power_field(sk_ctx* ctx, int64_t voxels, int64_t channels, const sk_c64* b_field, int iters,
                       sk_c64* vectors, float* values);

/* eig_dense_field (eigensolve.hpp:21, eigensolve.cpp:9-38): field in the
 * GramField layout; largest = 0 selects Extremal::smallest.  vectors Q x N
 * (unit column per voxel), values = extremal eigenvalue, second_values = the
 * runner-up (each output may be NULL).  FP64 cyclic Jacobi per voxel. */
int sk_eig_dense_field(sk_ctx* ctx, int64_t voxels, int64_t channels, const sk_c64* field, int largest,
                       sk_c64* vectors, float* values, float* second_values);

/* normalize_maps (maps.hpp:92-94, maps.cpp:101-176). */
int sk_normalize_maps(sk_ctx* ctx, int ndim, const int64_t* dims, int64_t channels, const sk_c64* raw,
                      const int64_t* calib_dims, const int64_t* center_offset, const sk_c64* calib,
                      double apod_width, sk_c64* out, int64_t* zeroed_voxels);

/* interpolate_maps / interpolate_real (maps.hpp:98-99, maps.cpp:54-99). */
int sk_interpolate_maps(sk_ctx* ctx, int ndim, const int64_t* low_dims, int64_t channels, const sk_c64* low,
                        const int64_t* full_dims, sk_c64* out);
int sk_interpolate_real(sk_ctx* ctx, int ndim, const int64_t* low_dims, const float* low,
                        const int64_t* full_dims, float* out);

/* support_mask (maps.hpp:105, maps.cpp:47-52). */
int sk_support_mask(sk_ctx* ctx, int64_t voxels, const float* lambda, double mask_threshold, uint8_t* mask);

/* ------------------------------------------------------------- metrics */
/* projection_residual (metrics.hpp, metrics.cpp:11-49): sqrt(sum_j ||rho_j -
 * c_j c_j^H rho_j / ||c_j||^2||^2 / sum_j ||rho_j||^2) with rho the unitary
 * image of the k-space stack (channels x dims, channel-major) and c the maps
 * (same shape).  FP64 accumulation, deterministic. */
int sk_projection_residual(sk_ctx* ctx, int ndim, const int64_t* dims, int64_t channels, const sk_c64* kspace,
                           const sk_c64* maps, double* value);

/* ------------------------------------------------- z-slab sharding (§8e) */
/* pipeline::compute_field + solve_field + the per-voxel half of finalize
 * (maps.hpp:115-123, maps.cpp:195-230, 117-172) restricted to rows
 * [slab_begin, slab_end) of axis 0 of the map grid (grid_dims_for or
 * cfg->grid_dims): maps = Q x slab voxels (SoS-normalised, phase referenced,
 * not yet interpolated), lambda = slab voxels.  Every rank computes the same
 * Gram and nullspace (deterministic), so concatenating the slabs along axis 0
 * reproduces the map-grid result; interpolation then runs per channel subset
 * (sk_interpolate_maps) with the renormalisation split below. */
int sk_estimate_raw_slab(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                         int64_t channels, const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg,
                         int64_t slab_begin, int64_t slab_end, sk_c64* maps, float* lambda, sk_provenance* prov);

/* Multi-GPU z-slab sharding with one exchange step (north_star:
 * "broadcast the shared nullspace filters").  sk_signal_basis runs
 * compute_gram + extract_nullspace (maps.cpp:180-186, nullspace.cpp:7-35) and
 * returns the nullspace in its complement form: the k = n - R signal
 * eigenvectors U_sig (n x k column-major, interleaved complex128; W = F F^H =
 * I - U_sig U_sig^H), plus R, sigma_1 and the cut margin.  u_sig holds
 * n * kmax values (host or device); if k > kmax the call fails with
 * SK_ERR_DIM after setting *k.  sk_estimate_raw_slab_basis is
 * sk_estimate_raw_slab with that basis supplied (K1 and K2 skipped), so every
 * rank expands the SAME filters the root broadcast. */
int sk_signal_basis(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                    int64_t channels, const sk_c64* calib, const sk_config* cfg, int64_t kmax, double* u_sig,
                    int64_t* k, int64_t* rank, double* sigma1, double* cut_margin);
int sk_estimate_raw_slab_basis(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                               int64_t channels, const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg,
                               const double* u_sig, int64_t k, double sigma1, int64_t slab_begin, int64_t slab_end,
                               sk_c64* maps, float* lambda, sk_provenance* prov);
/* Renormalisation after interpolation (maps.cpp:236-258) split over channel
 * subsets: sos[j] += sum_c |maps[c][j]|^2; then maps[c][j] /= sqrt(sos[j])
 * where sos[j] > 0, with sos the sum over all subsets (an all-reduce). */
int sk_sos_accumulate(sk_ctx* ctx, int64_t voxels, int64_t channels, const sk_c64* maps, float* sos);
int sk_renormalize_sos(sk_ctx* ctx, int64_t voxels, int64_t channels, sk_c64* maps, const float* sos);

/* Test hook for the K2 Rayleigh-Ritz eigensolver (no reference counterpart;
 * the reference uses Eigen's SelfAdjointEigenSolver, nullspace.cpp:13):
 * h is an n x n Hermitian complex128 matrix, column-major, interleaved
 * (re, im) doubles, host memory; on return it holds the eigenvectors and w
 * the eigenvalues ascending.  n <= 64 uses the one-CTA kernel, larger n
 * cuSOLVER Jacobi. */
int sk_debug_small_eigh(sk_ctx* ctx, int64_t n, double* h, double* w);

/* Test hooks for the K2 block kernels (the reference's dense path has no
 * equivalent entry point; they expose the steps eigen_dense/orthonormalise
 * stand-ins run between subspace products, maps.cpp:151-175).
 * sk_debug_cholqr: x (n x b complex128, column-major) <- x R^{-1}, R the
 *   Cholesky factor of x^H x, `passes` times (CholQR / CholQR2).
 * sk_debug_cross_gram: out (b x b complex128, column-major) = x^H y
 *   (y == NULL: x^H x). */
int sk_debug_cholqr(sk_ctx* ctx, int64_t n, int64_t b, double* x, int passes);
int sk_debug_cross_gram(sk_ctx* ctx, int64_t n, int64_t b, const double* x, const double* y, double* out);

/* ----------------------------------------------------------- full pipeline */
/* estimate_maps (maps.hpp:85-86, maps.cpp:265-330).  Outputs on full_dims:
 * maps Q x N_full, lambda_min_map N_full, support_mask N_full (each may be
 * NULL).  spectrum_normalized (n = Q*|Lambda| values, may be NULL) and prov
 * (may be NULL) carry the Provenance fields. */
int sk_estimate_maps(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                     int64_t channels, const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg,
                     sk_c64* maps, float* lambda_min_map, uint8_t* support_mask, double* spectrum_normalized,
                     sk_provenance* prov);

/* Stage dumps for parity checks (any may be NULL): the Gram (n x n), the
 * grid-resolution G field (GramField layout), the raw power-iteration maps
 * (Q x N_grid) and lambda on the grid.  Same semantics as sk_estimate_maps. */
int sk_estimate_maps_debug(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                           int64_t channels, const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg,
                           sk_c64* maps, float* lambda_min_map, uint8_t* support_mask,
                           double* spectrum_normalized, sk_provenance* prov, sk_c64* gram_out,
                           sk_c64* field_out, sk_c64* raw_maps_out, float* raw_lambda_out);

/* Parity probe (test hook; the config-scale parity suite): estimate_maps on
 * exactly the path sk_estimate_maps runs (same solver selection: no spectrum,
 * so the subspace eigensolver), plus in-place samples of the intermediates:
 * gram_vals[k] = Gram(gram_idx[2k], gram_idx[2k+1]) (calibration.hpp:25-30,
 * column-major n x n), field_vals[k] = G_j(row, col) for (j, row, col) =
 * field_idx[3k..3k+2] (spatial_gram.hpp:36-51, hi + lo in FP64), their
 * Frobenius norms over the whole Gram / map grid, and the native-grid lambda
 * (RawMaps::lambda, maps.hpp:110-113).  Complex samples are interleaved
 * float64.  Any output may be NULL (then n_* must be 0 for the samples). */
int sk_estimate_maps_probe(sk_ctx* ctx, int ndim, const int64_t* calib_dims, const int64_t* center_offset,
                           int64_t channels, const sk_c64* calib, const int64_t* full_dims, const sk_config* cfg,
                           sk_c64* maps, float* lambda_min_map, uint8_t* support_mask, sk_provenance* prov,
                           int64_t n_gram, const int64_t* gram_idx, double* gram_vals, double* gram_fro,
                           int64_t n_field, const int64_t* field_idx, double* field_vals, double* field_fro,
                           float* raw_lambda);

/* Multislice: `slices` independent calibrations (slice-major, each
 * channel-major), one estimate_maps per slice on this GPU, outputs
 * slice-major.  prov may be NULL or an array of `slices` records. */
int sk_estimate_maps_batched(sk_ctx* ctx, int64_t slices, int ndim, const int64_t* calib_dims,
                             const int64_t* center_offset, int64_t channels, const sk_c64* calib,
                             const int64_t* full_dims, const sk_config* cfg, sk_c64* maps, float* lambda_min_map,
                             uint8_t* support_mask, sk_provenance* prov);

#ifdef __cplusplus
}
#endif

#endif /* SENSKIT_B200_H */
