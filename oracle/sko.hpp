// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A CPU, FP64 restatement of the reference `senskit` hot path
// (/root/reference/proj, read at survey time; the reference cannot be built
// here because Eigen3 and its vendored headers are absent — see DESIGN.md).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library, and only as the checker or the
// timed CPU baseline.  The product path (paper_2302_13431_b200) never links
// or calls it.
//
// Every function cites the reference file:line it restates.  Containers are
// Eigen-free but keep the reference layouts bit for bit:
//   * stacks: channel-major, row-major voxels, data[q*N + j]  (types.hpp:58-74)
//   * matrices: column-major (Eigen default)
//   * GramField: values[j*Q*Q + col*Q + row]                   (spatial_gram.hpp:36-51)
#pragma once

#include <complex>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace sko {

using Index = std::int64_t;
using Cx = std::complex<double>;
using Dims = std::vector<Index>;

// types.hpp:22-32
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DimError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NullspaceEmptyError : std::runtime_error { using std::runtime_error::runtime_error; };

Index numel(const Dims& dims);
std::vector<Index> strides_of(const Dims& dims);
bool next_index(std::vector<Index>& idx, const Dims& dims);
inline Index center_index(Index extent) { return extent / 2; }  // types.hpp:45
Dims centers_of(const Dims& dims);
inline double voxel_coord(Index j, Index extent) {  // types.hpp:52-54
  return double(j - center_index(extent)) / double(extent);
}

// Column-major dense complex matrix (Eigen::MatrixXcd stand-in).
struct Mat {
  Index rows = 0, cols = 0;
  std::vector<Cx> d;
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), d(std::size_t(r * c)) {}
  Cx& operator()(Index r, Index c) { return d[std::size_t(r + c * rows)]; }
  const Cx& operator()(Index r, Index c) const { return d[std::size_t(r + c * rows)]; }
};

enum class Domain { image = 0, kspace = 1 };

// types.hpp:58-74
struct Stack {
  Dims dims;
  Index channels = 0;
  Domain domain = Domain::image;
  std::vector<Cx> data;
  Stack() = default;
  Stack(Dims d, Index q, Domain dom);
  Index voxels() const { return numel(dims); }
  Cx* channel(Index q) { return data.data() + q * voxels(); }
  const Cx* channel(Index q) const { return data.data() + q * voxels(); }
  void validate() const;
};

// types.hpp:79-85
struct Calib {
  Stack grid;
  Dims center_offset;
  const Dims& dims() const { return grid.dims; }
  Index channels() const { return grid.channels; }
};

Calib extract_calibration(const Stack& stack, const Dims& size);  // types.cpp:58-90

// kernels.hpp:9-24
enum class KernelShape { rect = 0, ellipsoid = 1 };
struct Support {
  KernelShape shape = KernelShape::rect;
  int tau = 0;
  Index count = 0, nd = 0;
  std::vector<int> offsets;  // count x nd, row-major
  Index size() const { return count; }
  Index ndim() const { return nd; }
  int off(Index i, Index a) const { return offsets[std::size_t(i * nd + a)]; }
};
Support make_support(KernelShape shape, int tau, int ndim);  // kernels.cpp:7-35

// parallel.hpp:17-40 / parallel.cpp:11-18
void set_max_threads(int n);
int max_threads();
template <typename Fn>
void parallel_for(Index begin, Index end, Fn&& fn);

// fft.hpp / fft.cpp:37-112
namespace fft {
void transform_nd(Cx* data, const Dims& dims, int sign);
void fftshift_nd(Cx* data, const Dims& dims);
void ifftshift_nd(Cx* data, const Dims& dims);
void image_to_kspace(Cx* data, const Dims& dims);
void kspace_to_image(Cx* data, const Dims& dims);
void image_to_kspace_unitary(Cx* data, const Dims& dims);
void kspace_to_image_unitary(Cx* data, const Dims& dims);
std::int64_t forward_transforms();
std::int64_t inverse_transforms();
void reset_transform_counters();
}  // namespace fft

// calibration.hpp:16-42
struct CalibMatrix {
  Mat entries;
  Index valid_shifts = 0, channels = 0, support_size = 0;
};
enum class GramMethod { explicit_product = 0, fft = 1 };
struct GramMatrix {
  Mat entries;
  GramMethod method = GramMethod::explicit_product;
  Index channels = 0, support_size = 0;
};
CalibMatrix build_calib_matrix(const Calib& calib, const Support& support);
GramMatrix gram_explicit(const CalibMatrix& c);
GramMatrix gram_fft(const Calib& calib, const Support& support);

// nullspace.hpp:11-27
struct NullspaceBasis {
  Mat filters;                  // n x R
  std::vector<double> spectrum; // descending sigma, n
  double threshold_ratio = 0.05;
  Index channels = 0, support_size = 0;
  Index rank() const { return filters.cols; }
};
NullspaceBasis extract_nullspace(const GramMatrix& gram, double threshold_ratio = 0.05);
std::vector<double> singular_spectrum_report(const NullspaceBasis& basis);

// spatial_gram.hpp:13-73
struct FilterField {
  Dims dims;
  Index channels = 0, filters = 0;
  std::vector<Cx> values;  // plane (r,q) at ((r*Q)+q)*N
  Index voxels() const { return numel(dims); }
  const Cx* plane(Index r, Index q) const { return values.data() + (r * channels + q) * voxels(); }
};
struct AggregateW {
  Mat entries;
  Index channels = 0, support_size = 0;
};
struct GramField {
  Dims dims;
  Index channels = 0;
  std::vector<Cx> values;  // N*Q*Q, voxel-major, col-major per voxel
  Index voxels() const { return numel(dims); }
  Cx* at(Index j) { return values.data() + j * channels * channels; }
  const Cx* at(Index j) const { return values.data() + j * channels * channels; }
};
constexpr std::size_t kDefaultFieldByteCap = std::size_t(1) << 30;
FilterField filter_field_naive(const NullspaceBasis& basis, const Support& support, const Dims& dims,
                               std::size_t max_bytes = kDefaultFieldByteCap);
GramField gram_field_naive(const FilterField& field);
AggregateW aggregate_w(const NullspaceBasis& basis);
GramField gram_field_fast(const AggregateW& w, const Support& support, const Dims& dims);
void espirit_inplace(GramField& g, Index support_size);

// eigensolve.hpp:8-27
enum class Extremal { smallest = 0, largest = 1 };
struct EigenResult {
  Dims dims;
  Index channels = 0;
  Mat vectors;  // Q x N
  std::vector<double> values, second_values;
  int iterations_used = 0;
};
EigenResult eig_dense_field(const GramField& field, Extremal which);
EigenResult eig_power_field(const GramField& b_field, int iters = 10);

// maps.hpp:16-123
enum class GridMode { full = 0, reduced = 1 };
enum class EigMethod { dense = 0, power = 1 };
enum class MapMethod { nullspace = 0, espirit = 1 };
enum class FieldPath { naive = 0, fast = 1 };
struct PipelineConfig {
  KernelShape kernel = KernelShape::rect;
  int tau = 3;
  GramMethod gram = GramMethod::explicit_product;
  double nullspace_threshold = 0.05;
  GridMode grid = GridMode::full;
  Index grid_pad = 24;
  EigMethod eig = EigMethod::dense;
  int power_iters = 10;
  MapMethod method = MapMethod::nullspace;
  FieldPath field = FieldPath::fast;
  double mask_threshold = 0.01;
  double apod_width = -1.0;
  std::size_t field_byte_cap = kDefaultFieldByteCap;
  static PipelineConfig baseline();
  static PipelineConfig pisco();
};
struct NormalizationRecord {
  bool sos = false, phase_referenced = false, renormalized_after_interpolation = false;
  std::vector<double> apod_sigma;
  Index zeroed_voxels = 0;
};
struct Provenance {
  Dims calib_dims, full_dims, grid_dims;
  Index channels = 0, support_size = 0, valid_shifts = 0, nullspace_rank = 0;
  double sigma1 = 0.0;
  std::vector<double> spectrum_normalized;
  std::map<std::string, double> stages;  // seconds
  double total_seconds = 0.0;
};
struct SensitivityResult {
  Stack maps;
  std::vector<double> lambda_min_map;
  std::vector<std::uint8_t> support_mask;
  NormalizationRecord normalization;
  Provenance provenance;
};
struct RawMaps {
  Stack maps;
  std::vector<double> lambda;
};

Dims reduced_grid_dims(const Dims& calib_dims, Index pad, const Dims& full_dims);
std::vector<std::uint8_t> support_mask(const std::vector<double>& lambda, double thr);
Stack interpolate_maps(const Stack& lowres, const Dims& full_dims);
std::vector<double> interpolate_real(const std::vector<double>& lowres, const Dims& low_dims,
                                     const Dims& full_dims);
NormalizationRecord normalize_maps(const Stack& raw, const Calib& calib, double apod_width,
                                   Stack& out);
GramMatrix compute_gram(const Calib& calib, const Support& support, const PipelineConfig& cfg);
Dims grid_dims_for(const Calib& calib, const Dims& full_dims, const PipelineConfig& cfg);
GramField compute_field(const NullspaceBasis& basis, const Support& support, const Dims& grid,
                        const PipelineConfig& cfg);
RawMaps solve_field(GramField field, Index support_size, const PipelineConfig& cfg);
SensitivityResult finalize(RawMaps&& raw, const Calib& calib, const Dims& full_dims,
                           const PipelineConfig& cfg);
SensitivityResult estimate_maps(const Calib& calib, const Dims& full_dims, const PipelineConfig& cfg);

// synthetic.hpp:12-45 (reference generator; used for reference KATs)
enum class PhantomKind { disk = 0, rectangles = 1 };
struct SyntheticScene {
  Stack true_maps;
  std::vector<double> phantom;
  std::vector<std::uint8_t> support_mask_true;
  Dims dims;
  Index channels = 0;
  int tau_gen = 0;
  std::uint64_t seed = 0;
  Support gen_support;
  Mat gen_coeffs;
};
SyntheticScene make_scene(Index channels, const Dims& dims, int tau_gen, std::uint64_t seed,
                          PhantomKind kind);
Stack forward_kspace(const SyntheticScene& scene, double noise_sigma, std::uint64_t seed);

// metrics.hpp
double projection_residual(const Stack& kspace, const Stack& maps);
double gauge_aligned_max_difference(const Stack& a, const Stack& b);
double dice_coefficient(const std::vector<std::uint8_t>& a, const std::vector<std::uint8_t>& b);

// LAPACK / BLAS bridge (scipy's bundled OpenBLAS, LP64), loaded at runtime.
namespace lapack {
void load(const std::string& path);
bool loaded();
void set_threads(int n);
// Hermitian eigensolve, lower triangle, column-major in place; eigenvalues ascending.
void zheevd(Index n, Cx* a, double* w, bool vectors = true);
// C = alpha * op(A) * op(B) + beta * C, column-major.
void zgemm(char ta, char tb, Index m, Index n, Index k, Cx alpha, const Cx* a, Index lda,
           const Cx* b, Index ldb, Cx beta, Cx* c, Index ldc);
}  // namespace lapack

}  // namespace sko

#include "sko_parallel.inl"
