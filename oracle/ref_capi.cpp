// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/sko.hpp for the rules).
//
// Flat C entry points over the UNMODIFIED reference library: this file is
// compiled together with /root/reference/proj/src/{types,kernels,fft,
// calibration,nullspace,spatial_gram,eigensolve,maps,memlog,parallel,
// synthetic,metrics,serialize}.cpp (oracle/Makefile.ref, output
// oracle/_ref/libsk_ref.so) against the Eigen-subset shim in
// oracle/ref_shim/.  It exports the same sko_* symbols, signatures and return
// codes as oracle/sko_capi.cpp (the FP64 restatement), so oracle/oracle.py can
// drive either library and the tests can compare them call for call.
// Return codes mirror senskit_main.cpp:23-27 (0 ok, 4 empty nullspace,
// 5 shape, 3 I/O, 6 length, 1 other).
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include <unsupported/Eigen/FFT>

#include "senskit/calibration.hpp"
#include "senskit/eigensolve.hpp"
#include "senskit/fft.hpp"
#include "senskit/kernels.hpp"
#include "senskit/maps.hpp"
#include "senskit/metrics.hpp"
#include "senskit/nullspace.hpp"
#include "senskit/parallel.hpp"
#include "senskit/spatial_gram.hpp"
#include "senskit/synthetic.hpp"
#include "senskit/types.hpp"

using namespace senskit;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const NullspaceEmptyError& e) {
    g_err = e.what();
    return 4;
  } catch (const DimError& e) {
    g_err = e.what();
    return 5;
  } catch (const IoError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::length_error& e) {
    g_err = e.what();
    return 6;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

Dims dims_of(int nd, const std::int64_t* d) { return Dims(d, d + nd); }
const Cx* cx(const double* p) { return reinterpret_cast<const Cx*>(p); }
Cx* cx(double* p) { return reinterpret_cast<Cx*>(p); }

template <class M> void put(const M& m, double* out) {
  if (!out) return;
  // Column-major copy (Eigen storage order), independent of the source stride.
  Cx* o = cx(out);
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = 0; i < m.rows(); ++i) o[i + j * m.rows()] = m(i, j);
}

CalibrationRegion make_calib(int nd, const std::int64_t* cdims, const std::int64_t* center_offset, std::int64_t q,
                             const double* data) {
  CalibrationRegion c;
  c.grid = ComplexImageStack(dims_of(nd, cdims), q, Domain::kspace);
  std::memcpy(c.grid.data.data(), data, std::size_t(c.grid.data.size()) * sizeof(Cx));
  c.center_offset = dims_of(nd, center_offset);
  return c;
}

GramField field_from(std::int64_t n, std::int64_t q, const double* buf) {
  GramField g;
  g.dims = {n};
  g.channels = q;
  g.values.resize(n * q * q);
  std::memcpy(g.values.data(), buf, std::size_t(n * q * q) * sizeof(Cx));
  return g;
}

}  // namespace

extern "C" {

struct sko_config {
  std::int32_t kernel, tau, gram;
  double nullspace_threshold;
  std::int32_t grid;
  std::int64_t grid_pad;
  std::int32_t eig, power_iters, method, field;
  double mask_threshold, apod_width;
};

const char* sko_last_error() { return g_err.c_str(); }

int sko_init(const char* lapack_path) {
  return guarded([&] {
    Eigen::shim::load(lapack_path);
    Eigen::shim::set_threads(1);  // Eigen without OpenMP: single-threaded dense algebra
  });
}
void sko_set_max_threads(int n) { set_max_threads(n); }
int sko_max_threads() { return max_threads(); }
void sko_set_lapack_threads(int n) { Eigen::shim::set_threads(n); }

int sko_make_support(int shape, int tau, int ndim, std::int32_t* offsets, std::int64_t* count) {
  return guarded([&] {
    const KernelSupport s = make_support(KernelShape(shape), tau, ndim);
    *count = s.size();
    if (offsets)
      for (Index i = 0; i < s.size(); ++i)
        for (Index a = 0; a < s.ndim(); ++a) offsets[i * s.ndim() + a] = s.offsets(i, a);
  });
}

int sko_extract_calibration(int nd, const std::int64_t* dims, std::int64_t q, const double* data,
                            const std::int64_t* size, double* out, std::int64_t* center_offset) {
  return guarded([&] {
    ComplexImageStack s(dims_of(nd, dims), q, Domain::kspace);
    std::memcpy(s.data.data(), data, std::size_t(s.data.size()) * sizeof(Cx));
    const CalibrationRegion c = extract_calibration(s, dims_of(nd, size));
    put(c.grid.data, out);
    for (int a = 0; a < nd; ++a) center_offset[a] = c.center_offset[std::size_t(a)];
  });
}

int sko_fft(int nd, const std::int64_t* dims, double* data, int op) {
  return guarded([&] {
    const Dims d = dims_of(nd, dims);
    Cx* p = cx(data);
    switch (op) {
      case 0: fft::transform_nd(p, d, -1); break;
      case 1: fft::transform_nd(p, d, +1); break;
      case 2: fft::fftshift_nd(p, d); break;
      case 3: fft::ifftshift_nd(p, d); break;
      case 4: fft::image_to_kspace(p, d); break;
      case 5: fft::kspace_to_image(p, d); break;
      case 6: fft::image_to_kspace_unitary(p, d); break;
      case 7: fft::kspace_to_image_unitary(p, d); break;
      default: throw DimError("unknown fft op");
    }
  });
}
void sko_fft_counters(std::int64_t* fwd, std::int64_t* inv) {
  *fwd = fft::forward_transforms();
  *inv = fft::inverse_transforms();
}
void sko_fft_reset_counters() { fft::reset_transform_counters(); }

int sko_gram(int method, int nd, const std::int64_t* cdims, const std::int64_t* center_offset, std::int64_t q,
             const double* calib, int shape, int tau, double* gram) {
  return guarded([&] {
    const CalibrationRegion c = make_calib(nd, cdims, center_offset, q, calib);
    const KernelSupport s = make_support(KernelShape(shape), tau, nd);
    const GramMatrix g = method == 1 ? gram_fft(c, s) : gram_explicit(build_calib_matrix(c, s));
    put(g.entries, gram);
  });
}

int sko_calib_matrix(int nd, const std::int64_t* cdims, std::int64_t q, const double* calib, int shape, int tau,
                     double* out, std::int64_t* rows, std::int64_t* cols) {
  return guarded([&] {
    std::vector<std::int64_t> co(static_cast<std::size_t>(nd), 0);
    const CalibrationRegion c = make_calib(nd, cdims, co.data(), q, calib);
    const CalibMatrix m = build_calib_matrix(c, make_support(KernelShape(shape), tau, nd));
    *rows = m.entries.rows();
    *cols = m.entries.cols();
    put(m.entries, out);
  });
}

int sko_extract_nullspace(std::int64_t n, const double* gram, double ratio, std::int64_t* rank, double* spectrum,
                          double* filters) {
  return guarded([&] {
    GramMatrix g;
    g.entries.resize(n, n);
    std::memcpy(g.entries.data(), gram, std::size_t(n * n) * sizeof(Cx));
    const NullspaceBasis b = extract_nullspace(g, ratio);
    *rank = b.rank();
    if (spectrum) std::memcpy(spectrum, b.spectrum.data(), std::size_t(b.spectrum.size()) * sizeof(double));
    put(b.filters, filters);
  });
}

int sko_aggregate_w(std::int64_t n, std::int64_t r, const double* filters, double* w) {
  return guarded([&] {
    NullspaceBasis b;
    b.filters.resize(n, r);
    std::memcpy(b.filters.data(), filters, std::size_t(n * r) * sizeof(Cx));
    put(aggregate_w(b).entries, w);
  });
}

int sko_gram_field_fast(std::int64_t q, const double* w, int shape, int tau, int nd, const std::int64_t* dims,
                        double* field) {
  return guarded([&] {
    const KernelSupport s = make_support(KernelShape(shape), tau, nd);
    AggregateW aw;
    aw.channels = q;
    aw.support_size = s.size();
    const Index n = q * s.size();
    aw.entries.resize(n, n);
    std::memcpy(aw.entries.data(), w, std::size_t(n * n) * sizeof(Cx));
    put(gram_field_fast(aw, s, dims_of(nd, dims)).values, field);
  });
}

int sko_gram_field_naive(std::int64_t q, std::int64_t r, const double* filters, int shape, int tau, int nd,
                         const std::int64_t* dims, double* field) {
  return guarded([&] {
    const KernelSupport s = make_support(KernelShape(shape), tau, nd);
    NullspaceBasis b;
    b.channels = q;
    b.support_size = s.size();
    b.filters.resize(q * s.size(), r);
    std::memcpy(b.filters.data(), filters, std::size_t(b.filters.size()) * sizeof(Cx));
    put(gram_field_naive(filter_field_naive(b, s, dims_of(nd, dims))).values, field);
  });
}

int sko_espirit_inplace(std::int64_t n, std::int64_t q, double* field, std::int64_t support_size) {
  return guarded([&] {
    GramField g = field_from(n, q, field);
    espirit_inplace(g, support_size);
    put(g.values, field);
  });
}

int sko_eig_power_field(std::int64_t n, std::int64_t q, const double* bfield, int iters, double* vectors,
                        double* values) {
  return guarded([&] {
    const GramField g = field_from(n, q, bfield);
    const EigenResult r = eig_power_field(g, iters);
    put(r.vectors, vectors);
    std::memcpy(values, r.values.data(), std::size_t(n) * sizeof(double));
  });
}

int sko_eig_dense_field(std::int64_t n, std::int64_t q, const double* field, int which, double* vectors,
                        double* values, double* second) {
  return guarded([&] {
    const GramField g = field_from(n, q, field);
    const EigenResult r = eig_dense_field(g, Extremal(which));
    put(r.vectors, vectors);
    std::memcpy(values, r.values.data(), std::size_t(n) * sizeof(double));
    if (second) std::memcpy(second, r.second_values.data(), std::size_t(n) * sizeof(double));
  });
}

int sko_normalize_maps(int nd, const std::int64_t* dims, std::int64_t q, const double* raw,
                       const std::int64_t* cdims, const std::int64_t* center_offset, const double* calib,
                       double apod_width, double* out, std::int64_t* zeroed) {
  return guarded([&] {
    ComplexImageStack r(dims_of(nd, dims), q, Domain::image);
    std::memcpy(r.data.data(), raw, std::size_t(r.data.size()) * sizeof(Cx));
    const CalibrationRegion c = make_calib(nd, cdims, center_offset, q, calib);
    auto [m, rec] = normalize_maps(r, c, apod_width);
    put(m.data, out);
    if (zeroed) *zeroed = rec.zeroed_voxels;
  });
}

int sko_interpolate_maps(int nd, const std::int64_t* low_dims, std::int64_t q, const double* low,
                         const std::int64_t* full_dims, double* out) {
  return guarded([&] {
    ComplexImageStack s(dims_of(nd, low_dims), q, Domain::image);
    std::memcpy(s.data.data(), low, std::size_t(s.data.size()) * sizeof(Cx));
    put(interpolate_maps(s, dims_of(nd, full_dims)).data, out);
  });
}

int sko_interpolate_real(int nd, const std::int64_t* low_dims, const double* low, const std::int64_t* full_dims,
                         double* out) {
  return guarded([&] {
    const Dims ld = dims_of(nd, low_dims);
    ArrayXd l(numel(ld));
    std::memcpy(l.data(), low, std::size_t(l.size()) * sizeof(double));
    const ArrayXd r = interpolate_real(l, ld, dims_of(nd, full_dims));
    std::memcpy(out, r.data(), std::size_t(r.size()) * sizeof(double));
  });
}

namespace {

PipelineConfig config_of(const sko_config* c) {
  PipelineConfig cfg;
  cfg.kernel = KernelShape(c->kernel);
  cfg.tau = c->tau;
  cfg.gram = GramMethod(c->gram);
  cfg.nullspace_threshold = c->nullspace_threshold;
  cfg.grid = GridMode(c->grid);
  cfg.grid_pad = c->grid_pad;
  cfg.eig = EigMethod(c->eig);
  cfg.power_iters = c->power_iters;
  cfg.method = MapMethod(c->method);
  cfg.field = FieldPath(c->field);
  cfg.mask_threshold = c->mask_threshold;
  cfg.apod_width = c->apod_width;
  return cfg;
}

// Samples taken inside the staged pipeline (for golden fixtures); all optional.
struct Samples {
  std::int64_t n_gram = 0;
  const std::int64_t* gram_idx = nullptr;  // (row, col) pairs
  double* gram_vals = nullptr;             // complex
  double* gram_fro = nullptr;              // ||Gram||_F
  std::int64_t n_field = 0;
  const std::int64_t* field_idx = nullptr;  // (voxel, row, col) triples
  double* field_vals = nullptr;             // complex
  double* field_fro = nullptr;              // ||G(x)||_F over the whole grid
};

// maps.cpp:265-330 with the same stage order; grid_override = explicit grid
// dims (pipeline::compute_field/finalize, maps.hpp:117-123).
void staged(const CalibrationRegion& c, const Dims& full, const PipelineConfig& cfg, const std::int64_t* grid_override,
            SensitivityResult& res, double* raw_maps, double* raw_lambda, double* gram_out, const Samples& smp) {
  using clock = std::chrono::steady_clock;
  auto el = [](clock::time_point a) { return std::chrono::duration<double>(clock::now() - a).count(); };
  const int nd = int(c.dims().size());
  c.grid.validate();
  if (full.size() != c.dims().size()) throw DimError("full_dims rank mismatch");
  for (std::size_t a = 0; a < full.size(); ++a)
    if (full[a] < c.dims()[a]) throw DimError("full_dims must be at least the calibration extent");
  const auto t0 = clock::now();
  Provenance prov;
  prov.config = cfg;
  const KernelSupport s = make_support(cfg.kernel, cfg.tau, nd);
  auto t = clock::now();
  const GramMatrix g = pipeline::compute_gram(c, s, cfg);
  prov.stages["gram"].seconds = el(t);
  put(g.entries, gram_out);
  if (smp.gram_fro) *smp.gram_fro = g.entries.norm();
  for (std::int64_t k = 0; k < smp.n_gram; ++k) {
    const Cx v = g.entries(smp.gram_idx[2 * k], smp.gram_idx[2 * k + 1]);
    smp.gram_vals[2 * k] = v.real();
    smp.gram_vals[2 * k + 1] = v.imag();
  }
  t = clock::now();
  const NullspaceBasis b = extract_nullspace(g, cfg.nullspace_threshold);
  prov.stages["nullspace"].seconds = el(t);
  prov.nullspace_rank = b.rank();
  prov.sigma1 = b.spectrum[0];
  prov.spectrum_normalized = singular_spectrum_report(b);
  const Dims grid = grid_override ? dims_of(nd, grid_override) : pipeline::grid_dims_for(c, full, cfg);
  prov.grid_dims = grid;
  t = clock::now();
  GramField f = pipeline::compute_field(b, s, grid, cfg);
  prov.stages["field"].seconds = el(t);
  if (smp.field_fro) *smp.field_fro = f.values.norm();
  const Index q = f.channels;
  for (std::int64_t k = 0; k < smp.n_field; ++k) {
    const Cx v = f.values[smp.field_idx[3 * k] * q * q + smp.field_idx[3 * k + 2] * q + smp.field_idx[3 * k + 1]];
    smp.field_vals[2 * k] = v.real();
    smp.field_vals[2 * k + 1] = v.imag();
  }
  t = clock::now();
  pipeline::RawMaps raw = pipeline::solve_field(std::move(f), s.size(), cfg);
  prov.stages["eigensolve"].seconds = el(t);
  put(raw.maps.data, raw_maps);
  if (raw_lambda) std::memcpy(raw_lambda, raw.lambda.data(), std::size_t(raw.lambda.size()) * sizeof(double));
  t = clock::now();
  res = pipeline::finalize(std::move(raw), c, full, cfg);
  prov.stages["post"].seconds = el(t);
  prov.total_seconds = el(t0);
  res.provenance = prov;
}

void export_result(const SensitivityResult& res, int nd, const Dims& full, double* maps, double* lambda,
                   std::uint8_t* mask, std::int64_t* grid_dims, std::int64_t* rank, double* sigma1, double* spectrum,
                   double* stage_seconds, std::int64_t* zeroed) {
  put(res.maps.data, maps);
  if (lambda)
    std::memcpy(lambda, res.lambda_min_map.data(), std::size_t(res.lambda_min_map.size()) * sizeof(double));
  if (mask) std::memcpy(mask, res.support_mask.data(), res.support_mask.size());
  if (grid_dims) {
    const Dims& gd = res.provenance.grid_dims.empty() ? full : res.provenance.grid_dims;
    for (int a = 0; a < nd; ++a) grid_dims[a] = gd[std::size_t(a)];
  }
  if (rank) *rank = res.provenance.nullspace_rank;
  if (sigma1) *sigma1 = res.provenance.sigma1;
  if (spectrum)
    std::memcpy(spectrum, res.provenance.spectrum_normalized.data(),
                std::size_t(res.provenance.spectrum_normalized.size()) * sizeof(double));
  if (stage_seconds) {
    const char* names[5] = {"gram", "nullspace", "field", "eigensolve", "post"};
    for (int i = 0; i < 5; ++i) {
      auto it = res.provenance.stages.find(names[i]);
      stage_seconds[i] = it == res.provenance.stages.end() ? 0.0 : it->second.seconds;
    }
  }
  if (zeroed) *zeroed = res.normalization.zeroed_voxels;
}

}  // namespace

int sko_estimate_maps(int nd, const std::int64_t* cdims, const std::int64_t* center_offset, std::int64_t q,
                      const double* calib, const std::int64_t* full_dims, const sko_config* cfgp,
                      const std::int64_t* grid_override, double* maps, double* lambda, std::uint8_t* mask,
                      std::int64_t* grid_dims, std::int64_t* rank, double* sigma1, double* spectrum,
                      double* stage_seconds, std::int64_t* zeroed, double* raw_maps, double* raw_lambda,
                      double* gram_out) {
  return guarded([&] {
    const PipelineConfig cfg = config_of(cfgp);
    const CalibrationRegion c = make_calib(nd, cdims, center_offset, q, calib);
    const Dims full = dims_of(nd, full_dims);
    SensitivityResult res;
    if (!grid_override && !raw_maps && !raw_lambda && !gram_out)
      res = estimate_maps(c, full, cfg);  // the reference entry point itself
    else
      staged(c, full, cfg, grid_override, res, raw_maps, raw_lambda, gram_out, Samples{});
    export_result(res, nd, full, maps, lambda, mask, grid_dims, rank, sigma1, spectrum, stage_seconds, zeroed);
  });
}

// Golden-fixture variant: the staged pipeline with Gram / G(x) sampled in
// place (no full-size copies of the 17 GB reference field) and the final maps,
// lambda and mask gathered at `n_vox` voxel indices (maps_s: Q x n_vox).
int skr_estimate_sampled(int nd, const std::int64_t* cdims, const std::int64_t* center_offset, std::int64_t q,
                         const double* calib, const std::int64_t* full_dims, const sko_config* cfgp,
                         const std::int64_t* grid_override, std::int64_t n_gram, const std::int64_t* gram_idx,
                         double* gram_vals, double* gram_fro, std::int64_t n_field, const std::int64_t* field_idx,
                         double* field_vals, double* field_fro, double* raw_lambda, std::int64_t n_vox,
                         const std::int64_t* vox_idx, double* maps_s, double* lambda_s, std::uint8_t* mask_s,
                         std::int64_t* grid_dims, std::int64_t* rank, double* sigma1, double* spectrum,
                         double* stage_seconds) {
  return guarded([&] {
    const PipelineConfig cfg = config_of(cfgp);
    const CalibrationRegion c = make_calib(nd, cdims, center_offset, q, calib);
    const Dims full = dims_of(nd, full_dims);
    Samples smp{n_gram, gram_idx, gram_vals, gram_fro, n_field, field_idx, field_vals, field_fro};
    SensitivityResult res;
    staged(c, full, cfg, grid_override, res, nullptr, raw_lambda, nullptr, smp);
    export_result(res, nd, full, nullptr, nullptr, nullptr, grid_dims, rank, sigma1, spectrum, stage_seconds,
                  nullptr);
    const Index nf = res.maps.voxels();
    for (std::int64_t k = 0; k < n_vox; ++k) {
      const Index j = vox_idx[k];
      for (Index ch = 0; ch < q; ++ch) {
        const Cx v = res.maps.data[ch * nf + j];
        maps_s[2 * (ch * n_vox + k)] = v.real();
        maps_s[2 * (ch * n_vox + k) + 1] = v.imag();
      }
      lambda_s[k] = res.lambda_min_map[j];
      mask_s[k] = res.support_mask[std::size_t(j)];
    }
  });
}

int sko_simulate(std::int64_t q, int nd, const std::int64_t* dims, int tau_gen, std::uint64_t seed, int kind,
                 double noise_sigma, std::uint64_t noise_seed, double* kspace, double* true_maps,
                 std::uint8_t* support_mask_true, double* phantom, double* gen_coeffs) {
  return guarded([&] {
    const SyntheticScene sc = make_scene(q, dims_of(nd, dims), tau_gen, seed, PhantomKind(kind));
    if (kspace) put(forward_kspace(sc, noise_sigma, noise_seed).data, kspace);
    put(sc.true_maps.data, true_maps);
    if (support_mask_true) std::memcpy(support_mask_true, sc.support_mask_true.data(), sc.support_mask_true.size());
    if (phantom) std::memcpy(phantom, sc.phantom.data(), std::size_t(sc.phantom.size()) * sizeof(double));
    put(sc.gen_coeffs, gen_coeffs);
  });
}

int sko_projection_residual(int nd, const std::int64_t* dims, std::int64_t q, const double* kspace,
                            const double* maps, double* out) {
  return guarded([&] {
    ComplexImageStack k(dims_of(nd, dims), q, Domain::kspace);
    std::memcpy(k.data.data(), kspace, std::size_t(k.data.size()) * sizeof(Cx));
    SensitivityResult m;
    m.maps = ComplexImageStack(dims_of(nd, dims), q, Domain::image);
    std::memcpy(m.maps.data.data(), maps, std::size_t(m.maps.data.size()) * sizeof(Cx));
    *out = projection_residual(k, m).value;
  });
}

}  // extern "C"
