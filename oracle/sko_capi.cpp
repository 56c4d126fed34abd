// ORACLE — TEST INFRASTRUCTURE ONLY (see sko.hpp).
//
// Flat C entry points over the FP64 restatement, for ctypes (tests/ and
// bench.py's CPU-baseline leg).  Complex buffers are interleaved float64
// (re, im) with the reference layouts.  Return codes mirror the reference
// CLI contract (senskit_main.cpp:23-27): 0 ok, 4 empty nullspace, 5 shape,
// 3 I/O, 6 length (field byte cap), 1 anything else.
#include <chrono>
#include <cstring>
#include <string>

#include "sko.hpp"

using namespace sko;

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

Calib make_calib(int nd, const std::int64_t* cdims, const std::int64_t* center_offset, std::int64_t q,
                 const double* data) {
  Calib c;
  c.grid = Stack(dims_of(nd, cdims), q, Domain::kspace);
  std::memcpy(c.grid.data.data(), data, c.grid.data.size() * sizeof(Cx));
  c.center_offset = dims_of(nd, center_offset);
  return c;
}

void put(const std::vector<Cx>& v, double* out) {
  if (out) std::memcpy(out, v.data(), v.size() * sizeof(Cx));
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
  return guarded([&] { lapack::load(lapack_path); });
}
void sko_set_max_threads(int n) { set_max_threads(n); }
int sko_max_threads() { return max_threads(); }
void sko_set_lapack_threads(int n) { lapack::set_threads(n); }

int sko_make_support(int shape, int tau, int ndim, std::int32_t* offsets, std::int64_t* count) {
  return guarded([&] {
    const Support s = make_support(KernelShape(shape), tau, ndim);
    *count = s.count;
    if (offsets)
      for (std::size_t i = 0; i < s.offsets.size(); ++i) offsets[i] = s.offsets[i];
  });
}

int sko_extract_calibration(int nd, const std::int64_t* dims, std::int64_t q, const double* data,
                            const std::int64_t* size, double* out, std::int64_t* center_offset) {
  return guarded([&] {
    Stack s(dims_of(nd, dims), q, Domain::kspace);
    std::memcpy(s.data.data(), data, s.data.size() * sizeof(Cx));
    const Calib c = extract_calibration(s, dims_of(nd, size));
    put(c.grid.data, out);
    for (int a = 0; a < nd; ++a) center_offset[a] = c.center_offset[std::size_t(a)];
  });
}

// op: 0 transform(-1), 1 transform(+1), 2 fftshift, 3 ifftshift, 4 image_to_kspace,
//     5 kspace_to_image, 6 image_to_kspace_unitary, 7 kspace_to_image_unitary
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

// method: 0 explicit (C^H C over valid shifts), 1 fft (gram_fft)
int sko_gram(int method, int nd, const std::int64_t* cdims, const std::int64_t* center_offset,
             std::int64_t q, const double* calib, int shape, int tau, double* gram) {
  return guarded([&] {
    const Calib c = make_calib(nd, cdims, center_offset, q, calib);
    const Support s = make_support(KernelShape(shape), tau, nd);
    const GramMatrix g = method == 1 ? gram_fft(c, s) : gram_explicit(build_calib_matrix(c, s));
    put(g.entries.d, gram);
  });
}

int sko_calib_matrix(int nd, const std::int64_t* cdims, std::int64_t q, const double* calib, int shape,
                     int tau, double* out, std::int64_t* rows, std::int64_t* cols) {
  return guarded([&] {
    std::vector<std::int64_t> co(static_cast<std::size_t>(nd), 0);
    const Calib c = make_calib(nd, cdims, co.data(), q, calib);
    const CalibMatrix m = build_calib_matrix(c, make_support(KernelShape(shape), tau, nd));
    *rows = m.entries.rows;
    *cols = m.entries.cols;
    put(m.entries.d, out);
  });
}

// filters: capacity n*n (first R columns written).
int sko_extract_nullspace(std::int64_t n, const double* gram, double ratio, std::int64_t* rank,
                          double* spectrum, double* filters) {
  return guarded([&] {
    GramMatrix g;
    g.entries = Mat(n, n);
    std::memcpy(g.entries.d.data(), gram, std::size_t(n * n) * sizeof(Cx));
    const NullspaceBasis b = extract_nullspace(g, ratio);
    *rank = b.rank();
    if (spectrum) std::memcpy(spectrum, b.spectrum.data(), b.spectrum.size() * sizeof(double));
    put(b.filters.d, filters);
  });
}

int sko_aggregate_w(std::int64_t n, std::int64_t r, const double* filters, double* w) {
  return guarded([&] {
    NullspaceBasis b;
    b.filters = Mat(n, r);
    std::memcpy(b.filters.d.data(), filters, std::size_t(n * r) * sizeof(Cx));
    put(aggregate_w(b).entries.d, w);
  });
}

int sko_gram_field_fast(std::int64_t q, const double* w, int shape, int tau, int nd, const std::int64_t* dims,
                        double* field) {
  return guarded([&] {
    const Support s = make_support(KernelShape(shape), tau, nd);
    AggregateW aw;
    aw.channels = q;
    aw.support_size = s.size();
    const Index n = q * s.size();
    aw.entries = Mat(n, n);
    std::memcpy(aw.entries.d.data(), w, std::size_t(n * n) * sizeof(Cx));
    put(gram_field_fast(aw, s, dims_of(nd, dims)).values, field);
  });
}

int sko_gram_field_naive(std::int64_t q, std::int64_t r, const double* filters, int shape, int tau, int nd,
                         const std::int64_t* dims, double* field) {
  return guarded([&] {
    const Support s = make_support(KernelShape(shape), tau, nd);
    NullspaceBasis b;
    b.channels = q;
    b.support_size = s.size();
    b.filters = Mat(q * s.size(), r);
    std::memcpy(b.filters.d.data(), filters, b.filters.d.size() * sizeof(Cx));
    put(gram_field_naive(filter_field_naive(b, s, dims_of(nd, dims))).values, field);
  });
}

int sko_espirit_inplace(std::int64_t n, std::int64_t q, double* field, std::int64_t support_size) {
  return guarded([&] {
    GramField g;
    g.dims = {n};
    g.channels = q;
    g.values.assign(cx(field), cx(field) + n * q * q);
    espirit_inplace(g, support_size);
    put(g.values, field);
  });
}

int sko_eig_power_field(std::int64_t n, std::int64_t q, const double* bfield, int iters, double* vectors,
                        double* values) {
  return guarded([&] {
    GramField g;
    g.dims = {n};
    g.channels = q;
    g.values.assign(cx(bfield), cx(bfield) + n * q * q);
    const EigenResult r = eig_power_field(g, iters);
    put(r.vectors.d, vectors);
    std::memcpy(values, r.values.data(), std::size_t(n) * sizeof(double));
  });
}

int sko_eig_dense_field(std::int64_t n, std::int64_t q, const double* field, int which, double* vectors,
                        double* values, double* second) {
  return guarded([&] {
    GramField g;
    g.dims = {n};
    g.channels = q;
    g.values.assign(cx(field), cx(field) + n * q * q);
    const EigenResult r = eig_dense_field(g, Extremal(which));
    put(r.vectors.d, vectors);
    std::memcpy(values, r.values.data(), std::size_t(n) * sizeof(double));
    if (second) std::memcpy(second, r.second_values.data(), std::size_t(n) * sizeof(double));
  });
}

int sko_normalize_maps(int nd, const std::int64_t* dims, std::int64_t q, const double* raw,
                       const std::int64_t* cdims, const std::int64_t* center_offset, const double* calib,
                       double apod_width, double* out, std::int64_t* zeroed) {
  return guarded([&] {
    Stack r(dims_of(nd, dims), q, Domain::image);
    std::memcpy(r.data.data(), raw, r.data.size() * sizeof(Cx));
    const Calib c = make_calib(nd, cdims, center_offset, q, calib);
    Stack m;
    const NormalizationRecord rec = normalize_maps(r, c, apod_width, m);
    put(m.data, out);
    if (zeroed) *zeroed = rec.zeroed_voxels;
  });
}

int sko_interpolate_maps(int nd, const std::int64_t* low_dims, std::int64_t q, const double* low,
                         const std::int64_t* full_dims, double* out) {
  return guarded([&] {
    Stack s(dims_of(nd, low_dims), q, Domain::image);
    std::memcpy(s.data.data(), low, s.data.size() * sizeof(Cx));
    put(interpolate_maps(s, dims_of(nd, full_dims)).data, out);
  });
}

int sko_interpolate_real(int nd, const std::int64_t* low_dims, const double* low, const std::int64_t* full_dims,
                         double* out) {
  return guarded([&] {
    const Dims ld = dims_of(nd, low_dims);
    std::vector<double> l(low, low + numel(ld));
    const auto r = interpolate_real(l, ld, dims_of(nd, full_dims));
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

// Full pipeline (maps.cpp:265-330).  grid_override: nullptr or nd extents
// (pipeline::compute_field/finalize with explicit grid dims, maps.hpp:117-123).
// Optional outputs may be null.  stage_seconds: gram, nullspace, field,
// eigensolve, post.
int sko_estimate_maps(int nd, const std::int64_t* cdims, const std::int64_t* center_offset, std::int64_t q,
                      const double* calib, const std::int64_t* full_dims, const sko_config* cfgp,
                      const std::int64_t* grid_override, double* maps, double* lambda, std::uint8_t* mask,
                      std::int64_t* grid_dims, std::int64_t* rank, double* sigma1, double* spectrum,
                      double* stage_seconds, std::int64_t* zeroed, double* raw_maps, double* raw_lambda,
                      double* gram_out) {
  return guarded([&] {
    PipelineConfig cfg;
    cfg.kernel = KernelShape(cfgp->kernel);
    cfg.tau = cfgp->tau;
    cfg.gram = GramMethod(cfgp->gram);
    cfg.nullspace_threshold = cfgp->nullspace_threshold;
    cfg.grid = GridMode(cfgp->grid);
    cfg.grid_pad = cfgp->grid_pad;
    cfg.eig = EigMethod(cfgp->eig);
    cfg.power_iters = cfgp->power_iters;
    cfg.method = MapMethod(cfgp->method);
    cfg.field = FieldPath(cfgp->field);
    cfg.mask_threshold = cfgp->mask_threshold;
    cfg.apod_width = cfgp->apod_width;
    const Calib c = make_calib(nd, cdims, center_offset, q, calib);
    const Dims full = dims_of(nd, full_dims);
    SensitivityResult res;
    if (!grid_override && !raw_maps && !raw_lambda && !gram_out) {
      res = estimate_maps(c, full, cfg);
    } else {
      // Same stages as estimate_maps, exposing intermediates.
      using clock = std::chrono::steady_clock;
      auto el = [](clock::time_point a) { return std::chrono::duration<double>(clock::now() - a).count(); };
      c.grid.validate();
      if (full.size() != c.dims().size()) throw DimError("full_dims rank mismatch");
      for (std::size_t a = 0; a < full.size(); ++a)
        if (full[a] < c.dims()[a]) throw DimError("full_dims must be at least the calibration extent");
      const auto t0 = clock::now();
      const Support s = make_support(cfg.kernel, cfg.tau, nd);
      auto t = clock::now();
      const GramMatrix g = compute_gram(c, s, cfg);
      res.provenance.stages["gram"] = el(t);
      put(g.entries.d, gram_out);
      t = clock::now();
      const NullspaceBasis b = extract_nullspace(g, cfg.nullspace_threshold);
      res.provenance.stages["nullspace"] = el(t);
      res.provenance.nullspace_rank = b.rank();
      res.provenance.sigma1 = b.spectrum[0];
      res.provenance.spectrum_normalized = singular_spectrum_report(b);
      const Dims grid = grid_override ? dims_of(nd, grid_override) : grid_dims_for(c, full, cfg);
      res.provenance.grid_dims = grid;
      t = clock::now();
      GramField f = compute_field(b, s, grid, cfg);
      res.provenance.stages["field"] = el(t);
      t = clock::now();
      RawMaps raw = solve_field(std::move(f), s.size(), cfg);
      res.provenance.stages["eigensolve"] = el(t);
      put(raw.maps.data, raw_maps);
      if (raw_lambda) std::memcpy(raw_lambda, raw.lambda.data(), raw.lambda.size() * sizeof(double));
      t = clock::now();
      Provenance keep = res.provenance;
      res = finalize(std::move(raw), c, full, cfg);
      keep.stages["post"] = el(t);
      keep.total_seconds = el(t0);
      res.provenance = keep;
    }
    put(res.maps.data, maps);
    if (lambda) std::memcpy(lambda, res.lambda_min_map.data(), res.lambda_min_map.size() * sizeof(double));
    if (mask) std::memcpy(mask, res.support_mask.data(), res.support_mask.size());
    if (grid_dims) {
      const Dims& gd = res.provenance.grid_dims.empty() ? full : res.provenance.grid_dims;
      for (int a = 0; a < nd; ++a) grid_dims[a] = gd[std::size_t(a)];
    }
    if (rank) *rank = res.provenance.nullspace_rank;
    if (sigma1) *sigma1 = res.provenance.sigma1;
    if (spectrum)
      std::memcpy(spectrum, res.provenance.spectrum_normalized.data(),
                  res.provenance.spectrum_normalized.size() * sizeof(double));
    if (stage_seconds) {
      const char* names[5] = {"gram", "nullspace", "field", "eigensolve", "post"};
      for (int i = 0; i < 5; ++i) stage_seconds[i] = res.provenance.stages[names[i]];
    }
    if (zeroed) *zeroed = res.normalization.zeroed_voxels;
  });
}

// Reference scene generator (synthetic.cpp) + forward model.  Any output may be null.
int sko_simulate(std::int64_t q, int nd, const std::int64_t* dims, int tau_gen, std::uint64_t seed, int kind,
                 double noise_sigma, std::uint64_t noise_seed, double* kspace, double* true_maps,
                 std::uint8_t* support_mask_true, double* phantom, double* gen_coeffs) {
  return guarded([&] {
    const SyntheticScene sc = make_scene(q, dims_of(nd, dims), tau_gen, seed, PhantomKind(kind));
    if (kspace) put(forward_kspace(sc, noise_sigma, noise_seed).data, kspace);
    put(sc.true_maps.data, true_maps);
    if (support_mask_true) std::memcpy(support_mask_true, sc.support_mask_true.data(), sc.support_mask_true.size());
    if (phantom) std::memcpy(phantom, sc.phantom.data(), sc.phantom.size() * sizeof(double));
    put(sc.gen_coeffs.d, gen_coeffs);
  });
}

int sko_projection_residual(int nd, const std::int64_t* dims, std::int64_t q, const double* kspace,
                            const double* maps, double* out) {
  return guarded([&] {
    Stack k(dims_of(nd, dims), q, Domain::kspace), m(dims_of(nd, dims), q, Domain::image);
    std::memcpy(k.data.data(), kspace, k.data.size() * sizeof(Cx));
    std::memcpy(m.data.data(), maps, m.data.size() * sizeof(Cx));
    *out = projection_residual(k, m);
  });
}

}  // extern "C"
