// ORACLE — TEST INFRASTRUCTURE ONLY (see sko.hpp).
//
// FP64 restatement of the reference hot path.  Each function cites the
// reference lines it follows; the arithmetic order is kept where it matters
// (Gram lag gather, W fold, power iteration restart rule, normalisation).
#include <atomic>
#include <chrono>
#include <cmath>
#include <dlfcn.h>

#include "sko.hpp"

namespace sko {

// ---------------------------------------------------------------- types.cpp
Index numel(const Dims& dims) {  // types.cpp:7-11
  Index n = 1;
  for (Index d : dims) n *= d;
  return n;
}

std::vector<Index> strides_of(const Dims& dims) {  // types.cpp:13-17
  std::vector<Index> s(dims.size(), 1);
  for (int a = int(dims.size()) - 2; a >= 0; --a) s[std::size_t(a)] = s[std::size_t(a + 1)] * dims[std::size_t(a + 1)];
  return s;
}

bool next_index(std::vector<Index>& idx, const Dims& dims) {  // types.cpp:19-25
  for (int a = int(dims.size()) - 1; a >= 0; --a) {
    if (++idx[std::size_t(a)] < dims[std::size_t(a)]) return true;
    idx[std::size_t(a)] = 0;
  }
  return false;
}

Dims centers_of(const Dims& dims) {  // types.cpp:27-31
  Dims c(dims.size());
  for (std::size_t a = 0; a < dims.size(); ++a) c[a] = center_index(dims[a]);
  return c;
}

Stack::Stack(Dims d, Index q, Domain dom) : dims(std::move(d)), channels(q), domain(dom) {
  Index n = 1;
  for (Index e : dims) n *= std::max<Index>(e, 0);
  data.assign(std::size_t(std::max<Index>(q, 0) * n), Cx(0, 0));
  validate();
}

void Stack::validate() const {  // types.cpp:49-56
  if (dims.empty()) throw DimError("stack needs at least one axis");
  for (Index d : dims)
    if (d < 1) throw DimError("stack axis extents must be >= 1");
  if (channels < 1) throw DimError("stack needs at least one channel");
  if (Index(data.size()) != channels * numel(dims))
    throw DimError("stack data length must be channels * voxels");
}

Calib extract_calibration(const Stack& stack, const Dims& size) {  // types.cpp:58-90
  stack.validate();
  if (size.size() != stack.dims.size()) throw DimError("calibration size rank does not match stack");
  for (std::size_t a = 0; a < size.size(); ++a)
    if (size[a] < 1 || size[a] > stack.dims[a])
      throw DimError("calibration size exceeds stack extent on axis " + std::to_string(a));
  const Dims parent_center = centers_of(stack.dims);
  const Dims region_center = centers_of(size);
  Dims start(size.size());
  for (std::size_t a = 0; a < size.size(); ++a) start[a] = parent_center[a] - region_center[a];
  Stack region(size, stack.channels, Domain::kspace);
  const auto src_strides = strides_of(stack.dims);
  const auto dst_strides = strides_of(size);
  const Index n_src = stack.voxels(), n_dst = region.voxels();
  std::vector<Index> idx(size.size(), 0);
  do {
    Index src = 0, dst = 0;
    for (std::size_t a = 0; a < size.size(); ++a) {
      src += (start[a] + idx[a]) * src_strides[a];
      dst += idx[a] * dst_strides[a];
    }
    for (Index q = 0; q < stack.channels; ++q)
      region.data[std::size_t(q * n_dst + dst)] = stack.data[std::size_t(q * n_src + src)];
  } while (next_index(idx, size));
  return Calib{std::move(region), region_center};
}

// ------------------------------------------------------------- parallel.cpp
namespace {
std::atomic<int> g_max_threads{0};
}
void set_max_threads(int n) { g_max_threads.store(n < 0 ? 0 : n); }
int max_threads() {  // parallel.cpp:11-18
  const int n = g_max_threads.load();
  if (n > 0) return n;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : int(hw);
}

// -------------------------------------------------------------- kernels.cpp
Support make_support(KernelShape shape, int tau, int ndim) {  // kernels.cpp:7-35
  if (tau < 0) throw DimError("kernel radius must be >= 0");
  if (ndim < 1) throw DimError("kernel dimension must be >= 1");
  const Index side = 2 * Index(tau) + 1;
  std::vector<int> kept;
  Dims box(std::size_t(ndim), side);
  std::vector<Index> idx(static_cast<std::size_t>(ndim), 0);
  do {
    long r2 = 0;
    for (int a = 0; a < ndim; ++a) {
      const long v = long(idx[std::size_t(a)]) - tau;
      r2 += v * v;
    }
    if (shape == KernelShape::ellipsoid && r2 > long(tau) * tau) continue;
    for (int a = 0; a < ndim; ++a) kept.push_back(int(idx[std::size_t(a)]) - tau);
  } while (next_index(idx, box));
  Support s;
  s.shape = shape;
  s.tau = tau;
  s.nd = ndim;
  s.count = Index(kept.size()) / ndim;
  s.offsets = std::move(kept);
  return s;
}

// ---------------------------------------------------------- calibration.cpp
namespace {
void check_calib(const Calib& calib, const Support& support) {  // calibration.cpp:12-20
  calib.grid.validate();
  if (Index(calib.grid.dims.size()) != support.ndim())
    throw DimError("support dimension does not match calibration region");
  for (Index d : calib.grid.dims)
    if (d <= 2 * support.tau)
      throw DimError("calibration region too small for kernel radius " + std::to_string(support.tau));
}
Index next_pow2(Index n) {  // calibration.cpp:22-26
  Index p = 1;
  while (p < n) p <<= 1;
  return p;
}
}  // namespace

CalibMatrix build_calib_matrix(const Calib& calib, const Support& support) {  // calibration.cpp:30-68
  check_calib(calib, support);
  const Index q_count = calib.grid.channels, lam = support.size(), nd = support.ndim();
  const Dims& ext = calib.grid.dims;
  const auto strides = strides_of(ext);
  const Index n_vox = calib.grid.voxels();
  Dims shift_ext(ext.size());
  Index p_rows = 1;
  for (std::size_t a = 0; a < ext.size(); ++a) {
    shift_ext[a] = ext[a] - 2 * support.tau;
    p_rows *= shift_ext[a];
  }
  CalibMatrix out;
  out.valid_shifts = p_rows;
  out.channels = q_count;
  out.support_size = lam;
  out.entries = Mat(p_rows, q_count * lam);
  std::vector<Index> idx(ext.size(), 0);
  Index row = 0;
  do {
    Index base = 0;
    for (Index a = 0; a < nd; ++a) base += (idx[std::size_t(a)] + support.tau) * strides[std::size_t(a)];
    for (Index i = 0; i < lam; ++i) {
      Index at = base;
      for (Index a = 0; a < nd; ++a) at -= support.off(i, a) * strides[std::size_t(a)];
      for (Index q = 0; q < q_count; ++q)
        out.entries(row, q * lam + i) = calib.grid.data[std::size_t(q * n_vox + at)];
    }
    ++row;
  } while (next_index(idx, shift_ext));
  return out;
}

namespace {
void hermitian_average(Mat& g) {  // (G + G^H) / 2
  const Index n = g.rows;
  for (Index c = 0; c < n; ++c)
    for (Index r = c; r < n; ++r) {
      const Cx a = g(r, c), b = std::conj(g(c, r));
      const Cx v = (a + b) / 2.0;
      g(r, c) = v;
      g(c, r) = std::conj(v);
    }
}
}  // namespace

GramMatrix gram_explicit(const CalibMatrix& c) {  // calibration.cpp:70-78
  GramMatrix g;
  g.method = GramMethod::explicit_product;
  g.channels = c.channels;
  g.support_size = c.support_size;
  const Index n = c.entries.cols, p = c.entries.rows;
  g.entries = Mat(n, n);
  if (lapack::loaded()) {
    lapack::zgemm('C', 'N', n, n, p, Cx(1, 0), c.entries.d.data(), p, c.entries.d.data(), p,
                  Cx(0, 0), g.entries.d.data(), n);
  } else {
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < n; ++i) {
        Cx acc = 0;
        for (Index r = 0; r < p; ++r) acc += std::conj(c.entries(r, i)) * c.entries(r, j);
        g.entries(i, j) = acc;
      }
  }
  hermitian_average(g.entries);
  return g;
}

GramMatrix gram_fft(const Calib& calib, const Support& support) {  // calibration.cpp:80-144
  check_calib(calib, support);
  const Index q_count = calib.grid.channels, lam = support.size(), nd = support.ndim();
  const Dims& ext = calib.grid.dims;
  const Index n_vox = calib.grid.voxels();
  Dims pad(ext.size());
  for (std::size_t a = 0; a < ext.size(); ++a) pad[a] = next_pow2(ext[a] + 2 * support.tau);
  const Index n_pad = numel(pad);
  const auto pad_strides = strides_of(pad);

  std::vector<std::vector<Cx>> spectra(static_cast<std::size_t>(q_count));  // :96-109
  for (Index q = 0; q < q_count; ++q) {
    std::vector<Cx> vol(static_cast<std::size_t>(n_pad), Cx(0, 0));
    std::vector<Index> idx(ext.size(), 0);
    Index src = 0;
    do {
      Index dst = 0;
      for (std::size_t a = 0; a < ext.size(); ++a) dst += idx[a] * pad_strides[a];
      vol[std::size_t(dst)] = calib.grid.data[std::size_t(q * n_vox + src)];
      ++src;
    } while (next_index(idx, ext));
    fft::transform_nd(vol.data(), pad, -1);
    spectra[std::size_t(q)] = std::move(vol);
  }

  std::vector<Index> lag_at(static_cast<std::size_t>(lam * lam));  // :113-122, lag n_s - n_t
  for (Index s = 0; s < lam; ++s)
    for (Index t = 0; t < lam; ++t) {
      Index at = 0;
      for (Index a = 0; a < nd; ++a) {
        const Index lag = support.off(s, a) - support.off(t, a);
        at += ((lag % pad[std::size_t(a)]) + pad[std::size_t(a)]) % pad[std::size_t(a)] * pad_strides[std::size_t(a)];
      }
      lag_at[std::size_t(s * lam + t)] = at;
    }

  GramMatrix g;
  g.method = GramMethod::fft;
  g.channels = q_count;
  g.support_size = lam;
  g.entries = Mat(q_count * lam, q_count * lam);
  parallel_for(0, q_count * q_count, [&](Index pair) {  // :131-140
    const Index p = pair / q_count, q = pair % q_count;
    std::vector<Cx> corr(static_cast<std::size_t>(n_pad));
    const auto& sp = spectra[std::size_t(p)];
    const auto& sq = spectra[std::size_t(q)];
    for (Index k = 0; k < n_pad; ++k) corr[std::size_t(k)] = std::conj(sp[std::size_t(k)]) * sq[std::size_t(k)];
    fft::transform_nd(corr.data(), pad, +1);
    for (auto& v : corr) v /= double(n_pad);
    for (Index s = 0; s < lam; ++s)
      for (Index t = 0; t < lam; ++t)
        g.entries(p * lam + s, q * lam + t) = corr[std::size_t(lag_at[std::size_t(s * lam + t)])];
  });
  hermitian_average(g.entries);  // :142
  return g;
}

// ------------------------------------------------------------ nullspace.cpp
NullspaceBasis extract_nullspace(const GramMatrix& gram, double threshold_ratio) {  // nullspace.cpp:7-35
  if (!(threshold_ratio > 0.0 && threshold_ratio < 1.0))
    throw DimError("nullspace threshold ratio must lie in (0,1)");
  const Index n = gram.entries.rows;
  if (n == 0 || gram.entries.cols != n) throw DimError("Gram matrix must be square");
  Mat vecs = gram.entries;
  std::vector<double> evals(static_cast<std::size_t>(n));
  lapack::zheevd(n, vecs.d.data(), evals.data(), true);  // ascending, as SelfAdjointEigenSolver
  std::vector<double> sigma_asc(static_cast<std::size_t>(n));
  for (Index i = 0; i < n; ++i) sigma_asc[std::size_t(i)] = std::sqrt(std::max(0.0, evals[std::size_t(i)]));
  NullspaceBasis basis;
  basis.threshold_ratio = threshold_ratio;
  basis.channels = gram.channels;
  basis.support_size = gram.support_size;
  basis.spectrum.assign(sigma_asc.rbegin(), sigma_asc.rend());
  const double cutoff = threshold_ratio * basis.spectrum[0];
  Index r = 0;
  while (r < n && sigma_asc[std::size_t(r)] < cutoff) ++r;
  if (r == 0)
    throw NullspaceEmptyError("calibration matrix has no approximate nullspace at ratio " +
                              std::to_string(threshold_ratio));
  basis.filters = Mat(n, r);
  std::copy(vecs.d.begin(), vecs.d.begin() + n * r, basis.filters.d.begin());
  return basis;
}

std::vector<double> singular_spectrum_report(const NullspaceBasis& basis) {  // nullspace.cpp:37-41
  const double s1 = basis.spectrum.empty() ? 0.0 : basis.spectrum[0];
  std::vector<double> out(basis.spectrum.size(), 0.0);
  if (s1 <= 0.0) return out;
  for (std::size_t i = 0; i < out.size(); ++i) out[i] = basis.spectrum[i] / s1;
  return out;
}

// --------------------------------------------------------- spatial_gram.cpp
namespace {
void check_grid(const Support& support, const Dims& dims) {  // spatial_gram.cpp:12-17
  if (Index(dims.size()) != support.ndim()) throw DimError("voxel grid rank does not match support dimension");
  for (Index d : dims)
    if (d < 1) throw DimError("voxel grid extents must be >= 1");
}
Index wrap_slot(const Support& s, Index row, int sign, const Dims& dims, const std::vector<Index>& strides) {
  Index at = 0;  // spatial_gram.cpp:21-29
  for (Index a = 0; a < s.ndim(); ++a) {
    const Index v = sign * Index(s.off(row, a));
    at += (((v % dims[std::size_t(a)]) + dims[std::size_t(a)]) % dims[std::size_t(a)]) * strides[std::size_t(a)];
  }
  return at;
}
}  // namespace

FilterField filter_field_naive(const NullspaceBasis& basis, const Support& support, const Dims& dims,
                               std::size_t max_bytes) {  // spatial_gram.cpp:33-64
  check_grid(support, dims);
  const Index r_count = basis.rank(), q_count = basis.channels, lam = support.size(), n = numel(dims);
  const std::size_t need = std::size_t(r_count) * std::size_t(q_count) * std::size_t(n) * sizeof(Cx);
  if (need > max_bytes)
    throw std::length_error("filter field would need " + std::to_string(need) + " bytes (cap " +
                            std::to_string(max_bytes) + ")");
  FilterField field;
  field.dims = dims;
  field.channels = q_count;
  field.filters = r_count;
  field.values.assign(std::size_t(r_count * q_count * n), Cx(0, 0));
  const auto strides = strides_of(dims);
  parallel_for(0, r_count * q_count, [&](Index plane) {
    const Index r = plane / q_count, q = plane % q_count;
    std::vector<Cx> vol(static_cast<std::size_t>(n), Cx(0, 0));
    for (Index i = 0; i < lam; ++i)
      vol[std::size_t(wrap_slot(support, i, +1, dims, strides))] += basis.filters(q * lam + i, r);
    fft::transform_nd(vol.data(), dims, +1);
    fft::fftshift_nd(vol.data(), dims);
    std::copy(vol.begin(), vol.end(), field.values.begin() + plane * n);
  });
  return field;
}

GramField gram_field_naive(const FilterField& field) {  // spatial_gram.cpp:66-85
  const Index q_count = field.channels, n = field.voxels();
  GramField out;
  out.dims = field.dims;
  out.channels = q_count;
  out.values.assign(std::size_t(n * q_count * q_count), Cx(0, 0));
  parallel_for(0, n, [&](Index j) {
    Cx* g = out.at(j);
    for (Index r = 0; r < field.filters; ++r)
      for (Index q = 0; q < q_count; ++q) {
        const Cx hq = field.plane(r, q)[j];
        for (Index p = 0; p < q_count; ++p) g[q * q_count + p] += std::conj(field.plane(r, p)[j]) * hq;
      }
  });
  return out;
}

AggregateW aggregate_w(const NullspaceBasis& basis) {  // spatial_gram.cpp:87-94
  if (basis.rank() < 1) throw NullspaceEmptyError("aggregate requires at least one filter");
  AggregateW w;
  w.channels = basis.channels;
  w.support_size = basis.support_size;
  const Index n = basis.filters.rows, r = basis.filters.cols;
  w.entries = Mat(n, n);
  if (lapack::loaded()) {
    lapack::zgemm('N', 'C', n, n, r, Cx(1, 0), basis.filters.d.data(), n, basis.filters.d.data(), n,
                  Cx(0, 0), w.entries.d.data(), n);
  } else {
    for (Index c = 0; c < n; ++c)
      for (Index k = 0; k < r; ++k) {
        const Cx b = std::conj(basis.filters(c, k));
        for (Index i = 0; i < n; ++i) w.entries(i, c) += basis.filters(i, k) * b;
      }
  }
  return w;
}

GramField gram_field_fast(const AggregateW& w, const Support& support, const Dims& dims) {  // :96-148
  check_grid(support, dims);
  const Index q_count = w.channels, lam = support.size(), n = numel(dims);
  const auto strides = strides_of(dims);
  GramField out;
  out.dims = dims;
  out.channels = q_count;
  out.values.assign(std::size_t(n * q_count * q_count), Cx(0, 0));
  std::vector<Index> lag_slot(static_cast<std::size_t>(lam * lam));  // frequency m_t - n_s
  for (Index s = 0; s < lam; ++s)
    for (Index t = 0; t < lam; ++t) {
      Index at = 0;
      for (Index a = 0; a < support.ndim(); ++a) {
        const Index v = Index(support.off(t, a)) - Index(support.off(s, a));
        at += (((v % dims[std::size_t(a)]) + dims[std::size_t(a)]) % dims[std::size_t(a)]) * strides[std::size_t(a)];
      }
      lag_slot[std::size_t(s * lam + t)] = at;
    }
  std::vector<std::pair<Index, Index>> pairs;
  for (Index p = 0; p < q_count; ++p)
    for (Index q = p; q < q_count; ++q) pairs.emplace_back(p, q);
  parallel_for(0, Index(pairs.size()), [&](Index k) {
    const auto [p, q] = pairs[std::size_t(k)];
    std::vector<Cx> kernel(static_cast<std::size_t>(n), Cx(0, 0));
    for (Index s = 0; s < lam; ++s)
      for (Index t = 0; t < lam; ++t)
        kernel[std::size_t(lag_slot[std::size_t(s * lam + t)])] += w.entries(q * lam + s, p * lam + t);
    fft::transform_nd(kernel.data(), dims, -1);
    fft::fftshift_nd(kernel.data(), dims);
    for (Index j = 0; j < n; ++j) {
      out.values[std::size_t(j * q_count * q_count + q * q_count + p)] = kernel[std::size_t(j)];
      if (p != q) out.values[std::size_t(j * q_count * q_count + p * q_count + q)] = std::conj(kernel[std::size_t(j)]);
    }
  });
  parallel_for(0, n, [&](Index j) {  // :140-146
    for (Index q = 0; q < q_count; ++q) {
      Cx& d = out.values[std::size_t(j * q_count * q_count + q * q_count + q)];
      d = Cx(d.real(), 0.0);
    }
  });
  return out;
}

void espirit_inplace(GramField& g, Index support_size) {  // spatial_gram.cpp:156-164
  const double inv = 1.0 / double(support_size);
  const Index q_count = g.channels;
  parallel_for(0, g.voxels(), [&](Index j) {
    Cx* m = g.at(j);
    for (Index i = 0; i < q_count * q_count; ++i) m[i] *= -inv;
    for (Index q = 0; q < q_count; ++q) m[q * q_count + q] += 1.0;
  });
}

// ----------------------------------------------------------- eigensolve.cpp
EigenResult eig_dense_field(const GramField& field, Extremal which) {  // eigensolve.cpp:9-38
  const Index q = field.channels, n = field.voxels();
  EigenResult out;
  out.dims = field.dims;
  out.channels = q;
  out.vectors = Mat(q, n);
  out.values.assign(std::size_t(n), 0.0);
  out.second_values.assign(std::size_t(n), 0.0);
  const int nt = max_threads();
  const Index chunk = (n + nt - 1) / nt;
  parallel_for(0, Index(nt), [&](Index t) {
    std::vector<Cx> a(static_cast<std::size_t>(q * q));
    std::vector<double> w(static_cast<std::size_t>(q));
    const Index lo = t * chunk, hi = std::min(n, lo + chunk);
    for (Index j = lo; j < hi; ++j) {
      std::copy(field.at(j), field.at(j) + q * q, a.begin());
      lapack::zheevd(q, a.data(), w.data(), true);
      const Index col = which == Extremal::smallest ? 0 : q - 1;
      for (Index r = 0; r < q; ++r) out.vectors(r, j) = a[std::size_t(col * q + r)];
      out.values[std::size_t(j)] = w[std::size_t(col)];
      if (which == Extremal::smallest)
        out.second_values[std::size_t(j)] = q > 1 ? w[1] : w[0];
      else
        out.second_values[std::size_t(j)] = q > 1 ? w[std::size_t(q - 2)] : w[std::size_t(q - 1)];
    }
  });
  return out;
}

EigenResult eig_power_field(const GramField& b_field, int iters) {  // eigensolve.cpp:40-74
  const Index q = b_field.channels, n = b_field.voxels();
  EigenResult out;
  out.dims = b_field.dims;
  out.channels = q;
  out.vectors = Mat(q, n);
  out.values.assign(std::size_t(n), 0.0);
  out.iterations_used = iters;
  const double init = 1.0 / std::sqrt(double(q));
  parallel_for(0, n, [&](Index j) {
    const Cx* b = b_field.at(j);
    std::vector<Cx> v(static_cast<std::size_t>(q), Cx(init, 0.0)), w(static_cast<std::size_t>(q));
    auto matvec = [&](const std::vector<Cx>& x, std::vector<Cx>& y) {
      std::fill(y.begin(), y.end(), Cx(0, 0));
      for (Index c = 0; c < q; ++c) {
        const Cx xc = x[std::size_t(c)];
        for (Index r = 0; r < q; ++r) y[std::size_t(r)] += b[c * q + r] * xc;
      }
    };
    auto norm = [&](const std::vector<Cx>& y) {
      double s = 0;
      for (const Cx& z : y) s += std::norm(z);
      return std::sqrt(s);
    };
    for (int it = 0; it < iters; ++it) {
      matvec(v, w);
      double nrm = norm(w);
      if (nrm < 1e-14) {
        if (it == 0) {
          std::fill(v.begin(), v.end(), Cx(0, 0));
          v[0] = 1.0;
          matvec(v, w);
          nrm = norm(w);
        }
        if (nrm < 1e-14) break;
      }
      for (Index r = 0; r < q; ++r) v[std::size_t(r)] = w[std::size_t(r)] / nrm;
    }
    for (Index r = 0; r < q; ++r) out.vectors(r, j) = v[std::size_t(r)];
    matvec(v, w);
    Cx dot = 0;
    for (Index r = 0; r < q; ++r) dot += std::conj(v[std::size_t(r)]) * w[std::size_t(r)];
    out.values[std::size_t(j)] = dot.real();
  });
  return out;
}

// ----------------------------------------------------------------- maps.cpp
PipelineConfig PipelineConfig::baseline() {  // maps.cpp:12-19
  PipelineConfig cfg;
  cfg.kernel = KernelShape::rect;
  cfg.gram = GramMethod::explicit_product;
  cfg.grid = GridMode::full;
  cfg.eig = EigMethod::dense;
  return cfg;
}
PipelineConfig PipelineConfig::pisco() {  // maps.cpp:21-28
  PipelineConfig cfg;
  cfg.kernel = KernelShape::ellipsoid;
  cfg.gram = GramMethod::fft;
  cfg.grid = GridMode::reduced;
  cfg.eig = EigMethod::power;
  return cfg;
}

Dims reduced_grid_dims(const Dims& calib_dims, Index pad, const Dims& full_dims) {  // maps.cpp:39-45
  if (calib_dims.size() != full_dims.size()) throw DimError("grid rank mismatch");
  Dims out(calib_dims.size());
  for (std::size_t a = 0; a < calib_dims.size(); ++a) out[a] = std::min(calib_dims[a] + pad, full_dims[a]);
  return out;
}

std::vector<std::uint8_t> support_mask(const std::vector<double>& lam, double thr) {  // maps.cpp:47-52
  std::vector<std::uint8_t> mask(lam.size());
  for (std::size_t j = 0; j < lam.size(); ++j) mask[j] = lam[j] < thr ? 1 : 0;
  return mask;
}

Stack interpolate_maps(const Stack& lowres, const Dims& full_dims) {  // maps.cpp:54-90
  lowres.validate();
  if (lowres.dims.size() != full_dims.size()) throw DimError("interpolation rank mismatch");
  for (std::size_t a = 0; a < full_dims.size(); ++a)
    if (full_dims[a] < lowres.dims[a])
      throw DimError("interpolation target smaller than source on axis " + std::to_string(a));
  const Dims& low = lowres.dims;
  const Index n_low = numel(low), n_full = numel(full_dims);
  const Dims c_low = centers_of(low), c_full = centers_of(full_dims);
  const auto s_full = strides_of(full_dims);
  Stack out(full_dims, lowres.channels, lowres.domain);
  parallel_for(0, lowres.channels, [&](Index q) {
    std::vector<Cx> spec(lowres.channel(q), lowres.channel(q) + n_low);
    fft::image_to_kspace(spec.data(), low);
    std::vector<Cx> padded(static_cast<std::size_t>(n_full), Cx(0, 0));
    std::vector<Index> idx(low.size(), 0);
    Index src = 0;
    do {
      Index dst = 0;
      for (std::size_t a = 0; a < low.size(); ++a) dst += (idx[a] - c_low[a] + c_full[a]) * s_full[a];
      padded[std::size_t(dst)] = spec[std::size_t(src++)];
    } while (next_index(idx, low));
    fft::kspace_to_image(padded.data(), full_dims);
    std::copy(padded.begin(), padded.end(), out.channel(q));
  });
  return out;
}

std::vector<double> interpolate_real(const std::vector<double>& lowres, const Dims& low_dims,
                                     const Dims& full_dims) {  // maps.cpp:92-99
  Stack wrap(low_dims, 1, Domain::image);
  for (std::size_t j = 0; j < lowres.size(); ++j) wrap.data[j] = Cx(lowres[j], 0.0);
  const Stack up = interpolate_maps(wrap, full_dims);
  std::vector<double> out(static_cast<std::size_t>(up.voxels()));
  for (std::size_t j = 0; j < out.size(); ++j) out[j] = up.data[j].real();
  return out;
}

NormalizationRecord normalize_maps(const Stack& raw, const Calib& calib, double apod_width,
                                   Stack& maps) {  // maps.cpp:101-176
  raw.validate();
  const Index q_count = raw.channels, n = raw.voxels();
  const Dims& dims = raw.dims;
  if (dims.size() != calib.dims().size()) throw DimError("map/calibration rank mismatch");
  for (std::size_t a = 0; a < dims.size(); ++a)
    if (dims[a] < calib.dims()[a]) throw DimError("map grid smaller than calibration region");
  if (q_count != calib.channels()) throw DimError("map/calibration channel mismatch");
  maps = raw;
  NormalizationRecord rec;
  rec.sos = true;
  Index zeroed = 0;
  for (Index j = 0; j < n; ++j) {
    double sos = 0;
    for (Index q = 0; q < q_count; ++q) sos += std::norm(maps.data[std::size_t(q * n + j)]);
    if (sos > 0) {
      const double inv = 1.0 / std::sqrt(sos);
      for (Index q = 0; q < q_count; ++q) maps.data[std::size_t(q * n + j)] *= inv;
    } else {
      ++zeroed;
    }
  }
  rec.zeroed_voxels = zeroed;
  const Dims& ext = calib.dims();
  rec.apod_sigma.resize(ext.size());
  for (std::size_t a = 0; a < ext.size(); ++a) rec.apod_sigma[a] = apod_width > 0 ? apod_width : double(ext[a]) / 4.0;
  const Dims grid_center = centers_of(dims);
  const auto grid_strides = strides_of(dims);
  const Index n_calib = calib.grid.voxels();
  Stack recon(dims, q_count, Domain::image);
  parallel_for(0, q_count, [&](Index q) {
    std::vector<Cx> vol(static_cast<std::size_t>(n), Cx(0, 0));
    std::vector<Index> idx(ext.size(), 0);
    Index src = 0;
    do {
      double w = 0;
      Index dst = 0;
      for (std::size_t a = 0; a < ext.size(); ++a) {
        const double f = double(idx[a] - calib.center_offset[a]);
        w += f * f / (2.0 * rec.apod_sigma[a] * rec.apod_sigma[a]);
        dst += (idx[a] - calib.center_offset[a] + grid_center[a]) * grid_strides[a];
      }
      vol[std::size_t(dst)] = calib.grid.data[std::size_t(q * n_calib + src)] * std::exp(-w);
      ++src;
    } while (next_index(idx, ext));
    fft::kspace_to_image(vol.data(), dims);
    std::copy(vol.begin(), vol.end(), recon.channel(q));
  });
  for (Index j = 0; j < n; ++j) {
    Cx combined = 0;
    for (Index q = 0; q < q_count; ++q)
      combined += std::conj(maps.data[std::size_t(q * n + j)]) * recon.data[std::size_t(q * n + j)];
    const double mag = std::abs(combined);
    if (mag > 0) {
      const Cx u = combined / mag;
      for (Index q = 0; q < q_count; ++q) maps.data[std::size_t(q * n + j)] *= u;
    }
  }
  rec.phase_referenced = true;
  return rec;
}

GramMatrix compute_gram(const Calib& calib, const Support& support, const PipelineConfig& cfg) {
  if (cfg.gram == GramMethod::fft) return gram_fft(calib, support);  // maps.cpp:180-186
  return gram_explicit(build_calib_matrix(calib, support));
}

Dims grid_dims_for(const Calib& calib, const Dims& full_dims, const PipelineConfig& cfg) {  // :188-193
  if (cfg.grid == GridMode::reduced) return reduced_grid_dims(calib.dims(), cfg.grid_pad, full_dims);
  return full_dims;
}

GramField compute_field(const NullspaceBasis& basis, const Support& support, const Dims& grid,
                        const PipelineConfig& cfg) {  // maps.cpp:195-205
  if (cfg.field == FieldPath::naive)
    return gram_field_naive(filter_field_naive(basis, support, grid, cfg.field_byte_cap));
  return gram_field_fast(aggregate_w(basis), support, grid);
}

RawMaps solve_field(GramField field, Index support_size, const PipelineConfig& cfg) {  // maps.cpp:207-230
  const Index q_count = field.channels, n = field.voxels();
  EigenResult eig;
  std::vector<double> lambda(static_cast<std::size_t>(n));
  if (cfg.eig == EigMethod::dense && cfg.method == MapMethod::nullspace) {
    eig = eig_dense_field(field, Extremal::smallest);
    for (Index j = 0; j < n; ++j) lambda[std::size_t(j)] = eig.values[std::size_t(j)] / double(support_size);
  } else {
    espirit_inplace(field, support_size);
    eig = cfg.eig == EigMethod::dense ? eig_dense_field(field, Extremal::largest)
                                      : eig_power_field(field, cfg.power_iters);
    for (Index j = 0; j < n; ++j) lambda[std::size_t(j)] = 1.0 - eig.values[std::size_t(j)];
  }
  RawMaps out;
  out.maps = Stack(field.dims, q_count, Domain::image);
  for (Index q = 0; q < q_count; ++q)
    for (Index j = 0; j < n; ++j) out.maps.data[std::size_t(q * n + j)] = eig.vectors(q, j);
  out.lambda = std::move(lambda);
  return out;
}

SensitivityResult finalize(RawMaps&& raw, const Calib& calib, const Dims& full_dims,
                           const PipelineConfig& cfg) {  // maps.cpp:232-261
  SensitivityResult result;
  Stack normalized;
  NormalizationRecord rec = normalize_maps(raw.maps, calib, cfg.apod_width, normalized);
  if (normalized.dims != full_dims) {
    result.maps = interpolate_maps(normalized, full_dims);
    result.lambda_min_map = interpolate_real(raw.lambda, normalized.dims, full_dims);
    const Index n = result.maps.voxels();
    for (Index j = 0; j < n; ++j) {
      double sos = 0;
      for (Index q = 0; q < result.maps.channels; ++q) sos += std::norm(result.maps.data[std::size_t(q * n + j)]);
      if (sos > 0) {
        const double inv = 1.0 / std::sqrt(sos);
        for (Index q = 0; q < result.maps.channels; ++q) result.maps.data[std::size_t(q * n + j)] *= inv;
      }
    }
    rec.renormalized_after_interpolation = true;
  } else {
    result.maps = std::move(normalized);
    result.lambda_min_map = std::move(raw.lambda);
  }
  result.support_mask = support_mask(result.lambda_min_map, cfg.mask_threshold);
  result.normalization = rec;
  return result;
}

SensitivityResult estimate_maps(const Calib& calib, const Dims& full_dims, const PipelineConfig& cfg) {
  calib.grid.validate();  // maps.cpp:265-330
  if (full_dims.size() != calib.dims().size()) throw DimError("full_dims rank mismatch");
  for (std::size_t a = 0; a < full_dims.size(); ++a)
    if (full_dims[a] < calib.dims()[a]) throw DimError("full_dims must be at least the calibration extent");
  using clock = std::chrono::steady_clock;
  auto elapsed = [](clock::time_point a, clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  };
  const auto t0 = clock::now();
  Provenance prov;
  prov.calib_dims = calib.dims();
  prov.full_dims = full_dims;
  prov.channels = calib.channels();
  const Support support = make_support(cfg.kernel, cfg.tau, int(calib.dims().size()));
  prov.support_size = support.size();
  prov.valid_shifts = 1;
  for (Index d : calib.dims()) prov.valid_shifts *= std::max<Index>(0, d - 2 * cfg.tau);

  auto t = clock::now();
  const GramMatrix gram = compute_gram(calib, support, cfg);
  prov.stages["gram"] = elapsed(t, clock::now());

  t = clock::now();
  const NullspaceBasis basis = extract_nullspace(gram, cfg.nullspace_threshold);
  prov.nullspace_rank = basis.rank();
  prov.sigma1 = basis.spectrum[0];
  prov.spectrum_normalized = singular_spectrum_report(basis);
  prov.stages["nullspace"] = elapsed(t, clock::now());

  const Dims grid_dims = grid_dims_for(calib, full_dims, cfg);
  prov.grid_dims = grid_dims;

  t = clock::now();
  GramField field = compute_field(basis, support, grid_dims, cfg);
  prov.stages["field"] = elapsed(t, clock::now());

  t = clock::now();
  RawMaps raw = solve_field(std::move(field), support.size(), cfg);
  prov.stages["eigensolve"] = elapsed(t, clock::now());

  t = clock::now();
  SensitivityResult result = finalize(std::move(raw), calib, full_dims, cfg);
  prov.stages["post"] = elapsed(t, clock::now());

  prov.total_seconds = elapsed(t0, clock::now());
  result.provenance = std::move(prov);
  return result;
}

// ------------------------------------------------------------ LAPACK bridge
namespace lapack {
namespace {
using zheevd_t = void (*)(const char*, const char*, const int*, Cx*, const int*, double*, Cx*,
                          const int*, double*, const int*, int*, const int*, int*, std::size_t,
                          std::size_t);
using zgemm_t = void (*)(const char*, const char*, const int*, const int*, const int*, const Cx*,
                         const Cx*, const int*, const Cx*, const int*, const Cx*, Cx*, const int*,
                         std::size_t, std::size_t);
using setthreads_t = void (*)(int);
zheevd_t g_zheevd = nullptr;
zgemm_t g_zgemm = nullptr;
setthreads_t g_set_threads = nullptr;
}  // namespace

void load(const std::string& path) {
  void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
  if (!h) throw std::runtime_error(std::string("cannot load LAPACK: ") + dlerror());
  g_zheevd = reinterpret_cast<zheevd_t>(dlsym(h, "scipy_zheevd_"));
  g_zgemm = reinterpret_cast<zgemm_t>(dlsym(h, "scipy_zgemm_"));
  g_set_threads = reinterpret_cast<setthreads_t>(dlsym(h, "scipy_openblas_set_num_threads"));
  if (!g_zheevd || !g_zgemm) throw std::runtime_error("LAPACK symbols scipy_zheevd_/scipy_zgemm_ missing");
  set_threads(1);  // Eigen in the reference runs these single-threaded (CMakeLists.txt:1-38)
}
bool loaded() { return g_zheevd != nullptr; }
void set_threads(int n) {
  if (g_set_threads) g_set_threads(n);
}

void zheevd(Index n, Cx* a, double* w, bool vectors) {
  if (!g_zheevd) throw std::runtime_error("LAPACK not loaded (call sko_init)");
  const char jobz = vectors ? 'V' : 'N', uplo = 'L';
  const int nn = int(n), lda = int(n);
  int info = 0, lwork = -1, lrwork = -1, liwork = -1, iwq = 0;
  Cx wq;
  double rwq = 0;
  g_zheevd(&jobz, &uplo, &nn, a, &lda, w, &wq, &lwork, &rwq, &lrwork, &iwq, &liwork, &info, 1, 1);
  lwork = int(wq.real()) + 1;
  lrwork = int(rwq) + 1;
  liwork = iwq + 1;
  std::vector<Cx> work(static_cast<std::size_t>(lwork));
  std::vector<double> rwork(static_cast<std::size_t>(lrwork));
  std::vector<int> iwork(static_cast<std::size_t>(liwork));
  g_zheevd(&jobz, &uplo, &nn, a, &lda, w, work.data(), &lwork, rwork.data(), &lrwork, iwork.data(),
           &liwork, &info, 1, 1);
  if (info != 0) throw std::runtime_error("Gram eigendecomposition failed");
}

void zgemm(char ta, char tb, Index m, Index n, Index k, Cx alpha, const Cx* a, Index lda, const Cx* b,
           Index ldb, Cx beta, Cx* c, Index ldc) {
  if (!g_zgemm) throw std::runtime_error("BLAS not loaded (call sko_init)");
  const int mm = int(m), nn = int(n), kk = int(k), la = int(lda), lb = int(ldb), lc = int(ldc);
  g_zgemm(&ta, &tb, &mm, &nn, &kk, &alpha, a, &la, b, &lb, &beta, c, &lc, 1, 1);
}
}  // namespace lapack

}  // namespace sko
