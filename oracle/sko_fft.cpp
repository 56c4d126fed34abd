// ORACLE — TEST INFRASTRUCTURE ONLY (see sko.hpp).
//
// Restates fft.cpp:37-112.  The reference delegates each 1-D line to
// Eigen::FFT<double> (kissfft backend, a recursive mixed-radix
// decimation-in-time FFT); this file implements that published algorithm from
// scratch: factor n into radices 4,2,3,5 then remaining odd primes, recurse on
// the strided sub-sequences, and combine with radix-specific butterflies.
// Inverse = conj o fwd o conj, exactly as fft.cpp:45-50.
#include <atomic>
#include <cmath>
#include <memory>
#include <mutex>
#include <unordered_map>

#include "sko.hpp"

namespace sko::fft {

namespace {

std::atomic<std::int64_t> g_forward{0};
std::atomic<std::int64_t> g_inverse{0};

struct Plan {
  Index n = 0;
  std::vector<Index> factors;  // pairs (radix, remaining length)
  std::vector<Cx> tw;          // exp(-2 pi i k / n)
};

std::shared_ptr<const Plan> make_plan(Index n) {
  auto p = std::make_shared<Plan>();
  p->n = n;
  p->tw.resize(std::size_t(n));
  for (Index k = 0; k < n; ++k) {
    const double ang = -2.0 * M_PI * double(k) / double(n);
    p->tw[std::size_t(k)] = Cx(std::cos(ang), std::sin(ang));
  }
  Index rem = n, r = 4;
  const double floor_sqrt = std::floor(std::sqrt(double(n)));
  while (rem > 1) {
    while (rem % r) {
      switch (r) {
        case 4: r = 2; break;
        case 2: r = 3; break;
        default: r += 2; break;
      }
      if (double(r) > floor_sqrt) r = rem;
    }
    rem /= r;
    p->factors.push_back(r);
    p->factors.push_back(rem);
  }
  return p;
}

std::shared_ptr<const Plan> plan_for(Index n) {
  static std::mutex mu;
  static std::unordered_map<Index, std::shared_ptr<const Plan>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  auto p = make_plan(n);
  cache.emplace(n, p);
  return p;
}

void butterfly2(Cx* out, Index fstride, const Plan& p, Index m) {
  Cx* a = out;
  Cx* b = out + m;
  for (Index k = 0; k < m; ++k) {
    const Cx t = b[k] * p.tw[std::size_t(k * fstride)];
    b[k] = a[k] - t;
    a[k] += t;
  }
}

void butterfly4(Cx* out, Index fstride, const Plan& p, Index m) {
  for (Index k = 0; k < m; ++k) {
    const Cx y0 = out[k];
    const Cx t1 = out[k + m] * p.tw[std::size_t(k * fstride)];
    const Cx t2 = out[k + 2 * m] * p.tw[std::size_t(2 * k * fstride)];
    const Cx t3 = out[k + 3 * m] * p.tw[std::size_t(3 * k * fstride)];
    const Cx s02 = y0 + t2, d02 = y0 - t2;
    const Cx s13 = t1 + t3, d13 = t1 - t3;
    const Cx mi_d13(d13.imag(), -d13.real());  // -i * d13
    out[k] = s02 + s13;
    out[k + 2 * m] = s02 - s13;
    out[k + m] = d02 + mi_d13;
    out[k + 3 * m] = d02 - mi_d13;
  }
}

void butterfly_generic(Cx* out, Index fstride, const Plan& p, Index m, Index radix) {
  std::vector<Cx> scratch(static_cast<std::size_t>(radix));
  const Index n = p.n;
  for (Index k = 0; k < m; ++k) {
    for (Index u = 0; u < radix; ++u) scratch[std::size_t(u)] = out[k + u * m];
    for (Index q = 0; q < radix; ++q) {
      const Index kk = k + q * m;
      Cx acc = scratch[0];
      Index tw_idx = 0;
      const Index step = (kk * fstride) % n;
      for (Index u = 1; u < radix; ++u) {
        tw_idx += step;
        if (tw_idx >= n) tw_idx -= n;
        acc += scratch[std::size_t(u)] * p.tw[std::size_t(tw_idx)];
      }
      out[kk] = acc;
    }
  }
}

void work(const Plan& p, Cx* out, const Cx* in, Index fstride, Index in_stride, const Index* f) {
  const Index radix = f[0];
  const Index m = f[1];
  if (m == 1) {
    for (Index i = 0; i < radix; ++i) out[i] = in[i * fstride * in_stride];
  } else {
    for (Index i = 0; i < radix; ++i)
      work(p, out + i * m, in + i * fstride * in_stride, fstride * radix, in_stride, f + 2);
  }
  switch (radix) {
    case 2: butterfly2(out, fstride, p, m); break;
    case 4: butterfly4(out, fstride, p, m); break;
    default: butterfly_generic(out, fstride, p, m, radix); break;
  }
}

// Forward (sign -1) unnormalized DFT of one contiguous line.
void fwd_line(const Plan& p, Cx* out, const Cx* in) {
  if (p.n == 1) {
    out[0] = in[0];
    return;
  }
  work(p, out, in, 1, 1, p.factors.data());
}

// fft.cpp:16-33: gather each line along `axis`, transform, scatter back.
template <typename Fn>
void for_each_line(Cx* data, const Dims& dims, std::size_t axis, Fn&& fn) {
  const Index n = dims[axis];
  Index outer = 1, inner = 1;
  for (std::size_t a = 0; a < axis; ++a) outer *= dims[a];
  for (std::size_t a = axis + 1; a < dims.size(); ++a) inner *= dims[a];
  std::vector<Cx> line(static_cast<std::size_t>(n)), out(static_cast<std::size_t>(n));
  for (Index o = 0; o < outer; ++o) {
    for (Index i = 0; i < inner; ++i) {
      Cx* base = data + o * n * inner + i;
      for (Index k = 0; k < n; ++k) line[std::size_t(k)] = base[k * inner];
      fn(line.data(), out.data());
      for (Index k = 0; k < n; ++k) base[k * inner] = out[std::size_t(k)];
    }
  }
}

// fft.cpp:58-76: dir = +1 fftshift (out[a] = in[(a - c) mod n]), -1 ifftshift.
void shift_impl(Cx* data, const Dims& dims, int dir) {
  const Index n = numel(dims);
  const auto strides = strides_of(dims);
  std::vector<Cx> scratch(data, data + n);
  std::vector<Index> idx(dims.size(), 0);
  Index dst = 0;
  do {
    Index src = 0;
    for (std::size_t a = 0; a < dims.size(); ++a) {
      const Index c = center_index(dims[a]);
      const Index s = dir > 0 ? (idx[a] - c + dims[a]) % dims[a] : (idx[a] + c) % dims[a];
      src += s * strides[a];
    }
    data[dst++] = scratch[std::size_t(src)];
  } while (next_index(idx, dims));
}

void scale(Cx* data, Index n, double s) {
  for (Index i = 0; i < n; ++i) data[i] *= s;
}

}  // namespace

// fft.cpp:37-54
void transform_nd(Cx* data, const Dims& dims, int sign) {
  for (std::size_t axis = 0; axis < dims.size(); ++axis) {
    if (dims[axis] == 1) continue;
    const auto plan = plan_for(dims[axis]);
    const Index n = dims[axis];
    if (sign < 0) {
      for_each_line(data, dims, axis, [&](Cx* in, Cx* out) { fwd_line(*plan, out, in); });
    } else {
      for_each_line(data, dims, axis, [&](Cx* in, Cx* out) {
        for (Index k = 0; k < n; ++k) in[k] = std::conj(in[k]);
        fwd_line(*plan, out, in);
        for (Index k = 0; k < n; ++k) out[k] = std::conj(out[k]);
      });
    }
  }
  (sign < 0 ? g_forward : g_inverse).fetch_add(1, std::memory_order_relaxed);
}

void fftshift_nd(Cx* data, const Dims& dims) { shift_impl(data, dims, +1); }
void ifftshift_nd(Cx* data, const Dims& dims) { shift_impl(data, dims, -1); }

// fft.cpp:81-88
void image_to_kspace(Cx* data, const Dims& dims) {
  ifftshift_nd(data, dims);
  transform_nd(data, dims, -1);
  fftshift_nd(data, dims);
  scale(data, numel(dims), 1.0 / double(numel(dims)));
}

// fft.cpp:90-94
void kspace_to_image(Cx* data, const Dims& dims) {
  ifftshift_nd(data, dims);
  transform_nd(data, dims, +1);
  fftshift_nd(data, dims);
}

// fft.cpp:96-112
void image_to_kspace_unitary(Cx* data, const Dims& dims) {
  ifftshift_nd(data, dims);
  transform_nd(data, dims, -1);
  fftshift_nd(data, dims);
  scale(data, numel(dims), 1.0 / std::sqrt(double(numel(dims))));
}

void kspace_to_image_unitary(Cx* data, const Dims& dims) {
  ifftshift_nd(data, dims);
  transform_nd(data, dims, +1);
  fftshift_nd(data, dims);
  scale(data, numel(dims), 1.0 / std::sqrt(double(numel(dims))));
}

std::int64_t forward_transforms() { return g_forward.load(); }
std::int64_t inverse_transforms() { return g_inverse.load(); }
void reset_transform_counters() {
  g_forward.store(0);
  g_inverse.store(0);
}

}  // namespace sko::fft
