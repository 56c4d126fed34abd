// Compiled C++ client of the drop-in boundary (include/senskit_b200.h): the
// way a reference-side shim calls the library, with no
// Python in between.  Built and run by tests/test_abi_cpp.py:
//   g++ -std=c++17 tests/abi_smoke.cpp -Iinclude -I/usr/local/cuda/include -Lpaper_2302_13431_b200/lib
//       -lsenskit_b200 -L/usr/local/cuda/lib64 -lcudart -o abi_smoke
//   ./abi_smoke            (exit 0 = every check passed; needs a GPU)
//   ./abi_smoke --no-gpu   (host-only entry points and argument errors)
//
// Input: a noiseless band-limited 8-coil scene evaluated directly in k-space
// on a 24 x 24 calibration block (smooth coil maps x a centred disc), so the
// Gram has a genuine nullspace.  Checks: return codes and error mapping
// (types.hpp:22-32 <-> SK_ERR_*), make_support (kernels.cpp:7-35), the
// pisco pipeline on host and on device buffers (identical results), outputs
// finite, maps of unit sum-of-squares, the mask = lambda < threshold, and the
// subspace solver reported in the provenance.
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "senskit_b200.h"

namespace {
int failures = 0;
void check(bool ok, const std::string& what) {
  if (!ok) {
    std::fprintf(stderr, "FAIL: %s (%s)\n", what.c_str(), sk_last_error());
    ++failures;
  }
}

sk_config pisco(int tau, int iters, int64_t pad) {
  sk_config c;
  std::memset(&c, 0, sizeof c);
  c.kernel = 1;  // ellipsoid
  c.tau = tau;
  c.gram = 1;  // fft
  c.nullspace_threshold = 0.05;
  c.grid = 1;  // reduced
  c.grid_pad = pad;
  c.eig = 1;  // power
  c.power_iters = iters;
  c.method = 0;
  c.field = 1;
  c.mask_threshold = 0.01;
  c.apod_width = -1.0;
  return c;
}

// k-space of c_q(x) * disc(x) on the centred E x E block of an N x N grid,
// evaluated as a direct (small) DFT of the image.
std::vector<sk_c64> scene(int q, int N, int E) {
  const double pi = 3.14159265358979323846;
  std::vector<std::complex<double>> img(size_t(q) * N * N);
  for (int c = 0; c < q; ++c) {
    const double ang = 2 * pi * c / q, cx = 1.5 * std::cos(ang), cy = 1.5 * std::sin(ang);
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        const double x = double(i - N / 2) / N, y = double(j - N / 2) / N;
        const double r2 = (x - cx) * (x - cx) + (y - cy) * (y - cy);
        const double rho = (x * x + y * y < 0.3 * 0.3) ? 1.0 : 0.0;
        img[(size_t(c) * N + i) * N + j] = std::polar(rho / (1.0 + r2 / 0.36), ang + x);
      }
  }
  std::vector<sk_c64> cal(size_t(q) * E * E);
  for (int c = 0; c < q; ++c)
    for (int a = 0; a < E; ++a)
      for (int b = 0; b < E; ++b) {
        const int fa = a - E / 2, fb = b - E / 2;
        std::complex<double> s = 0.0;
        for (int i = 0; i < N; ++i)
          for (int j = 0; j < N; ++j)
            s += img[(size_t(c) * N + i) * N + j] *
                 std::polar(1.0, -2 * pi * (double(fa) * (i - N / 2) + double(fb) * (j - N / 2)) / N);
        s /= N;
        cal[(size_t(c) * E + a) * E + b] = {float(s.real()), float(s.imag())};
      }
  return cal;
}
}  // namespace

int main(int argc, char** argv) {
  const bool gpu = !(argc > 1 && std::string(argv[1]) == "--no-gpu");
  // host-only entry points
  int64_t count = 0;
  check(sk_make_support(1, 3, 2, nullptr, &count) == SK_OK && count == 29, "make_support ellipsoid tau 3 -> 29");
  std::vector<int32_t> offs(size_t(count) * 2);
  check(sk_make_support(1, 3, 2, offs.data(), &count) == SK_OK && offs[0] == -3 && offs[1] == 0,
        "make_support lexicographic order");
  check(sk_make_support(0, -1, 2, nullptr, &count) == SK_ERR_DIM, "make_support tau < 0 -> SK_ERR_DIM");
  const int64_t cd[2] = {24, 24}, fd[2] = {64, 64};
  int64_t red[2] = {0, 0};
  check(sk_reduced_grid_dims(2, cd, 24, fd, red) == SK_OK && red[0] == 48 && red[1] == 48, "reduced_grid_dims");
  check(sk_estimate_maps(nullptr, 2, cd, cd, 8, nullptr, fd, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr) ==
            SK_ERR_DIM,
        "null context -> SK_ERR_DIM");
  if (!gpu) {
    std::printf("abi_smoke (host only): %s\n", failures ? "FAILED" : "ok");
    return failures ? 1 : 0;
  }

  sk_ctx* ctx = nullptr;
  check(sk_create(0, &ctx) == SK_OK && ctx, "sk_create(0)");
  if (!ctx) return 1;
  const int q = 8;
  const int64_t co[2] = {12, 12};
  const std::vector<sk_c64> cal = scene(q, 64, 24);
  sk_config cfg = pisco(3, 30, 24);
  const int64_t nf = 64 * 64;
  std::vector<sk_c64> maps(size_t(q) * nf);
  std::vector<float> lam(static_cast<size_t>(nf));
  std::vector<uint8_t> mask(static_cast<size_t>(nf));
  sk_provenance prov;
  check(sk_estimate_maps(ctx, 2, cd, co, q, cal.data(), fd, &cfg, maps.data(), lam.data(), mask.data(), nullptr,
                         &prov) == SK_OK,
        "estimate_maps (host buffers)");
  check(prov.nullspace_rank > 0 && prov.nullspace_rank < q * 29, "0 < R < n");
  check(prov.eig_solver_used == 2, "default nullspace solver is the subspace solver");
  check(prov.grid_dims[0] == 48 && prov.grid_dims[1] == 48, "grid_dims_for (reduced, pad 24)");
  int bad = 0, masked = 0, inconsistent = 0;
  for (int64_t j = 0; j < nf; ++j) {
    double sos = 0.0;
    for (int c = 0; c < q; ++c) {
      const sk_c64 v = maps[size_t(c * nf + j)];
      if (!std::isfinite(v.re) || !std::isfinite(v.im)) ++bad;
      sos += double(v.re) * v.re + double(v.im) * v.im;
    }
    if (std::fabs(sos - 1.0) > 1e-4) ++bad;  // renormalised after interpolation (maps.cpp:240-250)
    if (!std::isfinite(lam[size_t(j)])) ++bad;
    masked += mask[size_t(j)];
    if ((lam[size_t(j)] < cfg.mask_threshold) != (mask[size_t(j)] != 0)) ++inconsistent;
  }
  check(bad == 0, "finite maps with unit sum of squares, finite lambda");
  check(inconsistent == 0, "mask == (lambda < mask_threshold)");
  check(masked > nf / 20 && masked < nf, "support mask covers the disc");

  // the same call on device buffers (cudaMalloc'd by the caller)
  {
    sk_c64 *d_cal = nullptr, *d_maps = nullptr;
    float* d_lam = nullptr;
    uint8_t* d_mask = nullptr;
    cudaMalloc(&d_cal, cal.size() * sizeof(sk_c64));
    cudaMalloc(&d_maps, maps.size() * sizeof(sk_c64));
    cudaMalloc(&d_lam, lam.size() * sizeof(float));
    cudaMalloc(&d_mask, mask.size());
    cudaMemcpy(d_cal, cal.data(), cal.size() * sizeof(sk_c64), cudaMemcpyHostToDevice);
    sk_provenance p2;
    check(sk_estimate_maps(ctx, 2, cd, co, q, d_cal, fd, &cfg, d_maps, d_lam, d_mask, nullptr, &p2) == SK_OK,
          "estimate_maps (device buffers)");
    std::vector<sk_c64> m2(maps.size());
    std::vector<float> l2(lam.size());
    std::vector<uint8_t> k2(mask.size());
    cudaMemcpy(m2.data(), d_maps, m2.size() * sizeof(sk_c64), cudaMemcpyDeviceToHost);
    cudaMemcpy(l2.data(), d_lam, l2.size() * sizeof(float), cudaMemcpyDeviceToHost);
    cudaMemcpy(k2.data(), d_mask, k2.size(), cudaMemcpyDeviceToHost);
    double num = 0.0, den = 0.0, lerr = 0.0;
    int mdiff = 0;
    for (size_t i = 0; i < maps.size(); ++i) {
      const double dr = double(m2[i].re) - maps[i].re, di = double(m2[i].im) - maps[i].im;
      num += dr * dr + di * di;
      den += double(maps[i].re) * maps[i].re + double(maps[i].im) * maps[i].im;
    }
    for (size_t i = 0; i < lam.size(); ++i) {
      lerr = std::fmax(lerr, std::fabs(double(l2[i]) - lam[i]) / std::fmax(1e-30, std::fabs(double(lam[i]))));
      mdiff += k2[i] != mask[i];
    }
    // converged results (the subspace step plan may differ with the call history)
    check(p2.nullspace_rank == prov.nullspace_rank, "device-buffer call: same R");
    check(std::sqrt(num / den) < 1e-5 && lerr < 1e-4 && mdiff == 0, "device-buffer call: same maps / lambda / mask");
    cudaFree(d_cal);
    cudaFree(d_maps);
    cudaFree(d_lam);
    cudaFree(d_mask);
  }

  // same call with the C-ABI's error classes
  sk_config badcfg = cfg;
  badcfg.nullspace_threshold = 1.5;
  check(sk_estimate_maps(ctx, 2, cd, co, q, cal.data(), fd, &badcfg, maps.data(), lam.data(), mask.data(), nullptr,
                         nullptr) == SK_ERR_DIM,
        "threshold ratio outside (0,1) -> SK_ERR_DIM (nullspace.cpp:9-10)");
  const int64_t small_full[2] = {16, 16};
  check(sk_estimate_maps(ctx, 2, cd, co, q, cal.data(), small_full, &cfg, nullptr, nullptr, nullptr, nullptr,
                         nullptr) == SK_ERR_DIM,
        "full_dims smaller than the calibration -> SK_ERR_DIM (maps.cpp:268-271)");
  sk_destroy(ctx);
  std::printf("abi_smoke: R=%lld masked=%d total=%.3f ms launches ok: %s\n", (long long)prov.nullspace_rank, masked,
              prov.total_ms, failures ? "FAILED" : "ok");
  return failures ? 1 : 0;
}
