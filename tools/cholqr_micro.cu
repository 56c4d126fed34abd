// Warm, back-to-back timing of the sk_cholqr.cu kernels in isolation (the
// file is compiled in; host helpers of the runtime are stubbed).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/cholqr_micro tools/cholqr_micro.cu -lcublas -lcusolver
#include "../paper_2302_13431_b200/csrc/sk_cholqr.cu"

#include <cstdio>
#include <vector>

namespace skb {
void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    std::exit(1);
  }
}
void* Arena::get(const std::string&, size_t) { return nullptr; }
void fail(int, const std::string& m) {
  std::fprintf(stderr, "%s\n", m.c_str());
  std::exit(1);
}
Arena::~Arena() {}
void set_smem_limit(const void* f, size_t bytes) {
  check_cuda(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)), "smem");
}
}  // namespace skb

namespace skb { namespace {
__global__ void factor4_alone(const double2* s_in, long long* cyc, int* flag) {
  __shared__ double2 colb[2][4][kQ];
  __shared__ double2 Ls[kQ * kQLd];
  __shared__ double rsv[kQ];
  const int lane = threadIdx.x;
  double2 a[4][2];
  long long tot = 0;
  for (int w = 0; w < 16; ++w) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) a[c][h] = s_in[(lane + 32 * h) + kQ * (4 * w + c)];
    __syncwarp();
    const long long c0 = clock64();
    chol64_factor4(a, colb[w & 1], Ls, rsv, w, lane, flag);
    __syncwarp();
    const double2 v = colb[w & 1][3][63];
    if (v.x == 1234.5) flag[1] = 1;
    tot += clock64() - c0;
  }
  if (lane == 0) cyc[0] = tot / 16;
}
}  // namespace
}  // namespace skb

template <typename F>
float time_it(F f, int reps = 200) {
  for (int i = 0; i < 5; ++i) f();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

int main() {
  using namespace skb;
  const i64 n = 2592;
  std::vector<double2> hx(size_t(n * 64));
  unsigned s = 1;
  for (auto& v : hx) {
    s = s * 1664525u + 1013904223u;
    v.x = (s >> 8) * (1.0 / 16777216.0) - 0.5;
    s = s * 1664525u + 1013904223u;
    v.y = (s >> 8) * (1.0 / 16777216.0) - 0.5;
  }
  double2 *x, *S, *L, *D, *cp;
  unsigned* counter;
  int* flag;
  cudaMalloc(&x, hx.size() * sizeof(double2));
  cudaMalloc(&S, 64 * 64 * sizeof(double2));
  cudaMalloc(&L, 64 * 64 * sizeof(double2));
  cudaMalloc(&D, 4 * 256 * sizeof(double2));
  cudaMalloc(&cp, 64 * 16 * 256 * sizeof(double2));
  cudaMalloc(&counter, 4);
  cudaMalloc(&flag, 4);
  cudaMemset(counter, 0, 4);
  cudaMemset(flag, 0, 4);
  cudaMemcpy(x, hx.data(), hx.size() * sizeof(double2), cudaMemcpyHostToDevice);
  const int rows = int((n + 143) / 144);
  const size_t smem_g = size_t(1 * kQStage * kQLd + 10 * kQGramThreads) * sizeof(double2);
  set_smem_limit(reinterpret_cast<const void*>(gram64_kernel<true>), smem_g);
  auto gram = [&] { gram64_kernel<true><<<144, kQGramThreads, smem_g>>>(x, x, n, rows, cp, counter, S, 0); };
  const size_t smem_c = size_t(kQ * kQLd + 4 * 16 * 17) * sizeof(double2);
  set_smem_limit(reinterpret_cast<const void*>(chol64_kernel), smem_c);
  auto chol = [&] { chol64_kernel<<<1, kQCholThreads, smem_c>>>(S, L, D, flag); };
  const int trows = 18;
  const size_t smem_t = size_t(kQ * kQLd + 4 * 16 * 17 + trows * kQLd) * sizeof(double2);
  set_smem_limit(reinterpret_cast<const void*>(trsm64_kernel), smem_t);
  auto trsm = [&] { trsm64_kernel<<<unsigned((n + trows - 1) / trows), 288, smem_t>>>(x, n, trows, L, D, 0); };
  gram();
  chol();
  cudaDeviceSynchronize();
  std::printf("gram64<herm>     %7.2f us\n", time_it(gram));
  std::printf("chol64           %7.2f us\n", time_it(chol));
  std::printf("trsm64           %7.2f us  (operates in place; values drift, timing only)\n", time_it(trsm));
  {
    long long* c;
    cudaMallocManaged(&c, 8);
    factor4_alone<<<1, 32>>>(S, c, flag);
    cudaDeviceSynchronize();
    factor4_alone<<<1, 32>>>(S, c, flag);
    cudaDeviceSynchronize();
    std::printf("factor4 alone (one warp): %lld cycles per 4-pivot block\n", c[0]);
  }
  std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
