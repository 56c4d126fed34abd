// cuBLASLt TF32 GEMM algorithm sweep on the K2 steering-product shapes
// (C = A' V', A' the K-concatenated split Gram 2n x 2n, V' 2n x 4b): does any
// heuristic candidate beat cublasGemmEx's default choice?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lt_tf32_micro.cu -lcublasLt -lcublas -o tools/lt_tf32_micro
#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

int main() {
  const int shapes[][2] = {{5184, 256}, {7872, 256}, {3136, 256}, {14464, 512}};  // {2n, 4b}
  cublasLtHandle_t lt;
  cublasLtCreate(&lt);
  cublasHandle_t h;
  cublasCreate(&h);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void* ws;
  const size_t wsb = size_t(256) << 20;
  cudaMalloc(&ws, wsb);
  for (auto& s : shapes) {
    const int m = s[0], n = s[1], k = s[0];
    float *a, *b, *c;
    cudaMalloc(&a, size_t(m) * k * 4);
    cudaMalloc(&b, size_t(k) * n * 4);
    cudaMalloc(&c, size_t(m) * n * 4);
    cudaMemset(a, 0, size_t(m) * k * 4);
    cudaMemset(b, 0, size_t(k) * n * 4);
    const float one = 1.f, zero = 0.f;
    auto time_it = [&](auto fn) {
      for (int i = 0; i < 3; ++i) fn();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int i = 0; i < 20; ++i) fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      return 1e3f * ms / 20;
    };
    const float t0 = time_it([&] {
      cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &one, a, CUDA_R_32F, m, b, CUDA_R_32F, k, &zero, c,
                   CUDA_R_32F, m, CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT);
    });
    printf("m=%d n=%d k=%d  GemmEx default %.2f us (%.0f TFLOP/s)\n", m, n, k, t0, 2.0 * m * n * k / t0 / 1e6);
    cublasLtMatmulDesc_t op;
    cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F_FAST_TF32, CUDA_R_32F);
    cublasLtMatrixLayout_t la, lb, lc;
    cublasLtMatrixLayoutCreate(&la, CUDA_R_32F, m, k, m);
    cublasLtMatrixLayoutCreate(&lb, CUDA_R_32F, k, n, k);
    cublasLtMatrixLayoutCreate(&lc, CUDA_R_32F, m, n, m);
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb));
    std::vector<cublasLtMatmulHeuristicResult_t> res(32);
    int got = 0;
    cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 32, res.data(), &got);
    float best = 1e30f;
    int bi = -1;
    for (int i = 0; i < got; ++i) {
      if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
      const float t = time_it([&] {
        cublasLtMatmul(lt, op, &one, a, la, b, lb, &zero, c, lc, c, lc, &res[i].algo, ws, wsb, 0);
      });
      if (t < best) {
        best = t;
        bi = i;
      }
    }
    printf("   cublasLt: %d candidates, best #%d %.2f us (%.0f TFLOP/s)\n", got, bi, best, 2.0 * m * n * k / best / 1e6);
    cudaFree(a);
    cudaFree(b);
    cudaFree(c);
  }
  return 0;
}
