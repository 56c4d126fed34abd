// cuBLAS INT8 GEMM (int32 accumulate) on the K2 product shapes: is it fast
// enough to emulate the FP64 subspace steps by sliced integer products?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/i8gemm_micro.cu -lcublas -o tools/i8gemm_micro
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>

int main() {
  cublasHandle_t h;
  cublasCreate(&h);
  const int shapes[][3] = {{5184, 128, 2592}, {14464, 256, 7232}, {3136, 128, 1568}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& s : shapes) {
    const int m = s[0], n = s[1], k = s[2];
    int8_t *a, *b;
    int32_t* c;
    cudaMalloc(&a, size_t(m) * k);
    cudaMalloc(&b, size_t(k) * n);
    cudaMalloc(&c, size_t(m) * n * 4);
    cudaMemset(a, 1, size_t(m) * k);
    cudaMemset(b, 1, size_t(k) * n);
    const int32_t one = 1, zero = 0;
    for (int mode = 0; mode < 2; ++mode) {  // 0: NN (A m x k col-major), 1: TN (A stored k x m)
      const cublasOperation_t ta = mode ? CUBLAS_OP_T : CUBLAS_OP_N;
      const int lda = mode ? k : m;
      cublasStatus_t st = CUBLAS_STATUS_SUCCESS;
      for (int it = 0; it < 3; ++it)
        st = cublasGemmEx(h, ta, CUBLAS_OP_N, m, n, k, &one, a, CUDA_R_8I, lda, b, CUDA_R_8I, k, &zero, c, CUDA_R_32I,
                          m, CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT);
      cudaDeviceSynchronize();
      const int reps = 20;
      cudaEventRecord(e0);
      for (int it = 0; it < reps; ++it)
        cublasGemmEx(h, ta, CUBLAS_OP_N, m, n, k, &one, a, CUDA_R_8I, lda, b, CUDA_R_8I, k, &zero, c, CUDA_R_32I, m,
                     CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      int32_t h0 = 0;
      cudaMemcpy(&h0, c, 4, cudaMemcpyDeviceToHost);
      printf("m=%d n=%d k=%d %s status=%d  %.2f us  %.1f TOPS  c[0]=%d (expect %d)\n", m, n, k, mode ? "TN" : "NN",
             int(st), 1e3 * ms / reps, 2.0 * m * n * k / (ms / reps * 1e-3) / 1e12, h0, k);
    }
    cudaFree(a);
    cudaFree(b);
    cudaFree(c);
  }
  return 0;
}
