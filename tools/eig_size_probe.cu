// Probe (dev tool): cuSOLVER symmetric eigensolver time against n at the RHOSVD Gram sizes,
// full vectors / values only / top-k vectors (Xsyevdx), one call at a time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/eig_size_probe tools/eig_size_probe.cu -lcusolver -lcublas
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { auto e = (x); if (e) { printf("err %d at %s:%d\n", int(e), __FILE__, __LINE__); exit(1);} } while (0)

int main(int argc, char** argv) {
  std::vector<long> sizes = {800, 1300, 1600, 2000, 2600, 2842, 3526, 4200, 5394, 8283};
  if (argc > 1) { sizes.clear(); for (int i = 1; i < argc; ++i) sizes.push_back(atol(argv[i])); }
  cusolverDnHandle_t hs; cublasHandle_t hb;
  cusolverDnParams_t par;
  CK(cusolverDnCreate(&hs)); CK(cublasCreate(&hb)); CK(cusolverDnCreateParams(&par));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (long n : sizes) {
    // A = B diag(exp(-k/40)) B^T: a Gram-like spectrum spanning ~1e-30
    std::vector<double> hB(size_t(n) * n);
    std::mt19937_64 g(n);
    std::normal_distribution<double> nd;
    for (auto& v : hB) v = nd(g);
    double *B, *BS, *A, *A0, *W;
    CK(cudaMalloc(&B, 8 * n * n)); CK(cudaMalloc(&BS, 8 * n * n)); CK(cudaMalloc(&A, 8 * n * n));
    CK(cudaMalloc(&A0, 8 * n * n)); CK(cudaMalloc(&W, 8 * n));
    CK(cudaMemcpy(B, hB.data(), 8 * n * n, cudaMemcpyHostToDevice));
    std::vector<double> sc(n);
    for (long k = 0; k < n; ++k) sc[k] = std::exp(-double(k) * 60.0 / n);
    double* dsc; CK(cudaMalloc(&dsc, 8 * n)); CK(cudaMemcpy(dsc, sc.data(), 8 * n, cudaMemcpyHostToDevice));
    CK(cublasDdgmm(hb, CUBLAS_SIDE_RIGHT, n, n, B, n, dsc, 1, BS, n));
    const double one = 1, zero = 0;
    CK(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, n, n, n, &one, BS, n, BS, n, &zero, A0, n));
    int* info; CK(cudaMalloc(&info, sizeof(int)));
    for (int mode = 0; mode < 3; ++mode) {
      size_t db = 0, hbsz = 0;
      const long k = n * 2 / 5;
      int64_t found = 0;
      double vl = 0, vu = 0;
      if (mode < 2)
        CK(cusolverDnXsyevd_bufferSize(hs, par, mode == 0 ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR,
                                       CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, W, CUDA_R_64F, &db, &hbsz));
      else
        CK(cusolverDnXsyevdx_bufferSize(hs, par, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n,
                                        CUDA_R_64F, A, n, &vl, &vu, n - k + 1, n, &found, CUDA_R_64F, W, CUDA_R_64F, &db, &hbsz));
      void* dw; CK(cudaMalloc(&dw, db));
      std::vector<char> hw(hbsz + 1);
      float best = 1e30f;
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemcpy(A, A0, 8 * n * n, cudaMemcpyDeviceToDevice));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        if (mode < 2)
          CK(cusolverDnXsyevd(hs, par, mode == 0 ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR,
                              CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, W, CUDA_R_64F, dw, db,
                              hw.data(), hbsz, info));
        else
          CK(cusolverDnXsyevdx(hs, par, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n,
                               CUDA_R_64F, A, n, &vl, &vu, n - k + 1, n, &found, CUDA_R_64F, W, CUDA_R_64F, dw, db,
                               hw.data(), hbsz, info));
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      printf("n=%5ld %-22s %9.2f ms\n", n, mode == 0 ? "Xsyevd vectors" : mode == 1 ? "Xsyevd values only" : "Xsyevdx top 40%", best);
      fflush(stdout);
      CK(cudaFree(dw));
    }
    cudaFree(B); cudaFree(BS); cudaFree(A); cudaFree(A0); cudaFree(W); cudaFree(dsc); cudaFree(info);
  }
  return 0;
}
