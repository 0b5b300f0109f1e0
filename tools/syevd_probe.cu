// Probe: cuSOLVER symmetric eigensolver options at the Gram sizes of the path (dev tool).
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#include <cmath>

#define CK(x) do { auto e = (x); if (e) { printf("err %d at %s:%d\n", int(e), __FILE__, __LINE__); exit(1);} } while (0)

static void fill(double* dA, int64_t n, int64_t batch, unsigned seed) {
  std::vector<double> h(n * n * batch);
  srand(seed);
  for (int64_t b = 0; b < batch; ++b) {
    // Gram-like SPD with a decaying spectrum: A = Q diag(exp(-i/10)) Q^T approx via B B^T
    std::vector<double> B(n * n);
    for (auto& v : B) v = (rand() / double(RAND_MAX) - 0.5);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i <= j; ++i) {
        double s = 0;
        for (int64_t k = 0; k < n; k += 7) s += B[i + k * n] * B[j + k * n] * std::exp(-double(k) / 50);
        h[b * n * n + i + j * n] = h[b * n * n + j + i * n] = s;
      }
  }
  CK(cudaMemcpy(dA, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
}

int main() {
  cusolverDnHandle_t hs[3];
  cudaStream_t st[3];
  cusolverDnParams_t par;
  CK(cusolverDnCreateParams(&par));
  for (int i = 0; i < 3; ++i) {
    CK(cusolverDnCreate(&hs[i]));
    CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    CK(cusolverDnSetStream(hs[i], st[i]));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int64_t n : {400, 693, 1000, 1625, 2048}) {
    double *A, *A0, *W;
    CK(cudaMalloc(&A, 3 * n * n * 8)); CK(cudaMalloc(&A0, 3 * n * n * 8)); CK(cudaMalloc(&W, 3 * n * 8));
    fill(A0, n, 3, 1);
    int* info; CK(cudaMalloc(&info, 3 * sizeof(int)));
    size_t db = 0, hb = 0;
    CK(cusolverDnXsyevd_bufferSize(hs[0], par, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, W, CUDA_R_64F, &db, &hb));
    void* dw[3]; std::vector<char> hw[3];
    for (int i = 0; i < 3; ++i) { CK(cudaMalloc(&dw[i], db)); hw[i].resize(hb + 1); }
    // sequential 3x syevd
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0, st[0]);
      for (int i = 0; i < 3; ++i)
        CK(cusolverDnXsyevd(hs[0], par, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A + i * n * n, n, CUDA_R_64F, W + i * n, CUDA_R_64F, dw[i], db, hw[i].data(), hb, info + i));
      cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("n=%5ld  3x Xsyevd sequential: %8.2f ms\n", n, ms);
    }
    // 3 threads / streams
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
      CK(cudaDeviceSynchronize());
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int i = 0; i < 3; ++i) th.emplace_back([&, i] {
        cusolverDnXsyevd(hs[i], par, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A + i * n * n, n, CUDA_R_64F, W + i * n, CUDA_R_64F, dw[i], db, hw[i].data(), hb, info + i);
        cudaStreamSynchronize(st[i]);
      });
      for (auto& t : th) t.join();
      double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (rep == 2) printf("n=%5ld  3x Xsyevd 3 streams : %8.2f ms\n", n, ms);
    }
    // batched
    size_t dbb = 0, hbb = 0;
    auto stb = cusolverDnXsyevBatched_bufferSize(hs[0], par, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, W, CUDA_R_64F, &dbb, &hbb, 3);
    if (stb == CUSOLVER_STATUS_SUCCESS) {
      void* dwb; CK(cudaMalloc(&dwb, dbb + 8)); std::vector<char> hwb(hbb + 1);
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0, st[0]);
        auto s2 = cusolverDnXsyevBatched(hs[0], par, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, W, CUDA_R_64F, dwb, dbb, hwb.data(), hbb, info, 3);
        cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("n=%5ld  XsyevBatched(3)    : %8.2f ms (status %d)\n", n, ms, int(s2));
      }
      cudaFree(dwb);
    } else printf("n=%5ld  XsyevBatched unsupported (status %d)\n", n, int(stb));
    // eigenvalues only
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0, st[0]);
      CK(cusolverDnXsyevd(hs[0], par, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, W, CUDA_R_64F, dw[0], db, hw[0].data(), hb, info));
      cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("n=%5ld  1x Xsyevd novector : %8.2f ms\n", n, ms);
    }
    for (int i = 0; i < 3; ++i) cudaFree(dw[i]);
    cudaFree(A); cudaFree(A0); cudaFree(W); cudaFree(info);
  }
  return 0;
}
