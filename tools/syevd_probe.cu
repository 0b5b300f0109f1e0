// Probe: cuSOLVER symmetric eigensolver options at the Gram sizes of the path (dev tool).
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#include <cmath>
#include <chrono>

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
  for (int64_t n : {357, 693, 1625}) {
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
    // Jacobi (syevj)
    {
      syevjInfo_t sj;
      CK(cusolverDnCreateSyevjInfo(&sj));
      cusolverDnXsyevjSetTolerance(sj, 1e-14);
      cusolverDnXsyevjSetMaxSweeps(sj, 20);
      int lw = 0;
      CK(cusolverDnDsyevj_bufferSize(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, &lw, sj));
      double* wj; CK(cudaMalloc(&wj, size_t(lw) * 8 + 8));
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0, st[0]);
        CK(cusolverDnDsyevj(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, wj, lw, info, sj));
        cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        int sweeps = 0; double res = 0;
        cusolverDnXsyevjGetSweeps(hs[0], sj, &sweeps); cusolverDnXsyevjGetResidual(hs[0], sj, &res);
        if (rep == 2) printf("n=%5ld  1x Dsyevj          : %8.2f ms (sweeps %d residual %.2e)\n", n, ms, sweeps, res);
      }
      cudaFree(wj);
      cusolverDnDestroySyevjInfo(sj);
    }
    // 32-bit legacy Dsyevd
    {
      int lw = 0;
      CK(cusolverDnDsyevd_bufferSize(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, &lw));
      double* wd; CK(cudaMalloc(&wd, size_t(lw) * 8 + 8));
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0, st[0]);
        CK(cusolverDnDsyevd(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, wd, lw, info));
        cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("n=%5ld  1x Dsyevd (legacy) : %8.2f ms\n", n, ms);
      }
      cudaFree(wd);
    }
    // legacy Dsyevd (no host workspace) from 3 threads / streams
    {
      int lw = 0;
      CK(cusolverDnDsyevd_bufferSize(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, &lw));
      double* wd3[3];
      for (int i = 0; i < 3; ++i) CK(cudaMalloc(&wd3[i], size_t(lw) * 8 + 8));
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
        CK(cudaDeviceSynchronize());
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int i = 0; i < 3; ++i) th.emplace_back([&, i] {
          cusolverDnDsyevd(hs[i], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A + i * n * n, n, W + i * n, wd3[i], lw, info + i);
          cudaStreamSynchronize(st[i]);
        });
        for (auto& t : th) t.join();
        double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (rep == 2) printf("n=%5ld  3x Dsyevd legacy 3 streams: %8.2f ms\n", n, ms);
      }
      // sytrd alone from 3 threads
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
        CK(cudaDeviceSynchronize());
        int lt = 0;
        double *dd, *ee, *tt;
        CK(cudaMalloc(&dd, 3 * n * 8)); CK(cudaMalloc(&ee, 3 * n * 8)); CK(cudaMalloc(&tt, 3 * n * 8));
        CK(cusolverDnDsytrd_bufferSize(hs[0], CUBLAS_FILL_MODE_LOWER, n, A, n, dd, ee, tt, &lt));
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int i = 0; i < 3; ++i) th.emplace_back([&, i] {
          cusolverDnDsytrd(hs[i], CUBLAS_FILL_MODE_LOWER, n, A + i * n * n, n, dd + i * n, ee + i * n, tt + i * n, wd3[i], lt < lw ? lt : lw, info + i);
          cudaStreamSynchronize(st[i]);
        });
        for (auto& t : th) t.join();
        double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (rep == 2) printf("n=%5ld  3x Dsytrd 3 streams       : %8.2f ms\n", n, ms);
        cudaFree(dd); cudaFree(ee); cudaFree(tt);
      }
      for (int i = 0; i < 3; ++i) cudaFree(wd3[i]);
    }
    // legacy Dsyevd captured into a CUDA graph (launch-latency test)
    {
      int lw = 0;
      CK(cusolverDnDsyevd_bufferSize(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, &lw));
      double* wd; CK(cudaMalloc(&wd, size_t(lw) * 8 + 8));
      CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
      CK(cudaDeviceSynchronize());
      cudaGraph_t g = nullptr;
      cudaGraphExec_t ge = nullptr;
      auto c0 = cudaStreamBeginCapture(st[0], cudaStreamCaptureModeRelaxed);
      auto c1 = cusolverDnDsyevd(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, wd, lw, info);
      auto c2 = cudaStreamEndCapture(st[0], &g);
      size_t nodes = 0;
      if (g) cudaGraphGetNodes(g, nullptr, &nodes);
      printf("n=%5ld  graph capture of Dsyevd: begin %d solver %d end %d nodes %zu\n", n, int(c0), int(c1), int(c2), nodes);
      cudaGetLastError();
      if (c2 == cudaSuccess && g && cudaGraphInstantiate(&ge, g, 0) == cudaSuccess) {
        for (int rep = 0; rep < 3; ++rep) {
          CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
          CK(cudaDeviceSynchronize());
          cudaEventRecord(e0, st[0]);
          CK(cudaGraphLaunch(ge, st[0]));
          cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          if (rep == 2) printf("n=%5ld  1x Dsyevd graph    : %8.2f ms\n", n, ms);
        }
        // 3 graphs on 3 streams concurrently
        for (int rep = 0; rep < 3; ++rep) {
          CK(cudaDeviceSynchronize());
          cudaEventRecord(e0, st[0]);
          cudaEvent_t f; cudaEventCreate(&f); cudaEventRecord(f, st[0]);
          for (int i = 1; i < 3; ++i) cudaStreamWaitEvent(st[i], f, 0);
          for (int i = 0; i < 3; ++i) CK(cudaGraphLaunch(ge, st[i]));
          for (int i = 1; i < 3; ++i) { cudaEvent_t j; cudaEventCreate(&j); cudaEventRecord(j, st[i]); cudaStreamWaitEvent(st[0], j, 0); }
          cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          if (rep == 2) printf("n=%5ld  3x Dsyevd graph 3 streams (same buffers, timing only): %8.2f ms\n", n, ms);
        }
      }
      cudaFree(wd);
    }
    // sytrd alone
    {
      int lw = 0;
      double *dd, *ee, *tau;
      CK(cudaMalloc(&dd, n * 8)); CK(cudaMalloc(&ee, n * 8)); CK(cudaMalloc(&tau, n * 8));
      CK(cusolverDnDsytrd_bufferSize(hs[0], CUBLAS_FILL_MODE_LOWER, n, A, n, dd, ee, tau, &lw));
      double* wt; CK(cudaMalloc(&wt, size_t(lw) * 8 + 8));
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemcpy(A, A0, 3 * n * n * 8, cudaMemcpyDeviceToDevice));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0, st[0]);
        CK(cusolverDnDsytrd(hs[0], CUBLAS_FILL_MODE_LOWER, n, A, n, dd, ee, tau, wt, lw, info));
        cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("n=%5ld  1x Dsytrd          : %8.2f ms\n", n, ms);
      }
      cudaFree(wt); cudaFree(dd); cudaFree(ee); cudaFree(tau);
    }
    for (int i = 0; i < 3; ++i) cudaFree(dw[i]);
    cudaFree(A); cudaFree(A0); cudaFree(W); cudaFree(info);
  }
  return 0;
}
