// FP64 tensor-core GEMM for sm_100a: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).
//
// tcgen05 has no f64 kind (ptxas rejects .kind::f64), so FP64 tensor
// math on B200 is the DMMA path: operands staged global -> shared memory by
// cp.async (multi-stage ring), shared -> registers with conflict-free 64-bit
// loads, accumulators in registers.  Measured peak of this instruction on the
// pool's B200s: 37.0 TFLOP/s (tools/fp64_peak.cu; profiles/fp64_peak_r01.txt).
//
// One kernel serves every dense contraction of the path:
//   C = alpha * opA(A) * opB(B) + beta * C, column-major, with
//   opA(m,k) = TA ? A[k + m*lda] : A[m + k*lda]
//   opB(k,n) = TB ? B[n + k*ldb] : B[k + n*ldb]
// plus strided batches, deterministic split-K (partials + ordered reduction),
// per-batch K segments (grouped contractions), and a lower-triangle-only mode
// for Gram matrices (syevd reads the lower triangle only).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace latsum_b200 {

struct GemmParams {
  int64_t M, N, K;
  const double* A;
  int64_t lda, sA;  // batch strides in elements
  const double* B;
  int64_t ldb, sB;
  double* C;
  int64_t ldc, sC;
  double alpha, beta;
  int64_t batch;
  int splits;             // >1: write partials to C + split*M*N (ldc=M), reduce later
  const int64_t* kseg;    // optional [batch+1] K ranges (A/B not batch-strided then)
  int lower_only;         // skip tiles strictly above the diagonal (M == N Gram)
};

namespace gemm_cfg {
constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int WM = 64, WN = 32;  // warp tile: 2 x 4 warps
constexpr int PAD = 4;           // row stride = 4 (mod 16) doubles: conflict-free fragments
constexpr int SM_MMAJ = BK * (BM + PAD);   // [k][m] layout
constexpr int SM_KMAJ = BM * (BK + PAD);   // [m][k] layout
constexpr int SA = SM_MMAJ > SM_KMAJ ? SM_MMAJ : SM_KMAJ;
constexpr int SB = SA;
constexpr size_t SMEM_BYTES = size_t(STAGES) * (SA + SB) * sizeof(double);
}  // namespace gemm_cfg

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Loads the BM x BK tile of opA starting at (m0, k0) and the BK x BN tile of
// opB at (k0, n0) into one pipeline stage.  Out-of-range elements are zero.
template <bool TA, bool TB>
__device__ __forceinline__ void load_stage(double* As, double* Bs, const double* A, int64_t lda,
                                           const double* B, int64_t ldb, int64_t m0, int64_t n0,
                                           int64_t k0, int64_t kend, int64_t M, int64_t N) {
  using namespace gemm_cfg;
  const int tid = threadIdx.x;
#pragma unroll
  for (int it = 0; it < (BM * BK) / THREADS; ++it) {
    const int idx = tid + it * THREADS;
    if (!TA) {  // contiguous in m: [k][m]
      const int k = idx / BM, m = idx % BM;
      const int64_t gm = m0 + m, gk = k0 + k;
      const bool p = gm < M && gk < kend;
      cp_async8(As + k * (BM + PAD) + m, p ? A + gm + gk * lda : A, p);
    } else {  // contiguous in k: [m][k]
      const int m = idx / BK, k = idx % BK;
      const int64_t gm = m0 + m, gk = k0 + k;
      const bool p = gm < M && gk < kend;
      cp_async8(As + m * (BK + PAD) + k, p ? A + gk + gm * lda : A, p);
    }
  }
#pragma unroll
  for (int it = 0; it < (BN * BK) / THREADS; ++it) {
    const int idx = tid + it * THREADS;
    if (TB) {  // contiguous in n: [k][n]
      const int k = idx / BN, n = idx % BN;
      const int64_t gn = n0 + n, gk = k0 + k;
      const bool p = gn < N && gk < kend;
      cp_async8(Bs + k * (BN + PAD) + n, p ? B + gn + gk * ldb : B, p);
    } else {  // contiguous in k: [n][k]
      const int n = idx / BK, k = idx % BK;
      const int64_t gn = n0 + n, gk = k0 + k;
      const bool p = gn < N && gk < kend;
      cp_async8(Bs + n * (BK + PAD) + k, p ? B + gk + gn * ldb : B, p);
    }
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(gemm_cfg::THREADS, 1) dgemm_dmma_kernel(GemmParams p) {
  using namespace gemm_cfg;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * SA;

  const int64_t tiles_m = (p.M + BM - 1) / BM;
  const int64_t tm = blockIdx.x % tiles_m;
  const int64_t tn = blockIdx.y;
  if (p.lower_only && tn > tm) return;  // tile entirely above the diagonal (BM == BN)
  const int64_t m0 = tm * BM, n0 = tn * BN;

  int64_t b = blockIdx.z, split = 0;
  if (p.splits > 1) {
    split = b % p.splits;
    b /= p.splits;
  }
  const double* A = p.A;
  const double* B = p.B;
  double* C = p.C + b * p.sC;
  int64_t kbeg = 0, kend = p.K;
  if (p.kseg) {
    kbeg = p.kseg[b];
    kend = p.kseg[b + 1];
  } else {
    A += b * p.sA;
    B += b * p.sB;
  }
  if (p.splits > 1) {
    const int64_t span = kend - kbeg;
    const int64_t chunk = ((span + p.splits - 1) / p.splits + BK - 1) / BK * BK;
    const int64_t lo = kbeg + split * chunk;
    kend = lo + chunk < kend ? lo + chunk : kend;
    kbeg = lo;
  }

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % (BM / WM)) * WM;  // 0 or 64
  const int wn = (warp / (BM / WM)) * WN;  // 0, 32, 64, 96

  double acc[WM / 8][WN / 8][2];
#pragma unroll
  for (int i = 0; i < WM / 8; ++i)
#pragma unroll
    for (int j = 0; j < WN / 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t ktiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles)
      load_stage<TA, TB>(As + s * SA, Bs + s * SB, A, p.lda, B, p.ldb, m0, n0, kbeg + s * BK, kend,
                         p.M, p.N);
    cp_async_commit();
  }

  for (int64_t kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + STAGES - 1;
      if (nk < ktiles) {
        const int st = int(nk % STAGES);
        load_stage<TA, TB>(As + st * SA, Bs + st * SB, A, p.lda, B, p.ldb, m0, n0,
                           kbeg + nk * BK, kend, p.M, p.N);
      }
      cp_async_commit();
    }
    const double* as = As + int(kt % STAGES) * SA;
    const double* bs = Bs + int(kt % STAGES) * SB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[WM / 8], bf[WN / 8];
#pragma unroll
      for (int i = 0; i < WM / 8; ++i) {
        const int m = wm + i * 8 + g, k = kk + t;
        af[i] = TA ? as[m * (BK + PAD) + k] : as[k * (BM + PAD) + m];
      }
#pragma unroll
      for (int j = 0; j < WN / 8; ++j) {
        const int n = wn + j * 8 + g, k = kk + t;
        bf[j] = TB ? bs[k * (BN + PAD) + n] : bs[n * (BK + PAD) + k];
      }
#pragma unroll
      for (int i = 0; i < WM / 8; ++i)
#pragma unroll
        for (int j = 0; j < WN / 8; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: thread holds C[m0+wm+8i+g][n0+wn+8j+2t+{0,1}]
  const bool partial = p.splits > 1;
  double* Cp = partial ? p.C + (b * p.splits + split) * (p.M * p.N) : C;
  const int64_t ldc = partial ? p.M : p.ldc;
#pragma unroll
  for (int i = 0; i < WM / 8; ++i) {
    const int64_t gm = m0 + wm + i * 8 + g;
    if (gm >= p.M) continue;
#pragma unroll
    for (int j = 0; j < WN / 8; ++j) {
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int64_t gn = n0 + wn + j * 8 + 2 * t + x;
        if (gn >= p.N) continue;
        double* dst = Cp + gm + gn * ldc;
        if (partial) {
          *dst = acc[i][j][x];
        } else {
          const double v = p.alpha * acc[i][j][x];
          *dst = p.beta == 0.0 ? v : v + p.beta * *dst;
        }
      }
    }
  }
}

// C = alpha * sum_s partial_s + beta * C, in split order (deterministic).
__global__ void dgemm_reduce_splits(const double* __restrict__ ws, int splits, int64_t M, int64_t N,
                                    double* C, int64_t ldc, int64_t sC, double alpha, double beta,
                                    int lower_only) {
  const int64_t b = blockIdx.y;
  const int64_t total = M * N;
  const double* w = ws + b * splits * total;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = e % M, n = e / M;
    if (lower_only && n > m) continue;
    double s = 0.0;
    for (int q = 0; q < splits; ++q) s += w[q * total + e];
    double* dst = C + b * sC + m + n * ldc;
    const double v = alpha * s;
    *dst = beta == 0.0 ? v : v + beta * *dst;
  }
}

}  // namespace latsum_b200
