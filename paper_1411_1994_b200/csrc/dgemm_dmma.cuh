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

// Tile configuration: block tile BM x BN x BK, STAGES-deep cp.async ring, warp tile
// WM x WN (m8n8k4 fragments), PAD keeps shared-memory row strides = 4 (mod 16)
// doubles so every 64-bit fragment load is bank-conflict free.
template <int BM_, int BN_, int BK_, int STAGES_, int WM_, int WN_, int MINB_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_, WM = WM_, WN = WN_;
  static constexpr int MINB = MINB_;  // CTAs per SM the register budget targets
  static constexpr int THREADS = (BM / WM) * (BN / WN) * 32;
  static constexpr int PAD = 4;
  static constexpr int SA = (BK * (BM + PAD) > BM * (BK + PAD)) ? BK * (BM + PAD) : BM * (BK + PAD);
  static constexpr int SB = (BK * (BN + PAD) > BN * (BK + PAD)) ? BK * (BN + PAD) : BN * (BK + PAD);
  static constexpr size_t SMEM_BYTES = size_t(STAGES) * (SA + SB) * sizeof(double);
};

using CfgBig = GemmCfg<128, 128, 16, 4, 64, 32, 1>;    // 8 warps, 1 CTA/SM
using CfgWide = GemmCfg<128, 128, 16, 4, 32, 32, 1>;   // 16 warps, 1 CTA/SM
using CfgHalf = GemmCfg<128, 64, 16, 4, 64, 32, 2>;    // 4 warps, 2 CTAs/SM
using CfgDeep = GemmCfg<128, 128, 32, 3, 64, 32, 1>;   // 8 warps, BK=32

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

// Per-thread tile loader.  Each thread owns one fixed coordinate of the contiguous
// dimension and a strided set of the other, so a stage needs one pointer, one
// stride and two remaining-extent counters per operand (no 64-bit index math in
// the main loop).  Out-of-range elements are zero-filled by cp.async src-size 0.
template <int ROWS, int BKk, int THREADS, int PAD, bool KMAJOR>
struct OperandLoader {
  // KMAJOR == false: contiguous along the ROWS dimension (m or n); smem [k][row]
  // KMAJOR == true : contiguous along k;                       smem [row][k]
  static constexpr int ITERS = (ROWS * BKk) / THREADS;
  static constexpr int FIX = KMAJOR ? BKk : ROWS;    // extent of the contiguous dim
  static constexpr int STEP = THREADS / FIX;         // stride of the other dim per iter
  const double* ptr;   // element (row0 + r_fix/var, kbeg + k_fix/var) of this thread
  int64_t step_ld;     // STEP * ld
  int64_t stage_adv;   // pointer advance per BK
  int fix, var;        // this thread's coordinates in the tile
  int64_t row_rem;     // rows remaining from (row0 + thread row)
  int64_t k_rem;       // k remaining from (kbeg + thread k)

  __device__ __forceinline__ void init(const double* base, int64_t ld, int64_t row0,
                                       int64_t rows, int64_t kbeg, int64_t kend) {
    fix = threadIdx.x % FIX;
    var = threadIdx.x / FIX;
    const int r = KMAJOR ? var : fix, k = KMAJOR ? fix : var;
    ptr = KMAJOR ? base + (kbeg + k) + (row0 + r) * ld : base + (row0 + r) + (kbeg + k) * ld;
    step_ld = int64_t(STEP) * ld;
    stage_adv = KMAJOR ? BKk : int64_t(BKk) * ld;
    row_rem = rows - row0 - r;
    k_rem = kend - kbeg - k;
  }
  // stage s of this tile into smem buffer `dst`
  __device__ __forceinline__ void load(double* dst, int s) const {
    const double* src = ptr + int64_t(s) * stage_adv;
    const int64_t krem = k_rem - int64_t(s) * BKk;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int v = var + it * STEP;
      bool pred;
      double* d;
      if (KMAJOR) {
        pred = krem > 0 && row_rem - it * STEP > 0;
        d = dst + v * (BKk + PAD) + fix;
      } else {
        pred = row_rem > 0 && krem - it * STEP > 0;
        d = dst + v * (ROWS + PAD) + fix;
      }
      cp_async8(d, pred ? src + it * step_ld : src - int64_t(s) * stage_adv, pred);
    }
  }
};

template <class Cfg, bool TA, bool TB>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) dgemm_dmma_kernel(GemmParams p) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, PAD = Cfg::PAD, STAGES = Cfg::STAGES;
  constexpr int WM = Cfg::WM, WN = Cfg::WN, SA = Cfg::SA, SB = Cfg::SB;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * SA;

  const int64_t tiles_m = (p.M + BM - 1) / BM;
  const int64_t tm = blockIdx.x % tiles_m;
  const int64_t tn = blockIdx.y;
  if (p.lower_only && tn * BN > tm * BM + BM - 1) return;  // tile entirely above the diagonal
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
  // opA: rows = m; NoTrans contiguous in m, Trans contiguous in k.
  // opB: rows = n; NoTrans contiguous in k, Trans contiguous in n.
  OperandLoader<BM, BK, Cfg::THREADS, PAD, TA> la;
  OperandLoader<BN, BK, Cfg::THREADS, PAD, !TB> lb;
  la.init(A, p.lda, m0, p.M, kbeg, kend);
  lb.init(B, p.ldb, n0, p.N, kbeg, kend);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) {
      la.load(As + s * SA, s);
      lb.load(Bs + s * SB, s);
    }
    cp_async_commit();
  }

  // Fragments are double-buffered in registers: the 64-bit shared loads of k-step
  // s+1 are issued before the DMMAs of step s, and the stage barrier sits before the
  // last k-step of a stage so the next stage's first fragments overlap its DMMAs.
  constexpr int KSTEPS = BK / 4;
  double af[2][WM / 8], bf[2][WN / 8];
  auto load_frags = [&](int buf, const double* as, const double* bs, int kk) {
#pragma unroll
    for (int i = 0; i < WM / 8; ++i) {
      const int m = wm + i * 8 + g, k = kk + t;
      af[buf][i] = TA ? as[m * (BK + PAD) + k] : as[k * (BM + PAD) + m];
    }
#pragma unroll
    for (int j = 0; j < WN / 8; ++j) {
      const int n = wn + j * 8 + g, k = kk + t;
      bf[buf][j] = TB ? bs[k * (BN + PAD) + n] : bs[n * (BK + PAD) + k];
    }
  };
  if (ktiles > 0) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    load_frags(0, As, Bs, 0);
  }
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    const double* as = As + int(kt % STAGES) * SA;
    const double* bs = Bs + int(kt % STAGES) * SB;
#pragma unroll
    for (int s = 0; s < KSTEPS; ++s) {
      const int cur = s & 1;
      if (s + 1 < KSTEPS) {
        load_frags(cur ^ 1, as, bs, (s + 1) * 4);
      } else {
        // stage kt+1 must have landed; every warp is past stage kt-1, whose slot the
        // load for stage kt+STAGES-1 reuses
        cp_async_wait<STAGES - 3>();
        __syncthreads();
        const int64_t nk = kt + STAGES - 1;
        if (nk < ktiles) {
          const int st = int(nk % STAGES);
          la.load(As + st * SA, int(nk));
          lb.load(Bs + st * SB, int(nk));
        }
        cp_async_commit();
        if (kt + 1 < ktiles)
          load_frags(cur ^ 1, As + int((kt + 1) % STAGES) * SA, Bs + int((kt + 1) % STAGES) * SB, 0);
      }
#pragma unroll
      for (int i = 0; i < WM / 8; ++i)
#pragma unroll
        for (int j = 0; j < WN / 8; ++j)
          dmma884(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
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
