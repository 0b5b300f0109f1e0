// Symmetric eigensolver for the RHOSVD Grams (n ~ 300 .. 4000), replacing cuSOLVER syevd
// whose one-column-at-a-time tridiagonalisation is launch-latency bound (6.2 of 6.7 ms at
// n = 693) and whose concurrent calls serialise.
//
//   1. sytrd  : Householder tridiagonalisation (LAPACK dsytd2, lower) in ONE thread-block
//               cluster of 16 CTAs: warps own trailing columns, the two dependencies per
//               column (p.v and the next reflector) are cluster barriers (~0.2 us) instead
//               of kernel launches; the trailing matrix stays in L2.
//   2. stedc  : Cuppen divide and conquer on the tridiagonal (eig_dc.cuh).
//   3. ormtr  : eigenvectors Q_h Z with the reflectors applied in compact-WY blocks (GEMMs).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace latsum_b200 {
namespace eig {

namespace cg = cooperative_groups;

constexpr int TRD_CTAS = 16;  // cluster size (non-portable: 16)
constexpr int TRD_THREADS = 1024;
constexpr int TRD_WPC = TRD_THREADS / 32;  // warps per CTA
constexpr int TRD_WARPS = TRD_CTAS * TRD_WPC;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Workspace (global, L2-resident): two v buffers, the p buffer, per-CTA partial dots.
struct TrdWork {
  double* v0;
  double* v1;    // n each
  double* p;     // n
  double* part;  // 2 * TRD_CTAS
};

// Householder reflector of x = A[kk+1 .. n-1, kk] by one warp (LAPACK dlarfg): H = I - tau
// v v^T, v[kk+1] = 1, H x = (beta, 0, ..).  v -> vout[kk+1..n) and A[kk+2.., kk] (LAPACK
// layout), beta -> e[kk] and A[kk+1, kk], tau -> tau[kk].
__device__ __forceinline__ void householder_warp(double* A, int64_t lda, int n, int kk,
                                                 double* vout, double* e, double* tau, int lane) {
  double* x = A + int64_t(kk) * lda;
  const double alpha = x[kk + 1];
  double ss = 0.0;
  for (int r = kk + 2 + lane; r < n; r += 32) ss += x[r] * x[r];
  ss = warp_sum(ss);
  double beta, tk, scal;
  if (ss == 0.0) {  // H = I (also for a single element)
    beta = alpha;
    tk = 0.0;
    scal = 0.0;
  } else {
    const double nrm = sqrt(alpha * alpha + ss);
    beta = alpha >= 0.0 ? -nrm : nrm;
    tk = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
  for (int r = kk + 1 + lane; r < n; r += 32) {
    const double v = r == kk + 1 ? 1.0 : x[r] * scal;
    vout[r] = v;
    if (r > kk + 1) x[r] = v;
  }
  if (lane == 0) {
    e[kk] = beta;
    tau[kk] = tk;
    x[kk + 1] = beta;
  }
}

// One cluster tridiagonalises A (n x n, full symmetric storage): d[0..n), e[0..n-1),
// tau[0..n-1); reflector k has v[k+1] = 1 and v[k+2..n) in A[k+2.., k].  Column c >= 1 is
// owned by global warp (c - 1) % TRD_WARPS.  Step k, with reflector k and
// p_k = tau_k A22 v_k (plus per-CTA partials of p_k . v_k) published:
//   alpha = -tau_k/2 (p_k . v_k), w = p_k + alpha v_k, A22 -= v w^T + w v^T (owned columns;
//   the owner of column k+1 updates it first and builds reflector k+1)      | cluster barrier
//   p_{k+1}[c] = tau_{k+1} A22'[:, c] . v_{k+1} for owned c >= k+2            | cluster barrier
__global__ void __launch_bounds__(TRD_THREADS, 1)
k_sytrd_cluster(double* __restrict__ A, int64_t lda, int n, double* __restrict__ d,
                double* __restrict__ e, double* __restrict__ tau, TrdWork w) {
  cg::cluster_group cluster = cg::this_cluster();
  const int cta = int(cluster.block_rank());
  const int lane = threadIdx.x % 32, wib = threadIdx.x / 32;
  const int gw = cta * TRD_WPC + wib;
  __shared__ double red[TRD_WPC];
  __shared__ double alpha_s;

  if (n == 1) {
    if (threadIdx.x == 0 && cta == 0) d[0] = A[0];
    return;
  }
  if (gw == 0) {
    householder_warp(A, lda, n, 0, w.v0, e, tau, lane);
    if (lane == 0) d[0] = A[0];
  }
  cluster.sync();
  // p_0 over columns c >= 1
  {
    const double* v = w.v0;
    const double t0 = tau[0];
    double mypart = 0.0;
    for (int c = 1 + gw; c < n; c += TRD_WARPS) {
      const double* col = A + int64_t(c) * lda;
      double s = 0.0;
      if (t0 != 0.0)
        for (int r = 1 + lane; r < n; r += 32) s += col[r] * v[r];
      s = warp_sum(s) * t0;
      if (lane == 0) w.p[c] = s;
      mypart += s * v[c];
    }
    if (lane == 0) red[wib] = mypart;
    __syncthreads();
    if (threadIdx.x < 32) {
      double s = threadIdx.x < TRD_WPC ? red[threadIdx.x] : 0.0;
      s = warp_sum(s);
      if (threadIdx.x == 0) w.part[cta] = s;
    }
  }
  cluster.sync();

  extern __shared__ double sbuf[];  // sv[n], sw[n]: v_k and w_k (step broadcast, per CTA)
  double* sv = sbuf;
  double* sw = sbuf + n;
  for (int k = 0; k + 1 < n; ++k) {
    const bool odd = k & 1;
    const double* v = odd ? w.v1 : w.v0;
    double* vn = odd ? w.v0 : w.v1;
    const double* part_cur = w.part + (odd ? TRD_CTAS : 0);
    double* part_next = w.part + (odd ? 0 : TRD_CTAS);
    const double tk = tau[k];
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q = 0; q < TRD_CTAS; ++q) s += part_cur[q];
      alpha_s = -0.5 * tk * s;
    }
    __syncthreads();
    const double alpha = alpha_s;
    // stage v_k and w_k = p_k + alpha v_k in shared memory (one coalesced L2 pass per CTA)
    for (int r = k + 1 + threadIdx.x; r < n; r += TRD_THREADS) {
      const double vr = v[r];
      sv[r] = vr;
      sw[r] = w.p[r] + alpha * vr;
    }
    __syncthreads();
    // update owned columns c >= k+1 (ascending: the owner of k+1 starts with it)
    for (int c = 1 + gw; c < n; c += TRD_WARPS) {
      if (c < k + 1) continue;
      double* col = A + int64_t(c) * lda;
      if (tk != 0.0) {
        const double vc = sv[c], wc = sw[c];
#pragma unroll 8
        for (int r = k + 1 + lane; r < n; r += 32) col[r] -= sv[r] * wc + sw[r] * vc;
      }
      if (c == k + 1) {
        __syncwarp();
        if (lane == 0) d[c] = col[c];
        if (c + 1 < n) householder_warp(A, lda, n, c, vn, e, tau, lane);
      }
    }
    cluster.sync();  // reflector k+1 published, all columns updated
    if (k + 2 >= n) break;
    {
      const double t1 = tau[k + 1];
      for (int r = k + 2 + threadIdx.x; r < n; r += TRD_THREADS) sv[r] = vn[r];
      __syncthreads();
      double mypart = 0.0;
      for (int c = 1 + gw; c < n; c += TRD_WARPS) {
        if (c < k + 2) continue;
        const double* col = A + int64_t(c) * lda;
        double s = 0.0;
        if (t1 != 0.0) {
#pragma unroll 8
          for (int r = k + 2 + lane; r < n; r += 32) s += col[r] * sv[r];
        }
        s = warp_sum(s) * t1;
        if (lane == 0) w.p[c] = s;
        mypart += s * sv[c];
      }
      if (lane == 0) red[wib] = mypart;
      __syncthreads();
      if (threadIdx.x < 32) {
        double s = threadIdx.x < TRD_WPC ? red[threadIdx.x] : 0.0;
        s = warp_sum(s);
        if (threadIdx.x == 0) part_next[cta] = s;
      }
    }
    cluster.sync();
  }
}

}  // namespace eig
}  // namespace latsum_b200
