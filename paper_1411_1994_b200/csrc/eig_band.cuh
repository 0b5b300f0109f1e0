// Two-stage symmetric eigensolver for the RHOSVD Grams (n <= SB_NMAX), the default
// replacement of cuSOLVER syevd whose one-stage tridiagonalisation spends ~9 us per column
// on launch latency (6.3 of 6.7 ms at n = 693) and whose concurrent calls serialise.
//
//   1. k_sy2sb   full -> lower band of width BW in ONE 16-CTA thread-block cluster: per
//                panel of BW columns, CTA 0 factors the panel (a warp per column, the
//                column in registers, one __syncthreads per reflector) into V, T (compact
//                WY); the cluster applies Q^T A22 Q = A22 - W V^T - V W^T with
//                W = A22 V T - 1/2 V (T^T V^T A22 V T), each CTA owning a column slab; the
//                matrix stays in L2 and the per-panel dependencies are cluster barriers.
//   2. k_sb2st   band -> tridiagonal by bulge chasing (the successive-band-reduction
//                kernels of LAPACK dsb2st: Householder of length BW, one task = right
//                application to the block below + a new reflector + its two-sided
//                application to the next diagonal block).  The band (with room for the
//                bulges) lives in ONE CTA's shared memory; each warp runs a sweep, and
//                sweep s+1 starts task k once sweep s has finished task k+1 (the two then
//                touch disjoint elements), so ~n/(2 BW) sweeps are in flight.
//   3. eigenvalues by Sturm multisection (eig_sym.cuh), eigenvectors of the tridiagonal
//      by inverse iteration (k_tridiag_invit_sm, factors and iterate in shared memory).
//   4. k_band_backtransform  Z = Q1 Q2 Y for a few columns per CTA: the bulge reflectors
//      of one sweep act on disjoint rows, so a sweep is one parallel step (half-warp dot
//      products); the panels then apply I - V T V^T in reverse order.
#pragma once
#include <cooperative_groups.h>
#include "ozaki_i8.cuh"  // mbarrier / bulk-copy wrappers
#include <cuda_runtime.h>
#include <cstdint>

namespace latsum_b200 {
namespace band {

namespace cg = cooperative_groups;
constexpr unsigned FULL = 0xffffffffu;

constexpr int BW = 16;                 // band width (a half-warp)
constexpr int S2B_CTAS = 16;           // cluster size (non-portable: 16)
constexpr int S2B_THREADS = 512;       // 16 warps = the BW columns of a panel
constexpr int S2B_RPL = 26;            // panel rows per lane: n <= 832
constexpr int S2B_NMAX = 32 * S2B_RPL;
constexpr int S2B_MAXC = (S2B_NMAX + S2B_CTAS - 1) / S2B_CTAS;  // owned columns per CTA
constexpr int SB_LDB = 2 * BW + 2;     // band column stride in shared memory (bulge room)
#ifndef LATSUM_SB_WARPS
#define LATSUM_SB_WARPS 16
#endif
constexpr int SB_WARPS = LATSUM_SB_WARPS;  // sweeps in flight (one warp each): 16 beat 12 / 24 (2.22 vs 2.38 / 2.43 ms, n = 693)
constexpr int SB_KBIG = 64;            // progress encoding: sweep * SB_KBIG + tasks done
constexpr int SB_NMAX = 808;           // 34 (n + 16) + 768 doubles <= 227 KB
constexpr int BT_CPB = 4;              // eigenvector columns per back-transform CTA
constexpr int BT_THREADS = 512;

__host__ __device__ inline int s2b_panels(int n) { return n >= 2 ? (n - 2) / BW : 0; }
__host__ __device__ inline int sb_tasks_max(int n) { return n >= 2 ? (n - 2) / BW + 1 : 1; }
constexpr int S2B_LDV = S2B_NMAX;      // row stride of the panel's V in shared memory
inline size_t s2b_smem_doubles(int) {
  return size_t(BW) * S2B_LDV + S2B_MAXC * 2 * BW + S2B_MAXC * BW + 7 * BW * BW + BW;
}
inline size_t sb_smem_doubles(int n) { return size_t(SB_LDB) * (n + BW) + SB_WARPS * 32; }

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Reduce acc[16] over the 32 lanes; lane l returns the total of acc[l >> 1].
__device__ __forceinline__ double reduce16_scatter(const double (&acc)[16], int lane) {
  double a8[8], a4[4], a2[2];
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double send = b4 ? acc[j] : acc[j + 8];
    a8[j] = (b4 ? acc[j + 8] : acc[j]) + __shfl_xor_sync(FULL, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double send = b3 ? a8[j] : a8[j + 4];
    a4[j] = (b3 ? a8[j + 4] : a8[j]) + __shfl_xor_sync(FULL, send, 8);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double send = b2 ? a4[j] : a4[j + 2];
    a2[j] = (b2 ? a4[j + 2] : a4[j]) + __shfl_xor_sync(FULL, send, 4);
  }
  const double send = b1 ? a2[0] : a2[1];
  double r = (b1 ? a2[1] : a2[0]) + __shfl_xor_sync(FULL, send, 2);
  return r + __shfl_xor_sync(FULL, r, 1);
}

// Reduce p[8] over the 16 lanes of a half-warp; lane l returns the total of p[(l >> 1) & 7].
__device__ __forceinline__ double reduce8_half(const double (&p)[8], int lane) {
  double a4[4], a2[2];
  const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double send = b3 ? p[j] : p[j + 4];
    a4[j] = (b3 ? p[j + 4] : p[j]) + __shfl_xor_sync(FULL, send, 8);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double send = b2 ? a4[j] : a4[j + 2];
    a2[j] = (b2 ? a4[j + 2] : a4[j]) + __shfl_xor_sync(FULL, send, 4);
  }
  const double send = b1 ? a2[0] : a2[1];
  double r = (b1 ? a2[1] : a2[0]) + __shfl_xor_sync(FULL, send, 2);
  return r + __shfl_xor_sync(FULL, r, 1);
}

// ---------------------------------------------------------------- stage 1: full -> band
// A (n x n, full symmetric storage, lda) is reduced in place to lower band width BW:
// A = Q1 B Q1^T, Q1 = P_0 P_1 .. P_{npan-1}, P_p = I - V_p T_p V_p^T.  Panel p covers columns
// [pBW, pBW+BW) and rows [r0, n), r0 = (p+1)BW; reflector c of the panel has its unit entry
// at row r0 + c.  Outputs: Vw (npan x BW x n, column c of panel p at Vw + (p BW + c) n,
// zero above the unit entry: the caller zero-fills), Tw (npan x BW x BW, column-major
// upper triangular).  Wg: BW x n scratch.
struct S2BArgs {
  double* A;
  int64_t lda;
  int n;
  double* Vw;
  double* Tw;
  double* Wg;
  long long* prof;  // optional: per-phase cycles of CTA 0 (8 slots)
};

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Per panel (4 cluster barriers):
//   CTA 0: panel QR (V -> Vp, S = V^T V and tau in shared memory)            | barrier 1
//   all:   Y_own = A22[:, own]^T V (DMMA, K split over warps); P_own = V_own^T Y_own;
//          CTA 0's warp 15 builds T meanwhile (needed only after barrier 2)    | barrier 2
//   all:   Z = (sum_q P_q) T, M2 = T^T Z, X_own = Y_own T, W_own = X_own - 1/2 V_own M2  | barrier 3
//   all:   A22[:, own] -= [W V] [V_own W_own]^T (DMMA, K = 2 BW)              | barrier 4
__global__ void __launch_bounds__(S2B_THREADS, 1) k_sy2sb(S2BArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  const int n = a.n;
  const int64_t lda = a.lda;
  double* __restrict__ A = a.A;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;  // mma fragment coordinates
  extern __shared__ double sm[];
  double* Vs = sm;                          // BW x S2B_LDV: the panel's V, local rows, zero past m
  double* VWj = Vs + BW * S2B_LDV;          // S2B_MAXC x 2BW: (V, W) rows of the owned columns
  double* Ys = VWj + S2B_MAXC * 2 * BW;     // S2B_MAXC x BW: Y rows of the owned columns
  double* Zp = Ys + S2B_MAXC * BW;          // BW x BW: this CTA's share of V^T Y
  double* Zf = Zp + BW * BW;                // V^T A22 V T  (then reused)
  double* M2 = Zf + BW * BW;                // T^T Z
  double* Ts = M2 + BW * BW;                // T (row-major)
  double* Ss = Ts + BW * BW;                // V^T V (upper)
  double* taus = Ss + BW * BW;              // BW
  double* Pf = taus + BW;                   // BW x BW: sum of the P shares
  const int npan = s2b_panels(n);
  long long ph[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tclk = clock64();
  auto mark = [&](int slot) {
    if (a.prof) {
      const long long t = clock64();
      ph[slot] += t - tclk;
      tclk = t;
    }
  };
  for (int p = 0; p < npan; ++p) {
    const int j0 = p * BW, r0 = j0 + BW, m = n - r0;
    const int tmax = (m + 31) / 32;
    double* Vp = a.Vw + size_t(p) * BW * n;
    double* Tp = a.Tw + size_t(p) * BW * BW;
    for (int idx = tid; idx < S2B_MAXC * BW; idx += S2B_THREADS) Ys[idx] = 0.0;
    if (q == 0) {  // ---- panel QR: warp c owns column j0 + c, lane holds rows lane + 32t
      double x[S2B_RPL];
      const double* colp = A + int64_t(j0 + wid) * lda + r0;
#pragma unroll
      for (int t = 0; t < S2B_RPL; ++t) {
        const int r = lane + 32 * t;
        x[t] = r < m ? __ldcg(colp + r) : 0.0;
      }
      mark(8);
      // the serial chain per reflector is the owner's norm + scaling and one barrier; rows
      // past m hold zeros in x and Vs, so the loops need no row predicates.  Only the
      // columns right of the reflector read v (shared-memory bandwidth is the limit here);
      // V^T V for T is formed after the loop.
      for (int cc = 0; cc < BW; ++cc) {
        if (wid == cc) {
          const double alpha = __shfl_sync(FULL, x[0], cc);
          double s0 = (lane > cc) ? x[0] * x[0] : 0.0, s1 = 0.0;
#pragma unroll
          for (int t = 1; t < S2B_RPL; t += 2) {
            if (t < tmax) s1 += x[t] * x[t];
            if (t + 1 < S2B_RPL && t + 1 < tmax) s0 += x[t + 1] * x[t + 1];
          }
          const double ss = wsum(s0 + s1);
          double tau = 0.0, beta = alpha, scal = 0.0;
          if (m - cc > 1 && ss > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + ss), alpha);
            scal = 1.0 / (alpha - beta);
            tau = (beta - alpha) * (1.0 / beta);
          }
          double* vc = Vs + cc * S2B_LDV + lane;
          if (lane < cc) vc[0] = 0.0;
          if (lane == cc) {
            vc[0] = 1.0;
            x[0] = beta;
          }
          if (lane > cc) {
            x[0] *= scal;
            vc[0] = x[0];
          }
#pragma unroll
          for (int t = 1; t < S2B_RPL; ++t) {
            if (t < tmax) x[t] *= scal;
            vc[32 * t] = x[t];  // zeros past m
          }
          if (lane == 0) taus[cc] = tau;
        }
        __syncthreads();
        if (wid > cc) {  // apply P_cc to column wid: v read from shared memory once, kept in
                         // registers for the dot and the update (the loop was bound by the
                         // shared-memory wavefronts of reading v twice in 15 warps)
          const double* __restrict__ vc = Vs + cc * S2B_LDV + lane;  // zero above row cc, past m
          double vv[S2B_RPL];
#pragma unroll
          for (int t = 0; t < S2B_RPL; ++t) vv[t] = t < tmax ? vc[32 * t] : 0.0;
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int t = 0; t < S2B_RPL; t += 2) {
            s0 += vv[t] * x[t];
            if (t + 1 < S2B_RPL) s1 += vv[t + 1] * x[t + 1];
          }
          const double f = taus[cc] * wsum(s0 + s1);
#pragma unroll
          for (int t = 0; t < S2B_RPL; ++t) x[t] -= f * vv[t];
        }
      }
      mark(9);
      {  // column wid (R, beta, v) back to A; v to the panel's Vp
        double* colw = A + int64_t(j0 + wid) * lda + r0;
        double* vg = Vp + size_t(wid) * n + r0;
#pragma unroll
        for (int t = 0; t < S2B_RPL; ++t) {
          const int r = lane + 32 * t;
          if (t < tmax && r < m) {
            colw[r] = x[t];
            if (r >= wid) vg[r] = Vs[wid * S2B_LDV + r];
          }
        }
      }
      __syncthreads();
      // S = V^T V (upper): warp w forms the dots of v_w with v_c, c > w
      for (int cpair = wid; cpair < BW * BW; cpair += S2B_THREADS / 32) {
        const int ra = cpair / BW, cb = cpair % BW;
        if (cb <= ra) continue;  // uniform per warp
        const double* va = Vs + ra * S2B_LDV;
        const double* vb = Vs + cb * S2B_LDV;
        double sdot = 0.0;
        for (int r = cb + lane; r < m; r += 32) sdot += va[r] * vb[r];
        sdot = wsum(sdot);
        if (lane == 0) Ss[ra * BW + cb] = sdot;
      }
      __syncthreads();
    }
    mark(0);
    cluster.sync();  // ---- 1: panel published (V in Vp / A)
    mark(1);
    if (q != 0) {
      for (int idx = tid; idx < BW * S2B_LDV; idx += S2B_THREADS) {
        const int c = idx / S2B_LDV, r = idx % S2B_LDV;
        Vs[idx] = r < m ? __ldcg(Vp + size_t(c) * n + r0 + r) : 0.0;
      }
      __syncthreads();
    }
    const int cpc = (m + S2B_CTAS - 1) / S2B_CTAS;
    const int lo = min(m, q * cpc), hi = min(m, lo + cpc), ncol = hi - lo;
    if (q == 0 && wid == 15) {  // T (LAPACK dlarft, forward / columnwise): lane i keeps row i
      double trow[BW];
#pragma unroll
      for (int c = 0; c < BW; ++c) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int e = 0; e < c; e += 2) {
          if (e >= lane) a0 += trow[e] * Ss[e * BW + c];
          if (e + 1 < c && e + 1 >= lane) a1 += trow[e + 1] * Ss[(e + 1) * BW + c];
        }
        trow[c] = lane < c ? -taus[c] * (a0 + a1) : (lane == c ? taus[c] : 0.0);
      }
      if (lane < BW)
#pragma unroll
        for (int c = 0; c < BW; ++c) {
          Ts[lane * BW + c] = trow[c];
          Tp[lane + c * BW] = trow[c];  // column-major
        }
    } else if (ncol > 0) {
      // ---- Y_own = A22[:, own]^T V: mma m8n8k4, M = owned columns (8 per tile), N = BW
      // (two tiles), K = the m rows split over the warps
      const int MT = (ncol + 7) / 8, KS = 15 / MT;
      if (wid < MT * KS) {
        const int mt = wid % MT, ks = wid / MT;
        const int nsteps = (m + 3) / 4;
        const int s0 = ks * nsteps / KS, s1 = (ks + 1) * nsteps / KS;
        const int ii = mt * 8 + g;
        const bool iok = ii < ncol;
        const double* acol = A + int64_t(r0 + lo + (iok ? ii : 0)) * lda + r0;
        double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
        for (int st = s0; st < s1; st += 4) {
          double af[4], b0[4], b1[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = (st + u) * 4 + t4;
            const bool ok = st + u < s1 && k < m;
            af[u] = (ok && iok) ? __ldcg(acol + k) : 0.0;
            b0[u] = ok ? Vs[g * S2B_LDV + k] : 0.0;
            b1[u] = ok ? Vs[(8 + g) * S2B_LDV + k] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            dmma884(c00, c01, af[u], b0[u]);
            dmma884(c10, c11, af[u], b1[u]);
          }
        }
        if (iok) {
          double* yr = Ys + ii * BW + 2 * t4;
          atomicAdd(yr, c00);
          atomicAdd(yr + 1, c01);
          atomicAdd(yr + 8, c10);
          atomicAdd(yr + 9, c11);
        }
      }
    }
    __syncthreads();
    mark(2);
    if (tid < BW * BW) {  // this CTA's share of P = V^T Y
      const int ra = tid / BW, cb = tid % BW;
      double z = 0.0;
      for (int i = 0; i < ncol; ++i) z += Vs[ra * S2B_LDV + lo + i] * Ys[i * BW + cb];
      Zp[tid] = z;
    }
    cluster.sync();  // ---- 2: P shares and T published
    mark(3);
    if (tid < BW * BW) {
      double z = 0.0;
      for (int r = 0; r < S2B_CTAS; ++r) z += cluster.map_shared_rank(Zp, r)[tid];
      Pf[tid] = z;
      if (q != 0) Ts[tid] = __ldcg(Tp + (tid % BW) * BW + tid / BW);
    }
    __syncthreads();
    if (tid < BW * BW) {  // Z = P T (T upper triangular)
      const int ra = tid / BW, cb = tid % BW;
      double s = 0.0;
      for (int e = 0; e <= cb; ++e) s += Pf[ra * BW + e] * Ts[e * BW + cb];
      Zf[tid] = s;
    }
    __syncthreads();
    if (tid < BW * BW) {  // M2 = T^T Z
      const int ra = tid / BW, cb = tid % BW;
      double s = 0.0;
      for (int e = 0; e <= ra; ++e) s += Ts[e * BW + ra] * Zf[e * BW + cb];
      M2[tid] = s;
    }
    __syncthreads();
    for (int idx = tid; idx < ncol * BW; idx += S2B_THREADS) {  // X = Y T, W = X - 1/2 V M2
      const int ii = idx / BW, cb = idx % BW, i = lo + ii;
      double x = 0.0, s = 0.0;
#pragma unroll
      for (int e = 0; e < BW; ++e) {
        x += Ys[ii * BW + e] * Ts[e * BW + cb];
        s += Vs[e * S2B_LDV + i] * M2[e * BW + cb];
      }
      const double w = x - 0.5 * s;
      a.Wg[size_t(cb) * n + i] = w;
      VWj[ii * 2 * BW + cb] = Vs[cb * S2B_LDV + i];
      VWj[ii * 2 * BW + BW + cb] = w;
    }
    mark(4);
    cluster.sync();  // ---- 3: W published
    mark(5);
    // ---- A22[:, own] -= [W V] [V_own W_own]^T: mma m8n8k4, M = rows (8 per tile, one
    // row tile per warp at a time, its A fragments reused across the owned column tiles),
    // N = owned columns, K = 2 BW
    if (ncol > 0) {
      const int NT = (ncol + 7) / 8, RT = (m + 7) / 8;
      for (int rt = wid; rt < RT; rt += S2B_THREADS / 32) {
        const int i = rt * 8 + g;
        const bool iok = i < m;
        double af[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          af[u] = iok ? __ldcg(a.Wg + size_t(4 * u + t4) * n + i) : 0.0;
          af[4 + u] = Vs[(4 * u + t4) * S2B_LDV + i];  // zero past m
        }
        double cold[2 * ((S2B_MAXC + 7) / 8)];
#pragma unroll
        for (int nt = 0; nt < (S2B_MAXC + 7) / 8; ++nt) {
          const int jc = nt * 8 + 2 * t4;
          const double* ap = A + int64_t(r0 + lo + jc) * lda + r0 + i;
          cold[2 * nt] = (nt < NT && iok && jc < ncol) ? __ldcg(ap) : 0.0;
          cold[2 * nt + 1] = (nt < NT && iok && jc + 1 < ncol) ? __ldcg(ap + lda) : 0.0;
        }
#pragma unroll
        for (int nt = 0; nt < (S2B_MAXC + 7) / 8; ++nt) {
          if (nt < NT) {
            const int jj = nt * 8 + g;
            const double* vw = VWj + (jj < ncol ? jj : 0) * 2 * BW + t4;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) dmma884(c0, c1, af[u], jj < ncol ? vw[4 * u] : 0.0);
            const int jc = nt * 8 + 2 * t4;
            double* ap = A + int64_t(r0 + lo + jc) * lda + r0 + i;
            if (iok && jc < ncol) ap[0] = cold[2 * nt] - c0;
            if (iok && jc + 1 < ncol) ap[lda] = cold[2 * nt + 1] - c1;
          }
        }
      }
    }
    mark(6);
    cluster.sync();  // ---- 4: A22 updated
    mark(7);
  }
  if (a.prof && q == 0 && tid == 0)
    for (int i = 0; i < 12; ++i) a.prof[i] = ph[i];
}

// Progress flags between the sweep warps (shared memory, CTA scope): release / acquire
// instead of a sequentially consistent fence on both sides of every task.
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(v) : "memory");
}

// ---------------------------------------------------------------- stage 2: band -> tridiagonal
// Band in shared memory: element (r, c), r >= c, at AB[r + 33 c] (column stride
// SB_LDB = 34: the diagonal and 2 BW sub-diagonals, room for the bulges), zero-padded by BW
// columns, so every task reads and writes whole 16 x 16 blocks without predicates (the
// entries past n are zero and stay exactly zero).
__device__ __forceinline__ int sbi(int r, int c) { return r + (SB_LDB - 1) * c; }

// LAPACK dlarfg on x (lane i = lane & 15 holds x_i; zeros past the vector): v_0 = 1,
// H x = beta e_0.
__device__ __forceinline__ void warp_larfg(double x, int i, double& beta, double& tau, double& v) {
  const double alpha = __shfl_sync(FULL, x, 0);
  double ss = i >= 1 ? x * x : 0.0;
  ss += __shfl_xor_sync(FULL, ss, 8);
  ss += __shfl_xor_sync(FULL, ss, 4);
  ss += __shfl_xor_sync(FULL, ss, 2);
  ss += __shfl_xor_sync(FULL, ss, 1);
  if (ss == 0.0) {
    beta = alpha;
    tau = 0.0;
    v = i == 0 ? 1.0 : 0.0;
    return;
  }
  beta = -copysign(sqrt(alpha * alpha + ss), alpha);
  tau = (beta - alpha) / beta;
  v = i == 0 ? 1.0 : x * (1.0 / (alpha - beta));
}

// D <- H D H on the symmetric diagonal block [st, st+16) (LAPACK dlarfy); lane (i, h) =
// (lane & 15, lane >> 4) holds D[i][8h .. 8h+8); vsh: v (16).
__device__ __forceinline__ void sb_sym_apply(double* AB, int st, double tau, double vi,
                                             const double* vsh, double* wsh, int lane) {
  const int i = lane & 15, h = lane >> 4;
  double* lo = AB + sbi(st + i, st + 8 * h);        // D[i][8h+jj] = lo[33 jj]  (8h+jj <= i)
  const double* up = AB + sbi(st + 8 * h, st + i);  // D[i][8h+jj] = up[jj]     (8h+jj > i)
  double d[8], vj[8];
  double t = 0.0;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    d[jj] = 8 * h + jj <= i ? lo[(SB_LDB - 1) * jj] : up[jj];
    vj[jj] = vsh[8 * h + jj];
    t += d[jj] * vj[jj];
  }
  t += __shfl_xor_sync(FULL, t, 16);
  double w = tau * t;
  double s = w * vi;  // both half-warps hold the same (w_i, v_i): reduce within each
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  w -= 0.5 * tau * s * vi;
  if (h == 0) wsh[i] = w;
  __syncwarp();
#pragma unroll
  for (int jj = 0; jj < 8; ++jj)
    if (8 * h + jj <= i) lo[(SB_LDB - 1) * jj] = d[jj] - vi * wsh[8 * h + jj] - w * vj[jj];
  __syncwarp();
}

// The band of A (lower, width BW, full storage lda) -> d (n), e (n-1); reflectors of sweep
// s, task k: rows s+1+k BW + i, v_i at V2[s n + k BW + i] (v_0 = 1), tau at TAU2[s KS + k].
// Task 0 of sweep s annihilates column s below the subdiagonal and applies the reflector to
// the first diagonal block; task k >= 1 applies the previous reflector from the right to the
// block below (creating the bulge), annihilates the bulge's first column with a new
// reflector (applied from the left to the rest of the block) and applies it to the next
// diagonal block (LAPACK dsb2st_kernels types 1, 2, 3).
__global__ void __launch_bounds__(SB_WARPS * 32, 1)
k_sb2st(const double* __restrict__ A, int64_t lda, int n, double* __restrict__ dout,
        double* __restrict__ eout, double* __restrict__ V2, double* __restrict__ TAU2, int KS,
        unsigned long long* prof) {
  extern __shared__ double sm[];
  double* AB = sm;
  double* scr = AB + size_t(SB_LDB) * (n + BW);
  __shared__ int prog_s[SB_WARPS];
  volatile int* prog = prog_s;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int idx = tid; idx < (n + BW) * SB_LDB; idx += blockDim.x) {
    const int c = idx / SB_LDB, off = idx % SB_LDB, r = c + off;
    AB[idx] = (off <= BW && r < n) ? A[r + int64_t(c) * lda] : 0.0;
  }
  if (tid < SB_WARPS) prog[tid] = tid * SB_KBIG;
  __syncthreads();
  double* vsh = scr + w * 32;
  double* wsh = vsh + 16;
  const int i = lane & 15, h = lane >> 4;
  long long t_wait = 0, t_start = clock64(), ntask = 0;
  for (int s = w; s <= n - 3; s += SB_WARPS) {
    const int pw = (s + SB_WARPS - 1) % SB_WARPS;
    auto wait = [&](int need) {  // sweep s-1 has finished `need` tasks (or all)
      if (s == 0) return;
      const int target = (s - 1) * SB_KBIG + need;
      if (lane == 0) {
        const long long t0 = prof ? clock64() : 0;
        while (ld_acquire_cta(prog_s + pw) < target) __nanosleep(20);
        if (prof) t_wait += clock64() - t0;
        ++ntask;
      }
      __syncwarp();  // lane 0's acquire + the warp barrier order the other lanes' reads
    };
    auto publish = [&](int val) {
      __syncwarp();
      if (lane == 0) st_release_cta(prog_s + w, val);  // after the warp barrier: all lanes' writes
    };
    double* Vs2 = V2 + size_t(s) * n;
    double* Ts2 = TAU2 + size_t(s) * KS;
    // task 0
    wait(2);
    int st = s + 1;
    {
      double* col = AB + sbi(st + i, s);
      double beta, tau, vi;
      warp_larfg(*col, i, beta, tau, vi);
      if (h == 0) {
        *col = i == 0 ? beta : 0.0;
        vsh[i] = vi;
        if (st + i < n) Vs2[i] = vi;
      }
      if (lane == 0) Ts2[0] = tau;
      __syncwarp();
      sb_sym_apply(AB, st, tau, vi, vsh, wsh, lane);
      publish(s * SB_KBIG + 1);
      int k = 1;
      while (st + BW < n) {
        wait(k + 2);
        const int j1 = st + BW;
        double* bp = AB + sbi(j1 + i, st + 8 * h);  // B[i][8h+jj] = bp[33 jj]
        double b[8], vj[8];
        double t = 0.0;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          b[jj] = bp[(SB_LDB - 1) * jj];
          vj[jj] = vsh[8 * h + jj];
          t += b[jj] * vj[jj];
        }
        t += __shfl_xor_sync(FULL, t, 16);
        const double tt = tau * t;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) b[jj] -= tt * vj[jj];
        const double x0 = __shfl_sync(FULL, b[0], i);
        double beta2, tau2, v2;
        warp_larfg(x0, i, beta2, tau2, v2);
        if (h == 0) b[0] = i == 0 ? beta2 : 0.0;
        double pp[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) pp[jj] = (8 * h + jj >= 1) ? v2 * b[jj] : 0.0;
        const double u = reduce8_half(pp, lane);
        __syncwarp();  // everyone is done with the old v
        if (h == 0) vsh[i] = v2;
        if ((lane & 1) == 0) wsh[8 * h + ((lane >> 1) & 7)] = u;
        __syncwarp();
        const double tv = tau2 * v2;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          if (8 * h + jj >= 1) b[jj] -= tv * wsh[8 * h + jj];
          bp[(SB_LDB - 1) * jj] = b[jj];
        }
        if (h == 0 && j1 + i < n) Vs2[j1 - s - 1 + i] = v2;
        if (lane == 0) Ts2[k] = tau2;
        __syncwarp();
        sb_sym_apply(AB, j1, tau2, v2, vsh, wsh, lane);
        st = j1;
        tau = tau2;
        ++k;
        publish(s * SB_KBIG + k);
      }
    }
    publish((s + 1) * SB_KBIG);
  }
  if (prof && lane == 0) {
    atomicAdd(prof, (unsigned long long)t_wait);
    atomicAdd(prof + 1, (unsigned long long)(clock64() - t_start));
    atomicAdd(prof + 2, (unsigned long long)ntask);
  }
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x) {
    dout[j] = AB[sbi(j, j)];
    if (j + 1 < n) eout[j] = AB[sbi(j + 1, j)];
  }
}

// ---------------------------------------------------------------- tridiagonal eigenvalues
// All eigenvalues of T = (d, e) by Sturm-count multisection, one warp per eigenvalue: each
// lane counts at EV_PTS points, so a round narrows the bracket 65-fold.  The count is the
// number of sign changes of the characteristic-polynomial sequence
// p_j = (d_j - x) p_{j-1} - e_{j-1}^2 p_{j-2} (p_j / p_{j-1} = LDL^T pivot q_j, the
// quantity LAPACK dstebz tests): two FMAs per step instead of a division, rescaled by
// 2^+-500 before it over/underflows, an exact zero p_j counted as a negative pivot (as
// dstebz's pivmin replacement does); the EV_PTS chains are independent (ILP).
constexpr int EV_WARPS = 4;
constexpr int EV_PTS = 2;

__global__ void __launch_bounds__(32 * EV_WARPS)
k_tridiag_eigvals_ms(const double* __restrict__ dg, const double* __restrict__ eg, int n,
                     double* __restrict__ w) {
  extern __shared__ double sme[];
  double* d = sme;       // n
  double* e2 = sme + n;  // n - 1
  __shared__ double red[3][EV_WARPS];
  double gl = 1e308, gu = -1e308;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double dj = dg[j];
    const double el = j > 0 ? fabs(eg[j - 1]) : 0.0, er = j + 1 < n ? fabs(eg[j]) : 0.0;
    d[j] = dj;
    if (j + 1 < n) e2[j] = eg[j] * eg[j];
    gl = fmin(gl, dj - el - er);
    gu = fmax(gu, dj + el + er);
  }
  for (int o = 16; o > 0; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(FULL, gl, o));
    gu = fmax(gu, __shfl_xor_sync(FULL, gu, o));
  }
  const int lane = threadIdx.x % 32, wib = threadIdx.x / 32;
  if (lane == 0) {
    red[0][wib] = gl;
    red[1][wib] = gu;
  }
  __syncthreads();
  gl = red[0][0];
  gu = red[1][0];
  for (int q = 1; q < EV_WARPS; ++q) {
    gl = fmin(gl, red[0][q]);
    gu = fmax(gu, red[1][q]);
  }
  const double eps = 2.220446049250313e-16;
  const double tnorm = fmax(fabs(gl), fabs(gu));
  gl -= 2.0 * eps * tnorm * n + 1e-300;
  gu += 2.0 * eps * tnorm * n + 1e-300;
  const int i = blockIdx.x * EV_WARPS + wib;  // eigenvalue index (ascending)
  if (i >= n) return;
  double lo = gl, hi = gu;
  const double atol = 2.0 * eps * tnorm + 1e-300;
  constexpr double BIG = 0x1p500, SMALL = 0x1p-500;
  for (int round = 0; round < 24; ++round) {
    const double width = hi - lo;
    if (width <= fmax(2.0 * eps * fmax(fabs(lo), fabs(hi)), atol)) break;
    double x[EV_PTS], p0[EV_PTS], p1[EV_PTS];
    int cnt[EV_PTS];
#pragma unroll
    for (int q = 0; q < EV_PTS; ++q) {
      x[q] = lo + width * double(lane * EV_PTS + q + 1) * (1.0 / (32 * EV_PTS + 1));
      p0[q] = 1.0;
      p1[q] = d[0] - x[q];
      if (p1[q] == 0.0) p1[q] = -0x1p-60;
      cnt[q] = p1[q] < 0.0;
    }
    // steps in groups of 4 (one rescale per group: |p| grows by < (3 ||T||)^4 per group)
    auto step = [&](int j) {
      const double dj = d[j], ej = e2[j - 1];
#pragma unroll
      for (int q = 0; q < EV_PTS; ++q) {
        const double t = ej * p0[q];
        double pn = fma(dj - x[q], p1[q], -t);
        pn = pn == 0.0 ? -p1[q] * 0x1p-60 : pn;
        cnt[q] += (pn < 0.0) != (p1[q] < 0.0);
        p0[q] = p1[q];
        p1[q] = pn;
      }
    };
    int j = 1;
    for (; j + 3 < n; j += 4) {
      step(j);
      step(j + 1);
      step(j + 2);
      step(j + 3);
#pragma unroll
      for (int q = 0; q < EV_PTS; ++q) {
        const double a = fmax(fabs(p1[q]), fabs(p0[q]));
        const double sc = a > BIG ? SMALL : (a < SMALL ? BIG : 1.0);
        p0[q] *= sc;
        p1[q] *= sc;
      }
    }
    for (; j < n; ++j) step(j);
    // first point (lane-major) whose count exceeds i: eigenvalue i lies below it
    int f = EV_PTS;
#pragma unroll
    for (int q = EV_PTS - 1; q >= 0; --q)
      if (cnt[q] > i) f = q;
    const unsigned any = __ballot_sync(FULL, f < EV_PTS);
    double nlo = lo, nhi = hi;
    if (any) {
      const int L = __ffs(any) - 1;
      const int fl = __shfl_sync(FULL, f, L);
      const int idx = L * EV_PTS + fl;
      double xs = x[0];
#pragma unroll
      for (int q = 1; q < EV_PTS; ++q)
        if (fl == q) xs = x[q];
      nhi = __shfl_sync(FULL, xs, L);
      if (idx > 0) {
        const int pl = (idx - 1) / EV_PTS, pq = (idx - 1) % EV_PTS;
        double xp = x[0];
#pragma unroll
        for (int q = 1; q < EV_PTS; ++q)
          if (pq == q) xp = x[q];
        nlo = __shfl_sync(FULL, xp, pl);
      }
    } else {
      nlo = __shfl_sync(FULL, x[EV_PTS - 1], 31);
    }
    if (nlo == lo && nhi == hi) break;  // no representable progress
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) w[i] = 0.5 * (lo + hi);
}

// ---------------------------------------------------------------- inverse iteration
// Eigenvector of the tridiagonal (d, e) for lam[j], one thread per vector, the LU factors
// (LAPACK dgttrf with partial pivoting, tiny pivots perturbed as dlagtf) and the iterate in
// shared memory, interleaved across the block's threads (conflict-free).  Three inverse
// iteration solves from a pseudo-random start; Y[:, j] unit 2-norm.
__global__ void __launch_bounds__(64)
k_tridiag_invit_sm(const double* __restrict__ dg, const double* __restrict__ eg, int n,
                   const double* __restrict__ lam, int k, double tnorm, double* __restrict__ Y) {
  extern __shared__ double smv[];
  const int nt = blockDim.x, tj = threadIdx.x;
  double* u1 = smv;              // 1 / pivot
  double* u2 = u1 + size_t(n) * nt;
  double* u3 = u2 + size_t(n) * nt;
  double* ml = u3 + size_t(n) * nt;
  double* x = ml + size_t(n) * nt;
  unsigned char* sw = reinterpret_cast<unsigned char*>(x + size_t(n) * nt);
  const int j = blockIdx.x * nt + tj;
  if (j >= k) return;
#define IX(i) (size_t(i) * nt + tj)
  const double eps = 2.220446049250313e-16;
  const double tiny = eps * fmax(tnorm, 1e-300);
  const double l = lam[j];
  double a = dg[0] - l, b = n > 1 ? eg[0] : 0.0, c = 0.0;
  for (int r = 0; r + 1 < n; ++r) {
    const double sub = eg[r], dn = dg[r + 1] - l, up = r + 2 < n ? eg[r + 1] : 0.0;
    if (fabs(sub) > fabs(a)) {
      const double rs = 1.0 / sub, m = a * rs;
      u1[IX(r)] = rs;
      u2[IX(r)] = dn;
      u3[IX(r)] = up;
      ml[IX(r)] = m;
      sw[IX(r)] = 1;
      a = b - m * dn;
      b = c - m * up;
    } else {
      if (fabs(a) < tiny) a = a >= 0.0 ? tiny : -tiny;
      const double ra = 1.0 / a, m = sub * ra;
      u1[IX(r)] = ra;
      u2[IX(r)] = b;
      u3[IX(r)] = c;
      ml[IX(r)] = m;
      sw[IX(r)] = 0;
      a = dn - m * b;
      b = up - m * c;
    }
    c = 0.0;
  }
  if (fabs(a) < tiny) a = a >= 0.0 ? tiny : -tiny;
  u1[IX(n - 1)] = 1.0 / a;
  uint32_t hsh = 0x9E3779B9u * uint32_t(j + 1);
  for (int r = 0; r < n; ++r) {
    hsh ^= hsh << 13;
    hsh ^= hsh >> 17;
    hsh ^= hsh << 5;
    x[IX(r)] = double(hsh & 0xFFFFFF) / double(0x1000000) + 0.5;
  }
  for (int it = 0; it < 3; ++it) {
    double xi = x[IX(0)];
    for (int r = 0; r + 1 < n; ++r) {  // L^{-1} P
      double xn = x[IX(r + 1)];
      if (sw[IX(r)]) {
        const double t = xi;
        xi = xn;
        xn = t;
      }
      x[IX(r)] = xi;
      xi = xn - ml[IX(r)] * xi;
    }
    x[IX(n - 1)] = xi;
    double mx = 0.0, x1 = 0.0, x2 = 0.0;
    for (int r = n - 1; r >= 0; --r) {  // U^{-1}
      const double v = (x[IX(r)] - u2[IX(r)] * x1 - u3[IX(r)] * x2) * u1[IX(r)];
      x[IX(r)] = v;
      x2 = x1;
      x1 = v;
      mx = fmax(mx, fabs(v));
    }
    const double s = mx > 0.0 ? 1.0 / mx : 1.0;
    for (int r = 0; r < n; ++r) x[IX(r)] *= s;
  }
  double nrm = 0.0;
  for (int r = 0; r < n; ++r) nrm += x[IX(r)] * x[IX(r)];
  nrm = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
  double* out = Y + size_t(j) * n;
  for (int r = 0; r < n; ++r) out[r] = x[IX(r)] * nrm;
#undef IX
}

// ---------------------------------------------------------------- back-transformation
// Z[:, c] = Q1 Q2 Y[:, c] for BT_CPB columns per CTA (Z may alias Y).  Q2 = product of the
// sweeps' reflectors in generation order, applied last sweep first; the reflectors of one
// sweep cover disjoint BW-row blocks starting at row s+1, so thread t handles row s+1+t and
// the dot products are half-warp reductions.  Q1 = P_0 .. P_{npan-1}, applied last first.
// Row r of the back-transform's column block (BT_CPB = 4 contiguous doubles) as two 16-byte
// shared-memory accesses: lanes on consecutive rows then touch one contiguous span instead
// of four 4-way bank-conflicted 8-byte accesses.
static_assert(BT_CPB == 4, "ys rows are two double2");
__device__ __forceinline__ void ys_load(const double* ys, int r, bool act, double* y) {
  if (act) {
    const double2 a = reinterpret_cast<const double2*>(ys + r * BT_CPB)[0];
    const double2 b = reinterpret_cast<const double2*>(ys + r * BT_CPB)[1];
    y[0] = a.x, y[1] = a.y, y[2] = b.x, y[3] = b.y;
  } else {
    y[0] = y[1] = y[2] = y[3] = 0.0;
  }
}
__device__ __forceinline__ void ys_store(double* ys, int r, const double* y) {
  reinterpret_cast<double2*>(ys + r * BT_CPB)[0] = make_double2(y[0], y[1]);
  reinterpret_cast<double2*>(ys + r * BT_CPB)[1] = make_double2(y[2], y[3]);
}

__global__ void __launch_bounds__(BT_THREADS)
k_band_backtransform(int n, int k, const double* __restrict__ V2, const double* __restrict__ TAU2,
                     int KS, const double* __restrict__ Vw, const double* __restrict__ Tw,
                     int npan, const double* Y, double* Z, int dbuf) {
  extern __shared__ __align__(16) double smb[];
  double* ys = smb;                        // n x BT_CPB (row-major)
  double* wv = ys + size_t(n) * BT_CPB;    // BW x BT_CPB
  double* tw = wv + BW * BT_CPB;           // BW x BT_CPB
  const int c0 = blockIdx.x * BT_CPB, nc = min(BT_CPB, k - c0);
  const int tid = threadIdx.x;
  for (int idx = tid; idx < n * BT_CPB; idx += BT_THREADS) {
    const int r = idx % n, c = idx / n;
    ys[r * BT_CPB + c] = c < nc ? Y[size_t(c0 + c) * n + r] : 0.0;
  }
  __syncthreads();
  // Q2: sweeps last to first.  Reflector j of sweep s (rows s+1+16j .. +15) is applied by a
  // half-warp: lane (rq, c) = (l >> 2, l & 3) holds rows 4 rq .. 4 rq + 3 of column c, sums
  // its 4 products and the half-warp reduces over rq with two shuffles (16 lanes x 16
  // shuffles per reflector before: the shuffle unit was the limit).  The next sweep's
  // reflector entries are prefetched into registers.
  double nv[2][4], ntau[2];
  auto fetch = [&](int s) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int t = tid + half * BT_THREADS, j = t >> 4, rq = (t & 15) >> 2;
      const int rows = n - 1 - s;
      ntau[half] = (s >= 0 && 16 * j < rows) ? __ldg(TAU2 + size_t(s) * KS + j) : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ti = 16 * j + 4 * rq + i;
        nv[half][i] = (s >= 0 && ti < rows) ? __ldg(V2 + size_t(s) * n + ti) : 0.0;
      }
    }
  };
  fetch(n - 3);
  for (int s = n - 3; s >= 0; --s) {
    const int rows = n - 1 - s;
    double cv[2][4], ctau[2];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      ctau[half] = ntau[half];
#pragma unroll
      for (int i = 0; i < 4; ++i) cv[half][i] = nv[half][i];
    }
    fetch(s - 1);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int t = tid + half * BT_THREADS, j = t >> 4, l = t & 15, c = l & 3, rq = l >> 2;
      if (16 * j >= rows) continue;  // whole half-warp beyond the sweep (uniform)
      const int rb = s + 1 + 16 * j + 4 * rq;
      double y[4], p = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool act = 16 * j + 4 * rq + i < rows;
        y[i] = act ? ys[(rb + i) * BT_CPB + c] : 0.0;
        p += cv[half][i] * y[i];
      }
      const unsigned hm = 0xffffu << (threadIdx.x & 16);
      p += __shfl_xor_sync(hm, p, 4, 16);
      p += __shfl_xor_sync(hm, p, 8, 16);
      const double f = ctau[half] * p;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (16 * j + 4 * rq + i < rows) ys[(rb + i) * BT_CPB + c] = y[i] - f * cv[half][i];
    }
    __syncthreads();
  }
  // Q1: panels last to first; thread (pair = tid / 8, seg = tid % 8), pair = (row of V^T, column)
  const int pair = tid >> 3, seg = tid & 7;
  const int pc = pair / BT_CPB, pcol = pair % BT_CPB;  // pair < 64 (512 threads)
  // the panels' V (BW x n, contiguous) arrive by bulk copy (TMA engine), double-buffered
  // when two fit in shared memory: the next panel streams in while this one is applied
  const int nbuf = dbuf ? 2 : 1;
  double* vsb = tw + BW * BT_CPB;  // nbuf x (BW x n)
  uint64_t* bar = reinterpret_cast<uint64_t*>(vsb + size_t(nbuf) * BW * n);
  const uint32_t vbytes = uint32_t(BW) * uint32_t(n) * 8u;
  if (tid == 0) {
    for (int b = 0; b < nbuf; ++b) oz::mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int p, int b) {
    if (tid == 0 && p >= 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      oz::mbar_expect_tx(&bar[b], vbytes);
      oz::bulk_g2s(vsb + size_t(b) * BW * n, Vw + size_t(p) * BW * n, vbytes, &bar[b]);
    }
  };
  issue(npan - 1, 0);
  if (nbuf == 2) issue(npan - 2, 1);
  uint32_t phase[2] = {0u, 0u};
  for (int p = npan - 1; p >= 0; --p) {
    const int r0 = (p + 1) * BW;
    const int b = nbuf == 2 ? (npan - 1 - p) & 1 : 0;
    double* vs = vsb + size_t(b) * BW * n;
    oz::mbar_wait(&bar[b], phase[b]);
    phase[b] ^= 1u;
    double acc0 = 0.0, acc1 = 0.0;
    int r = r0 + pc + seg;
    for (; r + 8 < n; r += 16) {
      acc0 += vs[pc * n + r] * ys[r * BT_CPB + pcol];
      acc1 += vs[pc * n + r + 8] * ys[(r + 8) * BT_CPB + pcol];
    }
    if (r < n) acc0 += vs[pc * n + r] * ys[r * BT_CPB + pcol];
    double acc = acc0 + acc1;
    acc += __shfl_xor_sync(FULL, acc, 4);
    acc += __shfl_xor_sync(FULL, acc, 2);
    acc += __shfl_xor_sync(FULL, acc, 1);
    if (seg == 0) wv[pc * BT_CPB + pcol] = acc;
    __syncthreads();
    if (tid < BW * BT_CPB) {  // tw = T wv (T upper triangular, column-major)
      const int rr = tid / BT_CPB, cc = tid % BT_CPB;
      const double* Tp = Tw + size_t(p) * BW * BW;
      double s = 0.0;
      for (int e = rr; e < BW; ++e) s += __ldg(Tp + rr + e * BW) * wv[e * BT_CPB + cc];
      tw[tid] = s;
    }
    __syncthreads();
    for (int r = r0 + tid; r < n; r += BT_THREADS) {
      double y[BT_CPB];
      ys_load(ys, r, true, y);
#pragma unroll
      for (int e = 0; e < BW; ++e) {
        const double v = vs[e * n + r];
#pragma unroll
        for (int c = 0; c < BT_CPB; ++c) y[c] -= v * tw[e * BT_CPB + c];
      }
      ys_store(ys, r, y);
    }
    __syncthreads();  // vs consumed: refill it with panel p - nbuf
    issue(p - nbuf, b);
  }
  for (int idx = tid; idx < n * nc; idx += BT_THREADS) {
    const int r = idx % n, c = idx / n;
    Z[size_t(c0 + c) * n + r] = ys[r * BT_CPB + c];
  }
}

}  // namespace band
}  // namespace latsum_b200
