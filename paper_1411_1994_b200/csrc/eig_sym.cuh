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

// A[i, j] = A[j, i] for i < j: the Grams come from a lower-triangle SYRK (as syevd reads them)
__global__ void k_symmetrize_lower(double* __restrict__ A, int64_t lda, int n) {
  const int64_t total = int64_t(n) * n;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(idx % n), j = int(idx / n);
    if (i < j) A[i + int64_t(j) * lda] = A[j + int64_t(i) * lda];
  }
}

// out[0] = max |S - I| over the k x k matrix S (one block)
__global__ void k_max_offidentity(const double* __restrict__ S, int k, double* __restrict__ out) {
  double m = 0.0;
  for (int64_t idx = threadIdx.x; idx < int64_t(k) * k; idx += blockDim.x) {
    const int i = int(idx % k), j = int(idx / k);
    const double dv = fabs(S[idx] - (i == j ? 1.0 : 0.0));
    // fmax drops NaN: a non-finite vector must fail the check (-> the syevd fallback)
    m = (dv == dv && dv <= 1e300) ? fmax(m, dv) : INFINITY;
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < int(blockDim.x / 32); ++q) m = fmax(m, red[q]);
    out[0] = fmax(m, red[0]);
  }
}

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

// ---------------------------------------------------------------- tridiagonal eigenvalues
// All eigenvalues of the symmetric tridiagonal T = (d, e) by Sturm-count multisection: one
// warp per eigenvalue, the 32 lanes count at 32 interior points of the current bracket, so
// each round narrows it 33-fold (LAPACK dstebz's bisection, parallelised).  The counts are
// exact to ~eps ||T|| (Kahan), which bounds the absolute accuracy as for any backward-
// stable solver (syevd included).  w ascending.
constexpr int EIG_WARPS = 8;  // warps (eigenvalues) per block

__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2,
                                           int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (q < 0.0) ++cnt;
  for (int j = 1; j < n; ++j) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = d[j] - x - e2[j - 1] / q;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

__global__ void __launch_bounds__(32 * EIG_WARPS)
k_tridiag_eigvals(const double* __restrict__ dg, const double* __restrict__ eg, int n,
                  double* __restrict__ w) {
  extern __shared__ double sm[];
  double* d = sm;       // n
  double* e2 = sm + n;  // n - 1
  __shared__ double red[3][32 * EIG_WARPS / 32];
  double gl = 1e308, gu = -1e308, em = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double dj = dg[j];
    const double el = j > 0 ? fabs(eg[j - 1]) : 0.0, er = j + 1 < n ? fabs(eg[j]) : 0.0;
    d[j] = dj;
    if (j + 1 < n) e2[j] = eg[j] * eg[j];
    gl = fmin(gl, dj - el - er);
    gu = fmax(gu, dj + el + er);
    em = fmax(em, er * er);
  }
  for (int o = 16; o > 0; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
    gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
    em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
  }
  const int lane = threadIdx.x % 32, wib = threadIdx.x / 32;
  if (lane == 0) {
    red[0][wib] = gl;
    red[1][wib] = gu;
    red[2][wib] = em;
  }
  __syncthreads();
  gl = red[0][0], gu = red[1][0], em = red[2][0];
  for (int q = 1; q < EIG_WARPS; ++q) {
    gl = fmin(gl, red[0][q]);
    gu = fmax(gu, red[1][q]);
    em = fmax(em, red[2][q]);
  }
  const double eps = 2.220446049250313e-16;
  const double tnorm = fmax(fabs(gl), fabs(gu));
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, em) * 4.0;
  gl -= 2.0 * eps * tnorm * n + 2.0 * pivmin;
  gu += 2.0 * eps * tnorm * n + 2.0 * pivmin;
  const int i = blockIdx.x * EIG_WARPS + wib;  // eigenvalue index (ascending)
  if (i >= n) return;
  double lo = gl, hi = gu;
  // stop at the accuracy the Sturm counts support: eps ||T|| absolute (as syevd)
  const double atol = 2.0 * eps * tnorm + 4.0 * pivmin;
  for (int round = 0; round < 40; ++round) {
    const double width = hi - lo;
    if (width <= fmax(2.0 * eps * fmax(fabs(lo), fabs(hi)), atol)) break;
    const double x = lo + width * double(lane + 1) / 33.0;
    const int cnt = sturm_count(d, e2, n, x, pivmin);
    const unsigned above = __ballot_sync(0xffffffffu, cnt > i);  // x beyond eigenvalue i
    double nlo = lo, nhi = hi;
    if (above) {
      const int f = __ffs(above) - 1;
      nhi = __shfl_sync(0xffffffffu, x, f);
      if (f > 0) nlo = __shfl_sync(0xffffffffu, x, f - 1);
    } else {
      nlo = __shfl_sync(0xffffffffu, x, 31);
    }
    if (nlo == lo && nhi == hi) break;  // no representable progress
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) w[i] = 0.5 * (lo + hi);
}

// ---------------------------------------------------------------- inverse iteration
// Eigenvector of T for the eigenvalue lam[j] (one thread each): LU of T - lam I with partial
// pivoting (LAPACK dgttrf; pivots below eps ||T|| perturbed, as dlagtf), then two inverse
// iteration solves from a pseudo-random start.  Accurate as syevd's vectors (error
// ~ eps ||T|| / gap); callers orthonormalise the bases they build from them.
// Y[:, j] (n x k), unit 2-norm.  ws: 5 n doubles per thread.
// one thread per vector, blockDim.x vectors per block with their LU factors in shared memory
__global__ void __launch_bounds__(32)
k_tridiag_invit(const double* __restrict__ dg, const double* __restrict__ eg, int n,
                const double* __restrict__ lam, int k, double tnorm, double* __restrict__ Y) {
  extern __shared__ double smf[];  // blockDim.x x 5 n
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const double eps = 2.220446049250313e-16;
  const double tiny = eps * fmax(tnorm, 1e-300);
  const double l = lam[j];
  double* u1 = smf + int64_t(threadIdx.x) * 5 * n;  // U diagonal
  double* u2 = u1 + n;                               // U first super-diagonal
  double* u3 = u2 + n;                               // U second super-diagonal (fill from swaps)
  double* ml = u3 + n;                               // multipliers
  double* sw = ml + n;                               // 1: rows i, i+1 swapped at step i
  double* x = Y + int64_t(j) * n;
  double a = dg[0] - l, b = n > 1 ? eg[0] : 0.0, c = 0.0;  // current row (cols i, i+1, i+2)
  for (int i = 0; i + 1 < n; ++i) {
    const double sub = eg[i], dn = dg[i + 1] - l, up = i + 2 < n ? eg[i + 1] : 0.0;
    if (fabs(sub) > fabs(a)) {
      const double m = a / sub;
      u1[i] = sub;
      u2[i] = dn;
      u3[i] = up;
      ml[i] = m;
      sw[i] = 1.0;
      a = b - m * dn;
      b = c - m * up;
    } else {
      if (fabs(a) < tiny) a = a >= 0.0 ? tiny : -tiny;
      const double m = sub / a;
      u1[i] = a;
      u2[i] = b;
      u3[i] = c;
      ml[i] = m;
      sw[i] = 0.0;
      a = dn - m * b;
      b = up - m * c;
    }
    c = 0.0;
  }
  if (fabs(a) < tiny) a = a >= 0.0 ? tiny : -tiny;
  u1[n - 1] = a;
  // pseudo-random start (an all-ones start can be orthogonal to the eigenvector), kept
  // in the output column
  uint32_t h = 0x9E3779B9u * uint32_t(j + 1);
  for (int i = 0; i < n; ++i) {
    h ^= h << 13;
    h ^= h >> 17;
    h ^= h << 5;
    x[i] = double(h & 0xFFFFFF) / double(0x1000000) + 0.5;
  }
  for (int it = 0; it < 3; ++it) {
    double xi = x[0];
    for (int i = 0; i + 1 < n; ++i) {  // L^{-1} P, streaming x[i+1]
      double xn = x[i + 1];
      if (sw[i] != 0.0) {
        const double t = xi;
        xi = xn;
        xn = t;
      }
      x[i] = xi;
      xi = xn - ml[i] * xi;
    }
    x[n - 1] = xi;
    double mx = 0.0, x1 = 0.0, x2 = 0.0;  // x[i+1], x[i+2]
    for (int i = n - 1; i >= 0; --i) {  // U^{-1}
      const double v = (x[i] - u2[i] * x1 - u3[i] * x2) / u1[i];
      x[i] = v;
      x2 = x1;
      x1 = v;
      mx = fmax(mx, fabs(v));
    }
    const double s = mx > 0.0 ? 1.0 / mx : 1.0;
    for (int i = 0; i < n; ++i) x[i] *= s;
  }
  double nrm = 0.0;
  for (int i = 0; i < n; ++i) nrm += x[i] * x[i];
  nrm = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
  for (int i = 0; i < n; ++i) x[i] *= nrm;
}

// ---------------------------------------------------------------- back-transformation
// Q = H_0 H_1 .. H_{n-2} (sytrd 'L') applied to Y in compact-WY blocks of NB reflectors:
// Q_b = I - V_b T_b V_b^T (LAPACK dlarft, forward / columnwise).  k_wy_build materialises
// V_b (n x NB, unit lower trapezoidal from the reflectors stored in A) and T_b for every
// block (one CTA per block); the caller applies Y <- Y - V_b (T_b (V_b^T Y)) with GEMMs,
// last block first.
constexpr int WY_NB = 64;

__global__ void __launch_bounds__(256)
k_wy_build(const double* __restrict__ A, int64_t lda, int n, const double* __restrict__ tau,
           double* __restrict__ V, double* __restrict__ T) {
  const int blk = blockIdx.x;
  const int j0 = blk * WY_NB;  // first reflector of the block
  const int nr = n - 1;        // reflectors 0 .. n-2
  const int nb = min(WY_NB, nr - j0);
  double* Vb = V + int64_t(blk) * WY_NB * n;
  double* Tb = T + int64_t(blk) * WY_NB * WY_NB;
  extern __shared__ double wysm[];  // S and T: 2 x WY_NB x (WY_NB + 1)
  double (*S)[WY_NB + 1] = reinterpret_cast<double (*)[WY_NB + 1]>(wysm);
  double (*Ts)[WY_NB + 1] = reinterpret_cast<double (*)[WY_NB + 1]>(wysm + WY_NB * (WY_NB + 1));
  for (int idx = threadIdx.x; idx < WY_NB * n; idx += blockDim.x) {
    const int jj = idx / n, r = idx % n;
    const int kk = j0 + jj;  // reflector index
    double v = 0.0;
    if (jj < nb) {
      if (r == kk + 1) v = 1.0;
      else if (r > kk + 1) v = A[r + int64_t(kk) * lda];
    }
    Vb[r + int64_t(jj) * n] = v;
  }
  __syncthreads();
  // S = V_b^T V_b (upper part needed)
  for (int idx = threadIdx.x; idx < WY_NB * WY_NB; idx += blockDim.x) {
    const int p = idx / WY_NB, q = idx % WY_NB;
    double acc = 0.0;
    if (p < q && q < nb) {
      const double* vp = Vb + int64_t(p) * n;
      const double* vq = Vb + int64_t(q) * n;
      for (int r = j0 + q + 1; r < n; ++r) acc += vp[r] * vq[r];
    }
    S[p][q] = acc;
    Ts[p][q] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < nb; ++q) {
      const double tq = tau[j0 + q];
      // T[0:q, q] = -tau_q T[0:q, 0:q] S[0:q, q]
      for (int p = 0; p < q; ++p) {
        double acc = 0.0;
        for (int m = p; m < q; ++m) acc += Ts[p][m] * S[m][q];
        Ts[p][q] = -tq * acc;
      }
      Ts[q][q] = tq;
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < WY_NB * WY_NB; idx += blockDim.x) {
    const int p = idx % WY_NB, q = idx / WY_NB;
    Tb[p + q * WY_NB] = Ts[p][q];  // column-major
  }
}

// ---------------------------------------------------------------- shared-memory sytrd
// The same reduction with the trailing matrix resident in the cluster's shared memory
// (n <= SM_TRD_MAX): CTA q keeps the lower part L[c.., c] of the columns c = q (mod 16).
// Per column k (reflector v_k, tau_k in every CTA's smem):
//   A  p-partials: pacc[r] = sum_{own c <= r} L[r,c] v[c] (row gather) + for own c the
//      column dot sum_{r > c} L[r,c] v[r] (A = L + L^T - D)                | cluster barrier
//   B  reduce-scatter: CTA q sums the 16 partials of its rows r = q (mod 16) through
//      DSMEM, p = tau pacc, and its share of p.v                           | cluster barrier
//   C  gather p (DSMEM), alpha = -tau/2 p.v, w = p + alpha v, update own columns
//      L -= v w^T + w v^T; the owner of column k+1 then builds reflector k+1 | cluster barrier
//   D  every CTA copies v_{k+1} from the owner's shared memory.
// Outputs as k_sytrd_cluster (d, e, tau; reflectors below the subdiagonal of A).
constexpr int SM_TRD_THREADS = 512;
constexpr int SM_TRD_WARPS = SM_TRD_THREADS / 32;
constexpr int SM_TRD_MAXCOL = 64;  // columns per CTA (n <= 1024)
// doubles of shared memory for n: the owned lower columns plus 5 vectors
__host__ __device__ inline int64_t sm_trd_doubles(int n) {
  int64_t m = 0;
  for (int q = 0; q < TRD_CTAS; ++q) {  // the largest share (q = 0)
    int64_t t = 0;
    for (int c = q; c < n; c += TRD_CTAS) t += n - c;
    m = t > m ? t : m;
  }
  return m + 5 * int64_t(n) + 8;
}

__global__ void __launch_bounds__(SM_TRD_THREADS, 1)
k_sytrd_smem(double* __restrict__ A, int64_t lda, int n, double* __restrict__ d,
             double* __restrict__ e, double* __restrict__ tau, long long* __restrict__ prof) {
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = clock64();
#define TRD_MARK(i)                         \
  if (prof) {                               \
    const long long t1 = clock64();         \
    tacc[i] += t1 - t0;                     \
    t0 = t1;                                \
  }
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid % 32, wib = tid / 32;
  extern __shared__ double sm[];
  __shared__ int off[SM_TRD_MAXCOL + 1];
  __shared__ double red[SM_TRD_WARPS];
  __shared__ double scal[4];  // [0..1] tau by parity, [2] p.v partial, [3] alpha
  const int ncol = n > q ? (n - q + TRD_CTAS - 1) / TRD_CTAS : 0;  // owned columns
  if (tid == 0) {
    int o = 0;
    for (int lc = 0; lc <= ncol; ++lc) {
      off[lc] = o;
      if (lc < ncol) o += n - (q + TRD_CTAS * lc);
    }
  }
  __syncthreads();
  // the vectors sit at the same offset in every CTA (after the largest column share,
  // CTA 0's) so that DSMEM addresses map across the cluster
  int share0 = 0;
  for (int c = 0; c < n; c += TRD_CTAS) share0 += n - c;
  double* Lm = sm;
  double* vbuf = sm + share0;     // 2 n
  double* pacc = vbuf + 2 * n;    // n
  double* psl = pacc + n;         // n (own rows)
  double* wv = psl + n;           // n
  // load the owned lower columns
  for (int lc = wib; lc < ncol; lc += SM_TRD_WARPS) {
    const int c = q + TRD_CTAS * lc;
    const double* src = A + int64_t(c) * lda;
    for (int r = c + lane; r < n; r += 32) Lm[off[lc] + (r - c)] = src[r];
  }
  __syncthreads();
  auto Lat = [&](int r, int lc, int c) -> double& { return Lm[off[lc] + (r - c)]; };

  // reflector kk from the owner's column kk (local smem), by warp 0 of the owner CTA:
  // v -> vbuf[par] rows kk+1.., scal[par] = tau; global d, e, tau and A[kk+2.., kk]
  auto reflector = [&](int kk, int par) {
    const int lc = kk / TRD_CTAS;
    double* x = Lm + off[lc];  // x[r - kk] = L[r, kk]
    if (lane == 0) d[kk] = x[0];
    if (kk + 1 >= n) return;
    const double alpha = x[1];
    double ss = 0.0;
    for (int r = kk + 2 + lane; r < n; r += 32) ss += x[r - kk] * x[r - kk];
    ss = warp_sum(ss);
    double beta, tk, sc;
    if (ss == 0.0) {
      beta = alpha;
      tk = 0.0;
      sc = 0.0;
    } else {
      const double nrm = sqrt(alpha * alpha + ss);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tk = (beta - alpha) / beta;
      sc = 1.0 / (alpha - beta);
    }
    double* v = vbuf + par * n;
    double* col = A + int64_t(kk) * lda;
    for (int r = kk + 1 + lane; r < n; r += 32) {
      const double vr = r == kk + 1 ? 1.0 : x[r - kk] * sc;
      v[r] = vr;
      if (r > kk + 1) col[r] = vr;
    }
    if (lane == 0) {
      e[kk] = beta;
      tau[kk] = tk;
      col[kk + 1] = beta;
      scal[par] = tk;
    }
  };

  if (q == 0 && wib == 0) reflector(0, 0);
  cluster.sync();
  if (q != 0) {
    const double* vo = cluster.map_shared_rank(vbuf, 0);
    for (int r = 1 + tid; r < n; r += SM_TRD_THREADS) vbuf[r] = vo[r];
    if (tid == 0) scal[0] = *cluster.map_shared_rank(&scal[0], 0);
  }
  __syncthreads();

  for (int k = 0; k + 1 < n; ++k) {
    const int par = k & 1;
    const double* v = vbuf + par * n;
    const double tk = scal[par];
    // ---- A: symv partials over the owned columns c >= k+1
    for (int r = k + 1 + tid; r < n; r += SM_TRD_THREADS) {
      double s = 0.0;
      for (int lc = 0; lc < ncol; ++lc) {
        const int c = q + TRD_CTAS * lc;
        if (c > r) break;
        if (c >= k + 1) s += Lat(r, lc, c) * v[c];
      }
      pacc[r] = s;
    }
    __syncthreads();
    for (int lc = wib; lc < ncol; lc += SM_TRD_WARPS) {
      const int c = q + TRD_CTAS * lc;
      if (c < k + 1) continue;
      double s = 0.0;
      for (int r = c + 1 + lane; r < n; r += 32) s += Lat(r, lc, c) * v[r];
      s = warp_sum(s);
      if (lane == 0) pacc[c] += s;
    }
    TRD_MARK(0);
    cluster.sync();
    TRD_MARK(1);
    // ---- B: reduce-scatter of the own rows r = q (mod 16), r >= k+1
    {
      double dp = 0.0;
      // 16 threads per row: thread t reads CTA (t % 16)'s partial
      const int src = tid % TRD_CTAS, slot = tid / TRD_CTAS;  // 32 rows in flight
      const double* pr = cluster.map_shared_rank(pacc, src);
      const int r0 = ((k + 1 + TRD_CTAS - 1 - q) / TRD_CTAS) * TRD_CTAS + q;  // first own row >= k+1
      // warp-uniform trip count: both 16-lane halves shuffle together
      const int nown = r0 < n ? (n - 1 - r0) / TRD_CTAS + 1 : 0;  // own rows >= k+1
      const int per = SM_TRD_THREADS / TRD_CTAS;                    // rows per sweep
      for (int base = 0; base < nown; base += per) {
        const int j = base + slot;
        const int r = r0 + TRD_CTAS * j;
        double part = j < nown ? pr[r] : 0.0;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (src == 0 && j < nown) {
          const double pv = tk * part;
          psl[r] = pv;
          dp += pv * v[r];
        }
      }
      dp = warp_sum(dp);
      if (lane == 0) red[wib] = dp;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < SM_TRD_WARPS; ++w) t += red[w];
        scal[2] = t;
      }
    }
    TRD_MARK(2);
    cluster.sync();
    TRD_MARK(3);
    // ---- C: gather p, w, update, next reflector
    if (tid < 32) {
      double t = lane < TRD_CTAS ? *cluster.map_shared_rank(&scal[2], lane) : 0.0;
      t = warp_sum(t);
      if (lane == 0) scal[3] = -0.5 * tk * t;
    }
    __syncthreads();
    const double alpha = scal[3];
    for (int r = k + 1 + tid; r < n; r += SM_TRD_THREADS) {
      const double pr = *cluster.map_shared_rank(&psl[r], r % TRD_CTAS);
      wv[r] = pr + alpha * v[r];
    }
    __syncthreads();
    TRD_MARK(4);
    const int own1 = (k + 1) % TRD_CTAS == q;  // this CTA owns column k+1
    if (own1 && wib == 0) {
      const int lc = (k + 1) / TRD_CTAS, c = k + 1;
      if (tk != 0.0) {
        const double vc = v[c], wc = wv[c];
        for (int r = c + lane; r < n; r += 32) Lat(r, lc, c) -= v[r] * wc + wv[r] * vc;
      }
      __syncwarp();
      reflector(k + 1, par ^ 1);
    }
    if (tk != 0.0) {
      // warps 1.. (or all when column k+1 is elsewhere) update the other owned columns
      const int w0 = own1 ? 1 : 0, nw = own1 ? SM_TRD_WARPS - 1 : SM_TRD_WARPS;
      if (wib >= w0) {
        for (int lc = wib - w0; lc < ncol; lc += nw) {
          const int c = q + TRD_CTAS * lc;
          if (c < k + 2) continue;
          const double vc = v[c], wc = wv[c];
          for (int r = c + lane; r < n; r += 32) Lat(r, lc, c) -= v[r] * wc + wv[r] * vc;
        }
      }
    }
    TRD_MARK(5);
    cluster.sync();
    TRD_MARK(6);
    // ---- D: copy v_{k+1} and tau_{k+1} from the owner of column k+1
    if (k + 2 < n) {
      const int ow = (k + 1) % TRD_CTAS;
      if (ow != q) {
        double* vn = vbuf + (par ^ 1) * n;
        const double* vo = cluster.map_shared_rank(vbuf + (par ^ 1) * n, ow);
        for (int r = k + 2 + tid; r < n; r += SM_TRD_THREADS) vn[r] = vo[r];
        if (tid == 0) scal[par ^ 1] = *cluster.map_shared_rank(&scal[par ^ 1], ow);
      }
      __syncthreads();
    }
    TRD_MARK(7);
  }
  if (prof && tid == 0 && q == 0)
    for (int i = 0; i < 8; ++i) prof[i] = tacc[i];
  cluster.sync();  // no CTA exits while a peer may still read its shared memory
#undef TRD_MARK
}

}  // namespace eig
}  // namespace latsum_b200
