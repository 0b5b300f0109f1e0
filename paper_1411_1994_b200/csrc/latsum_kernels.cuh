// Stage kernels of the lattice-sum hot path (sm_100a, FP64).
//
// Layouts: every matrix is column-major with the
// grid index fastest, as Eigen stores the reference's side matrices.
//   ref_l   : 2N_l x Rd    distinct reference columns (t_{-k} = -t_k share one)
//   dict_l  : N_l  x d_l   distinct side-matrix columns, d_l = P_l * Rd, column
//                          c = p * Rd + j holds placement p (a sublattice shift list
//                          or one defect shift) of reference column j
//   terms   : T merged canonical terms (c0, c1, c2, w) sorted by c0
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace latsum_b200 {

// ---------------------------------------------------------------- helpers

// Deterministic block sum (fixed tree); blockDim.x must be a power of two <= 1024.
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = blockDim.x / 32;
  if (warp == 0) {
    v = lane < nw ? red[lane] : 0.0;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// erf(hi) - erf(lo) routed through erfc on the same-sign side (reference.hpp:21-25).
__device__ __forceinline__ double erf_difference(double lo, double hi) {
  if (lo >= 0.0) return erfc(lo) - erfc(hi);
  if (hi <= 0.0) return erfc(-hi) - erfc(-lo);
  return erf(hi) - erf(lo);
}

// ---------------------------------------------------------------- stage 1

// entry(i, k) = int over cell i of exp(-s_k x^2) dx (reference.hpp:33-54), one thread
// per (cell, distinct term).  Cell bounds lo = lower + i h, hi = lo + h are formed
// without FMA contraction exactly as the host does; the cell integral is the
// cancellation-free hybrid (4-point Gauss-Legendre when sqrt(s) h < 0.05, the
// reference's erf difference otherwise).
__global__ void k_ref_integrals(const double* __restrict__ s, int64_t n2, double lower, double h,
                                double* __restrict__ out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int k = blockIdx.y;
  if (i >= n2) return;
  const double sk = s[k];
  double v;
  if (sk == 0.0) {
    v = h;
  } else {
    const double rs = sqrt(sk);
    const double lo = __dadd_rn(lower, __dmul_rn(double(i), h));
    if (__dmul_rn(rs, h) < 0.05) {
      const double xg[4] = {-0.86113631159405257522, -0.33998104358485626480,
                            0.33998104358485626480, 0.86113631159405257522};
      const double wg[4] = {0.34785484513745385737, 0.65214515486254614263,
                            0.65214515486254614263, 0.34785484513745385737};
      const double half = __dmul_rn(0.5, h);
      const double mid = __dadd_rn(lo, half);
      double acc = 0.0;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const double x = __dadd_rn(mid, __dmul_rn(half, xg[g]));
        acc = __dadd_rn(acc, __dmul_rn(wg[g], exp(__dmul_rn(__dmul_rn(-sk, x), x))));
      }
      v = __dmul_rn(half, acc);
    } else {
      const double hi = __dadd_rn(lo, h);
      const double c = sqrt(M_PI) / (2.0 * rs);
      v = __dmul_rn(c, erf_difference(__dmul_rn(rs, lo), __dmul_rn(rs, hi)));
    }
  }
  out[i + k * n2] = v;
}

// from_raw for one mode (canonical.hpp:32-48): one block per column, ordered
// reduction of the squares, then col /= norm (zero column -> e_0).
__global__ void k_normalize_columns(double* __restrict__ m, int64_t rows, double* __restrict__ norms) {
  __shared__ double red[32];
  double* c = m + int64_t(blockIdx.x) * rows;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) s += c[i] * c[i];
  const double nrm = sqrt(block_sum(s, red));
  if (threadIdx.x == 0) norms[blockIdx.x] = nrm;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x)
    c[i] = nrm == 0.0 ? (i == 0 ? 1.0 : c[i]) : c[i] / nrm;
}

// ---------------------------------------------------------------- stage 2

// Value of dictionary column c at row i: sum over the placement's shifts of
// ref_j[N/2 - shift + i] (assembled_vector, lattice_sum.hpp:101-144; ascending
// order of the shift list).
struct DictArgs {
  const double* ref;       // 2N x Rd
  int64_t N;
  int Rd;
  const int64_t* pl_off;   // P+1
  const int64_t* pl_shift; // shifts
  double* dict;            // N x d
  double* partial;         // d x nchunk
  double* norms;           // d
  int64_t chunk;
  int nchunk;
  int64_t c0 = 0;          // first column handled by this launch (blockIdx.x + c0)
  // per placement: the stride n of a uniformly strided shift list summed by the sliding
  // recursion (k_dict_sliding), 0 for the direct sum; null: every placement direct
  const int64_t* pl_stride = nullptr;
};

// Dictionary entries of column c = (placement p, reference column j) for the DICT_RT rows
// i0 + tid + DICT_THREADS r of this thread: v[r] = sum_{s in placement p} ref_j[N/2 - shift_s
// + i].  Shifts outer, rows inner: the DICT_RT loads per shift are independent and coalesced
// across the block (the shift list sits in shared memory), so the 256-shift sublattice
// columns (cfg5) stream instead of forming one dependent L2 chain per entry.
constexpr int DICT_THREADS = 256, DICT_RT = 8, DICT_MAXSH = 1024;
static_assert(DICT_THREADS * DICT_RT == 2048, "2048-row sub-chunks; a block covers a chunk of them");

__device__ __forceinline__ void dict_values(const DictArgs& a, const double* __restrict__ rj,
                                            const int64_t* __restrict__ sh, int ns, int64_t i0,
                                            int64_t i1, double* v) {
#pragma unroll
  for (int r = 0; r < DICT_RT; ++r) v[r] = 0.0;
  for (int s = 0; s < ns; ++s) {
    const double* src = rj + (a.N / 2 - sh[s]);
#pragma unroll
    for (int r = 0; r < DICT_RT; ++r) {
      const int64_t i = i0 + threadIdx.x + int64_t(DICT_THREADS) * r;
      if (i < i1) v[r] += src[i];
    }
  }
}

// stage the placement's shift list in shared memory (long lists: read from global)
__device__ __forceinline__ const int64_t* dict_shifts(const DictArgs& a, int64_t p, int64_t* buf,
                                                      int& ns) {
  const int64_t s0 = a.pl_off[p], s1 = a.pl_off[p + 1];
  ns = int(s1 - s0);
  if (ns > DICT_MAXSH) return a.pl_shift + s0;
  for (int s = threadIdx.x; s < ns; s += blockDim.x) buf[s] = a.pl_shift[s0 + s];
  __syncthreads();
  return buf;
}

__global__ void __launch_bounds__(DICT_THREADS) k_dict_sumsq(DictArgs a) {
  __shared__ double red[32];
  __shared__ int64_t shb[DICT_MAXSH];
  const int64_t c = blockIdx.x + a.c0;
  const int64_t p = c / a.Rd, j = c % a.Rd;
  if (a.pl_stride && a.pl_stride[p] > 0) return;  // summed by k_dict_sliding
  const double* rj = a.ref + j * 2 * a.N;
  int ns;
  const int64_t* sh = dict_shifts(a, p, shb, ns);
  const int64_t c0 = blockIdx.y * a.chunk, c1 = min(a.N, c0 + a.chunk);
  double s = 0.0;
  for (int64_t i0 = c0; i0 < c1; i0 += DICT_THREADS * DICT_RT) {  // 2048-row sub-chunks
    double v[DICT_RT];
    dict_values(a, rj, sh, ns, i0, c1, v);
#pragma unroll
    for (int r = 0; r < DICT_RT; ++r) s += v[r] * v[r];
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) a.partial[c * a.nchunk + blockIdx.y] = s;
}

__global__ void k_dict_norms(DictArgs a, int64_t d) {
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x + a.c0;
  if (c >= d) return;
  if (a.pl_stride && a.pl_stride[c / a.Rd] > 0) return;  // k_dict_sliding wrote this norm
  double s = 0.0;
  for (int q = 0; q < a.nchunk; ++q) s += a.partial[c * a.nchunk + q];
  a.norms[c] = sqrt(s);
}

__global__ void __launch_bounds__(DICT_THREADS) k_dict_write(DictArgs a) {
  __shared__ int64_t shb[DICT_MAXSH];
  const int64_t c = blockIdx.x + a.c0;
  const int64_t p = c / a.Rd, j = c % a.Rd;
  const double* rj = a.ref + j * 2 * a.N;
  if (a.pl_stride && a.pl_stride[p] > 0) {  // raw values are in place (k_dict_sliding): scale them
    const double nrm = a.norms[c];
    const double inv = nrm == 0.0 ? 0.0 : 1.0 / nrm;
    double* out = a.dict + c * a.N;
    const int64_t c0 = blockIdx.y * a.chunk, c1 = min(a.N, c0 + a.chunk);
    for (int64_t i = c0 + threadIdx.x; i < c1; i += DICT_THREADS)
      out[i] = nrm == 0.0 ? (i == 0 ? 1.0 : 0.0) : out[i] * inv;
    return;
  }
  int ns;
  const int64_t* sh = dict_shifts(a, p, shb, ns);
  const int64_t c0 = blockIdx.y * a.chunk, c1 = min(a.N, c0 + a.chunk);
  const double nrm = a.norms[c];
  const double inv = nrm == 0.0 ? 0.0 : 1.0 / nrm;  // one division per column, not per entry
  double* out = a.dict + c * a.N;
  for (int64_t i0 = c0; i0 < c1; i0 += DICT_THREADS * DICT_RT) {  // 2048-row sub-chunks
    double v[DICT_RT];
    dict_values(a, rj, sh, ns, i0, c1, v);
#pragma unroll
    for (int r = 0; r < DICT_RT; ++r) {
      const int64_t i = i0 + threadIdx.x + int64_t(DICT_THREADS) * r;
      if (i < c1) out[i] = nrm == 0.0 ? (i == 0 ? 1.0 : 0.0) : v[r] * inv;
    }
  }
}

// The reference's default accumulation order (Accumulation::sliding, assembled_vector,
// lattice_sum.hpp:116-128) for a placement of L uniformly strided shifts c_k = c_0 + k n: the
// first n rows are direct sums over k (ascending), every later row reuses the overlap of
// consecutive windows, v[i] = v[i - n] + ref[hi + i] - ref[lo + i] with hi = N/2 - c_0 (the term
// entering) and lo = N/2 - (c_{L-1} + n) (the term leaving): O(N + L n) reads per column instead
// of O(L N) (cfg5: 256 shifts).  One thread per residue i mod n walks its chain, in the
// reference's own operation order.  Raw values go to the dictionary column and the column's sum
// of squares to the norm; k_dict_write then scales the column.  One block per column.
__global__ void __launch_bounds__(DICT_THREADS) k_dict_sliding(DictArgs a) {
  __shared__ double red[32];
  const int64_t c = blockIdx.x + a.c0;
  const int64_t p = c / a.Rd, j = c % a.Rd;
  const int64_t n = a.pl_stride[p];
  if (n <= 0) return;
  const int64_t s0 = a.pl_off[p], L = a.pl_off[p + 1] - s0;
  const double* __restrict__ rj = a.ref + j * 2 * a.N;
  const double* __restrict__ hi = rj + (a.N / 2 - a.pl_shift[s0]);
  const double* __restrict__ lo = rj + (a.N / 2 - (a.pl_shift[s0 + L - 1] + n));
  double* __restrict__ out = a.dict + c * a.N;
  double ss = 0.0;
  for (int64_t r = threadIdx.x; r < n && r < a.N; r += DICT_THREADS) {
    double v = 0.0;
    for (int64_t k = 0; k < L; ++k) v += rj[a.N / 2 - a.pl_shift[s0 + k] + r];
    out[r] = v;
    ss += v * v;
    int64_t i = r + n;
    for (; i + 3 * n < a.N; i += 4 * n) {  // the loads do not depend on the chain: issue them first
      const double h0 = hi[i], h1 = hi[i + n], h2 = hi[i + 2 * n], h3 = hi[i + 3 * n];
      const double l0 = lo[i], l1 = lo[i + n], l2 = lo[i + 2 * n], l3 = lo[i + 3 * n];
      v = v + h0 - l0;
      out[i] = v;
      ss += v * v;
      v = v + h1 - l1;
      out[i + n] = v;
      ss += v * v;
      v = v + h2 - l2;
      out[i + 2 * n] = v;
      ss += v * v;
      v = v + h3 - l3;
      out[i + 3 * n] = v;
      ss += v * v;
    }
    for (; i < a.N; i += n) {
      v = v + hi[i] - lo[i];
      out[i] = v;
      ss += v * v;
    }
  }
  ss = block_sum(ss, red);
  if (threadIdx.x == 0) a.norms[c] = sqrt(ss);
}

// Single-shift placements (windowed_canonical, lattice_sum.hpp:148-157: the defect columns, all
// but a few of a dictionary): one block per column does the whole column in one launch — the
// window's sum of squares (from L2), the norm, then the normalised column — with no partial-sum
// round trip and no second grid, so the blocks' L2-bound first halves overlap other blocks'
// HBM-bound second halves.  Same summation order as k_dict_sumsq / k_dict_norms with one chunk
// per column: the norms are bit-identical to that path's.
__global__ void __launch_bounds__(DICT_THREADS) k_dict_single(DictArgs a) {
  __shared__ double red[32];
  const int64_t c = blockIdx.x + a.c0;
  const int64_t p = c / a.Rd, j = c % a.Rd;
  const double* __restrict__ src = a.ref + j * 2 * a.N + (a.N / 2 - a.pl_shift[a.pl_off[p]]);
  double s = 0.0;
  for (int64_t i0 = 0; i0 < a.N; i0 += DICT_THREADS * DICT_RT) {
    double v[DICT_RT];
#pragma unroll
    for (int r = 0; r < DICT_RT; ++r) {
      const int64_t i = i0 + threadIdx.x + int64_t(DICT_THREADS) * r;
      v[r] = i < a.N ? src[i] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < DICT_RT; ++r) s += v[r] * v[r];
  }
  s = block_sum(s, red);
  const double nrm = sqrt(s);
  if (threadIdx.x == 0) a.norms[c] = nrm;
  const double inv = nrm == 0.0 ? 0.0 : 1.0 / nrm;
  double* __restrict__ out = a.dict + c * a.N;
  for (int64_t i0 = 0; i0 < a.N; i0 += DICT_THREADS * DICT_RT) {
    double v[DICT_RT];
#pragma unroll
    for (int r = 0; r < DICT_RT; ++r) {
      const int64_t i = i0 + threadIdx.x + int64_t(DICT_THREADS) * r;
      v[r] = i < a.N ? src[i] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < DICT_RT; ++r) {
      const int64_t i = i0 + threadIdx.x + int64_t(DICT_THREADS) * r;
      if (i < a.N) out[i] = nrm == 0.0 ? (i == 0 ? 1.0 : 0.0) : v[r] * inv;
    }
  }
}

// out[:, q] = dict[:, idx[q]] — the reference-form N x M_c side matrix (HBM-bound
// gather with 128-bit accesses when rows are even).
__global__ void k_gather_columns(const double* __restrict__ dict, int64_t rows,
                                 const int64_t* __restrict__ idx, double* __restrict__ out) {
  const int64_t q = blockIdx.y;
  const double* src = dict + idx[q] * rows;
  double* dst = out + q * rows;
  if ((rows & 1) == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows / 2;
         i += int64_t(gridDim.x) * blockDim.x)
      d2[i] = s2[i];
  } else {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows;
         i += int64_t(gridDim.x) * blockDim.x)
      dst[i] = src[i];
  }
}

// ---------------------------------------------------------------- stage 3 helpers

// out[:, c] = in[:, c] * scale[c]   (optionally in place)
__global__ void k_scale_columns(const double* __restrict__ in, int64_t rows, int64_t cols,
                                const double* __restrict__ scale, double* __restrict__ out) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x)
    out[e] = in[e] * scale[e / rows];
}

// out[:, q] = src[:, cols[q]] * (w ? w[q] : 1)   (rows x T gather, src leading dim ld)
__global__ void k_gather_scale(const double* __restrict__ src, int64_t rows, int64_t ld,
                               const int32_t* __restrict__ cols, const double* __restrict__ w,
                               int64_t T, double* __restrict__ out) {
  const int64_t total = rows * T;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = e / rows, i = e % rows;
    const double v = src[i + int64_t(cols[q]) * ld];
    out[e] = w ? v * w[q] : v;
  }
}

// dst[:, j] = src[:, n - 1 - j] for j < k   (ascending eigenvectors -> descending)
__global__ void k_reverse_columns(const double* __restrict__ src, int64_t rows, int64_t n,
                                  int64_t k, double* __restrict__ dst) {
  const int64_t total = rows * k;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / rows, i = e % rows;
    dst[e] = src[i + (n - 1 - j) * rows];
  }
}

// dst[:, j] = src[:, sel[j]]
__global__ void k_select_columns(const double* __restrict__ src, int64_t rows,
                                 const int64_t* __restrict__ sel, int64_t k,
                                 double* __restrict__ dst) {
  const int64_t total = rows * k;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / rows, i = e % rows;
    dst[e] = src[i + sel[j] * rows];
  }
}

// ||A||^2 = sum_{t,u} w_t w_u prod_l G_l[c_l(t), c_l(u)] (canonical.hpp:148-162 with the
// three M x M Grams replaced by d_l x d_l dictionary Grams).  A block owns NORM_TPB terms
// t (NORM_TPW per warp); the u terms stream through shared memory in chunks, lanes stride
// over u (coalesced), and each t's partial is reduced in a fixed order:
// partial[t] = w_t * sum_u (...).
constexpr int NORM_TPW = 4, NORM_WARPS = 8, NORM_TPB = NORM_TPW * NORM_WARPS, NORM_CHUNK = 1024;
__global__ void __launch_bounds__(NORM_WARPS * 32)
k_hadamard_norm_rows(const double* __restrict__ G0, const double* __restrict__ G1,
                     const double* __restrict__ G2, int64_t d0, int64_t d1, int64_t d2,
                     const int32_t* __restrict__ c0, const int32_t* __restrict__ c1,
                     const int32_t* __restrict__ c2, const double* __restrict__ w, int64_t T,
                     double* __restrict__ partial) {
  __shared__ int32_t s0[NORM_CHUNK], s1[NORM_CHUNK], s2[NORM_CHUNK];
  __shared__ double sw[NORM_CHUNK];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t tbase = int64_t(blockIdx.x) * NORM_TPB + warp * NORM_TPW;
  const double* g0[NORM_TPW];
  const double* g1[NORM_TPW];
  const double* g2[NORM_TPW];
  double acc[NORM_TPW];
#pragma unroll
  for (int q = 0; q < NORM_TPW; ++q) {
    const int64_t t = min(tbase + q, T - 1);
    g0[q] = G0 + int64_t(c0[t]) * d0;
    g1[q] = G1 + int64_t(c1[t]) * d1;
    g2[q] = G2 + int64_t(c2[t]) * d2;
    acc[q] = 0.0;
  }
  for (int64_t u0 = 0; u0 < T; u0 += NORM_CHUNK) {
    const int n = int((T - u0) < NORM_CHUNK ? (T - u0) : NORM_CHUNK);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      s0[i] = c0[u0 + i];
      s1[i] = c1[u0 + i];
      s2[i] = c2[u0 + i];
      sw[i] = w[u0 + i];
    }
    __syncthreads();
    for (int i = lane; i < n; i += 32) {
      const int a = s0[i], b = s1[i], cc = s2[i];
      const double wu = sw[i];
#pragma unroll
      for (int q = 0; q < NORM_TPW; ++q) acc[q] += wu * (g0[q][a] * g1[q][b] * g2[q][cc]);
    }
  }
#pragma unroll
  for (int q = 0; q < NORM_TPW; ++q) {
    double v = acc[q];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    const int64_t t = tbase + q;
    if (lane == 0 && t < T) partial[t] = w[t] * v;
  }
}

// Ordered sum of n values by one block (deterministic).
__global__ void k_sum(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// ---------------------------------------------------------------- stage 4 helpers

// X[t + T*(j + nj*kk)] = w_t * D2[k0+kk, c2_t] * D1[j0+j, c1_t] : the canonical slab
// operand (canonical.hpp:192-202 to_dense as one GEMM per z-slab).
__global__ void k_canonical_slab_operand(const double* __restrict__ D1, int64_t N1,
                                         const double* __restrict__ D2, int64_t N2,
                                         const int32_t* __restrict__ c1,
                                         const int32_t* __restrict__ c2,
                                         const double* __restrict__ w, int64_t T, int64_t j0,
                                         int64_t nj, int64_t k0, int64_t nk,
                                         double* __restrict__ X) {
  const int64_t total = T * nj * nk;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = e % T, j = (e / T) % nj, kk = e / (T * nj);
    X[e] = w[t] * D2[(k0 + kk) + int64_t(c2[t]) * N2] * D1[(j0 + j) + int64_t(c1[t]) * N1];
  }
}

// Tucker entries at probes: out[p] = sum_{b,c} W[p + np*(b + r1*c)] U1[j_p, b] U2[k_p, c]
// with W = U0[i_p, :] * core_(1) precomputed by a GEMM.
__global__ void k_tucker_probe_finish(const double* __restrict__ W, int64_t np, int64_t r1,
                                      int64_t r2, const double* __restrict__ U1, int64_t N1,
                                      const double* __restrict__ U2, int64_t N2,
                                      const int64_t* __restrict__ probes,
                                      double* __restrict__ out) {
  __shared__ double red[32];
  const int64_t p = blockIdx.x;
  const int64_t j = probes[3 * p + 1], k = probes[3 * p + 2];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < r1 * r2; e += blockDim.x) {
    const int64_t b = e % r1, c = e / r1;
    s += W[p + np * e] * U1[j + b * N1] * U2[k + c * N2];
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[p] = s;
}

// Canonical entries at probes (canonical.hpp:63-70) over merged terms.
__global__ void k_canonical_probes(const double* __restrict__ D0, int64_t N0,
                                   const double* __restrict__ D1, int64_t N1,
                                   const double* __restrict__ D2, int64_t N2,
                                   const int32_t* __restrict__ c0, const int32_t* __restrict__ c1,
                                   const int32_t* __restrict__ c2, const double* __restrict__ w,
                                   int64_t T, const int64_t* __restrict__ probes,
                                   double* __restrict__ out) {
  __shared__ double red[32];
  const int64_t p = blockIdx.x;
  const int64_t i = probes[3 * p], j = probes[3 * p + 1], k = probes[3 * p + 2];
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x)
    s += w[t] * D0[i + int64_t(c0[t]) * N0] * D1[j + int64_t(c1[t]) * N1] *
         D2[k + int64_t(c2[t]) * N2];
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[p] = s;
}

// rows gather: out[p + np*a] = U[idx_p + N*a]
__global__ void k_gather_rows(const double* __restrict__ U, int64_t N, int64_t r,
                              const int64_t* __restrict__ probes, int comp, int64_t np,
                              double* __restrict__ out) {
  const int64_t total = np * r;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = e % np, a = e / np;
    out[e] = U[probes[3 * p + comp] + N * a];
  }
}

}  // namespace latsum_b200

namespace latsum_b200 {

// ---------------------------------------------------------------- verification

// Brute-force windowed sum (lattice_sum.hpp:656-671 oracle_entry) at probe p over the
// sources [s0, s1): sum_s w_s sum_k w_k prod_l ref_l[N_l/2 - c_{s,l} + i_l, jmap[k]],
// the reference's own loop order per source; block partial -> part[p * nchunk + chunk].
struct VerifyArgs {
  const double* ref[3];     // 2N_l x Rd distinct unit columns
  int64_t N[3];
  const int32_t* jmap;      // R -> distinct column
  const double* wref;       // R reference weights
  int R;
  const int64_t* shifts;    // ns x 3
  const double* sw;         // ns
  int64_t ns;
  const int64_t* probes;    // np x 3
  int64_t chunk;
  int nchunk;
  double* part;
};

__global__ void k_verify_partial(VerifyArgs a) {
  __shared__ double red[32];
  const int64_t p = blockIdx.x;
  const int64_t i = a.probes[3 * p], j = a.probes[3 * p + 1], k = a.probes[3 * p + 2];
  const int64_t s0 = int64_t(blockIdx.y) * a.chunk;
  const int64_t s1 = min(a.ns, s0 + a.chunk);
  double acc = 0.0;
  for (int64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    const double* r0 = a.ref[0] + (a.N[0] / 2 - a.shifts[3 * s] + i);
    const double* r1 = a.ref[1] + (a.N[1] / 2 - a.shifts[3 * s + 1] + j);
    const double* r2 = a.ref[2] + (a.N[2] / 2 - a.shifts[3 * s + 2] + k);
    double e = 0.0;
    for (int q = 0; q < a.R; ++q) {
      const int64_t c = a.jmap[q];
      e += a.wref[q] * r0[c * 2 * a.N[0]] * r1[c * 2 * a.N[1]] * r2[c * 2 * a.N[2]];
    }
    acc += a.sw[s] * e;
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) a.part[p * a.nchunk + blockIdx.y] = acc;
}

__global__ void k_verify_finish(const double* __restrict__ part, int nchunk, int64_t np,
                                double* __restrict__ out) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= np) return;
  double s = 0.0;
  for (int c = 0; c < nchunk; ++c) s += part[p * nchunk + c];
  out[p] = s;
}

}  // namespace latsum_b200

namespace latsum_b200 {

// core'[j + r1 (i + r0 k)] = core[i + r0 (j + r1 k)]  (swap the first two modes)
__global__ void k_swap01(const double* __restrict__ in, int64_t r0, int64_t r1, int64_t r2,
                         double* __restrict__ out) {
  const int64_t total = r0 * r1 * r2;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % r0, j = (e / r0) % r1, k = e / (r0 * r1);
    out[j + r1 * (i + r0 * k)] = in[e];
  }
}

// sum of squares of the core entries with index_l == at inside the box [0, r) (one block)
__global__ void k_slice_mass(const double* __restrict__ core, int64_t d0, int64_t d1, int l,
                             int64_t at, int64_t b0, int64_t b1, int64_t b2,
                             double* __restrict__ out) {
  __shared__ double red[32];
  const int64_t n_a = l == 0 ? b1 : b0, n_b = l == 2 ? b1 : b2;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < n_a * n_b; e += blockDim.x) {
    const int64_t x = e % n_a, y = e / n_a;
    int64_t i, j, k;
    if (l == 0) { i = at; j = x; k = y; }
    else if (l == 1) { i = x; j = at; k = y; }
    else { i = x; j = y; k = at; }
    const double v = core[i + d0 * (j + d1 * k)];
    s += v * v;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// out (b0 x b1 x b2) = the leading box of core (d0 x d1 x d2)
__global__ void k_crop(const double* __restrict__ core, int64_t d0, int64_t d1, int64_t b0,
                       int64_t b1, int64_t b2, double* __restrict__ out) {
  const int64_t total = b0 * b1 * b2;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % b0, j = (e / b0) % b1, k = e / (b0 * b1);
    out[e] = core[i + d0 * (j + d1 * k)];
  }
}

// Per-block partial sums of squares of a column-major rows x cols block (leading dim ld);
// k_sum then adds the gridDim.x partials in order (deterministic).
__global__ void k_sumsq_partial(const double* __restrict__ v, int64_t rows, int64_t cols,
                                int64_t ld, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double x = v[(i % rows) + (i / rows) * ld];
    s += x * x;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Standard normal samples, counter-based (splitmix64 + Box-Muller): out[i] depends only on
// (seed, i), so the sketch is reproducible and independent of the launch shape.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void k_fill_gauss(double* __restrict__ out, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t a = splitmix64(seed ^ (uint64_t(i) * 2 + 0)), b = splitmix64(seed ^ (uint64_t(i) * 2 + 1));
    const double u1 = (double(a >> 11) + 0.5) * 0x1p-53, u2 = double(b >> 11) * 0x1p-53;
    out[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

__global__ void k_sumsq(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += v[i] * v[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

}  // namespace latsum_b200

namespace latsum_b200 {

// Low-rank canonical evaluation on a box (canonical.hpp:192-202 to_dense) for T <= 64
// merged terms, output-write bound (2 T flops per 8-byte point sits below the FP64 ridge):
// each thread keeps A0[i, :] = D0[i, c0_t] for cp_ipt rows in registers (zero-padded to
// the rank bucket MAXT: T rounded up to even below 24, so at most one FMA per point is
// padding), the block stages x_t(j,k) = w_t D1[j, c1_t] D2[k, c2_t] for CP_PAIRS (j,k)
// pairs in shared memory, double-buffered so the next batch's gathers overlap this batch's
// FMAs and stores; x is read as 16-byte pairs (one shared load per 2 cp_ipt FMAs); stores
// are coalesced along i.  Registers stay <= 128 (4 CTAs per SM; 2 for the 48 and 64 buckets) to keep
// stores in flight.
constexpr int CP_MAXT = 64, CP_PAIRS = 32, CP_THREADS = 128;
template <int MAXT>
constexpr int cp_ipt() { return MAXT <= 18 ? 4 : (MAXT <= 24 ? 2 : 1); }
template <int MAXT>
constexpr int cp_minb() { return (MAXT <= 18 || MAXT > 32) ? 2 : (MAXT <= 24 ? 3 : 4); }
template <int MAXT>
__global__ void __launch_bounds__(CP_THREADS, cp_minb<MAXT>())
k_cp_eval_small(const double* __restrict__ D0, int64_t ld0, const double* __restrict__ D1,
                int64_t ld1, const double* __restrict__ D2, int64_t ld2,
                const int32_t* __restrict__ c0, const int32_t* __restrict__ c1,
                const int32_t* __restrict__ c2, const double* __restrict__ w, int T, int64_t ni,
                int64_t nj, int64_t nk, double* __restrict__ out) {
  static_assert(MAXT % 2 == 0, "x is read in pairs");
  constexpr int CP_IPT = cp_ipt<MAXT>();
  __shared__ __align__(16) double xs[2][CP_PAIRS][MAXT];
  const int64_t ibase = blockIdx.x * int64_t(CP_THREADS * CP_IPT) + threadIdx.x;
  double a[CP_IPT][MAXT];
#pragma unroll
  for (int u = 0; u < CP_IPT; ++u) {
    const int64_t i = ibase + u * CP_THREADS;
#pragma unroll
    for (int t = 0; t < MAXT; ++t) a[u][t] = (t < T && i < ni) ? D0[i + int64_t(c0[t]) * ld0] : 0.0;
  }
  const int64_t npairs = nj * nk, stride = int64_t(gridDim.y) * CP_PAIRS;
  // the term table (weight, mode-1 and mode-2 columns) in shared memory, loaded once
  __shared__ double ws[MAXT];
  __shared__ int c1s[MAXT], c2s[MAXT];
  for (int t = threadIdx.x; t < MAXT; t += CP_THREADS) {
    ws[t] = t < T ? w[t] : 0.0;
    c1s[t] = t < T ? c1[t] : 0;
    c2s[t] = t < T ? c2[t] : 0;
  }
  __syncthreads();
  // staging is software-pipelined: the next batch's factor entries are loaded into
  // registers before this batch's FMAs and written to shared memory after them, so the L2
  // latency of the gathers overlaps the compute and the stores
  constexpr int NSLOT = (CP_PAIRS * MAXT + CP_THREADS - 1) / CP_THREADS;
  double g1[NSLOT], g2[NSLOT];
  auto gather = [&](int64_t p0) {
    const int64_t j0 = p0 % nj, k0 = p0 / nj;  // one division per batch
#pragma unroll
    for (int m = 0; m < NSLOT; ++m) {
      const int e = threadIdx.x + m * CP_THREADS;
      const int q = e / MAXT, t = e % MAXT;
      g1[m] = g2[m] = 0.0;
      if (e < CP_PAIRS * MAXT && p0 + q < npairs && t < T) {
        int64_t j = j0 + q, k = k0;
        while (j >= nj) {
          j -= nj;
          ++k;
        }
        g2[m] = D2[k + int64_t(c2s[t]) * ld2];
        g1[m] = D1[j + int64_t(c1s[t]) * ld1];
      }
    }
  };
  auto put = [&](int buf) {
#pragma unroll
    for (int m = 0; m < NSLOT; ++m) {
      const int e = threadIdx.x + m * CP_THREADS;
      if (e < CP_PAIRS * MAXT) (&xs[buf][0][0])[e] = ws[e % MAXT] * g2[m] * g1[m];
    }
  };
  int64_t p0 = int64_t(blockIdx.y) * CP_PAIRS;
  if (p0 < npairs) {
    gather(p0);
    put(0);
  }
  __syncthreads();
  for (int buf = 0; p0 < npairs; p0 += stride, buf ^= 1) {
    const bool more = p0 + stride < npairs;
    if (more) gather(p0 + stride);  // loads in flight during this batch
    const int nq = int((npairs - p0) < CP_PAIRS ? (npairs - p0) : CP_PAIRS);
    for (int q = 0; q < nq; ++q) {
      double s[CP_IPT];
#pragma unroll
      for (int u = 0; u < CP_IPT; ++u) s[u] = 0.0;
      const double2* x2 = reinterpret_cast<const double2*>(&xs[buf][q][0]);
#pragma unroll
      for (int t = 0; t < MAXT; t += 2) {
        const double2 x = x2[t / 2];
#pragma unroll
        for (int u = 0; u < CP_IPT; ++u) {
          s[u] += a[u][t] * x.x;
          s[u] += a[u][t + 1] * x.y;
        }
      }
      const int64_t p = p0 + q;
#pragma unroll
      for (int u = 0; u < CP_IPT; ++u) {
        const int64_t i = ibase + u * CP_THREADS;
        if (i < ni) out[i + ni * p] = s[u];
      }
    }
    if (more) put(buf ^ 1);  // consumed one iteration ago
    __syncthreads();  // buf consumed, buf ^ 1 staged
  }
}

}  // namespace latsum_b200
