// FP64-accurate GEMM on the INT8 tensor cores of sm_100a (Ozaki scheme I).
//
// C = A B (FP64) with A (M x K) and B (K x N).  Every row of A and column of B is scaled
// by a power of two into (-1, 1), rounded to the integer X = rint(2^54 x) (|error| <=
// 2^-55, unbiased) and written in balanced base 256 as S = 7 signed int8 digits,
//   X = sum_s d_s 2^{8(6-s)},  d_1..d_6 in [-128, 127],  d_0 in [-65, 65],
// so x = sum_s 2^{-6-8s} d_s and C = diag(2^e) [ sum_g 2^{-12-8g} D_g ] diag(2^f) with
// D_g = sum_{s+t=g} A_s B_t.  Each A_s B_t is exact in int32, the 28 pairs with s + t <= 6
// are kept (a dropped pair weighs <= 2^-54 K of the row/column maxima and has no sign
// bias), and the 7 group sums accumulate in TMEM as int32 (|D_g| <= 7 * 2^14 K < 2^31
// for K <= 16384).  The epilogue folds the groups exactly in int64 (two words: g = 0..3
// and g = 4..6), converts each once and adds them with one rounding.
//
// Data path: operands are pre-sliced into the canonical K-major "no swizzle" core-matrix
// layout (8 rows x 16 bytes) per (tile, k-block, slice), so each pipeline stage is one
// contiguous bulk copy per operand (cp.async.bulk, TMA engine) completing on an mbarrier.
// Tiles are 128 x 128 and every tile runs two passes over K, because TMEM (512 columns)
// holds four 128-column int32 groups: pass 1 accumulates groups 0..3 (the 10 pairs with
// s + t <= 3, slices 0..3 only), pass 2 groups 4..6 (18 pairs, all slices).  One thread
// issues tcgen05.mma.kind::i8 (M=128, N=128, K=32); the N=128 shape halves the shared-
// memory operand reads per product against N=64 (the MMA's smem port is the limit).
// Eight epilogue warps drain TMEM with tcgen05.ld after each pass.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace latsum_b200 {
namespace oz {

constexpr int S = 7;                 // slices per operand
constexpr int BM = 128, BN = 128;    // output tile (TMEM lanes x accumulator columns)
constexpr int BKB = 32;              // k-block (int8 elements = bytes) per stage
constexpr int STAGES = 4;
constexpr int A_BLK = BM * BKB;      // one slice's A block (bytes)
constexpr int B_BLK = BN * BKB;
constexpr int A_STAGE = S * A_BLK;   // 28 KB (pass 2; pass 1 loads the first 4 slices)
constexpr int B_STAGE = S * B_BLK;   // 28 KB
constexpr int P1_SLICES = 4;         // pass 1: groups g = s + t <= 3
constexpr int TMEM_COLS = 512;       // 4 groups x 128 columns
constexpr int KMAX = 16384;          // int32 accumulator headroom

// byte offset of (row r, k) inside a rows x BKB block in the canonical K-major layout
__host__ __device__ __forceinline__ int blk_off(int r, int k) {
  return (r >> 3) * (BKB / 16) * 128 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}

// 2^e with |x| * 2^-e < 1 for the largest |x| (frexp exponent); 0 for an all-zero line
__device__ __forceinline__ int line_exponent(double amax) {
  if (amax == 0.0) return 0;
  int e;
  frexp(amax, &e);
  return e;
}

// balanced base-256 digits of rint(2^54 x) for x in (-1, 1), most significant first
__device__ __forceinline__ void digits(double x, int8_t* d) {
  long long X = __double2ll_rn(x * 0x1p54);
#pragma unroll
  for (int s = S - 1; s > 0; --s) {
    const long long r = ((X + 128) & 255) - 128;
    d[s] = int8_t(r);
    X = (X - r) >> 8;
  }
  d[0] = int8_t(X);
}

// Operands are "lines" (rows of A, columns of B) of K elements: element (l, k) of the
// FP64 source is P[(l % L1) sl + (l / L1) sl2 + k sk] (L1 = L: a plain matrix; otherwise a
// batch of L/L1 matrices stacked as one operand).  One CTA slices a tile of ROWS lines over all
// k-blocks: pass 1 finds each line's scale 2^e (max |x| 2^-e < 1; 1 for a zero line),
// pass 2 re-reads the tile (L1/L2-resident) and writes its S digit blocks per k-block in
// the canonical K-major layout, 16 k-bytes of one line per thread as 16-byte stores.
// VEC: lines are contiguous (sk == 1) and 16-byte aligned, loads are double2.
template <int ROWS, bool VEC>
__device__ __forceinline__ void load16(const double* __restrict__ p, int64_t sk, int64_t k0,
                                       int64_t K, double* x) {
  if (VEC && k0 + 16 <= K) {
#pragma unroll
    for (int kk = 0; kk < 16; kk += 2) {
      const double2 v = *reinterpret_cast<const double2*>(p + k0 + kk);
      x[kk] = v.x;
      x[kk + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) x[kk] = k0 + kk < K ? p[(k0 + kk) * sk] : 0.0;
  }
}

// max |x| over k-blocks [kb0, kb1) of this thread's half (16 k of each 32-k block)
template <int ROWS, bool VEC>
__device__ __forceinline__ double slice_amax(const double* p, int64_t sk, int64_t K, int h,
                                             int64_t kb0, int64_t kb1) {
  double amax = 0.0;
  for (int64_t kb = kb0; kb < kb1; ++kb) {
    double x[16];
    load16<ROWS, VEC>(p, sk, kb * BKB + 16 * h, K, x);
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) amax = fmax(amax, fabs(x[kk]));
  }
  return amax;
}

// the S digit blocks of k-blocks [kb0, kb1) for line r (valid: l < L) of tile `tile`
template <int ROWS, bool VEC>
__device__ __forceinline__ void slice_digits(const double* p, int64_t sk, int64_t K, int h, int r,
                                             bool valid, double inv54, int64_t tile, int64_t KB,
                                             int64_t kb0, int64_t kb1, int8_t* __restrict__ out,
                                             int halves) {
  for (int64_t kb = kb0; kb < kb1; ++kb) {
    uint32_t w[S][4];
#pragma unroll
    for (int s = 0; s < S; ++s) w[s][0] = w[s][1] = w[s][2] = w[s][3] = 0u;
    if (valid) {
      double x[16];
      load16<ROWS, VEC>(p, sk, kb * BKB + 16 * h, K, x);
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        // balanced base-256 digits of X = rint(2^54 x): with Y = X + sum_i 128 256^i the
        // low digits are the bytes of Y minus 128 (byte ^ 0x80) and the top one Y >> 48
        const long long X = __double2ll_rn(x[kk] * inv54);
        const unsigned long long Y = static_cast<unsigned long long>(X + 0x808080808080LL);
        const uint32_t lo = uint32_t(Y) ^ 0x80808080u;        // d6 d5 d4 d3 (bytes 0..3)
        const uint32_t hi = uint32_t(Y >> 32) ^ 0x00008080u;  // d2 d1 d0 (bytes 0..2)
        const int pp = kk % 4;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const uint32_t src = s <= 2 ? hi : lo;
          const int m = s <= 2 ? 2 - s : 6 - s;  // byte of src holding digit s
          const uint32_t sel = (0x3210u & ~(0xFu << (4 * pp))) | (uint32_t(4 + m) << (4 * pp));
          w[s][kk / 4] = __byte_perm(w[s][kk / 4], src, sel);
        }
      }
    }
    // halves = 2 (B operand of the 2-SM kernel): [half][slice][64 lines], so that each CTA
    // of the pair loads its 64 lines of all slices with one contiguous copy
    const int hr = halves == 2 ? r / (ROWS / 2) : 0, rr = halves == 2 ? r % (ROWS / 2) : r;
    const int blk = ROWS / (halves == 2 ? 2 : 1) * BKB;
    int8_t* base = out + ((tile * KB + kb) * S) * int64_t(ROWS * BKB) + int64_t(hr) * S * blk +
                   blk_off(rr, 16 * h);
#pragma unroll
    for (int s = 0; s < S; ++s)
      *reinterpret_cast<uint4*>(base + s * blk) = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
  }
}

template <int ROWS, bool VEC>
__global__ void __launch_bounds__(2 * ROWS)
k_slice_tile(const double* __restrict__ P, int64_t sl, int64_t sk, int64_t L, int64_t K,
             int64_t KB, double* __restrict__ scale, int8_t* __restrict__ out, int64_t L1,
             int64_t sl2, int halves) {
  // persistent over tiles: one resident tile per CTA keeps the pass-2 re-read in L2
  __shared__ double part[ROWS];
  const int r = threadIdx.x % ROWS, h = threadIdx.x / ROWS;  // line in tile, k half
  const int64_t tiles = (L + ROWS - 1) / ROWS;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t l = tile * ROWS + r;
    const int64_t ll = l < L ? l : 0;  // line ll = (ll % L1, ll / L1)
    const double* p = P + (ll % L1) * sl + (ll / L1) * sl2;
    const double amax = l < L ? slice_amax<ROWS, VEC>(p, sk, K, h, 0, KB) : 0.0;
    if (h == 1) part[r] = amax;
    __syncthreads();
    if (h == 0) part[r] = fmax(amax, part[r]);
    __syncthreads();
    const double sc = ldexp(1.0, line_exponent(part[r]));
    __syncthreads();  // part[] is rewritten by the next tile
    if (h == 0 && l < L) scale[l] = sc;
    slice_digits<ROWS, VEC>(p, sk, K, h, r, l < L, 0x1p54 / sc, tile, KB, 0, KB, out, halves);
  }
}

// Long-line form of k_slice_tile: the work unit is LU lines of one tile (not all ROWS), with
// 256 / LU threads per line splitting its half-blocks (16 k) p, p + PARTS, ...; the line
// maxima meet in shared memory.  Persistent over units on 2 x 148 CTAs, so the lines in flight
// (2 x 148 x LU x K doubles; the caller picks LU to keep them within ~90 MB) stay L2-resident
// between the max pass and the digit pass: the FP64 operand is read from HBM once, where
// k_slice_tile's 2 x 148 whole tiles of long lines overflow L2 and read it twice.
// Digits are bit-identical to k_slice_tile's.
template <int ROWS, int LU, bool VEC>
__global__ void __launch_bounds__(256)
k_slice_lines(const double* __restrict__ P, int64_t sl, int64_t sk, int64_t L, int64_t K,
              int64_t KB, double* __restrict__ scale, int8_t* __restrict__ out, int64_t L1,
              int64_t sl2, int halves) {
  constexpr int PARTS = 256 / LU, UPT = ROWS / LU;  // units per tile
  __shared__ double part[PARTS][LU];
  const int u = threadIdx.x % LU, p = threadIdx.x / LU;
  const int64_t units = (L + ROWS - 1) / ROWS * UPT, HB = 2 * KB;
  for (int64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const int64_t tile = unit / UPT;
    const int r = int(unit % UPT) * LU + u;  // line within the tile
    const int64_t l = tile * ROWS + r;
    const int64_t ll = l < L ? l : 0;
    const double* pl = P + (ll % L1) * sl + (ll / L1) * sl2;
    double amax = 0.0;
    if (l < L)
      for (int64_t hb = p; hb < HB; hb += PARTS) {
        double x[16];
        load16<ROWS, VEC>(pl, sk, (hb / 2) * BKB + 16 * (hb % 2), K, x);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) amax = fmax(amax, fabs(x[kk]));
      }
    part[p][u] = amax;
    __syncthreads();
    double m = 0.0;
#pragma unroll
    for (int q = 0; q < PARTS; ++q) m = fmax(m, part[q][u]);
    const double sc = ldexp(1.0, line_exponent(m));
    __syncthreads();  // part[] is rewritten by the next unit
    if (p == 0 && l < L) scale[l] = sc;
    const double inv54 = 0x1p54 / sc;
    for (int64_t hb = p; hb < HB; hb += PARTS)
      slice_digits<ROWS, VEC>(pl, sk, K, int(hb % 2), r, l < L, inv54, tile, KB, hb / 2,
                              hb / 2 + 1, out, halves);
  }
}

// Few line tiles with a long K (the projected-CP evaluation's D0 and Y: 16-65 tiles of
// K = 8283 at cfg5): the persistent kernel would run on 16-65 SMs.  Split K over grid.y
// instead: pass 1 writes per-split line maxima, pass 2 (every split) takes their maximum —
// exact, so the digits are bit-identical to k_slice_tile's — and writes its k-blocks.
template <int ROWS, bool VEC>
__global__ void __launch_bounds__(2 * ROWS)
k_slice_pmax(const double* __restrict__ P, int64_t sl, int64_t sk, int64_t L, int64_t K,
             int64_t KB, int64_t L1, int64_t sl2, int64_t kbs, double* __restrict__ pmax) {
  __shared__ double part[ROWS];
  const int r = threadIdx.x % ROWS, h = threadIdx.x / ROWS;
  const int64_t l = blockIdx.x * int64_t(ROWS) + r, ll = l < L ? l : 0;
  const double* p = P + (ll % L1) * sl + (ll / L1) * sl2;
  const int64_t kb0 = blockIdx.y * kbs, kb1 = kb0 + kbs < KB ? kb0 + kbs : KB;
  const double amax = l < L ? slice_amax<ROWS, VEC>(p, sk, K, h, kb0, kb1) : 0.0;
  if (h == 1) part[r] = amax;
  __syncthreads();
  if (h == 0 && l < L) pmax[blockIdx.y * L + l] = fmax(amax, part[r]);
}

template <int ROWS, bool VEC>
__global__ void __launch_bounds__(2 * ROWS)
k_slice_split(const double* __restrict__ P, int64_t sl, int64_t sk, int64_t L, int64_t K,
              int64_t KB, int64_t L1, int64_t sl2, int64_t kbs, const double* __restrict__ pmax,
              double* __restrict__ scale, int8_t* __restrict__ out, int halves) {
  const int r = threadIdx.x % ROWS, h = threadIdx.x / ROWS;
  const int64_t tile = blockIdx.x, l = tile * ROWS + r, ll = l < L ? l : 0;
  const double* p = P + (ll % L1) * sl + (ll / L1) * sl2;
  double amax = 0.0;
  if (l < L)
    for (unsigned q = 0; q < gridDim.y; ++q) amax = fmax(amax, pmax[q * L + l]);
  const double sc = ldexp(1.0, line_exponent(amax));
  if (blockIdx.y == 0 && h == 0 && l < L) scale[l] = sc;
  const int64_t kb0 = blockIdx.y * kbs, kb1 = kb0 + kbs < KB ? kb0 + kbs : KB;
  slice_digits<ROWS, VEC>(p, sk, K, h, r, l < L, 0x1p54 / sc, tile, KB, kb0, kb1, out, halves);
}

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  // SmemDescriptor (cute/arch/mma_sm100_desc.hpp): start [0,14), LBO [16,30), SBO [32,46),
  // version 1 at [46,48), base offset 0, lbo mode 0, layout SWIZZLE_NONE (0) at [61,64)
  const uint64_t addr = (smem_u32(p) >> 4) & 0x3FFF;
  return addr | (uint64_t((lbo >> 4) & 0x3FFF) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
         (uint64_t(1) << 46);
}
// InstrDescriptor: c_format S32 (2) [4,6), a/b format s8 (1) [7,10) [10,13),
// K-major A and B, N>>3 at [17,23), M>>4 at [24,29)
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                            (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, int* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}



// Persistent, warp-specialised GEMM over the M x N output tiles; output column n lives at
// C + (n / nb) bs + (n % nb) ldc, so a batch of slabs sharing A is one launch.  Tile t:
// mt = t % tiles_m, nt = t / tiles_m (M tiles fastest: the CTAs sharing a B column tile run
// together, B streams from HBM once and the small A operand stays in L2).
//   warp 0 lane 0: producer, bulk copies of the (A, B) slices of each (pass, k-block);
//   warp 1 lane 0: MMA issuer, per k-block 10 (pass 1) or 18 (pass 2) tcgen05.mma;
//   warps 2-9    : epilogue; warp w owns TMEM lane quadrant w % 4 (tile rows) and column
//                  half (w - 2) / 4.  After pass 1 it folds D_0..D_3 into the exact integer
//                  hi = sum D_g 2^{8(3-g)} (a double: < 2^53 for K <= 1024), releases TMEM
//                  for pass 2, then folds lo = sum_{g>=4} D_g 2^{8(6-g)} likewise and
//                  writes (hi 2^-36 + lo 2^-60) 2^e_i 2^f_n (one rounding) while the next
//                  tile's MMAs run.
// Output addressing: tile row i (0 <= i < M) and column n land at
//   C + (i % mr) + (i / mr) rs + (n / nb) bs + (n % nb) ldc,
// i.e. a plain column-major C (mr = M, nb = N) or batches of row / column blocks (the
// evaluators' slabs, the batched Q = core x2 U1); C = alpha A op(B) + beta C.
struct OzOut {
  double* C;
  int64_t ldc, nb, bs, mr, rs;
  double beta;
  double alpha;  // C = alpha A op(B) + beta C
};

constexpr int EPI_WARPS = 8;
constexpr int PTHREADS = 32 * (2 + EPI_WARPS);
constexpr int EPI_COLS = BN / 2;  // columns per epilogue thread
constexpr size_t SMEM_BYTES = size_t(STAGES) * (A_STAGE + B_STAGE) + 128;
#ifdef LATSUM_OZ_TRACE
// summed over CTAs: MMA-thread cycles in the tile loop, cycles waiting for the epilogue
__device__ unsigned long long g_oz_trace[2];
#endif

// fold the NG groups of the 4-column chunk at TMEM column c into x (Horner, base 256, in
// int64: |D_g| < 2^31 so the fold stays below 2^55; converting once per element instead of
// once per group keeps the drain off the int->FP64 conversion pipe)
template <int NG, int W>
__device__ __forceinline__ void drainw(uint32_t taddr, double* x) {
  int v[NG][W];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    if (W == 16) tmem_ld16(taddr + uint32_t(g * BN), v[g]);
    else if (W == 8) tmem_ld8(taddr + uint32_t(g * BN), v[g]);
    else tmem_ld4(taddr + uint32_t(g * BN), v[g]);
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < W; ++j) {  // exact int64 Horner fold, one conversion per element
    long long h = v[0][j];
#pragma unroll
    for (int g = 1; g < NG; ++g) h = h * 256 + v[g][j];
    x[j] = __ll2double_rn(h);
  }
}

__global__ void __launch_bounds__(PTHREADS, 1)
k_gemm_i8(const int8_t* __restrict__ As, const double* __restrict__ ra,
          const int8_t* __restrict__ Bs, const double* __restrict__ cb, int64_t M, int64_t N,
          int64_t KB, OzOut o, int64_t tiles_m, int64_t tiles, int64_t tiles_n, int nfast) {
  // tile t -> (mt, nt): M tiles fastest (default: the CTAs running together share a B column
  // tile) or, nfast, N tiles fastest (a tall A streamed once, B kept in L2)
  auto tile_m = [&](int64_t t) { return nfast ? t / tiles_n : t % tiles_m; };
  auto tile_n = [&](int64_t t) { return nfast ? t % tiles_n : t / tiles_m; };
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, EPI_WARPS);  // one arrival per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int64_t it = 0;  // (pass, k-block) stages loaded by this CTA (ring position)
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int8_t* gA = As + (tile_m(t) * KB) * int64_t(A_STAGE);
        const int8_t* gB = Bs + (tile_n(t) * KB) * int64_t(B_STAGE);
        for (int pass = 0; pass < 2; ++pass) {
          const uint32_t nsl = pass == 0 ? P1_SLICES : S;
          for (int64_t kb = 0; kb < KB; ++kb, ++it) {
            const int st = int(it % STAGES);
            if (it >= STAGES) mbar_wait(&empty[st], uint32_t(((it / STAGES) - 1) & 1));
            mbar_expect_tx(&full[st], nsl * (A_BLK + B_BLK));
            bulk_g2s(sA + st * A_STAGE, gA + kb * A_STAGE, nsl * A_BLK, &full[st]);
            bulk_g2s(sB + st * B_STAGE, gB + kb * B_STAGE, nsl * B_BLK, &full[st]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int64_t it = 0, np = 0;  // np: passes issued (TMEM phase)
#ifdef LATSUM_OZ_TRACE
      long long w_tm = 0, t_begin = clock64();
#endif
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int pass = 0; pass < 2; ++pass, ++np) {
#ifdef LATSUM_OZ_TRACE
          const long long c0 = clock64();
#endif
          if (np > 0) mbar_wait(tmem_empty, uint32_t((np - 1) & 1));  // previous pass drained
#ifdef LATSUM_OZ_TRACE
          w_tm += clock64() - c0;
#endif
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          for (int64_t kb = 0; kb < KB; ++kb, ++it) {
            const int st = int(it % STAGES);
            mbar_wait(&full[st], uint32_t((it / STAGES) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint8_t* a0 = sA + st * A_STAGE;
            const uint8_t* b0 = sB + st * B_STAGE;
            const uint32_t acc0 = kb > 0 ? 1u : 0u;
            if (pass == 0) {
#pragma unroll
              for (int s = 0; s < P1_SLICES; ++s)
#pragma unroll
                for (int u = 0; u < P1_SLICES - s; ++u)  // g = s + u <= 3
                  mma_i8(tmem + uint32_t((s + u) * BN),
                         smem_desc(a0 + s * A_BLK, 128, (BKB / 16) * 128),
                         smem_desc(b0 + u * B_BLK, 128, (BKB / 16) * 128), s > 0 ? 1u : acc0);
            } else {
#pragma unroll
              for (int s = 0; s < S; ++s)
#pragma unroll
                for (int u = (s < 4 ? 4 - s : 0); u < S - s; ++u)  // 4 <= g <= 6
                  mma_i8(tmem + uint32_t((s + u - 4) * BN),
                         smem_desc(a0 + s * A_BLK, 128, (BKB / 16) * 128),
                         smem_desc(b0 + u * B_BLK, 128, (BKB / 16) * 128), s > 0 ? 1u : acc0);
            }
            mma_commit(&empty[st]);  // frees the stage when these MMAs retire
          }
          mma_commit(tmem_full);
        }
      }
#ifdef LATSUM_OZ_TRACE
      atomicAdd(&g_oz_trace[0], (unsigned long long)(clock64() - t_begin));
      atomicAdd(&g_oz_trace[1], (unsigned long long)w_tm);
#endif
    }
  } else {
    const int q = warp % 4, half = (warp - 2) / 4;
    const uint32_t tq = tmem + (uint32_t(q * 32) << 16) + uint32_t(half * EPI_COLS);
    int64_t np = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, np += 2) {
      const int64_t mt = tile_m(t), nt = tile_n(t);
      const int64_t i = mt * BM + q * 32 + lane;
      const int64_t n0 = nt * BN + half * EPI_COLS;
      // row / column scales, fetched before the accumulators are ready
      const double ri = i < M ? o.alpha * ra[i] : 0.0;
      const double c0s = n0 + lane < N ? cb[n0 + lane] : 0.0;
      const double c1s = n0 + 32 + lane < N ? cb[n0 + 32 + lane] : 0.0;
      double hv[EPI_COLS];
      mbar_wait(tmem_full, uint32_t(np & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int c = 0; c < EPI_COLS; c += 16) drainw<4, 16>(tq + uint32_t(c), hv + c);
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tmem_empty))
                     : "memory");
      mbar_wait(tmem_full, uint32_t((np + 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int c = 0; c < EPI_COLS; c += 4) {
        double lv[4];
        drainw<3, 4>(tq + uint32_t(c), lv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double cs = __shfl_sync(0xffffffffu, c + j < 32 ? c0s : c1s, (c + j) % 32);
          hv[c + j] = (hv[c + j] * 0x1p-36 + lv[j] * 0x1p-60) * ri * cs;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tmem_empty))
                     : "memory");
      if (i < M) {
        int64_t kk = n0 / o.nb, jj = n0 - kk * o.nb;
        double* ci = o.C + (i % o.mr) + (i / o.mr) * o.rs;
        if (o.beta == 0.0) {
#pragma unroll
          for (int j = 0; j < EPI_COLS; ++j) {
            if (n0 + j < N) ci[kk * o.bs + jj * o.ldc] = hv[j];
            if (++jj == o.nb) {
              jj = 0;
              ++kk;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < EPI_COLS; ++j) {
            if (n0 + j < N) {
              double* cp = ci + kk * o.bs + jj * o.ldc;
              *cp = hv[j] + o.beta * *cp;
            }
            if (++jj == o.nb) {
              jj = 0;
              ++kk;
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

}  // namespace oz
}  // namespace latsum_b200
