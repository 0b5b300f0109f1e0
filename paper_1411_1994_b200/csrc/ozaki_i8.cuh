// FP64-accurate GEMM on the INT8 tensor cores of sm_100a (Ozaki scheme I).
//
// C = A B (FP64) with A (M x K) and B (K x N).  Every row of A and column of B is scaled
// by a power of two into (-1, 1) and split into S = 8 signed 7-bit digits (slices):
//   A = diag(2^e) sum_s 2^{-7s} A_s,   B = sum_t 2^{-7t} B_t diag(2^f),
// so C = diag(2^e) [ sum_g 2^{-7g} D_g ] diag(2^f) with D_g = sum_{s+t=g} A_s B_t.
// Each A_s B_t is exact in int32 (|.| <= 127^2 K), the pairs with s+t > S+1 are below
// 2^{-7(S+2)} and dropped, and the S group sums D_2 .. D_{S+1} accumulate in TMEM as int32
// (|D_g| <= 8 * 127^2 * K < 2^31 for K <= 16k).  The FP64 epilogue combines them exactly
// up to one rounding per term, so the result has FP64-GEMM accuracy: the representation
// error is 2^{-56} of the row/column maxima.  36 int8 products replace one FP64 product;
// at the int8 tensor rate that is ~3.4x the DMMA rate.
//
// Data path: operands are pre-sliced into the canonical K-major "no swizzle" core-matrix
// layout (8 rows x 16 bytes) per (tile, k-block, slice), so each pipeline stage is one
// contiguous bulk copy (cp.async.bulk, TMA engine) completing on an mbarrier; one thread
// issues tcgen05.mma.kind::i8 (M=128, N=64, K=32) into 8 TMEM accumulators (512 columns);
// tcgen05.commit frees a stage; four warps read TMEM with tcgen05.ld for the epilogue.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace latsum_b200 {
namespace oz {

constexpr int S = 8;                 // slices per operand
constexpr int BM = 128, BN = 64;     // output tile (TMEM lanes x accumulator columns)
constexpr int BKB = 32;              // k-block (int8 elements = bytes) per stage
constexpr int STAGES = 4;
constexpr int A_BLK = BM * BKB;      // one slice's A block (bytes)
constexpr int B_BLK = BN * BKB;
constexpr int A_STAGE = S * A_BLK;   // 32 KB
constexpr int B_STAGE = S * B_BLK;   // 16 KB
constexpr int THREADS = 128;
constexpr int TMEM_COLS = S * BN;    // 512
constexpr size_t SMEM_BYTES = size_t(STAGES) * (A_STAGE + B_STAGE) + 1024;

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

// digits of x in (-1, 1): x = sum_s d_s 2^{-7s} + r, |r| < 2^{-7S}, d_s in [-127, 127]
__device__ __forceinline__ void digits(double x, int8_t* d) {
#pragma unroll
  for (int s = 0; s < S; ++s) {
    x *= 128.0;
    const double t = trunc(x);
    d[s] = int8_t(t);
    x -= t;
  }
}

// A (M x K, column-major, lda) -> slices [mtile][kblk][s][A_BLK], exponents e[M].
// One warp per row (rows are strided by lda; M*K is small for the evaluation).
__global__ void k_slice_rows(const double* __restrict__ A, int64_t lda, int64_t M, int64_t K,
                             int64_t KB, int8_t* __restrict__ out, int* __restrict__ ex) {
  const int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (i >= M) return;
  double amax = 0.0;
  for (int64_t k = lane; k < K; k += 32) amax = fmax(amax, fabs(A[i + k * lda]));
  for (int off = 16; off > 0; off >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  const int e = line_exponent(amax);
  if (lane == 0) ex[i] = e;
  const int64_t mt = i / BM;
  const int r = int(i % BM);
  for (int64_t k = lane; k < KB * BKB; k += 32) {
    int8_t d[S];
    const double x = k < K ? ldexp(A[i + k * lda], -e) : 0.0;
    digits(x, d);
    const int64_t kb = k / BKB;
    int8_t* base = out + ((mt * KB + kb) * S) * int64_t(A_BLK);
#pragma unroll
    for (int s = 0; s < S; ++s) base[s * A_BLK + blk_off(r, int(k % BKB))] = d[s];
  }
}

// B (K x N, column-major, ldb: columns contiguous in k) -> slices [ntile][kblk][s][B_BLK],
// exponents f[N].  One warp per column.
__global__ void k_slice_cols(const double* __restrict__ B, int64_t ldb, int64_t N, int64_t K,
                             int64_t KB, int8_t* __restrict__ out, int* __restrict__ ex) {
  const int64_t n = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (n >= N) return;
  const double* col = B + n * ldb;
  double amax = 0.0;
  for (int64_t k = lane; k < K; k += 32) amax = fmax(amax, fabs(col[k]));
  for (int off = 16; off > 0; off >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  const int f = line_exponent(amax);
  if (lane == 0) ex[n] = f;
  const int64_t nt = n / BN;
  const int r = int(n % BN);
  for (int64_t k = lane; k < KB * BKB; k += 32) {
    int8_t d[S];
    const double x = k < K ? ldexp(col[k], -f) : 0.0;
    digits(x, d);
    const int64_t kb = k / BKB;
    int8_t* base = out + ((nt * KB + kb) * S) * int64_t(B_BLK);
#pragma unroll
    for (int s = 0; s < S; ++s) base[s * B_BLK + blk_off(r, int(k % BKB))] = d[s];
  }
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
// InstrDescriptor: c_format S32 (2) [4,6), a/b format signed int8 (1) [7,10) [10,13),
// K-major A and B, N>>3 at [17,23), M>>4 at [24,29)
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                            (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
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
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// C[i + ldc n] = sum over the tile's int8 slice products (see header), for the tile
// (blockIdx.y, blockIdx.x) of an M x N output; KB k-blocks.
__global__ void __launch_bounds__(THREADS, 1)
k_gemm_i8(const int8_t* __restrict__ As, const int* __restrict__ ea, const int8_t* __restrict__ Bs,
          const int* __restrict__ eb, int64_t M, int64_t N, int64_t KB, double* __restrict__ C,
          int64_t ldc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int64_t nt = blockIdx.x, mt = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int8_t* gA = As + (mt * KB) * int64_t(A_STAGE);
  const int8_t* gB = Bs + (nt * KB) * int64_t(B_STAGE);
  if (threadIdx.x == 0) {
    // prologue: fill the ring
    for (int64_t kb = 0; kb < KB && kb < STAGES; ++kb) {
      mbar_expect_tx(&full[kb], A_STAGE + B_STAGE);
      bulk_g2s(sA + kb * A_STAGE, gA + kb * A_STAGE, A_STAGE, &full[kb]);
      bulk_g2s(sB + kb * B_STAGE, gB + kb * B_STAGE, B_STAGE, &full[kb]);
    }
    for (int64_t kb = 0; kb < KB; ++kb) {
      const int st = int(kb % STAGES);
      const uint32_t ph = uint32_t((kb / STAGES) & 1);
      mbar_wait(&full[st], ph);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint8_t* a0 = sA + st * A_STAGE;
      const uint8_t* b0 = sB + st * B_STAGE;
#pragma unroll
      for (int s = 0; s < S; ++s) {
#pragma unroll
        for (int t = 0; t < S; ++t) {
          if (s + t > S - 1) continue;  // keep groups g = s + t + 2 <= S + 1
          const int g = s + t;
          const uint64_t da = smem_desc(a0 + s * A_BLK, 128, (BKB / 16) * 128);
          const uint64_t db = smem_desc(b0 + t * B_BLK, 128, (BKB / 16) * 128);
          // the first product into group g at kb = 0 overwrites the accumulator
          const uint32_t acc = (kb > 0 || s > 0) ? 1u : 0u;
          mma_i8(tmem + uint32_t(g * BN), da, db, acc);
        }
      }
      mma_commit(&empty[st]);
      const int64_t nk = kb + STAGES;
      if (nk < KB) {  // refill this stage once its MMAs have drained it
        mbar_wait(&empty[st], ph);
        mbar_expect_tx(&full[st], A_STAGE + B_STAGE);
        bulk_g2s(sA + st * A_STAGE, gA + nk * A_STAGE, A_STAGE, &full[st]);
        bulk_g2s(sB + st * B_STAGE, gB + nk * B_STAGE, B_STAGE, &full[st]);
      }
    }
    mma_commit(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

  // epilogue: warp w owns TMEM lanes (tile rows) 32w .. 32w+31
  const int64_t i = mt * BM + warp * 32 + lane;
  const double si = i < M ? 1.0 : 0.0;
  const int ei = i < M ? ea[i] : 0;
  for (int c0 = 0; c0 < BN; c0 += 16) {
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll
    for (int g = 0; g < S; ++g) {
      uint32_t v[16];
      tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(g * BN + c0), v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      const double scale = ldexp(1.0, -7 * (g + 2));
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] += double(int32_t(v[j])) * scale;
    }
    if (i < M) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t n = nt * BN + c0 + j;
        if (n < N) C[i + ldc * n] = si * ldexp(acc[j], ei + eb[n]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TMEM_COLS));
}

}  // namespace oz
}  // namespace latsum_b200
