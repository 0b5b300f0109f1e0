// tcgen05.mma.kind::i8 issue-rate microbenchmark (dev tool): one CTA per SM issues a long
// stream of M=128 x N x K=32 MMAs from shared memory into TMEM; reports dense int8 TOPS for
// N = 64, 128, 256 (operand smem read pressure falls as N grows).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_mma_peak tools/i8_mma_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(const void* p, uint32_t lbo, uint32_t sbo) {
  return ((smem_u32(p) >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}

template <int N>
__global__ void k_peak(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 128 * 32 * 8 + N * 32 * 8; i += blockDim.x) smem[i] = uint8_t(i * 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (8u << 24);
  if (threadIdx.x == 0) {
    const uint8_t* A = smem;
    const uint8_t* B = smem + 128 * 32 * 8;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint64_t da = desc(A + s * 128 * 32, 128, 256);
        const uint64_t db = desc(B + s * N * 32, 128, 256);
        const uint32_t d = tmem + uint32_t((s % (512 / N)) * N);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                     "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0, 10000000;\n\t"
      "@P1 bra D;\n\tbra W;\n\tD:\n\t}\n" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x == 0) atomicAdd(sink, 1);
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// the Ozaki GEMM's issue pattern: per k-block 36 MMAs (s + u <= 7) into 8 groups of 64
// columns, stage ring of 4 x (8 A slices + 8 B slices)
__global__ void k_pattern(int iters, int* sink, long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int AS = 8 * 128 * 32, BS = 8 * 64 * 32;
  for (int i = threadIdx.x; i < 4 * (AS + BS); i += blockDim.x) smem[i] = uint8_t(i * 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(64 >> 3) << 17) | (8u << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const uint8_t* A = smem + (it % 4) * AS;
      const uint8_t* B = smem + 4 * AS + (it % 4) * BS;
#pragma unroll
      for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (s + u > 7) continue;
          const uint64_t da = desc(A + s * 128 * 32, 128, 256);
          const uint64_t db = desc(B + u * 64 * 32, 128, 256);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + uint32_t((s + u) * 64)),
                       "l"(da), "l"(db), "r"(idesc), "r"((it > 0 || s > 0) ? 1 : 0));
        }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0, 10000000;\n\t"
      "@P1 bra D;\n\tbra W;\n\tD:\n\t}\n" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x == 0) { atomicAdd(sink, 1); if (blockIdx.x == 0) *clk = clock64() - t0; }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

void run_pattern(int* sink, long long* clk) {
  const int smem = 4 * (8 * 128 * 32 + 8 * 64 * 32);
  cudaFuncSetAttribute(k_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int iters : {100, 2000, 20000}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k_pattern<<<148, 128, smem>>>(iters, sink, clk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    const double ops = 2.0 * 148 * double(iters) * 36 * 128.0 * 64 * 32;
    printf("ozaki pattern iters=%d: %.1f dense TOPS (%.3f ms, %.0f MHz effective) err=%s\n", iters,
           ops / ms / 1e9, ms, c / (ms * 1e3), cudaGetErrorString(cudaGetLastError()));
  }
}

template <int N>
void run(int* sink) {
  const int smem = 128 * 32 * 8 + N * 32 * 8;
  cudaFuncSetAttribute(k_peak<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
  k_peak<N><<<148, 128, smem>>>(100, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_peak<N><<<148, 128, smem>>>(iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double ops = 2.0 * 148 * iters * 8 * 128.0 * N * 32;
  printf("kind::i8 M=128 N=%3d K=32: %.1f dense TOPS (%.3f ms) err=%s\n", N, ops / ms / 1e9, ms,
         cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  int* sink;
  cudaMalloc(&sink, 4);
  long long* clk;
  cudaMalloc(&clk, 8);
  run_pattern(sink, clk);
  run<64>(sink);
  run<128>(sink);
  run<256>(sink);
  return 0;
}
