// Microbenchmark (experiment): MMA issue patterns for the dy-fused no-swizzle conv loop.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2305_14566_b200/csrc/ptx.cuh"
using namespace osg;

__device__ __forceinline__ void mma_f16_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc)
      : "memory");
}

constexpr int R = 8, BN = 32, PX = 130;
constexpr int kChunkStride = (R + 2) * PX * 16;

// MODE 0: lane 0 only (current).  MODE 1: whole warp, elect inside asm.
template <int MODE>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tslot;
  const bool go = MODE == 0 ? threadIdx.x == 0 : warp == 0;
  if (go) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t sa = ptx::smem_u32(smem) + (it & 1) * 0;  // stage base
      const uint32_t d_base = tbase + (it & 1) * R * BN;
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const uint32_t sbd = sa + 2 * kChunkStride + dx * 3 * BN * 32;
#pragma unroll
        for (int i = -1; i <= R; ++i) {
          const int r_hi = i + 1 < R - 1 ? i + 1 : R - 1;
          const int r_lo = i - 1 > 0 ? i - 1 : 0;
          const int nrows = r_hi - r_lo + 1;
          const int dy0 = i - r_hi + 1;
          const uint32_t a0 = sa + (uint32_t)(((i + 1) * PX + dx) * 16);
          const uint64_t da = ptx::smem_desc_noswz(a0, kChunkStride, 128);
          const uint64_t db = ptx::smem_desc(sbd + dy0 * BN * 32, 8 * 32, 6u);
          const uint32_t id = nrows == 3 ? ptx::idesc_f16(128, 3 * BN, false)
                            : nrows == 2 ? ptx::idesc_f16(128, 2 * BN, false) : ptx::idesc_f16(128, BN, false);
          if (MODE == 0) ptx::mma_f16(d_base + (R - 1 - r_hi) * BN, da, db, id, 1u);
          else mma_f16_elect(d_base + (R - 1 - r_hi) * BN, da, db, id);
        }
      }
    }
    if (MODE == 0 || (threadIdx.x & 31) == 0) {
      ptx::mma_commit(&bar);
      ptx::mbar_wait(&bar, 0);
    }
    __syncwarp(MODE == 0 ? 1u : 0xffffffffu);
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tbase); }
}

template <int M>
void run(long long* d) {
  cudaFuncSetAttribute(bench<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int iters = 200;
  bench<M><<<148, 128, 96 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  // per (dx, i) group: 30 MMAs; model floor: sum over i of max(N/2, 32 + N/4) = 3 * (2*40 + 2*48 + 6*56) = 1536
  printf("mode %d: %.1f cycles per 30-MMA chunk (model floor 1536), %.1f per MMA\n", M, (double)c / iters,
         (double)c / iters / 30);
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  run<0>(d); run<1>(d); run<0>(d); run<1>(d);
  return 0;
}
