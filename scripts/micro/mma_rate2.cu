// Microbenchmark (experiment): per-instruction cost of tcgen05.mma, M=128, unrolled issue.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2305_14566_b200/csrc/ptx.cuh"
using namespace osg;

template <int N, int ND, int UNROLL>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    const uint32_t sa = ptx::smem_u32(smem), sb = sa + 32768;
    const uint64_t da = ptx::smem_desc(sa, 1024, 2u), db = ptx::smem_desc(sb, 1024, 2u);
    constexpr uint32_t id = ptx::idesc_f16(128, N, false);
    for (int i = 0; i < 16; ++i) ptx::mma_f16(tbase, da, db, id, 1);
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += UNROLL) {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) ptx::mma_f16(tbase + (u % ND) * N, da + 2 * u, db, id, 1);
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 1);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tbase); }
}

template <int N, int ND, int U>
void run(long long* d) {
  cudaFuncSetAttribute(bench<N, ND, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 4096;
  bench<N, ND, U><<<148, 128, 64 * 1024>>>(iters, d);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d nd=%d unroll=%2d : %.1f cycles/MMA (floor N/2 = %d)\n", N, ND, U, (double)c / iters, N / 2);
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  run<32, 1, 1>(d); run<32, 1, 4>(d); run<32, 1, 16>(d); run<32, 4, 16>(d);
  run<64, 1, 16>(d); run<64, 4, 16>(d);
  run<96, 1, 16>(d); run<96, 4, 16>(d);
  run<128, 1, 16>(d); run<128, 4, 16>(d);
  run<256, 1, 1>(d); run<256, 1, 16>(d); run<256, 2, 16>(d);
  return 0;
}
