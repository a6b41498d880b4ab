// Microbenchmark (experiment, not product): tcgen05.mma issue rate for K-major A/B in
// shared memory, layouts no-swizzle / SW128, N in {32..256}, kind::f16 and kind::f8f6f4.
// One CTA per SM, one thread issues `iters` MMAs on a fixed smem tile; timed by clock64.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2305_14566_b200/csrc/ptx.cuh"
using namespace osg;

__global__ void __launch_bounds__(128, 1) bench(int layout, int N, int f8, int acc, int iters, long long* out, int nd) {
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
    uint64_t da, db;
    if (layout == 0) {  // no swizzle: core matrices 8x16B, LBO = 2048 (K), SBO = 128 (M/N)
      da = ptx::smem_desc_noswz(sa, 16384 / 8, 128);
      db = ptx::smem_desc_noswz(sb, 16384 / 8, 128);
    } else {            // SW128 K-major: 8 rows x 128 B atoms
      da = ptx::smem_desc(sa, 1024, 2u);
      db = ptx::smem_desc(sb, 1024, 2u);
    }
    const uint32_t id = f8 ? ptx::idesc_f8(128, N) : ptx::idesc_f16(128, N, false);
    // warm
    for (int i = 0; i < 16; ++i) {
      if (f8) ptx::mma_f8(tbase, da, db, id, acc); else ptx::mma_f16(tbase, da, db, id, acc);
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t dt = tbase + (uint32_t)((i % nd) * N);
      if (f8) ptx::mma_f8(dt, da, db, id, acc); else ptx::mma_f16(dt, da, db, id, acc);
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

int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 4096;
  printf("layout N acc nd : cycles/MMA (f16)\n");
  for (int layout = 0; layout < 2; ++layout)
    for (int acc = 1; acc >= 0; --acc)
      for (int nd : {1, 2, 4})
        for (int N : {16, 32, 64, 96, 128, 256}) {
          if (nd * N > 512) continue;
          bench<<<148, 128, 64 * 1024>>>(layout, N, 0, acc, iters, d, nd);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
          long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
          printf("%s N=%3d acc=%d nd=%d : %.1f\n", layout ? "SW128" : "noswz", N, acc, nd, (double)c / iters);
        }
  return 0;
}
