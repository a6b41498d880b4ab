// Microbenchmark (experiment): TMA load throughput of the no-swizzle conv A box
// {8 el, 130 px, 10 rows, 2 chunks} from (a) NHWC with 96-B pixels (f8, C=32) and
// (b) a row-blocked layout [B][H][chunk][W][16 B]. 148 CTAs, 4-stage ring, 1 thread.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2305_14566_b200/csrc/ptx.cuh"
using namespace osg;

__global__ void __launch_bounds__(32, 1) load_bench(const __grid_constant__ CUtensorMap tm, int blocked, int H,
                                                     int W, int items, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[4];
  constexpr int kBox = 2 * 10 * 130 * 16;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  const int per_img = (H / 8) * (W / 128);
  for (int it = 0; it < items * 3; ++it) {
    const int s = it & 3;
    if (it >= 4) ptx::mbar_wait(&full[s], ((it >> 2) - 1) & 1);
    const int item = blockIdx.x + (it / 3) * gridDim.x;
    const int b = item / per_img, rem = item % per_img;
    const int y0 = (rem / (W / 128)) * 8 - 1, x0 = (rem % (W / 128)) * 128 - 1;
    const int kc = it % 3;
    ptx::mbar_arrive_expect_tx(&full[s], blocked == 2 ? 46080 : kBox);
    if (blocked == 2)  // dims {64, W/8, chunks, H, B}, 18 units of 8 px
      ptx::tma_load_5d(smem + s * 46080, &tm, &full[s], 0, (x0 - 7) / 8 - (x0 < 7 ? 1 : 0), 2 * kc, y0, b);
    else if (blocked)  // dims {8, W, chunks, H, B}
      ptx::tma_load_5d(smem + s * kBox, &tm, &full[s], 0, x0, 2 * kc, y0, b);
    else          // dims {8, W, H, chunks, B}
      ptx::tma_load_5d(smem + s * kBox, &tm, &full[s], 0, x0, y0, 2 * kc, b);
  }
  for (int it = items * 3 - 4; it < items * 3; ++it) ptx::mbar_wait(&full[it & 3], (it >> 2) & 1);
  if (blockIdx.x == 0) out[0] = clock64() - t0;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  const int B = 16, H = 512, W = 512, NCH = 6;  // 96-B pixels
  const size_t bytes = (size_t)B * H * W * NCH * 16;
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(load_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 46080 + 1024);
  const int items_total = B * (H / 8) * (W / 128);
  const int items = items_total / 148;
  for (int blocked = 0; blocked < 3; ++blocked) {
    CUtensorMap tm;
    cuuint64_t dims[5], strides[4];
    if (blocked == 2) {
      cuuint64_t d5[5] = {64, (cuuint64_t)W / 8, 4, (cuuint64_t)H, (cuuint64_t)B};
      cuuint64_t s4[4] = {128, (cuuint64_t)W * 16, (cuuint64_t)W * 96, (cuuint64_t)H * W * 96};
      for (int i = 0; i < 5; ++i) dims[i] = d5[i];
      for (int i = 0; i < 4; ++i) strides[i] = s4[i];
    } else if (!blocked) {
      cuuint64_t d5[5] = {8, (cuuint64_t)W, (cuuint64_t)H, 4, (cuuint64_t)B};
      cuuint64_t s4[4] = {96, (cuuint64_t)W * 96, 16, (cuuint64_t)H * W * 96};
      for (int i = 0; i < 5; ++i) dims[i] = d5[i];
      for (int i = 0; i < 4; ++i) strides[i] = s4[i];
    } else {
      cuuint64_t d5[5] = {8, (cuuint64_t)W, 4, (cuuint64_t)H, (cuuint64_t)B};
      cuuint64_t s4[4] = {16, (cuuint64_t)W * 16, (cuuint64_t)W * 96, (cuuint64_t)H * W * 96};
      for (int i = 0; i < 5; ++i) dims[i] = d5[i];
      for (int i = 0; i < 4; ++i) strides[i] = s4[i];
    }
    cuuint32_t box[5] = {8, 130, blocked ? 2u : 10u, blocked ? 10u : 2u, 1};
    if (blocked == 2) { box[0] = 64; box[1] = 18; box[2] = 2; box[3] = 10; }
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode %d\n", r); return 1; }
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      load_bench<<<148, 32, 4 * 46080 + 1024>>>(tm, blocked, H, W, items, d);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double moved = 148.0 * items * 3 * (blocked == 2 ? 46080 : 41600);
      printf("%s: %.3f ms, %.0f GB/s smem-fill (%.2f GB of boxes)\n", blocked == 2 ? "blocked128" : blocked ? "blocked" : "NHWC96", ms,
             moved / ms / 1e6, moved / 1e9);
    }
  }
  return 0;
}
