// Micro-test: 2-D TMA load of a u32 image box {132, 6} at negative / positive coordinates
// (the stem's input ring), checked against a host copy.  nvcc -arch=sm_100a tma_u32_box.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

#include "../../paper_2305_14566_b200/csrc/ptx.cuh"
using namespace osg;

__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, uint32_t* out, int BW) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint32_t* buf = reinterpret_cast<uint32_t*>(dsm);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, 6 * (BW < 0 ? -BW : BW) * 4);
    if (BW < 0) ptx::tma_load_2d(buf, &m, &bar, c0, c1);
    else ptx::tma_load_4d(buf, &m, &bar, c0, c1, 0, 0);
  }
  ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 6 * (BW < 0 ? -BW : BW); i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int W = 384, H = 64;
  std::vector<uint32_t> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = 0x01000000u + i;
  uint32_t *d, *o;
  cudaMalloc(&d, W * H * 4);
  cudaMalloc(&o, 6 * 132 * 4);
  cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, 1, 1};
  cuuint64_t strides[3] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * 4};
  int bw = argc > 1 ? atoi(argv[1]) : 132;
  int dt = argc > 2 ? atoi(argv[2]) : 0;
  cuuint32_t box[4] = {(cuuint32_t)bw, 6, 1, 1}, es[4] = {1, 1, 1, 1};
  if (dt == 3) {  // the same bytes viewed as u8: box {4 bw, 6}
    dims[0] = (cuuint64_t)W * 4;
    box[0] = (cuuint32_t)bw * 4;
  }
  CUresult r = cuTensorMapEncodeTiled(&m, dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : dt == 3 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_INT32, 4, d, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("box %d dt %d encode %d\n", bw, dt, (int)r);
  int cases[3][2] = {{100, 10}, {-4, -1}, {-1, 3}};
  for (auto& c : cases) {
    k<<<1, 128, 8192>>>(m, dt == 3 ? 4 * c[0] : c[0], c[1], o, bw);  // 4-D map
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint32_t> g(6 * 132);
    cudaMemcpy(g.data(), o, g.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < 6; ++y)
      for (int x = 0; x < bw; ++x) {
        int gx = c[0] + x, gy = c[1] + y;
        uint32_t ex = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? h[gy * W + gx] : 0u;
        bad += g[y * bw + x] != ex;
      }
    printf("coords (%d,%d): %s, mismatches %d\n", c[0], c[1], cudaGetErrorString(e), bad);
  }
  return 0;
}
