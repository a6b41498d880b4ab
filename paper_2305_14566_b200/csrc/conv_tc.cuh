// conv_tc.cuh -- implicit-GEMM convolution on tcgen05 tensor cores (sm_100a).
//
// D[M = pixels, N = C_out] = A[M, K = taps x C_in] * W[N, K]^T, fp32 accumulation in TMEM.
// A is never materialised: for tap (dy, dx) and channel chunk kc the 128-pixel M tile
// (hb rows x wb cols of the output grid of one image) is one 4-D TMA box of the NHWC
// input starting at (kc*BK, x0*s + dx - r, y0*s + dy - r, b); the box's out-of-bounds
// elements are zero-filled by TMA, which IS the convolution's zero 'same' padding, and
// the stride-2 convolutions use TMA element strides (every other input pixel).
// The smem image of the box is a K-major, BK*2-byte-swizzled 128 x BK operand, the
// canonical UMMA layout, consumed directly by tcgen05.mma.
//
// Warp roles (256 threads, 1 CTA/SM, persistent over (m_tile, n_tile) work items):
//   warp 0: TMA producer (one lane)      warp 1: MMA issuer (one lane)
//   warp 2: TMEM allocator               warps 4-7: epilogue (TMEM -> regs -> global)
// Pipelines: smem ring full/empty (STAGES), TMEM accumulator full/empty (2 buffers).
// Epilogues (fused): +bias, +residual, ReLU, nearest-up x2 + skip add, rounding to the
// 16-bit storage type (the canonical rounding points of DESIGN.md R9).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "ptx.cuh"

namespace osg {

enum ConvMode : int { kReluBias = 0, kResidualRelu = 1, kUpAdd = 2, kBias = 3 };

struct ConvArgs {
  int B, Ho, Wo;          // conv output grid (mode 2: the low-resolution grid)
  int Cin, Cout;
  int ksize, stride;      // 1 or 3; 1 or 2
  int wb, hb;             // M tile = hb x wb output pixels (wb * hb == 128)
  int tiles_x, tiles_y;   // Wo / wb, Ho / hb
  int n_tiles_n;          // Cout / BN
  int kchunks;            // Cin / BK
  int num_work;           // B * tiles_y * tiles_x * n_tiles_n
  const float* bias;      // [Cout]
  const void* res;        // residual (mode 1, [B][Ho][Wo][Cout]) or skip (mode 2, [B][2Ho][2Wo][Cout])
  void* out;              // [B][Ho][Wo][Cout] (mode 2: [B][2Ho][2Wo][Cout])
  int split;              // res/out stored as [Cout] hi | [Cout] lo per pixel (x2 precision mode)
};

template <typename T>
struct StoreT;
template <>
struct StoreT<__half> {
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ float2 unpack(uint32_t u) {
    __half2 h = *reinterpret_cast<__half2*>(&u);
    return __half22float2(h);
  }
};
template <>
struct StoreT<__nv_bfloat16> {
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ float2 unpack(uint32_t u) {
    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
    return __bfloat1622float2(h);
  }
};

// Row I/O of the epilogue. A pixel's channels are stored either plain ([C]) or split
// ([C] hi | [C] lo, hi = round(v), lo = round(v - hi): the "x2" precision mode in which
// the next convolution runs its K loop over both halves with the same exact weights).
template <typename T, int CH>
__device__ __forceinline__ void add_row(float (&v)[CH], const T* base, size_t pix, int n0, int C, int split) {
  const size_t stride = split ? 2 * (size_t)C : (size_t)C;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 1 && !split) break;
    const uint4* rs = reinterpret_cast<const uint4*>(base + pix * stride + h * C + n0);
#pragma unroll
    for (int j = 0; j < CH / 8; ++j) {
      uint4 rv = __ldg(rs + j);
      uint32_t rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = StoreT<T>::unpack(rr[e]);
        v[8 * j + 2 * e] += f.x;
        v[8 * j + 2 * e + 1] += f.y;
      }
    }
  }
}
template <typename T, int CH>
__device__ __forceinline__ void store_row(const float (&v)[CH], T* base, size_t pix, int n0, int C, int split) {
  const size_t stride = split ? 2 * (size_t)C : (size_t)C;
  uint4* hs = reinterpret_cast<uint4*>(base + pix * stride + n0);
#pragma unroll
  for (int j = 0; j < CH / 8; ++j) {
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = StoreT<T>::pack(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
    hs[j] = make_uint4(o[0], o[1], o[2], o[3]);
    if (split) {
      uint32_t l[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 hv = StoreT<T>::unpack(o[e]);
        l[e] = StoreT<T>::pack(v[8 * j + 2 * e] - hv.x, v[8 * j + 2 * e + 1] - hv.y);
      }
      reinterpret_cast<uint4*>(base + pix * stride + C + n0)[j] = make_uint4(l[0], l[1], l[2], l[3]);
    }
  }
}

template <int BN, int BK, int STAGES>
struct ConvSmem {
  static constexpr int kA = 128 * BK * 2;
  static constexpr int kB = ((BN * BK * 2 + 1023) / 1024) * 1024;
  static constexpr int kStage = kA + kB;
  static constexpr int kBars = (2 * STAGES + 4) * 8 + 16;
  static constexpr int kTotal = STAGES * kStage + kBars + 1024;  // + alignment slack
  static constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                                          : (2 * BN <= 256) ? 256 : 512;
  static constexpr uint32_t kLayout = BK == 64 ? 2u : BK == 32 ? 4u : 6u;  // SW128 / SW64 / SW32
  static constexpr uint32_t kSBO = 8 * BK * 2;                              // 8 rows of BK*2 bytes
};

template <typename T, int BN, int BK, int STAGES, int MODE>
__global__ void __launch_bounds__(256, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const ConvArgs args) {
  using S = ConvSmem<BN, BK, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<S::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int r = args.ksize >> 1;
  const int taps = args.ksize * args.ksize;
  const int kiters = taps * args.kchunks;
  constexpr uint32_t kTx = S::kA + BN * BK * 2;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x) {
        const int nt = w % args.n_tiles_n;
        int m = w / args.n_tiles_n;
        const int tx = m % args.tiles_x;
        m /= args.tiles_x;
        const int ty = m % args.tiles_y;
        const int b = m / args.tiles_y;
        const int x0 = tx * args.wb * args.stride - r;
        const int y0 = ty * args.hb * args.stride - r;
        for (int it = 0; it < kiters; ++it) {
          const int tap = it / args.kchunks;
          const int kc = it - tap * args.kchunks;
          const int dy = tap / args.ksize, dx = tap - (tap / args.ksize) * args.ksize;
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStage;
          uint8_t* sb = sa + S::kA;
          ptx::mbar_arrive_expect_tx(&full[stage], kTx);
          ptx::tma_load_4d(sa, &tmA, &full[stage], kc * BK, x0 + dx, y0 + dy, b);
          ptx::tma_load_2d(sb, &tmB, &full[stage], tap * args.Cin + kc * BK, nt * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = ptx::idesc_f16(128, BN, std::is_same<T, __nv_bfloat16>::value);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int it = 0; it < kiters; ++it) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * S::kStage);
          const uint32_t sb = sa + S::kA;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t da = ptx::smem_desc(sa + k * 32, S::kSBO, S::kLayout);
            const uint64_t db = ptx::smem_desc(sb + k * 32, S::kSBO, S::kLayout);
            ptx::mma_f16(d_tmem, da, db, idesc, (it | k) != 0);
          }
          ptx::mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;               // TMEM lane quadrant of this warp
    const int row = q * 32 + lane;        // M row = pixel within the tile
    const int py = row / args.wb, px = row - (row / args.wb) * args.wb;
    int local = 0;
    for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int nt = w % args.n_tiles_n;
      int m = w / args.n_tiles_n;
      const int tx = m % args.tiles_x;
      m /= args.tiles_x;
      const int ty = m % args.tiles_y;
      const int b = m / args.tiles_y;
      const int y = ty * args.hb + py, x = tx * args.wb + px;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      constexpr int CH = BN < 32 ? BN : 32;
#pragma unroll 1
      for (int c = 0; c < BN; c += CH) {
        uint32_t u[32];
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c;
        if constexpr (CH == 32) {
          ptx::tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(u));
        } else {
          ptx::tmem_ld_32x32b_x16(taddr, *reinterpret_cast<uint32_t(*)[16]>(u));
        }
        ptx::tmem_ld_wait();
        const int n0 = nt * BN + c;
        float v[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) v[j] = __uint_as_float(u[j]) + __ldg(args.bias + n0 + j);
        if constexpr (MODE == kUpAdd) {
          const size_t W2 = 2 * (size_t)args.Wo;
#pragma unroll 1
          for (int a = 0; a < 4; ++a) {
            const size_t pix = ((size_t)b * 2 * args.Ho + 2 * y + (a >> 1)) * W2 + 2 * x + (a & 1);
            float u[CH];
#pragma unroll
            for (int j = 0; j < CH; ++j) u[j] = v[j];
            add_row<T, CH>(u, static_cast<const T*>(args.res), pix, n0, args.Cout, args.split);
            store_row<T, CH>(u, static_cast<T*>(args.out), pix, n0, args.Cout, args.split);
          }
        } else {
          const size_t pix = ((size_t)b * args.Ho + y) * args.Wo + x;
          if constexpr (MODE == kResidualRelu)
            add_row<T, CH>(v, static_cast<const T*>(args.res), pix, n0, args.Cout, args.split);
          if constexpr (MODE != kBias) {
#pragma unroll
            for (int j = 0; j < CH; ++j) v[j] = fmaxf(v[j], 0.0f);
          }
          store_row<T, CH>(v, static_cast<T*>(args.out), pix, n0, args.Cout, args.split);
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<S::kTmemCols>(tmem_base);
  }
}

}  // namespace osg
