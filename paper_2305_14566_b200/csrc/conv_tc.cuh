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
#include <cuda_fp8.h>

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace osg {

enum ConvMode : int { kReluBias = 0, kResidualRelu = 1, kUpAdd = 2, kBias = 3, kHeadFused = 4 };
// plan-level request (make_conv_plan only): kHeadFused with the tensor-core head (arch headtc=1):
// R = 4 rows per work item, the plan's mode is kHeadFused and ConvPlan::head_tc is set
constexpr int kHeadFusedTc = 5;

// Storage of an activation tensor, per pixel (R9):
//   kStorePlain  [C] 16-bit
//   kStoreX2     [C] hi | [C] lo, both 16-bit (hi = round(v), lo = round(v - hi))
//   kStoreF8     [C] fp16 hi | [C] e4m3 lo8 = sat(round((v - hi) * 2^6)), 3C bytes per pixel.
// A convolution over an F8 input runs its K loop over the hi chunks (kind::f16, 16-bit
// weights) and then the lo chunks (kind::f8f6f4, E5M2 weights W * 2^-6) into ONE fp32
// accumulator: (lo 2^6)(W 2^-6) = lo W.
enum StoreKind : int { kStorePlain = 0, kStoreX2 = 1, kStoreF8 = 2 };
constexpr float kLoScale = 64.0f;
constexpr float kLoInv = 1.0f / 64.0f;

// fp8 TMA maps of an F8 tensor's lo part (input A, lo weights B, output O, residual R).
struct LoMaps {
  CUtensorMap A, B, O, R;
};

// q = v / d, r = v % d for v >= 0, d > 0: a shift and a mask when d is a power of two (the work
// decode of the persistent kernels runs per item on every epilogue thread; signed division is
// ~25 instructions)
__device__ __forceinline__ void udivmod(int v, int d, int& q, int& r) {
  if ((d & (d - 1)) == 0) {
    q = v >> (__ffs(d) - 1);
    r = v & (d - 1);
  } else {
    q = (int)((unsigned)v / (unsigned)d);
    r = v - q * d;
  }
}

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
  int split;              // StoreKind of res/out
  int kch_lo;             // F8 input: number of lo K chunks (after the kchunks hi chunks), else 0
  int lo2;                // per-tap kernel: a lo chunk holds 2 BK channels (128-B rows, SW128)
  // batch-index offsets of the tensors (a launch over images [0, B) of the work space reads
  // input image b + b_in, residual b + b_res, writes b + b_out, head tile b + b_head)
  int b_in, b_res, b_out, b_head;
  // row-chunked (RC) layout flags of the input / residual / output tensors: [B][H][chunk][W][16 B]
  // with the 16-B chunks of a pixel in the order hi chunks, then lo chunks; else NHWC
  int in_rc, res_rc, out_rc;
  int dbg;  // experiments only (OMNISEG_DBG, conv3_nz_kernel): 1 skip epilogue math/stores, 2 skip MMAs, 4 skip loads,
            // 8 record MMA-warp cycle counters into dbg_out[blockIdx.x][4]
  unsigned long long* dbg_out;
  // nz / stride-2 kernels: the weights pre-arranged as the per-K-step smem image
  // [n tile][K step][9 tap slots][BN rows][32 B, SW32 swizzled] (build_conv_wimage), loaded with
  // one bulk copy per K step instead of 9 TMA boxes of 32-byte rows
  const uint8_t* wimg;
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

// ---- F8 lo helpers: e4m3 pairs, low byte = first value
__device__ __forceinline__ uint32_t f8_pack4(float a, float b, float c, float d) {
  const uint32_t p0 = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
  const uint32_t p1 = __nv_cvt_float2_to_fp8x2(make_float2(c, d), __NV_SATFINITE, __NV_E4M3);
  return p0 | (p1 << 16);
}
__device__ __forceinline__ float2 f8_unpack2(uint32_t u16) {
  const __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(u16 & 0xFFFFu), __NV_E4M3);
  const float2 f = __half22float2(__half2(hr));
  return make_float2(f.x * kLoInv, f.y * kLoInv);
}
// 16 values -> 16 fp16 hi (two uint4) + 16 e4m3 lo (one uint4)
__device__ __forceinline__ void split_f8_16(const float* v, uint4& h0, uint4& h1, uint4& lo) {
  uint32_t h[8], l[4];
#pragma unroll
  for (int e = 0; e < 8; ++e) h[e] = StoreT<__half>::pack(v[2 * e], v[2 * e + 1]);
  // (v - hi) 2^6 as one packed FMA per pair: fma(v, 2^6, -hi 2^6) rounds 2^6 (v - hi), which is
  // exact (v - hi is exact by Sterbenz, the scaling by a power of two too): bit-identical
  const float2 s64 = make_float2(kLoScale, kLoScale), m64 = make_float2(-kLoScale, -kLoScale);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 a = __ffma2_rn(make_float2(v[4 * e], v[4 * e + 1]), s64,
                                __fmul2_rn(StoreT<__half>::unpack(h[2 * e]), m64));
    const float2 b = __ffma2_rn(make_float2(v[4 * e + 2], v[4 * e + 3]), s64,
                                __fmul2_rn(StoreT<__half>::unpack(h[2 * e + 1]), m64));
    l[e] = f8_pack4(a.x, a.y, b.x, b.y);
  }
  h0 = make_uint4(h[0], h[1], h[2], h[3]);
  h1 = make_uint4(h[4], h[5], h[6], h[7]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}
// v[0..16) += the 16 lo values of one uint4 of e4m3
__device__ __forceinline__ void add_f8_16(float* v, const uint4& q) {
  // v += lo 2^-6 as packed FMAs (the scaling by a power of two is exact: bit-identical)
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  const float2 inv = make_float2(kLoInv, kLoInv);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)((w[e] >> (16 * k)) & 0xFFFFu), __NV_E4M3);
      const float2 r = __ffma2_rn(__half22float2(__half2(hr)), inv, make_float2(v[4 * e + 2 * k], v[4 * e + 2 * k + 1]));
      v[4 * e + 2 * k] = r.x;
      v[4 * e + 2 * k + 1] = r.y;
    }
  }
}
// smem image of one F8 lo box row of CH bytes: 32-B swizzle (CH = 32) / none (CH = 16)
template <int CH>
__device__ __forceinline__ uint32_t lo_off(int r, int j) {
  if constexpr (CH == 32)
    return r * 32 + 16 * (j ^ ((r >> 2) & 1));
  else
    return r * 16;
}

// Row I/O of the epilogue. A pixel's channels are stored either plain ([C]) or split
// ([C] hi | [C] lo, hi = round(v), lo = round(v - hi): the "x2" precision mode in which
// the next convolution runs its K loop over both halves with the same exact weights).
template <typename T, int CH>
__device__ __forceinline__ void add_row(float (&v)[CH], const T* base, size_t pix, int n0, int C, int split) {
  if (split == kStoreF8) {
    const uint8_t* px = reinterpret_cast<const uint8_t*>(base) + pix * 3 * (size_t)C;
    const uint4* hs = reinterpret_cast<const uint4*>(px + 2 * n0);
    const uint4* ls = reinterpret_cast<const uint4*>(px + 2 * (size_t)C + n0);
#pragma unroll
    for (int j = 0; j < CH / 8; ++j) {
      const uint4 rv = __ldg(hs + j);
      const uint32_t rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = StoreT<T>::unpack(rr[e]);
        v[8 * j + 2 * e] += f.x;
        v[8 * j + 2 * e + 1] += f.y;
      }
    }
#pragma unroll
    for (int j = 0; j < CH / 16; ++j) add_f8_16(v + 16 * j, __ldg(ls + j));
    return;
  }
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
  if (split == kStoreF8) {
    uint8_t* px = reinterpret_cast<uint8_t*>(base) + pix * 3 * (size_t)C;
    uint4* hs = reinterpret_cast<uint4*>(px + 2 * n0);
    uint4* ls = reinterpret_cast<uint4*>(px + 2 * (size_t)C + n0);
#pragma unroll
    for (int j = 0; j < CH / 16; ++j) split_f8_16(v + 16 * j, hs[2 * j], hs[2 * j + 1], ls[j]);
    return;
  }
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


// ---------------------------------------------------------------------------------------
// TMA epilogue (modes 0, 1, 3): each epilogue warp owns 32 M rows = a bw x bh pixel box.
// TMEM -> registers -> bias (+ residual from a TMA-loaded smem tile) -> ReLU -> 16-bit
// (hi, and lo in the x2 mode) -> swizzled STS -> one TMA store per box. The smem images
// use the 64-B (CH = 32) / 32-B (CH = 16) swizzle of the output / residual tensor maps.
template <int CH>
struct EpiTile {
  static constexpr int kRow = CH * 2;
  static constexpr int kBuf = 32 * kRow;
  static constexpr int kWarpBytes = 6 * kBuf;   // out hi, out lo, 2 x (res hi, res lo)
  static constexpr int kBytes = 4 * kWarpBytes; // 4 epilogue warps
  static __device__ __forceinline__ uint32_t off(int r, int j) {
    if constexpr (CH == 32)
      return r * 64 + 16 * (j ^ ((r >> 1) & 3));
    else
      return r * 32 + 16 * (j ^ ((r >> 2) & 1));
  }
};

struct EpiState {
  uint8_t* buf;         // this warp's 6 kBuf-sized buffers (EpiTile::kWarpBytes)
  uint64_t* rbar;       // this warp's 2 residual mbarriers (double-buffered prefetch)
  uint32_t rphase[2];
  int res_base = 2;     // buffer index of residual slot 0 (0 when the warp has no out buffers)
  int res_rc = 0;       // residual / output tensors in the row-chunked layout (see ConvArgs)
  int out_rc = 0;
  // byte offsets of the out / residual slots (epi_layout); a slot is [hi kBuf][lo]
  int out_off[2] = {0, 0}, res_off[2] = {0, 0};
  int oslot = 0;
};

// Slot layout in the warp's 6 kBuf: a slot holds hi (kBuf) + lo (x2: kBuf, F8: kBuf/2, plain:
// none). Plain / F8 slots take 1.5 kBuf, so there is room for TWO output slots (double-
// buffered TMA stores: the next chunk's STS does not wait for the previous store) beside the
// two residual slots; x2 keeps one output slot.
// lean (residual epilogues, F8 / plain storage): ONE output slot + the two residual slots (4.5
// kBuf per warp instead of 6), so the nz kernel's operand ring gets another stage
template <int CH>
__device__ __forceinline__ void epi_layout(EpiState& es, int split, bool lean = false) {
  constexpr int kB = EpiTile<CH>::kBuf;
  if (lean && split != kStoreX2) {
    es.out_off[0] = es.out_off[1] = 0;
    es.res_off[0] = kB + kB / 2;
    es.res_off[1] = 3 * kB;
  } else if (split == kStoreX2) {
    es.out_off[0] = es.out_off[1] = 0;
    es.res_off[0] = es.res_base * kB;
    es.res_off[1] = (es.res_base + 2) * kB;
  } else {
    es.out_off[0] = 0;
    es.out_off[1] = kB + kB / 2;
    const int rb = es.res_base ? 3 * kB : 0;
    es.res_off[0] = rb;
    es.res_off[1] = rb + kB + kB / 2;
  }
}

// smem image offsets of one warp box (32 pixels x CH channels). NHWC boxes are 64-B (CH = 32)
// / 32-B (CH = 16) swizzled pixel rows; row-chunked (RC) boxes are [16-B chunk][32 px][16 B].
// j16: index of a 16-bit 8-channel unit; j8: index of an e4m3 16-channel unit.
template <int CH>
__device__ __forceinline__ uint32_t off16(int rc, int px, int j16) {
  return rc ? (uint32_t)(j16 * 512 + px * 16) : EpiTile<CH>::off(px, j16);
}
template <int CH>
__device__ __forceinline__ uint32_t off8(int rc, int px, int j8) {
  return rc ? (uint32_t)(j8 * 512 + px * 16) : lo_off<CH>(px, j8);
}

// Issue the TMA loads of one residual chunk into buffer slot `slot` (lane 0). F8: the lo part
// comes from the e4m3 map tmR2. RC: 5-D maps {128 B = 8 px, W/8, chunk, H, B}; the chunks of channels
// [n0, n0 + CH) are n0/8.. (hi), C/8 + n0/8.. (x2 lo) and C/8 + n0/16.. (F8 lo).
// SK / RC >= 0: storage kind / row-chunked flag of the residual known at compile time (the
// product configurations: the runtime kind / layout branches fold away); -1: runtime
template <int CH, int SK = -1, int RC = -1>
__device__ __forceinline__ void epi_res_issue(EpiState& es, int slot, const CUtensorMap* tmR, const CUtensorMap* tmR2,
                                              int n0, int Cout, int split_, int xb, int yb, int b, uint32_t lane) {
  using E = EpiTile<CH>;
  const int split = SK >= 0 ? SK : split_;
  if (lane == 0) {
    uint8_t* hi = es.buf + es.res_off[slot];
    const uint32_t tx = split == kStoreF8 ? E::kBuf + 32 * CH : (split ? 2 : 1) * E::kBuf;
    ptx::mbar_arrive_expect_tx(&es.rbar[slot], tx);
    if (RC >= 0 ? RC != 0 : es.res_rc != 0) {
      ptx::tma_load_5d(hi, tmR, &es.rbar[slot], 0, xb / 8, n0 / 8, yb, b);
      if (split == kStoreF8)
        ptx::tma_load_5d(hi + E::kBuf, tmR2, &es.rbar[slot], 0, xb / 8, Cout / 8 + n0 / 16, yb, b);
      else if (split)
        ptx::tma_load_5d(hi + E::kBuf, tmR, &es.rbar[slot], 0, xb / 8, Cout / 8 + n0 / 8, yb, b);
      return;
    }
    ptx::tma_load_4d(hi, tmR, &es.rbar[slot], n0, xb, yb, b);
    if (split == kStoreF8)
      ptx::tma_load_4d(hi + E::kBuf, tmR2, &es.rbar[slot], n0, xb, yb, b);
    else if (split)
      ptx::tma_load_4d(hi + E::kBuf, tmR, &es.rbar[slot], Cout + n0, xb, yb, b);
  }
}

// Accumulator -> bias (+ residual from a TMA-loaded smem tile) -> ReLU (MODE != kBias), for
// one CH-wide chunk of the warp's 32 rows. (xb, yb, b): box origin; n0: first channel.
// The residual of this chunk was issued earlier into `slot` (epi_res_issue).
// SB: `bias` points to a shared-memory copy (16-B aligned): vector LDS instead of per-element
// uniform global loads (the fused head's epilogue is issue-bound)
template <typename T, int CH, int MODE, bool SB = false, int SK = -1, int RC = -1>
__device__ __forceinline__ void epi_values(EpiState& es, int slot, uint32_t taddr, const float* bias, int n0,
                                           int split_, uint32_t lane, float (&v)[CH]) {
  using E = EpiTile<CH>;
  const int split = SK >= 0 ? SK : split_;
  uint8_t* res_hi = es.buf + es.res_off[slot];
  uint8_t* res_lo = res_hi + E::kBuf;
  constexpr bool kRes = MODE == kResidualRelu || MODE == kHeadFused;
  uint32_t u[32];
  if constexpr (CH == 32) {
    ptx::tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(u));
  } else {
    ptx::tmem_ld_32x32b_x16(taddr, *reinterpret_cast<uint32_t(*)[16]>(u));
  }
  ptx::tmem_ld_wait();
  if constexpr (SB) {
#pragma unroll
    for (int j = 0; j < CH; j += 4) {  // + bias, packed, from shared memory
      const float4 b4 = *reinterpret_cast<const float4*>(bias + n0 + j);
      const float2 r0 = __fadd2_rn(make_float2(__uint_as_float(u[j]), __uint_as_float(u[j + 1])), make_float2(b4.x, b4.y));
      const float2 r1 =
          __fadd2_rn(make_float2(__uint_as_float(u[j + 2]), __uint_as_float(u[j + 3])), make_float2(b4.z, b4.w));
      v[j] = r0.x;
      v[j + 1] = r0.y;
      v[j + 2] = r1.x;
      v[j + 3] = r1.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < CH; j += 4) {  // + bias, packed (bias + n0 is 16-B aligned: n0 % 16 == 0)
      const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + n0 + j));
      const float2 r0 = __fadd2_rn(make_float2(__uint_as_float(u[j]), __uint_as_float(u[j + 1])), make_float2(b4.x, b4.y));
      const float2 r1 =
          __fadd2_rn(make_float2(__uint_as_float(u[j + 2]), __uint_as_float(u[j + 3])), make_float2(b4.z, b4.w));
      v[j] = r0.x;
      v[j + 1] = r0.y;
      v[j + 2] = r1.x;
      v[j + 3] = r1.y;
    }
  }
  if constexpr (kRes) {
    const int rc = RC >= 0 ? RC : es.res_rc;
    ptx::mbar_wait(&es.rbar[slot], es.rphase[slot]);
    es.rphase[slot] ^= 1;
    if (split == kStoreF8) {
#pragma unroll
      for (int j = 0; j < CH / 16; ++j)
        add_f8_16(v + 16 * j, *reinterpret_cast<const uint4*>(res_lo + off8<CH>(rc, lane, j)));
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && split != kStoreX2) break;
      const uint8_t* rb = h ? res_lo : res_hi;
#pragma unroll
      for (int j = 0; j < CH / 8; ++j) {
        const uint4 rv = *reinterpret_cast<const uint4*>(rb + off16<CH>(rc, lane, j));
        const uint32_t rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __fadd2_rn(StoreT<T>::unpack(rr[e]), make_float2(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]));
          v[8 * j + 2 * e] = f.x;
          v[8 * j + 2 * e + 1] = f.y;
        }
      }
    }
    __syncwarp();  // every lane has read the residual tile before it is reloaded
  }
  if constexpr (MODE != kBias) {
#pragma unroll
    for (int j = 0; j < CH; ++j) v[j] = fmaxf(v[j], 0.0f);
  }
}

// One CH-wide chunk: values -> 16-bit (hi, + lo in x2 / F8) -> STS -> TMA store.
template <typename T, int CH, int SK = -1>
__device__ __forceinline__ void epi_store(EpiState& es, const CUtensorMap* tmO, const CUtensorMap* tmO2,
                                          const float (&v)[CH], int n0, int Cout, int split, int xb, int yb, int b,
                                          uint32_t lane);

// SK >= 0: the residual / output storage kind known at compile time (see epi_res_issue)
template <typename T, int CH, int MODE, int SK = -1>
__device__ __forceinline__ void epi_chunk(EpiState& es, int slot, const CUtensorMap* tmO, const CUtensorMap* tmO2,
                                          uint32_t taddr, const float* bias, int n0, int Cout, int split, int xb,
                                          int yb, int b, uint32_t lane) {
  float v[CH];
  epi_values<T, CH, MODE, false, SK>(es, slot, taddr, bias, n0, split, lane, v);
  epi_store<T, CH, SK>(es, tmO, tmO2, v, n0, Cout, split, xb, yb, b, lane);
}

// The store half of epi_chunk: v (final values) -> storage kind -> STS -> TMA store.
template <typename T, int CH, int SK>
__device__ __forceinline__ void epi_store(EpiState& es, const CUtensorMap* tmO, const CUtensorMap* tmO2,
                                          const float (&v)[CH], int n0, int Cout, int split_, int xb, int yb, int b,
                                          uint32_t lane) {
  const int split = SK >= 0 ? SK : split_;
  uint8_t* out_hi = es.buf + es.out_off[es.oslot];
  uint8_t* out_lo = out_hi + EpiTile<CH>::kBuf;
  const bool dbl = es.out_off[1] != es.out_off[0];
  es.oslot ^= dbl ? 1 : 0;
  const int rc = es.out_rc;
  // the store that last read this slot is done reading smem (one store may stay in flight
  // when the output is double-buffered)
  if (lane == 0) {
    if (dbl)
      ptx::bulk_wait_read1();
    else
      ptx::bulk_wait_read0();
  }
  __syncwarp();
  if (split == kStoreF8) {
#pragma unroll
    for (int j = 0; j < CH / 16; ++j) {
      uint4 h0, h1, lo;
      split_f8_16(v + 16 * j, h0, h1, lo);
      *reinterpret_cast<uint4*>(out_hi + off16<CH>(rc, lane, 2 * j)) = h0;
      *reinterpret_cast<uint4*>(out_hi + off16<CH>(rc, lane, 2 * j + 1)) = h1;
      *reinterpret_cast<uint4*>(out_lo + off8<CH>(rc, lane, j)) = lo;
    }
  } else {
#pragma unroll
    for (int j = 0; j < CH / 8; ++j) {
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) o[e] = StoreT<T>::pack(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
      *reinterpret_cast<uint4*>(out_hi + off16<CH>(rc, lane, j)) = make_uint4(o[0], o[1], o[2], o[3]);
      if (split) {
        uint32_t l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 hv = StoreT<T>::unpack(o[e]);
          l[e] = StoreT<T>::pack(v[8 * j + 2 * e] - hv.x, v[8 * j + 2 * e + 1] - hv.y);
        }
        *reinterpret_cast<uint4*>(out_lo + off16<CH>(rc, lane, j)) = make_uint4(l[0], l[1], l[2], l[3]);
      }
    }
  }
  ptx::fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    if (rc) {
      ptx::tma_store_5d(tmO, out_hi, 0, xb / 8, n0 / 8, yb, b);
      if (split == kStoreF8)
        ptx::tma_store_5d(tmO2, out_lo, 0, xb / 8, Cout / 8 + n0 / 16, yb, b);
      else if (split)
        ptx::tma_store_5d(tmO, out_lo, 0, xb / 8, Cout / 8 + n0 / 8, yb, b);
    } else {
      ptx::tma_store_4d(tmO, out_hi, n0, xb, yb, b);
      if (split == kStoreF8)
        ptx::tma_store_4d(tmO2, out_lo, n0, xb, yb, b);
      else if (split)
        ptx::tma_store_4d(tmO, out_lo, Cout + n0, xb, yb, b);
    }
    ptx::bulk_commit();
  }
}

constexpr int kHeadDescs = 16;  // task descriptors per epilogue warp (tasks of one scale)
// A task of the item's window scale, compacted per epilogue warp (head_tasks): canvas pointer of
// window pixel (0, 0), the window rows / columns that land on owned canvas pixels, row pitch.
struct HeadTask {
  uint32_t* base;
  int t, Wt, ylo, yhi, xlo, xhi, pad_;
};

// Lanes t < ntasks describe task t if it runs at this window's level (lf); the valid ones are
// compacted in task order into d[0..n) (warp-private shared memory; __syncwarp before use).
__device__ __forceinline__ int head_tasks(const HeadArgs& ha, int lf, int oy, int ox, HeadTask* d, uint32_t lane) {
  const int t = (int)lane;
  const bool on = t < ha.ntasks && ha.tt.log2f[t] == lf;
  const unsigned m = __ballot_sync(0xffffffffu, on);
  if (on) {
    const int cy0 = oy - (ha.pad >> lf), cx0 = ox - (ha.pad >> lf);  // canvas coords of window pixel (0, 0); pad >= 0
    const int Wt = ha.tt.Wt[t];
    HeadTask h;
    h.t = t;
    h.Wt = Wt;
    h.ylo = max(0, max(ha.tt.row0[t], 0) - cy0);
    h.yhi = min(ha.tt.Ht[t], ha.tt.row1[t]) - cy0;
    h.xlo = max(0, -cx0);
    h.xhi = Wt - cx0;
    h.base = ha.tt.canvas[t] + ((int64_t)(cy0 - ha.tt.row0[t]) * Wt + cx0);
    h.pad_ = 0;
    const int k = __popc(m & ((1u << lane) - 1u));
    if (k < kHeadDescs) d[k] = h;
  }
  __syncwarp();
  return __popc(m) <= kHeadDescs ? __popc(m) : -1;  // -1: more tasks than descriptors (generic path)
}

// OMNISEG_CHECKS: the descriptor's bounds and address agree with the direct canvas formula.
__device__ __forceinline__ void head_check(const HeadArgs& ha, const HeadTask& d, int lf, int oy, int ox, int x, int y,
                                           bool in) {
#if OMNISEG_CHECKS
  const int t = d.t, f = 1 << lf;
  const int cy = oy + y - ha.pad / f, cx = ox + x - ha.pad / f;
  const bool ok = cy >= 0 && cy < ha.tt.Ht[t] && cx >= 0 && cx < ha.tt.Wt[t] && cy >= ha.tt.row0[t] &&
                  cy < ha.tt.row1[t];
  OS_DCHECK(ok == in, "head stitch: descriptor bounds differ from the canvas formula");
  if (in)
    OS_DCHECK(d.base + (int64_t)y * d.Wt + x == ha.tt.canvas[t] + (int64_t)(cy - ha.tt.row0[t]) * ha.tt.Wt[t] + cx,
              "head stitch: descriptor address differs from the canvas formula");
#else
  (void)ha, (void)d, (void)lf, (void)oy, (void)ox, (void)x, (void)y, (void)in;
#endif
}

// Fused dynamic head + stitch (MODE kHeadFused, last decoder conv, CH = BN = all C0 channels):
// D0 = ReLU(acc + b + U0) (the storage-rounded value in plain 16-bit modes, the exact fp32
// value in x2 modes, i.e. hi + lo to 2^-22), F = precls(D0), then per task of the tile's
// scale z = W3 ReLU(W2 ReLU(W1 F + b1) + b2) + b3, p = sigmoid(z), and the fixed-point
// canvas atomics of kernels.cu's head_stitch_kernel. D0 itself is never written.
template <typename T, int CH>
__device__ __forceinline__ void epi_head(EpiState& es, int slot, uint32_t taddr, const float* bias, int split,
                                         int xb, int yb, int b, uint32_t lane, const HeadArgs& ha, const float* s_w,
                                         const float* s_b, const float* s_th, int lf, int oy, int ox,
                                         const HeadTask* ht = nullptr, int nht = 0) {
  float v[CH];
  epi_values<T, CH, kHeadFused>(es, slot, taddr, bias, 0, split, lane, v);
  if (!split) {
#pragma unroll
    for (int j = 0; j < CH; ++j) v[j] = float(T(v[j]));
  }
  // precls, weights TRANSPOSED in smem (s_w[j * 8 + o], zero rows beyond C0): input-outer
  // order so the 8 accumulators are independent FMA chains (two float4 loads per input)
  float F[kHead];
#pragma unroll
  for (int o = 0; o < kHead; ++o) F[o] = s_b[o];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const float4 w0 = *reinterpret_cast<const float4*>(s_w + j * 8);
    const float4 w1 = *reinterpret_cast<const float4*>(s_w + j * 8 + 4);
    F[0] = fmaf(w0.x, v[j], F[0]);
    F[1] = fmaf(w0.y, v[j], F[1]);
    F[2] = fmaf(w0.z, v[j], F[2]);
    F[3] = fmaf(w0.w, v[j], F[3]);
    F[4] = fmaf(w1.x, v[j], F[4]);
    F[5] = fmaf(w1.y, v[j], F[5]);
    F[6] = fmaf(w1.z, v[j], F[6]);
    F[7] = fmaf(w1.w, v[j], F[7]);
  }
  const int y = yb, x = xb + (int)lane;  // hb = 1: the warp's 32 pixels of one row
  if (ha.out_F) {
#pragma unroll
    for (int o = 0; o < kHead; ++o) ha.out_F[(((int64_t)b * ha.P + y) * ha.P + x) * kHead + o] = F[o];
  }
  const int f = 1 << lf;
  const int nloop = ht ? nht : ha.ntasks;
  for (int k = 0; k < nloop; ++k) {
    int t = k;
    if (ht) {
      t = ht[k].t;
    } else if (ha.tiles && ha.tt.log2f[t] != lf) {
      continue;
    }
    // theta in smem with W1 / W2 transposed: [i * 8 + o] (see the theta load)
    const float* th = s_th + t * 156;
    float h1[kHead], h2[kHead];
#pragma unroll
    for (int o = 0; o < kHead; ++o) h1[o] = th[64 + o];
#pragma unroll
    for (int i = 0; i < kHead; ++i) {
      const float4 a4 = *reinterpret_cast<const float4*>(th + i * 8);
      const float4 b4 = *reinterpret_cast<const float4*>(th + i * 8 + 4);
      h1[0] = fmaf(a4.x, F[i], h1[0]);
      h1[1] = fmaf(a4.y, F[i], h1[1]);
      h1[2] = fmaf(a4.z, F[i], h1[2]);
      h1[3] = fmaf(a4.w, F[i], h1[3]);
      h1[4] = fmaf(b4.x, F[i], h1[4]);
      h1[5] = fmaf(b4.y, F[i], h1[5]);
      h1[6] = fmaf(b4.z, F[i], h1[6]);
      h1[7] = fmaf(b4.w, F[i], h1[7]);
    }
#pragma unroll
    for (int o = 0; o < kHead; ++o) {
      h1[o] = fmaxf(h1[o], 0.f);
      h2[o] = th[136 + o];
    }
#pragma unroll
    for (int i = 0; i < kHead; ++i) {
      const float4 a4 = *reinterpret_cast<const float4*>(th + 72 + i * 8);
      const float4 b4 = *reinterpret_cast<const float4*>(th + 72 + i * 8 + 4);
      h2[0] = fmaf(a4.x, h1[i], h2[0]);
      h2[1] = fmaf(a4.y, h1[i], h2[1]);
      h2[2] = fmaf(a4.z, h1[i], h2[2]);
      h2[3] = fmaf(a4.w, h1[i], h2[3]);
      h2[4] = fmaf(b4.x, h1[i], h2[4]);
      h2[5] = fmaf(b4.y, h1[i], h2[5]);
      h2[6] = fmaf(b4.z, h1[i], h2[6]);
      h2[7] = fmaf(b4.w, h1[i], h2[7]);
    }
#pragma unroll
    for (int o = 0; o < kHead; ++o) h2[o] = fmaxf(h2[o], 0.f);
    const float4 c4 = *reinterpret_cast<const float4*>(th + 144);
    const float4 d4 = *reinterpret_cast<const float4*>(th + 148);
    float z = th[152];
    z = fmaf(c4.x, h2[0], z);
    z = fmaf(c4.y, h2[1], z);
    z = fmaf(c4.z, h2[2], z);
    z = fmaf(c4.w, h2[3], z);
    z = fmaf(d4.x, h2[4], z);
    z = fmaf(d4.y, h2[5], z);
    z = fmaf(d4.z, h2[6], z);
    z = fmaf(d4.w, h2[7], z);
    if (ht) {  // the stitch through the item's compacted task descriptor
      const HeadTask d = ht[k];
      const bool in = x >= d.xlo && x < d.xhi && y >= d.ylo && y < d.yhi;
      head_check(ha, d, lf, oy, ox, x, y, in);
      if (in) atomicAdd(d.base + (int64_t)y * d.Wt + x, stitch_value(__frcp_rn(1.0f + __expf(-z)), z, ha.tt.vote));
      continue;
    }
    const float p = 1.0f / (1.0f + expf(-z));
    if (ha.out_p) {
      ha.out_p[(((int64_t)b * ha.ntasks + t) * ha.P + y) * ha.P + x] = p;
    } else {
      const int cy = oy + y - ha.pad / f, cx = ox + x - ha.pad / f;
      const int Wt = ha.tt.Wt[t];
      if (cy >= 0 && cy < ha.tt.Ht[t] && cx >= 0 && cx < Wt && cy >= ha.tt.row0[t] && cy < ha.tt.row1[t]) {
        atomicAdd(ha.tt.canvas[t] + (int64_t)(cy - ha.tt.row0[t]) * Wt + cx, stitch_value(p, z, ha.tt.vote));
      }
    }
  }
}

// The fused head for TWO pixels per thread (rows r0, r1 of the warp's column): every shared
// weight load feeds both, and the FMAs run as packed f32x2 (__ffma2_rn, sm_100) -- the same
// fp32 arithmetic per pixel, half the FMA and load instructions of epi_head. v0 / v1: the D0
// values (epi_values) of the two pixels; (x, y0) / (x, y1): their window coordinates.
template <typename T, int CH>
__device__ __forceinline__ void epi_head2(const float (&v0)[CH], const float (&v1)[CH], int x, int y0, int y1, int b,
                                          const HeadArgs& ha, const float* s_w, const float* s_b, const float* s_th,
                                          int lf, int oy, int ox, const HeadTask* ht = nullptr, int nht = 0) {
  // precls with transposed weights (s_w[j * 8 + o]): input-outer, 8 independent packed chains
  float2 F[kHead];
#pragma unroll
  for (int o = 0; o < kHead; ++o) F[o] = make_float2(s_b[o], s_b[o]);
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const float4 w0 = *reinterpret_cast<const float4*>(s_w + j * 8);
    const float4 w1 = *reinterpret_cast<const float4*>(s_w + j * 8 + 4);
    const float2 vj = make_float2(v0[j], v1[j]);
    F[0] = __ffma2_rn(make_float2(w0.x, w0.x), vj, F[0]);
    F[1] = __ffma2_rn(make_float2(w0.y, w0.y), vj, F[1]);
    F[2] = __ffma2_rn(make_float2(w0.z, w0.z), vj, F[2]);
    F[3] = __ffma2_rn(make_float2(w0.w, w0.w), vj, F[3]);
    F[4] = __ffma2_rn(make_float2(w1.x, w1.x), vj, F[4]);
    F[5] = __ffma2_rn(make_float2(w1.y, w1.y), vj, F[5]);
    F[6] = __ffma2_rn(make_float2(w1.z, w1.z), vj, F[6]);
    F[7] = __ffma2_rn(make_float2(w1.w, w1.w), vj, F[7]);
  }
  if (ha.out_F) {
#pragma unroll
    for (int o = 0; o < kHead; ++o) {
      ha.out_F[(((int64_t)b * ha.P + y0) * ha.P + x) * kHead + o] = F[o].x;
      ha.out_F[(((int64_t)b * ha.P + y1) * ha.P + x) * kHead + o] = F[o].y;
    }
  }
  const int f = 1 << lf;
  const int nloop = ht ? nht : ha.ntasks;
  for (int k = 0; k < nloop; ++k) {
    int t = k;
    if (ht) {
      t = ht[k].t;
    } else if (ha.tiles && ha.tt.log2f[t] != lf) {
      continue;
    }
    const float* th = s_th + t * 156;  // W1 / W2 transposed: [i * 8 + o]
    float2 h1[kHead], h2[kHead];
#pragma unroll
    for (int o = 0; o < kHead; ++o) h1[o] = make_float2(th[64 + o], th[64 + o]);
#pragma unroll
    for (int i = 0; i < kHead; ++i) {
      const float4 a4 = *reinterpret_cast<const float4*>(th + i * 8);
      const float4 b4 = *reinterpret_cast<const float4*>(th + i * 8 + 4);
      h1[0] = __ffma2_rn(make_float2(a4.x, a4.x), F[i], h1[0]);
      h1[1] = __ffma2_rn(make_float2(a4.y, a4.y), F[i], h1[1]);
      h1[2] = __ffma2_rn(make_float2(a4.z, a4.z), F[i], h1[2]);
      h1[3] = __ffma2_rn(make_float2(a4.w, a4.w), F[i], h1[3]);
      h1[4] = __ffma2_rn(make_float2(b4.x, b4.x), F[i], h1[4]);
      h1[5] = __ffma2_rn(make_float2(b4.y, b4.y), F[i], h1[5]);
      h1[6] = __ffma2_rn(make_float2(b4.z, b4.z), F[i], h1[6]);
      h1[7] = __ffma2_rn(make_float2(b4.w, b4.w), F[i], h1[7]);
    }
#pragma unroll
    for (int o = 0; o < kHead; ++o) {
      h1[o] = make_float2(fmaxf(h1[o].x, 0.f), fmaxf(h1[o].y, 0.f));
      h2[o] = make_float2(th[136 + o], th[136 + o]);
    }
#pragma unroll
    for (int i = 0; i < kHead; ++i) {
      const float4 a4 = *reinterpret_cast<const float4*>(th + 72 + i * 8);
      const float4 b4 = *reinterpret_cast<const float4*>(th + 72 + i * 8 + 4);
      h2[0] = __ffma2_rn(make_float2(a4.x, a4.x), h1[i], h2[0]);
      h2[1] = __ffma2_rn(make_float2(a4.y, a4.y), h1[i], h2[1]);
      h2[2] = __ffma2_rn(make_float2(a4.z, a4.z), h1[i], h2[2]);
      h2[3] = __ffma2_rn(make_float2(a4.w, a4.w), h1[i], h2[3]);
      h2[4] = __ffma2_rn(make_float2(b4.x, b4.x), h1[i], h2[4]);
      h2[5] = __ffma2_rn(make_float2(b4.y, b4.y), h1[i], h2[5]);
      h2[6] = __ffma2_rn(make_float2(b4.z, b4.z), h1[i], h2[6]);
      h2[7] = __ffma2_rn(make_float2(b4.w, b4.w), h1[i], h2[7]);
    }
#pragma unroll
    for (int o = 0; o < kHead; ++o) h2[o] = make_float2(fmaxf(h2[o].x, 0.f), fmaxf(h2[o].y, 0.f));
    const float4 c4 = *reinterpret_cast<const float4*>(th + 144);
    const float4 d4 = *reinterpret_cast<const float4*>(th + 148);
    float2 z = make_float2(th[152], th[152]);
    z = __ffma2_rn(make_float2(c4.x, c4.x), h2[0], z);
    z = __ffma2_rn(make_float2(c4.y, c4.y), h2[1], z);
    z = __ffma2_rn(make_float2(c4.z, c4.z), h2[2], z);
    z = __ffma2_rn(make_float2(c4.w, c4.w), h2[3], z);
    z = __ffma2_rn(make_float2(d4.x, d4.x), h2[4], z);
    z = __ffma2_rn(make_float2(d4.y, d4.y), h2[5], z);
    z = __ffma2_rn(make_float2(d4.z, d4.z), h2[6], z);
    z = __ffma2_rn(make_float2(d4.w, d4.w), h2[7], z);
    if (ht) {  // the stitch through the item's compacted task descriptor
      const HeadTask d = ht[k];
      const bool xin = x >= d.xlo && x < d.xhi;
      head_check(ha, d, lf, oy, ox, x, y0, xin && y0 >= d.ylo && y0 < d.yhi);
      head_check(ha, d, lf, oy, ox, x, y1, xin && y1 >= d.ylo && y1 < d.yhi);
      // sigmoid with the fast exp / reciprocal (relative error ~1e-7, far inside the 2^-20
      // fixed point the stitch rounds to; the vote decision uses z itself)
      if (xin && y0 >= d.ylo && y0 < d.yhi)
        atomicAdd(d.base + (int64_t)y0 * d.Wt + x, stitch_value(__frcp_rn(1.0f + __expf(-z.x)), z.x, ha.tt.vote));
      if (xin && y1 >= d.ylo && y1 < d.yhi)
        atomicAdd(d.base + (int64_t)y1 * d.Wt + x, stitch_value(__frcp_rn(1.0f + __expf(-z.y)), z.y, ha.tt.vote));
      continue;
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float zz = k ? z.y : z.x;
      const int y = k ? y1 : y0;
      const float p = 1.0f / (1.0f + expf(-zz));
      if (ha.out_p) {
        ha.out_p[(((int64_t)b * ha.ntasks + t) * ha.P + y) * ha.P + x] = p;
      } else {
        const int cy = oy + y - ha.pad / f, cx = ox + x - ha.pad / f;
        const int Wt = ha.tt.Wt[t];
        if (cy >= 0 && cy < ha.tt.Ht[t] && cx >= 0 && cx < Wt && cy >= ha.tt.row0[t] && cy < ha.tt.row1[t]) {
          atomicAdd(ha.tt.canvas[t] + (int64_t)(cy - ha.tt.row0[t]) * Wt + cx, stitch_value(p, zz, ha.tt.vote));
        }
      }
    }
  }
}

// Tensor-core dynamic head, second half (CUDA cores): h1 = ReLU(W1' D0 + b1') of one task
// (layer 1 and precls ran on the tensor cores, epi_head_tc), then h2 = ReLU(W2 h1 + b2),
// z = W3 h2 + b3, p = sigmoid(z) and the fixed-point stitch -- the arithmetic of epi_head.
__device__ __forceinline__ void head_tail(const float (&h1)[kHead], const float* th, const HeadArgs& ha, int t, int x,
                                          int y, int lf, int oy, int ox) {
  float h2[kHead];
#pragma unroll
  for (int o = 0; o < kHead; ++o) h2[o] = th[136 + o];
#pragma unroll
  for (int i = 0; i < kHead; ++i) {
    const float4 a4 = *reinterpret_cast<const float4*>(th + 72 + i * 8);
    const float4 b4 = *reinterpret_cast<const float4*>(th + 72 + i * 8 + 4);
    h2[0] = fmaf(a4.x, h1[i], h2[0]);
    h2[1] = fmaf(a4.y, h1[i], h2[1]);
    h2[2] = fmaf(a4.z, h1[i], h2[2]);
    h2[3] = fmaf(a4.w, h1[i], h2[3]);
    h2[4] = fmaf(b4.x, h1[i], h2[4]);
    h2[5] = fmaf(b4.y, h1[i], h2[5]);
    h2[6] = fmaf(b4.z, h1[i], h2[6]);
    h2[7] = fmaf(b4.w, h1[i], h2[7]);
  }
  const float4 c4 = *reinterpret_cast<const float4*>(th + 144);
  const float4 d4 = *reinterpret_cast<const float4*>(th + 148);
  float z = th[152];
  z = fmaf(c4.x, fmaxf(h2[0], 0.f), z);
  z = fmaf(c4.y, fmaxf(h2[1], 0.f), z);
  z = fmaf(c4.z, fmaxf(h2[2], 0.f), z);
  z = fmaf(c4.w, fmaxf(h2[3], 0.f), z);
  z = fmaf(d4.x, fmaxf(h2[4], 0.f), z);
  z = fmaf(d4.y, fmaxf(h2[5], 0.f), z);
  z = fmaf(d4.z, fmaxf(h2[6], 0.f), z);
  z = fmaf(d4.w, fmaxf(h2[7], 0.f), z);
  const float p = 1.0f / (1.0f + expf(-z));
  const int f = 1 << lf;
  const int cy = oy + y - ha.pad / f, cx = ox + x - ha.pad / f;
  const int Wt = ha.tt.Wt[t];
  if (cy >= 0 && cy < ha.tt.Ht[t] && cx >= 0 && cx < Wt && cy >= ha.tt.row0[t] && cy < ha.tt.row1[t])
    atomicAdd(ha.tt.canvas[t] + (int64_t)(cy - ha.tt.row0[t]) * Wt + cx, stitch_value(p, z, ha.tt.vote));
}

// Per-tap kernel epilogue shape: the output-only modes (kReluBias, kBias) with BN >= 32 run 8
// epilogue warps that split the channels (a pair per TMEM lane quadrant; chunks of tap_epi_ch
// channels); the up-add runs 8 warps split by output row; the residual mode 4 warps.
__host__ __device__ constexpr bool tap_split8(int bn, int mode) {
  return (mode == kReluBias || mode == kBias) && bn >= 32;
}
__host__ __device__ constexpr int tap_epi_ch(int bn, int mode) {
  return tap_split8(bn, mode) ? (bn >= 64 ? 32 : bn / 2) : (bn < 32 ? bn : 32);
}
__host__ __device__ constexpr int tap_epi_warps(int bn, int mode) {
  return (mode == kUpAdd || tap_split8(bn, mode)) ? 8 : 4;
}

template <int BN, int BK, int STAGES, int MODE = kReluBias, int CL = 1>
struct ConvSmem {
  static constexpr bool UP = MODE == kUpAdd;
  static constexpr int kA = 128 * BK * 2;
  // CL = 2 (CTA pair, cta_group::2): each CTA holds half of the N rows of B
  static constexpr int kB = ((BN / CL * BK * 2 + 1023) / 1024) * 1024;
  static constexpr int kStage = kA + kB;
  static constexpr int kBars = (2 * STAGES + 4 + 16) * 8 + 16;  // full/empty, tfull/tempty, 2 x 8 epilogue warps
  static constexpr int kEpiOff = ((STAGES * kStage + kBars + 1023) / 1024) * 1024;
  // epilogue smem: the TMA epilogue tiles, or the up-add tiles (4 x 64 rows x CH ch per warp)
  static constexpr int kCH = BN < 32 ? BN : 32;
  // up-add: 8 epilogue warps x 2 slots x (skip hi, skip lo) 64-pixel buffers, the output
  // computed in place over the skip
  static constexpr int kUpBytes = 8 * 4 * 64 * kCH * 2;
  static constexpr int kEpiBytes = UP ? kUpBytes
                                  : tap_split8(BN, MODE) ? 8 * 3 * EpiTile<tap_epi_ch(BN, MODE)>::kBuf
                                                         : EpiTile<kCH>::kBytes;
  static constexpr int kTotal = kEpiOff + kEpiBytes + 1024;  // + alignment slack
  static constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                                          : (2 * BN <= 256) ? 256 : 512;
  static constexpr uint32_t kLayout = BK == 64 ? 2u : BK == 32 ? 4u : 6u;  // SW128 / SW64 / SW32
  static constexpr uint32_t kSBO = 8 * BK * 2;                              // 8 rows of BK*2 bytes
  static constexpr uint32_t kLayoutLo = BK == 64 ? 4u : 6u;                 // F8 lo rows: BK bytes
  static constexpr uint32_t kSBOLo = 8 * BK;
};

// CL = 2: a CTA pair (cluster of two, cta_group::2) processes work items in pairs (two M
// tiles, the same N tile and K sequence) as ONE M = 256 MMA: each CTA loads its own 128-pixel
// A tile and HALF of the B (weight) rows into its own shared memory, both CTAs' TMA bytes
// complete on the leader's `full` barrier, the leader (rank 0) issues the pair MMAs and
// multicasts its commits to both CTAs' `empty` / `tfull` barriers, and both epilogues release
// the accumulators on the leader's `tempty`. Per SM that is 2/3 of the shared-memory fill of
// the 1-CTA kernel (A + B/2 instead of A + B per K step), which is what bounds the 256-channel
// layers (measured: their MMA warp waited on loads a third of the time; multicasting B, which
// halves L2 reads but not the smem fill, did not help).
template <typename T, int BN, int BK, int STAGES, int MODE, int CL = 1>
__global__ void __launch_bounds__(tap_epi_warps(BN, MODE) == 8 ? 384 : 256, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmR,
                   const ConvArgs args, const __grid_constant__ LoMaps lo) {
  using S = ConvSmem<BN, BK, STAGES, MODE, CL>;
  static_assert(S::kTotal <= 227 * 1024, "shared memory");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  // epilogue warps: 8 for the up-add (a pair per TMEM lane quadrant, one per output row), else 4
  constexpr int EW = tap_epi_warps(BN, MODE);
  uint64_t* rbar = tempty + 2;  // two residual / skip barriers per epilogue warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 2 * EW);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  static_assert(CL == 1 || CL == 2, "cluster size");
  const uint32_t crank = CL == 2 ? ptx::cluster_ctarank() : 0;
  // work item w -> (n tile, m tile); CL = 2: pairs (2p, 2p + 1) share the n tile
  auto decode = [&](int w, int& nt, int& m) {
    if constexpr (CL == 2) {
      const int pp = w >> 1;
      nt = pp % args.n_tiles_n;
      m = 2 * (pp / args.n_tiles_n) + (w & 1);
    } else {
      nt = w % args.n_tiles_n;
      m = w / args.n_tiles_n;
    }
  };

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);  // CL = 2: the leader's multicast commit arrives in both CTAs
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], CL == 2 ? 2 * EW : 32 * EW);  // CL = 2: one arrival per epilogue warp of the pair
    }
    for (int a = 0; a < 2 * EW; ++a) ptx::mbar_init(&rbar[a], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CL == 2)
      ptx::tmem_alloc_cg2<S::kTmemCols>(tmem_slot);
    else
      ptx::tmem_alloc<S::kTmemCols>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (CL == 2)
    ptx::cluster_sync();  // both CTAs' barriers initialised before any cross-CTA arrive
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int r = args.ksize >> 1;
  const int taps = args.ksize * args.ksize;
  const int kct = args.kchunks + args.kch_lo;  // hi chunks, then (F8 input) lo chunks
  const int kiters = taps * kct;
  // bytes landing on one K step's `full` barrier (CL = 2: the leader's, from both CTAs)
  constexpr uint32_t kTx = CL * (S::kA + BN / CL * BK * 2);
  constexpr uint32_t kTxLo = CL * (128 * BK + BN / CL * BK);  // F8 lo chunk: BK bytes per row

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x) {
        int nt, m;
        decode(w, nt, m);
        const int tx = m % args.tiles_x;
        m /= args.tiles_x;
        const int ty = m % args.tiles_y;
        const int b = m / args.tiles_y;
        const int x0 = tx * args.wb * args.stride - r;
        const int y0 = ty * args.hb * args.stride - r;
        for (int it = 0; it < kiters; ++it) {
          const int tap = it / kct;
          const int kc = it - tap * kct;
          const int dy = tap / args.ksize, dx = tap - (tap / args.ksize) * args.ksize;
          if constexpr (MODE == kUpAdd)  // epilogue-bound: let the epilogue warps have the issue slots
            ptx::mbar_wait_backoff(&empty[stage], phase ^ 1);
          else
            ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStage;
          uint8_t* sb = sa + S::kA;
          if constexpr (CL == 2) {
            // both CTAs: own A tile + own half of the B rows, completing on the LEADER's barrier;
            // the leader expects both CTAs' bytes
            const uint32_t fb = ptx::mapa(&full[stage], 0);
            if (kc < args.kchunks) {
              if (crank == 0) ptx::mbar_arrive_expect_tx(&full[stage], kTx);
              ptx::tma_load_4d_cg2(sa, &tmA, fb, kc * BK, x0 + dx, y0 + dy, b + args.b_in);
              ptx::tma_load_2d_cg2(sb, &tmB, fb, tap * args.Cin + kc * BK, nt * BN + crank * (BN / 2));
            } else {
              const int kl = kc - args.kchunks, kw = args.lo2 ? 2 * BK : BK;
              if (crank == 0) ptx::mbar_arrive_expect_tx(&full[stage], args.lo2 ? 2 * kTxLo : kTxLo);
              ptx::tma_load_4d_cg2(sa, &lo.A, fb, kl * kw, x0 + dx, y0 + dy, b + args.b_in);
              ptx::tma_load_2d_cg2(sb, &lo.B, fb, tap * args.Cin + kl * kw, nt * BN + crank * (BN / 2));
            }
          } else if (kc < args.kchunks) {
            ptx::mbar_arrive_expect_tx(&full[stage], kTx);
            ptx::tma_load_4d(sa, &tmA, &full[stage], kc * BK, x0 + dx, y0 + dy, b + args.b_in);
            ptx::tma_load_2d(sb, &tmB, &full[stage], tap * args.Cin + kc * BK, nt * BN);
          } else {
            // lo chunk: BK e4m3 channels (BK-byte rows), or 2 BK (lo2: 128-byte rows, as many TMA
            // rows as a hi chunk for twice the MMAs of a BK-wide lo chunk)
            const int kl = kc - args.kchunks, kw = args.lo2 ? 2 * BK : BK;
            ptx::mbar_arrive_expect_tx(&full[stage], args.lo2 ? 2 * kTxLo : kTxLo);
            ptx::tma_load_4d(sa, &lo.A, &full[stage], kl * kw, x0 + dx, y0 + dy, b + args.b_in);
            ptx::tma_load_2d(sb, &lo.B, &full[stage], tap * args.Cin + kl * kw, nt * BN);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (CL == 1 || crank == 0) {
      // ------------------------------------------------------------ MMA issuer (warp-collective;
      // CL = 2: the leader issues M = 256 pair MMAs)
      constexpr uint32_t idesc = ptx::idesc_f16(128 * CL, BN, std::is_same<T, __nv_bfloat16>::value);
      constexpr uint32_t idesc8 = ptx::idesc_f8(128 * CL, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      unsigned long long c_te = 0, c_full = 0, t_start = OS_CLK();
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        unsigned long long t0 = OS_CLK();
        ptx::mbar_wait_backoff(&tempty[acc], acc_phase ^ 1);
        c_te += OS_CLK() - t0;
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int it = 0; it < kiters; ++it) {
          t0 = OS_CLK();
          ptx::mbar_wait(&full[stage], phase);
          c_full += OS_CLK() - t0;
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * S::kStage);
          const uint32_t sb = sa + S::kA;
          if (it % kct < args.kchunks) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t da = ptx::smem_desc(sa + k * 32, S::kSBO, S::kLayout);
              const uint64_t db = ptx::smem_desc(sb + k * 32, S::kSBO, S::kLayout);
              if constexpr (CL == 2)
                ptx::mma_f16_cg2_w(d_tmem, da, db, idesc, (it | k) != 0);
              else
                ptx::mma_f16_w(d_tmem, da, db, idesc, (it | k) != 0);
            }
          } else if (BK == 64 && args.lo2) {
            // F8 lo chunk of 2 BK = 128 channels: 128-byte rows (SW128), 32 K per MMA
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t da = ptx::smem_desc(sa + k * 32, 1024, 2u);
              const uint64_t db = ptx::smem_desc(sb + k * 32, 1024, 2u);
              if constexpr (CL == 2)
                ptx::mma_f8_cg2_w(d_tmem, da, db, idesc8, 1u);
              else
                ptx::mma_f8_w(d_tmem, da, db, idesc8, 1u);
            }
          } else if constexpr (BK >= 32) {
            // F8 lo chunk: BK bytes per row (SW64 / SW32), 32 K per MMA
#pragma unroll
            for (int k = 0; k < BK / 32; ++k) {
              const uint64_t da = ptx::smem_desc(sa + k * 32, S::kSBOLo, S::kLayoutLo);
              const uint64_t db = ptx::smem_desc(sb + k * 32, S::kSBOLo, S::kLayoutLo);
              if constexpr (CL == 2)
                ptx::mma_f8_cg2_w(d_tmem, da, db, idesc8, 1u);
              else
                ptx::mma_f8_w(d_tmem, da, db, idesc8, 1u);
            }
          }
          if constexpr (CL == 2)
            ptx::mma_commit_cg2_mc_w(&empty[stage], 0x3);
          else
            ptx::mma_commit_w(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CL == 2)
          ptx::mma_commit_cg2_mc_w(&tfull[acc], 0x3);
        else
          ptx::mma_commit_w(&tfull[acc]);
      }
      if (OS_EXP && (args.dbg & 8) && lane == 0) {
        args.dbg_out[blockIdx.x * 4 + 0] = OS_CLK() - t_start;
        args.dbg_out[blockIdx.x * 4 + 1] = c_te;
        args.dbg_out[blockIdx.x * 4 + 2] = c_full;
        args.dbg_out[blockIdx.x * 4 + 3] = local;
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;               // TMEM lane quadrant of this warp
    const int ew = warp - 4, half = ew >> 2;
    const int row = q * 32 + lane;        // M row = pixel within the tile
    const int py = row / args.wb, px = row - (row / args.wb) * args.wb;
    constexpr int CH = tap_epi_ch(BN, MODE);
    constexpr bool kSplit8 = tap_split8(BN, MODE);  // the warp pair of a quadrant splits the channels
    EpiState es{smem + S::kEpiOff + ew * (S::kEpiBytes / EW), &rbar[2 * ew], {0, 0}, 2, args.res_rc, args.out_rc};
    epi_layout<CH>(es, args.split);
    const int bw = args.wb < 32 ? args.wb : 32;
    const int box_dx = (q * 32) % args.wb, box_dy = (q * 32) / args.wb;
    (void)bw;
    // up-add (TMA path): the skip rows are double-buffered ACROSS work items (slot k & 1 holds the
    // k-th load of this warp) so their HBM latency overlaps the previous row's math and stores
    int up_k = 0;
    auto up_issue = [&](int slot, int w2, int c2, int a2) {
      if (lane != 0) return;
      constexpr int kUB = 64 * CH * 2;
      const bool f8 = args.split == kStoreF8;
      int nt2, m2;
      decode(w2, nt2, m2);
      const int tx2 = m2 % args.tiles_x;
      m2 /= args.tiles_x;
      const int ty2 = m2 % args.tiles_y;
      const int b2 = m2 / args.tiles_y + args.b_res;
      const int ox = 2 * (tx2 * args.wb + box_dx), oyy = 2 * (ty2 * args.hb + box_dy) + a2;
      const int n0 = nt2 * BN + c2;
      uint8_t* sk_hi = es.buf + 2 * slot * kUB;
      uint8_t* sk_lo = sk_hi + kUB;
      ptx::bulk_wait_read0();  // the store computed in place in this slot two steps ago has read it
      ptx::mbar_arrive_expect_tx(&es.rbar[slot], f8 ? kUB + kUB / 2 : (args.split ? 2 : 1) * kUB);
      if (args.res_rc) {
        ptx::tma_load_5d(sk_hi, &tmR, &es.rbar[slot], 0, ox / 8, n0 / 8, oyy, b2);
        if (f8)
          ptx::tma_load_5d(sk_lo, &lo.R, &es.rbar[slot], 0, ox / 8, args.Cout / 8 + n0 / 16, oyy, b2);
        else if (args.split)
          ptx::tma_load_5d(sk_lo, &tmR, &es.rbar[slot], 0, ox / 8, args.Cout / 8 + n0 / 8, oyy, b2);
      } else {
        ptx::tma_load_4d(sk_hi, &tmR, &es.rbar[slot], n0, ox, oyy, b2);
        if (f8)
          ptx::tma_load_4d(sk_lo, &lo.R, &es.rbar[slot], n0, ox, oyy, b2);
        else if (args.split)
          ptx::tma_load_4d(sk_lo, &tmR, &es.rbar[slot], args.Cout + n0, ox, oyy, b2);
      }
    };
    if constexpr (MODE == kUpAdd) {
      if (args.wb >= 32 && (int)blockIdx.x < args.num_work) up_issue(0, blockIdx.x, 0, half);
    }
    int local = 0;
    for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      int nt, m;
      decode(w, nt, m);
      const int tx = m % args.tiles_x;
      m /= args.tiles_x;
      const int ty = m % args.tiles_y;
      const int b = m / args.tiles_y;
      const int y = ty * args.hb + py, x = tx * args.wb + px;
      constexpr bool kRes = MODE == kResidualRelu;
      const int xb = tx * args.wb + box_dx, yb = ty * args.hb + box_dy;
      if constexpr (kRes)
        epi_res_issue<CH>(es, 0, &tmR, &lo.R, nt * BN, args.Cout, args.split, xb, yb, b + args.b_res, lane);
      ptx::mbar_wait_backoff(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int c = kSplit8 ? half * CH : 0; c < BN; c += kSplit8 ? 2 * CH : CH) {
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c;
        const int n0 = nt * BN + c;
        const int slot = (c / CH) & 1;
        if constexpr (kRes) {
          if (c + CH < BN)
            epi_res_issue<CH>(es, slot ^ 1, &tmR, &lo.R, n0 + CH, args.Cout, args.split, xb, yb, b + args.b_res, lane);
        }
        if constexpr (MODE == kUpAdd) {
          uint32_t u[32];
          if constexpr (CH == 32) {
            ptx::tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(u));
          } else {
            ptx::tmem_ld_32x32b_x16(taddr, *reinterpret_cast<uint32_t(*)[16]>(u));
          }
          ptx::tmem_ld_wait();
          float v[CH];
#pragma unroll
          for (int j = 0; j < CH; ++j) v[j] = __uint_as_float(u[j]) + __ldg(args.bias + n0 + j);
          if (args.wb >= 32) {
            // TMA path: the warp's 32 low-res pixels (one row) -> two output rows of 64 pixels
            using E = EpiTile<CH>;
            constexpr int kUB = 64 * CH * 2;  // one 64-row buffer; 2 slots x (skip hi, skip lo)
            const bool f8 = args.split == kStoreF8;
            const int orc = args.out_rc;  // RC output: [chunk][64 px][16 B] boxes; the skip stays NHWC
            auto oo16 = [&](int rr, int j) { return orc ? (uint32_t)(j * 1024 + rr * 16) : E::off(rr, j); };
            auto oo8 = [&](int rr, int j) { return orc ? (uint32_t)(j * 1024 + rr * 16) : lo_off<CH>(rr, j); };
            const int src = args.res_rc;  // RC skip: [chunk][64 px][16 B]
            auto so16 = [&](int rr, int j) { return src ? (uint32_t)(j * 1024 + rr * 16) : E::off(rr, j); };
            auto so8 = [&](int rr, int j) { return src ? (uint32_t)(j * 1024 + rr * 16) : lo_off<CH>(rr, j); };
            auto ostore = [&](const uint8_t* o_hi, const uint8_t* o_lo, int ox, int oyy) {
              if (orc) {
                ptx::tma_store_5d(&tmO, o_hi, 0, ox / 8, n0 / 8, oyy, b + args.b_out);
                if (f8)
                  ptx::tma_store_5d(&lo.O, o_lo, 0, ox / 8, args.Cout / 8 + n0 / 16, oyy, b + args.b_out);
                else if (args.split)
                  ptx::tma_store_5d(&tmO, o_lo, 0, ox / 8, args.Cout / 8 + n0 / 8, oyy, b + args.b_out);
              } else {
                ptx::tma_store_4d(&tmO, o_hi, n0, ox, oyy, b + args.b_out);
                if (f8)
                  ptx::tma_store_4d(&lo.O, o_lo, n0, ox, oyy, b + args.b_out);
                else if (args.split)
                  ptx::tma_store_4d(&tmO, o_lo, args.Cout + n0, ox, oyy, b + args.b_out);
              }
              ptx::bulk_commit();
            };
            {
              // this warp's output row a = half; the skip of this (item, chunk) was issued one
              // step ahead into slot up_k & 1: issue the next one (next chunk / item) now. The
              // output is computed in place over the skip buffer and stored from there.
              const int a = half;
              const int ox = 2 * xb, oyy = 2 * yb + a;
              const int slot = up_k & 1;
              {
                int w2 = w, c2 = c + CH;
                if (c2 >= BN) c2 = 0, w2 += gridDim.x;
                if (w2 < args.num_work) up_issue(slot ^ 1, w2, c2, a);
              }
              ++up_k;
              uint8_t* sk_hi = es.buf + 2 * slot * kUB;
              uint8_t* sk_lo = sk_hi + kUB;
              uint8_t* o_hi = sk_hi;
              uint8_t* o_lo = sk_lo;
              ptx::mbar_wait(&es.rbar[slot], es.rphase[slot]);
              es.rphase[slot] ^= 1;
              // phase 1: skip + up-sampled conv value for the lane's two output pixels (all
              // reads of the slot complete before phase 2 overwrites it in place -- the skip
              // and output layouts may differ)
              float x[2][CH];
#pragma unroll
              for (int q2 = 0; q2 < 2; ++q2) {
                const int rr = 2 * (int)lane + q2;
#pragma unroll
                for (int j = 0; j < CH / 8; ++j) {
                  const uint4 h4 = *reinterpret_cast<const uint4*>(sk_hi + so16(rr, j));
                  uint4 l4 = make_uint4(0, 0, 0, 0);
                  if (args.split == kStoreX2) l4 = *reinterpret_cast<const uint4*>(sk_lo + so16(rr, j));
                  const uint32_t hh[4] = {h4.x, h4.y, h4.z, h4.w}, ll[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float2 fh = StoreT<T>::unpack(hh[e]);
                    const float2 fl = StoreT<T>::unpack(ll[e]);
                    x[q2][8 * j + 2 * e] = fh.x + fl.x + v[8 * j + 2 * e];
                    x[q2][8 * j + 2 * e + 1] = fh.y + fl.y + v[8 * j + 2 * e + 1];
                  }
                }
                if (f8) {
#pragma unroll
                  for (int j = 0; j < CH / 16; ++j)
                    add_f8_16(x[q2] + 16 * j, *reinterpret_cast<const uint4*>(sk_lo + so8(rr, j)));
                }
              }
              __syncwarp();
              // phase 2: round to the storage kind and write in the output layout
#pragma unroll
              for (int q2 = 0; q2 < 2; ++q2) {
                const int rr = 2 * (int)lane + q2;
                if (f8) {
#pragma unroll
                  for (int j = 0; j < CH / 16; ++j) {
                    uint4 h0, h1, l4;
                    split_f8_16(x[q2] + 16 * j, h0, h1, l4);
                    *reinterpret_cast<uint4*>(o_hi + oo16(rr, 2 * j)) = h0;
                    *reinterpret_cast<uint4*>(o_hi + oo16(rr, 2 * j + 1)) = h1;
                    *reinterpret_cast<uint4*>(o_lo + oo8(rr, j)) = l4;
                  }
                } else {
#pragma unroll
                  for (int j = 0; j < CH / 8; ++j) {
                    uint32_t o[4], l[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                      const float x0 = x[q2][8 * j + 2 * e], x1 = x[q2][8 * j + 2 * e + 1];
                      o[e] = StoreT<T>::pack(x0, x1);
                      const float2 hv = StoreT<T>::unpack(o[e]);
                      l[e] = StoreT<T>::pack(x0 - hv.x, x1 - hv.y);
                    }
                    *reinterpret_cast<uint4*>(o_hi + oo16(rr, j)) = make_uint4(o[0], o[1], o[2], o[3]);
                    if (args.split) *reinterpret_cast<uint4*>(o_lo + oo16(rr, j)) = make_uint4(l[0], l[1], l[2], l[3]);
                  }
                }
              }
              ptx::fence_proxy_async();
              __syncwarp();
              if (lane == 0) ostore(o_hi, o_lo, ox, oyy);
            }
          } else if (half == 0) {
            const size_t W2 = 2 * (size_t)args.Wo;
#pragma unroll 1
            for (int a = 0; a < 4; ++a) {
              const size_t pin = (size_t)(2 * y + (a >> 1)) * W2 + 2 * x + (a & 1);
              const size_t img = (size_t)2 * args.Ho * W2;
              float uu[CH];
#pragma unroll
              for (int j = 0; j < CH; ++j) uu[j] = v[j];
              add_row<T, CH>(uu, static_cast<const T*>(args.res), (size_t)(b + args.b_res) * img + pin, n0, args.Cout,
                             args.split);
              store_row<T, CH>(uu, static_cast<T*>(args.out), (size_t)(b + args.b_out) * img + pin, n0, args.Cout,
                               args.split);
            }
          }
        } else {
          epi_chunk<T, CH, MODE>(es, slot, &tmO, &lo.O, taddr, args.bias, n0, args.Cout, args.split, xb, yb,
                                 b + args.b_out, lane);
        }
      }
      ptx::tc_fence_before();
      if constexpr (CL == 2) {  // one arrival per warp on the leader's barrier
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(&tempty[acc], 0));
      } else {
        ptx::mbar_arrive(&tempty[acc]);
      }
    }
    if (lane == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  if constexpr (CL == 2)
    ptx::cluster_sync();  // no CTA leaves while its peer may still signal or read it
  else
    __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    if constexpr (CL == 2)
      ptx::tmem_dealloc_cg2<S::kTmemCols>(tmem_base);
    else
      ptx::tmem_dealloc<S::kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------------------
// Multi-row variant for 3x3 stride-1 convolutions with N <= 128 (the thin, bandwidth-bound
// levels). One work item = R vertically adjacent 128-pixel M blocks (R * hb image rows of
// one wb-wide column segment) x one N tile. For each (dx, K chunk) a single TMA box of
// R*hb + 2 input rows (dx-shifted, zero-filled outside the image) serves all three dy taps
// of all R blocks: the A operand of block r, tap dy starts (r*hb + dy)*wb pixels into the
// box, a multiple of 8 rows, so it stays aligned to the swizzle atom. The three B boxes
// (taps (0,dx), (1,dx), (2,dx)) are shared by the R blocks. Per 128 output pixels this
// moves 3(R*hb+2)/(R*hb) instead of 9 input rows and 9/R instead of 9 weight tiles through
// L2 -> SMEM. Accumulators: R x BN TMEM columns, double buffered (2 R BN <= 512).
// Compile-time tile configuration of the multi-row kernel: R = 256/BN blocks (so two
// accumulator buffers fill the 512 TMEM columns), the largest K chunk giving >= 3 stages in
// 200 KB of shared memory (else 16 with >= 2 stages).
constexpr int kStageBudget = 168 * 1024;     // smem for the operand ring (the TMA epilogue takes 48 KB)
constexpr int kStageBudgetTap = 168 * 1024;    // per-tap kernel (its TMA epilogue takes 48 KB)
constexpr int kStageBudgetTapUp = 96 * 1024;   // per-tap up-add kernel (its epilogue takes 128 KB)

struct RowsCfg {
  static constexpr int stage_bytes(int bn, int bk, int r, int hb) {
    return (((r * hb + 2) * (128 / hb) * bk * 2 + 1023) / 1024) * 1024 + 3 * (((bn * bk * 2 + 1023) / 1024) * 1024);
  }
  static constexpr int R(int bn) { return 256 / bn; }
  static constexpr int BK(int bn, int hb) {
    return 3 * stage_bytes(bn, 64, R(bn), hb) <= kStageBudget   ? 64
           : 3 * stage_bytes(bn, 32, R(bn), hb) <= kStageBudget ? 32
                                                                : 16;
  }
  static constexpr int STAGES(int bn, int hb) {
    return kStageBudget / stage_bytes(bn, BK(bn, hb), R(bn), hb) > 6
               ? 6
               : kStageBudget / stage_bytes(bn, BK(bn, hb), R(bn), hb);
  }
};

template <int BN, int BK, int R, int ROWS, int WB, int STAGES>
struct RowsSmem {
  static constexpr int kA = ((ROWS * WB * BK * 2 + 1023) / 1024) * 1024;
  static constexpr int kBt = ((BN * BK * 2 + 1023) / 1024) * 1024;  // one tap's B tile
  static constexpr int kStage = kA + 3 * kBt;
  static constexpr int kBars = (2 * STAGES + 12) * 8 + 16;
  static constexpr int kEpiOff = ((STAGES * kStage + kBars + 1023) / 1024) * 1024;
  static constexpr int kTotal = kEpiOff + EpiTile<(BN < 32 ? BN : 32)>::kBytes + 1024;
  static constexpr uint32_t kTmemCols = (2 * R * BN <= 32) ? 32 : (2 * R * BN <= 64) ? 64 : (2 * R * BN <= 128) ? 128
                                         : (2 * R * BN <= 256) ? 256 : 512;
  static constexpr uint32_t kLayout = BK == 64 ? 2u : BK == 32 ? 4u : 6u;
  static constexpr uint32_t kSBO = 8 * BK * 2;
  static constexpr uint32_t kLayoutLo = BK == 64 ? 4u : 6u;  // F8 lo rows: BK bytes
  static constexpr uint32_t kSBOLo = 8 * BK;
};

template <typename T, int BN, int BK, int R, int HB, int STAGES, int MODE>
__global__ void __launch_bounds__(256, 1)
    conv3_rows_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmR,
                      const ConvArgs args, const __grid_constant__ LoMaps lo) {
  constexpr int WB = 128 / HB;
  constexpr int ROWS = R * HB + 2;
  using S = RowsSmem<BN, BK, R, ROWS, WB, STAGES>;
  static_assert(S::kTotal <= 227 * 1024, "shared memory");
  static_assert(2 * R * BN <= 512, "TMEM");
  static_assert(WB % 8 == 0, "swizzle alignment of the shifted A operands");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;  // 8 residual barriers (two per epilogue warp)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 8);
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
    for (int a = 0; a < 8; ++a) ptx::mbar_init(&rbar[a], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<S::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int kct = args.kchunks + args.kch_lo;  // hi chunks, then (F8 input) lo chunks
  const int kiters = 3 * kct;                   // (dx, kc)
  constexpr uint32_t kTx = ROWS * WB * BK * 2 + 3 * BN * BK * 2;
  constexpr uint32_t kTxLo = ROWS * WB * BK + 3 * BN * BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x) {
        const int nt = w % args.n_tiles_n;
        int m = w / args.n_tiles_n;
        const int tx = m % args.tiles_x;
        m /= args.tiles_x;
        const int tyg = m % args.tiles_y;
        const int b = m / args.tiles_y;
        const int x0 = tx * WB - 1;
        const int y0 = tyg * R * HB - 1;
        for (int it = 0; it < kiters; ++it) {
          const int dx = it / kct;
          const int kc = it - dx * kct;
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStage;
          const bool hi = kc < args.kchunks;
          const int kk = hi ? kc : kc - args.kchunks;
          const CUtensorMap* mA = hi ? &tmA : &lo.A;
          const CUtensorMap* mB = hi ? &tmB : &lo.B;
          ptx::mbar_arrive_expect_tx(&full[stage], hi ? kTx : kTxLo);
          ptx::tma_load_4d(sa, mA, &full[stage], kk * BK, x0 + dx, y0, b + args.b_in);
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
            ptx::tma_load_2d(sa + S::kA + dy * S::kBt, mB, &full[stage], (dy * 3 + dx) * args.Cin + kk * BK,
                             nt * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // MMA issuer (warp-collective)
      constexpr uint32_t idesc = ptx::idesc_f16(128, BN, std::is_same<T, __nv_bfloat16>::value);
      constexpr uint32_t idesc8 = ptx::idesc_f8(128, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
        const int acc = local & 1;
        ptx::mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_base = tmem_base + acc * R * BN;
        for (int it = 0; it < kiters; ++it) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * S::kStage);
          if (it % kct >= args.kchunks) {
            if constexpr (BK >= 32) {
              // F8 lo chunk: BK bytes per row, 32 K per MMA (always accumulates: hi chunks precede)
#pragma unroll
              for (int dy = 0; dy < 3; ++dy) {
                const uint32_t sb = sa + S::kA + dy * S::kBt;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                  const uint32_t a0 = sa + (uint32_t)((r * HB + dy) * WB * BK);
#pragma unroll
                  for (int k = 0; k < BK / 32; ++k) {
                    const uint64_t da = ptx::smem_desc(a0 + k * 32, S::kSBOLo, S::kLayoutLo);
                    const uint64_t db = ptx::smem_desc(sb + k * 32, S::kSBOLo, S::kLayoutLo);
                    ptx::mma_f8_w(d_base + r * BN, da, db, idesc8, 1u);
                  }
                }
              }
            }
            ptx::mma_commit_w(&empty[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
#pragma unroll
          for (int dy = 0; dy < 3; ++dy) {
            const uint32_t sb = sa + S::kA + dy * S::kBt;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const uint32_t a0 = sa + (uint32_t)((r * HB + dy) * WB * BK * 2);
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                const uint64_t da = ptx::smem_desc(a0 + k * 32, S::kSBO, S::kLayout);
                const uint64_t db = ptx::smem_desc(sb + k * 32, S::kSBO, S::kLayout);
                ptx::mma_f16_w(d_base + r * BN, da, db, idesc, (it | dy | k) != 0);
              }
            }
          }
          ptx::mma_commit_w(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit_w(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    constexpr int CH = BN < 32 ? BN : 32;
    EpiState es{smem + S::kEpiOff + q * EpiTile<CH>::kWarpBytes, &rbar[2 * q], {0, 0}, 2, args.res_rc, args.out_rc};
    epi_layout<CH>(es, args.split);
    const int box_dx = (q * 32) % WB, box_dy = (q * 32) / WB;
    int local = 0;
    for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
      const int acc = local & 1;
      const int nt = w % args.n_tiles_n;
      int m = w / args.n_tiles_n;
      const int tx = m % args.tiles_x;
      m /= args.tiles_x;
      const int tyg = m % args.tiles_y;
      const int b = m / args.tiles_y;
      constexpr bool kRes = MODE == kResidualRelu;
      constexpr int NC = BN / CH;
      const int xb = tx * WB + box_dx;
      const int yb0 = tyg * R * HB + box_dy;
      if constexpr (kRes)
        epi_res_issue<CH>(es, 0, &tmR, &lo.R, nt * BN, args.Cout, args.split, xb, yb0, b + args.b_res, lane);
      ptx::mbar_wait_backoff(&tfull[acc], (local >> 1) & 1);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int i = 0; i < R * NC; ++i) {
        const int r = i / NC, c = (i - r * NC) * CH;
        const int slot = i & 1;
        if constexpr (kRes) {
          if (i + 1 < R * NC) {
            const int r1 = (i + 1) / NC, c1 = (i + 1 - r1 * NC) * CH;
            epi_res_issue<CH>(es, slot ^ 1, &tmR, &lo.R, nt * BN + c1, args.Cout, args.split, xb, yb0 + r1 * HB,
                              b + args.b_res, lane);
          }
        }
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN + r * BN + c;
        epi_chunk<T, CH, MODE>(es, slot, &tmO, &lo.O, taddr, args.bias, nt * BN + c, args.Cout, args.split, xb,
                               yb0 + r * HB, b + args.b_out, lane);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<S::kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------------------
// Multi-row 3x3 stride-1 kernel with a NO-SWIZZLE A operand (image width >= 128, N <= 64).
// The input is in the row-chunked (RC) layout [B][H][16-B chunk][W][16 B], so one image row
// of one chunk is W*16 contiguous bytes. Per 32-byte K step (two chunks) one 5-D TMA box
// {128 B = 8 px, 18 units, 2 chunks, R+2 rows, 1} brings the (R+2) input rows x 144 pixels
// [x0 - 8, x0 + 136) (OOB zero-filled = the conv padding) into smem as [row][chunk][144 px]
// [16 B] -- 128-B TMA rows (a 16-B inner box dimension is limited to 16 B per cycle per SM,
// measured). In the K-major no-swizzle UMMA layout every pixel is one 16-B core-matrix row,
// so the operand of block r, tap (dy, dx) starts at row r+dy, pixel 7+dx of the box (LBO =
// the chunk plane): all 9 taps of all R blocks come from one load (~(R+2)/R input reads per
// output). Weights: 9 per-tap SW32 boxes per chunk, shared by the R blocks.
// EK: epilogue kind -- 0 output only (two compact output slots, 3 kBuf per warp), 1 output +
// residual (6 kBuf), 2 fused head (residual slots only, 4 kBuf).
template <int BN, int R, int STAGES, bool DYF = false, int EW = 8, int EK = 0, int CL = 1>
struct NzSmem {
  static constexpr bool HEAD = EK == 2;
  static constexpr int kPx = 144;                                   // 18 units of 8 pixels
  static constexpr int kChunkStride = kPx * 16;                      // LBO of the A operand
  static constexpr int kRowStride = 2 * kChunkStride;                // two chunks (K = 32 B) per row
  static constexpr int kABytes = (R + 2) * kRowStride;
  static constexpr int kA = ((kABytes + 1023) / 1024) * 1024;
  // one tap's BN x 16-channel weight tile (SW32); the dy-stacked variant packs the three dy
  // tiles of one dx back to back, so they must be exactly BN*32 bytes apart
  // tap slots back to back (one bulk copy per K step); CL = 2 (CTA pair): this CTA's half of N
  static constexpr int kBt = BN / CL * 32;
  static constexpr int kStage = kA + ((9 * kBt + 1023) / 1024) * 1024;
  // full / empty per stage, tfull / tempty x 2, two residual barriers per epilogue warp, + TMEM slot
  static constexpr int kBars = (2 * STAGES + 4 + 2 * EW) * 8 + 16;
  static constexpr int kEpiOff = ((STAGES * kStage + kBars + 1023) / 1024) * 1024;
  // EW epilogue warps; with 8 (fused head: no output tiles) each warp keeps residual slots only
  // EK 3 / 4: lean residual / output-only epilogue (one output slot, epi_layout lean): 4.5 / 1.5 kBuf
  static constexpr int kWarpEpi =
      (EK == 4 ? 3 : EK == 3 ? 9 : EK == 2 ? 8 : EK == 1 ? 12 : 6) * EpiTile<(BN < 32 ? BN : 32)>::kBuf / 2;
  static constexpr int kHeadOff = kEpiOff + EW * kWarpEpi;
  static constexpr int kHeadTasks = 8;  // fused head supports up to 8 tasks per batch
  static constexpr int kHeadBytes = HEAD ? (kHeadTasks * 156 + kHead * 64 + kHead) * 4 + EW * kHeadDescs * 32 : 0;
  // tensor-core dynamic head (fp16 activations, see epi_head_tc): per epilogue half the D0 row
  // as UMMA A operands (128 px x BN channels, fp16 hi and lo, no-swizzle K-major), the item's B
  // operand W1' = W1 Wpre (BN x BN, hi and lo), b1' and one MMA-completion mbarrier per half
  // (2 halves x 2 rows in flight x hi / lo A tiles; layer-1 results in TMEM columns past the
  // two accumulator buffers)
  static constexpr int kTcA = 128 * BN * 2;                          // one A tile (hi or lo)
  static constexpr int kTcB = BN * BN * 2;                           // one B tile
  static constexpr int kTcOff = ((kHeadOff + kHeadBytes + 1023) / 1024) * 1024;
  static constexpr bool kTc = EK == 2 && BN <= 32 && R == 4;  // = NzCfg::tc(BN, EK, R)
  static constexpr int kTcBytes = kTc ? 8 * kTcA + 2 * kTcB + BN * 4 + 64 : 0;
  static constexpr int kTotal = kTcOff + kTcBytes + 1024;
  static constexpr uint32_t kTmemCols = kTc || 2 * R * BN > 256 ? 512 : 256;
};

struct NzCfg {
  // R output rows per work item: 2 R BN = 512 TMEM columns (two accumulator buffers), at most 8
  // rows (the (R+2)-row input box must leave room for >= 2 ring stages). The optional tensor-core
  // head (arch headtc=1, BN <= 32) runs R = 4: half the accumulator columns stay free for its
  // layer-1 results and the smaller input box leaves shared memory for its A tiles.
  static constexpr int R(int bn) { return 256 / bn < 8 ? 256 / bn : 8; }
  static constexpr int RTC = 4;
  static constexpr bool tc(int bn, int ek, int r) { return ek == 2 && bn <= 32 && r == RTC; }
  static constexpr int stage_bytes(int bn, int r, int cl = 1) {
    return (((r + 2) * 2 * 144 * 16 + 1023) / 1024) * 1024 + ((9 * (bn / cl) * 32 + 1023) / 1024) * 1024;
  }
  // CTA pairs (CL = 2): half the weight image per stage
  static constexpr int STAGES_CL2(int bn, int ek) {
    return budget(bn, ek, R(bn)) / stage_bytes(bn, R(bn), 2) > 6 ? 6 : budget(bn, ek, R(bn)) / stage_bytes(bn, R(bn), 2);
  }
  // ring depth from what the 8 epilogue warps (kind ek, see NzSmem) leave of 227 KB
  static constexpr int STAGES(int bn, int ek, int r) {
    return budget(bn, ek, r) / stage_bytes(bn, r) > 6 ? 6 : budget(bn, ek, r) / stage_bytes(bn, r);
  }
  static constexpr int STAGES(int bn, int ek) { return STAGES(bn, ek, R(bn)); }
  static constexpr int tc_bytes(int bn) { return 8 * 128 * bn * 2 + 2 * bn * bn * 2 + bn * 4 + 64; }
  static constexpr int budget(int bn, int ek, int r) {
    return 227 * 1024 - 3 * 1024 - 8 * (ek == 4 ? 3 : ek == 3 ? 9 : ek == 2 ? 8 : ek == 1 ? 12 : 6) * 32 * (bn < 32 ? bn : 32) -
           (ek == 2 ? 7680 + 8 * kHeadDescs * 32 : 0) - (tc(bn, ek, r) ? 1024 + tc_bytes(bn) : 0);
  }

};

// The MMAs of one 32-byte K chunk of conv3_nz_kernel (warp-collective issue). F8: the lo
// chunk (e4m3 activations x e5m2 weights, kind::f8f6f4); otherwise 16-bit (kind::f16).
template <int BN, int R, bool DYF, bool F8, bool BF, typename S, int CL = 1>
__device__ __forceinline__ void nz_mma_chunk(uint32_t sa, uint32_t d_base, int kc) {
  if constexpr (DYF) {
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {
      const uint32_t sbd = sa + S::kA + dx * 3 * S::kBt;
#pragma unroll
      for (int i = -1; i <= R; ++i) {
        const int r_hi = i + 1 < R - 1 ? i + 1 : R - 1;
        const int r_lo = i - 1 > 0 ? i - 1 : 0;
        const int nrows = r_hi - r_lo + 1;
        const int dy0 = i - r_hi + 1;
        const uint32_t a0 = sa + (uint32_t)((i + 1) * S::kRowStride + (7 + dx) * 16);
        const uint64_t da = ptx::smem_desc_noswz(a0, S::kChunkStride, 128);
        const uint64_t db = ptx::smem_desc(sbd + dy0 * BN * 32, 8 * 32, 6u);
        if constexpr (F8)
          ptx::mma_f8_w(d_base + (R - 1 - r_hi) * BN, da, db, ptx::idesc_f8(128, nrows * BN), 1u);
        else
          ptx::mma_f16_w(d_base + (R - 1 - r_hi) * BN, da, db, ptx::idesc_f16(128, nrows * BN, BF), 1u);
      }
    }
  } else {
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      const int dy = tap / 3, dx = tap % 3;
      const uint64_t db = ptx::smem_desc(sa + S::kA + tap * S::kBt, 8 * 32, 6u);  // SW32, 8 rows x 32 B
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t a0 = sa + (uint32_t)((r + dy) * S::kRowStride + (7 + dx) * 16);
        const uint64_t da = ptx::smem_desc_noswz(a0, S::kChunkStride, 128);
        if constexpr (CL == 2) {  // CTA pair: M = 256 over both CTAs' A tiles, N = BN over their B halves
          if constexpr (F8)
            ptx::mma_f8_cg2_w(d_base + r * BN, da, db, ptx::idesc_f8(256, BN), 1u);
          else
            ptx::mma_f16_cg2_w(d_base + r * BN, da, db, ptx::idesc_f16(256, BN, BF), (kc | tap) != 0);
        } else if constexpr (F8) {
          ptx::mma_f8_w(d_base + r * BN, da, db, ptx::idesc_f8(128, BN), 1u);
        } else {
          ptx::mma_f16_w(d_base + r * BN, da, db, ptx::idesc_f16(128, BN, BF), (kc | tap) != 0);
        }
      }
    }
  }
}

// DYF ("dy-fused"): the three dy weight tiles of a dx are stacked along N, so ONE MMA with
// ONE A fetch (input row i, shift dx) produces the contributions to output rows i+1, i, i-1
// (N = 3 BN; 2 BN / BN at the band edges). The R accumulators are laid out in reverse row
// order (row r at column (R-1-r) BN) so those three are contiguous; because one MMA covers
// accumulators first-written by different MMAs, they are zeroed by the epilogue
// (tcgen05.st) after each use and every MMA accumulates. ~1.9x (BN=32) / 1.5x (BN=64) less
// tensor-core operand traffic than one MMA per (tap, row).
// LEAN (kResidualRelu / kReluBias, F8 / plain storage): the lean epilogue layout (EK 3 / 4), more ring stages
template <typename T, int BN, int R, int STAGES, int MODE, bool DYF, int CL = 1, bool LEAN = false>
__global__ void __launch_bounds__(384, 1)
    conv3_nz_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmR,
                    const ConvArgs args, const __grid_constant__ HeadArgs hargs, const __grid_constant__ LoMaps lo) {
  // epilogue warps: 8 (2 per TMEM lane quadrant, alternating rows) for the residual and
  // fused-head epilogues, whose per-row work exceeds the MMA time of thin layers; 4 otherwise
  // 8 epilogue warps (2 per TMEM lane quadrant, alternating rows): a single warp per SM
  // sub-partition leaves the epilogue latency-bound (measured: it, not the loads or MMAs, set
  // the pace of the thin layers)
  constexpr int EW = 8;
  using S = NzSmem<BN, R, STAGES, DYF, EW,
                   MODE == kHeadFused ? 2 : MODE == kResidualRelu ? (LEAN ? 3 : 1) : (LEAN ? 4 : 0), CL>;
  static_assert(!LEAN || MODE == kResidualRelu || MODE == kReluBias, "lean epilogue: residual / output-only modes");
  static_assert(!DYF || 3 * BN <= 256, "dy-fused N");
  // CL = 2: CTA pair (cta_group::2, see conv_tc_kernel): items in pairs (two M items, one N tile),
  // each CTA's A rows + its half of the weight image complete on the leader's `full` barrier
  static_assert(CL == 1 || (!DYF && MODE != kHeadFused), "CTA pairs: plain multi-row layers only");
  const uint32_t crank = CL == 2 ? ptx::cluster_ctarank() : 0;
  auto decode = [&](int w, int& nt, int& m) {
    if constexpr (CL == 2) {
      const int pp = w >> 1;
      nt = pp % args.n_tiles_n;
      m = 2 * (pp / args.n_tiles_n) + (w & 1);
    } else {
      udivmod(w, args.n_tiles_n, m, nt);
    }
  };
  static_assert(S::kTotal <= 227 * 1024, "shared memory");
  static_assert(2 * R * BN <= 512, "TMEM");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;  // two residual barriers per epilogue warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 2 * EW);
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
      ptx::mbar_init(&tempty[a], CL == 2 ? 2 * EW : 32 * EW);
    }
    for (int a = 0; a < 2 * EW; ++a) ptx::mbar_init(&rbar[a], 1);
    if constexpr (S::kTc) {
      uint64_t* hmb = reinterpret_cast<uint64_t*>(smem + S::kTcOff + 8 * S::kTcA + 2 * S::kTcB + BN * 4);
      for (int i = 0; i < 8; ++i) ptx::mbar_init(&hmb[i], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CL == 2)
      ptx::tmem_alloc_cg2<S::kTmemCols>(tmem_slot);
    else
      ptx::tmem_alloc<S::kTmemCols>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (CL == 2)
    ptx::cluster_sync();
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // 32-byte K chunks: kchunks hi chunks (16 fp16 channels), then kch_lo F8 lo chunks (32 e4m3)
  const int kiters = args.kchunks + args.kch_lo;
  constexpr uint32_t kTx = CL * (S::kABytes + 9 * S::kBt);

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x) {
        int nt, m;
        decode(w, nt, m);
        const int tx = m % args.tiles_x;
        m /= args.tiles_x;
        const int tyg = m % args.tiles_y;
        const int b = m / args.tiles_y;
        const int u0 = tx * 16 - 1;  // first 8-pixel unit of the box (pixels [x0 - 8, x0 + 136))
        const int y0 = tyg * R - 1;
        for (int kc = 0; kc < kiters; ++kc) {
          if constexpr (MODE == kHeadFused)  // epilogue-bound: leave the issue slots to the head math
            ptx::mbar_wait_backoff(&empty[stage], phase ^ 1);
          else
            ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStage;
          const bool hi = kc < args.kchunks;
          const int kk = hi ? kc : kc - args.kchunks;
          if (OS_EXP && (args.dbg & 4)) {
            ptx::mbar_arrive(&full[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          (void)hi;
          (void)kk;
          if constexpr (CL == 2) {
            // own A rows + own half of the K step's weight image (3-D map {32 B, BN/2 rows, 9
            // tap planes} over the pair-layout image, tmB) -> the leader's barrier
            const uint32_t fb = ptx::mapa(&full[stage], 0);
            if (crank == 0) ptx::mbar_arrive_expect_tx(&full[stage], kTx);
            ptx::tma_load_5d_cg2(sa, &tmA, fb, 0, u0, 2 * kc, y0, b + args.b_in);
            ptx::tma_load_3d_cg2(sa + S::kA, &tmB, fb, 0, 0, (((nt * kiters + kc) * 2) + (int)crank) * 9);
          } else {
            ptx::mbar_arrive_expect_tx(&full[stage], kTx);
            // chunks 2kc, 2kc+1 of the RC input: hi chunks first, then (F8) the lo chunks
            ptx::tma_load_5d(sa, &tmA, &full[stage], 0, u0, 2 * kc, y0, b + args.b_in);
            ptx::bulk_load(sa + S::kA, args.wimg + ((size_t)nt * kiters + kc) * 9 * BN * 32, 9 * BN * 32,
                           &full[stage]);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (CL == 1 || crank == 0) {  // MMA issuer (warp-collective; the hi/lo kind branch is per
                                  // chunk, outside the MMA loops; CL = 2: the leader only)
      constexpr bool kBf = std::is_same<T, __nv_bfloat16>::value;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      unsigned long long c_te = 0, c_full = 0, c_all = 0, t_start = OS_CLK();
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
        const int acc = local & 1;
        // DYF: the epilogue zeroes every buffer and arrives once up front (real phases)
        unsigned long long t0 = OS_CLK();
        ptx::mbar_wait_backoff(&tempty[acc], DYF ? ((local >> 1) & 1) : (((local >> 1) & 1) ^ 1));
        c_te += OS_CLK() - t0;
        ptx::tc_fence_after();
        const uint32_t d_base = tmem_base + acc * R * BN;
        for (int kc = 0; kc < kiters; ++kc) {
          t0 = OS_CLK();
          ptx::mbar_wait(&full[stage], phase);
          c_full += OS_CLK() - t0;
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * S::kStage);
          if (OS_EXP && (args.dbg & 2)) {
          } else if (kc >= args.kchunks) {  // F8 lo chunk: same smem image, kind::f8f6f4
            nz_mma_chunk<BN, R, DYF, true, kBf, S, CL>(sa, d_base, kc);
          } else {
            nz_mma_chunk<BN, R, DYF, false, kBf, S, CL>(sa, d_base, kc);
          }
          if constexpr (CL == 2)
            ptx::mma_commit_cg2_mc_w(&empty[stage], 0x3);
          else
            ptx::mma_commit_w(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CL == 2)
          ptx::mma_commit_cg2_mc_w(&tfull[acc], 0x3);
        else
          ptx::mma_commit_w(&tfull[acc]);
      }
      c_all = OS_CLK() - t_start;
      if (OS_EXP && (args.dbg & 8) && lane == 0) {
        args.dbg_out[blockIdx.x * 4 + 0] = c_all;
        args.dbg_out[blockIdx.x * 4 + 1] = c_te;
        args.dbg_out[blockIdx.x * 4 + 2] = c_full;
        args.dbg_out[blockIdx.x * 4 + 3] = local;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;            // TMEM lane quadrant
    const int ew = warp - 4;           // epilogue warp index
    constexpr int NH = EW / 4;         // warps per quadrant (they alternate rows)
    const int half = ew / 4;
    constexpr int CH = BN < 32 ? BN : 32;
    EpiState es{smem + S::kEpiOff + ew * S::kWarpEpi, &rbar[2 * ew], {0, 0}, MODE == kHeadFused ? 0 : 2, args.res_rc,
                args.out_rc};
    epi_layout<CH>(es, args.split, LEAN);
    float* s_th = reinterpret_cast<float*>(smem + S::kHeadOff);
    float* s_w = s_th + S::kHeadTasks * 156;
    float* s_b = s_w + kHead * 64;
    const float* th_g = nullptr;         // this item's transposed theta rows (global, or s_th)
    HeadTask* s_ht = reinterpret_cast<HeadTask*>(s_b + kHead) + ew * kHeadDescs;  // this warp's task descriptors
    bool h_ok = false;
    int h_n = 0;
    (void)s_ht;
    const int et = ew * 32 + (int)lane;  // 0 .. 32*EW-1 over the epilogue warps
    // tensor-core head (the row loop below): fp16 activations, all BN channels in one chunk
    constexpr bool kTcHead = S::kTc && std::is_same<T, __half>::value && CH == BN;
    uint8_t* tc_a = smem + S::kTcOff + half * 4 * S::kTcA;  // this half's A tiles: 2 rows x (hi, lo)
    uint8_t* tc_b = smem + S::kTcOff + 8 * S::kTcA;         // B tiles: hi, lo
    float* tc_b1 = reinterpret_cast<float*>(tc_b + 2 * S::kTcB);
    uint64_t* tc_bar = reinterpret_cast<uint64_t*>(tc_b + 2 * S::kTcB + BN * 4);
    uint32_t tc_phase = 0;
    int tl[BN / 8 > 0 ? BN / 8 : 1];
    int ns = 0;
    bool tc = false;
    (void)tc_a;
    (void)tc_bar;
    (void)tc_phase;
    (void)tl;
    // the fused head's conv bias (two-row path): in the theta staging area, which only the
    // tensor-core head uses
    float* s_bias = s_th;
    (void)s_bias;
    if constexpr (MODE == kHeadFused) {
      for (int i = et; i < kHead * CH; i += 32 * EW) {  // transposed: s_w[j * 8 + o]
        const int o = i / CH, j = i - o * CH;
        s_w[j * 8 + o] = j < hargs.C0 ? hargs.Wpre[o * hargs.C0 + j] : 0.f;
      }
      if (et < kHead) s_b[et] = hargs.bpre[et];
      if (!S::kTc && et < BN) s_bias[et] = args.bias[et];
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");  // s_w / s_b / s_bias complete
    }
    if constexpr (DYF) {
      // zero both accumulator buffers (this warp's lanes; the NH warps of a quadrant split the
      // columns) and release them to the MMA warp
      for (int c = half * (2 * R * BN / NH); c < (half + 1) * (2 * R * BN / NH); c += 16)
        ptx::tmem_st_zero16(tmem_base + ((uint32_t)(q * 32) << 16) + c);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[0]);
      ptx::mbar_arrive(&tempty[1]);
    }
    int local = 0;
    for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
      const int acc = local & 1;
      int nt, m, tx, tyg, b;
      decode(w, nt, m);
      udivmod(m, args.tiles_x, m, tx);
      udivmod(m, args.tiles_y, b, tyg);
      int lf = 0, oy = 0, ox = 0;
      if constexpr (MODE == kHeadFused) {
        // the window's theta (W1 / W2 transposed, rows of 156 floats, written by the controller)
        // is read straight from global memory by the head (warp-uniform float4 loads, L1
        // broadcast): no per-item staging and no epilogue-wide barrier. The tensor-core head
        // stages it in shared memory for the B-operand build.
        th_g = hargs.theta_t + (int64_t)(b + args.b_head) * hargs.ntasks * 156;
        if constexpr (S::kTc) {
          asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");  // previous theta no longer read
          for (int i = et; i < hargs.ntasks * 156; i += 32 * EW) s_th[i] = th_g[i];
          asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
          th_g = s_th;
        }
        if (hargs.tiles) {
          const uint32_t id = hargs.tiles[hargs.first + b + args.b_head];
          lf = id >> 30;
          oy = min((int)((id >> 15) & 0x7FFF) * hargs.S, (hargs.Hp >> lf) - hargs.P);
          ox = min((int)(id & 0x7FFF) * hargs.S, (hargs.Wp >> lf) - hargs.P);
        }
        h_ok = hargs.tiles != nullptr && hargs.out_p == nullptr && hargs.out_F == nullptr;
        if (h_ok) h_n = head_tasks(hargs, lf, oy, ox, s_ht, lane);
        if constexpr (kTcHead) {
          // tensor-core head for this item: the window's tasks of its scale, at most BN / 8
          ns = 0;
          if (hargs.tiles && !hargs.out_F) {
            for (int t = 0; t < hargs.ntasks; ++t)
              if (hargs.tt.log2f[t] == lf) {
#pragma unroll
                for (int k = 0; k < BN / 8; ++k)
                  if (k == ns) tl[k] = t;  // constant indices: tl stays in registers
                ++ns;
              }
          }
          tc = ns >= 1 && ns <= BN / 8 && !(OS_EXP && hargs.no_tc);
          if (tc) {
            // B = W1' (rows n = task * 8 + o, K = BN input channels of precls), fp16 hi / lo in
            // the no-swizzle K-major layout: W1'[n][k] = sum_j W1_t[o][j] Wpre[j][k];
            // b1'[n] = b1_t[o] + sum_j W1_t[o][j] bpre[j] (layer 1 folded through precls)
            for (int i = et; i < BN * BN; i += 32 * EW) {
              const int n = i / BN, k = i - n * BN, ti = n >> 3, o = n & 7;
              float wv = 0.f;
              if (ti < ns) {
                const float* th = s_th + tl[ti] * 156;
#pragma unroll
                for (int j = 0; j < kHead; ++j) wv = fmaf(th[j * 8 + o], s_w[k * 8 + j], wv);
              }
              const __half hv = __float2half_rn(wv);
              const __half lv = __float2half_rn(wv - __half2float(hv));
              const int off = (k >> 3) * (BN * 16) + (n >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
              *reinterpret_cast<__half*>(tc_b + off) = hv;
              *reinterpret_cast<__half*>(tc_b + S::kTcB + off) = lv;
            }
            if (et < BN) {
              const int ti = et >> 3, o = et & 7;
              float bv = 0.f;
              if (ti < ns) {
                const float* th = s_th + tl[ti] * 156;
                bv = th[64 + o];
#pragma unroll
                for (int j = 0; j < kHead; ++j) bv = fmaf(th[j * 8 + o], s_b[j], bv);
              }
              tc_b1[et] = bv;
            }
            ptx::fence_proxy_async();
            asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
          }
        }
      }
      constexpr bool kRes = MODE == kResidualRelu || MODE == kHeadFused;
      constexpr int NC = BN / CH;
      const int xb = tx * 128 + q * 32;
      constexpr int RM = R / NH;  // rows of this warp: r = j * NH + half
      // the first residual chunk does not depend on the accumulator: issue it before waiting
      if constexpr (kRes)
        epi_res_issue<CH>(es, 0, &tmR, &lo.R, nt * BN, args.Cout, args.split, xb, tyg * R + half, b + args.b_res, lane);
      ptx::mbar_wait_backoff(&tfull[acc], (local >> 1) & 1);
      ptx::tc_fence_after();
      if (kTcHead && tc) {
        // Tensor-core dynamic head. Phase 1, for each of the warp's RM rows: D0 = ReLU(acc + b +
        // U0) -> fp16 hi + lo into the row's A tiles (pixel m = 32 q + lane: the 4 quadrant warps
        // of the half fill the 128-pixel row) -> named barrier of the half -> the quadrant-0 warp
        // issues D = A_hi B_hi + A_lo B_hi + A_hi B_lo (M = 128, N = BN: every task's layer-1
        // pre-activation W1' D0) into the row's own TMEM columns past the accumulator buffers
        // and commits to the row's mbarrier. Phase 2: wait, load the warp's 32 lanes, run
        // W2 / W3 / sigmoid / stitch on the CUDA cores (head_tail). All RM rows' MMAs are in
        // flight before the first wait.
        static_assert(!kTcHead || RM * NH * BN <= 512 - 2 * R * BN, "TMEM columns for the head");
#pragma unroll
        for (int i = 0; i < RM; ++i) {
          const int r = i * NH + half, slot = i & 1;
          if (i + 1 < RM)
            epi_res_issue<CH>(es, slot ^ 1, &tmR, &lo.R, 0, args.Cout, args.split, xb, tyg * R + (i + 1) * NH + half,
                              b + args.b_res, lane);
          const uint32_t taddr =
              tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN + (DYF ? (R - 1 - r) : r) * BN;
          float v[CH];
          epi_values<T, CH, kHeadFused>(es, slot, taddr, args.bias, 0, args.split, lane, v);
          if (!args.split) {
#pragma unroll
            for (int j = 0; j < CH; ++j) v[j] = float(T(v[j]));
          }
          uint8_t* ta = tc_a + i * 2 * S::kTcA;
          const int m = q * 32 + (int)lane;
#pragma unroll
          for (int g = 0; g < CH / 8; ++g) {
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const __half2 h2 = __floats2half2_rn(v[8 * g + 2 * e], v[8 * g + 2 * e + 1]);
              const float2 hf = __half22float2(h2);
              const __half2 l2 = __floats2half2_rn(v[8 * g + 2 * e] - hf.x, v[8 * g + 2 * e + 1] - hf.y);
              hw[e] = *reinterpret_cast<const uint32_t*>(&h2);
              lw[e] = *reinterpret_cast<const uint32_t*>(&l2);
            }
            const int off = g * 2048 + (m >> 3) * 128 + (m & 7) * 16;
            *reinterpret_cast<uint4*>(ta + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(ta + S::kTcA + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
          ptx::fence_proxy_async();
          ptx::tc_fence_before();
          asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory");
          if (q == 0) {
            ptx::tc_fence_after();
            constexpr uint32_t id = ptx::idesc_f16(128, BN, false);
            const uint32_t a_hi = ptx::smem_u32(ta), a_lo = a_hi + S::kTcA;
            const uint32_t b_hi = ptx::smem_u32(tc_b), b_lo = b_hi + S::kTcB;
            const uint32_t d = tmem_base + 2 * R * BN + (half * RM + i) * BN;
#pragma unroll
            for (int kk = 0; kk < CH / 16; ++kk) {
              const uint64_t dah = ptx::smem_desc_noswz(a_hi + kk * 4096, 2048, 128);
              const uint64_t dal = ptx::smem_desc_noswz(a_lo + kk * 4096, 2048, 128);
              const uint64_t dbh = ptx::smem_desc_noswz(b_hi + kk * BN * 32, BN * 16, 128);
              const uint64_t dbl = ptx::smem_desc_noswz(b_lo + kk * BN * 32, BN * 16, 128);
              ptx::mma_f16_w(d, dah, dbh, id, kk > 0 ? 1u : 0u);
              ptx::mma_f16_w(d, dal, dbh, id, 1u);
              ptx::mma_f16_w(d, dah, dbl, id, 1u);
            }
            ptx::mma_commit_w(&tc_bar[half * RM + i]);
          }
        }
        // every accumulator row of this warp has been read: zero them (DYF) and hand the buffer
        // back to the MMA warp before waiting for the head MMAs
        if constexpr (DYF) {
          for (int j = 0; j < RM; ++j) {
            const int r = j * NH + half;
            for (int c = 0; c < BN; c += 16)
              ptx::tmem_st_zero16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN + (R - 1 - r) * BN + c);
          }
          ptx::tmem_st_wait();
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
#pragma unroll
        for (int i = 0; i < RM; ++i) {
          const int r = i * NH + half;
          ptx::mbar_wait(&tc_bar[half * RM + i], tc_phase);
          ptx::tc_fence_after();
          uint32_t hr[CH];
          const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16) + 2 * R * BN + (half * RM + i) * BN;
          if constexpr (CH == 32)
            ptx::tmem_ld_32x32b_x32(tq, *reinterpret_cast<uint32_t(*)[32]>(hr));
          else
            ptx::tmem_ld_32x32b_x16(tq, *reinterpret_cast<uint32_t(*)[16]>(hr));
          ptx::tmem_ld_wait();
#pragma unroll
          for (int ti = 0; ti < BN / 8; ++ti) {  // constant indices: hr / tl stay in registers
            if (ti < ns) {
              float h1[kHead];
#pragma unroll
              for (int o = 0; o < kHead; ++o) h1[o] = fmaxf(__uint_as_float(hr[ti * 8 + o]) + tc_b1[ti * 8 + o], 0.f);
              head_tail(h1, s_th + tl[ti] * 156, hargs, tl[ti], xb + (int)lane, tyg * R + r, lf, oy, ox);
            }
          }
        }
        tc_phase ^= 1;
        continue;  // accumulator already released
      } else if constexpr (MODE == kHeadFused && NC == 1 && RM % 2 == 0) {
        // two rows (pixels (xb + lane, r0) and (xb + lane, r1)) per pass: both residual slots
        // are consumed by epi_values before the head math, so the next pair's residual loads
        // are issued right away and overlap it
        // the product configuration (F8 split, row-chunked residual) runs a copy of the pass
        // loop with the storage kind / layout known at compile time
        auto passes = [&](auto f8rc_tag) {
          constexpr bool F8RC = decltype(f8rc_tag)::value;
#pragma unroll 1
          for (int i = 0; i < RM; i += 2) {
            const int r0 = i * NH + half, r1 = (i + 1) * NH + half;
            epi_res_issue<CH, F8RC ? (int)kStoreF8 : -1, F8RC ? 1 : -1>(es, 1, &tmR, &lo.R, 0, args.Cout, args.split, xb, tyg * R + r1, b + args.b_res,
                                      lane);
            const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN;
            float v0[CH], v1[CH];
            constexpr bool kSB = !S::kTc;  // s_bias staged (the tensor-core build keeps theta there)
            const float* bsrc = kSB ? s_bias : args.bias;
            epi_values<T, CH, kHeadFused, kSB, F8RC ? (int)kStoreF8 : -1, F8RC ? 1 : -1>(es, 0, tq + (DYF ? (R - 1 - r0) : r0) * BN, bsrc, 0, args.split, lane,
                                             v0);
            epi_values<T, CH, kHeadFused, kSB, F8RC ? (int)kStoreF8 : -1, F8RC ? 1 : -1>(es, 1, tq + (DYF ? (R - 1 - r1) : r1) * BN, bsrc, 0, args.split, lane,
                                             v1);
            if (i + 2 < RM)
              epi_res_issue<CH, F8RC ? (int)kStoreF8 : -1, F8RC ? 1 : -1>(es, 0, &tmR, &lo.R, 0, args.Cout, args.split, xb, tyg * R + (i + 2) * NH + half,
                                      b + args.b_res, lane);
            if (!F8RC && !args.split) {
#pragma unroll
              for (int j = 0; j < CH; ++j) {
                v0[j] = float(T(v0[j]));
                v1[j] = float(T(v1[j]));
              }
            }
            epi_head2<T, CH>(v0, v1, xb + (int)lane, tyg * R + r0, tyg * R + r1, b + args.b_head, hargs, s_w, s_b,
                             th_g, lf, oy, ox, h_ok && h_n >= 0 ? s_ht : nullptr, h_n);
          }
        };
        if (args.split == kStoreF8 && es.res_rc)
          passes(std::true_type{});
        else
          passes(std::false_type{});
      } else {
        // F8 storage (the product dtype) runs a copy of the chunk loop with the kind known at
        // compile time
        auto chunks = [&](auto f8_tag) {
          constexpr int SK = decltype(f8_tag)::value ? (int)kStoreF8 : -1;
#pragma unroll 1
          for (int i = 0; i < RM * NC; ++i) {
            const int r = (i / NC) * NH + half, c = (i % NC) * CH;
            const int slot = i & 1;
            if constexpr (kRes) {
              if (i + 1 < RM * NC) {
                const int r1 = ((i + 1) / NC) * NH + half, c1 = ((i + 1) % NC) * CH;
                epi_res_issue<CH, SK>(es, slot ^ 1, &tmR, &lo.R, nt * BN + c1, args.Cout, args.split, xb, tyg * R + r1,
                                      b + args.b_res, lane);
              }
            }
            const uint32_t taddr =
                tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN + (DYF ? (R - 1 - r) : r) * BN + c;
            if (OS_EXP && (args.dbg & 1)) {
              if constexpr (kRes) {
                ptx::mbar_wait(&es.rbar[slot], es.rphase[slot]);
                es.rphase[slot] ^= 1;
              }
            } else if constexpr (MODE == kHeadFused) {
              epi_head<T, CH>(es, slot, taddr, args.bias, args.split, xb, tyg * R + r, b + args.b_head, lane, hargs,
                              s_w, s_b, th_g, lf, oy, ox, h_ok && h_n >= 0 ? s_ht : nullptr, h_n);
            } else {
              epi_chunk<T, CH, MODE, SK>(es, slot, &tmO, &lo.O, taddr, args.bias, nt * BN + c, args.Cout, args.split,
                                         xb, tyg * R + r, b + args.b_out, lane);
            }
          }
        };
        if (MODE != kHeadFused && args.split == kStoreF8)
          chunks(std::true_type{});
        else
          chunks(std::false_type{});
      }
      if constexpr (DYF) {
        for (int j = 0; j < RM; ++j) {
          const int r = j * NH + half;
          for (int c = 0; c < BN; c += 16)
            ptx::tmem_st_zero16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN + (R - 1 - r) * BN + c);
        }
        ptx::tmem_st_wait();
      }
      ptx::tc_fence_before();
      if constexpr (CL == 2) {  // one arrival per warp on the leader's barrier
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(&tempty[acc], 0));
      } else {
        ptx::mbar_arrive(&tempty[acc]);
      }
    }
    if (lane == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  if constexpr (CL == 2)
    ptx::cluster_sync();
  else
    __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    if constexpr (CL == 2)
      ptx::tmem_dealloc_cg2<S::kTmemCols>(tmem_base);
    else
      ptx::tmem_dealloc<S::kTmemCols>(tmem_base);
  }
}

}  // namespace osg

namespace osg {

// ---------------------------------------------------------------------------------------
// Stride-2 3x3 convolution over a ROW-CHUNKED input (the U-Net down convs of the levels whose
// tensors are row-chunked). Like conv3_nz_kernel, one 5-D TMA box per 32-byte K step brings
// 2R+1 full input rows x 144 pixels (128-B TMA rows) into smem; the M tile is 128 consecutive
// INPUT pixels of one input row, so the MMA computes the stride-1 response at every input
// column and the epilogue keeps the even ones (output pixel x0/2 + m/2 at TMEM lane m): 2x MMA
// work for 1x loads -- a strided pixel walk is not a UMMA operand layout, and this layer's
// MMA time is far below its load time. Only the even-row outputs are computed: input row i
// of the box feeds output row i/2 (dy = 0) and i/2 - 1 (dy = 2) when i is even, (i-1)/2 (dy = 1)
// when odd; with the R accumulators in reverse row order the even case is ONE MMA with the
// [dy0 | dy2] weight tiles stacked along N (N = 2 BN). Accumulators are zeroed by the epilogue.
template <int BN, int R, int STAGES>
struct S2Smem {
  static constexpr int kPx = 144;
  static constexpr int kChunkStride = kPx * 16;
  static constexpr int kRowStride = 2 * kChunkStride;
  static constexpr int kABytes = (2 * R + 1) * kRowStride;
  static constexpr int kA = ((kABytes + 1023) / 1024) * 1024;
  static constexpr int kBt = BN * 32;  // one tap's BN x 32-B weight tile (SW32); per dx: [dy0][dy2][dy1]
  static constexpr int kStage = kA + ((9 * kBt + 1023) / 1024) * 1024;
  static constexpr int kBars = (2 * STAGES + 8) * 8 + 16;
  static constexpr int kEpiOff = ((STAGES * kStage + kBars + 1023) / 1024) * 1024;
  static constexpr int kCH = BN < 32 ? BN : 32;
  static constexpr int kEpiBuf = 16 * kCH * 2;                 // 16 output pixels x CH 16-bit channels
  static constexpr int kTotal = kEpiOff + 8 * 4 * kEpiBuf + 1024;  // 8 warps x 2 x (hi, lo)
  static constexpr uint32_t kTmemCols = (2 * R * BN <= 256) ? 256 : 512;
};

struct S2Cfg {
  static constexpr int R(int bn) { return 256 / bn < 4 ? 256 / bn : 4; }
  static constexpr int stage_bytes(int bn) {
    return (((2 * R(bn) + 1) * 2 * 144 * 16 + 1023) / 1024) * 1024 + ((9 * bn * 32 + 1023) / 1024) * 1024;
  }
  static constexpr int budget(int bn) { return 227 * 1024 - 3 * 1024 - 32 * 16 * (bn < 32 ? bn : 32) * 2; }
  static constexpr int STAGES(int bn) { return budget(bn) / stage_bytes(bn) > 4 ? 4 : budget(bn) / stage_bytes(bn); }
};

template <int BN, int R, bool F8, bool BF, typename S>
__device__ __forceinline__ void s2_mma_chunk(uint32_t sa, uint32_t d_base) {
#pragma unroll
  for (int dx = 0; dx < 3; ++dx) {
    const uint32_t sbd = sa + S::kA + dx * 3 * S::kBt;  // [dy0][dy2][dy1]
#pragma unroll
    for (int i = 0; i <= 2 * R; ++i) {
      const uint32_t a0 = sa + (uint32_t)(i * S::kRowStride + (7 + dx) * 16);
      const uint64_t da = ptx::smem_desc_noswz(a0, S::kChunkStride, 128);
      int col, n, slot;
      if (i & 1) {  // dy = 1 -> output row (i-1)/2
        col = (R - 1 - (i - 1) / 2) * BN;
        n = BN;
        slot = 2;
      } else if (i == 0) {  // dy = 0 only -> row 0
        col = (R - 1) * BN;
        n = BN;
        slot = 0;
      } else if (i == 2 * R) {  // dy = 2 only -> row R-1
        col = 0;
        n = BN;
        slot = 1;
      } else {  // dy = 0 -> row i/2 and dy = 2 -> row i/2 - 1 (adjacent, reverse order)
        col = (R - 1 - i / 2) * BN;
        n = 2 * BN;
        slot = 0;
      }
      const uint64_t db = ptx::smem_desc(sbd + slot * S::kBt, 8 * 32, 6u);
      if constexpr (F8)
        ptx::mma_f8_w(d_base + col, da, db, ptx::idesc_f8(128, n), 1u);
      else
        ptx::mma_f16_w(d_base + col, da, db, ptx::idesc_f16(128, n, BF), 1u);
    }
  }
}

template <typename T, int BN, int R, int STAGES>
__global__ void __launch_bounds__(384, 1)
    conv3s2_rc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, const ConvArgs args,
                      const __grid_constant__ LoMaps lo) {
  using S = S2Smem<BN, R, STAGES>;
  constexpr int CH = S::kCH;
  static_assert(2 * BN <= 256, "stacked N");
  static_assert(S::kTotal <= 227 * 1024, "shared memory");
  static_assert(2 * R * BN <= 512, "TMEM");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
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
      ptx::mbar_init(&tempty[a], 256);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<S::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int kiters = args.kchunks + args.kch_lo;
  constexpr uint32_t kTx = S::kABytes + 9 * BN * 32;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x) {
        const int nt = w % args.n_tiles_n;
        int m = w / args.n_tiles_n;
        const int tx = m % args.tiles_x;  // 128 input pixels -> 64 output pixels
        m /= args.tiles_x;
        const int tyg = m % args.tiles_y;
        const int b = m / args.tiles_y;
        const int u0 = tx * 16 - 1;
        const int y0 = 2 * tyg * R - 1;
        for (int kc = 0; kc < kiters; ++kc) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStage;
          const bool hi = kc < args.kchunks;
          const int kk = hi ? kc : kc - args.kchunks;
          ptx::mbar_arrive_expect_tx(&full[stage], kTx);
          ptx::tma_load_5d(sa, &tmA, &full[stage], 0, u0, 2 * kc, y0, b + args.b_in);
          (void)hi;
          (void)kk;
          ptx::bulk_load(sa + S::kA, args.wimg + ((size_t)nt * kiters + kc) * 9 * BN * 32, 9 * BN * 32, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr bool kBf = std::is_same<T, __nv_bfloat16>::value;
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    unsigned long long c_te = 0, c_full = 0, t_start = OS_CLK();
    for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
      const int acc = local & 1;
      unsigned long long t0 = OS_CLK();
      ptx::mbar_wait_backoff(&tempty[acc], (local >> 1) & 1);  // the epilogue zeroes and arrives up front
      c_te += OS_CLK() - t0;
      ptx::tc_fence_after();
      const uint32_t d_base = tmem_base + acc * R * BN;
      for (int kc = 0; kc < kiters; ++kc) {
        t0 = OS_CLK();
        ptx::mbar_wait(&full[stage], phase);
        c_full += OS_CLK() - t0;
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(smem + stage * S::kStage);
        if (kc >= args.kchunks)
          s2_mma_chunk<BN, R, true, kBf, S>(sa, d_base);
        else
          s2_mma_chunk<BN, R, false, kBf, S>(sa, d_base);
        ptx::mma_commit_w(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      ptx::mma_commit_w(&tfull[acc]);
    }
    if (OS_EXP && (args.dbg & 8) && lane == 0) {
      args.dbg_out[blockIdx.x * 4 + 0] = OS_CLK() - t_start;
      args.dbg_out[blockIdx.x * 4 + 1] = c_te;
      args.dbg_out[blockIdx.x * 4 + 2] = c_full;
      args.dbg_out[blockIdx.x * 4 + 3] = local;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue: even TMEM lanes are outputs
    // 8 warps: a pair per TMEM lane quadrant, alternating output rows. Each output pixel's
    // CH = 32 channels are shared by its lane pair: the even lane (which holds the pixel in
    // TMEM) keeps channels 0-15, the odd lane takes 16-31 through a shuffle, so all 32 lanes
    // convert and store. Output staging double-buffered (two (hi, lo) sets per warp).
    const int q = warp & 3, ew = warp - 4, half = ew >> 2;
    uint8_t* obase = smem + S::kEpiOff + ew * 4 * S::kEpiBuf;
    int oslot = 0;
    const int px = (int)lane >> 1;  // output pixel within the warp's 16
    const bool odd = (lane & 1) != 0;
    constexpr bool kPair = CH == 32;  // lane-pair channel split
    constexpr int CW = kPair ? 16 : CH;  // channels converted by one lane
    const int cb = (kPair && odd) ? 16 : 0;
    const int rc = args.out_rc;
    // NHWC box images: 16 rows of CH*2 bytes, 64-B (CH = 32) / 32-B swizzle; RC: [chunk][16 px][16 B]
    auto o16 = [&](int j16) { return rc ? (uint32_t)(j16 * 256 + px * 16) : EpiTile<CH>::off(px, j16); };
    auto o8 = [&](int j8) { return rc ? (uint32_t)(j8 * 256 + px * 16) : lo_off<CH>(px, j8); };
    {
      const int c0 = half * (R * BN), c1 = c0 + R * BN;  // the pair splits the zeroing of both buffers
      for (int c = c0; c < c1; c += 16) ptx::tmem_st_zero16(tmem_base + ((uint32_t)(q * 32) << 16) + c);
    }
    ptx::tmem_st_wait();
    ptx::tc_fence_before();
    ptx::mbar_arrive(&tempty[0]);
    ptx::mbar_arrive(&tempty[1]);
    int local = 0;
    for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
      const int acc = local & 1;
      const int nt = w % args.n_tiles_n;
      int m = w / args.n_tiles_n;
      const int tx = m % args.tiles_x;
      m /= args.tiles_x;
      const int tyg = m % args.tiles_y;
      const int b = m / args.tiles_y;
      ptx::mbar_wait_backoff(&tfull[acc], (local >> 1) & 1);
      ptx::tc_fence_after();
      const int xo = tx * 64 + q * 16;
#pragma unroll 1
      for (int i = 0; i < (R / 2) * (BN / CH); ++i) {
        const int r = (i / (BN / CH)) * 2 + half, c = (i % (BN / CH)) * CH;
        const int n0 = nt * BN + c;
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN + (R - 1 - r) * BN + c;
        uint32_t u[32];
        if constexpr (CH == 32) {
          ptx::tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(u));
        } else {
          ptx::tmem_ld_32x32b_x16(taddr, *reinterpret_cast<uint32_t(*)[16]>(u));
        }
        ptx::tmem_ld_wait();
        float v[CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          float x0 = fmaxf(__uint_as_float(u[j]) + __ldg(args.bias + n0 + j), 0.0f);
          if constexpr (kPair) {
            const float x1 = fmaxf(__uint_as_float(u[16 + j]) + __ldg(args.bias + n0 + 16 + j), 0.0f);
            const float from_even = __shfl_sync(0xffffffffu, x1, (int)lane ^ 1);
            x0 = odd ? from_even : x0;
          }
          v[j] = x0;
        }
        uint8_t* o_hi = obase + oslot * 2 * S::kEpiBuf;
        uint8_t* o_lo = o_hi + S::kEpiBuf;
        oslot ^= 1;
        if (lane == 0) ptx::bulk_wait_read1();  // the store that last used this slot has read it
        __syncwarp();
        if (!kPair && odd) {
          // without the pair split only the even lanes hold output pixels
        } else if (args.split == kStoreF8) {
#pragma unroll
          for (int j = 0; j < CW / 16; ++j) {
            uint4 h0, h1, l4;
            split_f8_16(v + 16 * j, h0, h1, l4);
            *reinterpret_cast<uint4*>(o_hi + o16(cb / 8 + 2 * j)) = h0;
            *reinterpret_cast<uint4*>(o_hi + o16(cb / 8 + 2 * j + 1)) = h1;
            *reinterpret_cast<uint4*>(o_lo + o8(cb / 16 + j)) = l4;
          }
        } else {
#pragma unroll
          for (int j = 0; j < CW / 8; ++j) {
            uint32_t o[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              o[e] = StoreT<T>::pack(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
              const float2 hv = StoreT<T>::unpack(o[e]);
              l[e] = StoreT<T>::pack(v[8 * j + 2 * e] - hv.x, v[8 * j + 2 * e + 1] - hv.y);
            }
            *reinterpret_cast<uint4*>(o_hi + o16(cb / 8 + j)) = make_uint4(o[0], o[1], o[2], o[3]);
            if (args.split) *reinterpret_cast<uint4*>(o_lo + o16(cb / 8 + j)) = make_uint4(l[0], l[1], l[2], l[3]);
          }
        }
        ptx::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          const int y = tyg * R + r, bo = b + args.b_out;
          if (rc) {
            ptx::tma_store_5d(&tmO, o_hi, 0, xo / 8, n0 / 8, y, bo);
            if (args.split == kStoreF8)
              ptx::tma_store_5d(&lo.O, o_lo, 0, xo / 8, args.Cout / 8 + n0 / 16, y, bo);
            else if (args.split)
              ptx::tma_store_5d(&tmO, o_lo, 0, xo / 8, args.Cout / 8 + n0 / 8, y, bo);
          } else {
            ptx::tma_store_4d(&tmO, o_hi, n0, xo, y, bo);
            if (args.split == kStoreF8)
              ptx::tma_store_4d(&lo.O, o_lo, n0, xo, y, bo);
            else if (args.split)
              ptx::tma_store_4d(&tmO, o_lo, args.Cout + n0, xo, y, bo);
          }
          ptx::bulk_commit();
        }
      }
      for (int j = 0; j < R / 2; ++j) {
        const int r = j * 2 + half;
        for (int c = 0; c < BN; c += 16)
          ptx::tmem_st_zero16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN + (R - 1 - r) * BN + c);
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<S::kTmemCols>(tmem_base);
  }
}

}  // namespace osg

namespace osg {

// ---------------------------------------------------------------------------------------
// Fused window gather + stem conv (A5 + the first A6 layer). For each kept window of the
// batch, the 3x3x3 stem is a K = 27 (padded to 32) GEMM over an im2col operand that four
// converter warps build directly in shared memory from the RGBX level image of the window's
// scale (L_f, padded frame; the window's zero 'same' padding applied by masking), so the
// 64-B/px im2col tensor of a separate gather kernel never touches HBM. Work item = R output
// rows x 128 pixels of one window; per row two K = 16 MMAs (M = 128, N = BN). Epilogue: the
// 8-warp TMA epilogue of the convs (bias, ReLU, storage split, row-chunked / NHWC store).
struct StemArgs {
  const uint32_t* tiles;   // kept-window ids (pack_tile), batch b = tiles[first + b]
  const uint32_t* L[4];    // RGBX u32 padded-frame levels f = 1, 2, 4, 8 (row length Wp / f)
  const float* bias;
  const void* w;           // [BN][32] 16-bit stem weights, K = (dy*3 + dx)*3 + c
  int first, P, S, Hp, Wp;
  int num_work, tiles_x, tiles_y;
  int split, out_rc, Cout, b_out;
  unsigned long long* dbg_out;  // experiments (OMNISEG_DBG & 8): MMA-warp cycle counters
};

// TMA maps of the four RGBX levels (u32 elements, dims {Wp/f, Hp/f}, box {kStemBoxW, R + 2}):
// the stem's input ring is filled by TMA (window halo included, image-edge OOB -> 0).
struct StemInMaps {
  CUtensorMap m[4];
};
// 136 pixels: the 128-pixel tile + the 3x3 halo, started 4 pixels early -- a tiled TMA box must
// start 16-byte aligned in its innermost dimension (measured: a start at -1 faults with an
// illegal instruction, scripts/micro/tma_u32_box.cu), so the box covers [x0 - 4, x0 + 132)
constexpr int kStemBoxW = 136;

template <int BN, int R, int NA>
struct StemSmem {
  // K = 48: the 3x3 window's 9 pixels x RGBX (k = (dy*3 + dx)*4 + c, X and k >= 36 weighted 0),
  // so one RGBX word of the level image becomes two fp16 pairs by byte permutes
  static constexpr int kKC = 6;                  // 16-byte K chunks
  static constexpr int kA = kKC * 128 * 16;      // one row: [kc][128 px][16 B]
  static constexpr int kB = kKC * BN * 16;       // [kc][BN][16 B]
  static constexpr int kCH = BN < 32 ? BN : 32;  // output box width (make_stem_plan's maps)
  static constexpr int kBOff = NA * kA;
  // TMA input ring: kNI items of (R + 2) rows x kStemBoxW RGBX words
  static constexpr int kNI = 6;
  static constexpr int kIn = (((R + 2) * kStemBoxW * 4) + 127) / 128 * 128;
  static constexpr int kInOff = ((kBOff + kB + 127) / 128) * 128;
  static constexpr int kBarOff = ((kInOff + kNI * kIn + 1023) / 1024) * 1024;
  // epilogue warps: 16 for 32 channels (one output row each per 4-row item), else 8
  static constexpr int kEW = (BN == 32 && R == 4) ? 16 : 8;
  static constexpr int kThreads = 256 + 32 * kEW;
  static constexpr int kBars = (2 * NA + 2 * kNI + 4 + 2 * kEW) * 8 + 16;
  static constexpr int kEpiOff = ((kBarOff + kBars + 1023) / 1024) * 1024;
  static constexpr int kTotal = kEpiOff + kEW * 3 * EpiTile<kCH>::kBuf + 1024;
  static constexpr uint32_t kTmemCols = (2 * R * BN <= 32) ? 32 : (2 * R * BN <= 64) ? 64 : (2 * R * BN <= 128) ? 128
                                        : (2 * R * BN <= 256) ? 256 : 512;
};

template <typename T, int BN, int R, int NA>
__global__ void __launch_bounds__(StemSmem<BN, R, NA>::kThreads, 1)
    stem_tc_kernel(const __grid_constant__ CUtensorMap tmO, const __grid_constant__ StemArgs args,
                   const __grid_constant__ LoMaps lo, const __grid_constant__ CUtensorMap in0,
                   const __grid_constant__ CUtensorMap in1, const __grid_constant__ CUtensorMap in2,
                   const __grid_constant__ CUtensorMap in3) {
  using S = StemSmem<BN, R, NA>;
  constexpr int CH = S::kCH;
  static_assert(S::kTotal <= 227 * 1024, "shared memory");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* afull = reinterpret_cast<uint64_t*>(smem + S::kBarOff);
  uint64_t* aempty = afull + NA;
  uint64_t* tfull = aempty + NA;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;  // unused by the output-only epilogue (EpiState needs the slots)
  uint64_t* infull = rbar + 2 * S::kEW;
  uint64_t* inempty = infull + S::kNI;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(inempty + S::kNI);
  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < NA; ++i) {
      ptx::mbar_init(&afull[i], 128);
      ptx::mbar_init(&aempty[i], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 32 * S::kEW);
    }
    for (int a = 0; a < 2 * S::kEW; ++a) ptx::mbar_init(&rbar[a], 1);
    for (int i = 0; i < S::kNI; ++i) {
      ptx::mbar_init(&infull[i], 1);
      ptx::mbar_init(&inempty[i], 4);  // one arrival per converter warp
    }
    ptx::fence_barrier_init();
  }
  // weights -> smem B operand (no-swizzle K-major: [kc][n][8 x 16-bit])
  if (tid < 128) {
    const uint4* wsrc = static_cast<const uint4*>(args.w);
    for (int i = tid; i < BN * S::kKC; i += 128) {
      const int n = i / S::kKC, kc = i % S::kKC;
      *reinterpret_cast<uint4*>(smem + S::kBOff + kc * BN * 16 + n * 16) = wsrc[n * S::kKC + kc];
    }
    ptx::fence_proxy_async();
  }
  if (warp == 5) ptx::tmem_alloc<S::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------ im2col converters: thread = output pixel
    // The (R+2) x 130 RGBX neighbourhood of the item arrives in the TMA input ring (producer:
    // warp 6, kNI items ahead); each thread reads its (R+2) x 3 words from shared memory,
    // applies the window's zero padding and releases the slot.
    const int px = tid;
    int stage = 0;
    uint32_t phase = 0;
    int istage = 0;
    uint32_t iphase = 0;
    for (int w = blockIdx.x; w < args.num_work; w += gridDim.x) {
      const int tx = w % args.tiles_x;
      const int tyg = (w / args.tiles_x) % args.tiles_y;
      const int x = tx * 128 + px;  // window column
      const int y0 = tyg * R;
      uint32_t win[R + 2][3];
      ptx::mbar_wait(&infull[istage], iphase);
      const uint32_t* in = reinterpret_cast<const uint32_t*>(smem + S::kInOff + istage * S::kIn);
#pragma unroll
      for (int i = 0; i < R + 2; ++i) {
        const int yy = y0 + i - 1;
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int xx = x + dx - 1;
          const uint32_t v = in[i * kStemBoxW + px + dx + 3];  // box column 0 = window column x0 - 4
          win[i][dx] = (yy >= 0 && yy < args.P && xx >= 0 && xx < args.P) ? v : 0u;  // window zero padding
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&inempty[istage]);
      if (++istage == S::kNI) {
        istage = 0;
        iphase ^= 1;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ptx::mbar_wait(&aempty[stage], phase ^ 1);
        uint8_t* a = smem + stage * S::kA;
        uint32_t o[24];  // 48 16-bit K values: pixel p -> o[2p] = (R, G), o[2p+1] = (B, X)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
            const uint32_t q = win[r + dy][dx];
            const int p2 = (dy * 3 + dx) * 2;
            if constexpr (std::is_same<T, __half>::value) {
              // byte b -> fp16 bits 0x6400 | b = 1024 + b (exact), minus 1024 in one packed op
              o[p2] = ptx::hsub2_u32(__byte_perm(q, 0x64646464u, 0x4140), 0x64006400u);
              o[p2 + 1] = ptx::hsub2_u32(__byte_perm(q, 0x64646464u, 0x4342), 0x64006400u);
            } else {
              o[p2] = StoreT<T>::pack(float(q & 255), float((q >> 8) & 255));
              o[p2 + 1] = StoreT<T>::pack(float((q >> 16) & 255), float(q >> 24));
            }
          }
#pragma unroll
        for (int k = 18; k < 24; ++k) o[k] = 0u;
#pragma unroll
        for (int kc = 0; kc < S::kKC; ++kc)
          *reinterpret_cast<uint4*>(a + kc * 2048 + px * 16) =
              make_uint4(o[4 * kc], o[4 * kc + 1], o[4 * kc + 2], o[4 * kc + 3]);
        ptx::fence_proxy_async();  // generic-proxy smem writes -> visible to tcgen05.mma
        ptx::mbar_arrive(&afull[stage]);
        if (++stage == NA) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 6) {
    // ------------------------------------------ TMA producer of the input ring
    if (lane == 0) {
      int istage = 0;
      uint32_t iphase = 0;
      constexpr uint32_t kTx = (R + 2) * kStemBoxW * 4;
      for (int w = blockIdx.x; w < args.num_work; w += gridDim.x) {
        const int tx = w % args.tiles_x;
        int m = w / args.tiles_x;
        const int tyg = m % args.tiles_y;
        const int b = m / args.tiles_y;
        const uint32_t id = __ldg(args.tiles + args.first + b);
        const int lf = id >> 30, f = 1 << lf;
        const int oy = min((int)((id >> 15) & 0x7FFF) * args.S, args.Hp / f - args.P);
        const int ox = min((int)(id & 0x7FFF) * args.S, args.Wp / f - args.P);
        ptx::mbar_wait(&inempty[istage], iphase ^ 1);
        ptx::mbar_arrive_expect_tx(&infull[istage], kTx);
        // static addresses of the __grid_constant__ maps (a dynamic index would copy the
        // parameter struct to local memory, where TMA cannot read a tensor map)
        const CUtensorMap* mp = lf == 0 ? &in0 : lf == 1 ? &in1 : lf == 2 ? &in2 : &in3;
        ptx::tma_load_2d(smem + S::kInOff + istage * S::kIn, mp, &infull[istage], ox + tx * 128 - 4, oy + tyg * R - 1);
        if (++istage == S::kNI) {
          istage = 0;
          iphase ^= 1;
        }
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------ MMA issuer (warp-collective)
    constexpr bool kBf = std::is_same<T, __nv_bfloat16>::value;
    constexpr uint32_t idesc = ptx::idesc_f16(128, BN, kBf);
    const uint32_t sb = ptx::smem_u32(smem + S::kBOff);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    unsigned long long c_te = 0, c_full = 0, t_start = OS_CLK();
    for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
      const int acc = local & 1;
      unsigned long long t0 = OS_CLK();
      ptx::mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
      c_te += OS_CLK() - t0;
      ptx::tc_fence_after();
      for (int r = 0; r < R; ++r) {
        t0 = OS_CLK();
        ptx::mbar_wait(&afull[stage], phase);
        c_full += OS_CLK() - t0;
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(smem + stage * S::kA);
        const uint32_t d = tmem_base + acc * R * BN + r * BN;
#pragma unroll
        for (int ks = 0; ks < S::kKC / 2; ++ks) {
          const uint64_t da = ptx::smem_desc_noswz(sa + ks * 2 * 2048, 2048, 128);
          const uint64_t db = ptx::smem_desc_noswz(sb + ks * 2 * BN * 16, BN * 16, 128);
          ptx::mma_f16_w(d, da, db, idesc, ks);
        }
        ptx::mma_commit_w(&aempty[stage]);
        if (++stage == NA) {
          stage = 0;
          phase ^= 1;
        }
      }
      ptx::mma_commit_w(&tfull[acc]);
    }
    if (OS_EXP && args.dbg_out && lane == 0) {
      args.dbg_out[blockIdx.x * 4 + 0] = OS_CLK() - t_start;
      args.dbg_out[blockIdx.x * 4 + 1] = c_te;
      args.dbg_out[blockIdx.x * 4 + 2] = c_full;
      args.dbg_out[blockIdx.x * 4 + 3] = local;
    }
  } else if (warp >= 8) {
    // ------------------------------------------ epilogue (kEW warps: 8 -> rows alternate per
    // pair of warps on a TMEM lane quadrant; 16 -> one row per warp)
    const int q = warp & 3, ew = warp - 8, half = ew >> 2;
    EpiState es{smem + S::kEpiOff + ew * 3 * EpiTile<CH>::kBuf, &rbar[2 * ew], {0, 0}, 0, 0, args.out_rc};
    epi_layout<CH>(es, args.split);
    float bias_r[S::kEW == 16 ? 1 : CH];  // 16 warps: the bias is read (L1-resident) per row
    if constexpr (S::kEW != 16) {
#pragma unroll
      for (int j = 0; j < CH; ++j) bias_r[j] = __ldg(args.bias + j);
    }
    int local = 0;
    // F8 storage (the product dtype) runs a copy of the item loop with the kind known at compile time
    auto items = [&](auto f8_tag) {
    constexpr int SK = decltype(f8_tag)::value ? (int)kStoreF8 : -1;
    for (int w = blockIdx.x; w < args.num_work; w += gridDim.x, ++local) {
      const int acc = local & 1;
      int tx, m, tyg, b;
      udivmod(w, args.tiles_x, m, tx);
      udivmod(m, args.tiles_y, b, tyg);
      ptx::mbar_wait_backoff(&tfull[acc], (local >> 1) & 1);
      ptx::tc_fence_after();
      const int xb = tx * 128 + q * 32;
      if constexpr (S::kEW == 16) {
        uint32_t u[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN + half * BN, u);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);  // the accumulator row is in registers
        float v[CH];
        const float4* b4 = reinterpret_cast<const float4*>(args.bias);
#pragma unroll
        for (int j = 0; j < CH; j += 4) {
          const float4 bb = __ldg(b4 + j / 4);
          const float2 t0 = __fadd2_rn(make_float2(__uint_as_float(u[j]), __uint_as_float(u[j + 1])),
                                       make_float2(bb.x, bb.y));
          const float2 t1 = __fadd2_rn(make_float2(__uint_as_float(u[j + 2]), __uint_as_float(u[j + 3])),
                                       make_float2(bb.z, bb.w));
          v[j] = fmaxf(t0.x, 0.f);
          v[j + 1] = fmaxf(t0.y, 0.f);
          v[j + 2] = fmaxf(t1.x, 0.f);
          v[j + 3] = fmaxf(t1.y, 0.f);
        }
        epi_store<T, CH, SK>(es, &tmO, &lo.O, v, 0, args.Cout, args.split, xb, tyg * R + half, b + args.b_out, lane);
        continue;
      } else if constexpr (BN == CH && CH == 32) {
        // one 32-channel chunk per row: bias held in registers, the next row's accumulator
        // loaded from TMEM while this row is converted and stored
        constexpr int NI = R / 2;
        uint32_t u[2][32];
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN;
        ptx::tmem_ld_32x32b_x32(tb + half * BN, u[0]);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          if (i + 1 < NI) ptx::tmem_ld_32x32b_x32(tb + ((i + 1) * 2 + half) * BN, u[(i + 1) & 1]);
          float v[CH];
#pragma unroll
          for (int j = 0; j < CH; j += 2) {
            const float2 t2 = __fadd2_rn(make_float2(__uint_as_float(u[i & 1][j]), __uint_as_float(u[i & 1][j + 1])),
                                         make_float2(bias_r[j], bias_r[j + 1]));
            v[j] = fmaxf(t2.x, 0.f);
            v[j + 1] = fmaxf(t2.y, 0.f);
          }
          epi_store<T, CH, SK>(es, &tmO, &lo.O, v, 0, args.Cout, args.split, xb, tyg * R + i * 2 + half,
                               b + args.b_out, lane);
          ptx::tmem_ld_wait();
        }
      } else {
#pragma unroll 1
        for (int i = 0; i < (R / 2) * (BN / CH); ++i) {
          const int r = (i / (BN / CH)) * 2 + half, c = (i % (BN / CH)) * CH;
          const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * R * BN + r * BN + c;
          epi_chunk<T, CH, kReluBias, SK>(es, 0, &tmO, &lo.O, taddr, args.bias, c, args.Cout, args.split, xb,
                                          tyg * R + r, b + args.b_out, lane);
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
    };
    if (args.split == kStoreF8)
      items(std::true_type{});
    else
      items(std::false_type{});
    if (lane == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<S::kTmemCols>(tmem_base);
  }
}

}  // namespace osg
