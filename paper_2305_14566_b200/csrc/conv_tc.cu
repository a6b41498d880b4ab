// conv_tc.cu -- host side of the tcgen05 implicit-GEMM convolution: TMA tensor maps,
// tile-shape selection, template dispatch and the persistent launch.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <unordered_set>
#include <type_traits>

#include "common.cuh"
#include "conv_plan.h"
#include "conv_tc.cuh"

namespace osg {

namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw Error(-2, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  return fn;
}

CUtensorMapSwizzle swz(int bytes) {
  return bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
}

template <typename T, int BN, int BK>
struct Cfg {
  static constexpr int kStageBytes = ConvSmem<BN, BK, 1>::kStage;
  static constexpr int kStages0 = kStageBudgetTap / kStageBytes;
  static constexpr int STAGES = kStages0 > 8 ? 8 : (kStages0 < 2 ? 2 : kStages0);
  using Smem = ConvSmem<BN, BK, STAGES>;
};

template <typename T, int BN, int BK>
void launch_tpl(const ConvPlan& p, cudaStream_t s) {
  using C = Cfg<T, BN, BK>;
  constexpr int smem = C::Smem::kTotal;
  auto launch_mode = [&](auto kern) {
    // all instantiations share one function-pointer type: remember each kernel separately
    static std::mutex mu;
    static std::unordered_set<const void*> done;
    {
      std::lock_guard<std::mutex> g(mu);
      if (done.insert(reinterpret_cast<const void*>(kern)).second)
        OS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    kern<<<p.grid, 256, smem, s>>>(p.tmA, p.tmB, p.tmO, p.tmR, p.args);
  };
  switch (p.mode) {
    case kReluBias: launch_mode(conv_tc_kernel<T, BN, BK, C::STAGES, kReluBias>); break;
    case kResidualRelu: launch_mode(conv_tc_kernel<T, BN, BK, C::STAGES, kResidualRelu>); break;
    case kUpAdd: launch_mode(conv_tc_kernel<T, BN, BK, C::STAGES, kUpAdd>); break;
    default: launch_mode(conv_tc_kernel<T, BN, BK, C::STAGES, kBias>); break;
  }
}

template <typename T, int BN, int HB>
void launch_rows(const ConvPlan& p, cudaStream_t s) {
  constexpr int R = RowsCfg::R(BN);
  constexpr int BK = RowsCfg::BK(BN, HB);
  constexpr int ST = RowsCfg::STAGES(BN, HB);
  static_assert(ST >= 2, "multi-row tile does not fit shared memory");
  constexpr int smem = RowsSmem<BN, BK, R, R * HB + 2, 128 / HB, ST>::kTotal;
  auto go = [&](auto kern) {
    static std::mutex mu;
    static std::unordered_set<const void*> done;
    {
      std::lock_guard<std::mutex> g(mu);
      if (done.insert(reinterpret_cast<const void*>(kern)).second)
        OS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    kern<<<p.grid, 256, smem, s>>>(p.tmA, p.tmB, p.tmO, p.tmR, p.args);
  };
  switch (p.mode) {
    case kReluBias: go(conv3_rows_kernel<T, BN, BK, R, HB, ST, kReluBias>); break;
    case kResidualRelu: go(conv3_rows_kernel<T, BN, BK, R, HB, ST, kResidualRelu>); break;
    default: go(conv3_rows_kernel<T, BN, BK, R, HB, ST, kBias>); break;
  }
}

template <typename T, int BN, bool DYF>
void launch_nz(const ConvPlan& p, cudaStream_t s) {
  constexpr int R = NzCfg::R(BN);
  constexpr int ST = NzCfg::STAGES(BN, 4, false);   // plain epilogue (4 warps)
  constexpr int STR = NzCfg::STAGES(BN, 8, false);  // residual epilogue (8 warps)
  constexpr int STH = NzCfg::STAGES(BN, 8, true);   // fused head (8 warps, residual slots only)
  static_assert(ST >= 2 && STR >= 2 && STH >= 2, "no-swizzle tile does not fit shared memory");
  int smem = NzSmem<BN, R, ST, DYF, 4, false>::kTotal, threads = 256;
  if (p.mode == kResidualRelu) {
    smem = NzSmem<BN, R, STR, DYF, 8, false>::kTotal;
    threads = 384;
  } else if (p.mode == kHeadFused) {
    smem = NzSmem<BN, R, STH, DYF, 8, true>::kTotal;
    threads = 384;
  }
  auto go = [&](auto kern) {
    static std::mutex mu;
    static std::unordered_set<const void*> done;
    {
      std::lock_guard<std::mutex> g(mu);
      if (done.insert(reinterpret_cast<const void*>(kern)).second)
        OS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    kern<<<p.grid, threads, smem, s>>>(p.tmA, p.tmB, p.tmO, p.tmR, p.args, p.head);
  };
  switch (p.mode) {
    case kReluBias: go(conv3_nz_kernel<T, BN, R, ST, kReluBias, DYF>); break;
    case kResidualRelu: go(conv3_nz_kernel<T, BN, R, STR, kResidualRelu, DYF>); break;
    case kHeadFused: go(conv3_nz_kernel<T, BN, R, STH, kHeadFused, DYF>); break;
    default: go(conv3_nz_kernel<T, BN, R, ST, kBias, DYF>); break;
  }
}

template <typename T>
void dispatch(const ConvPlan& p, cudaStream_t s) {
  if (p.mode == kHeadFused && p.nz_R == 0) throw Error(-1, "fused head needs the no-swizzle conv kernel");
  if (p.nz_R > 0) {
    static const bool dyf = getenv("OMNISEG_NO_DYF") == nullptr;
    if (p.bn == 16) return dyf ? launch_nz<T, 16, true>(p, s) : launch_nz<T, 16, false>(p, s);
    if (p.bn == 32) return dyf ? launch_nz<T, 32, true>(p, s) : launch_nz<T, 32, false>(p, s);
    if (p.bn == 64) return dyf ? launch_nz<T, 64, true>(p, s) : launch_nz<T, 64, false>(p, s);
    throw Error(-1, "unsupported no-swizzle conv shape");
  }
  if (p.rows_R > 0) {
#define OS_RCASE(N_, H_) \
  if (p.bn == N_ && p.hb == H_) return launch_rows<T, N_, H_>(p, s);
    OS_RCASE(16, 1) OS_RCASE(32, 1) OS_RCASE(64, 1) OS_RCASE(128, 1)
    OS_RCASE(16, 2) OS_RCASE(32, 2) OS_RCASE(64, 2) OS_RCASE(128, 2)
#undef OS_RCASE
    throw Error(-1, "unsupported multi-row conv shape");
  }
#define OS_CASE(N_, K_) \
  if (p.bn == N_ && p.bk == K_) return launch_tpl<T, N_, K_>(p, s);
  OS_CASE(16, 16) OS_CASE(16, 32) OS_CASE(16, 64)
  OS_CASE(32, 16) OS_CASE(32, 32) OS_CASE(32, 64)
  OS_CASE(64, 16) OS_CASE(64, 32) OS_CASE(64, 64)
  OS_CASE(128, 16) OS_CASE(128, 32) OS_CASE(128, 64)
  OS_CASE(256, 16) OS_CASE(256, 32) OS_CASE(256, 64)
#undef OS_CASE
  throw Error(-1, "unsupported conv tile shape");
}

int stages_for(int bn, int bk) {
  const int a = 128 * bk * 2, b = ((bn * bk * 2 + 1023) / 1024) * 1024;
  int st = kStageBudgetTap / (a + b);
  return st > 8 ? 8 : (st < 2 ? 2 : st);
}
}  // namespace

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    OS_CUDA(cudaGetDevice(&dev));
    OS_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

ConvPlan make_conv_plan(bool bf16, const void* in, int B, int Hin, int Win, int Cin, const void* w,
                        const float* bias, int Cout, int k, int stride, int mode, const void* res, void* out,
                        bool split_out, int B_in, int B_res, int B_out) {
  if (B_in < 0) B_in = B;
  if (B_res < 0) B_res = B;
  if (B_out < 0) B_out = B;
  OS_REQUIRE(Cin % 16 == 0 && Cout % 16 == 0, "conv channels must be multiples of 16");
  OS_REQUIRE(k == 1 || k == 3, "conv kernel size must be 1 or 3");
  OS_REQUIRE(stride == 1 || stride == 2, "conv stride must be 1 or 2");
  ConvPlan p{};
  p.mode = mode;
  p.bf16 = bf16;
  // K chunk = one swizzle row (128/64/32 bytes); N tile = largest power of two <= 256 dividing Cout
  p.bk = Cin % 64 == 0 ? 64 : Cin % 32 == 0 ? 32 : 16;
  p.bn = 256;
  while (Cout % p.bn) p.bn >>= 1;
  const int Ho = (Hin - 1) / stride + 1, Wo = (Win - 1) / stride + 1;
  ConvArgs& a = p.args;
  a.B = B;
  a.Ho = Ho;
  a.Wo = Wo;
  a.Cin = Cin;
  a.Cout = Cout;
  a.ksize = k;
  a.stride = stride;
  if (Wo >= 128) {
    OS_REQUIRE(Wo % 128 == 0, "output width must be a multiple of 128 or divide 128");
    a.wb = 128;
    a.hb = 1;
  } else {
    OS_REQUIRE(128 % Wo == 0, "output width must divide 128");
    a.wb = Wo;
    a.hb = 128 / Wo;
    OS_REQUIRE(Ho % a.hb == 0, "output height incompatible with the 128-pixel M tile");
  }
  a.tiles_x = Wo / a.wb;
  a.tiles_y = Ho / a.hb;
  a.n_tiles_n = Cout / p.bn;
  a.kchunks = Cin / p.bk;
  // no-swizzle multi-row variant (conv3_nz_kernel): 3x3 stride 1, width >= 128, N <= 64
  if (k == 3 && stride == 1 && mode != kUpAdd && p.bn <= 64 && a.hb == 1 && Cout == p.bn && Cin % 16 == 0 &&
      a.tiles_y % NzCfg::R(p.bn) == 0 && getenv("OMNISEG_NO_NZ") == nullptr) {
    const int R = NzCfg::R(p.bn);
    // A: 5-D view {8 ch, W, H, Cin/8, B} with the chunk dimension (16-B stride) outside the
    // pixel dimensions, box {8, 130, R+2, 2, 1} -> smem [chunk][row][px][16 B]
    cuuint64_t dims[5] = {8, (cuuint64_t)Win, (cuuint64_t)Hin, (cuuint64_t)(Cin / 8), (cuuint64_t)B_in};
    cuuint64_t strides[4] = {(cuuint64_t)Cin * 2, (cuuint64_t)Win * Cin * 2, 16, (cuuint64_t)Hin * Win * Cin * 2};
    cuuint32_t box[5] = {8, 130, (cuuint32_t)(R + 2), 2, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    const CUtensorMapDataType dt0 = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUresult r = encode_fn()(&p.tmA, dt0, 5, const_cast<void*>(in), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) {
      p.nz_R = R;
      p.bk = 16;
      a.kchunks = Cin / 16;
      a.tiles_y /= R;
    }
  }
  // multi-row variant for 3x3 stride-1 convs with N <= 128 (see conv3_rows_kernel)
  if (p.nz_R == 0 && k == 3 && stride == 1 && mode != kUpAdd && p.bn <= 128 && (a.hb == 1 || a.hb == 2) &&
      Cout == p.bn && getenv("OMNISEG_NO_ROWS") == nullptr) {
    const int R = RowsCfg::R(p.bn);
    const int bk = RowsCfg::BK(p.bn, a.hb);
    if (a.tiles_y % R == 0 && Cin % bk == 0) {
      p.rows_R = R;
      p.hb = a.hb;
      p.bk = bk;
      a.kchunks = Cin / bk;
      a.tiles_y /= R;
    }
  }
  a.num_work = B * a.tiles_x * a.tiles_y * a.n_tiles_n;
  a.bias = bias;
  a.res = res;
  a.out = out;
  a.split = split_out ? 1 : 0;
  const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  if (p.nz_R == 0) {
    cuuint64_t dims[4] = {(cuuint64_t)Cin, (cuuint64_t)Win, (cuuint64_t)Hin, (cuuint64_t)B_in};
    cuuint64_t strides[3] = {(cuuint64_t)Cin * 2, (cuuint64_t)Win * Cin * 2, (cuuint64_t)Hin * Win * Cin * 2};
    cuuint32_t box[4] = {(cuuint32_t)p.bk, (cuuint32_t)(a.wb * stride), (cuuint32_t)(a.hb * stride), 1};
    if (p.rows_R > 0) box[2] = (cuuint32_t)(p.rows_R * a.hb + 2);
    cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
    CUresult r = encode_fn()(&p.tmA, dt, 4, const_cast<void*>(in), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, swz(p.bk * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(A) failed: " + std::to_string((int)r));
  }
  {
    const int taps = k * k;
    cuuint64_t dims[2] = {(cuuint64_t)taps * Cin, (cuuint64_t)Cout};
    cuuint64_t strides[1] = {(cuuint64_t)taps * Cin * 2};
    cuuint32_t box[2] = {(cuuint32_t)p.bk, (cuuint32_t)p.bn};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&p.tmB, dt, 2, const_cast<void*>(w), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, swz(p.bk * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(B) failed: " + std::to_string((int)r));
  }
  {
    // output / residual maps for the TMA epilogue: [B][Ho][Wo][Cst], one warp box
    // = CH channels x (bw x bh) pixels, 64-B (CH=32) / 32-B (CH=16) swizzle
    const int CH = p.bn < 32 ? p.bn : 32;
    const int Cst = split_out ? 2 * Cout : Cout;
    const int bw = a.wb < 32 ? a.wb : 32, bh = 32 / bw;
    cuuint64_t dims[4] = {(cuuint64_t)Cst, (cuuint64_t)Wo, (cuuint64_t)Ho, (cuuint64_t)B_out};
    cuuint64_t dims_r[4] = {(cuuint64_t)Cst, (cuuint64_t)Wo, (cuuint64_t)Ho, (cuuint64_t)B_res};
    cuuint64_t strides[3] = {(cuuint64_t)Cst * 2, (cuuint64_t)Wo * Cst * 2, (cuuint64_t)Ho * Wo * Cst * 2};
    cuuint32_t box[4] = {(cuuint32_t)CH, (cuuint32_t)bw, (cuuint32_t)bh, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle sw = CH == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    if (mode == kUpAdd && a.wb >= 32) {
      // up-add: full-resolution skip / output, one box = 64 output pixels of one row
      cuuint64_t d2[4] = {(cuuint64_t)Cst, (cuuint64_t)(2 * Wo), (cuuint64_t)(2 * Ho), (cuuint64_t)B_out};
      cuuint64_t d2r[4] = {(cuuint64_t)Cst, (cuuint64_t)(2 * Wo), (cuuint64_t)(2 * Ho), (cuuint64_t)B_res};
      cuuint64_t st2[3] = {(cuuint64_t)Cst * 2, (cuuint64_t)2 * Wo * Cst * 2, (cuuint64_t)4 * Ho * Wo * Cst * 2};
      cuuint32_t bx2[4] = {(cuuint32_t)CH, 64, 1, 1};
      CUresult r = encode_fn()(&p.tmO, dt, 4, out, d2, st2, bx2, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(up out) failed: " + std::to_string((int)r));
      r = encode_fn()(&p.tmR, dt, 4, const_cast<void*>(res), d2r, st2, bx2, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(up skip) failed: " + std::to_string((int)r));
    }
    if (mode != kUpAdd) {
      CUresult r = encode_fn()(&p.tmO, dt, 4, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(out) failed: " + std::to_string((int)r));
      if (res) {
        r = encode_fn()(&p.tmR, dt, 4, const_cast<void*>(res), dims_r, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(res) failed: " + std::to_string((int)r));
      } else {
        p.tmR = p.tmO;
      }
    }
  }
  p.stages = (p.rows_R > 0 || p.nz_R > 0) ? 0 : stages_for(p.bn, p.bk);
  p.grid = a.num_work < num_sms() ? a.num_work : num_sms();
  p.flops = 2.0 * (double)B * Ho * Wo * Cout * (double)k * k * Cin;
  p.hb = a.hb;
  return p;
}

// Re-point a plan at a different batch size (same buffers): only the work count changes.
void set_conv_batch(ConvPlan& p, int B) {
  ConvArgs& a = p.args;
  a.num_work = B * a.tiles_x * a.tiles_y * a.n_tiles_n;
  p.grid = a.num_work < num_sms() ? a.num_work : num_sms();
  p.flops = 2.0 * (double)B * a.Ho * a.Wo * a.Cout * (double)a.ksize * a.ksize * a.Cin;
}

void run_conv(const ConvPlan& p, cudaStream_t s) {
  if (p.args.num_work <= 0) return;
  if (p.bf16)
    dispatch<__nv_bfloat16>(p, s);
  else
    dispatch<__half>(p, s);
  OS_CUDA(cudaGetLastError());
}

}  // namespace osg
