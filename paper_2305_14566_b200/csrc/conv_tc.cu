// conv_tc.cu -- host side of the tcgen05 implicit-GEMM convolution: TMA tensor maps,
// tile-shape selection, template dispatch and the persistent launch.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
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

template <typename T, int BN, int BK, int MODE, int CL = 1>
struct Cfg {
  static constexpr int kStageBytes = ConvSmem<BN, BK, 1, MODE, CL>::kStage;
  static constexpr int kStages0 = (MODE == kUpAdd ? kStageBudgetTapUp : kStageBudgetTap) / kStageBytes;
  static constexpr int STAGES = kStages0 > 8 ? 8 : (kStages0 < 2 ? 2 : kStages0);
  using Smem = ConvSmem<BN, BK, STAGES, MODE, CL>;
};

template <typename T, int BN, int BK>
void launch_tpl(const ConvPlan& p, cudaStream_t s) {
  using C0 = Cfg<T, BN, BK, kReluBias>;
  using C1 = Cfg<T, BN, BK, kResidualRelu>;
  using CU = Cfg<T, BN, BK, kUpAdd>;
  using C3 = Cfg<T, BN, BK, kBias>;
  auto launch_mode = [&](auto kern, int smem, int cl) {
    // all instantiations share one function-pointer type: remember each kernel separately
    static std::mutex mu;
    static std::unordered_set<const void*> done;
    {
      std::lock_guard<std::mutex> g(mu);
      if (done.insert(reinterpret_cast<const void*>(kern)).second)
        OS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    const int threads = tap_epi_warps(BN, p.mode) == 8 ? 384 : 256;
    if (cl == 1) {
      kern<<<p.grid, threads, smem, s>>>(p.tmA, p.tmB, p.tmO, p.tmR, p.args, p.lo);
      return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    OS_CUDA(cudaLaunchKernelEx(&cfg, kern, p.tmA, p.tmB, p.tmO, p.tmR, p.args, p.lo));
  };
  if constexpr (BN == 256 || BN == 128) {
    if (p.cl == 2) {  // CTA pair (cta_group::2): half the B rows per CTA -> a deeper ring
      using P0 = Cfg<T, BN, BK, kReluBias, 2>;
      using P1 = Cfg<T, BN, BK, kResidualRelu, 2>;
      using P3 = Cfg<T, BN, BK, kBias, 2>;
      switch (p.mode) {
        case kReluBias: launch_mode(conv_tc_kernel<T, BN, BK, P0::STAGES, kReluBias, 2>, P0::Smem::kTotal, 2); break;
        case kResidualRelu:
          launch_mode(conv_tc_kernel<T, BN, BK, P1::STAGES, kResidualRelu, 2>, P1::Smem::kTotal, 2);
          break;
        case kBias: launch_mode(conv_tc_kernel<T, BN, BK, P3::STAGES, kBias, 2>, P3::Smem::kTotal, 2); break;
        default: throw Error(-1, "CTA-pair conv: unsupported mode");
      }
      return;
    }
  }
  switch (p.mode) {
    case kReluBias: launch_mode(conv_tc_kernel<T, BN, BK, C0::STAGES, kReluBias>, C0::Smem::kTotal, 1); break;
    case kResidualRelu:
      launch_mode(conv_tc_kernel<T, BN, BK, C1::STAGES, kResidualRelu>, C1::Smem::kTotal, 1);
      break;
    case kUpAdd: launch_mode(conv_tc_kernel<T, BN, BK, CU::STAGES, kUpAdd>, CU::Smem::kTotal, 1); break;
    default: launch_mode(conv_tc_kernel<T, BN, BK, C3::STAGES, kBias>, C3::Smem::kTotal, 1); break;
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
    kern<<<p.grid, 256, smem, s>>>(p.tmA, p.tmB, p.tmO, p.tmR, p.args, p.lo);
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
  constexpr int ST = NzCfg::STAGES(BN, 0);   // output-only epilogue
  constexpr int STR = NzCfg::STAGES(BN, 1);  // residual epilogue
  constexpr int STH = NzCfg::STAGES(BN, 2);  // fused head (residual slots only)
  static_assert(ST >= 2 && STR >= 2 && STH >= 2, "no-swizzle tile does not fit shared memory");
  constexpr int RT = NzCfg::RTC;
  constexpr int STT = NzCfg::STAGES(BN, 2, RT);  // tensor-core head
  constexpr int STL0 = NzCfg::STAGES(BN, 4);  // lean output-only epilogue
  const bool lean0 = p.mode == kReluBias && p.args.split != kStoreX2 && STL0 > ST;
  int smem = lean0 ? NzSmem<BN, R, STL0, DYF, 8, 4>::kTotal : NzSmem<BN, R, ST, DYF, 8, 0>::kTotal;
  const int threads = 384;
  // residual convs in F8 / plain storage: the lean epilogue layout buys another ring stage
  constexpr int STL = NzCfg::STAGES(BN, 3);
  const bool lean = p.mode == kResidualRelu && p.args.split != kStoreX2 && STL > STR;
  if (p.mode == kResidualRelu) smem = lean ? NzSmem<BN, R, STL, DYF, 8, 3>::kTotal : NzSmem<BN, R, STR, DYF, 8, 1>::kTotal;
  else if (p.mode == kHeadFused) smem = p.head_tc ? NzSmem<BN, RT, STT, DYF, 8, 2>::kTotal : NzSmem<BN, R, STH, DYF, 8, 2>::kTotal;
  OS_REQUIRE(p.nz_R == (p.head_tc ? RT : R), "nz plan: rows per work item mismatch");
  auto go = [&](auto kern) {
    static std::mutex mu;
    static std::unordered_set<const void*> done;
    {
      std::lock_guard<std::mutex> g(mu);
      if (done.insert(reinterpret_cast<const void*>(kern)).second)
        OS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    kern<<<p.grid, threads, smem, s>>>(p.tmA, p.tmB, p.tmO, p.tmR, p.args, p.head, p.lo);
  };
  if constexpr (BN == 128 && !DYF) {
    if (p.cl == 2) {  // CTA pair (cta_group::2), cluster (2, 1, 1)
      constexpr int ST2 = NzCfg::STAGES_CL2(BN, 0), STR2 = NzCfg::STAGES_CL2(BN, 1), STL2 = NzCfg::STAGES_CL2(BN, 3),
                    STL20 = NzCfg::STAGES_CL2(BN, 4);
      auto go2 = [&](auto kern, int sm) {
        static std::mutex mu;
        static std::unordered_set<const void*> done;
        {
          std::lock_guard<std::mutex> g(mu);
          if (done.insert(reinterpret_cast<const void*>(kern)).second)
            OS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(p.grid);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        OS_CUDA(cudaLaunchKernelEx(&cfg, kern, p.tmA, p.tmB, p.tmO, p.tmR, p.args, p.head, p.lo));
      };
      if (p.mode == kReluBias && p.args.split != kStoreX2 && STL20 > ST2)
        go2(conv3_nz_kernel<T, BN, R, STL20, kReluBias, false, 2, true>, NzSmem<BN, R, STL20, false, 8, 4, 2>::kTotal);
      else if (p.mode == kReluBias)
        go2(conv3_nz_kernel<T, BN, R, ST2, kReluBias, false, 2>, NzSmem<BN, R, ST2, false, 8, 0, 2>::kTotal);
      else if (p.mode == kResidualRelu && p.args.split != kStoreX2 && STL2 > STR2)
        go2(conv3_nz_kernel<T, BN, R, STL2, kResidualRelu, false, 2, true>, NzSmem<BN, R, STL2, false, 8, 3, 2>::kTotal);
      else if (p.mode == kResidualRelu)
        go2(conv3_nz_kernel<T, BN, R, STR2, kResidualRelu, false, 2>, NzSmem<BN, R, STR2, false, 8, 1, 2>::kTotal);
      else
        throw Error(-1, "nz CTA pair: unsupported mode");
      return;
    }
  }
  switch (p.mode) {
    case kReluBias:
      if constexpr (STL0 > ST) {
        if (lean0) {
          go(conv3_nz_kernel<T, BN, R, STL0, kReluBias, DYF, 1, true>);
          break;
        }
      }
      go(conv3_nz_kernel<T, BN, R, ST, kReluBias, DYF>);
      break;
    case kResidualRelu:
      if constexpr (STL > STR) {
        if (lean) {
          go(conv3_nz_kernel<T, BN, R, STL, kResidualRelu, DYF, 1, true>);
          break;
        }
      }
      go(conv3_nz_kernel<T, BN, R, STR, kResidualRelu, DYF>);
      break;
    case kHeadFused:
      if constexpr (BN <= 32) {
        if (p.head_tc) {
          go(conv3_nz_kernel<T, BN, RT, STT, kHeadFused, DYF>);
          break;
        }
      }
      go(conv3_nz_kernel<T, BN, R, STH, kHeadFused, DYF>);
      break;
    default: go(conv3_nz_kernel<T, BN, R, ST, kBias, DYF>); break;
  }
}

template <typename T, int BN>
void launch_s2(const ConvPlan& p, cudaStream_t s) {
  constexpr int R = S2Cfg::R(BN);
  constexpr int ST = S2Cfg::STAGES(BN);
  static_assert(ST >= 2, "stride-2 tile does not fit shared memory");
  constexpr int smem = S2Smem<BN, R, ST>::kTotal;
  auto kern = conv3s2_rc_kernel<T, BN, R, ST>;
  static std::once_flag once;
  std::call_once(once, [&] { OS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); });
  kern<<<p.grid, 384, smem, s>>>(p.tmA, p.tmB, p.tmO, p.args, p.lo);
}

template <typename T>
void dispatch(const ConvPlan& p, cudaStream_t s) {
  if (p.s2_R > 0) {
    if (p.bn == 16) return launch_s2<T, 16>(p, s);
    if (p.bn == 32) return launch_s2<T, 32>(p, s);
    if (p.bn == 64) return launch_s2<T, 64>(p, s);
    if (p.bn == 128) return launch_s2<T, 128>(p, s);
    throw Error(-1, "unsupported stride-2 conv shape");
  }
  if (p.mode == kHeadFused && p.nz_R == 0) throw Error(-1, "fused head needs the no-swizzle conv kernel");
  if (p.nz_R > 0) {
    static const bool dyf = !exp_flag("OMNISEG_NO_DYF");
    if (p.bn == 16) return dyf ? launch_nz<T, 16, true>(p, s) : launch_nz<T, 16, false>(p, s);
    if (p.bn == 32) return dyf ? launch_nz<T, 32, true>(p, s) : launch_nz<T, 32, false>(p, s);
    if (p.bn == 64) return dyf ? launch_nz<T, 64, true>(p, s) : launch_nz<T, 64, false>(p, s);
    if (p.bn == 128) return launch_nz<T, 128, false>(p, s);  // 3 x 128 > 256: no dy stacking
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

int stages_for(int bn, int bk) {  // informational (ConvPlan::stages): the non-up-add ring depth
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

bool s2_eligible(int Hin, int Win, int Cin, int Cout, int k, int stride, int mode) {
  int bn = 256;
  while (Cout % bn) bn >>= 1;
  return k == 3 && stride == 2 && mode == kReluBias && bn <= 128 && bn >= 16 && Cout == bn && Cin % 16 == 0 &&
         Win % 128 == 0 && Hin % 2 == 0 && (Hin / 2) % S2Cfg::R(bn) == 0;
}

bool nz_eligible(int Hin, int Win, int Cin, int Cout, int k, int stride, int mode) {
  int bn = 256;
  while (Cout % bn) bn >>= 1;
  return k == 3 && stride == 1 && mode != kUpAdd && bn <= 128 && Cout == bn && Cin % 16 == 0 && Win >= 128 &&
         Win % 128 == 0 && Hin % NzCfg::R(bn) == 0 && (bn <= 64 || mode != kHeadFused);
}

ConvPlan make_conv_plan(bool bf16, const void* in, int B, int Hin, int Win, int Cin, const void* w,
                        const float* bias, int Cout, int k, int stride, int mode, const void* res, void* out,
                        int split_out, int B_in, int B_res, int B_out, int in_kind, const void* w_lo, int in_rc,
                        int res_rc, int out_rc) {
  if (B_in < 0) B_in = B;
  if (B_res < 0) B_res = B;
  if (B_out < 0) B_out = B;
  OS_REQUIRE(Cin % 16 == 0 && Cout % 16 == 0, "conv channels must be multiples of 16");
  OS_REQUIRE(k == 1 || k == 3, "conv kernel size must be 1 or 3");
  OS_REQUIRE(stride == 1 || stride == 2, "conv stride must be 1 or 2");
  const bool f8in = in_kind == kStoreF8;
  OS_REQUIRE(!f8in || (Cin % 32 == 0 && w_lo != nullptr && !bf16), "F8 input needs Cin % 32 == 0, fp16 and lo weights");
  OS_REQUIRE(split_out != kStoreF8 || (Cout % 32 == 0 && !bf16), "F8 output needs Cout % 32 == 0 and fp16");
  ConvPlan p{};
  if (mode == kHeadFusedTc) {
    mode = kHeadFused;
    p.head_tc = !bf16 && Cout <= 32;
  }
  p.mode = mode;
  p.bf16 = bf16;
  // K chunk = one swizzle row (128/64/32 bytes); N tile = largest power of two <= 256 dividing Cout
  p.bk = Cin % 64 == 0 ? 64 : Cin % 32 == 0 ? 32 : 16;
  p.bn = 256;
  while (Cout % p.bn) p.bn >>= 1;
  if (p.bn == 256 && p.bk == 64 && exp_flag("OMNISEG_TAP_BK32")) p.bk = 32;  // experiment: deeper ring
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
  a.kch_lo = f8in ? Cin / p.bk : 0;
  // input pixel bytes and the element count of its (hi) channel axis
  const uint64_t in_px = f8in ? 3ull * Cin : 2ull * Cin;
  const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const CUtensorMapDataType d8 = CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const void* in_lo = f8in ? static_cast<const uint8_t*>(in) + 2 * Cin : nullptr;
  a.in_rc = in_rc;
  a.res_rc = res_rc;
  a.out_rc = out_rc;
  {
    const int Wout = mode == kUpAdd ? 2 * Wo : Wo;  // up-add: the full-resolution output
    OS_REQUIRE(!out_rc || (Wout >= 128 && Wout % 128 == 0 && (mode != kUpAdd || a.wb >= 32)),
               "row-chunked output needs width >= 128");
    OS_REQUIRE(!res_rc || (Wout >= 128 && Wout % 128 == 0 && (mode != kUpAdd || a.wb >= 32)),
               "row-chunked residual / skip needs width >= 128");
  }
  // no-swizzle multi-row variant (conv3_nz_kernel): 3x3 stride 1, width >= 128, N <= 64, and
  // the input in the row-chunked layout (which only that kernel reads)
  OS_REQUIRE(!in_rc || nz_eligible(Hin, Win, Cin, Cout, k, stride, mode) ||
                 s2_eligible(Hin, Win, Cin, Cout, k, stride, mode),
             "row-chunked input needs the nz / stride-2 row-chunked conv");
  if (in_rc && stride == 2) {
    // stride-2 kernel: the same RC view, box {128, 18, 2, 2R+1, 1}; 128 input px -> 64 output px
    const int R = S2Cfg::R(p.bn);
    const uint64_t nch = in_px / 16;
    cuuint64_t dims[5] = {128, (cuuint64_t)Win / 8, nch, (cuuint64_t)Hin, (cuuint64_t)B_in};
    cuuint64_t strides[4] = {128, (cuuint64_t)Win * 16, nch * Win * 16, (cuuint64_t)Hin * nch * Win * 16};
    cuuint32_t box[5] = {128, 18, 2, (cuuint32_t)(2 * R + 1), 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode_fn()(&p.tmA, d8, 5, const_cast<void*>(in), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(A rc s2) failed: " + std::to_string((int)r));
    p.s2_R = R;
    p.bk = 16;
    a.kchunks = Cin / 16;
    a.kch_lo = f8in ? Cin / 32 : 0;
    a.tiles_x = Win / 128;
    a.tiles_y = Ho / R;
  } else if (in_rc) {
    const int R = p.head_tc ? NzCfg::RTC : NzCfg::R(p.bn);
    // A: 5-D u8 view {128 B = 8 px of one chunk, W/8 units, chunk, H, B} of [B][H][chunk][W][16 B],
    // box {128, 18, 2, R+2, 1} -> smem [row][chunk][144 px][16 B]
    const uint64_t nch = in_px / 16;
    cuuint64_t dims[5] = {128, (cuuint64_t)Win / 8, nch, (cuuint64_t)Hin, (cuuint64_t)B_in};
    cuuint64_t strides[4] = {128, (cuuint64_t)Win * 16, nch * Win * 16, (cuuint64_t)Hin * nch * Win * 16};
    cuuint32_t box[5] = {128, 18, 2, (cuuint32_t)(R + 2), 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode_fn()(&p.tmA, d8, 5, const_cast<void*>(in), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(A rc) failed: " + std::to_string((int)r));
    p.nz_R = R;
    p.bk = 16;
    a.kchunks = Cin / 16;
    a.kch_lo = f8in ? Cin / 32 : 0;
    a.tiles_y /= R;
    // 128-channel layers (level 2): CTA pairs (cta_group::2) with half the weight image per CTA;
    // the image is built in the pair layout and read through a 3-D map (build_conv_wimage)
    if (p.bn == 128 && (mode == kReluBias || mode == kResidualRelu) && (a.tiles_x * a.tiles_y) % 2 == 0 &&
        !exp_flag("OMNISEG_NO_PAIR"))
      p.cl = 2;
  }
  // multi-row variant for 3x3 stride-1 convs with N <= 128 (see conv3_rows_kernel)
  if (p.nz_R == 0 && k == 3 && stride == 1 && mode != kUpAdd && p.bn <= 128 && (a.hb == 1 || a.hb == 2) &&
      Cout == p.bn && !exp_flag("OMNISEG_NO_ROWS")) {
    const int R = RowsCfg::R(p.bn);
    const int bk = RowsCfg::BK(p.bn, a.hb);
    if (a.tiles_y % R == 0 && Cin % bk == 0 && (!f8in || bk >= 32)) {
      p.rows_R = R;
      p.hb = a.hb;
      p.bk = bk;
      a.kchunks = Cin / bk;
      a.kch_lo = f8in ? Cin / bk : 0;
      a.tiles_y /= R;
    }
  }
  OS_REQUIRE(!f8in || p.nz_R > 0 || p.s2_R > 0 || p.bk >= 32, "F8 input needs K chunks of >= 32 channels");
  a.num_work = B * a.tiles_x * a.tiles_y * a.n_tiles_n;
  a.dbg = exp_int("OMNISEG_DBG");
  a.bias = bias;
  a.res = res;
  a.out = out;
  a.split = split_out;
  // per-tap layers with 256 / 128-wide N tiles (levels 3-4, the down convs): CTA pairs
  // (cta_group::2, M = 256), each CTA holding half of the weight rows; pairs need an even M-tile
  // count per N tile
  if (p.nz_R == 0 && p.s2_R == 0 && p.rows_R == 0 && (p.bn == 256 || p.bn == 128) && mode != kUpAdd &&
      (a.tiles_x * a.tiles_y) % 2 == 0 && !exp_flag("OMNISEG_NO_PAIR"))
    p.cl = 2;
  // per-tap kernel: 128-channel lo chunks when the K chunk is 64 (one SW128 row like the hi chunks)
  a.lo2 = (f8in && p.nz_R == 0 && p.s2_R == 0 && p.rows_R == 0 && p.bk == 64 && Cin % 128 == 0) ? 1 : 0;
  if (a.lo2) a.kch_lo = Cin / 128;
  if (p.nz_R == 0 && p.s2_R == 0) {
    cuuint64_t dims[4] = {(cuuint64_t)Cin, (cuuint64_t)Win, (cuuint64_t)Hin, (cuuint64_t)B_in};
    cuuint64_t strides[3] = {in_px, (cuuint64_t)Win * in_px, (cuuint64_t)Hin * Win * in_px};
    cuuint32_t box[4] = {(cuuint32_t)p.bk, (cuuint32_t)(a.wb * stride), (cuuint32_t)(a.hb * stride), 1};
    if (p.rows_R > 0) box[2] = (cuuint32_t)(p.rows_R * a.hb + 2);
    cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
    CUresult r = encode_fn()(&p.tmA, dt, 4, const_cast<void*>(in), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, swz(p.bk * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(A) failed: " + std::to_string((int)r));
    if (f8in) {
      cuuint32_t bl[4] = {box[0] * (a.lo2 ? 2u : 1u), box[1], box[2], box[3]};
      r = encode_fn()(&p.lo.A, d8, 4, const_cast<void*>(in_lo), dims, strides, bl, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      swz(p.bk * (a.lo2 ? 2 : 1)), CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(A lo) failed: " + std::to_string((int)r));
    }
  }
  {
    const int taps = k * k;
    cuuint64_t dims[2] = {(cuuint64_t)taps * Cin, (cuuint64_t)Cout};
    cuuint64_t strides[1] = {(cuuint64_t)taps * Cin * 2};
    cuuint32_t box[2] = {(cuuint32_t)p.bk, (cuuint32_t)(p.bn / p.cl)};  // CL = 2: each CTA loads half
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&p.tmB, dt, 2, const_cast<void*>(w), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, swz(p.bk * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(B) failed: " + std::to_string((int)r));
    if (f8in) {
      // lo weights: e5m2 bytes [Cout][taps*Cin]; a lo chunk is bk (nz: 32) bytes wide
      const int bkl = (p.nz_R > 0 || p.s2_R > 0) ? 32 : p.bk * (a.lo2 ? 2 : 1);
      cuuint64_t s1[1] = {(cuuint64_t)taps * Cin};
      cuuint32_t b1[2] = {(cuuint32_t)bkl, (cuuint32_t)(p.bn / p.cl)};
      r = encode_fn()(&p.lo.B, d8, 2, const_cast<void*>(w_lo), dims, s1, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      swz(bkl), CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(B lo) failed: " + std::to_string((int)r));
    }
  }
  {
    // output / residual maps for the TMA epilogue: [B][Ho][Wo][C], one warp box = CH channels
    // x (bw x bh) pixels, 64-B (CH=32) / 32-B (CH=16) swizzle; x2 stores [C hi | C lo] per
    // pixel (lo at channel Cout), F8 a fp16 hi map + an e4m3 lo map (CH-byte rows, 32-B / no swizzle)
    const bool tap = p.nz_R == 0 && p.rows_R == 0 && p.s2_R == 0;  // per-tap kernel (conv_tc_kernel)
    const int CH = tap ? tap_epi_ch(p.bn, mode) : (p.bn < 32 ? p.bn : 32);
    const bool f8o = split_out == kStoreF8;
    const int Cst = split_out == kStoreX2 ? 2 * Cout : Cout;
    const uint64_t opx = f8o ? 3ull * Cout : 2ull * Cst;
    int bw = a.wb < 32 ? a.wb : 32, bh = 32 / bw;
    if (p.s2_R > 0) bw = 16, bh = 1;  // stride-2 RC kernel: a warp stores 16 output pixels
    cuuint64_t dims[4] = {(cuuint64_t)Cst, (cuuint64_t)Wo, (cuuint64_t)Ho, (cuuint64_t)B_out};
    cuuint64_t dims_r[4] = {(cuuint64_t)Cst, (cuuint64_t)Wo, (cuuint64_t)Ho, (cuuint64_t)B_res};
    cuuint64_t strides[3] = {opx, (cuuint64_t)Wo * opx, (cuuint64_t)Ho * Wo * opx};
    cuuint32_t box[4] = {(cuuint32_t)CH, (cuuint32_t)bw, (cuuint32_t)bh, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle sw = CH == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    const CUtensorMapSwizzle swl = CH == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    auto enc = [&](CUtensorMap* m, CUtensorMapDataType t, const void* base, const cuuint64_t* d, const cuuint64_t* st,
                   const cuuint32_t* bx, CUtensorMapSwizzle z, const char* what) {
      CUresult r = encode_fn()(m, t, 4, const_cast<void*>(base), d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, z,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(-2, std::string("cuTensorMapEncodeTiled(") + what + ") failed: " +
                                                 std::to_string((int)r));
    };
    auto lo_of = [&](const void* base) { return static_cast<const void*>(static_cast<const uint8_t*>(base) + 2 * Cout); };
    // row-chunked out / residual: 5-D u8 {128 B, W/8, chunk, H, B}; box = 32 (up-add: 64) pixels x the
    // chunks of CH channels (hi; x2 lo: the same box at chunk Cout/8 + ..; F8 lo: CH/16 chunks)
    auto enc_rc = [&](CUtensorMap* m, const void* base, int Wd, int Hd, int Bd, int px, int chunks, const char* what) {
      const uint64_t nch = opx / 16;
      // 128-B units of 8 pixels as the inner box dimension (16-B TMA rows are issue-limited)
      cuuint64_t d5[5] = {128, (cuuint64_t)Wd / 8, nch, (cuuint64_t)Hd, (cuuint64_t)Bd};
      cuuint64_t s5[4] = {128, (cuuint64_t)Wd * 16, nch * Wd * 16, (cuuint64_t)Hd * nch * Wd * 16};
      cuuint32_t b5[5] = {128, (cuuint32_t)px / 8, (cuuint32_t)chunks, 1, 1};
      cuuint32_t e5[5] = {1, 1, 1, 1, 1};
      CUresult r = encode_fn()(m, d8, 5, const_cast<void*>(base), d5, s5, b5, e5, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(-2, std::string("cuTensorMapEncodeTiled(") + what + ") failed: " +
                                                 std::to_string((int)r));
    };
    if (mode == kUpAdd && a.wb >= 32) {
      // up-add: full-resolution skip / output, one box = 64 output pixels of one row
      cuuint64_t d2[4] = {(cuuint64_t)Cst, (cuuint64_t)(2 * Wo), (cuuint64_t)(2 * Ho), (cuuint64_t)B_out};
      cuuint64_t d2r[4] = {(cuuint64_t)Cst, (cuuint64_t)(2 * Wo), (cuuint64_t)(2 * Ho), (cuuint64_t)B_res};
      cuuint64_t st2[3] = {opx, 2ull * Wo * opx, 4ull * Ho * Wo * opx};
      cuuint32_t bx2[4] = {(cuuint32_t)CH, 64, 1, 1};
      if (out_rc) {
        enc_rc(&p.tmO, out, 2 * Wo, 2 * Ho, B_out, 64, CH / 8, "up out rc");
        if (f8o) enc_rc(&p.lo.O, out, 2 * Wo, 2 * Ho, B_out, 64, CH / 16, "up out lo rc");
      } else {
        enc(&p.tmO, dt, out, d2, st2, bx2, sw, "up out");
        if (f8o) enc(&p.lo.O, d8, lo_of(out), d2, st2, bx2, swl, "up out lo");
      }
      if (res_rc) {
        enc_rc(&p.tmR, res, 2 * Wo, 2 * Ho, B_res, 64, CH / 8, "up skip rc");
        if (f8o) enc_rc(&p.lo.R, res, 2 * Wo, 2 * Ho, B_res, 64, CH / 16, "up skip lo rc");
      } else {
        enc(&p.tmR, dt, res, d2r, st2, bx2, sw, "up skip");
        if (f8o) enc(&p.lo.R, d8, lo_of(res), d2r, st2, bx2, swl, "up skip lo");
      }
    }
    if (mode != kUpAdd) {
      if (out_rc) {
        enc_rc(&p.tmO, out, Wo, Ho, B_out, bw, CH / 8, "out rc");
        if (f8o) enc_rc(&p.lo.O, out, Wo, Ho, B_out, bw, CH / 16, "out lo rc");
      } else {
        enc(&p.tmO, dt, out, dims, strides, box, sw, "out");
        if (f8o) enc(&p.lo.O, d8, lo_of(out), dims, strides, box, swl, "out lo");
      }
      if (res && res_rc) {
        enc_rc(&p.tmR, res, Wo, Ho, B_res, 32, CH / 8, "res rc");
        if (f8o) enc_rc(&p.lo.R, res, Wo, Ho, B_res, 32, CH / 16, "res lo rc");
      } else if (res) {
        enc(&p.tmR, dt, res, dims_r, strides, box, sw, "res");
        if (f8o) enc(&p.lo.R, d8, lo_of(res), dims_r, strides, box, swl, "res lo");
      } else {
        p.tmR = p.tmO;
      }
    }
  }
  p.stages = (p.rows_R > 0 || p.nz_R > 0 || p.s2_R > 0) ? 0 : stages_for(p.bn, p.bk);
  p.grid = a.num_work < num_sms() ? a.num_work : num_sms();
  if (p.cl == 2) p.grid &= ~1;  // whole clusters (num_work is even)
  p.flops = 2.0 * (double)B * Ho * Wo * Cout * (double)k * k * Cin;
  p.hb = a.hb;
  return p;
}

// Re-point a plan at a different batch size (same buffers): only the work count changes.
void set_conv_batch(ConvPlan& p, int B) {
  ConvArgs& a = p.args;
  a.num_work = B * a.tiles_x * a.tiles_y * a.n_tiles_n;
  p.grid = a.num_work < num_sms() ? a.num_work : num_sms();
  if (p.cl == 2) p.grid &= ~1;
  p.flops = 2.0 * (double)B * a.Ho * a.Wo * a.Cout * (double)a.ksize * a.ksize * a.Cin;
}

// ---- per-K-step weight images of the nz / stride-2 kernels (ConvArgs::wimg)
namespace {
struct SlotMap {
  int tap[9];
};
// one thread per (n tile, K step, slot, row n, 16-B half j)
__global__ void wimage_kernel(const uint8_t* w16, const uint8_t* wlo, uint8_t* dst, int ntn, int BN, int taps_cin,
                              int Cin, int khi, int klo, SlotMap sm, int cl) {
  const int nks = khi + klo;
  const int64_t total = (int64_t)ntn * nks * 9 * BN * 2;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int j = (int)(i & 1);
  int64_t r = i >> 1;
  const int n = (int)(r % BN);
  r /= BN;
  const int slot = (int)(r % 9);
  r /= 9;
  const int ks = (int)(r % nks);
  const int nt = (int)(r / nks);
  const int co = nt * BN + n, tap = sm.tap[slot];
  const uint8_t* src = ks < khi ? w16 + ((int64_t)co * taps_cin + (int64_t)tap * Cin + 16 * ks + 8 * j) * 2
                                : wlo + (int64_t)co * taps_cin + (int64_t)tap * Cin + 32 * (ks - khi) + 16 * j;
  // cl = 2 (CTA pair): [nt][ks][half][slot][n % (BN/2)][32 B], each CTA's half of a K step contiguous
  const int bnh = BN / cl, hf = n / bnh, nl = n - hf * bnh;
  uint8_t* d = dst + ((((int64_t)nt * nks + ks) * cl + hf) * 9 + slot) * bnh * 32 + nl * 32 + 16 * (j ^ ((nl >> 2) & 1));
  *reinterpret_cast<uint4*>(d) = *reinterpret_cast<const uint4*>(src);
}
}  // namespace

size_t conv_wimage_bytes(const ConvPlan& p) {
  if (p.nz_R == 0 && p.s2_R == 0) return 0;
  return (size_t)p.args.n_tiles_n * (p.args.kchunks + p.args.kch_lo) * 9 * p.bn * 32;
}

void build_conv_wimage(ConvPlan& p, const void* w, const void* w_lo, void* dst, cudaStream_t s) {
  const size_t bytes = conv_wimage_bytes(p);
  if (!bytes) return;
  SlotMap sm;
  for (int tap = 0; tap < 9; ++tap) {
    const int dy = tap / 3, dx = tap % 3;
    int slot;
    if (p.s2_R > 0) slot = dx * 3 + (dy == 0 ? 0 : dy == 2 ? 1 : 2);  // [dx][dy0, dy2, dy1]
    else if (!exp_flag("OMNISEG_NO_DYF") && p.bn <= 64) slot = dx * 3 + dy;  // dy-fused: [dx][dy]
    else slot = tap;
    sm.tap[slot] = tap;
  }
  const int64_t total = (int64_t)bytes / 16;
  wimage_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
      static_cast<const uint8_t*>(w), static_cast<const uint8_t*>(w_lo), static_cast<uint8_t*>(dst),
      p.args.n_tiles_n, p.bn, 9 * p.args.Cin, p.args.Cin, p.args.kchunks, p.args.kch_lo, sm, p.cl);
  OS_CUDA(cudaGetLastError());
  p.args.wimg = static_cast<const uint8_t*>(dst);
  if (p.cl == 2 && p.nz_R > 0) {
    // 3-D view {32 B, BN/2 rows, planes} of the pair-layout image; box = one CTA's 9 tap slots
    const int bnh = p.bn / 2;
    const uint64_t planes = (uint64_t)p.args.n_tiles_n * (p.args.kchunks + p.args.kch_lo) * 2 * 9;
    cuuint64_t dims[3] = {32, (cuuint64_t)bnh, (cuuint64_t)planes};
    cuuint64_t strides[2] = {32, (cuuint64_t)bnh * 32};
    cuuint32_t box[3] = {32, (cuuint32_t)bnh, 9};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_fn()(&p.tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, dst, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(weight image pair) failed: " + std::to_string((int)r));
  }
}

constexpr int kStemR = 4, kStemNA = 8;

bool stem_fusable(int P, int Cout) {
  int bn = 256;
  while (Cout % bn) bn >>= 1;
  return P % 128 == 0 && P % kStemR == 0 && Cout == bn && (bn == 16 || bn == 32 || bn == 64);
}

StemPlan make_stem_plan(const ConvPlan& stem_conv, const void* w, int P) {
  StemPlan p;
  p.conv = stem_conv;
  StemArgs& a = p.args;
  a = StemArgs{};
  a.bias = stem_conv.args.bias;
  a.w = w;
  a.P = P;
  a.tiles_x = P / 128;
  a.tiles_y = P / kStemR;
  a.split = stem_conv.args.split;
  a.out_rc = stem_conv.args.out_rc;
  a.Cout = stem_conv.args.Cout;
  return p;
}

template <typename T, int BN>
void launch_stem(const StemPlan& p, cudaStream_t s) {
  using S = StemSmem<BN, kStemR, kStemNA>;
  auto kern = stem_tc_kernel<T, BN, kStemR, kStemNA>;
  static std::once_flag once;
  std::call_once(once, [&] { OS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal)); });
  kern<<<p.grid, S::kThreads, S::kTotal, s>>>(p.conv.tmO, p.args, p.conv.lo, p.inm.m[0], p.inm.m[1], p.inm.m[2],
                                              p.inm.m[3]);
}

// TMA map of one RGBX level (u32 elements {Wp/f, Hp/f}), box {kStemBoxW, kStemR + 2}; reads past
// the image edge return 0 (the converters zero everything outside the window anyway).
void encode_level_map(CUtensorMap* m, const uint32_t* L, int Hl, int Wl) {
  cuuint64_t dims[2] = {(cuuint64_t)Wl, (cuuint64_t)Hl};
  cuuint64_t strides[1] = {(cuuint64_t)Wl * 4};
  cuuint32_t box[2] = {(cuuint32_t)kStemBoxW, (cuuint32_t)(kStemR + 2)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(L), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(-2, "cuTensorMapEncodeTiled(stem level) failed: " + std::to_string((int)r));
}

void run_stem(StemPlan& p, const uint32_t* tiles, int first, int n, const uint32_t* const L[4], int S, int Hp, int Wp,
              cudaStream_t s) {
  StemArgs& a = p.args;
  a.tiles = tiles;
  for (int i = 0; i < 4; ++i) a.L[i] = L[i];
  a.first = first;
  a.S = S;
  a.Hp = Hp;
  a.Wp = Wp;
  a.num_work = n * a.tiles_x * a.tiles_y;
  if (a.num_work <= 0) return;
  p.grid = a.num_work < num_sms() ? a.num_work : num_sms();
  if (Hp != p.inm_Hp || Wp != p.inm_Wp || L[0] != p.inm_ptr[0] || L[1] != p.inm_ptr[1] || L[2] != p.inm_ptr[2] ||
      L[3] != p.inm_ptr[3]) {
    for (int l = 0; l < 4; ++l) {
      p.inm_ptr[l] = L[l];
      if (L[l]) encode_level_map(&p.inm.m[l], L[l], Hp >> l, Wp >> l);
    }
    p.inm_Hp = Hp;
    p.inm_Wp = Wp;
  }
  static unsigned long long* sdbg = nullptr;
  const bool dbg = (exp_int("OMNISEG_DBG") & 8) != 0;
  if (dbg && !sdbg) OS_CUDA(cudaMalloc(&sdbg, 148 * 4 * 8));
  a.dbg_out = dbg ? sdbg : nullptr;
  const int bn = p.conv.bn;
  if (p.conv.bf16) {
    if (bn == 16) launch_stem<__nv_bfloat16, 16>(p, s);
    else if (bn == 32) launch_stem<__nv_bfloat16, 32>(p, s);
    else launch_stem<__nv_bfloat16, 64>(p, s);
  } else {
    if (bn == 16) launch_stem<__half, 16>(p, s);
    else if (bn == 32) launch_stem<__half, 32>(p, s);
    else launch_stem<__half, 64>(p, s);
  }
  OS_CUDA(cudaGetLastError());
  if (dbg) {
    unsigned long long hb[148 * 4];
    OS_CUDA(cudaStreamSynchronize(s));
    OS_CUDA(cudaMemcpy(hb, sdbg, sizeof(hb), cudaMemcpyDeviceToHost));
    double t = 0, te = 0, fu = 0, nn = 0;
    for (int i = 0; i < p.grid; ++i) t += hb[4 * i], te += hb[4 * i + 1], fu += hb[4 * i + 2], nn += hb[4 * i + 3];
    fprintf(stderr, "[stem] per item: total %.0f, wait tempty %.0f, wait afull %.0f cycles (%.0f items/CTA)\n", t / nn,
            te / nn, fu / nn, nn / p.grid);
  }
}

bool exp_flag(const char* name) {
#if OMNISEG_EXPERIMENTS
  return getenv(name) != nullptr;
#else
  (void)name;
  return false;
#endif
}
int exp_int(const char* name) {
#if OMNISEG_EXPERIMENTS
  const char* v = getenv(name);
  return v ? atoi(v) : 0;
#else
  (void)name;
  return 0;
#endif
}

void run_conv(const ConvPlan& p0, cudaStream_t s) {
  if (p0.args.num_work <= 0) return;
  OS_REQUIRE((p0.nz_R == 0 && p0.s2_R == 0) || p0.args.wimg != nullptr, "conv plan: weight image not built");
  ConvPlan p = p0;
  static unsigned long long* dbuf = nullptr;
  if ((p.args.dbg & 8) && p.rows_R == 0) {  // experiment: MMA-warp cycle counters
    if (!dbuf) OS_CUDA(cudaMalloc(&dbuf, 148 * 4 * 8));
    p.args.dbg_out = dbuf;
  } else {
    p.args.dbg &= ~8;
  }
  if (p.bf16)
    dispatch<__nv_bfloat16>(p, s);
  else
    dispatch<__half>(p, s);
  OS_CUDA(cudaGetLastError());
  if (p.args.dbg & 8) {
    unsigned long long h[148 * 4];
    OS_CUDA(cudaStreamSynchronize(s));
    OS_CUDA(cudaMemcpy(h, dbuf, sizeof(h), cudaMemcpyDeviceToHost));
    double a = 0, te = 0, fu = 0, n = 0;
    for (int i = 0; i < p.grid; ++i) {
      a += h[4 * i];
      te += h[4 * i + 1];
      fu += h[4 * i + 2];
      n += h[4 * i + 3];
    }
    fprintf(stderr, "[%s BN=%d Cin=%d Wo=%d mode=%d] per item: total %.0f, wait tempty %.0f, wait full %.0f cycles (%.0f items/CTA)\n",
            p.s2_R ? "s2" : p.nz_R ? "nz" : "tap", p.bn, p.args.Cin, p.args.Wo, p.mode, a / n, te / n, fu / n, n / p.grid);
  }
}

}  // namespace osg
