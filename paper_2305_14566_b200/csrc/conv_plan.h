// conv_plan.h -- host interface of the tcgen05 convolution (conv_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "conv_tc.cuh"

namespace osg {

struct ConvPlan {
  CUtensorMap tmA, tmB;  // activation (4-D NHWC) and weight (2-D [Cout][taps*Cin]) TMA maps
  CUtensorMap tmO, tmR;  // output / residual maps of the TMA epilogue (unused for kUpAdd)
  LoMaps lo;             // e4m3 / e5m2 maps of the F8 lo parts (input, weights, output, residual)
  ConvArgs args;
  int bn, bk, stages, mode, grid;
  int rows_R = 0;        // > 0: the multi-row 3x3 kernel (conv3_rows_kernel) with R blocks
  int nz_R = 0;          // > 0: the no-swizzle multi-row 3x3 kernel (conv3_nz_kernel)
  int s2_R = 0;          // > 0: the stride-2 row-chunked-input kernel (conv3s2_rc_kernel)
  int cl = 1;            // per-tap kernel cluster size (2: CTA pairs multicasting the weight tiles)
  int hb = 1;
  bool bf16;
  bool head_tc = false;  // kHeadFused with the tensor-core head (R = NzCfg::RTC)
  HeadArgs head{};       // kHead mode (fused dynamic head + stitch), set by the caller per launch
  double flops;          // algorithmic FLOPs of one launch (2 * M * N * K)
};

// Plan one convolution: input [B][Hin][Win][Cin], weights [Cout][k][k][Cin] (16-bit,
// K-major), fp32 bias; output grid Ho = ceil(Hin/stride) etc. `res` per ConvMode.
// in_rc / res_rc / out_rc: tensors in the row-chunked layout [B][H][16-B chunk][W][16 B] (hi
// chunks, then lo chunks) instead of NHWC; an RC input requires nz_eligible().
// split_out: StoreKind of res/out. in_kind: StoreKind of the input; for x2 inputs the
// caller passes Cin = 2 x channels and weights duplicated along K ([W | W]); for F8 inputs
// Cin = channels, w = fp16 weights and w_lo = e5m2(W * 2^-6) bytes of the same layout.
// B = images per launch (work items); B_in / B_res / B_out = batch extents of the input,
// residual and output tensors (default B; the args.b_* offsets select the images).
ConvPlan make_conv_plan(bool bf16, const void* in, int B, int Hin, int Win, int Cin, const void* w,
                        const float* bias, int Cout, int k, int stride, int mode, const void* res, void* out,
                        int split_out = 0, int B_in = -1, int B_res = -1, int B_out = -1, int in_kind = 0,
                        const void* w_lo = nullptr, int in_rc = 0, int res_rc = 0, int out_rc = 0);
// The no-swizzle multi-row conv (the only reader of row-chunked inputs) applies to this shape.
bool nz_eligible(int Hin, int Win, int Cin, int Cout, int k, int stride, int mode);
// The stride-2 kernel over a row-chunked input (conv3s2_rc_kernel) applies to this shape.
bool s2_eligible(int Hin, int Win, int Cin, int Cout, int k, int stride, int mode);
void set_conv_batch(ConvPlan& p, int B);
// nz / stride-2 plans read their weights as per-K-step smem images: the caller allocates
// conv_wimage_bytes(p) bytes (0: not needed) and builds them once (stream-ordered).
size_t conv_wimage_bytes(const ConvPlan& p);
void build_conv_wimage(ConvPlan& p, const void* w, const void* w_lo, void* dst, cudaStream_t s);

// Fused window gather + stem (stem_tc_kernel): the stem conv's output maps come from its
// ConvPlan (a 1x1 conv over the unfused im2col input); windows are read from the RGBX levels.
struct StemPlan {
  ConvPlan conv;   // output maps, bias, weights, storage kind
  StemArgs args;
  int grid = 0;
  StemInMaps inm{};                       // TMA maps of the RGBX levels (rebuilt when they change)
  const void* inm_ptr[4] = {nullptr, nullptr, nullptr, nullptr};
  int inm_Hp = 0, inm_Wp = 0;
};
bool stem_fusable(int P, int Cout);
StemPlan make_stem_plan(const ConvPlan& stem_conv, const void* w, int P);
void run_stem(StemPlan& p, const uint32_t* tiles, int first, int n, const uint32_t* const L[4], int S, int Hp, int Wp,
              cudaStream_t s);
void run_conv(const ConvPlan& p, cudaStream_t s);
int num_sms();

}  // namespace osg
