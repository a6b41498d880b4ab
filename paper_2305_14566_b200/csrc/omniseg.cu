// omniseg.cu -- the C ABI (include/omniseg.h, include/omniseg_debug.h): argument
// validation, weight packing, workspace, the launch sequence of one slide / band, and
// the NCCL collectives of the multi-GPU band path. All arithmetic runs in the kernels
// of kernels.cu and conv_tc.cu.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-op unless a tool (ncu --nvtx, nsys) attaches

#include "../../include/omniseg.h"
#include "../../include/omniseg_debug.h"
#include "common.cuh"
#include "conv_plan.h"
#include "kernels.h"

using namespace osg;

namespace {

thread_local std::string g_last_error;

// NVTX range of one pipeline stage on the calling (host) thread: the enqueue timeline of a
// segment call (ncu --nvtx --nvtx-include "omniseg/..." selects a stage's kernels).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t bytes) {
    if (bytes <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (bytes == 0) return;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(-3, "cudaMalloc(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e));
    }
    n = bytes;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
  void* so = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  void load() {
    if (so) return;
    so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!so) throw Error(-4, std::string("dlopen libnccl.so.2 failed: ") + dlerror());
    commInitRank = (decltype(commInitRank))dlsym(so, "ncclCommInitRank");
    allReduce = (decltype(allReduce))dlsym(so, "ncclAllReduce");
    broadcast = (decltype(broadcast))dlsym(so, "ncclBroadcast");
    commDestroy = (decltype(commDestroy))dlsym(so, "ncclCommDestroy");
    errStr = (decltype(errStr))dlsym(so, "ncclGetErrorString");
    send = (decltype(send))dlsym(so, "ncclSend");
    recv = (decltype(recv))dlsym(so, "ncclRecv");
    groupStart = (decltype(groupStart))dlsym(so, "ncclGroupStart");
    groupEnd = (decltype(groupEnd))dlsym(so, "ncclGroupEnd");
    if (!commInitRank || !allReduce || !broadcast || !commDestroy || !errStr || !send || !recv || !groupStart ||
        !groupEnd)
      throw Error(-4, "libnccl.so.2 lacks required symbols");
  }
  void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(-4, std::string(what) + ": " + errStr(r));
  }
};
Nccl g_nccl;

// ---------------------------------------------------------------- arch
struct Arch {
  int levels = 5, base = 32, head = 8, ncls = 6, slide_mag = 40, batch = 64, device = -1;
  std::vector<int> scale_codes{5, 10, 20, 40};
  bool bf16 = false;
  int split = kStoreF8;     // StoreKind of the activations: f8 (fp16 + e4m3 lo; default), x2 (hi + lo 16-bit), plain
  int xlevels = -1;         // split storage only for tensors at U-Net levels < xlevels (-1: all levels)
  int xa = 1;               // 0: residual-block intermediates (conv_a outputs) stored plain 16-bit
  int xal = 64;             // with xa = 1: conv_a outputs keep the split kind only at levels < xal
  int xap = 0;              // conv_a outputs stored plain 16-bit at levels < xap (precision budget)
  int plainl = 0;           // bitmask of U-Net levels whose tensors are all stored plain 16-bit
  int xa_level(int l) const { return xa && l < xal && l >= xap ? l : 1000; }  // level passed to sp() for conv_a outputs
  int vote = 0;             // fusion rule: 0 mean of p (R11), 1 hard majority vote
  int fgmin = 0;            // drop foreground components below fgmin level-8 pixels
  int maskfg = 0;           // AND the output masks with the foreground
  int headtc = 0;           // 1: the fused head's layer 1 (+ precls) on tcgen05 (measured slower)
  // L2-resident schedule of the shallow levels: the U-Net levels < glev run per
  // group of grp windows (their intermediates in a group-sized scratch slice that stays in L2,
  // only the skips E_l per window), the deeper levels over the whole batch. grp = 0: every layer
  // over the whole batch.
  int grp = 0, glev = 2;
  std::vector<int> vthr;    // vote fusion: literal vote-count threshold per scale code; empty = majority
  int sp(int level) const {
    if (level < 31 && ((plainl >> level) & 1)) return kStorePlain;
    return level < (xlevels < 0 ? 64 : xlevels) ? split : kStorePlain;
  }
  // bytes per channel of a tensor stored with kind k
  static int bpc(int k) { return k == kStoreX2 ? 4 : k == kStoreF8 ? 3 : 2; }
  // channel padding: 16 (MMA K step), 32 in the f8 mode (an e4m3 MMA consumes 32 channels)
  int padc(int c) const { return split == kStoreF8 ? (c + 31) / 32 * 32 : (c + 15) / 16 * 16; }
};

Arch parse_arch(const char* s) {
  OS_REQUIRE(s != nullptr, "arch string is NULL");
  Arch a;
  std::stringstream ss(s);
  std::string kv;
  while (std::getline(ss, kv, ';')) {
    if (kv.empty()) continue;
    auto eq = kv.find('=');
    OS_REQUIRE(eq != std::string::npos, "arch: expected key=value, got '" + kv + "'");
    std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
    auto toi = [&](const std::string& x) {
      try {
        size_t pos = 0;
        int r = std::stoi(x, &pos);
        OS_REQUIRE(pos == x.size(), "arch: bad integer '" + x + "' for " + k);
        return r;
      } catch (const std::logic_error&) {
        throw Error(-1, "arch: bad integer '" + x + "' for " + k);
      }
    };
    if (k == "levels") a.levels = toi(v);
    else if (k == "base") a.base = toi(v);
    else if (k == "head") a.head = toi(v);
    else if (k == "ncls") a.ncls = toi(v);
    else if (k == "slide_mag") a.slide_mag = toi(v);
    else if (k == "batch") a.batch = toi(v);
    else if (k == "device") a.device = toi(v);
    else if (k == "xlevels") a.xlevels = toi(v);
    else if (k == "xa") a.xa = toi(v);
    else if (k == "xal") a.xal = toi(v);
    else if (k == "fgmin") a.fgmin = toi(v);
    else if (k == "maskfg") a.maskfg = toi(v);
    else if (k == "headtc") a.headtc = toi(v);
    else if (k == "grp") a.grp = toi(v);
    else if (k == "xap") a.xap = toi(v);
    else if (k == "plainl") a.plainl = toi(v);
    else if (k == "glev") a.glev = toi(v);
    else if (k == "vthr") {
      a.vthr.clear();
      std::stringstream s2(v);
      std::string x;
      while (std::getline(s2, x, ',')) {
        a.vthr.push_back(toi(x));
        OS_REQUIRE(a.vthr.back() >= 0, "arch: vthr entries must be >= 0");
      }
    }
    else if (k == "fusion") {
      OS_REQUIRE(v == "mean" || v == "vote", "arch: fusion must be mean or vote");
      a.vote = v == "vote";
    }
    else if (k == "dtype") {
      OS_REQUIRE(v == "fp16" || v == "bf16" || v == "fp16x2" || v == "bf16x2" || v == "fp16f8",
                 "arch: dtype must be fp16, bf16, fp16x2, bf16x2 or fp16f8");
      a.bf16 = v.rfind("bf16", 0) == 0;
      a.split = v == "fp16f8" ? kStoreF8 : v.size() > 4 ? kStoreX2 : kStorePlain;
    } else if (k == "scale_codes") {
      a.scale_codes.clear();
      std::stringstream s2(v);
      std::string x;
      while (std::getline(s2, x, ',')) a.scale_codes.push_back(toi(x));
    } else {
      throw Error(-1, "arch: unknown key '" + k + "'");
    }
  }
  OS_REQUIRE(a.levels >= 2 && a.levels <= 6, "arch: levels must be in [2, 6]");
  OS_REQUIRE(a.base >= 8 && a.base <= 64 && (a.base & (a.base - 1)) == 0, "arch: base must be 8, 16, 32 or 64");
  OS_REQUIRE((a.base << (a.levels - 1)) <= 2048, "arch: too many channels");
  OS_REQUIRE(a.head == kHead, "arch: head must be 8 (3-layer 8-channel dynamic head)");
  OS_REQUIRE(a.ncls >= 1 && a.ncls <= 64, "arch: ncls out of range");
  OS_REQUIRE(!a.scale_codes.empty() && a.scale_codes.size() <= 8, "arch: 1..8 scale codes");
  OS_REQUIRE(a.batch >= 1 && a.batch <= 4096, "arch: batch out of range");
  OS_REQUIRE(a.grp >= 0 && a.grp <= a.batch, "arch: grp must be in [0, batch]");
  OS_REQUIRE(a.glev >= 1 && a.glev <= 8, "arch: glev must be in [1, 8]");
  OS_REQUIRE(a.slide_mag >= 1, "arch: slide_mag must be positive");
  OS_REQUIRE(a.vthr.empty() || a.vthr.size() == a.scale_codes.size(), "arch: vthr needs one entry per scale code");
  return a;
}

int pad16(int c) { return (c + 15) / 16 * 16; }

struct Layer {
  DevBuf w;      // [coutp][k*k][cinp] 16-bit
  DevBuf wlo;    // f8 inputs: [coutp][k*k][cinp] e5m2 bytes of W * 2^-6 (the lo term's weights)
  mutable DevBuf wimg;  // per-K-step smem image of the weights for nz / stride-2 plans
  DevBuf b;      // [coutp] fp32
  int in_kind = 0;  // StoreKind of the layer's input
  int cin = 0, cout = 0, cinp = 0, coutp = 0, k = 3, stride = 1;
  int alg_k = 0; // algorithmic K if not k*k*cin (the stem: 27)
  DevBuf wpx;    // stem only: [coutp][48] weights of the fused stem's pixel-major RGBX im2col
};

struct LevelBufs {
  DevBuf E, A, Bt;
  int P = 0, C = 0;
};

}  // namespace

// ==================================================================== the handle
struct omniseg {
  Arch arch;
  int device = 0;
  std::vector<int> C, Cp;  // channels per level (real, padded to 16)
  Layer stem;
  std::vector<Layer> enc_a, enc_b, down, up, dec_a, dec_b;
  DevBuf Wpre, bpre, Wc, bc;
  int nin = 0;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // progressive D2H of finished canvas rows (host outputs)
  cudaEvent_t copy_ev = nullptr;

  // workspace (per patch size / batch capacity)
  int ws_P = 0, ws_B = 0;
  DevBuf X0;
  std::vector<LevelBufs> lv;
  std::vector<int> rc;   // per level: A_l / Bt_l stored row-chunked (see ensure_workspace)
  std::vector<int> erc;  // per level: E_l (encoder output / skip) stored row-chunked
  DevBuf g, gpart, theta, theta_t, task_cls, task_scl;
  // plans in launch order for one batch (rebuilt with the workspace)
  struct Step {
    int kind;  // 0 conv, 1 gap+controller marker
    ConvPlan plan;
  };
  std::vector<ConvPlan> enc_plans, dec_plans;
  std::vector<const Layer*> enc_layers, dec_layers;
  ConvPlan head_plan{};   // dec0.b with the dynamic head + stitch fused into its epilogue
  StemPlan stem_plan{};   // window gather + stem fused (stem_tc_kernel)
  bool stem_fused = false;
  bool head_fusable = false;
  // front end / canvases
  DevBuf cc_lab, cc_size;  // SURVEY N2 component-labelling scratch
  DevBuf r_slide, r_mask, r_40, r_10;  // SURVEY N3 render staging (host inputs / outputs)
  DevBuf slide, L1, L2, L4, L8, luma8, gm, fg, hist, state, keep, tiles, counts, grids, canvas, area, prob, mask, flag;
  std::vector<uint32_t> h_tiles;
  int64_t n_tiles = 0;
  int H8 = 0, W8 = 0, otsu_t = -1, g_pad = -1;
  int64_t fg_r0 = 0, fg_r1 = 0;

  // timing
  cudaEvent_t ev[12] = {};
  double timings[11] = {};
  int conv_launches = 0, launches = 0;

  // per-conv-launch profiling (omniseg_debug_set_profile): event pairs on the stream
  bool profile = false;
  std::vector<cudaEvent_t> pev;
  std::vector<int> player;
  std::vector<double> pflops;
  int pn = 0;                        // event pairs used in the current call
  std::vector<double> layer_ms, layer_flops, layer_n;
  double prof_ms = 0, prof_flops = 0, prof_launches = 0;

  // debug: injected global detection state for single-GPU band emulation
  bool inject = false;
  uint8_t inj_pc[4] = {0, 0, 0, 0};
  unsigned long long inj_hist[256] = {};
  std::vector<uint8_t> inj_fg;  // pre-filter level-8 foreground of the whole slide (band fgmin emulation)
  unsigned long long last_hist[256] = {};

  // NCCL
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;

  ~omniseg() {
    for (auto& e : pev)
      if (e) cudaEventDestroy(e);
    if (comm) g_nccl.commDestroy(comm);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (copy_ev) cudaEventDestroy(copy_ev);
  }
};

namespace {

template <typename T>
T to16(float v);
template <>
__half to16<__half>(float v) {
  return __float2half_rn(v);
}
template <>
__nv_bfloat16 to16<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// Upload one conv: blob order [cout][k][k][cin] fp32 -> device [coutp][k*k][cinp] 16-bit.
// x2 inputs: the K axis of every tap is [W | W] (kdup = 2). f8 inputs: also the lo weights
// e5m2(W * 2^-6), RNE and saturating (R9).
template <typename T>
void upload_conv(Layer& L, const float* w, const float* b, int cin, int cout, int k, int stride, int cinp, int coutp,
                 int in_kind = kStorePlain) {
  const int kdup = in_kind == kStoreX2 ? 2 : 1;
  L.in_kind = in_kind;
  L.cin = cin;
  L.cout = cout;
  L.cinp = cinp * kdup;
  L.coutp = coutp;
  L.k = k;
  L.stride = stride;
  const int ck = cinp * kdup;
  std::vector<T> hw((size_t)coutp * k * k * ck, to16<T>(0.f));
  for (int o = 0; o < cout; ++o)
    for (int t = 0; t < k * k; ++t)
      for (int d = 0; d < kdup; ++d)
        for (int c = 0; c < cin; ++c)
          hw[((size_t)o * k * k + t) * ck + d * cinp + c] = to16<T>(w[((size_t)o * k * k + t) * cin + c]);
  std::vector<float> hb(coutp, 0.f);
  for (int o = 0; o < cout; ++o) hb[o] = b[o];
  L.w.ensure(hw.size() * sizeof(T));
  L.b.ensure(hb.size() * sizeof(float));
  OS_CUDA(cudaMemcpy(L.w.p, hw.data(), hw.size() * sizeof(T), cudaMemcpyHostToDevice));
  OS_CUDA(cudaMemcpy(L.b.p, hb.data(), hb.size() * sizeof(float), cudaMemcpyHostToDevice));
  if (in_kind == kStoreF8) {
    std::vector<uint8_t> hl((size_t)coutp * k * k * cinp, 0);
    for (int o = 0; o < cout; ++o)
      for (int t = 0; t < k * k; ++t)
        for (int c = 0; c < cin; ++c)
          hl[((size_t)o * k * k + t) * cinp + c] = (uint8_t)__nv_cvt_float_to_fp8(
              w[((size_t)o * k * k + t) * cin + c] * kLoInv, __NV_SATFINITE, __NV_E5M2);
    L.wlo.ensure(hl.size());
    OS_CUDA(cudaMemcpy(L.wlo.p, hl.data(), hl.size(), cudaMemcpyHostToDevice));
  }
}

// Stem as a 1x1 conv over the 32-channel im2col input of the gather kernel:
// column (dy*3 + dx)*3 + c  <->  blob weight [o][dy][dx][c] (identical flattening).
template <typename T>
void upload_stem(Layer& L, const float* w, const float* b, int cout, int coutp) {
  std::vector<float> w32((size_t)cout * 32, 0.f);
  for (int o = 0; o < cout; ++o)
    for (int j = 0; j < 27; ++j) w32[(size_t)o * 32 + j] = w[(size_t)o * 27 + j];
  upload_conv<T>(L, w32.data(), b, 32, cout, 1, 1, 32, coutp);
  L.alg_k = 27;
  // fused stem (stem_tc_kernel): column (dy*3 + dx)*4 + c, c < 3; the X byte and 36..47 weigh 0
  std::vector<T> w48((size_t)coutp * 48, to16<T>(0.f));
  for (int o = 0; o < cout; ++o)
    for (int p = 0; p < 9; ++p)
      for (int c = 0; c < 3; ++c) w48[(size_t)o * 48 + p * 4 + c] = to16<T>(w[(size_t)o * 27 + p * 3 + c]);
  L.wpx.ensure(w48.size() * sizeof(T));
  OS_CUDA(cudaMemcpy(L.wpx.p, w48.data(), w48.size() * sizeof(T), cudaMemcpyHostToDevice));
}

size_t param_count(const Arch& a) {
  size_t n = 0;
  auto conv = [&](int co, int k, int ci) { n += (size_t)co * k * k * ci + co; };
  std::vector<int> C(a.levels);
  for (int l = 0; l < a.levels; ++l) C[l] = a.base << l;
  conv(C[0], 3, 3);
  for (int l = 0; l < a.levels; ++l) {
    conv(C[l], 3, C[l]);
    conv(C[l], 3, C[l]);
    if (l < a.levels - 1) conv(C[l + 1], 3, C[l]);
  }
  for (int l = a.levels - 2; l >= 0; --l) {
    conv(C[l], 1, C[l + 1]);
    conv(C[l], 3, C[l]);
    conv(C[l], 3, C[l]);
  }
  conv(kHead, 1, C[0]);
  const int nin = C[a.levels - 1] + a.ncls + (int)a.scale_codes.size();
  n += (size_t)kTheta * nin + kTheta;
  return n;
}

template <typename T>
void load_weights(omniseg* h, const float* blob) {
  const Arch& a = h->arch;
  const int L = a.levels;
  size_t o = 0;
  auto take = [&](size_t n) {
    const float* p = blob + o;
    o += n;
    return p;
  };
  // in_level: U-Net level of the layer's input tensor (x2 inputs duplicate the K axis)
  auto conv = [&](Layer& dst, int co, int k, int ci, int stride, int in_level) {
    const float* w = take((size_t)co * k * k * ci);
    const float* b = take(co);
    upload_conv<T>(dst, w, b, ci, co, k, stride, a.padc(ci), a.padc(co), a.sp(in_level));
  };
  {
    const float* w = take((size_t)h->C[0] * 27);
    const float* b = take(h->C[0]);
    upload_stem<T>(h->stem, w, b, h->C[0], h->Cp[0]);
  }
  h->enc_a.resize(L);
  h->enc_b.resize(L);
  h->down.resize(L);
  h->up.resize(L);
  h->dec_a.resize(L);
  h->dec_b.resize(L);
  for (int l = 0; l < L; ++l) {
    conv(h->enc_a[l], h->C[l], 3, h->C[l], 1, l);
    conv(h->enc_b[l], h->C[l], 3, h->C[l], 1, a.xa_level(l));
    if (l < L - 1) conv(h->down[l], h->C[l + 1], 3, h->C[l], 2, l);
  }
  for (int l = L - 2; l >= 0; --l) {
    conv(h->up[l], h->C[l], 1, h->C[l + 1], 1, l + 1);
    conv(h->dec_a[l], h->C[l], 3, h->C[l], 1, l);
    conv(h->dec_b[l], h->C[l], 3, h->C[l], 1, a.xa_level(l));
  }
  {
    const float* w = take((size_t)kHead * h->C[0]);
    const float* b = take(kHead);
    h->Wpre.ensure((size_t)kHead * h->C[0] * 4);
    h->bpre.ensure(kHead * 4);
    OS_CUDA(cudaMemcpy(h->Wpre.p, w, (size_t)kHead * h->C[0] * 4, cudaMemcpyHostToDevice));
    OS_CUDA(cudaMemcpy(h->bpre.p, b, kHead * 4, cudaMemcpyHostToDevice));
  }
  {
    const float* w = take((size_t)kTheta * h->nin);
    const float* b = take(kTheta);
    h->Wc.ensure((size_t)kTheta * h->nin * 4);
    h->bc.ensure(kTheta * 4);
    OS_CUDA(cudaMemcpy(h->Wc.p, w, (size_t)kTheta * h->nin * 4, cudaMemcpyHostToDevice));
    OS_CUDA(cudaMemcpy(h->bc.p, b, kTheta * 4, cudaMemcpyHostToDevice));
  }
}

// Level widths P >> l must suit the 128-pixel M tile: multiple of 128 or divisor of 128.
void check_patch(const omniseg* h, int P) {
  const int L = h->arch.levels;
  OS_REQUIRE(P >= 16 && P % 16 == 0, "patch must be a positive multiple of 16");
  OS_REQUIRE(P % (1 << (L - 1)) == 0, "patch must be divisible by 2^(levels-1)");
  for (int l = 0; l < L; ++l) {
    const int w = P >> l;
    OS_REQUIRE(w % 128 == 0 || 128 % w == 0, "patch: level width " + std::to_string(w) +
                                                  " must be a multiple or a divisor of 128");
    OS_REQUIRE((int64_t)w * w >= 128, "patch: coarsest level must hold at least 128 pixels");
  }
}

// Allocate the per-batch workspace and build the convolution plans.
void ensure_workspace(omniseg* h, int P) {
  const int B = h->arch.batch;
  if (h->ws_P == P && h->ws_B == B) return;
  check_patch(h, P);
  const int L = h->arch.levels;
  const Arch& ar = h->arch;
  h->X0.ensure((size_t)B * P * P * 32 * 2);  // exact u8 values in 16-bit: never split
  h->lv.clear();
  h->lv.resize(L);
  for (int l = 0; l < L; ++l) {
    LevelBufs& q = h->lv[l];
    q.P = P >> l;
    q.C = h->Cp[l];
    const size_t n = (size_t)B * q.P * q.P * q.C * Arch::bpc(ar.sp(l));
    q.E.ensure(n);
    q.A.ensure(n);
    q.Bt.ensure(n);
  }
  h->g.ensure((size_t)B * h->C[L - 1] * 4);
  h->gpart.ensure(gap_scratch_floats(B, h->Cp[L - 1]) * 4);
  h->theta.ensure((size_t)B * kMaxTasks * kTheta * 4);
  h->theta_t.ensure((size_t)B * kMaxTasks * 156 * 4);
  const bool bf = ar.bf16;
  h->enc_plans.clear();
  h->dec_plans.clear();
  h->enc_layers.clear();
  h->dec_layers.clear();
  // Tensor layouts. Per level l: A_l (stem / down / up output = the RB input
  // and residual), Bt_l (conv_a output) and E_l (RB output: skip, down input; in the decoder
  // E_l then receives D_l, the next up-conv's input). A_l and Bt_l are read only by the 3x3
  // convs of their level: where those run the no-swizzle multi-row kernel (levels of width
  // >= 128 and <= 64 channels) they are stored row-chunked (RC) for its 128-B TMA rows; E_l
  // and every other tensor are NHWC.
  h->rc.assign(L, 0);
  for (int l = 0; l < L; ++l)
    h->rc[l] = nz_eligible(P >> l, P >> l, h->enc_a[l].cinp, h->enc_a[l].coutp, 3, 1, kReluBias) &&
               nz_eligible(P >> l, P >> l, h->enc_b[l].cinp, h->enc_b[l].coutp, 3, 1, kResidualRelu) &&
               !exp_flag("OMNISEG_NO_NZ");
  // out_level: U-Net level of the output (and residual / skip) tensor
  auto plan = [&](const Layer& ly, const void* in, int Hin, const void* res, void* out, int mode, int out_level,
                  int in_rc, int res_rc, int out_rc) {
    ConvPlan p = make_conv_plan(bf, in, B, Hin, Hin, ly.cinp, ly.w.p, ly.b.as<float>(), ly.coutp, ly.k, ly.stride,
                                mode, res, out, ar.sp(out_level), -1, -1, -1, ly.in_kind, ly.wlo.p, in_rc, res_rc,
                                out_rc);
    if (const size_t wb = conv_wimage_bytes(p)) {
      ly.wimg.ensure(wb);
      build_conv_wimage(p, ly.w.p, ly.wlo.p, ly.wimg.p, h->stream);
    }
    return p;
  };
  auto enc = [&](const Layer& ly, const void* in, int Hin, const void* res, void* out, int mode, int ol, int irc,
                 int rrc, int orc) {
    h->enc_plans.push_back(plan(ly, in, Hin, res, out, mode, ol, irc, rrc, orc));
    h->enc_layers.push_back(&ly);
  };
  auto dec = [&](const Layer& ly, const void* in, int Hin, const void* res, void* out, int mode, int ol, int irc,
                 int rrc, int orc) {
    h->dec_plans.push_back(plan(ly, in, Hin, res, out, mode, ol, irc, rrc, orc));
    h->dec_layers.push_back(&ly);
  };
  // E_l (the skip) is row-chunked too where the level is and its down conv can read it
  // (conv3s2_rc_kernel); the decoder's D_l reuses the E_l buffer in NHWC (the next up-conv's
  // per-tap A operand).
  h->erc.assign(L, 0);
  for (int l = 0; l + 1 < L; ++l)
    h->erc[l] = h->rc[l] && s2_eligible(P >> l, P >> l, h->down[l].cinp, h->down[l].coutp, 3, 2, kReluBias) &&
                h->down[l].coutp <= 128 &&  // 2x MMA work: up to N = 128 (down1: 78 -> 74 ms per cfg4 step)
                !exp_flag("OMNISEG_NO_S2");
  const auto& rc = h->rc;
  const auto& erc = h->erc;
  enc(h->stem, h->X0.p, P, nullptr, h->lv[0].A.p, kReluBias, 0, 0, 0, rc[0]);
  for (int l = 0; l < L; ++l) {
    LevelBufs& q = h->lv[l];
    enc(h->enc_a[l], q.A.p, q.P, nullptr, q.Bt.p, kReluBias, ar.xa_level(l), rc[l], 0, rc[l]);
    enc(h->enc_b[l], q.Bt.p, q.P, q.A.p, q.E.p, kResidualRelu, l, rc[l], rc[l], erc[l]);
    if (l < L - 1)
      enc(h->down[l], q.E.p, q.P, nullptr, h->lv[l + 1].A.p, kReluBias, l + 1, erc[l], 0, rc[l + 1]);
  }
  for (int l = L - 2; l >= 0; --l) {
    LevelBufs& q = h->lv[l];
    dec(h->up[l], h->lv[l + 1].E.p, q.P / 2, q.E.p, q.A.p, kUpAdd, l, 0, erc[l], rc[l]);
    dec(h->dec_a[l], q.A.p, q.P, nullptr, q.Bt.p, kReluBias, ar.xa_level(l), rc[l], 0, rc[l]);
    dec(h->dec_b[l], q.Bt.p, q.P, q.A.p, q.E.p, kResidualRelu, l, rc[l], rc[l], 0);
  }
  // fused window gather + stem
  h->stem_fused = stem_fusable(P, h->stem.coutp) && h->stem.cinp == 32;
  if (h->stem_fused) {
    // the stem kernel's epilogue stores 32-channel boxes (the per-tap output-only plan splits
    // the channels over 16-wide warp pairs): its output maps come from a residual-mode plan
    // of the same conv (no residual given), whose epilogue box is min(C, 32) channels wide
    ConvPlan mp = make_conv_plan(bf, h->X0.p, B, P, P, h->stem.cinp, h->stem.w.p, h->stem.b.as<float>(),
                                 h->stem.coutp, 1, 1, kResidualRelu, nullptr, h->lv[0].A.p, ar.sp(0), -1, -1, -1,
                                 kStorePlain, nullptr, 0, 0, rc[0]);
    mp.args.split = h->enc_plans[0].args.split;
    h->stem_plan = make_stem_plan(mp, h->stem.wpx.p, P);
  }
  // fused head: only with the no-swizzle kernel and all C0 channels in one N tile
  h->head_fusable = false;
  if (!exp_flag("OMNISEG_NO_HEAD_FUSION") && rc[0]) {
    LevelBufs& q = h->lv[0];
    ConvPlan hp = plan(h->dec_b[0], q.Bt.p, q.P, q.A.p, q.E.p,
                       h->arch.headtc ? kHeadFusedTc : kHeadFused, 0, rc[0], rc[0], 0);
    if (hp.nz_R > 0 && hp.bn == h->Cp[0] && h->C[0] <= 32) {
      h->head_plan = hp;
      h->head_fusable = true;
    }
  }
  h->ws_P = P;
  h->ws_B = B;
}

struct Tasks {
  int n = 0;
  int f[kMaxTasks], log2f[kMaxTasks], cls[kMaxTasks], scl[kMaxTasks];
  int64_t Ht[kMaxTasks], Wt[kMaxTasks], r0[kMaxTasks], r1[kMaxTasks];
  int factors[kMaxScales], nf = 0;  // distinct factors, descending
  int fmax = 1;
};

Tasks make_tasks(const omniseg* h, const int* scales, const int* classes, int n, int64_t H, int64_t W) {
  OS_REQUIRE(n >= 1 && n <= kMaxTasks, "n_tasks must be in [1, 32]");
  OS_REQUIRE(scales && classes, "scales/classes must not be NULL");
  Tasks t;
  t.n = n;
  bool used[4] = {false, false, false, false};
  for (int i = 0; i < n; ++i) {
    const auto& sc = h->arch.scale_codes;
    auto it = std::find(sc.begin(), sc.end(), scales[i]);
    OS_REQUIRE(it != sc.end(), "scale " + std::to_string(scales[i]) + " is not in scale_codes");
    OS_REQUIRE(scales[i] > 0 && h->arch.slide_mag % scales[i] == 0, "scale must divide slide_mag");
    const int f = h->arch.slide_mag / scales[i];
    OS_REQUIRE(f == 1 || f == 2 || f == 4 || f == 8, "level factor slide_mag/scale must be 1, 2, 4 or 8");
    OS_REQUIRE(classes[i] >= 0 && classes[i] < h->arch.ncls, "class index out of range");
    t.f[i] = f;
    t.log2f[i] = f == 1 ? 0 : f == 2 ? 1 : f == 4 ? 2 : 3;
    t.cls[i] = classes[i];
    t.scl[i] = (int)(it - sc.begin());
    t.Ht[i] = (H + f - 1) / f;
    t.Wt[i] = (W + f - 1) / f;
    used[t.log2f[i]] = true;
  }
  for (int l = 3; l >= 0; --l)
    if (used[l]) t.factors[t.nf++] = 1 << l;
  t.fmax = t.factors[0];
  return t;
}

void record(omniseg* h, int i) { OS_CUDA(cudaEventRecord(h->ev[i], h->stream)); }

// Algorithmic FLOPs of one conv launch over n tiles: 2 * M * N_real * K_real (real channel
// counts: no padding, no x2 doubling, stem K = 27).
double conv_alg_flops(const ConvPlan& p, const Layer& ly, int n) {
  const double M = (double)n * p.args.Ho * p.args.Wo;
  const double K = ly.alg_k ? ly.alg_k : (double)ly.k * ly.k * ly.cin;
  return 2.0 * M * ly.cout * K;
}

template <typename F>
void run_prof(omniseg* h, const ConvPlan& p, const Layer& ly, int layer_idx, int n, F&& launch) {
  if (h->profile) {
    if ((int)h->pev.size() < 2 * (h->pn + 1)) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        OS_CUDA(cudaEventCreate(&e));
        h->pev.push_back(e);
      }
    }
    OS_CUDA(cudaEventRecord(h->pev[2 * h->pn], h->stream));
    launch();
    OS_CUDA(cudaEventRecord(h->pev[2 * h->pn + 1], h->stream));
    if ((int)h->player.size() <= h->pn) {
      h->player.resize(h->pn + 1);
      h->pflops.resize(h->pn + 1);
    }
    h->player[h->pn] = layer_idx;
    h->pflops[h->pn] = conv_alg_flops(p, ly, n);
    h->pn++;
  } else {
    launch();
  }
}
void run_conv_prof(omniseg* h, const ConvPlan& p, const Layer& ly, int layer_idx, int n) {
  run_prof(h, p, ly, layer_idx, n, [&] { run_conv(p, h->stream); });
}

// Resolve the event pairs of the finished call into the accumulators.
void collect_profile(omniseg* h) {
  if (!h->profile) return;
  for (int i = 0; i < h->pn; ++i) {
    float ms = 0;
    OS_CUDA(cudaEventElapsedTime(&ms, h->pev[2 * i], h->pev[2 * i + 1]));
    const int l = h->player[i];
    if ((int)h->layer_ms.size() <= l) {
      h->layer_ms.resize(l + 1, 0);
      h->layer_flops.resize(l + 1, 0);
      h->layer_n.resize(l + 1, 0);
    }
    h->layer_ms[l] += ms;
    h->layer_flops[l] += h->pflops[i];
    h->layer_n[l] += 1;
    h->prof_ms += ms;
    h->prof_flops += h->pflops[i];
    h->prof_launches += 1;
  }
  h->pn = 0;
}

// Run trunk + GAP/controller + head for `n` tiles already gathered into X0.
void fill_head(HeadArgs& ha, omniseg* h, int ntasks, int P, int S, int Hp, int Wp, int pad, const uint32_t* tiles,
               int first, const HeadTaskTable& tt, float* out_p, float* out_F) {
  ha.Wpre = h->Wpre.as<float>();
  ha.bpre = h->bpre.as<float>();
  ha.theta = h->theta.as<float>();
  ha.theta_t = h->theta_t.as<float>();
  ha.ntasks = ntasks;
  ha.C0 = h->C[0];
  ha.P = P;
  ha.S = S;
  ha.Hp = Hp;
  ha.Wp = Wp;
  ha.pad = pad;
  ha.tiles = tiles;
  ha.first = first;
  ha.out_p = out_p;
  ha.out_F = out_F;
  ha.no_tc = exp_flag("OMNISEG_NO_TC_HEAD") ? 1 : 0;
  ha.tt = tt;
}

template <typename T>
void run_trunk_and_head(omniseg* h, int n, int P, const uint32_t* tiles, int first, bool stem_done, const HeadTaskTable& tt,
                        int ntasks, int S, int Hp, int Wp, int pad, float* out_p, float* out_F, float* out_g) {
  const int L = h->arch.levels;
  cudaStream_t s = h->stream;
  const size_t ne = h->enc_plans.size();
  // ---------------- encoder (the stem already ran fused with the window gather when stem_done)
  for (size_t i = stem_done ? 1 : 0; i < ne; ++i) {
    set_conv_batch(h->enc_plans[i], n);
    run_conv_prof(h, h->enc_plans[i], *h->enc_layers[i], (int)i, n);
    h->conv_launches++;
  }
  const LevelBufs& bl = h->lv[L - 1];
  launch_gap_controller<T>(bl.E.as<T>(), n, bl.P * bl.P, bl.C, h->arch.sp(L - 1), h->C[L - 1], h->Wc.as<float>(),
                           h->bc.as<float>(), h->arch.ncls, (int)h->arch.scale_codes.size(), h->task_cls.as<int>(),
                           h->task_scl.as<int>(), ntasks, h->gpart.as<float>(), h->g.as<float>(), h->theta.as<float>(),
                           h->theta_t.as<float>(), s);
  h->launches += 2;
  if (out_g) OS_CUDA(cudaMemcpyAsync(out_g, h->g.p, (size_t)n * h->C[L - 1] * 4, cudaMemcpyDefault, s));
  // ---------------- decoder
  const size_t ndec = h->dec_plans.size();
  const bool fuse = h->head_fusable && ntasks <= 8;
  bool head_done = false;
  for (size_t i = 0; i < ndec; ++i) {
    if (fuse && i + 1 == ndec) {
      ConvPlan& hp = h->head_plan;
      set_conv_batch(hp, n);
      fill_head(hp.head, h, ntasks, P, S, Hp, Wp, pad, tiles, first, tt, out_p, out_F);
      run_conv_prof(h, hp, *h->dec_layers[i], (int)(ne + i), n);
      head_done = true;
    } else {
      set_conv_batch(h->dec_plans[i], n);
      run_conv_prof(h, h->dec_plans[i], *h->dec_layers[i], (int)(ne + i), n);
    }
    h->conv_launches++;
  }
  if (!head_done) {
    launch_head<T>(h->lv[0].E.as<T>(), n, h->Cp[0], h->C[0], h->arch.sp(0), P, h->Wpre.as<float>(),
                   h->bpre.as<float>(), h->theta.as<float>(), ntasks, tiles, first, tt, S, Hp, Wp, pad, out_p, out_F, s);
    h->launches++;
  }
  OS_CUDA(cudaGetLastError());
}

// Batch-index offsets of a plan's input / residual / output / head-tile tensors.
void set_boffs(ConvPlan& p, int bin, int bres, int bout, int bhead = 0) {
  p.args.b_in = bin;
  p.args.b_res = bres;
  p.args.b_out = bout;
  p.args.b_head = bhead;
}

// The L2-resident schedule (arch grp / glev) of one batch of n windows whose
// gather + stem is fused: per group of G windows, the levels < GL run back to back with their
// stem / down / up outputs and conv_a outputs in the scratch slice [0, G) of the level buffers
// (rewritten by every group, so it stays in L2) and only the skips E_l in the windows' own
// slots; the levels >= GL and the GAP + controller run once over the batch; then per group the
// decoder levels < GL down to the fused head. Same kernels, same arithmetic per window: the
// outputs are bit-identical to the batch-wide schedule.
template <typename T>
void run_grouped(omniseg* h, int n, int P, const uint32_t* tiles, int first, const HeadTaskTable& tt, int ntasks, int S,
                 int Hp, int Wp, int pad, const uint32_t* const Lv[4]) {
  const int L = h->arch.levels, GL = std::min(h->arch.glev, L - 1), G = h->arch.grp;
  cudaStream_t s = h->stream;
  const size_t ne = h->enc_plans.size(), ndec = h->dec_plans.size();
  auto enc_idx = [](int l, int j) { return 1 + 3 * l + j; };          // j: 0 conv_a, 1 conv_b, 2 down
  auto dec_idx = [L](int l, int j) { return 3 * (L - 2 - l) + j; };  // j: 0 up, 1 conv_a, 2 conv_b
  auto run = [&](ConvPlan& p, size_t layer_list_idx, bool dec, int nn) {
    set_conv_batch(p, nn);
    run_conv_prof(h, p, dec ? *h->dec_layers[layer_list_idx] : *h->enc_layers[layer_list_idx],
                  (int)(dec ? ne + layer_list_idx : layer_list_idx), nn);
    h->conv_launches++;
  };
  // ---- encoder, levels < GL, per group
  for (int g0 = 0; g0 < n; g0 += G) {
    const int gn = std::min(G, n - g0);
    h->stem_plan.args.b_out = 0;
    run_prof(h, h->enc_plans[0], *h->enc_layers[0], 0, gn,
             [&] { run_stem(h->stem_plan, tiles, first + g0, gn, Lv, S, Hp, Wp, s); });
    h->conv_launches++;
    for (int l = 0; l < GL; ++l) {
      ConvPlan& a = h->enc_plans[enc_idx(l, 0)];
      ConvPlan& b = h->enc_plans[enc_idx(l, 1)];
      ConvPlan& d = h->enc_plans[enc_idx(l, 2)];
      set_boffs(a, 0, 0, 0);
      run(a, enc_idx(l, 0), false, gn);
      set_boffs(b, 0, 0, g0);  // E_l: the window's own slot (skip)
      run(b, enc_idx(l, 1), false, gn);
      set_boffs(d, g0, 0, l + 1 < GL ? 0 : g0);  // the batch phase reads A_GL per window
      run(d, enc_idx(l, 2), false, gn);
    }
  }
  // ---- levels >= GL over the batch
  for (size_t i = enc_idx(GL, 0); i < ne; ++i) {
    set_boffs(h->enc_plans[i], 0, 0, 0);
    run(h->enc_plans[i], i, false, n);
  }
  const LevelBufs& bl = h->lv[L - 1];
  launch_gap_controller<T>(bl.E.as<T>(), n, bl.P * bl.P, bl.C, h->arch.sp(L - 1), h->C[L - 1], h->Wc.as<float>(),
                           h->bc.as<float>(), h->arch.ncls, (int)h->arch.scale_codes.size(), h->task_cls.as<int>(),
                           h->task_scl.as<int>(), ntasks, h->gpart.as<float>(), h->g.as<float>(), h->theta.as<float>(),
                           h->theta_t.as<float>(), s);
  h->launches += 2;
  for (int l = L - 2; l >= GL; --l)
    for (int j = 0; j < 3; ++j) {
      set_boffs(h->dec_plans[dec_idx(l, j)], 0, 0, 0);
      run(h->dec_plans[dec_idx(l, j)], dec_idx(l, j), true, n);
    }
  // ---- decoder, levels < GL, per group, down to the fused head
  for (int g0 = 0; g0 < n; g0 += G) {
    const int gn = std::min(G, n - g0);
    for (int l = GL - 1; l >= 0; --l) {
      ConvPlan& u = h->dec_plans[dec_idx(l, 0)];
      ConvPlan& a = h->dec_plans[dec_idx(l, 1)];
      set_boffs(u, l + 1 >= GL ? g0 : 0, g0, 0);  // D_{l+1} (per window from the batch phase, else scratch), skip E_l
      run(u, dec_idx(l, 0), true, gn);
      set_boffs(a, 0, 0, 0);
      run(a, dec_idx(l, 1), true, gn);
      if (l > 0) {
        ConvPlan& b = h->dec_plans[dec_idx(l, 2)];
        set_boffs(b, 0, 0, 0);  // D_l into the scratch slice of E_l (its skips there are consumed)
        run(b, dec_idx(l, 2), true, gn);
      } else {
        ConvPlan& hp = h->head_plan;
        fill_head(hp.head, h, ntasks, P, S, Hp, Wp, pad, tiles, first, tt, nullptr, nullptr);
        set_boffs(hp, 0, 0, 0, g0);
        set_conv_batch(hp, gn);
        run_conv_prof(h, hp, *h->dec_layers[ndec - 1], (int)(ne + ndec - 1), gn);
        h->conv_launches++;
      }
    }
  }
  // back to the batch-wide offsets for the other entry points
  for (auto& p : h->enc_plans) set_boffs(p, 0, 0, 0);
  for (auto& p : h->dec_plans) set_boffs(p, 0, 0, 0);
  set_boffs(h->head_plan, 0, 0, 0, 0);
  OS_CUDA(cudaGetLastError());
}

void upload_tasks(omniseg* h, const Tasks& t) {
  h->task_cls.ensure(kMaxTasks * 4);
  h->task_scl.ensure(kMaxTasks * 4);
  OS_CUDA(cudaMemcpyAsync(h->task_cls.p, t.cls, t.n * 4, cudaMemcpyHostToDevice, h->stream));
  OS_CUDA(cudaMemcpyAsync(h->task_scl.p, t.scl, t.n * 4, cudaMemcpyHostToDevice, h->stream));
}

// One slide or one band. row0/row1: owned rows of the padded 40x frame.
template <typename T>
void segment(omniseg* h, const uint8_t* rgb, int64_t H, int64_t W, int64_t row0, int64_t row1, int64_t b0,
             int64_t b1, int pad, int P, int S, const Tasks& tk, float* out_prob, uint8_t* out_mask,
             uint64_t* out_area) {
  cudaStream_t s = h->stream;
  h->conv_launches = 0;
  h->launches = 0;
  const int Hp = (int)((H + 2 * pad + 127) / 128 * 128), Wp = (int)((W + 2 * pad + 127) / 128 * 128);
  const int H8 = Hp / 8, W8 = Wp / 8;
  h->H8 = H8;
  h->W8 = W8;
  NvtxRange nv_call("omniseg/segment");
  ensure_workspace(h, P);
  record(h, 0);
  // ---- upload (the band's slide rows [b0, b1))
  nvtxRangePushA("omniseg/upload");
  const int64_t rows = b1 - b0;
  const size_t slide_bytes = (size_t)rows * W * 3;
  const uint8_t* dslide = rgb;
  if (!is_device_ptr(rgb)) {
    h->slide.ensure(slide_bytes);
    OS_CUDA(cudaMemcpyAsync(h->slide.p, rgb, slide_bytes, cudaMemcpyHostToDevice, s));
    dslide = h->slide.as<uint8_t>();
  }
  nvtxRangePop();
  record(h, 1);
  // ---- front end
  nvtxRangePushA("omniseg/front_end");
  h->state.ensure(sizeof(DevState));
  DevState* st = h->state.as<DevState>();
  if (b0 == 0) launch_pad_colour(dslide, W, st, s);
  if (h->inject) OS_CUDA(cudaMemcpyAsync(st, h->inj_pc, 4, cudaMemcpyHostToDevice, s));
  if (h->comm) {
    g_nccl.check(g_nccl.broadcast(st, st, 4, ncclUint8, 0, h->comm, s), "ncclBroadcast(pad colour)");
  }
  bool needf[4] = {false, false, false, false};
  for (int i = 0; i < tk.n; ++i) needf[tk.log2f[i]] = true;
  const bool l1_needed = needf[0] && h->stem_fused && !exp_flag("OMNISEG_NO_STEM_FUSION");
  if (l1_needed) h->L1.ensure((size_t)Hp * Wp * 4);
  if (needf[1]) h->L2.ensure((size_t)(Hp / 2) * (Wp / 2) * 4);
  if (needf[2]) h->L4.ensure((size_t)(Hp / 4) * (Wp / 4) * 4);
  if (needf[3]) h->L8.ensure((size_t)H8 * W8 * 4);
  h->luma8.ensure((size_t)H8 * W8);
  h->gm.ensure((size_t)H8 * W8);
  h->fg.ensure((size_t)H8 * W8);
  // level-8 rows: fg needed on [m0, m1) (tiles touching the band), luma on m0-3 .. m1+3
  const int64_t halo = (int64_t)P * tk.fmax;
  const int m0 = (int)std::max<int64_t>(0, (row0 - halo) / 8), m1 = (int)std::min<int64_t>(H8, (row1 + halo + 7) / 8);
  const int l0 = std::max(0, m0 - 3), l1 = std::min(H8, m1 + 3);
  h->fg_r0 = m0;
  h->fg_r1 = m1;
  // slide rows needed: padded rows [8 l0, 8 l1) -> slide rows [8 l0 - pad, 8 l1 - pad) clipped to [0, H)
  const int64_t need0 = std::max<int64_t>(0, 8 * (int64_t)l0 - pad), need1 = std::min<int64_t>(H, 8 * (int64_t)l1 - pad);
  OS_REQUIRE(need1 <= need0 || (need0 >= b0 && need1 <= b1), "band: rgb_band does not hold the rows the halo needs");
  FrontParams fp{};
  fp.slide = dslide;
  fp.slide_row0 = b0;
  fp.slide_rows = rows;
  fp.H = H;
  fp.W = W;
  fp.pad = pad;
  fp.Hp = Hp;
  fp.Wp = Wp;
  fp.H8 = H8;
  fp.W8 = W8;
  fp.r8_0 = l0;
  fp.r8_1 = l1;
  fp.own8_0 = (int)(row0 / 8);
  fp.own8_1 = (int)(row1 / 8);
  launch_pyramid(fp, st, l1_needed ? h->L1.as<uint32_t>() : nullptr, needf[1] ? h->L2.as<uint32_t>() : nullptr,
                 needf[2] ? h->L4.as<uint32_t>() : nullptr,
                 needf[3] ? h->L8.as<uint32_t>() : nullptr, h->luma8.as<uint8_t>(), s);
  // the median reads luma rows [m0-3, m1+3) with edge replication only at the frame border
  launch_median(h->luma8.as<uint8_t>(), h->gm.as<uint8_t>(), H8, W8, m0, m1, s);
  h->hist.ensure(256 * 8);
  OS_CUDA(cudaMemsetAsync(h->hist.p, 0, 256 * 8, s));
  const int ir0 = pad / 8, ir1 = (int)(pad / 8 + H / 8), ic0 = pad / 8, ic1 = (int)(pad / 8 + W / 8);
  launch_hist(h->gm.as<uint8_t>(), W8, std::max(ir0, fp.own8_0), std::min(ir1, fp.own8_1), ic0, ic1,
              h->hist.as<unsigned long long>(), s);
  if (h->comm)
    g_nccl.check(g_nccl.allReduce(h->hist.p, h->hist.p, 256, ncclUint64, ncclSum, h->comm, s), "ncclAllReduce(hist)");
  if (h->inject) OS_CUDA(cudaMemcpyAsync(h->hist.p, h->inj_hist, 256 * 8, cudaMemcpyHostToDevice, s));
  OS_CUDA(cudaMemcpyAsync(h->last_hist, h->hist.p, 256 * 8, cudaMemcpyDeviceToHost, s));
  launch_otsu(h->hist.as<unsigned long long>(), st, s);
  // a band call of a multi-rank communicator always takes the exchange path (even a rank whose
  // band is the whole frame: the other ranks' empty bands join the same all-reduce)
  const bool partial = row0 > 0 || row1 < Hp || (h->comm && h->world > 1);
  if (h->arch.fgmin > 0 && partial) {
    // Tiny-component removal needs whole components: a band computes the foreground
    // of its OWNED level-8 rows only, the bands' disjoint rows are summed over the ranks
    // (ncclAllReduce of the H8 x W8 u8 grid: the union), and every rank labels the whole grid.
    OS_REQUIRE(h->comm || !h->inj_fg.empty(), "band fgmin needs a communicator (omniseg_comm_init)");
    OS_CUDA(cudaMemsetAsync(h->fg.p, 0, (size_t)H8 * W8, s));
    launch_fg(h->gm.as<uint8_t>(), h->fg.as<uint8_t>(), W8, std::max(m0, fp.own8_0), std::min(m1, fp.own8_1), ir0, ir1,
              ic0, ic1, st, s);
    if (h->comm)
      g_nccl.check(g_nccl.allReduce(h->fg.p, h->fg.p, (size_t)H8 * W8, ncclUint8, ncclSum, h->comm, s),
                   "ncclAllReduce(foreground)");
    if (!h->inj_fg.empty()) {
      OS_REQUIRE(h->inj_fg.size() == (size_t)H8 * W8, "injected foreground has the wrong size");
      OS_CUDA(cudaMemcpyAsync(h->fg.p, h->inj_fg.data(), h->inj_fg.size(), cudaMemcpyHostToDevice, s));
    }
    h->fg_r0 = 0;
    h->fg_r1 = H8;
    const size_t nfg = (size_t)H8 * W8;
    h->cc_lab.ensure(nfg * 4);
    h->cc_size.ensure(nfg * 4);
    launch_fg_components(h->fg.as<uint8_t>(), W8, 0, H8, h->arch.fgmin, h->cc_lab.as<int>(), h->cc_size.as<int>(), s);
  } else {
    launch_fg(h->gm.as<uint8_t>(), h->fg.as<uint8_t>(), W8, m0, m1, ir0, ir1, ic0, ic1, st, s);
    if (h->arch.fgmin > 0) {
      const size_t nfg = (size_t)(m1 - m0) * W8;
      h->cc_lab.ensure(nfg * 4);
      h->cc_size.ensure(nfg * 4);
      launch_fg_components(h->fg.as<uint8_t>(), W8, m0, m1, h->arch.fgmin, h->cc_lab.as<int>(), h->cc_size.as<int>(),
                           s);
    }
  }
  // candidate grids (canonical order: factor descending, row, col)
  std::vector<ScaleGrid> grids(tk.nf);
  int total = 0;
  for (int i = 0; i < tk.nf; ++i) {
    const int f = tk.factors[i];
    ScaleGrid& g = grids[i];
    g.f = f;
    g.log2f = f == 1 ? 0 : f == 2 ? 1 : f == 4 ? 2 : 3;
    g.Ey = Hp / f;
    g.Ex = Wp / f;
    OS_REQUIRE(g.Ey >= P && g.Ex >= P, "patch larger than the padded slide at some scale");
    g.ny = (g.Ey - P + S - 1) / S + 1;
    g.nx = (g.Ex - P + S - 1) / S + 1;
    OS_REQUIRE(g.ny < 32768 && g.nx < 32768, "tile grid too large");
    g.base = total;
    total += g.ny * g.nx;
  }
  h->grids.ensure(sizeof(ScaleGrid) * kMaxScales);
  OS_CUDA(cudaMemcpyAsync(h->grids.p, grids.data(), sizeof(ScaleGrid) * tk.nf, cudaMemcpyHostToDevice, s));
  h->keep.ensure(total);
  h->tiles.ensure((size_t)total * 4);
  h->counts.ensure((kMaxScales + 1) * 4);
  launch_tile_keep(h->fg.as<uint8_t>(), W8, h->grids.as<ScaleGrid>(), tk.nf, total, P, S, row0, row1,
                   h->keep.as<uint8_t>(), s);
  launch_compact(h->keep.as<uint8_t>(), total, h->grids.as<ScaleGrid>(), tk.nf, h->tiles.as<uint32_t>(),
                 h->counts.as<int>(), s);
  h->launches += 9;
  int counts[kMaxScales + 1];
  DevState hst;
  OS_CUDA(cudaMemcpyAsync(counts, h->counts.p, sizeof(counts), cudaMemcpyDeviceToHost, s));
  OS_CUDA(cudaMemcpyAsync(&hst, st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  OS_CUDA(cudaStreamSynchronize(s));
  h->n_tiles = counts[kMaxScales];
  h->otsu_t = hst.otsu_t;
  h->g_pad = hst.g_pad;
  nvtxRangePop();
  record(h, 2);
  // ---- canvases (owned rows only)
  HeadTaskTable tt{};
  tt.vote = h->arch.vote;
  int64_t canvas_px = 0;
  std::vector<int64_t> off(tk.n);
  std::vector<int64_t> r0(tk.n), r1(tk.n);
  for (int t = 0; t < tk.n; ++t) {
    omniseg_band_rows(H, row0, row1, pad, tk.f[t], &r0[t], &r1[t]);
    off[t] = canvas_px;
    canvas_px += (r1[t] - r0[t]) * tk.Wt[t];
  }
  h->canvas.ensure((size_t)std::max<int64_t>(canvas_px, 1) * 4);
  OS_CUDA(cudaMemsetAsync(h->canvas.p, 0, (size_t)canvas_px * 4, s));
  for (int t = 0; t < tk.n; ++t) {
    tt.canvas[t] = h->canvas.as<uint32_t>() + off[t];
    tt.Ht[t] = (int)tk.Ht[t];
    tt.Wt[t] = (int)tk.Wt[t];
    tt.row0[t] = (int)r0[t];
    tt.row1[t] = (int)r1[t];
    tt.log2f[t] = tk.log2f[t];
  }
  upload_tasks(h, tk);
  // ---- outputs: the caller's device buffers, or device staging + D2H for host buffers
  const bool prob_dev = is_device_ptr(out_prob), mask_dev = is_device_ptr(out_mask);
  float* dprob = nullptr;
  uint8_t* dmask = nullptr;
  if (out_prob) {
    if (prob_dev) dprob = out_prob;
    else {
      h->prob.ensure((size_t)std::max<int64_t>(canvas_px, 1) * 4);
      dprob = h->prob.as<float>();
    }
  }
  if (out_mask) {
    if (mask_dev) dmask = out_mask;
    else {
      h->mask.ensure((size_t)std::max<int64_t>(canvas_px, 1));
      dmask = h->mask.as<uint8_t>();
    }
  }
  h->area.ensure(kMaxTasks * 8);
  OS_CUDA(cudaMemsetAsync(h->area.p, 0, kMaxTasks * 8, s));
  // Host outputs are finalised and copied back PROGRESSIVELY: windows are ordered (scale
  // descending, row, column), so once the batch loop has passed a window row of scale f, the
  // canvas rows above the next pending window of that scale can no longer change. Those rows
  // are finalised on the compute stream and their D2H runs on a copy stream under the
  // remaining trunk work (bit-identical to finalising at the end).
  const bool host_out = (out_prob && !prob_dev) || (out_mask && !mask_dev);
  std::vector<int64_t> done(r0);
  auto finalize_rows = [&](int t, int64_t ra, int64_t rb) {
    if (rb <= ra) return;
    const int64_t base = off[t] + (ra - r0[t]) * tk.Wt[t], n = (rb - ra) * tk.Wt[t];
    FgMaskArgs fm;
    if (h->arch.maskfg) {
      fm.fg8 = h->fg.as<uint8_t>();
      fm.W8 = W8;
      fm.f = tk.f[t];
      fm.pad = pad;
      fm.Wt = (int)tk.Wt[t];
      fm.cy0 = ra;
    }
    launch_finalize(tt.canvas[t] + base - off[t], n, dprob ? dprob + base : nullptr, dmask ? dmask + base : nullptr,
                    h->area.as<unsigned long long>() + t, h->arch.vote, h->arch.vthr.empty() ? 0 : h->arch.vthr[tk.scl[t]],
                    fm, s);
    h->launches++;
    if (host_out) {
      OS_CUDA(cudaEventRecord(h->copy_ev, s));
      OS_CUDA(cudaStreamWaitEvent(h->copy_stream, h->copy_ev, 0));
      if (out_prob && !prob_dev)
        OS_CUDA(cudaMemcpyAsync(out_prob + base, dprob + base, (size_t)n * 4, cudaMemcpyDeviceToHost, h->copy_stream));
      if (out_mask && !mask_dev)
        OS_CUDA(cudaMemcpyAsync(out_mask + base, dmask + base, (size_t)n, cudaMemcpyDeviceToHost, h->copy_stream));
    }
    done[t] = rb;
  };
  // per-scale ranges of the (host copy of the) kept-window list
  int64_t sb[4] = {0, 0, 0, 0}, se[4] = {0, 0, 0, 0};
  if (host_out && h->n_tiles > 0) {
    h->h_tiles.resize(h->n_tiles);
    OS_CUDA(cudaMemcpyAsync(h->h_tiles.data(), h->tiles.p, h->n_tiles * 4, cudaMemcpyDeviceToHost, s));
    OS_CUDA(cudaStreamSynchronize(s));
    for (int l = 0; l < 4; ++l) sb[l] = se[l] = -1;
    for (int64_t i = 0; i < h->n_tiles; ++i) {
      const int l = h->h_tiles[i] >> 30;
      if (sb[l] < 0) sb[l] = i;
      se[l] = i + 1;
    }
  }
  auto progress = [&](int64_t k) {  // windows [0, k) are done
    for (int t = 0; t < tk.n; ++t) {
      const int l = tk.log2f[t], f = 1 << l;
      int64_t safe;
      if (sb[l] < 0 || k >= se[l]) safe = r1[t];
      else if (k <= sb[l]) safe = r0[t];
      else {
        const int ty = (h->h_tiles[k] >> 15) & 0x7FFF;
        const int64_t oy = std::min<int64_t>((int64_t)ty * S, Hp / f - P);
        safe = std::max(r0[t], std::min(r1[t], oy - pad / f));
      }
      if (safe - done[t] >= 256 || (safe == r1[t] && safe > done[t])) finalize_rows(t, done[t], safe);
    }
  };
  // ---- hot loop over batches of kept tiles
  const int B = h->arch.batch;
  const bool fused = h->stem_fused && !exp_flag("OMNISEG_NO_STEM_FUSION");
  const uint32_t* Lv[4] = {h->L1.as<uint32_t>(), h->L2.as<uint32_t>(), h->L4.as<uint32_t>(), h->L8.as<uint32_t>()};
  nvtxRangePushA("omniseg/windows");
  for (int64_t first = 0; first < h->n_tiles; first += B) {
    NvtxRange nv_batch("omniseg/batch");
    const int n = (int)std::min<int64_t>(B, h->n_tiles - first);
    if (fused && h->arch.grp > 0 && h->head_fusable && tk.n <= 8) {
      run_grouped<T>(h, n, P, h->tiles.as<uint32_t>(), (int)first, tt, tk.n, S, Hp, Wp, pad, Lv);
      if (host_out) progress(first + n);
      continue;
    }
    if (fused) {
      // window gather + stem in one kernel (A5 + the first conv of A6)
      run_prof(h, h->enc_plans[0], *h->enc_layers[0], 0, n, [&] {
        run_stem(h->stem_plan, h->tiles.as<uint32_t>(), (int)first, n, Lv, S, Hp, Wp, s);
      });
      h->conv_launches++;
    } else {
      launch_gather<T>(h->tiles.as<uint32_t>(), (int)first, n, P, S, fp, st, h->L2.as<uint32_t>(),
                       h->L4.as<uint32_t>(), h->L8.as<uint32_t>(), h->X0.as<T>(), s);
      h->launches++;
    }
    run_trunk_and_head<T>(h, n, P, h->tiles.as<uint32_t>(), (int)first, fused, tt, tk.n, S, Hp, Wp, pad, nullptr, nullptr,
                          nullptr);
    if (host_out) progress(first + n);
  }
  nvtxRangePop();
  record(h, 3);
  // ---- finalize the remaining rows
  NvtxRange nv_fin("omniseg/finalize");
  for (int t = 0; t < tk.n; ++t) finalize_rows(t, done[t], r1[t]);
  if (h->comm)
    g_nccl.check(g_nccl.allReduce(h->area.p, h->area.p, tk.n, ncclUint64, ncclSum, h->comm, s), "ncclAllReduce(area)");
  record(h, 4);
  if (host_out) {  // the compute stream waits for the progressive copies
    OS_CUDA(cudaEventRecord(h->copy_ev, h->copy_stream));
    OS_CUDA(cudaStreamWaitEvent(s, h->copy_ev, 0));
  }
  if (out_area) OS_CUDA(cudaMemcpyAsync(out_area, h->area.p, tk.n * 8, cudaMemcpyDefault, s));
  record(h, 5);
  OS_CUDA(cudaStreamSynchronize(s));
  collect_profile(h);
  float ms;
  auto el = [&](int a, int b) {
    OS_CUDA(cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]));
    return (double)ms;
  };
  for (double& v : h->timings) v = 0;
  h->timings[0] = el(0, 1);
  h->timings[1] = el(1, 2);
  h->timings[3] = el(2, 3);  // gather + trunk + gap/controller + head (per-kind split: bench.py)
  h->timings[6] = el(3, 4);
  h->timings[7] = el(4, 5);
  h->timings[8] = el(0, 5);
  h->timings[9] = h->conv_launches;
  h->timings[10] = h->conv_launches + h->launches;
}

// A rank whose band owns no rows (more ranks than 8*stride row units, dist.band_partition):
// no compute, but the same collective sequence as segment() -- receive the pad colour, add a
// zero histogram, add zero areas -- so the other ranks' NCCL calls complete.
void segment_empty(omniseg* h, int64_t H, int64_t W, int pad, const Tasks& tk, uint64_t* out_area) {
  cudaStream_t s = h->stream;
  h->conv_launches = 0;
  h->launches = 0;
  const int Hp = (int)((H + 2 * pad + 127) / 128 * 128), Wp = (int)((W + 2 * pad + 127) / 128 * 128);
  h->H8 = Hp / 8;
  h->W8 = Wp / 8;
  h->fg_r0 = h->fg_r1 = 0;
  h->n_tiles = 0;
  h->state.ensure(sizeof(DevState));
  DevState* st = h->state.as<DevState>();
  OS_CUDA(cudaMemsetAsync(st, 0, sizeof(DevState), s));
  if (h->inject) OS_CUDA(cudaMemcpyAsync(st, h->inj_pc, 4, cudaMemcpyHostToDevice, s));
  if (h->comm) g_nccl.check(g_nccl.broadcast(st, st, 4, ncclUint8, 0, h->comm, s), "ncclBroadcast(pad colour)");
  h->hist.ensure(256 * 8);
  OS_CUDA(cudaMemsetAsync(h->hist.p, 0, 256 * 8, s));
  if (h->comm)
    g_nccl.check(g_nccl.allReduce(h->hist.p, h->hist.p, 256, ncclUint64, ncclSum, h->comm, s), "ncclAllReduce(hist)");
  if (h->inject) OS_CUDA(cudaMemcpyAsync(h->hist.p, h->inj_hist, 256 * 8, cudaMemcpyHostToDevice, s));
  OS_CUDA(cudaMemcpyAsync(h->last_hist, h->hist.p, 256 * 8, cudaMemcpyDeviceToHost, s));
  launch_otsu(h->hist.as<unsigned long long>(), st, s);
  if (h->arch.fgmin > 0 && h->comm) {  // the band foreground exchange of segment() (zero rows)
    h->fg.ensure((size_t)h->H8 * h->W8);
    OS_CUDA(cudaMemsetAsync(h->fg.p, 0, (size_t)h->H8 * h->W8, s));
    g_nccl.check(g_nccl.allReduce(h->fg.p, h->fg.p, (size_t)h->H8 * h->W8, ncclUint8, ncclSum, h->comm, s),
                 "ncclAllReduce(foreground)");
  }
  h->area.ensure(kMaxTasks * 8);
  OS_CUDA(cudaMemsetAsync(h->area.p, 0, kMaxTasks * 8, s));
  if (h->comm)
    g_nccl.check(g_nccl.allReduce(h->area.p, h->area.p, tk.n, ncclUint64, ncclSum, h->comm, s), "ncclAllReduce(area)");
  if (out_area) OS_CUDA(cudaMemcpyAsync(out_area, h->area.p, tk.n * 8, cudaMemcpyDefault, s));
  DevState hst;
  OS_CUDA(cudaMemcpyAsync(&hst, st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  OS_CUDA(cudaStreamSynchronize(s));
  h->otsu_t = hst.otsu_t;
  h->g_pad = hst.g_pad;
  for (double& v : h->timings) v = 0;
}

int fail(const Error& e) {
  g_last_error = e.what();
  return e.code;
}

void validate_common(int64_t H, int64_t W, int pad, int P, int S, bool vote) {
  OS_REQUIRE(H >= 2 && W >= 2, "H and W must be >= 2");
  OS_REQUIRE(pad >= 0 && pad % 8 == 0, "pad must be a non-negative multiple of 8");
  OS_REQUIRE(S >= 8 && S <= P && S % 8 == 0, "stride must satisfy 8 <= stride <= patch, stride % 8 == 0");
  OS_REQUIRE(P % 8 == 0, "patch must be a multiple of 8");
  OS_REQUIRE((H / 8) * (W / 8) < (int64_t(1) << 28), "slide too large for the exact Otsu (interior >= 2^28 px)");
  const int per_axis = (P + S - 1) / S + 1;
  if (vote)
    OS_REQUIRE(per_axis * per_axis <= 65535, "vote fusion: coverage count could exceed 16 bits");
  else
    OS_REQUIRE(per_axis * per_axis <= 15, "coverage count could exceed 15: need (ceil(P/S)+1)^2 <= 15");
}

}  // namespace

// ==================================================================== C ABI
extern "C" {

omniseg_t* omniseg_create(const char* arch, const void* weights, size_t nbytes) {
  try {
    auto h = std::make_unique<omniseg>();
    h->arch = parse_arch(arch);
    if (h->arch.device >= 0) OS_CUDA(cudaSetDevice(h->arch.device));
    OS_CUDA(cudaGetDevice(&h->device));
    int major = 0, minor = 0;
    OS_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, h->device));
    OS_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, h->device));
    if (major != 10 || minor != 0)
      throw Error(-2, "libomniseg is built for sm_100a (B200); device is sm_" + std::to_string(major) +
                          std::to_string(minor));
    const int L = h->arch.levels;
    for (int l = 0; l < L; ++l) {
      h->C.push_back(h->arch.base << l);
      h->Cp.push_back(h->arch.padc(h->arch.base << l));
    }
    h->nin = h->C[L - 1] + h->arch.ncls + (int)h->arch.scale_codes.size();
    OS_REQUIRE(weights != nullptr, "weights is NULL");
    const size_t need = param_count(h->arch) * 4;
    OS_REQUIRE(nbytes == need, "weights: expected " + std::to_string(need) + " bytes, got " + std::to_string(nbytes));
    std::vector<float> blob(need / 4);
    OS_CUDA(cudaMemcpy(blob.data(), weights, need, cudaMemcpyDefault));
    if (h->arch.bf16)
      load_weights<__nv_bfloat16>(h.get(), blob.data());
    else
      load_weights<__half>(h.get(), blob.data());
    OS_CUDA(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
    OS_CUDA(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    OS_CUDA(cudaEventCreateWithFlags(&h->copy_ev, cudaEventDisableTiming));
    h->stream = h->own_stream;
    for (auto& e : h->ev) OS_CUDA(cudaEventCreate(&e));
    return h.release();
  } catch (const Error& e) {
    fail(e);
    return nullptr;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return nullptr;
  }
}

int omniseg_set_stream(omniseg_t* h, void* stream) {
  if (!h) return fail(Error(-1, "handle is NULL"));
  h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
  return 0;
}

int64_t omniseg_output_size(const omniseg_t* h, int64_t H, int64_t W, int scale) {
  if (!h || scale <= 0 || h->arch.slide_mag % scale) return -1;
  const int64_t f = h->arch.slide_mag / scale;
  return ((H + f - 1) / f) * ((W + f - 1) / f);
}

int omniseg_band_rows(int64_t H, int64_t row0, int64_t row1, int pad, int f, int64_t* r0_t, int64_t* r1_t) {
  if (f <= 0 || !r0_t || !r1_t) return fail(Error(-1, "band_rows: bad arguments"));
  const int64_t Ht = (H + f - 1) / f;
  auto cdiv = [](int64_t a, int64_t b) { return a >= 0 ? (a + b - 1) / b : -((-a) / b); };
  *r0_t = std::min<int64_t>(Ht, std::max<int64_t>(0, cdiv(row0 - pad, f)));
  *r1_t = std::min<int64_t>(Ht, std::max<int64_t>(0, cdiv(row1 - pad, f)));
  return 0;
}

int omniseg_segment_slide(omniseg_t* h, const uint8_t* rgb_u8, int64_t H, int64_t W, int pad, int patch, int stride,
                          const int* scales, const int* classes, int n_tasks, float* out_prob, uint8_t* out_mask,
                          uint64_t* out_area) {
  try {
    OS_REQUIRE(h != nullptr, "handle is NULL");
    OS_REQUIRE(rgb_u8 != nullptr, "rgb_u8 is NULL");
    OS_CUDA(cudaSetDevice(h->device));
    validate_common(H, W, pad, patch, stride, h->arch.vote != 0);
    Tasks tk = make_tasks(h, scales, classes, n_tasks, H, W);
    const int64_t Hp = (H + 2 * pad + 127) / 128 * 128;
    if (h->arch.bf16)
      segment<__nv_bfloat16>(h, rgb_u8, H, W, 0, Hp, 0, H, pad, patch, stride, tk, out_prob, out_mask, out_area);
    else
      segment<__half>(h, rgb_u8, H, W, 0, Hp, 0, H, pad, patch, stride, tk, out_prob, out_mask, out_area);
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(Error(-2, e.what()));
  }
}

int omniseg_comm_init(omniseg_t* h, const void* id, int world, int rank) {
  try {
    OS_REQUIRE(h && id, "comm_init: NULL argument");
    OS_REQUIRE(world >= 1 && rank >= 0 && rank < world, "comm_init: bad world/rank");
    OS_CUDA(cudaSetDevice(h->device));
    g_nccl.load();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    if (h->comm) g_nccl.commDestroy(h->comm);
    h->comm = nullptr;
    g_nccl.check(g_nccl.commInitRank(&h->comm, world, uid, rank), "ncclCommInitRank");
    h->world = world;
    h->rank = rank;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// Argument agreement of the band entry points: a check that fails on one rank only (a bad band,
// a host buffer on the root) would otherwise return on that rank and leave its peers blocked in
// the next collective. Every rank reports its verdict through one int all-reduce before any
// other collective, and all of them fail together (the failing rank with its own message).
static void agree_args(omniseg_t* h, const std::string& bad, const char* what) {
  if (!h->comm) {
    OS_REQUIRE(bad.empty(), bad);
    return;
  }
  cudaStream_t s = h->stream;
  h->flag.ensure(sizeof(int));
  const int mine = bad.empty() ? 0 : 1;
  OS_CUDA(cudaMemcpyAsync(h->flag.p, &mine, sizeof(int), cudaMemcpyHostToDevice, s));
  g_nccl.check(g_nccl.allReduce(h->flag.p, h->flag.p, 1, ncclInt32, ncclSum, h->comm, s),
               (std::string("ncclAllReduce(") + what + " arguments)").c_str());
  int nbad = 0;
  OS_CUDA(cudaMemcpyAsync(&nbad, h->flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  OS_CUDA(cudaStreamSynchronize(s));
  OS_REQUIRE(bad.empty(), bad);
  OS_REQUIRE(nbad == 0, std::string(what) + ": bad arguments on " + std::to_string(nbad) + " other rank(s)");
}

int omniseg_segment_band(omniseg_t* h, const uint8_t* rgb_band, int64_t H, int64_t W, int64_t row0, int64_t row1,
                         int pad, int patch, int stride, const int* scales, const int* classes, int n_tasks,
                         float* out_prob, uint8_t* out_mask, uint64_t* out_area) {
  try {
    OS_REQUIRE(h != nullptr, "handle is NULL");
    OS_CUDA(cudaSetDevice(h->device));
    Tasks tk;
    int64_t b0 = 0, b1 = 0;
    std::string bad;
    try {
      validate_common(H, W, pad, patch, stride, h->arch.vote != 0);
      tk = make_tasks(h, scales, classes, n_tasks, H, W);
      const int64_t Hp = (H + 2 * pad + 127) / 128 * 128;
      OS_REQUIRE(row0 >= 0 && row0 <= row1 && row1 <= Hp, "band: need 0 <= row0 <= row1 <= Hp");
      if (row0 == row1) {
        OS_REQUIRE(row0 > 0, "band 0 must not be empty (it holds the pad colour, the broadcast root)");
      } else {
        OS_REQUIRE(row0 % (8 * stride) == 0 && (row1 == Hp || row1 % (8 * stride) == 0),
                   "band: row0/row1 must be multiples of 8*stride (row1 may be Hp)");
        const int64_t halo = (int64_t)patch * tk.fmax + 64;
        b0 = std::max<int64_t>(0, std::min<int64_t>(H, row0 - pad - halo));
        b1 = std::max<int64_t>(0, std::min<int64_t>(H, row1 - pad + halo));
        OS_REQUIRE(b1 > b0 || rgb_band != nullptr, "band: empty");
        if (row0 == 0) OS_REQUIRE(b0 == 0, "band 0 must start at slide row 0");
      }
    } catch (const Error& e) {
      if (e.code != -1) throw;  // CUDA / allocation errors are not argument errors
      bad = e.what();
    }
    agree_args(h, bad, "segment_band");
    if (row0 == row1) {  // an empty band: collectives only
      segment_empty(h, H, W, pad, tk, out_area);
      return 0;
    }
    if (h->arch.bf16)
      segment<__nv_bfloat16>(h, rgb_band, H, W, row0, row1, b0, b1, pad, patch, stride, tk, out_prob, out_mask,
                             out_area);
    else
      segment<__half>(h, rgb_band, H, W, row0, row1, b0, b1, pad, patch, stride, tk, out_prob, out_mask, out_area);
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(Error(-2, e.what()));
  }
}

int omniseg_gather_bands(omniseg_t* h, int root, int64_t H, int64_t W, int pad, const int64_t* cuts,
                         const int* scales, int n_tasks, const float* band_prob, const uint8_t* band_mask,
                         float* out_prob, uint8_t* out_mask) {
  try {
    OS_REQUIRE(h && cuts && scales, "gather_bands: NULL argument");
    OS_REQUIRE(h->comm != nullptr, "gather_bands: needs omniseg_comm_init");
    OS_REQUIRE(root >= 0 && root < h->world, "gather_bands: bad root");
    OS_CUDA(cudaSetDevice(h->device));
    std::vector<int> classes(n_tasks, 0);
    const Tasks tk = make_tasks(h, scales, classes.data(), n_tasks, H, W);
    const int64_t Hp = (H + 2 * pad + 127) / 128 * 128;
    OS_REQUIRE(cuts[0] == 0 && cuts[h->world] == Hp, "gather_bands: cuts must run from 0 to Hp");
    for (int r = 0; r < h->world; ++r) OS_REQUIRE(cuts[r] <= cuts[r + 1], "gather_bands: cuts must be ascending");
    const bool me_root = h->rank == root;
    cudaStream_t s = h->stream;
    NvtxRange nv("omniseg/gather_bands");
    // Per-rank buffer checks can fail on one rank only (e.g. a host out_prob on the root); a
    // rank that returned here would leave its peers blocked in the send / recv group. So every
    // rank reports its verdict through one tiny all-reduce first, and all of them fail together.
    std::string bad;
    if (band_prob && !is_device_ptr(band_prob)) bad = "gather_bands: band_prob must be device memory";
    if (band_mask && !is_device_ptr(band_mask)) bad = "gather_bands: band_mask must be device memory";
    if (me_root && !((!band_prob || (out_prob && is_device_ptr(out_prob))) &&
                     (!band_mask || (out_mask && is_device_ptr(out_mask)))))
      bad = "gather_bands: the root needs device out_prob / out_mask for every band output given";
    agree_args(h, bad, "gather_bands");
    // per task: offset of the task in the full output and in each rank's band output
    std::vector<int64_t> full_off(tk.n);
    int64_t acc = 0;
    for (int t = 0; t < tk.n; ++t) {
      full_off[t] = acc;
      acc += tk.Ht[t] * tk.Wt[t];
    }
    g_nccl.check(g_nccl.groupStart(), "ncclGroupStart");
    for (int r = 0; r < h->world; ++r) {
      if (!me_root && r != h->rank) continue;
      int64_t boff = 0;
      for (int t = 0; t < tk.n; ++t) {
        int64_t r0, r1;
        omniseg_band_rows(H, cuts[r], cuts[r + 1], pad, tk.f[t], &r0, &r1);
        const int64_t n = (r1 - r0) * tk.Wt[t];
        if (n > 0) {
          const int64_t dst = full_off[t] + r0 * tk.Wt[t];
          if (r == h->rank) {  // my band: send to the root (a self send/recv pair on the root)
            if (band_prob) g_nccl.check(g_nccl.send(band_prob + boff, n, ncclFloat32, root, h->comm, s), "ncclSend");
            if (band_mask) g_nccl.check(g_nccl.send(band_mask + boff, n, ncclUint8, root, h->comm, s), "ncclSend");
          }
          if (me_root) {
            if (band_prob) g_nccl.check(g_nccl.recv(out_prob + dst, n, ncclFloat32, r, h->comm, s), "ncclRecv");
            if (band_mask) g_nccl.check(g_nccl.recv(out_mask + dst, n, ncclUint8, r, h->comm, s), "ncclRecv");
          }
        }
        boff += n;
      }
    }
    g_nccl.check(g_nccl.groupEnd(), "ncclGroupEnd");
    OS_CUDA(cudaStreamSynchronize(s));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(Error(-2, e.what()));
  }
}

int omniseg_render_overlay(omniseg_t* h, const uint8_t* rgb_u8, int64_t H, int64_t W, const uint8_t* masks,
                           const int* scales, const int* classes, int n_tasks, uint8_t* out40, uint8_t* out10) {
  try {
    OS_REQUIRE(h && rgb_u8 && masks, "render_overlay: NULL argument");
    OS_REQUIRE(out40 || out10, "render_overlay: no output requested");
    OS_REQUIRE(H >= 1 && W >= 1, "render_overlay: bad size");
    OS_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    const Tasks tk = make_tasks(h, scales, classes, n_tasks, H, W);
    for (int t = 0; t < tk.n; ++t) OS_REQUIRE(tk.cls[t] < 6, "render_overlay: palette has 6 classes");
    int64_t mtot = 0;
    std::vector<int64_t> moff(tk.n);
    for (int t = 0; t < tk.n; ++t) {
      moff[t] = mtot;
      mtot += tk.Ht[t] * tk.Wt[t];
    }
    const uint8_t* dslide = rgb_u8;
    if (!is_device_ptr(rgb_u8)) {
      h->r_slide.ensure((size_t)H * W * 3);
      OS_CUDA(cudaMemcpyAsync(h->r_slide.p, rgb_u8, (size_t)H * W * 3, cudaMemcpyHostToDevice, s));
      dslide = h->r_slide.as<uint8_t>();
    }
    const uint8_t* dmask = masks;
    if (!is_device_ptr(masks)) {
      h->r_mask.ensure((size_t)mtot);
      OS_CUDA(cudaMemcpyAsync(h->r_mask.p, masks, (size_t)mtot, cudaMemcpyHostToDevice, s));
      dmask = h->r_mask.as<uint8_t>();
    }
    RenderTasks rt{};
    rt.n = tk.n;
    for (int t = 0; t < tk.n; ++t) {
      rt.m[t] = dmask + moff[t];
      rt.f[t] = tk.f[t];
      rt.lf[t] = tk.log2f[t];
      rt.Wt[t] = (int)tk.Wt[t];
      rt.cls[t] = tk.cls[t];
    }
    uint8_t* d40 = out40;
    if (!out40 || !is_device_ptr(out40)) {
      h->r_40.ensure((size_t)H * W * 3);
      d40 = h->r_40.as<uint8_t>();
    }
    const int64_t n10 = ((H + 3) / 4) * ((W + 3) / 4) * 3;
    uint8_t* d10 = nullptr;
    if (out10) {
      d10 = out10;
      if (!is_device_ptr(out10)) {
        h->r_10.ensure((size_t)n10);
        d10 = h->r_10.as<uint8_t>();
      }
    }
    launch_overlay(dslide, H, W, rt, d40, d10, s);
    OS_CUDA(cudaGetLastError());
    if (out40 && d40 != out40) OS_CUDA(cudaMemcpyAsync(out40, d40, (size_t)H * W * 3, cudaMemcpyDeviceToHost, s));
    if (out10 && d10 != out10) OS_CUDA(cudaMemcpyAsync(out10, d10, (size_t)n10, cudaMemcpyDeviceToHost, s));
    OS_CUDA(cudaStreamSynchronize(s));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(Error(-2, e.what()));
  }
}

int omniseg_get_tiles(const omniseg_t* h, uint32_t* tiles, int64_t cap, int64_t* n) {
  try {
    OS_REQUIRE(h && n, "get_tiles: NULL argument");
    *n = h->n_tiles;
    if (tiles && cap > 0 && h->n_tiles > 0)
      OS_CUDA(cudaMemcpy(tiles, h->tiles.p, std::min<int64_t>(cap, h->n_tiles) * 4, cudaMemcpyDeviceToHost));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

int omniseg_get_fgmask(const omniseg_t* h, uint8_t* mask, int64_t cap, int64_t* h8, int64_t* w8, int* otsu_t,
                       int* g_pad) {
  try {
    OS_REQUIRE(h, "get_fgmask: NULL handle");
    if (h8) *h8 = h->H8;
    if (w8) *w8 = h->W8;
    if (otsu_t) *otsu_t = h->otsu_t;
    if (g_pad) *g_pad = h->g_pad;
    const int64_t n = (int64_t)h->H8 * h->W8;
    if (mask && cap >= n && n > 0) {
      // rows outside [fg_r0, fg_r1) were not computed by this call: report them as 0
      std::memset(mask, 0, n);
      const int64_t a = h->fg_r0 * h->W8, b = h->fg_r1 * h->W8;
      if (b > a) OS_CUDA(cudaMemcpy(mask + a, h->fg.as<uint8_t>() + a, b - a, cudaMemcpyDeviceToHost));
    }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

int omniseg_get_timings(const omniseg_t* h, double* out, int cap) {
  if (!h || !out) return fail(Error(-1, "get_timings: NULL argument"));
  for (int i = 0; i < cap && i < 11; ++i) out[i] = h->timings[i];
  return 0;
}

const char* omniseg_last_error(void) { return g_last_error.c_str(); }

void omniseg_destroy(omniseg_t* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  delete h;
}

// ---------------------------------------------------------------- debug entry points
int omniseg_debug_predict_tiles(omniseg_t* h, const uint8_t* tiles_u8, int n, int P, const int* cls, const int* scl,
                                int n_tasks, float* out_p, float* out_g, float* out_F) {
  try {
    OS_REQUIRE(h && tiles_u8 && cls && scl && out_p, "predict_tiles: NULL argument");
    OS_REQUIRE(n >= 1 && n <= h->arch.batch, "predict_tiles: 1 <= n <= batch");
    OS_REQUIRE(n_tasks >= 1 && n_tasks <= kMaxTasks, "predict_tiles: bad n_tasks");
    OS_CUDA(cudaSetDevice(h->device));
    for (int t = 0; t < n_tasks; ++t) {
      OS_REQUIRE(cls[t] >= 0 && cls[t] < h->arch.ncls, "predict_tiles: class out of range");
      OS_REQUIRE(scl[t] >= 0 && scl[t] < (int)h->arch.scale_codes.size(), "predict_tiles: scale index out of range");
    }
    ensure_workspace(h, P);
    cudaStream_t s = h->stream;
    DevBuf dt, dp, dF, dg;
    const uint8_t* src = tiles_u8;
    const size_t tb = (size_t)n * P * P * 3;
    if (!is_device_ptr(tiles_u8)) {
      dt.ensure(tb);
      OS_CUDA(cudaMemcpyAsync(dt.p, tiles_u8, tb, cudaMemcpyHostToDevice, s));
      src = dt.as<uint8_t>();
    }
    Tasks tk;
    tk.n = n_tasks;
    for (int t = 0; t < n_tasks; ++t) {
      tk.cls[t] = cls[t];
      tk.scl[t] = scl[t];
    }
    upload_tasks(h, tk);
    dp.ensure((size_t)n * n_tasks * P * P * 4);
    if (out_F) dF.ensure((size_t)n * P * P * kHead * 4);
    if (out_g) dg.ensure((size_t)n * h->C[h->arch.levels - 1] * 4);
    HeadTaskTable tt{};
    if (h->arch.bf16) {
      launch_gather_raw<__nv_bfloat16>(src, n, P, h->X0.as<__nv_bfloat16>(), s);
      run_trunk_and_head<__nv_bfloat16>(h, n, P, nullptr, 0, false, tt, n_tasks, P, P, P, 0, dp.as<float>(),
                                        out_F ? dF.as<float>() : nullptr, out_g ? dg.as<float>() : nullptr);
    } else {
      launch_gather_raw<__half>(src, n, P, h->X0.as<__half>(), s);
      run_trunk_and_head<__half>(h, n, P, nullptr, 0, false, tt, n_tasks, P, P, P, 0, dp.as<float>(),
                                 out_F ? dF.as<float>() : nullptr, out_g ? dg.as<float>() : nullptr);
    }
    OS_CUDA(cudaMemcpyAsync(out_p, dp.p, (size_t)n * n_tasks * P * P * 4, cudaMemcpyDefault, s));
    if (out_F) OS_CUDA(cudaMemcpyAsync(out_F, dF.p, (size_t)n * P * P * kHead * 4, cudaMemcpyDefault, s));
    if (out_g) OS_CUDA(cudaMemcpyAsync(out_g, dg.p, (size_t)n * h->C[h->arch.levels - 1] * 4, cudaMemcpyDefault, s));
    OS_CUDA(cudaStreamSynchronize(s));
    collect_profile(h);
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(Error(-2, e.what()));
  }
}

int omniseg_debug_conv(omniseg_t* h, const float* x, int B, int H, int W, int Cin, const float* w, const float* b,
                       int Cout, int k, int stride, const float* r, int mode, float* y) {
  try {
    OS_REQUIRE(h && x && w && b && y, "debug_conv: NULL argument");
    // mode | 16: x2 storage of input / residual / output; mode | 32: f8 storage; mode | 64:
    // residual (not an up-add skip) and output row-chunked. The input is row-chunked exactly
    // when the no-swizzle multi-row kernel applies (its only layout).
    const int split = (mode & 32) ? kStoreF8 : (mode & 16) ? kStoreX2 : kStorePlain;
    const bool orc_req = (mode & 64) != 0;
    const bool res_nhwc = (mode & 128) != 0;  // mode | 128: residual / skip NHWC even with an RC output
    mode &= 15;
    OS_REQUIRE(mode >= 0 && mode <= 3, "debug_conv: bad mode");
    OS_REQUIRE((mode != 1 && mode != 2) || r, "debug_conv: mode needs r");
    OS_REQUIRE(mode != 2 || (k == 1 && stride == 1), "debug_conv: mode 2 is a 1x1 stride-1 conv");
    OS_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    const bool bf = h->arch.bf16;
    const int pc = split == kStoreF8 ? 32 : 16;
    const int cinp = (Cin + pc - 1) / pc * pc, coutp = (Cout + pc - 1) / pc * pc;
    const int Ho = (H - 1) / stride + 1, Wo = (W - 1) / stride + 1;
    const int oh = mode == 2 ? 2 * Ho : Ho, ow = mode == 2 ? 2 * Wo : Wo;
    const int sm = split == kStoreX2 ? 2 : 1;
    const int bpc = Arch::bpc(split);
    Layer L;
    std::vector<float> wv(w, w + (size_t)Cout * k * k * Cin), bv(b, b + Cout);
    if (bf)
      upload_conv<__nv_bfloat16>(L, wv.data(), bv.data(), Cin, Cout, k, stride, cinp, coutp, split);
    else
      upload_conv<__half>(L, wv.data(), bv.data(), Cin, Cout, k, stride, cinp, coutp, split);
    DevBuf f32in, xin, rin, f32r, out, f32o;
    const int64_t rows_in = (int64_t)B * H * W, rows_out = (int64_t)B * oh * ow;
    f32in.ensure(rows_in * Cin * 4);
    xin.ensure(rows_in * cinp * bpc);
    OS_CUDA(cudaMemcpyAsync(f32in.p, x, rows_in * Cin * 4, cudaMemcpyHostToDevice, s));
    if (r) {
      f32r.ensure(rows_out * Cout * 4);
      rin.ensure(rows_out * coutp * bpc);
      OS_CUDA(cudaMemcpyAsync(f32r.p, r, rows_out * Cout * 4, cudaMemcpyHostToDevice, s));
    }
    out.ensure(rows_out * coutp * bpc);
    f32o.ensure(rows_out * Cout * 4);
    const int in_rc = (nz_eligible(H, W, cinp * sm, coutp, k, stride, mode) ||
                       (orc_req && s2_eligible(H, W, cinp * sm, coutp, k, stride, mode))) ? 1 : 0;
    const int out_rc = orc_req && ow >= 128 && ow % 128 == 0 ? 1 : 0;
    const int res_rc = res_nhwc ? 0 : out_rc;
    if (bf) {
      launch_f32_to_t<__nv_bfloat16>(f32in.as<float>(), xin.as<__nv_bfloat16>(), rows_in, Cin, cinp, split,
                                     in_rc ? W : 0, s);
      if (r)
        launch_f32_to_t<__nv_bfloat16>(f32r.as<float>(), rin.as<__nv_bfloat16>(), rows_out, Cout, coutp, split,
                                       res_rc ? ow : 0, s);
    } else {
      launch_f32_to_t<__half>(f32in.as<float>(), xin.as<__half>(), rows_in, Cin, cinp, split, in_rc ? W : 0, s);
      if (r)
        launch_f32_to_t<__half>(f32r.as<float>(), rin.as<__half>(), rows_out, Cout, coutp, split, res_rc ? ow : 0, s);
    }
    ConvPlan p = make_conv_plan(bf, xin.p, B, H, W, cinp * sm, L.w.p, L.b.as<float>(), coutp, k, stride, mode,
                                r ? rin.p : nullptr, out.p, split, -1, -1, -1, split, L.wlo.p, in_rc, res_rc, out_rc);
    if (const size_t wb = conv_wimage_bytes(p)) {
      L.wimg.ensure(wb);
      build_conv_wimage(p, L.w.p, L.wlo.p, L.wimg.p, s);
    }
    run_conv(p, s);
    if (bf)
      launch_t_to_f32<__nv_bfloat16>(out.as<__nv_bfloat16>(), f32o.as<float>(), rows_out, Cout, coutp, split,
                                     out_rc ? ow : 0, s);
    else
      launch_t_to_f32<__half>(out.as<__half>(), f32o.as<float>(), rows_out, Cout, coutp, split, out_rc ? ow : 0, s);
    OS_CUDA(cudaMemcpyAsync(y, f32o.p, rows_out * Cout * 4, cudaMemcpyDeviceToHost, s));
    OS_CUDA(cudaStreamSynchronize(s));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(Error(-2, e.what()));
  }
}

int omniseg_debug_band_globals(omniseg_t* h, const uint8_t* pc, const uint64_t* hist) {
  if (!h) return fail(Error(-1, "band_globals: NULL handle"));
  if (!pc || !hist) {
    h->inject = false;
    return 0;
  }
  h->inject = true;
  for (int c = 0; c < 3; ++c) h->inj_pc[c] = pc[c];
  h->inj_pc[3] = 0;
  for (int i = 0; i < 256; ++i) h->inj_hist[i] = hist[i];
  return 0;
}

int omniseg_debug_band_fg(omniseg_t* h, const uint8_t* fg8, int64_t n) {
  if (!h) return fail(Error(-1, "band_fg: NULL handle"));
  if (!fg8 || n <= 0) {
    h->inj_fg.clear();
    return 0;
  }
  h->inj_fg.assign(fg8, fg8 + n);
  return 0;
}

int omniseg_debug_get_detection(const omniseg_t* h, uint8_t* pc, uint64_t* hist) {
  try {
    OS_REQUIRE(h && pc && hist, "get_detection: NULL argument");
    DevState st;
    OS_CUDA(cudaMemcpy(&st, h->state.p, sizeof(st), cudaMemcpyDeviceToHost));
    for (int c = 0; c < 3; ++c) pc[c] = st.pc[c];
    for (int i = 0; i < 256; ++i) hist[i] = h->last_hist[i];
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

int omniseg_debug_set_profile(omniseg_t* h, int on) {
  if (!h) return fail(Error(-1, "set_profile: NULL handle"));
  h->profile = on != 0;
  h->pn = 0;
  h->layer_ms.clear();
  h->layer_flops.clear();
  h->layer_n.clear();
  h->prof_ms = h->prof_flops = h->prof_launches = 0;
  return 0;
}

int omniseg_debug_get_profile(const omniseg_t* h, double* out, int cap, int* n_layers) {
  if (!h || !out) return fail(Error(-1, "get_profile: NULL argument"));
  const int nl = (int)h->layer_ms.size();
  if (n_layers) *n_layers = nl;
  std::vector<double> v = {h->prof_ms, h->prof_flops, h->prof_launches};
  for (int l = 0; l < nl; ++l) {
    v.push_back(h->layer_ms[l]);
    v.push_back(h->layer_flops[l]);
    v.push_back(h->layer_n[l]);
  }
  for (int i = 0; i < cap && i < (int)v.size(); ++i) out[i] = v[i];
  return 0;
}

}  // extern "C"
