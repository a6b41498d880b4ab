// kernels.h -- host launchers of the non-GEMM kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace osg {

// Small device-resident state of one segment call.
struct DevState {
  uint8_t pc[4];   // pad colour (R, G, B, 0)
  int otsu_t;
  int g_pad;       // luma of the pad colour
  int pad_;
};


void launch_pad_colour(const uint8_t* slide, int64_t W, DevState* st, cudaStream_t s);
void launch_pyramid(const FrontParams& p, const DevState* st, uint32_t* L1, uint32_t* L2, uint32_t* L4, uint32_t* L8,
                    uint8_t* luma8, cudaStream_t s);
void launch_median(const uint8_t* g, uint8_t* out, int H8, int W8, int r0, int r1, cudaStream_t s);
void launch_hist(const uint8_t* gm, int W8, int r0, int r1, int c0, int c1, unsigned long long* hist, cudaStream_t s);
void launch_otsu(const unsigned long long* hist, DevState* st, cudaStream_t s);
void launch_fg(const uint8_t* gm, uint8_t* fg, int W8, int r0, int r1, int ir0, int ir1, int ic0, int ic1,
               const DevState* st, cudaStream_t s);
void launch_tile_keep(const uint8_t* fg, int W8, const ScaleGrid* grids, int nscales, int total, int P, int S,
                      int64_t own0, int64_t own1, uint8_t* keep, cudaStream_t s);
void launch_compact(const uint8_t* keep, int total, const ScaleGrid* grids, int nscales, uint32_t* tiles, int* counts,
                    cudaStream_t s);
template <typename T>
void launch_gather(const uint32_t* tiles, int first, int n, int P, int S, const FrontParams& fp, const DevState* st,
                   const uint32_t* L2, const uint32_t* L4, const uint32_t* L8, T* X, cudaStream_t s);
template <typename T>
void launch_gather_raw(const uint8_t* tiles, int n, int P, T* X, cudaStream_t s);
template <typename T>
void launch_gap_controller(const T* E, int n, int hw, int C, int split, int Cb, const float* Wc, const float* bc,
                           int ncls, int nscl, const int* task_cls, const int* task_scl, int ntasks, float* part,
                           float* g, float* theta, float* theta_t, cudaStream_t s);
size_t gap_scratch_floats(int n, int C);
template <typename T>
void launch_head(const T* D0, int n, int C0p, int C0, int split, int P, const float* Wpre, const float* bpre,
                 const float* theta, int ntasks, const uint32_t* tiles, int first, const HeadTaskTable& tt, int S,
                 int Hp, int Wp, int pad, float* out_p, float* out_F, cudaStream_t s);
// N3 render: per task its mask (task-scale canvas, row stride Wt), level factor, class code.
struct RenderTasks {
  const uint8_t* m[kMaxTasks];
  int f[kMaxTasks], lf[kMaxTasks], Wt[kMaxTasks], cls[kMaxTasks];
  int n;
};
void launch_overlay(const uint8_t* slide, int64_t H, int64_t W, const RenderTasks& rt, uint8_t* out40, uint8_t* out10,
                    cudaStream_t s);
// Optional foreground filter of the finalized mask: canvas row of element 0 = cy0.
struct FgMaskArgs {
  const uint8_t* fg8 = nullptr;  // level-8 foreground (full grid, row stride W8); NULL: off
  int W8 = 0, f = 1, pad = 0, Wt = 1;
  int64_t cy0 = 0;
};
// vote: 0 mean fusion, 1 hard vote; vthr (vote only): 0 = majority ("at least half"), else the
// literal vote-count threshold min(vthr, coverage) (arch key vthr).
void launch_finalize(const uint32_t* acc, int64_t n, float* prob, uint8_t* mask, unsigned long long* area, int vote,
                     int vthr, const FgMaskArgs& fm, cudaStream_t s);
// Tiny-component removal on level-8 foreground rows [r0, r1) (lab, size: scratch of
// (r1 - r0) W ints each).
void launch_fg_components(uint8_t* fg, int W, int r0, int r1, int min_area, int* lab, int* size, cudaStream_t s);
template <typename T>
void launch_f32_to_t(const float* in, T* out, int64_t rows, int cin, int cpad, int split, int rc_w, cudaStream_t s);
template <typename T>
void launch_t_to_f32(const T* in, float* out, int64_t rows, int cout, int cpad, int split, int rc_w, cudaStream_t s);

// conv_tc.cu
struct ConvPlan;  // opaque per-layer plan (TMA maps + launch config)

}  // namespace osg
