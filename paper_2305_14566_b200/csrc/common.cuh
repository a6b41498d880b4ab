// common.cuh -- shared types of the omniseg kernels and the C-ABI orchestrator.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace osg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define OS_CUDA(call)                                                                             \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      throw ::osg::Error(-2, std::string(#call " failed: ") + cudaGetErrorString(e_) + " at " + \
                                     __FILE__ + ":" + std::to_string(__LINE__));                  \
  } while (0)

#define OS_REQUIRE(cond, msg)                                  \
  do {                                                         \
    if (!(cond)) throw ::osg::Error(-1, std::string(msg)); \
  } while (0)

// Experiment switches (DESIGN.md §8 "measured non-wins": kernel-variant toggles, MMA-warp cycle
// counters). Compiled OUT of the product build; `scripts/build_variant.sh NAME
// -DOMNISEG_EXPERIMENTS=1` builds a variant that reads the toggles from the environment.
#ifndef OMNISEG_EXPERIMENTS
#define OMNISEG_EXPERIMENTS 0
#endif
#define OS_EXP (OMNISEG_EXPERIMENTS != 0)
#if OMNISEG_EXPERIMENTS
#define OS_CLK() clock64()
#else
#define OS_CLK() 0ull
#endif
// Bounds-checked build (`scripts/build_variant.sh checks -DOMNISEG_CHECKS=1`; the stand-in for
// compute-sanitizer, which this GPU pool does not allow): device-side checks of the global
// writes the atomics / finalize / labelling make; a failure prints the site and traps.
#ifndef OMNISEG_CHECKS
#define OMNISEG_CHECKS 0
#endif
#if OMNISEG_CHECKS
#define OS_DCHECK(cond, what)                                                                          \
  do {                                                                                                 \
    if (!(cond)) {                                                                                     \
      printf("OMNISEG_CHECKS failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                       \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define OS_DCHECK(cond, what) \
  do {                        \
  } while (0)
#endif
// true iff the experiment build runs with the environment variable `name` set
bool exp_flag(const char* name);
int exp_int(const char* name);

constexpr int kMaxScales = 4;   // level factors 8, 4, 2, 1
constexpr int kMaxTasks = 32;
constexpr int kTheta = 153;     // W1 b1 W2 b2 W3 b3 of the 8-8-8-1 dynamic head
constexpr int kHead = 8;

// One scale's candidate-tile grid (front end, DESIGN.md §6 K4).
struct ScaleGrid {
  int f;          // level factor
  int log2f;
  int ny, nx;     // grid size
  int Ey, Ex;     // level-f padded extent
  int base;       // first candidate index of this scale (canonical order)
  int kept_base;  // filled after compaction
};

struct FrontParams {
  const uint8_t* slide;  // rows [slide_row0, slide_row0 + slide_rows) of the H x W x 3 slide
  int64_t slide_row0, slide_rows;
  int64_t H, W;
  int pad;
  int Hp, Wp;            // padded frame
  int H8, W8;            // level-8 grid
  int r8_0, r8_1;        // level-8 rows computed by this call (band: with halo)
  int own8_0, own8_1;    // level-8 rows owned (histogram counts only these)
};

// Per-task stitch targets passed by value to the head (kernel or fused epilogue).
struct HeadTaskTable {
  uint32_t* canvas[kMaxTasks];  // fixed-point accumulators, rows [row0, row1) of the task canvas
  int Ht[kMaxTasks], Wt[kMaxTasks];
  int row0[kMaxTasks], row1[kMaxTasks];
  int log2f[kMaxTasks];
  int vote;  // fusion rule: 0 mean of p (R11), 1 hard majority vote
};

// Canvas accumulator update of one window-task pixel (R12). Mean fusion: count << 28 plus
// round(p 2^20); vote fusion ("majority of the testing results", P:97 votes): count << 16
// plus the window's binary decision p >= 1/2, taken as z >= 0 (sigma(z) >= 1/2 exactly, the
// fp64 oracle's decision without fp32 rounding of p).
__device__ __forceinline__ uint32_t stitch_value(float p, float z, int vote) {
  return vote ? (1u << 16) + (z >= 0.f ? 1u : 0u) : (1u << 28) + __float2uint_rn(p * 1048576.0f);
}

// Everything the dynamic head + stitch needs (fused into the last decoder conv).
struct HeadArgs {
  const float* Wpre;    // [8][C0] precls weights (fp32)
  const float* bpre;    // [8]
  const float* theta;   // [B][ntasks][153] controller output
  const float* theta_t; // [B][ntasks][156] the same with W1 / W2 transposed ([in * 8 + out]), 16-B rows
  int ntasks, C0, P, S, Hp, Wp, pad;
  const uint32_t* tiles;  // kept-tile ids (NULL: debug windows, every task applies)
  int first;              // index of batch tile 0 in `tiles`
  float* out_p;           // debug: [B][ntasks][P][P] probabilities instead of stitching
  float* out_F;           // debug: [B][P][P][8]
  int no_tc;              // experiments only: force the CUDA-core head
  HeadTaskTable tt;
};

__host__ __device__ inline uint32_t pack_tile(int log2f, int ty, int tx) {
  return (uint32_t(log2f) << 30) | (uint32_t(ty) << 15) | uint32_t(tx);
}

}  // namespace osg
