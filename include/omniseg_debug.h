/*
 * omniseg_debug.h -- test-only entry points of libomniseg.so (same library, same
 * kernels as the product path). They expose single stages so the GPU parity tests
 * can compare each against the oracle. Conventions as in omniseg.h.
 */
#ifndef OMNISEG_DEBUG_H
#define OMNISEG_DEBUG_H

#include <stddef.h>
#include <stdint.h>

#include "omniseg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Trunk + GAP + controller + dynamic head on n given windows.
 *   tiles_u8 : n x P x P x 3 uint8 (host or device).
 *   cls[t], scl[t]: n_tasks (class index, scale-code index) pairs; every tile runs every task.
 *   out_p    : float[n][n_tasks][P][P] (host or device): sigmoid probabilities.
 *   out_g    : float[n][C_bottleneck] or NULL: the GAP feature.
 *   out_F    : float[n][P][P][8] or NULL: the precls feature F. */
int omniseg_debug_predict_tiles(omniseg_t* h, const uint8_t* tiles_u8, int n, int P,
                                const int* cls, const int* scl, int n_tasks,
                                float* out_p, float* out_g, float* out_F);

/* One implicit-GEMM convolution through the tcgen05 kernel.
 *   x   : float[B][H][W][Cin] host, values rounded to the storage dtype on upload.
 *   w   : float[Cout][k][k][Cin] host (k = 1 or 3), b: float[Cout].
 *   r   : float residual / skip input (mode 1: [B][Ho][Wo][Cout]; mode 2: [B][2H][2W][Cout]) or NULL.
 *   mode: 0 y = relu(conv + b); 1 y = relu(conv + b + r); 2 y[2i+a][2j+c] = r[...] + conv + b
 *         (1x1 + nearest-up x2 + skip add); 3 y = conv + b. mode | 16: x, r, y use the
 *         split hi|lo storage of the x2 precision modes (dtype fp16x2 / bf16x2).
 *   y   : float output (storage dtype values widened to fp32). */
int omniseg_debug_conv(omniseg_t* h, const float* x, int B, int H, int W, int Cin,
                       const float* w, const float* b, int Cout, int k, int stride,
                       const float* r, int mode, float* y);

/* Single-GPU emulation of the multi-GPU band path: inject the global pad colour (3 u8)
 * and global interior histogram (256 u64) that the NCCL broadcast / all-reduce would
 * deliver, so that omniseg_segment_band on one GPU without a communicator reproduces a
 * rank's result. NULL arguments switch injection off. */
int omniseg_debug_band_globals(omniseg_t* h, const uint8_t* pc, const uint64_t* hist);
/* Single-GPU emulation of the band foreground exchange (fgmin > 0: the ncclAllReduce of the
 * ranks' owned level-8 foreground rows): inject the whole slide's PRE-filter level-8
 * foreground (H8 x W8 u8, host). NULL switches injection off. */
int omniseg_debug_band_fg(omniseg_t* h, const uint8_t* fg8, int64_t n);
/* The pad colour and the (global) histogram used by the last segment call. */
int omniseg_debug_get_detection(const omniseg_t* h, uint8_t* pc, uint64_t* hist);

/* Per-launch CUDA-event timing of every tcgen05 convolution (on the library's stream),
 * accumulated over calls until the next set_profile. on = 0 disables; either call resets. */
int omniseg_debug_set_profile(omniseg_t* h, int on);
/* out[0] total conv ms, out[1] total algorithmic conv FLOPs (2 M N K with the network's
 * real channel counts: no padding, no x2 doubling, stem K = 27), out[2] launches, then per
 * layer position l (stem, enc.., dec..): out[3+3l] ms, out[4+3l] FLOPs, out[5+3l] launches. */
int omniseg_debug_get_profile(const omniseg_t* h, double* out, int cap, int* n_layers);

#ifdef __cplusplus
}
#endif
#endif
