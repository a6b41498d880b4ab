/*
 * omniseg.h -- C ABI of libomniseg.so: slide-wise Omni-Seg prediction on B200 (sm_100a).
 *
 * The operation (arxiv 2305.14566, /root/reference/PAPER.md):
 *   P:53 §2      three-step pipeline: tissue detection + patch extraction,
 *                Omni-Seg segmentation, slide-wise aggregation;
 *   P:57-61 §2.1 pad the WSI (colour = mean of the top-left 2x2), detect the
 *                foreground (median blur + Otsu), drop blank regions;
 *   P:66-69 §2.2 tile the slide at each class's magnification (40x/10x/5x) into
 *                overlapping 512x512 windows, predict each with the Omni-Seg
 *                dynamic network (BASELINE.json north_star: residual U-Net, GAP,
 *                controller -> 3 dynamic 1x1 layers, sigmoid);
 *   P:86-87 §2.3 merge the predictions of each tissue type back into a slide-level
 *                map; P:97 majority of overlapping tiles decides (read as the
 *                overlap-normalised mean thresholded at 1/2, R11).
 * The interface follows north_star: omniseg_create(arch, weights) and
 * omniseg_segment_slide(rgb_u8, H, W, pad, patch, stride, scales[], classes[],
 * out_prob, out_mask). Concrete readings of everything the paper leaves open are
 * listed in DESIGN.md §2 (R1..R14) and are cited below as "R<n>".
 *
 * Conventions (all entry points):
 *   - Return codes: 0 = ok, OMNISEG_EINVAL (-1) parameter error, OMNISEG_ECUDA (-2)
 *     CUDA error, OMNISEG_ENOMEM (-3) allocation failure, OMNISEG_ENCCL (-4)
 *     collective error. On error, omniseg_last_error() returns a thread-local
 *     message; outputs are unspecified.
 *   - Synchronous: outputs are complete when a call returns.
 *   - Pointers may be host or device memory (detected with
 *     cudaPointerGetAttributes); device pointers must be on the handle's device.
 *     The library never retains caller pointers; the caller owns every array.
 *   - A handle is not thread-safe: one handle per thread/device.
 */
#ifndef OMNISEG_H
#define OMNISEG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OMNISEG_OK      0
#define OMNISEG_EINVAL (-1)
#define OMNISEG_ECUDA  (-2)
#define OMNISEG_ENOMEM (-3)
#define OMNISEG_ENCCL  (-4)

typedef struct omniseg omniseg_t;   /* opaque; owns device weights, workspace, streams */

/* Create a predictor.
 *   arch   : ';'-separated key=value string, e.g.
 *            "levels=5;base=32;head=8;ncls=6;scale_codes=5,10,20,40;slide_mag=40;dtype=fp16f8;batch=64"
 *            levels/base: U-Net depth and base width (channels base*2^l); head must be 8
 *            (3-layer 8-channel dynamic head, BASELINE configs[0]); ncls classes;
 *            scale_codes: magnifications with a one-hot code each (order = code index);
 *            slide_mag: magnification of the input slide (level factor f = slide_mag/scale);
 *            dtype: activation storage, fp32 accumulation (R9):
 *              fp16f8 (default, the parity-gated product precision): each activation stored
 *                as fp16 hi + e4m3 residual lo8 = e4m3((v - hi) * 2^6) (3 bytes / channel);
 *                every convolution runs its K loop over the hi chunks (tcgen05 kind::f16,
 *                exact fp16 weights) and the lo chunks (kind::f8f6f4, e5m2(W * 2^-6)) into
 *                one fp32 accumulator (1.5x the fp16 tensor work);
 *              fp16x2 / bf16x2: hi + lo 16-bit pairs, K loop over [W | W] (2x tensor work);
 *              fp16 / bf16: plain 16-bit storage (reported, not parity-gated: a random
 *                network amplifies their rounding beyond the 1e-2 gate, R9);
 *            batch: tiles per trunk launch; device: CUDA ordinal (default: current);
 *            fusion=mean|vote (R11 / R11b); vthr=t5,t10,... (vote fusion only: one literal
 *            vote-count threshold per scale code, mask = votes >= min(thr, coverage); 0 =
 *            majority); fgmin=N, maskfg=0|1 (R7b); precision knobs xlevels / xa / xal
 *            (DESIGN.md §8).
 *   weights: flat little-endian fp32 blob in the order of DESIGN.md §3;
 *            nbytes must equal 4 * param_count(arch). Host or device; copied.
 * Returns NULL on error (see omniseg_last_error). */
omniseg_t* omniseg_create(const char* arch, const void* weights, size_t nbytes);

/* Segment one slide (all kept tiles of all task scales) on the handle's GPU.
 *   rgb_u8  : H x W x 3 uint8, row-major, tightly packed (pitch 3W). Host or device.
 *   H, W    : slide size in pixels at slide_mag; H, W >= 2.
 *   pad     : padding per side in slide pixels (R2); pad % 8 == 0.
 *             The padded frame is roundup(H+2pad,128) x roundup(W+2pad,128).
 *   patch   : window size P at every scale; multiple of 16 and of 2^(levels-1).
 *   stride  : window stride S at every scale; 8 <= S <= P, S % 8 == 0.
 *   scales  : n_tasks magnifications (each in scale_codes; f = slide_mag/scale in {1,2,4,8});
 *   classes : n_tasks class indices (< ncls).
 *   out_prob: float[sum_t Ht*Wt] or NULL, Ht = ceil(H/f_t), Wt = ceil(W/f_t), tasks
 *             concatenated in order: overlap-normalised probability (0 where no kept
 *             tile covers the pixel), R10-R11.
 *   out_mask: uint8[sum_t Ht*Wt] or NULL: prob >= 1/2 (decided exactly on the
 *             fixed-point accumulator, R12); with fusion=vote the vote fraction / majority
 *             (or the vthr count threshold) instead.
 *   out_area: uint64[n_tasks] or NULL: number of mask pixels per task.
 * Errors: EINVAL for any violated precondition above, and when the coverage count of
 * a pixel could exceed 15 (ceil(P/S)+1)^2 > 15, which the u32 fixed-point canvas
 * cannot hold (R12). */
int omniseg_segment_slide(omniseg_t* h, const uint8_t* rgb_u8, int64_t H, int64_t W,
                          int pad, int patch, int stride,
                          const int* scales, const int* classes, int n_tasks,
                          float* out_prob, uint8_t* out_mask, uint64_t* out_area);

/* Number of canvas pixels of a task at magnification `scale`: ceil(H/f)*ceil(W/f). */
int64_t omniseg_output_size(const omniseg_t* h, int64_t H, int64_t W, int scale);

/* Multi-GPU, one process per GPU. The caller joins an NCCL clique
 * (128-byte ncclUniqueId from rank 0, broadcast by the caller, e.g. via
 * torch.distributed) of `world` ranks. */
int omniseg_comm_init(omniseg_t* h, const void* nccl_unique_id, int world, int rank);

/* Segment the row band [row0, row1) of the PADDED 40x frame (row0, row1 multiples of
 * 8*stride*f_max/8... see DESIGN.md §7: multiples of 8*S, row1 = Hp for the last band).
 *   rgb_band: slide rows [b0, b1) with b0 = clamp(row0 - pad - halo, 0, H),
 *             b1 = clamp(row1 - pad + halo, 0, H), halo = patch * f_max + 64 (one
 *             window at the coarsest scale plus the detection median's reach), H x W
 *             layout otherwise as in omniseg_segment_slide.
 *   Each rank computes every kept tile whose window intersects its owned rows; the
 *   Otsu histogram is all-reduced over ranks (R6) so tile lists match the 1-GPU run;
 *   outputs cover only the task-canvas rows owned by this band, per task, tasks
 *   concatenated; out_area is all-reduced (global per-task areas on every rank).
 *   With fgmin > 0 (tiny-component removal needs whole components) each rank computes the
 *   foreground of its owned level-8 rows and the H8 x W8 grid is all-reduced (disjoint rows:
 *   the union) before every rank labels the whole grid; this needs a communicator.
 * Canvas values are bit-identical to omniseg_segment_slide's (fixed point, R12). */
int omniseg_segment_band(omniseg_t* h, const uint8_t* rgb_band, int64_t H, int64_t W,
                         int64_t row0, int64_t row1, int pad, int patch, int stride,
                         const int* scales, const int* classes, int n_tasks,
                         float* out_prob, uint8_t* out_mask, uint64_t* out_area);

/* An EMPTY band (row0 == row1 > 0: more ranks than 8*stride row units) computes nothing but
 * joins the same collectives (pad-colour broadcast, histogram and area all-reduces), so a
 * world larger than the slide's row-unit count still completes; out_area gets the global areas.
 *
 * Band gather (the north_star NCCL step, SURVEY §8(e) collective 2): after
 * omniseg_segment_band on every rank, gather every rank's owned canvas rows into full-slide
 * outputs on rank `root` (device-resident), one ncclSend/ncclRecv pair per (rank, task) in one
 * NCCL group (the root's own band too, as a self pair).
 *   cuts      : world+1 band boundaries of the PADDED 40x frame (cuts[r] = row0 of rank r,
 *               cuts[world] = Hp), as passed to each rank's segment_band.
 *   scales    : the n_tasks magnifications of the segment_band calls (classes are not needed).
 *   band_prob / band_mask: this rank's segment_band outputs (device; NULL = not gathered).
 *   out_prob / out_mask  : root only: device buffers laid out as omniseg_segment_slide's
 *               outputs (tasks concatenated, ceil(H/f) x ceil(W/f) each); ignored elsewhere.
 * Collective: every rank of the communicator must call it with the same cuts / scales.
 * Errors: EINVAL without a communicator or for host buffers; ENCCL on NCCL failure. Buffer
 * errors found on any one rank (e.g. a host out_prob on the root) are agreed on by one int
 * all-reduce before any transfer, so every rank returns the error instead of blocking. */
int omniseg_gather_bands(omniseg_t* h, int root, int64_t H, int64_t W, int pad, const int64_t* cuts,
                         const int* scales, int n_tasks, const float* band_prob, const uint8_t* band_mask,
                         float* out_prob, uint8_t* out_mask);

/* Owned canvas rows of band [row0,row1) for a task at factor f: [r0_t, r1_t) with
 * r0_t = clamp(ceil((row0 - pad)/f), 0, Ht) (likewise r1_t). Pure arithmetic helper. */
int omniseg_band_rows(int64_t H, int64_t row0, int64_t row1, int pad, int f,
                      int64_t* r0_t, int64_t* r1_t);

/* 40x merge + colour overlay + 10x overlay (§2.3 "stained with different colors
 * on WSIs ... a final downsampled prediction of the 10x WSI ... by directly resizing the final
 * prediction of the 40x image"). rgb_u8: the H x W x 3 slide; masks: the per-task masks
 * exactly as omniseg_segment_slide returns them (tasks concatenated, each ceil(H/f) x ceil(W/f)
 * u8 0/1) for the same scales[] / classes[]. Each task mask is upsampled nearest-neighbour to
 * 40x; where several classes are positive the lowest class code wins (TUFT > CAP > PT > DT >
 * PTC > VES, codes 0..5); a positive pixel becomes round(0.4 colour + 0.6 base) per channel with
 * the fixed palette TUFT (255,0,0), CAP (255,128,0), PT (0,255,0), DT (0,128,255), PTC
 * (255,0,255), VES (128,0,128) (the paper gives no values), others keep the slide pixel.
 * out40: H x W x 3 (or NULL); out10: ceil(H/4) x ceil(W/4) x 3 factor-4 area mean of the 40x
 * overlay, round half up, partial edge blocks averaging their pixels (or NULL). Host or device
 * pointers; synchronous. -1 on bad arguments (class code >= 6, no output). */
int omniseg_render_overlay(omniseg_t* h, const uint8_t* rgb_u8, int64_t H, int64_t W, const uint8_t* masks,
                           const int* scales, const int* classes, int n_tasks, uint8_t* out40, uint8_t* out10);

/* Introspection (valid after the last segment call on this handle). */
/* Kept tiles in canonical order (scale descending, then row, then column), packed
 * (log2 f) << 30 | ty << 15 | tx  (grid indices; origin = min(i*S, E-P), R3). */
int omniseg_get_tiles(const omniseg_t* h, uint32_t* tiles, int64_t cap, int64_t* n);
/* Level-8 foreground mask (Hp/8 x Wp/8 u8), Otsu threshold and the luma of the pad colour. */
int omniseg_get_fgmask(const omniseg_t* h, uint8_t* mask, int64_t cap, int64_t* h8, int64_t* w8,
                       int* otsu_t, int* g_pad);
/* Per-stage device times of the last call, milliseconds (CUDA events on the
 * library's stream): [0] upload, [1] pyramid+detection+selection, [3] the batch loop
 * (window gather fused into the stem kernel, trunk convs, GAP+controller, the dynamic head
 * and stitch fused into the last decoder conv -- their per-kind split is the per-conv
 * profile of omniseg_debug_get_profile), [6] finalize of the remaining rows + area
 * reduction, [7] output download wait, [8] total; [2], [4], [5] are 0 (fused into [3]).
 * Also the conv-kernel launch count [9] and total launches [10]. */
int omniseg_get_timings(const omniseg_t* h, double* out, int cap);

/* Use this CUDA stream (cudaStream_t cast to void*; NULL = the library's own). */
int omniseg_set_stream(omniseg_t* h, void* stream);

const char* omniseg_last_error(void);
void omniseg_destroy(omniseg_t* h);

#ifdef __cplusplus
}
#endif
#endif /* OMNISEG_H */
