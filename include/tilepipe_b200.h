/*
 * tilepipe_b200 — C ABI of the B200-native attention-pipeline hot path.
 *
 * Every entry point takes plain pointers and sizes; device pointers are
 * borrowed (the caller owns the memory, e.g. torch tensors), `stream` is a
 * cudaStream_t passed as void*. Calls are stream-ordered and return an int
 * status (0 = TP_OK); on failure tp_last_error() describes the cause. Nothing
 * is allocated per call: the YOLO plan works inside a caller-provided
 * workspace.
 *
 * Reference interfaces each entry point replaces (paths relative to the
 * reference package root, pkg/src/tilepipe/):
 *   tp_gather_tiles          detector.py:223-247 (cut_tile), pipeline.py:291-294 (_tile_for)
 *   tp_yolo_*                detector.py:77-96   (Detector.detect body: YOLO v2-608)
 *   tp_region_decode         detector.py:86-96 output contract + geometry.py:237-256 (to_global)
 *   tp_project_rects         geometry.py:237-256 (to_global, foreign-detector path)
 *   tp_attention_boxes       pipeline.py:313-316 (attention_pass confidence filter + box list)
 *   tp_select_active         pipeline.py:319-354 (merge_temporal + select_active)
 *   tp_build_jobs            pipeline.py:366     (final_pass: sorted(active_ids) tile order)
 *   tp_nccl_gather_dets      distribution/client.py:176-203, 242-377 (result collection from
 *                            workers, frame order)
 *   tp_collect_final         pipeline.py:357-375 (final_pass tagged list, crop-id order)
 *   tp_postprocess           postprocess.py:54-187 + pipeline.py:378-385
 *                            (nms_keep_indices, merge_split, postprocess, finish_detections)
 */
#ifndef TILEPIPE_B200_H
#define TILEPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TP_API __attribute__((visibility("default")))
#else
#define TP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define TP_MODEL_SIDE 608
#define TP_GRID 19
#define TP_ANCHORS 5
#define TP_CLASSES 80
#define TP_HEAD_CH 425 /* 5 * (4 + 1 + 80) */

enum { TP_RESAMPLE_NEAREST = 0, TP_RESAMPLE_BILINEAR = 1 };
/* 16-bit operand/activation format of the conv stack (fp32 accumulation either way).
 * TP_DTYPE_F16X2 is the fp32-parity plan (no reference counterpart; serves the north-star
 * 1e-3 score bar against the fp32 CPU reference): every activation is stored as exact fp16
 * pairs hi = fp16(x), lo = fp16(x - hi), interleaved per 16 channels ([hi 16 | lo 16]: real
 * channel c at stored channel 32*(c/16) + c%16, its lo part 16 further), so a C-channel
 * tensor has 2C stored channels and K spans both parts (weights duplicated per 16-channel
 * group); products are exact and accumulate in fp32, so activations carry ~22 bits. The
 * gather writes integer pixel values (exact in fp16) and layer 0 scales by 1/255 in fp32.
 * TP_DTYPE_F16F8 (the default parity plan) keeps the same contract at 3/4 of the tensor
 * work: every activation but the layer-0 input and the head is two planes, hi = fp16(x)
 * [pix][C] and lo = e4m3((x - hi) * 2^TP_LO_EXP) [pix][C] bytes ("HL8"); a consumer runs K
 * over hi with fp16 weights w * 2^c (kind::f16) and over lo with e4m3 weights
 * w * 2^(c - TP_LO_EXP) (kind::f8f6f4, twice the rate) into one fp32 accumulator and scales
 * it by 2^-c. tp_yolo_create_ex takes the extra weights and scales. */
enum { TP_DTYPE_BF16 = 0, TP_DTYPE_F16 = 1, TP_DTYPE_F16X2 = 2, TP_DTYPE_F16F8 = 3 };
#define TP_LO_EXP 11

/* One 608x608 tile to produce: crop square (x, y, side) of batch frame `frame`. */
typedef struct tp_tile_job {
  int32_t frame;   /* index into the device frame batch */
  int32_t crop_id; /* unified crop id (GridPlan) */
  int32_t x, y, side;
  int32_t cell;    /* row * grid_cols + col of the crop in its grid */
  int32_t pad0, pad1;
} tp_tile_job_t;

/* Region-layer output record, one per kept (cell, anchor). */
typedef struct tp_det {
  float lx, ly, lw, lh;     /* crop-local 608-space rect, clipped to [0,608]^2 */
  int32_t gx, gy, gw, gh;   /* to_global(local, crop, W, H): integer global rect */
  float conf;               /* sigmoid(obj) * softmax(cls)[argmax] */
  int32_t cls;              /* argmax class (COCO-80 index) */
  int32_t crop_id;
  int32_t frame;
} tp_det_t;

/* Postprocess record: global rect in fp64 (the reference Rect arithmetic). */
typedef struct tp_pdet {
  double x, y, w, h;
  double conf;
  int32_t cls;
  int32_t cell;    /* grid cell of the crop that produced it */
  int32_t crop_id;
  int32_t src;     /* index in the caller's input order */
} tp_pdet_t;

#define TP_MAX_CLASSES 128
enum { TP_RULE_NONE = 0, TP_RULE_VERTICAL = 1, TP_RULE_HORIZONTAL = 2, TP_RULE_BOTH = 3 };

typedef struct tp_post_policy {
  double nms_iou;
  double gap_px;
  double tol_px;
  double min_conf;          /* final confidence filter; < 0 disables */
  int32_t merge_before_nms;
  int32_t nms_per_crop;
  int32_t do_nms;           /* 0: skip NMS (merge_split only) */
  int32_t do_merge;         /* 0: skip merge (NMS only) */
  int32_t grid_cols;
  int32_t n_cells;          /* <= 256 */
  uint8_t class_rule[TP_MAX_CLASSES];
} tp_post_policy_t;

TP_API const char* tp_last_error(void);
TP_API int tp_version(void);
TP_API int tp_device_sm_count(int* out);

/* K1/K2: crop gather + resample (+ normalise). frames: u8 [n][H][W][3] with
 * frame_stride bytes between frames. out_u8: optional [n_jobs][608][608][3].
 * out_act: optional 16-bit (act_dtype) [n_jobs][610][614][4] layer-0 input: tile pixel
 * (v, u) at [v+1][u+2] as (r, g, b, 0) with values / 255 (the integer values for the
 * parity plans TP_DTYPE_F16X2 / TP_DTYPE_F16F8); the halo (rows 0 / 609, columns 0, 1, 610..613) must be pre-zeroed and
 * is never written.
 * n_jobs_dev: optional device count overriding n_jobs (n_jobs is then the max). */
TP_API int tp_gather_tiles(const uint8_t* frames, int64_t frame_stride, int H, int W,
                    const tp_tile_job_t* jobs, int n_jobs, const int32_t* n_jobs_dev,
                    int mode, uint8_t* out_u8, void* out_act, int act_dtype, void* stream);

/* K3/K4: YOLO v2-608 forward plan (23 tcgen05 implicit-GEMM conv layers,
 * maxpools, route/reorg). Weights are 16-bit [cout_pad][taps*cin] K-major with
 * BN folded in (layer 0: [32][144], 3 kernel rows x 3 window variants x 4 pixels x rgb0 — see
 * paper_1810_10551_b200/yolo.py L0_VARIANTS); biases fp32 [cout_pad]. */
typedef struct tp_yolo_net tp_yolo_net;
TP_API size_t tp_yolo_workspace_bytes(int max_tiles, int dtype);
TP_API int tp_yolo_create(int max_tiles, const void* const* weights, const float* const* biases,
                   void* workspace, size_t workspace_bytes, int dtype, tp_yolo_net** out);
/* TP_DTYPE_F16F8 plan: weights_lo[l] = e4m3 [cout_pad][taps*cin] lo-pass weights of every
 * layer with an HL8 input (NULL for the others), alphas[l] = accumulator scale 2^-c of
 * those layers (1 elsewhere; ignored for layer 0). Other dtypes: weights_lo and alphas may
 * be NULL (tp_yolo_create). */
TP_API int tp_yolo_create_ex(int max_tiles, const void* const* weights,
                             const void* const* weights_lo, const float* const* biases,
                             const float* alphas, void* workspace, size_t workspace_bytes,
                             int dtype, tp_yolo_net** out);
/* Which conv slots read an HL8 input in the TP_DTYPE_F16F8 plan: bit l of the mask. */
TP_API uint32_t tp_yolo_hl8_inputs(void);
TP_API void* tp_yolo_input(tp_yolo_net* net);        /* 16-bit [max_tiles][610][614][4] pixels */
TP_API int tp_yolo_num_steps(void);
TP_API const float* tp_yolo_head(tp_yolo_net* net);  /* fp32 [max_tiles][19][19][448] */
TP_API int tp_yolo_head_cstride(void);
TP_API int tp_yolo_forward(tp_yolo_net* net, int n_tiles, const int32_t* n_tiles_dev, void* stream);
/* Debug/parity: run layers [first, last] only and expose any layer's output. */
TP_API int tp_yolo_forward_range(tp_yolo_net* net, int n_tiles, const int32_t* n_tiles_dev,
                          int first, int last, void* stream);
TP_API int tp_yolo_layer_output(tp_yolo_net* net, int layer, void** ptr, int* res, int* cstride);
/* lo plane (e4m3 bytes, same [pixel][channel] index as the hi plane) of an HL8 step output;
 * *ptr = NULL for other outputs. */
TP_API int tp_yolo_layer_output_lo(tp_yolo_net* net, int layer, void** ptr);
/* Kernel the plan chose for conv slot 0..22: 0 conv_tc, 1 conv_pair (cta_group::2),
 * 2 conv_l0, 3 conv_box, 4 conv_pair_rect (cta_group::2, pooled); -1 on a bad argument. */
TP_API int tp_yolo_layer_kernel(tp_yolo_net* net, int conv);
/* TP_DTYPE_F16F8 plan: layer 5 (1x1, step 3) runs inside layer 4's kernel (step 2) by
 * default — layer 4's output stays on chip and its buffer is not written. fused = 0 keeps
 * the two launches (every step output materialised, for per-layer checks); the results are
 * bit-identical either way. TP_ERR_UNSUPPORTED when asked to fuse a plan that cannot. */
TP_API int tp_yolo_set_fused(tp_yolo_net* net, int fused);
/* 1 if `step` currently runs inside the previous step's kernel (its input buffer is not
 * written by a forward), else 0. */
TP_API int tp_yolo_step_fused(tp_yolo_net* net, int step);
TP_API int tp_yolo_destroy(tp_yolo_net* net);

/* Generic implicit-GEMM conv (one layer), for tests. Activations are compact NHWC 16-bit
 * [n][res][res][cstride]; the zero padding of 3x3 convs is implicit (TMA out-of-bounds
 * fill). cin_stride == 16 is the layer-0 mode (K = 16 per kernel row): input is the
 * gather's padded pixel image [n][res+2][res+6][4] and the conv must pool. pool != 0 fuses a 2x2/2 max pool
 * (out is then [n][res/2][res/2][out_cstride]). */
TP_API int tp_conv(const void* in, int n_img, int res, int cin_stride, const void* weight,
                   const float* bias, int cout, int cout_pad, int ksize, int leaky, void* out,
                   int out_cstride, int out_coff, int out_fp32, int reorg, int dtype, int pool,
                   void* stream);

/* K5: region decode + threshold + sort + project. head: fp32 compact
 * [n][19][19][cstride]. out: [n][max_per_tile] sorted by (-conf, cell*5+anchor). */
TP_API int tp_region_decode(const float* head, int head_cstride, int n_tiles, const int32_t* n_tiles_dev,
                     const tp_tile_job_t* jobs, int frame_w, int frame_h, float thresh,
                     const float* anchors_host, tp_det_t* out, int max_per_tile,
                     int32_t* counts, void* stream);

/* to_global for rects from a foreign (host) Detector plugin: local fp64 [n][4],
 * crop_xyside int32 [n][3]; frame_w <= 0 disables the frame clip. out int32 [n][4]. */
TP_API int tp_project_rects(const double* local, const int32_t* crop_xyside, int n, int frame_w,
                            int frame_h, int32_t* out, void* stream);

/* Attention boxes per frame: concat over the frame's A attention tiles (crop
 * order, detector order) of dets with conf >= min_conf. boxes: fp64
 * [n_frames][max_boxes][4] (x, y, w, h). */
TP_API int tp_attention_boxes(const tp_det_t* dets, const int32_t* counts, int max_per_tile,
                       int n_frames, int tiles_per_frame, double min_conf, double* boxes,
                       int32_t* box_counts, int max_boxes, void* stream);

/* K6: merge_temporal over `window` slots + select_active. boxes/box_counts are
 * slot-indexed: slot s holds frame (s - (window-1)) of the batch, so slots
 * 0..window-2 carry history. crops: fp64 [n_crops][4]. Outputs per frame:
 * active bitmask words [n_frames][mask_words], sorted active crop ids,
 * counts, and the first-seen-deduplicated merged box list. max_merged <= 512 (the
 * kernel's window capacity); a window holding more than 512 boxes reports its true box
 * count in merged_counts (> max_merged) and must be treated as a failure. */
TP_API int tp_select_active(const double* boxes, const int32_t* box_counts, int max_boxes,
                     int n_frames, int window, const double* crops, int n_crops,
                     int crop_id_base, double margin, double frame_w, double frame_h,
                     uint32_t* active_mask, int mask_words, int32_t* active_ids,
                     int32_t* active_counts, double* merged, int32_t* merged_counts,
                     int max_merged, void* stream);

/* Stage-2 job list from per-frame active ids (frame-major, crop-id ascending). */
TP_API int tp_build_jobs(const int32_t* active_ids, const int32_t* active_counts, int n_frames,
                  int max_active, const int32_t* crop_table /* [n_crops][4] x,y,side,cell */,
                  int crop_id_base, tp_tile_job_t* jobs, int32_t* frame_job_start,
                  int32_t* n_jobs_dev, void* stream);

/* final_pass tagged list per frame: concat over the frame's jobs (in job order)
 * of their dets, converted to fp64 postprocess records. */
TP_API int tp_collect_final(const tp_det_t* dets, const int32_t* counts, int max_per_tile,
                     const tp_tile_job_t* jobs, const int32_t* frame_job_start, int n_frames,
                     tp_pdet_t* out, int32_t* out_counts, int max_per_frame, void* stream);

/* K7: per-frame postprocess (NMS / merge_split / both / variants + min_conf
 * filter). keep_idx (optional): NMS keep indices in keep order per frame. */
TP_API int tp_postprocess(const tp_pdet_t* dets, const int32_t* counts, int n_frames,
                   int max_per_frame, const tp_post_policy_t* policy, tp_pdet_t* out,
                   int32_t* out_counts, int32_t* keep_idx, int32_t* keep_counts, void* stream);

/* Synthetic frame renderer (input generator): per frame, counts[f] <= 64 rectangles
 * rects int32 [n][max_obj][4] = (x0, y0, x1, y1) exclusive ends, colours u8 [n][max_obj][3],
 * painted in order over background bg_rgb (r | g<<8 | b<<16) into u8 [n][H][W][3].
 * Same bytes as the reference render_frame (synthetic.py:183-196). */
TP_API int tp_render_frames(const int32_t* rects, const uint8_t* colors, const int32_t* counts,
                            int n_frames, int max_obj, int H, int W, uint32_t bg_rgb,
                            uint8_t* out, void* stream);

/* Crop-parallel stage 2 (replaces the reference's remote dispatch of one
 * frame's tiles, pkg/src/tilepipe/distribution/client.py:82-96). tp_slice_jobs copies rank's
 * contiguous slice of the device job list (sizes differ by <= 1, larger first) and writes
 * its count; tp_unslice_dets maps all-gathered per-rank compact slices ([world][max_slice]
 * tiles of src_per_tile records + the tiles' true counts) back to global job order
 * (dst_per_tile records per tile). A tile with more than src_per_tile records is clamped
 * and sets *overflow (may be NULL) — the caller must fail, not use the result. */
TP_API int tp_slice_jobs(const tp_tile_job_t* jobs, const int32_t* n_jobs_dev, int rank,
                         int world, tp_tile_job_t* out, int32_t* n_out_dev, int max_out,
                         void* stream);
TP_API int tp_unslice_dets(const tp_det_t* gathered, const int32_t* gathered_counts,
                           int max_slice, const int32_t* n_jobs_dev, int world, int max_jobs,
                           int src_per_tile, int dst_per_tile, tp_det_t* dets, int32_t* counts,
                           int32_t* overflow, void* stream);

/* Result gather (replaces the reference's collection of worker results,
 * pkg/src/tilepipe/distribution/client.py:176-203 evaluate_remote and :242-377): all-gather
 * every rank's padded record slice (rec_bytes_per_rank bytes) and counts (counts_per_rank
 * int32) in rank order, both inside one ncclGroupStart/End on `stream`. `nccl_comm` is an
 * ncclComm_t borrowed from the caller (torch.distributed's ProcessGroupNCCL._comm_ptr());
 * NCCL is resolved from the libnccl.so.2 already loaded in the process. Either size may be
 * 0 (that gather is skipped). tp_nccl_available() = 1 when NCCL resolves. */
TP_API int tp_nccl_available(void);
TP_API int tp_nccl_gather_dets(void* nccl_comm, const void* local_recs, int64_t rec_bytes_per_rank,
                               const int32_t* local_counts, int64_t counts_per_rank,
                               void* all_recs, int32_t* all_counts, void* stream);


/* Profiling only (TP_CONV_DEBUG bit 32 set in the environment when the net/conv runs):
 * per-role cycle totals of conv_tc_kernel summed over CTAs — 0 producer, 1 producer
 * empty-wait, 2 MMA issuer, 3 issuer accumulator-wait, 4 issuer stage-wait, 5 epilogue
 * warp 0, 6 epilogue accumulator-wait, 7 launches. No reference counterpart. */
TP_API int tp_debug_conv_counters(uint64_t* out, int n, int reset);
/* 2x2/2 max pool on compact NHWC 16-bit activations (exposed for tests). */
TP_API int tp_maxpool2(const void* in, int n_img, int res, int cstride, int dtype, void* out,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif
