/*
 * The drop-in boundary from plain C (no Python, no torch): one frame through
 * tp_gather_tiles -> tp_yolo_create_ex / tp_yolo_forward (the default fp32-parity plan,
 * TP_DTYPE_F16F8) -> tp_region_decode, with device memory from cudaMalloc.
 *
 *   tp_capi_demo <blob> <frame.raw> <W> <H> <out_head.f32> <out_dets.bin>
 *
 * <blob> is written by tests/test_gpu_capi.py from the Python plan's own device weights
 * (yolo.YoloNet): "TPW1", n_layers, then per layer: hi bytes (u64 count + fp16 data),
 * lo bytes (u64 count + e4m3 data, 0 = none), bias bytes (u64 count + fp32), alpha (f32).
 * The frame is u8 [H][W][3]. The program cuts the two attention squares of the
 * "1 att, 3 fin, 20 over" grid (x = 0 and W - H, side H: pipeline.py:224-238's P1
 * attention grid for 16:9 frames), runs the YOLO plan and the region decode, and writes
 * the fp32 head [2][19][19][448] and the raw tp_det_t records + counts.
 * Exit status 0 on success; every C-ABI status is checked (tp_last_error on failure).
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/tilepipe_b200.h"

#define CK(x)                                                                     \
  do {                                                                            \
    int _s = (x);                                                                 \
    if (_s != 0) {                                                                \
      fprintf(stderr, "%s:%d %s -> %d: %s\n", __FILE__, __LINE__, #x, _s,          \
              tp_last_error());                                                   \
      return 1;                                                                   \
    }                                                                             \
  } while (0)
#define CU(x)                                                                     \
  do {                                                                            \
    cudaError_t _e = (x);                                                         \
    if (_e != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x,                  \
              cudaGetErrorString(_e));                                            \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static void* read_chunk(FILE* f, uint64_t* n) {
  if (fread(n, 8, 1, f) != 1) return NULL;
  if (*n == 0) return NULL;
  void* p = malloc(*n);
  if (p == NULL || fread(p, 1, *n, f) != *n) return NULL;
  return p;
}

static void* to_device(const void* h, uint64_t n) {
  void* d = NULL;
  if (n == 0 || cudaMalloc(&d, n) != cudaSuccess) return NULL;
  if (cudaMemcpy(d, h, n, cudaMemcpyHostToDevice) != cudaSuccess) return NULL;
  return d;
}

int main(int argc, char** argv) {
  if (argc != 7) {
    fprintf(stderr, "usage: %s blob frame.raw W H out_head.f32 out_dets.bin\n", argv[0]);
    return 2;
  }
  const int W = atoi(argv[3]), H = atoi(argv[4]);
  FILE* fb = fopen(argv[1], "rb");
  char magic[4];
  int32_t n_layers = 0;
  if (fb == NULL || fread(magic, 1, 4, fb) != 4 || memcmp(magic, "TPW1", 4) != 0 ||
      fread(&n_layers, 4, 1, fb) != 1 || n_layers != 23) {
    fprintf(stderr, "bad weight blob\n");
    return 1;
  }
  const void* w_hi[23];
  const void* w_lo[23];
  const float* bias[23];
  float alpha[23];
  for (int l = 0; l < n_layers; ++l) {
    uint64_t n_hi, n_lo, n_b;
    void* hi = read_chunk(fb, &n_hi);
    void* lo = read_chunk(fb, &n_lo);
    void* b = read_chunk(fb, &n_b);
    if (hi == NULL || b == NULL || fread(&alpha[l], 4, 1, fb) != 1) {
      fprintf(stderr, "truncated blob at layer %d\n", l);
      return 1;
    }
    w_hi[l] = to_device(hi, n_hi);
    w_lo[l] = lo != NULL ? to_device(lo, n_lo) : NULL;
    bias[l] = (const float*)to_device(b, n_b);
    free(hi);
    free(lo);
    free(b);
  }
  fclose(fb);

  /* frame -> device */
  const size_t frame_bytes = (size_t)W * H * 3;
  uint8_t* frame = (uint8_t*)malloc(frame_bytes);
  FILE* ff = fopen(argv[2], "rb");
  if (ff == NULL || frame == NULL || fread(frame, 1, frame_bytes, ff) != frame_bytes) {
    fprintf(stderr, "bad frame file\n");
    return 1;
  }
  fclose(ff);
  uint8_t* d_frame = (uint8_t*)to_device(frame, frame_bytes);

  /* the two attention squares of P1 (crop ids 0 and 1) */
  const int n_tiles = 2;
  tp_tile_job_t jobs[2] = {{0, 0, 0, 0, H, 0, 0, 0}, {0, 1, W - H, 0, H, 1, 0, 0}};
  tp_tile_job_t* d_jobs = (tp_tile_job_t*)to_device(jobs, sizeof(jobs));

  /* the plan: workspace sized by the library, weights borrowed */
  const size_t ws_bytes = tp_yolo_workspace_bytes(n_tiles, TP_DTYPE_F16F8);
  void* ws = NULL;
  CU(cudaMalloc(&ws, ws_bytes));
  tp_yolo_net* net = NULL;
  CK(tp_yolo_create_ex(n_tiles, w_hi, w_lo, bias, alpha, ws, ws_bytes, TP_DTYPE_F16F8, &net));

  cudaStream_t st;
  CU(cudaStreamCreate(&st));
  CK(tp_gather_tiles(d_frame, (int64_t)frame_bytes, H, W, d_jobs, n_tiles, NULL,
                     TP_RESAMPLE_NEAREST, NULL, tp_yolo_input(net), TP_DTYPE_F16F8, st));
  CK(tp_yolo_forward(net, n_tiles, NULL, st));

  /* region decode + projection (detector threshold 0.25, the YOLO v2 VOC/COCO anchors) */
  const float anchors[10] = {0.57273f, 0.677385f, 1.87446f, 2.06253f, 3.33843f,
                             5.47434f, 7.88282f, 3.52778f, 9.77052f, 9.16828f};
  const int max_per_tile = TP_GRID * TP_GRID * TP_ANCHORS;
  tp_det_t* d_dets = NULL;
  int32_t* d_counts = NULL;
  CU(cudaMalloc((void**)&d_dets, sizeof(tp_det_t) * max_per_tile * n_tiles));
  CU(cudaMalloc((void**)&d_counts, sizeof(int32_t) * n_tiles));
  CK(tp_region_decode(tp_yolo_head(net), tp_yolo_head_cstride(), n_tiles, NULL, d_jobs, W, H,
                      0.25f, anchors, d_dets, max_per_tile, d_counts, st));
  CU(cudaStreamSynchronize(st));

  /* results -> files */
  const size_t head_n = (size_t)n_tiles * TP_GRID * TP_GRID * tp_yolo_head_cstride();
  float* head = (float*)malloc(head_n * 4);
  CU(cudaMemcpy(head, tp_yolo_head(net), head_n * 4, cudaMemcpyDeviceToHost));
  FILE* fo = fopen(argv[5], "wb");
  if (fo == NULL || fwrite(head, 4, head_n, fo) != head_n) return 1;
  fclose(fo);
  int32_t counts[2];
  CU(cudaMemcpy(counts, d_counts, sizeof(counts), cudaMemcpyDeviceToHost));
  tp_det_t* dets = (tp_det_t*)malloc(sizeof(tp_det_t) * max_per_tile * n_tiles);
  CU(cudaMemcpy(dets, d_dets, sizeof(tp_det_t) * max_per_tile * n_tiles, cudaMemcpyDeviceToHost));
  FILE* fd = fopen(argv[6], "wb");
  if (fd == NULL || fwrite(counts, 4, 2, fd) != 2) return 1;
  for (int t = 0; t < n_tiles; ++t)
    if (fwrite(dets + (size_t)t * max_per_tile, sizeof(tp_det_t), counts[t], fd) != (size_t)counts[t])
      return 1;
  fclose(fd);
  printf("tp_capi_demo: 2 attention tiles, %d + %d detections, version %d\n", counts[0],
         counts[1], tp_version());
  CK(tp_yolo_destroy(net));
  return 0;
}
