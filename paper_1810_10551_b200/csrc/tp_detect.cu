// K5 — region-layer decode + confidence filter + deterministic sort + to_global.
//
// Implements the detector output contract of the reference boundary
// (pkg/src/tilepipe/detector.py:86-96: crop-local 608-space detections sorted by
// descending confidence, rects inside [0,608]^2 with positive size, geometry.py:31-36)
// for a YOLO v2 region layer, and fuses the projection the pipeline applies to every
// detection (to_global, geometry.py:237-256, called at pipeline.py:315 and :373).
//
// Per tile (one CTA): 19x19 cells x 5 anchors. For candidate i = cell*5 + anchor:
//   obj  = 1/(1+exp(-to)),  p = softmax(cls) at argmax (first max), conf = obj / sum_k exp(l_k - max)
//   cx = (col + sig(tx)) * 32, cy = (row + sig(ty)) * 32, w = aw*exp(tw)*32, h = ah*exp(th)*32
//   rect = [max(0,cx-w/2), min(608,cx+w/2)] x [...]; kept iff conf >= thresh and w,h > 0.
// Every float op uses the _rn intrinsics so nvcc cannot contract it into an FMA: the
// numpy restatement (oracle/yolo_ref.py::region_decode) performs the same op sequence.
// Sorted by (-conf, i). Projection follows the reference fp64 sequence exactly
// (mul then add, clip, round-half-even, >= 1 px), so given identical local rects the
// global rects are bit-identical.
#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

namespace {

constexpr int G = TP_GRID;
constexpr int NCAND = G * G * TP_ANCHORS;  // 1805
constexpr int SORT_N = 2048;

struct Anchors {
  float w[TP_ANCHORS], h[TP_ANCHORS];
};

__device__ __forceinline__ float sigmoid_rn(float x) {
  return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-x)));
}

struct Cand {
  bool keep;
  float conf, x1, y1, w, h;
  int cls;
};

__device__ Cand decode_one(const float* __restrict__ head, int cstride, int tile, int i,
                           const Anchors& an, float thresh) {
  const int cell = i / TP_ANCHORS, a = i - cell * TP_ANCHORS;
  const int row = cell / G, col = cell - row * G;
  const float* v = head + (((long long)tile * G + row) * G + col) * cstride +
                   a * (5 + TP_CLASSES);
  Cand c;
  const float obj = sigmoid_rn(v[4]);
  // conf = obj / s with s >= 1 exactly (the arg-max term is exp(0) = 1 and the rest are
  // >= 0), and correctly rounded division is monotonic, so obj < thresh already decides
  // rejection: skip the 80-class softmax (a dependent expf chain) for those candidates.
  if (obj < thresh) {
    c.keep = false;
    return c;
  }
  float m = v[5];
  int best = 0;
  for (int k = 1; k < TP_CLASSES; ++k) {
    const float l = v[5 + k];
    if (l > m) {
      m = l;
      best = k;
    }
  }
  float s = 0.0f;
  for (int k = 0; k < TP_CLASSES; ++k) s = __fadd_rn(s, expf(__fsub_rn(v[5 + k], m)));
  c.conf = __fdiv_rn(obj, s);
  c.cls = best;
  const float cx = __fmul_rn(__fadd_rn((float)col, sigmoid_rn(v[0])), 32.0f);
  const float cy = __fmul_rn(__fadd_rn((float)row, sigmoid_rn(v[1])), 32.0f);
  const float bw = __fmul_rn(__fmul_rn(an.w[a], expf(v[2])), 32.0f);
  const float bh = __fmul_rn(__fmul_rn(an.h[a], expf(v[3])), 32.0f);
  const float hw = __fmul_rn(bw, 0.5f), hh = __fmul_rn(bh, 0.5f);
  const float x1 = fmaxf(0.0f, __fsub_rn(cx, hw));
  const float y1 = fmaxf(0.0f, __fsub_rn(cy, hh));
  const float x2 = fminf(608.0f, __fadd_rn(cx, hw));
  const float y2 = fminf(608.0f, __fadd_rn(cy, hh));
  c.x1 = x1;
  c.y1 = y1;
  c.w = __fsub_rn(x2, x1);
  c.h = __fsub_rn(y2, y1);
  // NaN-safe: a non-finite logit never passes
  c.keep = (c.conf >= thresh) && (c.w > 0.0f) && (c.h > 0.0f);
  return c;
}

// to_global (geometry.py:237-256) for one edge pair; returns integer lo and hi.
__device__ __forceinline__ void project_axis(double g0, double s, double lo, double len,
                                             double frame_extent, int& ilo, int& ihi) {
  const double hi_local = __dadd_rn(lo, len);  // Rect.x2 = x + w
  double a = __dadd_rn(g0, __dmul_rn(lo, s));
  double b = __dadd_rn(g0, __dmul_rn(hi_local, s));
  a = fmin(a, frame_extent - 1.0);
  b = fmin(b, frame_extent);
  a = fmax(0.0, a);
  ilo = __double2int_rn(a);
  const int rb = __double2int_rn(b);
  ihi = max(ilo + 1, rb);
}

__global__ void __launch_bounds__(512) decode_kernel(const float* __restrict__ head, int cstride,
                                                     const int32_t* __restrict__ n_tiles_dev,
                                                     const tp_tile_job_t* __restrict__ jobs,
                                                     int frame_w, int frame_h, float thresh,
                                                     Anchors an, tp_det_t* __restrict__ out,
                                                     int max_per_tile, int32_t* __restrict__ counts) {
  __shared__ unsigned long long keys[SORT_N];
  __shared__ int n_keep;
  const int tile = blockIdx.x;
  if (n_tiles_dev != nullptr && tile >= *n_tiles_dev) return;
  if (threadIdx.x == 0) n_keep = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < NCAND; i += blockDim.x) {
    Cand c = decode_one(head, cstride, tile, i, an, thresh);
    if (c.keep) {
      const int slot = atomicAdd(&n_keep, 1);
      // descending conf (positive floats order like their bit patterns), then ascending i
      keys[slot] = ((unsigned long long)(0xFFFFFFFFu - __float_as_uint(c.conf)) << 32) |
                   (unsigned)i;
    }
  }
  __syncthreads();
  const int n = n_keep;
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  for (int i = n + threadIdx.x; i < np2; i += blockDim.x) keys[i] = ~0ull;
  __syncthreads();
  // bitonic sort (ascending) of np2 keys
  for (int k = 2; k <= np2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = keys[i], b = keys[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  const int n_out = min(n, max_per_tile);
  const tp_tile_job_t job = jobs[tile];
  const double s = __ddiv_rn((double)job.side, 608.0);
  for (int r = threadIdx.x; r < n_out; r += blockDim.x) {
    const int i = (int)(keys[r] & 0xFFFFFFFFu);
    Cand c = decode_one(head, cstride, tile, i, an, thresh);
    tp_det_t d;
    d.lx = c.x1;
    d.ly = c.y1;
    d.lw = c.w;
    d.lh = c.h;
    int x1, x2, y1, y2;
    project_axis((double)job.x, s, (double)c.x1, (double)c.w, (double)frame_w, x1, x2);
    project_axis((double)job.y, s, (double)c.y1, (double)c.h, (double)frame_h, y1, y2);
    d.gx = x1;
    d.gy = y1;
    d.gw = x2 - x1;
    d.gh = y2 - y1;
    d.conf = c.conf;
    d.cls = c.cls;
    d.crop_id = job.crop_id;
    d.frame = job.frame;
    out[(long long)tile * max_per_tile + r] = d;
  }
  if (threadIdx.x == 0) counts[tile] = n_out;
}

// attention_pass box list (pipeline.py:307-316): per frame, its A attention tiles in
// crop order, each tile's dets in detector order, kept iff conf >= min_conf.
// One warp per frame; ballot + popc compaction keeps the order.
__global__ void attention_boxes_kernel(const tp_det_t* __restrict__ dets,
                                       const int32_t* __restrict__ counts, int max_per_tile,
                                       int n_frames, int tiles_per_frame, double min_conf,
                                       double* __restrict__ boxes, int32_t* __restrict__ box_counts,
                                       int max_boxes) {
  const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (f >= n_frames) return;
  int n = 0;
  for (int a = 0; a < tiles_per_frame; ++a) {
    const int tile = f * tiles_per_frame + a;
    const int cnt = counts[tile];
    for (int base = 0; base < cnt; base += 32) {
      const int k = base + lane;
      tp_det_t d;
      bool take = false;
      if (k < cnt) {
        d = dets[(long long)tile * max_per_tile + k];
        take = (double)d.conf >= min_conf;
      }
      const unsigned m = __ballot_sync(0xffffffffu, take);
      const int pos = n + __popc(m & ((1u << lane) - 1u));
      if (take) {
        if (pos < max_boxes) {
          double* b = boxes + ((long long)f * max_boxes + pos) * 4;
          b[0] = d.gx;
          b[1] = d.gy;
          b[2] = d.gw;
          b[3] = d.gh;
        }
      }
      n += __popc(m);
    }
  }
  if (lane == 0) box_counts[f] = n;  // true count; > max_boxes means truncated
}

// final_pass tagged list (pipeline.py:365-375): frame f's jobs in job order (crop-id
// ascending), each tile's dets in detector order, widened to fp64 records.
__global__ void collect_final_kernel(const tp_det_t* __restrict__ dets,
                                     const int32_t* __restrict__ counts, int max_per_tile,
                                     const tp_tile_job_t* __restrict__ jobs,
                                     const int32_t* __restrict__ frame_job_start, int n_frames,
                                     tp_pdet_t* __restrict__ out, int32_t* __restrict__ out_counts,
                                     int max_per_frame) {
  const int f = blockIdx.x;
  if (f >= n_frames) return;
  const int j0 = frame_job_start[f], j1 = frame_job_start[f + 1];
  int n = 0;
  for (int j = j0; j < j1; ++j) {
    const int cnt = counts[j];
    const int cell = jobs[j].cell;
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
      const int pos = n + k;
      if (pos >= max_per_frame) continue;
      const tp_det_t d = dets[(long long)j * max_per_tile + k];
      tp_pdet_t r;
      r.x = d.gx;
      r.y = d.gy;
      r.w = d.gw;
      r.h = d.gh;
      r.conf = (double)d.conf;
      r.cls = d.cls;
      r.cell = cell;
      r.crop_id = d.crop_id;
      r.src = pos;
      out[(long long)f * max_per_frame + pos] = r;
    }
    n += cnt;
  }
  if (threadIdx.x == 0) out_counts[f] = n;  // true count; > max_per_frame means truncated
}

// to_global for detections produced by a foreign (host) detector plugin.
__global__ void project_kernel(const double* __restrict__ local, const int32_t* __restrict__ crop,
                               int n, int frame_w, int frame_h, int32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s = __ddiv_rn((double)crop[3 * i + 2], 608.0);
  const double* r = local + 4 * (long long)i;
  int x1, x2, y1, y2;
  if (frame_w > 0) {
    project_axis((double)crop[3 * i], s, r[0], r[2], (double)frame_w, x1, x2);
    project_axis((double)crop[3 * i + 1], s, r[1], r[3], (double)frame_h, y1, y2);
  } else {  // no frame clip (to_global without frame dims)
    const double gx = crop[3 * i], gy = crop[3 * i + 1];
    x1 = __double2int_rn(__dadd_rn(gx, __dmul_rn(r[0], s)));
    y1 = __double2int_rn(__dadd_rn(gy, __dmul_rn(r[1], s)));
    x2 = max(x1 + 1, __double2int_rn(__dadd_rn(gx, __dmul_rn(__dadd_rn(r[0], r[2]), s))));
    y2 = max(y1 + 1, __double2int_rn(__dadd_rn(gy, __dmul_rn(__dadd_rn(r[1], r[3]), s))));
  }
  out[4 * i] = x1;
  out[4 * i + 1] = y1;
  out[4 * i + 2] = x2 - x1;
  out[4 * i + 3] = y2 - y1;
}

}  // namespace

extern "C" int tp_project_rects(const double* local, const int32_t* crop_xyside, int n,
                                int frame_w, int frame_h, int32_t* out, void* stream) {
  if (local == nullptr || crop_xyside == nullptr || out == nullptr || n < 0) {
    tp_set_error("tp_project_rects: bad argument");
    return TP_ERR_ARG;
  }
  if (n == 0) return TP_OK;
  project_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(local, crop_xyside, n, frame_w,
                                                                     frame_h, out);
  TP_LAUNCH_CHECK();
  return TP_OK;
}

extern "C" int tp_region_decode(const float* head, int head_cstride, int n_tiles,
                                const int32_t* n_tiles_dev, const tp_tile_job_t* jobs, int frame_w,
                                int frame_h, float thresh, const float* anchors_host,
                                tp_det_t* out, int max_per_tile, int32_t* counts, void* stream) {
  if (head == nullptr || jobs == nullptr || out == nullptr || counts == nullptr ||
      anchors_host == nullptr || max_per_tile < 1 || head_cstride < TP_HEAD_CH) {
    tp_set_error("tp_region_decode: bad argument");
    return TP_ERR_ARG;
  }
  if (n_tiles <= 0) return TP_OK;
  Anchors an;
  for (int a = 0; a < TP_ANCHORS; ++a) {
    an.w[a] = anchors_host[2 * a];
    an.h[a] = anchors_host[2 * a + 1];
  }
  decode_kernel<<<n_tiles, 512, 0, (cudaStream_t)stream>>>(head, head_cstride, n_tiles_dev, jobs,
                                                           frame_w, frame_h, thresh, an, out,
                                                           max_per_tile, counts);
  TP_LAUNCH_CHECK();
  return TP_OK;
}

extern "C" int tp_attention_boxes(const tp_det_t* dets, const int32_t* counts, int max_per_tile,
                                  int n_frames, int tiles_per_frame, double min_conf,
                                  double* boxes, int32_t* box_counts, int max_boxes,
                                  void* stream) {
  if (dets == nullptr || counts == nullptr || boxes == nullptr || box_counts == nullptr ||
      tiles_per_frame < 1 || max_boxes < 1) {
    tp_set_error("tp_attention_boxes: bad argument");
    return TP_ERR_ARG;
  }
  if (n_frames <= 0) return TP_OK;
  const int warps = 4;
  attention_boxes_kernel<<<(n_frames + warps - 1) / warps, 32 * warps, 0, (cudaStream_t)stream>>>(
      dets, counts, max_per_tile, n_frames, tiles_per_frame, min_conf, boxes, box_counts,
      max_boxes);
  TP_LAUNCH_CHECK();
  return TP_OK;
}

extern "C" int tp_collect_final(const tp_det_t* dets, const int32_t* counts, int max_per_tile,
                                const tp_tile_job_t* jobs, const int32_t* frame_job_start,
                                int n_frames, tp_pdet_t* out, int32_t* out_counts,
                                int max_per_frame, void* stream) {
  if (dets == nullptr || counts == nullptr || jobs == nullptr || frame_job_start == nullptr ||
      out == nullptr || out_counts == nullptr || max_per_frame < 1) {
    tp_set_error("tp_collect_final: bad argument");
    return TP_ERR_ARG;
  }
  if (n_frames <= 0) return TP_OK;
  collect_final_kernel<<<n_frames, 256, 0, (cudaStream_t)stream>>>(
      dets, counts, max_per_tile, jobs, frame_job_start, n_frames, out, out_counts,
      max_per_frame);
  TP_LAUNCH_CHECK();
  return TP_OK;
}
