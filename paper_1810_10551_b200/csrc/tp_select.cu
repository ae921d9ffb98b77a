// K6 — temporal attention merge + active-crop selection + stage-2 job list.
//
// Reference: merge_temporal (pkg/src/tilepipe/pipeline.py:319-338: union of the last
// `window` models' boxes, first-seen de-duplication by Rect equality) and
// select_active (pipeline.py:341-354: crop active iff it strictly intersects any box
// dilated by the margin and clipped to the frame; Rect.dilated geometry.py:71-77,
// intersects geometry.py:80-82). Arithmetic is fp64 with the reference's exact op
// order (x2 = x + w recomputed from the dilated rect), so selections are bit-exact
// for any box values, not just integers.
//
// One CTA per frame. De-duplication: each box compares against all earlier ones;
// order-preserving compaction with warp ballots. Selection: one lane per crop, the
// whole box list broadcast from shared memory; __ballot_sync gives 32 crops' active
// bits at once and popc prefixes compact them into ascending crop-id order.
#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

namespace {

constexpr int MAX_IN = 512;  // boxes in one window (all slots); static smem budget
constexpr int MAX_CROPS = 1024;

__global__ void __launch_bounds__(256) select_kernel(
    const double* __restrict__ boxes, const int32_t* __restrict__ box_counts, int max_boxes,
    int n_frames, int window, const double* __restrict__ crops, int n_crops, int crop_id_base,
    double margin, double frame_w, double frame_h, uint32_t* __restrict__ active_mask,
    int mask_words, int32_t* __restrict__ active_ids, int32_t* __restrict__ active_counts,
    double* __restrict__ merged, int32_t* __restrict__ merged_counts, int max_merged) {
  __shared__ double bx[MAX_IN], by[MAX_IN], bw[MAX_IN], bh[MAX_IN];
  __shared__ unsigned char keep[MAX_IN];
  __shared__ double dx1[MAX_IN], dy1[MAX_IN], dw[MAX_IN], dh[MAX_IN];
  __shared__ int warp_tot[8];
  __shared__ int n_in_s, n_kept_s, n_total_s;
  const int f = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;

  if (tid == 0) {
    int n = 0;
    for (int s = 0; s < window; ++s) n += min(box_counts[f + s], max_boxes);
    n_total_s = n;
    n_in_s = min(n, MAX_IN);
  }
  __syncthreads();
  const int n_in = n_in_s;
  // gather the window's boxes in slot order
  {
    int base = 0;
    for (int s = 0; s < window; ++s) {
      const int cnt = min(box_counts[f + s], max_boxes);
      for (int k = tid; k < cnt; k += blockDim.x) {
        const int i = base + k;
        if (i < MAX_IN) {
          const double* b = boxes + ((long long)(f + s) * max_boxes + k) * 4;
          bx[i] = b[0];
          by[i] = b[1];
          bw[i] = b[2];
          bh[i] = b[3];
        }
      }
      base += cnt;
    }
  }
  __syncthreads();
  // first-seen de-duplication (Rect equality == all four fields equal)
  for (int i = tid; i < n_in; i += blockDim.x) {
    bool dup = false;
    for (int j = 0; j < i && !dup; ++j)
      dup = bx[j] == bx[i] && by[j] == by[i] && bw[j] == bw[i] && bh[j] == bh[i];
    keep[i] = dup ? 0 : 1;
  }
  __syncthreads();
  // order-preserving compaction of kept boxes into the dilated arrays + merged output
  if (tid == 0) n_kept_s = 0;
  __syncthreads();
  for (int base = 0; base < n_in; base += blockDim.x) {
    const int i = base + tid;
    const bool k = i < n_in && keep[i];
    const unsigned m = __ballot_sync(0xffffffffu, k);
    if (lane == 0) warp_tot[wid] = __popc(m);
    __syncthreads();
    int off = n_kept_s;
    for (int w = 0; w < wid; ++w) off += warp_tot[w];
    const int pos = off + __popc(m & ((1u << lane) - 1u));
    if (k) {
      // Rect.dilated: clip to the frame, then width = x2 - x1
      const double x1 = fmax(0.0, __dsub_rn(bx[i], margin));
      const double y1 = fmax(0.0, __dsub_rn(by[i], margin));
      const double x2 = fmin(frame_w, __dadd_rn(__dadd_rn(bx[i], bw[i]), margin));
      const double y2 = fmin(frame_h, __dadd_rn(__dadd_rn(by[i], bh[i]), margin));
      dx1[pos] = x1;
      dy1[pos] = y1;
      dw[pos] = __dsub_rn(x2, x1);
      dh[pos] = __dsub_rn(y2, y1);
      if (pos < max_merged) {
        double* o = merged + ((long long)f * max_merged + pos) * 4;
        o[0] = bx[i];
        o[1] = by[i];
        o[2] = bw[i];
        o[3] = bh[i];
      }
    }
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < nw; ++w) t += warp_tot[w];
      n_kept_s += t;
    }
    __syncthreads();
  }
  const int n_kept = n_kept_s;
  // selection: lane = crop; ballot -> 32 active bits per warp-iteration
  for (int c0 = wid * 32; c0 < ((n_crops + 31) / 32) * 32; c0 += nw * 32) {
    const int c = c0 + lane;
    bool hit = false;
    if (c < n_crops) {
      const double cx = crops[4 * c], cy = crops[4 * c + 1], cw = crops[4 * c + 2],
                   ch = crops[4 * c + 3];
      const double cx2 = __dadd_rn(cx, cw), cy2 = __dadd_rn(cy, ch);
      for (int b = 0; b < n_kept && !hit; ++b) {
        if (!(dw[b] > 0.0 && dh[b] > 0.0)) continue;  // degenerate box: Rect would reject it
        const double ex2 = __dadd_rn(dx1[b], dw[b]), ey2 = __dadd_rn(dy1[b], dh[b]);
        hit = fmin(cx2, ex2) > fmax(cx, dx1[b]) && fmin(cy2, ey2) > fmax(cy, dy1[b]);
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0 && (c0 >> 5) < mask_words) active_mask[(long long)f * mask_words + (c0 >> 5)] = m;
  }
  __syncthreads();
  // ascending compaction of active ids (warp 0 walks the mask words)
  if (wid == 0) {
    int n = 0;
    const int words = (n_crops + 31) / 32;
    for (int w = 0; w < words; ++w) {
      const unsigned m = active_mask[(long long)f * mask_words + w];
      if ((m >> lane) & 1u) {
        const int pos = n + __popc(m & ((1u << lane) - 1u));
        active_ids[(long long)f * n_crops + pos] = crop_id_base + w * 32 + lane;
      }
      n += __popc(m);
    }
    if (lane == 0) {
      active_counts[f] = n;
      // a window holding more than MAX_IN boxes was truncated: report its true size
      // (> MAX_IN >= max_merged) so the host raises instead of using the partial result
      merged_counts[f] = n_total_s > MAX_IN ? n_total_s : n_kept;
    }
  }
}

__global__ void build_jobs_kernel(const int32_t* __restrict__ active_ids,
                                  const int32_t* __restrict__ active_counts, int n_frames,
                                  int max_active, const int32_t* __restrict__ crop_table,
                                  int crop_id_base, tp_tile_job_t* __restrict__ jobs,
                                  int32_t* __restrict__ frame_job_start,
                                  int32_t* __restrict__ n_jobs_dev) {
  __shared__ int start[4097];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int f = 0; f < n_frames; ++f) {
      start[f] = acc;
      acc += active_counts[f];
    }
    start[n_frames] = acc;
    *n_jobs_dev = acc;
  }
  __syncthreads();
  for (int f = threadIdx.x; f <= n_frames; f += blockDim.x) frame_job_start[f] = start[f];
  for (int f = 0; f < n_frames; ++f) {
    const int cnt = active_counts[f];
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
      const int cid = active_ids[(long long)f * max_active + k];
      const int li = cid - crop_id_base;
      tp_tile_job_t j;
      j.frame = f;
      j.crop_id = cid;
      j.x = crop_table[4 * li];
      j.y = crop_table[4 * li + 1];
      j.side = crop_table[4 * li + 2];
      j.cell = crop_table[4 * li + 3];
      j.pad0 = 0;
      j.pad1 = 0;
      jobs[start[f] + k] = j;
    }
  }
}

}  // namespace

extern "C" int tp_select_active(const double* boxes, const int32_t* box_counts, int max_boxes,
                                int n_frames, int window, const double* crops, int n_crops,
                                int crop_id_base, double margin, double frame_w, double frame_h,
                                uint32_t* active_mask, int mask_words, int32_t* active_ids,
                                int32_t* active_counts, double* merged, int32_t* merged_counts,
                                int max_merged, void* stream) {
  if (boxes == nullptr || box_counts == nullptr || crops == nullptr || active_mask == nullptr ||
      active_ids == nullptr || active_counts == nullptr || merged == nullptr ||
      merged_counts == nullptr || window < 1 || n_crops < 1 || n_crops > MAX_CROPS ||
      mask_words < (n_crops + 31) / 32 || margin < 0 || max_merged < 1 || max_merged > MAX_IN) {
    tp_set_error("tp_select_active: bad argument (max_merged must be 1..%d)", MAX_IN);
    return TP_ERR_ARG;
  }
  if (n_frames <= 0) return TP_OK;
  select_kernel<<<n_frames, 256, 0, (cudaStream_t)stream>>>(
      boxes, box_counts, max_boxes, n_frames, window, crops, n_crops, crop_id_base, margin,
      frame_w, frame_h, active_mask, mask_words, active_ids, active_counts, merged,
      merged_counts, max_merged);
  TP_LAUNCH_CHECK();
  return TP_OK;
}

extern "C" int tp_build_jobs(const int32_t* active_ids, const int32_t* active_counts, int n_frames,
                             int max_active, const int32_t* crop_table, int crop_id_base,
                             tp_tile_job_t* jobs, int32_t* frame_job_start, int32_t* n_jobs_dev,
                             void* stream) {
  if (active_ids == nullptr || active_counts == nullptr || crop_table == nullptr ||
      jobs == nullptr || frame_job_start == nullptr || n_jobs_dev == nullptr || n_frames < 0 ||
      n_frames > 4096) {
    tp_set_error("tp_build_jobs: bad argument");
    return TP_ERR_ARG;
  }
  build_jobs_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(active_ids, active_counts, n_frames,
                                                         max_active, crop_table, crop_id_base,
                                                         jobs, frame_job_start, n_jobs_dev);
  TP_LAUNCH_CHECK();
  return TP_OK;
}
