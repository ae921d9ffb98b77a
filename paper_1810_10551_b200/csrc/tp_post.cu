// K7 — per-frame postprocess: greedy per-class NMS, cross-border merge, min_conf filter.
//
// Reference: nms_keep_indices (pkg/src/tilepipe/postprocess.py:54-73), merge_split with
// _gap/_cells_adjacent/_can_merge (:81-163), postprocess and its variants (:166-187),
// finish_detections (pipeline.py:378-385), iou (geometry.py:85-91).
//
// Semantics reproduced exactly:
//  * NMS visits candidates by (-conf, input index) and keeps a candidate iff its IoU with
//    every kept box of the same class is < threshold; IoU in fp64 with the reference's
//    op order (x2 = x + w, inter = (x2-x1)*(y2-y1), iou = inter / ((aA + bA) - inter)).
//    nms_per_crop groups by crop id in first-appearance order.
//  * merge_split repeatedly merges the lexicographically first mergeable pair (i, j),
//    i < j, into slot i (union rect, max confidence, union of grid cells), deletes j and
//    restarts. Cell sets are 256-bit masks over row*cols+col, so "adjacent along an
//    axis" is a shift-and-AND. After merging (i, j) only pairs (a, i) with a < i and
//    pairs whose first index is >= i can have changed, so the rescan starts there —
//    this returns the same first pair the full restart would.
// One CTA (512 threads) per frame; all working state in shared memory (<= 2048 entries).
#include <mutex>

#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

namespace {

constexpr int MAXN = 2048;
constexpr int NT = 512;

struct Work {
  double *x, *y, *w, *h, *conf;
  int *cls, *crop, *src, *order, *kept, *grank;
  short* cell;
  unsigned long long* cells;  // [MAXN][4]
};

__device__ __forceinline__ Work carve(uint8_t* sm) {
  Work W;
  double* d = reinterpret_cast<double*>(sm);
  W.x = d;
  W.y = d + MAXN;
  W.w = d + 2 * MAXN;
  W.h = d + 3 * MAXN;
  W.conf = d + 4 * MAXN;
  W.cells = reinterpret_cast<unsigned long long*>(d + 5 * MAXN);
  int* i = reinterpret_cast<int*>(W.cells + 4 * MAXN);
  W.cls = i;
  W.crop = i + MAXN;
  W.src = i + 2 * MAXN;
  W.order = i + 3 * MAXN;
  W.kept = i + 4 * MAXN;
  W.grank = i + 5 * MAXN;
  W.cell = reinterpret_cast<short*>(i + 6 * MAXN);
  return W;
}
constexpr size_t kSmemBytes = (size_t)MAXN * (5 * 8 + 4 * 8 + 6 * 4 + 2) + 64;

__device__ __forceinline__ double iou_ref(const Work& W, int a, int b) {
  const double ax2 = __dadd_rn(W.x[a], W.w[a]), ay2 = __dadd_rn(W.y[a], W.h[a]);
  const double bx2 = __dadd_rn(W.x[b], W.w[b]), by2 = __dadd_rn(W.y[b], W.h[b]);
  const double x1 = fmax(W.x[a], W.x[b]), y1 = fmax(W.y[a], W.y[b]);
  const double x2 = fmin(ax2, bx2), y2 = fmin(ay2, by2);
  if (x2 <= x1 || y2 <= y1) return 0.0;
  const double inter = __dmul_rn(__dsub_rn(x2, x1), __dsub_rn(y2, y1));
  const double aa = __dmul_rn(W.w[a], W.h[a]), ab = __dmul_rn(W.w[b], W.h[b]);
  return __ddiv_rn(inter, __dsub_rn(__dadd_rn(aa, ab), inter));
}

// ---- 256-bit cell sets
struct Cells {
  unsigned long long v[4];
};
__device__ __forceinline__ Cells load_cells(const Work& W, int i) {
  Cells c;
#pragma unroll
  for (int k = 0; k < 4; ++k) c.v[k] = W.cells[4 * i + k];
  return c;
}
__device__ __forceinline__ Cells shl(const Cells& a, int s) {  // toward higher cell index
  Cells r;
  const int ws = s >> 6, bs = s & 63;
#pragma unroll
  for (int k = 3; k >= 0; --k) {
    const int src = k - ws;
    unsigned long long lo = src >= 0 ? a.v[src] : 0ull;
    unsigned long long lo2 = src - 1 >= 0 ? a.v[src - 1] : 0ull;
    r.v[k] = bs ? ((lo << bs) | (lo2 >> (64 - bs))) : lo;
  }
  return r;
}
__device__ __forceinline__ Cells shr(const Cells& a, int s) {  // toward lower cell index
  Cells r;
  const int ws = s >> 6, bs = s & 63;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int src = k + ws;
    unsigned long long hi = src < 4 ? a.v[src] : 0ull;
    unsigned long long hi2 = src + 1 < 4 ? a.v[src + 1] : 0ull;
    r.v[k] = bs ? ((hi >> bs) | (hi2 << (64 - bs))) : hi;
  }
  return r;
}
__device__ __forceinline__ bool any_and(const Cells& a, const Cells& b) {
  return ((a.v[0] & b.v[0]) | (a.v[1] & b.v[1]) | (a.v[2] & b.v[2]) | (a.v[3] & b.v[3])) != 0ull;
}
// keep only cells whose column != col (used before horizontal shifts)
__device__ __forceinline__ Cells drop_column(const Cells& a, int col, int cols, int n_cells) {
  Cells r = a;
  for (int c = col; c < n_cells; c += cols) r.v[c >> 6] &= ~(1ull << (c & 63));
  return r;
}

__device__ bool can_merge(const Work& W, int a, int b, const tp_post_policy_t& P) {
  if (W.cls[a] != W.cls[b]) return false;
  const int cls = W.cls[a];
  const int rule = (cls >= 0 && cls < TP_MAX_CLASSES) ? P.class_rule[cls] : 0;
  if (rule == TP_RULE_NONE) return false;
  const Cells A = load_cells(W, a), B = load_cells(W, b);
  const double ax2 = __dadd_rn(W.x[a], W.w[a]), ay2 = __dadd_rn(W.y[a], W.h[a]);
  const double bx2 = __dadd_rn(W.x[b], W.w[b]), by2 = __dadd_rn(W.y[b], W.h[b]);
  if (rule & TP_RULE_VERTICAL) {
    const int C = P.grid_cols;
    const bool adj = any_and(shl(A, C), B) || any_and(shr(A, C), B);
    if (adj) {
      const double gap = __dsub_rn(fmax(W.y[a], W.y[b]), fmin(ay2, by2));
      if (gap <= P.gap_px && fabs(__dsub_rn(W.x[a], W.x[b])) <= P.tol_px &&
          fabs(__dsub_rn(ax2, bx2)) <= P.tol_px)
        return true;
    }
  }
  if (rule & TP_RULE_HORIZONTAL) {
    const int C = P.grid_cols;
    const bool adj = any_and(shl(drop_column(A, C - 1, C, P.n_cells), 1), B) ||
                     any_and(shr(drop_column(A, 0, C, P.n_cells), 1), B);
    if (adj) {
      const double gap = __dsub_rn(fmax(W.x[a], W.x[b]), fmin(ax2, bx2));
      if (gap <= P.gap_px && fabs(__dsub_rn(W.y[a], W.y[b])) <= P.tol_px &&
          fabs(__dsub_rn(ay2, by2)) <= P.tol_px)
        return true;
    }
  }
  return false;
}

// Permute all per-entry fields so that new[k] = old[idx[k]], k < m (field by field).
__device__ void permute(Work& W, const int* idx, int m) {
  constexpr int PER = MAXN / NT;
#define TP_PERMUTE_FIELD(T, arr)                                          \
  {                                                                       \
    T tmp[PER];                                                           \
    _Pragma("unroll") for (int r = 0; r < PER; ++r) {                     \
      const int k = threadIdx.x + r * NT;                                 \
      if (k < m) tmp[r] = arr[idx[k]];                                    \
    }                                                                     \
    __syncthreads();                                                      \
    _Pragma("unroll") for (int r = 0; r < PER; ++r) {                     \
      const int k = threadIdx.x + r * NT;                                 \
      if (k < m) arr[k] = tmp[r];                                         \
    }                                                                     \
    __syncthreads();                                                      \
  }
  TP_PERMUTE_FIELD(double, W.x)
  TP_PERMUTE_FIELD(double, W.y)
  TP_PERMUTE_FIELD(double, W.w)
  TP_PERMUTE_FIELD(double, W.h)
  TP_PERMUTE_FIELD(double, W.conf)
  TP_PERMUTE_FIELD(int, W.cls)
  TP_PERMUTE_FIELD(int, W.crop)
  TP_PERMUTE_FIELD(int, W.src)
  TP_PERMUTE_FIELD(short, W.cell)
  for (int q = 0; q < 4; ++q) {
    unsigned long long tmp[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int k = threadIdx.x + r * NT;
      if (k < m) tmp[r] = W.cells[4 * idx[k] + q];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int k = threadIdx.x + r * NT;
      if (k < m) W.cells[4 * k + q] = tmp[r];
    }
    __syncthreads();
  }
#undef TP_PERMUTE_FIELD
}

__device__ __forceinline__ bool nms_before(const Work& W, int i, int j) {
  if (W.grank[i] != W.grank[j]) return W.grank[i] < W.grank[j];
  if (W.conf[i] != W.conf[j]) return W.conf[i] > W.conf[j];
  return i < j;
}

// Greedy NMS over W[0..n). Returns kept count; W.kept holds kept indices in keep order.
__device__ int run_nms(Work& W, int n, double thr, bool per_crop, int* s_int) {
  // group ranks (first appearance index of the crop id) for per-crop mode
  for (int i = threadIdx.x; i < n; i += NT) {
    int g = 0;
    if (per_crop) {
      g = i;
      for (int j = 0; j < i; ++j)
        if (W.crop[j] == W.crop[i]) {
          g = j;
          break;
        }
    }
    W.grank[i] = g;
  }
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  for (int i = threadIdx.x; i < np2; i += NT) W.order[i] = i < n ? i : -1;
  __syncthreads();
  for (int k = 2; k <= np2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np2; i += NT) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int a = W.order[i], b = W.order[ixj];
          // -1 (padding) sorts last
          const bool a_after_b = (a < 0) ? (b >= 0) : (b >= 0 && nms_before(W, b, a));
          const bool up = (i & k) == 0;
          if (a_after_b == up) {
            W.order[i] = b;
            W.order[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // Greedy NMS in batches of 32 candidates (sort order): every thread tests the batch
  // against the kept list and against itself (32x32 suppression bits), then warp 0
  // resolves the batch in order with bit operations. Same decisions as the one-at-a-time
  // scan (candidate c survives iff no KEPT earlier candidate suppresses it); 2 barriers
  // per 32 candidates instead of 2 per candidate.
  unsigned* s_sup = reinterpret_cast<unsigned*>(&s_int[4]);  // [0] by-kept mask, [1..32] rows
  int kn = 0;
  if (threadIdx.x == 0) s_int[0] = 0;
  __syncthreads();  // n == 0 runs no batch: the count must still be visible to everyone
  for (int base = 0; base < n; base += 32) {
    const int m = min(32, n - base);
    for (int t = threadIdx.x; t < 33; t += NT) s_sup[t] = 0u;
    __syncthreads();
    // (a) batch candidate c vs kept k
    for (int t = threadIdx.x; t < m * kn; t += NT) {
      const int c = t / kn, k = t - c * kn;
      const int i = W.order[base + c], j = W.kept[k];
      if (W.cls[j] != W.cls[i] || (per_crop && W.crop[j] != W.crop[i])) continue;
      if (!(iou_ref(W, j, i) < thr)) atomicOr(&s_sup[0], 1u << c);
    }
    // (b) c1 < c2 inside the batch: does c1 (if kept) suppress c2?
    for (int t = threadIdx.x; t < m * m; t += NT) {
      const int c1 = t / m, c2 = t - c1 * m;
      if (c2 <= c1) continue;
      const int i1 = W.order[base + c1], i2 = W.order[base + c2];
      if (W.cls[i1] != W.cls[i2] || (per_crop && W.crop[i1] != W.crop[i2])) continue;
      if (!(iou_ref(W, i1, i2) < thr)) atomicOr(&s_sup[1 + c1], 1u << c2);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // resolve in order
      unsigned alive = ~s_sup[0] & (m == 32 ? 0xffffffffu : ((1u << m) - 1u));
      unsigned keep = 0u;
      for (int c = 0; c < m; ++c) {
        if (alive & (1u << c)) {
          keep |= 1u << c;
          alive &= ~s_sup[1 + c];
        }
      }
      const int lane = threadIdx.x;
      if (keep & (1u << lane)) W.kept[kn + __popc(keep & ((1u << lane) - 1u))] = W.order[base + lane];
      if (lane == 0) s_int[0] = kn + __popc(keep);
    }
    __syncthreads();
    kn = s_int[0];
  }
  return s_int[0];
}

// merge_split fixpoint over W[0..n) (list order). Returns the new length.
__device__ int run_merge(Work& W, int n, const tp_post_policy_t& P, int* s_int) {
  int lo = 0;
  for (;;) {
    if (threadIdx.x == 0) s_int[1] = 0x7fffffff;
    __syncthreads();
    // pairs (a, lo) with a < lo
    for (int a = threadIdx.x; a < lo; a += NT)
      if (can_merge(W, a, lo, P)) atomicMin(&s_int[1], a * MAXN + lo);
    // pairs lo <= a < b < n: row a per warp, columns b per lane; a row is skipped once a
    // pair of an earlier row is known (racy but monotone bound)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int a = lo + warp; a < n - 1; a += NT / 32) {
      if (a * MAXN >= *(volatile int*)&s_int[1]) break;
      for (int b = a + 1 + lane; b < n; b += 32) {
        if (a * MAXN + b >= *(volatile int*)&s_int[1]) break;
        if (can_merge(W, a, b, P)) {
          atomicMin(&s_int[1], a * MAXN + b);
          break;
        }
      }
    }
    __syncthreads();
    const int best = s_int[1];
    if (best == 0x7fffffff) break;
    const int i = best / MAXN, j = best % MAXN;
    if (threadIdx.x == 0) {
      const double ax2 = __dadd_rn(W.x[i], W.w[i]), ay2 = __dadd_rn(W.y[i], W.h[i]);
      const double bx2 = __dadd_rn(W.x[j], W.w[j]), by2 = __dadd_rn(W.y[j], W.h[j]);
      const double x1 = fmin(W.x[i], W.x[j]), y1 = fmin(W.y[i], W.y[j]);
      const double x2 = fmax(ax2, bx2), y2 = fmax(ay2, by2);
      W.x[i] = x1;
      W.y[i] = y1;
      W.w[i] = __dsub_rn(x2, x1);
      W.h[i] = __dsub_rn(y2, y1);
      W.conf[i] = fmax(W.conf[i], W.conf[j]);
      for (int q = 0; q < 4; ++q) W.cells[4 * i + q] |= W.cells[4 * j + q];
    }
    __syncthreads();
    // delete j: new[k] = old[k + (k >= j)]
    for (int k = threadIdx.x; k < n - 1; k += NT) W.order[k] = k < j ? k : k + 1;
    __syncthreads();
    permute(W, W.order, n - 1);
    n -= 1;
    lo = i;
  }
  return n;
}

__global__ void __launch_bounds__(NT, 1)
    postprocess_kernel(const tp_pdet_t* __restrict__ dets, const int32_t* __restrict__ counts,
                       int max_per_frame, const tp_post_policy_t P, tp_pdet_t* __restrict__ out,
                       int32_t* __restrict__ out_counts, int32_t* __restrict__ keep_idx,
                       int32_t* __restrict__ keep_counts) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_int[40];  // [0..3] scalars, [4..36] NMS batch suppression bits
  Work W = carve(smem);
  const int f = blockIdx.x;
  int n = min(counts[f], max_per_frame);
  if (n > MAXN) n = MAXN;  // host rejects this case before launch
  const tp_pdet_t* in = dets + (long long)f * max_per_frame;
  for (int i = threadIdx.x; i < n; i += NT) {
    const tp_pdet_t d = in[i];
    W.x[i] = d.x;
    W.y[i] = d.y;
    W.w[i] = d.w;
    W.h[i] = d.h;
    W.conf[i] = d.conf;
    W.cls[i] = d.cls;
    W.crop[i] = d.crop_id;
    W.src[i] = d.src;
    W.cell[i] = (short)d.cell;
    for (int q = 0; q < 4; ++q) W.cells[4 * i + q] = 0ull;
    if (d.cell >= 0 && d.cell < 256) W.cells[4 * i + (d.cell >> 6)] = 1ull << (d.cell & 63);
  }
  __syncthreads();

  // reference precedence: nms_per_crop wins over merge_before_nms (postprocess.py:175-185)
  const bool merge_first = P.merge_before_nms && !P.nms_per_crop && P.do_merge && P.do_nms;
  if (merge_first) n = run_merge(W, n, P, s_int);
  if (P.do_nms) {
    const int kn = run_nms(W, n, P.nms_iou, P.nms_per_crop != 0, s_int);
    if (keep_idx != nullptr) {
      for (int k = threadIdx.x; k < kn; k += NT)
        keep_idx[(long long)f * max_per_frame + k] = merge_first ? W.kept[k] : W.src[W.kept[k]];
      if (threadIdx.x == 0) keep_counts[f] = kn;
    }
    permute(W, W.kept, kn);
    n = kn;
  }
  if (P.do_merge && !merge_first) n = run_merge(W, n, P, s_int);

  // final confidence filter (finish_detections), order-preserving
  if (threadIdx.x == 0) s_int[2] = 0;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int m = 0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const bool take = i < n && (P.min_conf < 0.0 || W.conf[i] >= P.min_conf);
      const unsigned b = __ballot_sync(0xffffffffu, take);
      if (take) {
        const int pos = m + __popc(b & ((1u << lane) - 1u));
        tp_pdet_t o;
        o.x = W.x[i];
        o.y = W.y[i];
        o.w = W.w[i];
        o.h = W.h[i];
        o.conf = W.conf[i];
        o.cls = W.cls[i];
        o.cell = W.cell[i];
        o.crop_id = W.crop[i];
        o.src = W.src[i];
        out[(long long)f * max_per_frame + pos] = o;
      }
      m += __popc(b);
    }
    if (lane == 0) out_counts[f] = m;
  }
}

}  // namespace

extern "C" int tp_postprocess(const tp_pdet_t* dets, const int32_t* counts, int n_frames,
                              int max_per_frame, const tp_post_policy_t* policy, tp_pdet_t* out,
                              int32_t* out_counts, int32_t* keep_idx, int32_t* keep_counts,
                              void* stream) {
  if (dets == nullptr || counts == nullptr || policy == nullptr || out == nullptr ||
      out_counts == nullptr || max_per_frame < 1 || policy->n_cells > 256 ||
      policy->grid_cols < 1 || (keep_idx != nullptr && keep_counts == nullptr)) {
    tp_set_error("tp_postprocess: bad argument");
    return TP_ERR_ARG;
  }
  if (max_per_frame > MAXN) {
    tp_set_error("tp_postprocess: max_per_frame %d exceeds %d", max_per_frame, MAXN);
    return TP_ERR_CAPACITY;
  }
  if (n_frames <= 0) return TP_OK;
  {  // dynamic-smem opt-in: a per-device function attribute, set once per device
    static std::mutex mu;
    static uint64_t done = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    std::lock_guard<std::mutex> lock(mu);
    if (!(done & bit)) {
      TP_CUDA_CHECK(cudaFuncSetAttribute(postprocess_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemBytes));
      done |= bit;
    }
  }
  postprocess_kernel<<<n_frames, NT, kSmemBytes, (cudaStream_t)stream>>>(
      dets, counts, max_per_frame, *policy, out, out_counts, keep_idx, keep_counts);
  TP_LAUNCH_CHECK();
  return TP_OK;
}
