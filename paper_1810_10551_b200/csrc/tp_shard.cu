// Crop-parallel stage 2 across ranks (one 8K frame's active crops
// spread over GPUs). Every rank holds the same device job list (stage 1 + selection are
// replicated); rank r evaluates the contiguous slice [lo_r, lo_r + n_r) of it, sizes
// differing by at most one with the larger slices first — the reference's dispatch rule
// (pkg/src/tilepipe/distribution/client.py:82-96). After an all-gather of the per-rank
// padded slices (rank order == job order), tp_unslice_dets puts every tile's detection
// records back at its global job index, so collect_final / postprocess see exactly the
// single-GPU input. The job count stays on the device: no host synchronisation.
#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

namespace {

__device__ __forceinline__ void slice_of(int n, int rank, int world, int& lo, int& cnt) {
  const int base = n / world, extra = n % world;
  cnt = base + (rank < extra ? 1 : 0);
  lo = rank * base + min(rank, extra);
}

__global__ void slice_jobs_kernel(const tp_tile_job_t* __restrict__ jobs,
                                  const int32_t* __restrict__ n_dev, int rank, int world,
                                  tp_tile_job_t* __restrict__ out, int32_t* __restrict__ n_out,
                                  int max_out) {
  int lo, cnt;
  slice_of(*n_dev, rank, world, lo, cnt);
  if (cnt > max_out) cnt = max_out;  // the caller sizes max_out = ceil(max jobs / world)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
    out[i] = jobs[lo + i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = cnt;
}

// gathered: [world][max_slice] tiles of src_per_tile records (+ the tiles' TRUE counts);
// dst: global job order, dst_per_tile records per tile. A tile whose count exceeds
// src_per_tile lost records in the compact exchange: it is clamped and *overflow set
// (the host raises StageFailure; never a silent truncation).
__global__ void unslice_kernel(const tp_det_t* __restrict__ src, const int32_t* __restrict__ src_counts,
                               int max_slice, const int32_t* __restrict__ n_dev, int world,
                               int src_per_tile, int dst_per_tile, tp_det_t* __restrict__ dst,
                               int32_t* __restrict__ dst_counts, int32_t* __restrict__ overflow) {
  const int j = blockIdx.x;  // global job index
  const int n = *n_dev;
  if (j >= n) return;
  const int base = n / world, extra = n % world;
  // rank owning job j: the first `extra` ranks hold base+1 jobs
  int r, i;
  if (j < extra * (base + 1)) {
    r = j / (base + 1);
    i = j - r * (base + 1);
  } else {
    const int jj = j - extra * (base + 1);
    r = extra + jj / base;
    i = jj - (r - extra) * base;
  }
  const long long s = (long long)r * max_slice + i;
  int cnt = src_counts[s];
  if (cnt > src_per_tile) {
    if (threadIdx.x == 0 && overflow != nullptr) atomicOr(overflow, 1);
    cnt = src_per_tile;
  }
  if (cnt > dst_per_tile) cnt = dst_per_tile;
  if (threadIdx.x == 0) dst_counts[j] = cnt;
  for (int k = threadIdx.x; k < cnt; k += blockDim.x)
    dst[(long long)j * dst_per_tile + k] = src[s * src_per_tile + k];
}

}  // namespace

extern "C" int tp_slice_jobs(const tp_tile_job_t* jobs, const int32_t* n_jobs_dev, int rank,
                             int world, tp_tile_job_t* out, int32_t* n_out_dev, int max_out,
                             void* stream) {
  if (jobs == nullptr || n_jobs_dev == nullptr || out == nullptr || n_out_dev == nullptr ||
      world < 1 || rank < 0 || rank >= world || max_out < 1) {
    tp_set_error("tp_slice_jobs: bad argument");
    return TP_ERR_ARG;
  }
  const int blocks = (max_out + 255) / 256;
  slice_jobs_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(jobs, n_jobs_dev, rank, world, out,
                                                              n_out_dev, max_out);
  TP_LAUNCH_CHECK();
  return TP_OK;
}

extern "C" int tp_unslice_dets(const tp_det_t* gathered, const int32_t* gathered_counts,
                               int max_slice, const int32_t* n_jobs_dev, int world, int max_jobs,
                               int src_per_tile, int dst_per_tile, tp_det_t* dets, int32_t* counts,
                               int32_t* overflow, void* stream) {
  if (gathered == nullptr || gathered_counts == nullptr || n_jobs_dev == nullptr ||
      dets == nullptr || counts == nullptr || world < 1 || max_slice < 1 || max_jobs < 1 ||
      src_per_tile < 1 || dst_per_tile < 1) {
    tp_set_error("tp_unslice_dets: bad argument");
    return TP_ERR_ARG;
  }
  unslice_kernel<<<max_jobs, 256, 0, (cudaStream_t)stream>>>(
      gathered, gathered_counts, max_slice, n_jobs_dev, world, src_per_tile, dst_per_tile, dets,
      counts, overflow);
  TP_LAUNCH_CHECK();
  return TP_OK;
}
