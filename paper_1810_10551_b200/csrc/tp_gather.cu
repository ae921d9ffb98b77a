// K1/K2 — frame ingest + crop gather: crop square -> 608x608 tile.
//
// Replaces the reference tile cutter `cut_tile` (pkg/src/tilepipe/detector.py:223-247),
// which maps output pixel u to source floor(u*side/608) and zero-fills crop area that
// lies outside the frame. Mode NEAREST is bit-exact with it. Mode BILINEAR is the
// north-star downscale: 8-bit fixed-point weights, half-pixel centres, identical
// integer arithmetic to oracle/resample_ref.py so it is bit-exact as well.
//
// One CTA per (tile, 8 output rows); a warp task is 32 consecutive columns of one row
// (608 = 19 x 32, so a warp never straddles rows). Each lane produces one pixel: 3 bytes
// of the u8 tile and/or one 16-byte slot of the layer-0 input ([tile][610][610][8],
// fp16/bf16, zero 1-px halo): slot X of a row holds [q(X-1) rgb0 | q(X) rgb0] for tile
// pixels q (zero outside [0, 608)), so slots x and x+1 are layer 0's 32-byte A row
// [q(x-1) q(x) q(x) q(x+1)] — the conv's TMA map reads it through an overlapping view. Every store is one aligned 16-byte vector; a warp writes 512 B
// contiguous. Index math is 32-bit (divisions by the constant 608 / 1216 become
// multiply-highs); the value/255 table is built once per CTA. HBM-bound on the writes.
#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

namespace {

constexpr int S = TP_MODEL_SIDE;
constexpr int SP = S + 2;  // padded side of the layer-0 activation buffer (8 halves / slot)

struct Tap {
  int i0, i1, f;  // source offsets (relative to crop origin) and 8-bit weight of i1
};

__device__ __forceinline__ Tap bilinear_tap(int u, int side) {
  // source centre = (u + 0.5) * side / 608 - 0.5 ; fixed point with 8 fraction bits
  int num = (2 * u + 1) * side - S;  // = 1216 * centre
  if (num < 0) num = 0;
  // num * 256 < 2^32 for side <= 13000: unsigned 32-bit division by a constant
  const int s256 = (int)(((uint32_t)num * 256u) / (uint32_t)(2 * S));
  Tap t;
  t.i0 = s256 >> 8;
  t.f = s256 & 255;
  t.i1 = min(t.i0 + 1, side - 1);
  return t;
}

__device__ __forceinline__ void load_px(const uint8_t* __restrict__ frame, int H, int W, int gx,
                                        int gy, int& r, int& g, int& b) {
  if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
    const uint8_t* p = frame + ((size_t)gy * W + gx) * 3;
    r = p[0];
    g = p[1];
    b = p[2];
  } else {
    r = g = b = 0;
  }
}

constexpr int GATHER_ROWS = 8;  // output rows per CTA
constexpr int SEGS = S / 32;      // 19 warp tasks per row

__global__ void __launch_bounds__(256) gather_kernel(const uint8_t* __restrict__ frames,
                                                     int64_t frame_stride, int H, int W,
                                                     const tp_tile_job_t* __restrict__ jobs,
                                                     const int32_t* __restrict__ n_jobs_dev,
                                                     int mode, uint8_t* __restrict__ out_u8,
                                                     __nv_bfloat16* __restrict__ out_act,
                                                     int act_f16) {
  const int t = blockIdx.y;  // tile
  if (n_jobs_dev != nullptr && t >= *n_jobs_dev) return;
  const tp_tile_job_t job = jobs[t];
  const uint8_t* frame = frames + (int64_t)job.frame * frame_stride;
  const int side = job.side;

  // exact value/255 in the activation type, looked up instead of divided (bit-identical)
  __shared__ uint16_t lut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    if (act_f16) {
      __half h = __float2half_rn((float)i / 255.0f);
      lut[i] = *reinterpret_cast<uint16_t*>(&h);
    } else {
      __nv_bfloat16 h = __float2bfloat16_rn((float)i / 255.0f);
      lut[i] = *reinterpret_cast<uint16_t*>(&h);
    }
  }
  __syncthreads();
  auto pk2 = [&](int a, int b) -> uint32_t { return (uint32_t)lut[a] | ((uint32_t)lut[b] << 16); };

  const uint32_t lane = threadIdx.x & 31;
  for (int task = threadIdx.x >> 5; task < GATHER_ROWS * SEGS; task += blockDim.x >> 5) {
    const int row = task / SEGS;
    const int v = blockIdx.x * GATHER_ROWS + row;  // output row
    const int u = (task - row * SEGS) * 32 + (int)lane;
    int sy0, sy1 = 0, fy = 0;
    if (mode == TP_RESAMPLE_NEAREST) {
      sy0 = job.y + (v * side) / S;
    } else {
      const Tap ty = bilinear_tap(v, side);
      sy0 = job.y + ty.i0;
      sy1 = job.y + ty.i1;
      fy = ty.f;
    }
    // RGB of tile column uu on this output row (zero outside [0, 608) and the frame)
    auto sample = [&](int uu, int& r, int& g, int& b) {
      if (uu < 0 || uu >= S) {
        r = g = b = 0;
        return;
      }
      if (mode == TP_RESAMPLE_NEAREST) {
        load_px(frame, H, W, job.x + (uu * side) / S, sy0, r, g, b);
      } else {
        const Tap tx = bilinear_tap(uu, side);
        int r00, g00, b00, r01, g01, b01, r10, g10, b10, r11, g11, b11;
        load_px(frame, H, W, job.x + tx.i0, sy0, r00, g00, b00);
        load_px(frame, H, W, job.x + tx.i1, sy0, r01, g01, b01);
        load_px(frame, H, W, job.x + tx.i0, sy1, r10, g10, b10);
        load_px(frame, H, W, job.x + tx.i1, sy1, r11, g11, b11);
        const int w00 = (256 - tx.f) * (256 - fy), w01 = tx.f * (256 - fy);
        const int w10 = (256 - tx.f) * fy, w11 = tx.f * fy;
        r = (r00 * w00 + r01 * w01 + r10 * w10 + r11 * w11 + 32768) >> 16;
        g = (g00 * w00 + g01 * w01 + g10 * w10 + g11 * w11 + 32768) >> 16;
        b = (b00 * w00 + b01 * w01 + b10 * w10 + b11 * w11 + 32768) >> 16;
      }
    };
    int r, g, b;
    sample(u, r, g, b);
    if (out_u8 != nullptr) {
      uint8_t* o = out_u8 + (((size_t)t * S + v) * S + u) * 3;
      o[0] = (uint8_t)r;
      o[1] = (uint8_t)g;
      o[2] = (uint8_t)b;
    }
    if (out_act == nullptr) continue;
    const uint32_t me_rg = pk2(r, g), me_b0 = pk2(b, 0);
    uint32_t r_rg = __shfl_down_sync(0xffffffffu, me_rg, 1), r_b0 = __shfl_down_sync(0xffffffffu, me_b0, 1);
    if (lane == 31) {  // the right neighbour across the warp's edge is re-sampled
      int rr, gr, br;
      sample(u + 1, rr, gr, br);
      r_rg = pk2(rr, gr);
      r_b0 = pk2(br, 0);
    }
    // slot u+1 of padded row v+1: [q(u) rgb0 | q(u+1) rgb0]
    __nv_bfloat16* row_o = out_act + ((size_t)t * SP + (v + 1)) * SP * 8;
    *reinterpret_cast<uint4*>(row_o + (u + 1) * 8) = make_uint4(me_rg, me_b0, r_rg, r_b0);
    if (u == 0)  // slot 0: [q(-1) = 0 | q(0)]
      *reinterpret_cast<uint4*>(row_o) = make_uint4(0u, 0u, me_rg, me_b0);
  }
}

}  // namespace

extern "C" int tp_gather_tiles(const uint8_t* frames, int64_t frame_stride, int H, int W,
                               const tp_tile_job_t* jobs, int n_jobs, const int32_t* n_jobs_dev,
                               int mode, uint8_t* out_u8, void* out_act, int act_dtype,
                               void* stream) {
  if (frames == nullptr || jobs == nullptr || H < 1 || W < 1 || n_jobs < 0 ||
      (mode != TP_RESAMPLE_NEAREST && mode != TP_RESAMPLE_BILINEAR)) {
    tp_set_error("tp_gather_tiles: bad argument");
    return TP_ERR_ARG;
  }
  if (out_u8 == nullptr && out_act == nullptr) {
    tp_set_error("tp_gather_tiles: no output requested");
    return TP_ERR_ARG;
  }
  if (n_jobs == 0) return TP_OK;
  static_assert(S % 32 == 0 && S % GATHER_ROWS == 0, "tile side must split into warps/rows");
  dim3 grid(S / GATHER_ROWS, n_jobs);
  gather_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(frames, frame_stride, H, W, jobs,
                                                        n_jobs_dev, mode, out_u8,
                                                        (__nv_bfloat16*)out_act,
                                                        act_dtype == TP_DTYPE_F16);
  TP_LAUNCH_CHECK();
  return TP_OK;
}
