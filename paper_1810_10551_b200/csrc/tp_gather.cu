// K1/K2 — frame ingest + crop gather: crop square -> 608x608 tile.
//
// Replaces the reference tile cutter `cut_tile` (pkg/src/tilepipe/detector.py:223-247),
// which maps output pixel u to source floor(u*side/608) and zero-fills crop area that
// lies outside the frame. Mode NEAREST is bit-exact with it. Mode BILINEAR is the
// north-star downscale: 8-bit fixed-point weights, half-pixel centres, identical
// integer arithmetic to oracle/resample_ref.py so it is bit-exact as well.
//
// One CTA per (tile, 16 output rows); a warp task is 32 consecutive columns of one row
// (608 = 19 x 32, so a warp never straddles rows). Each lane produces one pixel: 3 bytes
// of the u8 tile and/or one 16-byte slot of the layer-0 input ([tile][610][610][8],
// fp16/bf16, zero 1-px halo): slot X of a row holds [q(X-1) rgb0 | q(X) rgb0] for tile
// pixels q (zero outside [0, 608)), so slots x and x+1 are layer 0's 32-byte A row
// [q(x-1) q(x) q(x) q(x+1)] — the conv's TMA map reads it through an overlapping view. Every store is one aligned 16-byte vector; a warp writes 512 B
// contiguous. Column source offsets / bilinear taps and the value/255 table are built
// once per CTA in shared memory; a pixel then costs a table read, its byte loads, LUT
// lookups, one shuffle pair and a 16-byte store.
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

constexpr int GATHER_ROWS = 16;  // output rows per CTA (amortises the column tables)
constexpr int SEGS = S / 32;       // 19 warp tasks per row
// Bilinear staging: a warp copies the byte span of both source rows that one chunk of 64
// output columns (+ the right neighbour) reads into shared memory with 16-byte coalesced
// loads, then samples the 2x2 taps from there (12 byte loads per pixel from global were
// LSU/latency bound: 35% of the HBM peak).
constexpr int BCHUNK = 64;
constexpr int BSTAGE = 1536;  // bytes per staged row span: side <= ~4600 px (8K attention crops); 6 CTAs per SM

template <int MODE>
__global__ void __launch_bounds__(256) gather_kernel(const uint8_t* __restrict__ frames,
                                                     int64_t frame_stride, int H, int W,
                                                     const tp_tile_job_t* __restrict__ jobs,
                                                     const int32_t* __restrict__ n_jobs_dev,
                                                     uint8_t* __restrict__ out_u8,
                                                     __nv_bfloat16* __restrict__ out_act,
                                                     int act_dtype) {
  const int t = blockIdx.y;  // tile
  if (n_jobs_dev != nullptr && t >= *n_jobs_dev) return;
  const tp_tile_job_t job = jobs[t];
  const uint8_t* frame = frames + (int64_t)job.frame * frame_stride;
  const int side = job.side;
  constexpr bool nearest = MODE == TP_RESAMPLE_NEAREST;

  // Per-CTA tables, shared by all GATHER_ROWS rows of this tile:
  //   lut: exact value/255 in the activation type (bit-identical to dividing); the
  //   integer value itself for TP_DTYPE_F16X2 (layer 0 then scales by 1/255 in fp32)
  //   cx0/cx1: byte offset 3*x of the column's source tap(s) in a frame row, -1 outside
  //   the frame (or outside the tile for u = 608); cf: bilinear weight of tap 1
  __shared__ uint16_t lut[256];
  // nearest: int cx0[S + 1]; bilinear: int4 {cx0, cx1, cf, 0}[S + 1] (one 16-byte read)
  __shared__ __align__(16) uint8_t tabmem[(S + 1) * (nearest ? 4 : 16)];
  int* cx0 = reinterpret_cast<int*>(tabmem);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    if (act_dtype == TP_DTYPE_F16X2) {  // fp32-parity plan: the integer value (exact)
      __half h = __float2half_rn((float)i);
      lut[i] = *reinterpret_cast<uint16_t*>(&h);
    } else if (act_dtype == TP_DTYPE_F16) {
      __half h = __float2half_rn((float)i / 255.0f);
      lut[i] = *reinterpret_cast<uint16_t*>(&h);
    } else {
      __nv_bfloat16 h = __float2bfloat16_rn((float)i / 255.0f);
      lut[i] = *reinterpret_cast<uint16_t*>(&h);
    }
  }
  for (int u = threadIdx.x; u <= S; u += blockDim.x) {
    int x0, x1 = -1, f = 0;
    if (nearest) {
      x0 = job.x + (u * side) / S;
    } else {
      const Tap tx = bilinear_tap(u, side);
      x0 = job.x + tx.i0;
      x1 = job.x + tx.i1;
      f = tx.f;
    }
    const bool in_tile = u < S;
    const int o0 = in_tile && x0 >= 0 && x0 < W ? 3 * x0 : -1;
    if (nearest)
      cx0[u] = o0;
    else
      reinterpret_cast<int4*>(tabmem)[u] = make_int4(o0, in_tile && x1 >= 0 && x1 < W ? 3 * x1 : -1, f, 0);
  }
  __syncthreads();
  auto pk2 = [&](int a, int b) -> uint32_t { return (uint32_t)lut[a] | ((uint32_t)lut[b] << 16); };

  const size_t row_bytes = (size_t)W * 3;
  // slot u+1 of padded row v+1 = [q(u) rgb0 | q(u+1) rgb0] (+ slot 0 = [0 | q(0)])
  auto emit = [&](int v, int u, uint32_t me_rg, uint32_t me_b0, uint32_t r_rg, uint32_t r_b0) {
    __nv_bfloat16* row_o = out_act + ((size_t)t * SP + (v + 1)) * SP * 8;
    *reinterpret_cast<uint4*>(row_o + (u + 1) * 8) = make_uint4(me_rg, me_b0, r_rg, r_b0);
    if (u == 0) *reinterpret_cast<uint4*>(row_o) = make_uint4(0u, 0u, me_rg, me_b0);
  };

  if constexpr (!nearest) {
  if (3 * (BCHUNK * side / S + 3) + 32 <= BSTAGE - 16 && row_bytes % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(frame) & 15) == 0) {
    // The last 16 bytes of each staging row stay zero: out-of-frame taps point there, so
    // the tap loads need no predicates.
    __shared__ __align__(16) uint8_t stg[8][2][BSTAGE];
    constexpr int ZOFF = BSTAGE - 16;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* st0 = stg[warp][0];
    uint8_t* st1 = stg[warp][1];
    if (lane < 2) reinterpret_cast<uint4*>(stg[warp][lane] + ZOFF)[0] = make_uint4(0u, 0u, 0u, 0u);
    const bool exact_int = act_dtype == TP_DTYPE_F16X2;
    // q(u) packed as two 32-bit words (rg, b0) in the activation type. The parity plan
    // stores the integer value itself: fp16(1024 + n) has bits 0x6400 + n, so one packed
    // half2 subtraction of 1024 turns two bytes into two exact fp16 integers.
    auto pack = [&](int r, int g, int b, uint32_t& rg, uint32_t& b0) {
      if (exact_int) {
        const __half2 k1024 = __halves2half2(__ushort_as_half(0x6400), __ushort_as_half(0x6400));
        __half2 hrg = __hsub2(__halves2half2(__ushort_as_half((unsigned short)(0x6400 | r)),
                                             __ushort_as_half((unsigned short)(0x6400 | g))), k1024);
        __half2 hb = __hsub2(__halves2half2(__ushort_as_half((unsigned short)(0x6400 | b)),
                                            __ushort_as_half(0x6400)), k1024);
        rg = *reinterpret_cast<uint32_t*>(&hrg);
        b0 = *reinterpret_cast<uint32_t*>(&hb);
      } else {
        rg = pk2(r, g);
        b0 = pk2(b, 0);
      }
    };
    for (int rr = (int)warp; rr < GATHER_ROWS; rr += 8) {
      const int v = blockIdx.x * GATHER_ROWS + rr;
      const Tap ty = bilinear_tap(v, side);
      const int s0 = job.y + ty.i0, s1 = job.y + ty.i1, fy = ty.f, fy0 = 256 - fy;
      const uint8_t* r0 = s0 >= 0 && s0 < H ? frame + (size_t)s0 * row_bytes : nullptr;
      const uint8_t* r1 = s1 >= 0 && s1 < H ? frame + (size_t)s1 * row_bytes : nullptr;
      __nv_bfloat16* row_o = out_act != nullptr ? out_act + ((size_t)t * SP + (v + 1)) * SP * 8 : nullptr;
      // slot u of the padded row = [q(u-1) | q(u)] is written by the lane owning q(u);
      // q(u-1) comes from the lane to the left, or from the previous 32 columns (carried)
      uint32_t prev_rg = 0u, prev_b0 = 0u;
      for (int c0 = 0; c0 < S; c0 += BCHUNK) {
        // source columns of outputs c0 .. c0 + BCHUNK - 1
        const int xa = max(job.x + bilinear_tap(c0, side).i0, 0);
        const int xb = min(job.x + bilinear_tap(min(c0 + BCHUNK - 1, S - 1), side).i1, W - 1);
        const int base = (3 * xa) & ~15;
        const int nvec = xb >= xa ? (3 * xb + 3 - base + 15) >> 4 : 0;
        __syncwarp();  // the previous chunk's smem reads are done
        for (int k = (int)lane; k < nvec; k += 32) {
          const uint4 z = make_uint4(0u, 0u, 0u, 0u);
          reinterpret_cast<uint4*>(st0)[k] =
              r0 ? __ldg(reinterpret_cast<const uint4*>(r0 + base) + k) : z;
          reinterpret_cast<uint4*>(st1)[k] =
              r1 ? __ldg(reinterpret_cast<const uint4*>(r1 + base) + k) : z;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < BCHUNK / 32; ++j) {
          const int u = c0 + j * 32 + (int)lane;  // S % 32 == 0: uniform per warp
          if (c0 + j * 32 >= S) break;
          const int4 tb = reinterpret_cast<const int4*>(tabmem)[u];  // o0, o1, fx
          const int i0 = tb.x >= 0 ? tb.x - base : ZOFF, i1 = tb.y >= 0 ? tb.y - base : ZOFF;
          const int fx = tb.z, fx0 = 256 - fx;
          int ch[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {  // separable form of the 2x2 weights: exact
            const int h0 = st0[i0 + k] * fx0 + st0[i1 + k] * fx;
            const int h1 = st1[i0 + k] * fx0 + st1[i1 + k] * fx;
            ch[k] = (h0 * fy0 + h1 * fy + 32768) >> 16;
          }
          if (out_u8 != nullptr) {
            uint8_t* o = out_u8 + (((size_t)t * S + v) * S + u) * 3;
            o[0] = (uint8_t)ch[0];
            o[1] = (uint8_t)ch[1];
            o[2] = (uint8_t)ch[2];
          }
          if (row_o == nullptr) continue;
          uint32_t me_rg, me_b0;
          pack(ch[0], ch[1], ch[2], me_rg, me_b0);
          uint32_t l_rg = __shfl_up_sync(0xffffffffu, me_rg, 1);
          uint32_t l_b0 = __shfl_up_sync(0xffffffffu, me_b0, 1);
          if (lane == 0) {
            l_rg = prev_rg;
            l_b0 = prev_b0;
          }
          prev_rg = __shfl_sync(0xffffffffu, me_rg, 31);
          prev_b0 = __shfl_sync(0xffffffffu, me_b0, 31);
          *reinterpret_cast<uint4*>(row_o + u * 8) = make_uint4(l_rg, l_b0, me_rg, me_b0);
          if (u == S - 1) *reinterpret_cast<uint4*>(row_o + S * 8) = make_uint4(me_rg, me_b0, 0u, 0u);
        }
      }
    }
    return;
  }
  }  // staged bilinear

  const uint32_t lane = threadIdx.x & 31;
  // 4 tasks in flight per warp: their frame loads overlap (long-scoreboard bound otherwise)
#pragma unroll 4
  for (int task = threadIdx.x >> 5; task < GATHER_ROWS * SEGS; task += blockDim.x >> 5) {
    const int row = task / SEGS;
    const int v = blockIdx.x * GATHER_ROWS + row;  // output row
    const int u = (task - row * SEGS) * 32 + (int)lane;
    // source row(s) of this output row; nullptr = outside the frame (reads as 0)
    const uint8_t *r0, *r1 = nullptr;
    int fy = 0;
    if (nearest) {
      const int sy = job.y + (v * side) / S;
      r0 = sy >= 0 && sy < H ? frame + (size_t)sy * row_bytes : nullptr;
    } else {
      const Tap ty = bilinear_tap(v, side);
      const int s0 = job.y + ty.i0, s1 = job.y + ty.i1;
      r0 = s0 >= 0 && s0 < H ? frame + (size_t)s0 * row_bytes : nullptr;
      r1 = s1 >= 0 && s1 < H ? frame + (size_t)s1 * row_bytes : nullptr;
      fy = ty.f;
    }
    // RGB of tile column uu on this output row (zero outside the tile and the frame)
    auto sample = [&](int uu, int& r, int& g, int& b) {
      const int o0 = nearest ? cx0[uu] : reinterpret_cast<const int4*>(tabmem)[uu].x;
      if (nearest) {
        if (o0 < 0 || r0 == nullptr) {
          r = g = b = 0;
        } else {
          r = __ldg(r0 + o0);
          g = __ldg(r0 + o0 + 1);
          b = __ldg(r0 + o0 + 2);
        }
        return;
      }
      const int4 tb = reinterpret_cast<const int4*>(tabmem)[uu];
      const int o1 = tb.y, fx = tb.z;
      auto px = [&](const uint8_t* rp, int o, int k) -> int {
        return (rp != nullptr && o >= 0) ? (int)__ldg(rp + o + k) : 0;
      };
      const int w00 = (256 - fx) * (256 - fy), w01 = fx * (256 - fy);
      const int w10 = (256 - fx) * fy, w11 = fx * fy;
      int ch[3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        ch[k] = (px(r0, o0, k) * w00 + px(r0, o1, k) * w01 + px(r1, o0, k) * w10 +
                 px(r1, o1, k) * w11 + 32768) >> 16;
      r = ch[0];
      g = ch[1];
      b = ch[2];
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
    emit(v, u, me_rg, me_b0, r_rg, r_b0);
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
  if (mode == TP_RESAMPLE_NEAREST)
    gather_kernel<TP_RESAMPLE_NEAREST><<<grid, 256, 0, (cudaStream_t)stream>>>(
        frames, frame_stride, H, W, jobs, n_jobs_dev, out_u8, (__nv_bfloat16*)out_act, act_dtype);
  else
    gather_kernel<TP_RESAMPLE_BILINEAR><<<grid, 256, 0, (cudaStream_t)stream>>>(
        frames, frame_stride, H, W, jobs, n_jobs_dev, out_u8, (__nv_bfloat16*)out_act, act_dtype);
  TP_LAUNCH_CHECK();
  return TP_OK;
}
