// Synthetic frame renderer (input generator): flat background with
// class-coloured filled rectangles drawn in painter's order — the same bytes as the
// reference's render_frame (pkg/src/tilepipe/synthetic.py:183-196), produced directly
// in HBM so 4K/8K benchmark clips never cross PCIe.
//
// One thread per 16-byte output chunk (16 bytes = 5 1/3 pixels); each thread tests its
// pixels against the frame's rectangle list (<= 64, staged in shared memory) from last
// to first, so the topmost rectangle wins.
#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

namespace {

constexpr int MAX_OBJ = 64;

__global__ void __launch_bounds__(256) render_kernel(const int32_t* __restrict__ rects,
                                                     const uint8_t* __restrict__ colors,
                                                     const int32_t* __restrict__ counts,
                                                     int max_obj, int H, int W, uint32_t bg,
                                                     uint8_t* __restrict__ out) {
  __shared__ int4 r_s[MAX_OBJ];
  __shared__ uint32_t c_s[MAX_OBJ];
  const int f = blockIdx.y;
  const int n = min(counts[f], MAX_OBJ);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int32_t* r = rects + ((long long)f * max_obj + i) * 4;
    r_s[i] = make_int4(r[0], r[1], r[2], r[3]);
    const uint8_t* c = colors + ((long long)f * max_obj + i) * 3;
    c_s[i] = (uint32_t)c[0] | ((uint32_t)c[1] << 8) | ((uint32_t)c[2] << 16);
  }
  __syncthreads();
  const long long frame_bytes = (long long)H * W * 3;
  uint8_t* img = out + (long long)f * frame_bytes;
  const long long n_chunks = (frame_bytes + 15) / 16;
  for (long long ch = blockIdx.x * (long long)blockDim.x + threadIdx.x; ch < n_chunks;
       ch += (long long)gridDim.x * blockDim.x) {
    uint8_t buf[16];
    const long long b0 = ch * 16;
    long long cached_px = -1;
    uint32_t col = bg;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const long long b = b0 + k;
      const long long px = b / 3;
      if (px != cached_px && b < frame_bytes) {
        cached_px = px;
        const int y = (int)(px / W), x = (int)(px - (long long)y * W);
        col = bg;
        for (int i = n - 1; i >= 0; --i) {
          const int4 r = r_s[i];
          if (x >= r.x && x < r.z && y >= r.y && y < r.w) {
            col = c_s[i];
            break;
          }
        }
      }
      buf[k] = (uint8_t)(col >> (8 * (int)(b - px * 3)));
    }
    if (b0 + 16 <= frame_bytes) {
      *reinterpret_cast<uint4*>(img + b0) = *reinterpret_cast<uint4*>(buf);
    } else {
      for (int k = 0; b0 + k < frame_bytes; ++k) img[b0 + k] = buf[k];
    }
  }
}

}  // namespace

extern "C" int tp_render_frames(const int32_t* rects, const uint8_t* colors, const int32_t* counts,
                                int n_frames, int max_obj, int H, int W, uint32_t bg_rgb,
                                uint8_t* out, void* stream) {
  if (rects == nullptr || colors == nullptr || counts == nullptr || out == nullptr || H < 1 ||
      W < 1 || max_obj < 1 || max_obj > MAX_OBJ || ((long long)H * W * 3) % 16 != 0) {
    tp_set_error("tp_render_frames: bad argument (max_obj <= %d, H*W*3 %% 16 == 0)", MAX_OBJ);
    return TP_ERR_ARG;
  }
  if (n_frames <= 0) return TP_OK;
  dim3 grid(148 * 4, n_frames);
  render_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(rects, colors, counts, max_obj, H, W,
                                                        bg_rgb, out);
  TP_LAUNCH_CHECK();
  return TP_OK;
}
