// fp32-parity mode support: activations carried as exact fp16 pairs (hi, lo).
//
// The north-star score bar (1e-3 relative vs the fp32 CPU reference) is below what 16-bit
// activation storage can guarantee through 23 layers (rounding flips caused by a different
// fp32 accumulation order compound). In this mode every activation x is stored as
// hi = fp16(x), lo = fp16(x - hi) in a doubled channel dimension ([hi C | lo C]) and the
// conv weights are duplicated over both halves, so the same tcgen05 kernels compute
// sum (hi + lo) * w with ~22 significant bits per activation and fp32 accumulation.
// Convs write fp32 (the head epilogue); tp_split_store applies the fused 2x2 max pool /
// space-to-depth reorg and writes the next layer's hi/lo input. Weights are exact fp16.
#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

namespace {

__global__ void split_store_kernel(const float* __restrict__ src, int n, int res,
                                   int src_cstride, int C, int pool, int reorg,
                                   __half* __restrict__ dst, int dst_cstride, int coff,
                                   int lo_off) {
  // output geometry: pool / reorg halve the side; reorg multiplies channels by 4
  const int ores = (pool || reorg) ? res >> 1 : res;
  const int oc = reorg ? 4 * C : C;
  const long long total = (long long)n * ores * ores * oc;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % oc);
    long long r = i / oc;
    const int x = (int)(r % ores);
    r /= ores;
    const int y = (int)(r % ores);
    const int img = (int)(r / ores);
    float v;
    if (pool) {
      const float* s = src + (((long long)img * res + 2 * y) * res + 2 * x) * src_cstride + c;
      v = fmaxf(fmaxf(s[0], s[src_cstride]),
                fmaxf(s[(long long)res * src_cstride], s[(long long)res * src_cstride + src_cstride]));
    } else if (reorg) {  // out channel (dy*2+dx)*C + c' <- pixel (2y+dy, 2x+dx) channel c'
      const int sub = c / C, cc = c - sub * C;
      const int sy = 2 * y + (sub >> 1), sx = 2 * x + (sub & 1);
      v = src[(((long long)img * res + sy) * res + sx) * src_cstride + cc];
    } else {
      v = src[(((long long)img * res + y) * res + x) * src_cstride + c];
    }
    const __half hi = __float2half_rn(v);
    const __half lo = __float2half_rn(__fsub_rn(v, __half2float(hi)));
    __half* d = dst + (((long long)img * ores + y) * ores + x) * dst_cstride + coff + c;
    d[0] = hi;
    d[lo_off] = lo;
  }
}

// u8 tiles [n][608][608][3] -> [n][608][608][32] fp16: channels 0..2 = hi(v/255),
// 16..18 = lo(v/255), others 0 (layer 0's input: logical 16 channels, split to 32)
__global__ void split_input_kernel(const uint8_t* __restrict__ tiles, int n,
                                   __half* __restrict__ dst) {
  const long long total = (long long)n * TP_MODEL_SIDE * TP_MODEL_SIDE;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < total;
       p += (long long)gridDim.x * blockDim.x) {
    __half h[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) h[k] = __float2half_rn(0.f);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float v = __fdiv_rn((float)tiles[p * 3 + k], 255.0f);
      h[k] = __float2half_rn(v);
      h[16 + k] = __float2half_rn(__fsub_rn(v, __half2float(h[k])));
    }
    uint4* d = reinterpret_cast<uint4*>(dst + p * 32);
    const uint4* s = reinterpret_cast<const uint4*>(h);
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = s[k];
  }
}

int grid_for(long long total) {
  long long b = (total + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return (int)(b > 0 ? b : 1);
}

}  // namespace

extern "C" int tp_split_store(const float* src, int n, int res, int src_cstride, int C, int pool,
                              int reorg, void* dst, int dst_cstride, int coff, int lo_off,
                              void* stream) {
  if (src == nullptr || dst == nullptr || n < 0 || res < 1 || C < 1 || (pool && reorg) ||
      ((pool || reorg) && (res & 1)) || coff < 0 || lo_off < 1) {
    tp_set_error("tp_split_store: bad argument");
    return TP_ERR_ARG;
  }
  if (n == 0) return TP_OK;
  const int ores = (pool || reorg) ? res >> 1 : res;
  const long long total = (long long)n * ores * ores * (reorg ? 4 * C : C);
  split_store_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(
      src, n, res, src_cstride, C, pool, reorg, (__half*)dst, dst_cstride, coff, lo_off);
  TP_LAUNCH_CHECK();
  return TP_OK;
}

extern "C" int tp_split_input(const uint8_t* tiles, int n, void* dst, void* stream) {
  if (tiles == nullptr || dst == nullptr || n < 0) {
    tp_set_error("tp_split_input: bad argument");
    return TP_ERR_ARG;
  }
  if (n == 0) return TP_OK;
  split_input_kernel<<<grid_for((long long)n * TP_MODEL_SIDE * TP_MODEL_SIDE), 256, 0,
                       (cudaStream_t)stream>>>(tiles, n, (__half*)dst);
  TP_LAUNCH_CHECK();
  return TP_OK;
}
