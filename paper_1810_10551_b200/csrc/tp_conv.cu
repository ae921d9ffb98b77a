// K3/K4 — YOLO v2-608 conv stack as tcgen05/TMEM implicit-GEMM kernels.
//
// No reference kernel exists (the reference detector is an abstract boundary,
// pkg/src/tilepipe/detector.py:77-96); the topology is yolov2-608 (Darknet-19 +
// passthrough head) as cited by PAPER.md:85,120, restated in oracle/yolo_ref.py.
//
// Activation layout: compact NHWC [tile][R][R][C] (fp16 or bf16). A 3x3/1 same conv is a
// GEMM over output pixels, K = taps x C; the zero padding is TMA out-of-bounds fill, so
// no halo is stored and no M row is wasted on one:
//   * FLAT tiles (conv_tc_kernel / conv_pair_kernel, non-pooled layers): M tile = 128
//     consecutive compact pixels (256 for a CTA pair), A loaded per (tap, 64-channel
//     block) with TMA im2col (window corner -1, tap = im2col offset).
//   * RECT tiles (conv_tc_kernel, pooled 3x3 layers without a box variant): a 16x8 pixel
//     rectangle loaded as a 4-D box {C, 16, 8, 1}; the epilogue pools in registers.
//   * box tiles (conv_box_kernel: 3x3 with cin 32/64 and resident weights): one box
//     {C, 10, 18} per 8x16 tile, the nine taps are descriptor row offsets into it.
//   * layer 0 (conv_l0_kernel): reads the gather's padded 8-byte rgb0 pixels as
//     overlapping 64-byte rows of 8 pixels starting at every even column; even columns
//     take one MMA per kernel row, odd columns two (see the kernel comment).
//
// Kernels are persistent and warp-specialised, one CTA per SM (320 threads): warps 0-7
// epilogue (two warpgroups on alternate accumulators, one TMEM lane quadrant per warp:
// tcgen05.ld -> +bias (BN folded) -> leaky(0.1) -> [2x2 max] -> 16-bit -> TMA store or
// direct store / reorg / fp32 head), warp 8 TMA producer, warp 9 TMEM allocator + MMA
// issuer (warp-convergent loop, one elected lane issues tcgen05.mma).
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <unordered_map>

#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

namespace {

enum ConvMode { MODE_SW128 = 0, MODE_SW64 = 1 };
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
// Warp roles: the warp scheduler favours HIGHER warp ids, so the two single-thread roles
// (TMA producer, MMA issuer) take the top ids and are never starved by epilogue warps.
constexpr uint32_t kProdWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
constexpr int RECT_W = 16, RECT_H = 8;

struct ConvParams {
  int n_img;
  const int32_t* n_img_dev;
  int res, img_px;  // activations are compact NHWC: img_px = res * res
  int ksize;
  int cin;         // channels per tap used by K (multiple of BK)
  int cout;        // real output channels
  int bn;          // N tile
  int n_blocks_n;
  int num_kb;      // k-blocks per output tile
  int kb_per_tap;
  int stages;
  uint32_t a_stage_bytes, b_stage_bytes;
  uint32_t tmem_cols;
  uint32_t idesc;  // operand format (bf16 or fp16) + shape
  int f16;         // activations stored as fp16 (else bf16)
  int rect;        // RECT tiles + fused 2x2 maxpool
  int tiles_x, tiles_y;
  const float* bias;
  void* out;
  int out_cstride, out_coff, out_fp32, leaky, reorg;
  int sub;         // RECT super-tile: SUB stacked 16x8 sub-tiles (halo variant)
  int halo;        // RECT + weights resident in smem + one {BK,16,10} halo box per (dx, cb)
  uint32_t bres_bytes, bchunk_bytes;
  int n_bchunks;
  uint32_t stage_bytes;  // epilogue store staging (TMA-store variants): 8 warps x 2 KB
  int nbuf;  // box kernel: TMEM accumulator buffers (2 or 4)
  // fp32-parity plan (TP_DTYPE_F16X2): outputs leave as exact fp16 pairs hi = fp16(v),
  // lo = fp16(v - hi), interleaved per 16 channels ([hi 16 | lo 16], stored channel of real
  // channel c = 32 (c / 16) + c % 16, its lo part +16); out_coff is in stored channels.
  int split;
  float alpha;  // accumulator scale: 1/255 for layer 0's integer pixels, 2^-c for HL8 inputs
  // HL8 activations (TP_DTYPE_F16F8, the fp32-parity plan): a hi plane fp16(x) [pix][C]
  // plus a lo plane e4m3((x - hi) * 2^TP_LO_EXP) [pix][C] bytes. Input side: each tap's K
  // runs kb_hi hi blocks (64 channels, kind::f16 against fp16 weights w * 2^c) then the
  // lo blocks (128 channels, kind::f8f6f4 against e4m3 weights w * 2^(c - TP_LO_EXP)) into
  // the same fp32 accumulator; both stage kinds are 128 rows x 128 bytes. Output side:
  // out_lo (!= nullptr) receives the lo plane at the hi plane's [pixel][channel] index.
  int lo_in;
  int kb_hi;
  void* out_lo;
  // conv_swap_kernel<false> with a fused 1x1 consumer (fuse != 0; the F16F8 plan's layer
  // 4 -> layer 5, whose input buffer nothing else reads): the 1x1's fp16 / e4m3 weights
  // [64][128], bias, accumulator scale and HL8 output planes (f5_cstride channels per pixel)
  int fuse;
  const void* f5_w;
  const void* f5_wlo;
  const float* f5_bias;
  float f5_alpha;
  int f5_leaky;
  void* f5_out;
  void* f5_out_lo;
  int f5_cstride;
  // profiling only (TP_CONV_DEBUG bits): 1 skip epilogue, 2 skip MMAs, 4 skip stores,
  // 8 skip TMEM loads, 16 no TMA (stale operands), 32 role cycle counters (g_conv_prof),
  // 64 unmerged pool-in-M MMAs (box kernel A/B)
  int dbg;
};


__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(tp::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(tp::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 4-D tiled box {C, W, H, N}; out-of-bounds elements (the conv's zero padding) read as 0
__device__ __forceinline__ void tma_load_4d(void* smem_dst, const void* tmap, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(tp::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(tp::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3)
      : "memory");
}
// im2col box: consecutive output pixels (W, then H, then N inside the map's bounding box),
// each contributing the input pixel at window corner + (ow, oh); coordinates are the
// first pixel's window corner. Out-of-bounds pixels read as 0 (tools/im2col_probe.cu).
__device__ __forceinline__ void tma_load_im2col(void* smem_dst, const void* tmap, uint64_t* bar,
                                                int32_t c, int32_t w, int32_t h, int32_t n,
                                                uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(tp::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(tp::smem_u32(bar)), "r"(c), "r"(w), "r"(h),
      "r"(n), "h"(ow), "h"(oh)
      : "memory");
}
// first compact pixel of an M tile -> (image, y, x)
struct PixPos {
  int n, y, x;
};
__device__ __forceinline__ PixPos pix_pos(int pix, int res, int img_px) {
  PixPos r;
  r.n = pix / img_px;
  const int rem = pix - r.n * img_px;
  r.y = rem / res;
  r.x = rem - r.y * res;
  return r;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* smem_src, int32_t c0,
                                             int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(tp::smem_u32(smem_src)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const void* tmap, const void* smem_src, int32_t c0,
                                             int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(tp::smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {  // <= 1 bulk group still reading smem
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// Profiling counters (TP_CONV_DEBUG bit 32): per-role cycle totals summed over CTAs.
//   0 producer total, 1 producer empty-wait, 2 mma total, 3 mma tempty-wait, 4 mma full-wait,
//   5 epilogue total (warp 0), 6 epilogue tfull-wait (warp 0), 7 launches
__device__ unsigned long long g_conv_prof[8];
#define PROF_T0(v) long long v = (p.dbg & 32) ? clock64() : 0
#define PROF_ADD(acc, t0) \
  if (p.dbg & 32) acc += clock64() - (t0)

// Epilogue variants, chosen at compile time (EPI_SPLIT: TMA-stored hi/lo fp16 pairs).
// EPI_HL8: TMA-stored fp16 hi plane (as EPI_PLAIN) + directly stored e4m3 lo plane.
enum Epi { EPI_PLAIN = 0, EPI_POOL = 1, EPI_REORG = 2, EPI_F32 = 3, EPI_SPLIT = 4, EPI_HL8 = 5 };

// 2*NP fp32 values -> NP packed fp16 pairs hi = fp16(v) and NP packed lo = fp16(v - hi)
template <int NP>
__device__ __forceinline__ void split_pairs(const float* f, uint32_t* hi, uint32_t* lo) {
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    __half2 h = __floats2half2_rn(f[2 * j], f[2 * j + 1]);
    const float2 hf = __half22float2(h);
    __half2 l = __floats2half2_rn(f[2 * j] - hf.x, f[2 * j + 1] - hf.y);
    hi[j] = *reinterpret_cast<uint32_t*>(&h);
    lo[j] = *reinterpret_cast<uint32_t*>(&l);
  }
}
// 16 split values to a stored [hi 16 | lo 16] group at o (16-bit elements)
__device__ __forceinline__ void store_split16(__nv_bfloat16* o, const float* f) {
  uint32_t hi[8], lo[8];
  split_pairs<8>(f, hi, lo);
  *reinterpret_cast<uint4*>(o) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4*>(o + 8) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
  *reinterpret_cast<uint4*>(o + 16) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  *reinterpret_cast<uint4*>(o + 24) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
}
// HL8 lo plane: 16 fp32 values -> hi (8 packed fp16 pairs, as __floats2half2_rn) and the
// residuals (v - hi) * 2^TP_LO_EXP as 16 e4m3 bytes (4 words, byte j = channel j; RN,
// saturating at +-448 — only for |v| beyond ~448, where the hi part alone carries 2^-12)
constexpr float kLoScale = 2048.0f;  // 2^TP_LO_EXP
static_assert(TP_LO_EXP == 11, "kLoScale");
__device__ __forceinline__ uint32_t e4m3x4(float a, float b, float c, float d) {
  uint16_t lo, hi;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(b), "f"(a));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(d), "f"(c));
  return (uint32_t)lo | ((uint32_t)hi << 16);
}
__device__ __forceinline__ void split_hl8(const float* f, uint32_t* hi, uint32_t* lo) {
  float r[16];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    __half2 h = __floats2half2_rn(f[2 * j], f[2 * j + 1]);
    const float2 hf = __half22float2(h);
    r[2 * j] = (f[2 * j] - hf.x) * kLoScale;
    r[2 * j + 1] = (f[2 * j + 1] - hf.y) * kLoScale;
    hi[j] = *reinterpret_cast<uint32_t*>(&h);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) lo[j] = e4m3x4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
}
// 16 HL8 values to the hi plane (fp16, 32 B at oh) and the lo plane (16 B at ol)
__device__ __forceinline__ void store_hl8(__half* oh, uint8_t* ol, const float* f) {
  uint32_t hi[8], lo[4];
  split_hl8(f, hi, lo);
  *reinterpret_cast<uint4*>(oh) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4*>(oh + 8) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
  *reinterpret_cast<uint4*>(ol) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}
// one scalar HL8 value (hi fp16 + lo e4m3 byte)
__device__ __forceinline__ void store_hl8_1(__half* oh, uint8_t* ol, float v) {
  const __half h = __float2half_rn(v);
  uint16_t pr;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(pr) : "f"(0.0f), "f"((v - __half2float(h)) * kLoScale));
  *oh = h;
  *ol = (uint8_t)(pr & 0xFF);
}
// tcgen05 MMA with e4m3 A/B (kind::f8f6f4, K = 32 per instruction: 32 bytes per row, the
// same operand bytes per instruction as kind::f16's K = 16), fp32 accumulate
__device__ __forceinline__ void mma_f8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Darknet's reorg (yolov2-608 [reorg] stride=2: forward_reorg_layer -> reorg_cpu(...,
// forward = 0), darknet src/blas.c): it reads the C x R x R input as C/4 x 2R x 2R memory and
// writes a 4C x R/2 x R/2 output, which is not a clean space-to-depth. Input element
// (c, y, x) lands at output (C, Y, X): with a = c % 4, h2 = (R/2) a + y/2, w2 = R (y % 2) + x,
// k = (2 (h2 % 2) + w2 % 2) (C/4) + c / 4 and P = w2/2 + R (h2/2) + R^2 k (NCHW flat),
// C = P / (R/2)^2, Y, X = the rest (oracle/yolo_ref.py reorg is the same map).
__device__ __forceinline__ void reorg_dest(int c, int y, int x, int R, int cin, int& Y, int& X,
                                           int& C) {
  const int hr = R >> 1;
  const int h2 = hr * (c & 3) + (y >> 1), w2 = R * (y & 1) + x;
  const int k = (2 * (h2 & 1) + (w2 & 1)) * (cin >> 2) + (c >> 2);
  const int P = (w2 >> 1) + R * (h2 >> 1) + R * R * k;
  C = P / (hr * hr);
  const int r = P - C * hr * hr;
  Y = r / hr;
  X = r - Y * hr;
}
constexpr int kMaxBias = 1024;

// Walks a CTA's contiguous tile range: t = mt * n_blocks_n + nb, and for RECT tiles
// mt = (img * tiles_y + by) * tiles_x + bx. Divisions only at the start.
struct TileIter {
  int nb, mt, img, by, bx;
  __device__ __forceinline__ void init(int t, const ConvParams& p) {
    mt = t / p.n_blocks_n;
    nb = t - mt * p.n_blocks_n;
    const int per = p.tiles_x * p.tiles_y;
    img = mt / per;
    const int r = mt - img * per;
    by = r / p.tiles_x;
    bx = r - by * p.tiles_x;
  }
  __device__ __forceinline__ void next(const ConvParams& p) {
    if (++nb == p.n_blocks_n) {
      nb = 0;
      ++mt;
      if (++bx == p.tiles_x) {
        bx = 0;
        if (++by == p.tiles_y) {
          by = 0;
          ++img;
        }
      }
    }
  }
};

template <int MODE, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmA2,
                   const __grid_constant__ CUtensorMap tmB2, const ConvParams p) {
  constexpr int BK = MODE == MODE_SW128 ? 64 : 32;
  constexpr bool RECT = EPI == EPI_POOL;
  // FLAT plain / fp32 / split outputs leave through per-warp swizzled smem slabs + TMA stores
  constexpr bool TSTORE = EPI == EPI_PLAIN || EPI == EPI_F32 || EPI == EPI_SPLIT || EPI == EPI_HL8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* smA = smem;
  uint8_t* smB = smem + (size_t)S * p.a_stage_bytes;  // B stages, or resident B (halo)
  uint8_t* smC = smB + (size_t)S * p.b_stage_bytes + p.bres_bytes;  // 1024-aligned
  uint64_t* bars = reinterpret_cast<uint64_t*>(smC + p.stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + 2;
  uint64_t* bres_bar = bars + 2 * S + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 5);
  float* bias_s = reinterpret_cast<float*>(bars + 2 * S + 6);

  const uint32_t warp = tp::warp_id();
  const uint32_t lane = tp::lane_id();
  const int cout_pad = p.bn * p.n_blocks_n;

  if (warp == kProdWarp && lane == 0) {
    tp::tma_prefetch(&tmA);
    tp::tma_prefetch(&tmB);
    for (int s = 0; s < S; ++s) {
      tp::mbar_init(&full[s], 1);
      tp::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tp::mbar_init(&tfull[a], 1);
      tp::mbar_init(&tempty[a], 4);
    }
    tp::mbar_init(bres_bar, 1);
    tp::fence_mbar_init();
  }
  if (warp == kMmaWarp) tp::tmem_alloc(tmem_slot, p.tmem_cols);
  for (int i = threadIdx.x; i < cout_pad; i += blockDim.x) bias_s[i] = p.bias[i];
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_img = p.n_img_dev != nullptr ? min(*p.n_img_dev, p.n_img) : p.n_img;
  const int m_blocks = RECT ? n_img * p.tiles_x * p.tiles_y : (n_img * p.img_px + 127) / 128;
  const int total_tiles = m_blocks * p.n_blocks_n;
  // contiguous, balanced tile range per CTA
  const int per_cta = total_tiles / (int)gridDim.x, extra = total_tiles % (int)gridDim.x;
  const int t_begin = (int)blockIdx.x * per_cta + min((int)blockIdx.x, extra);
  const int n_tiles = per_cta + ((int)blockIdx.x < extra ? 1 : 0);

  if (warp == kProdWarp) {
    if (lane == 0) {
      // ================= TMA producer =================
      int s = 0;
      uint32_t ph = 0;
      long long pr_wait = 0;
      PROF_T0(pr_start);
      const uint32_t tx_bytes = p.a_stage_bytes + p.b_stage_bytes;
      TileIter it;
      it.init(t_begin, p);
      if (RECT && p.halo && n_tiles > 0) {  // weights resident for the whole kernel
        tp::mbar_arrive_expect_tx(bres_bar, p.bres_bytes);
        for (int j = 0; j < p.n_bchunks; ++j)
          tp::tma_load_2d(smB + (size_t)j * p.bchunk_bytes, &tmB, bres_bar, j * BK, 0);
      }
      const int lo = p.ksize == 3 ? -1 : 0;  // im2col window corner (zero padding 1 or 0)
      for (int i = 0; i < n_tiles; ++i, it.next(p)) {
        const int n0 = it.nb * p.bn;
        // RECT: tile origin inside image it.img; FLAT: first compact pixel of the tile
        const int rx = it.bx * RECT_W, ry = it.by * RECT_H * p.sub;
        const PixPos f0 = RECT ? PixPos{0, 0, 0} : pix_pos(it.mt * 128, p.res, p.img_px);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          PROF_T0(tw);
          tp::mbar_wait(&empty[s], ph ^ 1);
          PROF_ADD(pr_wait, tw);
          uint8_t* a_dst = smA + (size_t)s * p.a_stage_bytes;
          uint8_t* b_dst = smB + (size_t)s * p.b_stage_bytes;
          if (p.dbg & 16) {  // profiling: no TMA, stale operands
            tp::mbar_arrive(&full[s]);
            if (++s == S) {
              s = 0;
              ph ^= 1;
            }
            continue;
          }
          tp::mbar_arrive_expect_tx(&full[s], tx_bytes);
          if (RECT && p.halo) {  // halo box {BK, 16, 8*SUB+2} for kernel column dx, block cb
            const int dx = kb / p.kb_per_tap - 1;
            const int cb = kb % p.kb_per_tap;
            tma_load_4d(a_dst, &tmA, &full[s], cb * BK, rx + dx, ry - 1, it.img);
          } else {
            const int tap = kb / p.kb_per_tap;
            const int cb = kb - tap * p.kb_per_tap;
            if (RECT) {
              const int dy = p.ksize == 3 ? tap / 3 - 1 : 0;
              const int dx = p.ksize == 3 ? tap % 3 - 1 : 0;
              tma_load_4d(a_dst, &tmA, &full[s], cb * BK, rx + dx, ry + dy, it.img);
            } else {  // im2col: 128 consecutive compact pixels, window shifted by the tap
              const int ox = p.ksize == 3 ? tap % 3 : 0, oy = p.ksize == 3 ? tap / 3 : 0;
              if (cb >= p.kb_hi) {  // HL8 lo block: 128 e4m3 channels (same stage bytes)
                const int cl = cb - p.kb_hi;
                tma_load_im2col(a_dst, &tmA2, &full[s], cl * 128, f0.x + lo, f0.y + lo, f0.n,
                                (uint16_t)ox, (uint16_t)oy);
                tp::tma_load_2d(b_dst, &tmB2, &full[s], tap * p.cin + cl * 128, n0);
                if (++s == S) {
                  s = 0;
                  ph ^= 1;
                }
                continue;
              }
              tma_load_im2col(a_dst, &tmA, &full[s], cb * BK, f0.x + lo, f0.y + lo, f0.n,
                              (uint16_t)ox, (uint16_t)oy);
            }
            tp::tma_load_2d(b_dst, &tmB, &full[s], tap * p.cin + cb * BK, n0);
          }
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      if (p.dbg & 32) {
        atomicAdd(&g_conv_prof[0], (unsigned long long)(clock64() - pr_start));
        atomicAdd(&g_conv_prof[1], (unsigned long long)pr_wait);
        if (blockIdx.x == 0) atomicAdd(&g_conv_prof[7], 1ull);
      }
    }
  } else if (warp == kMmaWarp) {
    {
      // ================= MMA issuer: the warp runs the loop convergent (descriptors stay
      // in uniform registers) and one elected lane issues; a divergent lane-0 loop made
      // the compiler wrap every tcgen05.mma in an ELECT/R2UR waterfall (~2.5x slower).
      const uint32_t idesc = p.idesc;
      int s = 0;
      uint32_t ph = 0;
      uint32_t aph[2] = {0, 0};
      if (RECT && p.halo && n_tiles > 0) tp::mbar_wait(bres_bar, 0);
      // descriptors are built once; per MMA only the start-address field (addr >> 4, low
      // bits) moves, so each issue is one 64-bit add — rebuilding them per instruction
      // made the single issuing thread the bottleneck for N <= 128 (~90+ cycles/MMA).
      constexpr uint32_t row_bytes = BK * 2;
      constexpr uint32_t sbo = 8 * row_bytes;
      constexpr uint32_t lay = MODE == MODE_SW128 ? 2 : 4;
      const uint64_t a_desc0 = tp::umma_desc(tp::smem_u32(smA), 16, sbo, lay);
      const uint64_t b_desc0 = tp::umma_desc(tp::smem_u32(smB), 16, sbo, lay);
      const uint32_t a_step = p.a_stage_bytes >> 4, b_step = p.b_stage_bytes >> 4;
      const uint32_t bch = p.bchunk_bytes >> 4;
      long long w_te = 0, w_fu = 0;
      PROF_T0(m_start);
      for (int i = 0; i < n_tiles; ++i) {
        const int acc = i & 1;
        PROF_T0(t1);
        tp::mbar_wait(&tempty[acc], aph[acc] ^ 1);
        PROF_ADD(w_te, t1);
        aph[acc] ^= 1;
        tp::tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * p.sub * p.bn);
        int cbk = 0;  // K block within the tap (>= kb_hi: an HL8 lo block)
        for (int kb = 0; kb < p.num_kb; ++kb) {
          const bool lo_blk = cbk >= p.kb_hi;
          if (++cbk == p.kb_per_tap) cbk = 0;
          PROF_T0(t2);
          tp::mbar_wait(&full[s], ph);
          PROF_ADD(w_fu, t2);
          tp::tc_fence_after();
          const uint64_t ad0 = a_desc0 + (uint64_t)(s * a_step);
          const uint64_t bd0 = b_desc0 + (uint64_t)(s * b_step);
          if (!tp::elect_one()) {
          } else if (p.dbg & 2) {
            // profiling: no MMA
          } else if (RECT && p.halo) {
            // three kernel rows dy = sub-windows of the halo box, 16 pixel rows apart
            constexpr uint32_t row16 = RECT_W * row_bytes / 16;  // one pixel row, >> 4
            const int dx = kb / p.kb_per_tap - 1;
            const int cb = kb % p.kb_per_tap;
            for (int j = 0; j < p.sub; ++j) {
              const uint64_t aj = ad0 + (uint64_t)(j * RECT_H * row16);
              const uint32_t dj = d_tmem + j * p.bn;
#pragma unroll
              for (int dy = 0; dy < 3; ++dy) {
                const int chunk = (dy * 3 + dx + 1) * p.kb_per_tap + cb;
                const uint64_t aw = aj + dy * row16;
                const uint64_t bw = b_desc0 + (uint64_t)(chunk * bch);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                  tp::mma_bf16(dj, aw + 2 * k, bw + 2 * k, idesc, (kb | dy | k) != 0);
              }
            }
          } else if (lo_blk) {  // 128 e4m3 channels = 4 x K32, 32 bytes per step as below
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_f8(d_tmem, ad0 + 2 * k, bd0 + 2 * k, idesc, 1);
          } else {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tp::mma_bf16(d_tmem, ad0 + 2 * k, bd0 + 2 * k, idesc, (kb | k) != 0);
          }
          if (tp::elect_one()) tp::mma_commit(&empty[s]);  // frees the stage when these retire
          __syncwarp();
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        if (tp::elect_one()) tp::mma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        __syncwarp();
      }
      if ((p.dbg & 32) && lane == 0) {
        atomicAdd(&g_conv_prof[2], (unsigned long long)(clock64() - m_start));
        atomicAdd(&g_conv_prof[3], (unsigned long long)w_te);
        atomicAdd(&g_conv_prof[4], (unsigned long long)w_fu);
      }
    }
  } else {
    // ================= epilogue: two warpgroups, one per TMEM accumulator =================
    // group g takes the CTA's local tiles i with i % 2 == g; its 4 warps cover the 4
    // TMEM lane quadrants, all BN columns.
    const int g = (int)warp >> 2;
    const float alpha = p.alpha;
    const uint32_t q = warp & 3;
    const int row = (int)(q * 32 + lane);
    const bool f16 = p.f16 != 0;
    const bool leaky = p.leaky != 0;
    const int ores = p.res >> 1, oimg = ores * ores;
    const int total_px = n_img * p.img_px;
    const int nchunks = p.bn >> 4;
    uint32_t ph = 0;
    TileIter it;
    it.init(t_begin, p);
    uint32_t slab = 0;  // TSTORE staging slabs used by this warp
    long long e_wait = 0;
    PROF_T0(e_start);
    for (int i = 0; i < n_tiles; ++i, it.next(p)) {
      if ((i & 1) != g) continue;
      const int n0 = it.nb * p.bn;
      PROF_T0(t3);
      tp::mbar_wait(&tfull[g], ph);
      PROF_ADD(e_wait, t3);
      ph ^= 1;
      tp::tc_fence_after();
      if (p.dbg & 1) {
        tp::tc_fence_before();
        __syncwarp();
        if (lane == 0) tp::mbar_arrive(&tempty[g]);
        continue;
      }

      for (int jt = 0; jt < p.sub; ++jt) {  // stacked 16x8 sub-tiles of a RECT super-tile
      bool valid, writer = true;
      int out_px = 0, sub = 0;
      if (RECT) {
        const int x = it.bx * RECT_W + (row & (RECT_W - 1));
        const int y = (it.by * p.sub + jt) * RECT_H + (row >> 4);
        valid = it.img < n_img && x < p.res && y < p.res;
        writer = ((x | y) & 1) == 0;
        out_px = it.img * oimg + (y >> 1) * ores + (x >> 1);
      } else {
        const int pix = it.mt * 128 + row;
        valid = pix < total_px;
        out_px = pix;
        if (valid && EPI == EPI_REORG) {  // (image, y, x) of the input pixel for reorg_dest
          const PixPos q0 = pix_pos(pix, p.res, p.img_px);
          sub = q0.y * p.res + q0.x;
          out_px = q0.n;
        }
      }
      const uint32_t t_row =
          tmem_base + ((q * 32u) << 16) + (uint32_t)((g * p.sub + jt) * p.bn);
      int rg_px[4] = {0, 0, 0, 0}, rg_cb[4] = {0, 0, 0, 0};  // reorg: per a = c % 4
      if (EPI == EPI_REORG && valid) {
        const int y = sub / p.res, x = sub - y * p.res;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          int Y, X, C;
          reorg_dest(a, y, x, p.res, p.cout, Y, X, C);  // channel 4m + a -> C + 4m
          rg_px[a] = (out_px * ores + Y) * ores + X;
          rg_cb[a] = C;
        }
      }
      uint32_t v[16];
      const bool do_ld = (p.dbg & 8) == 0;
      if (do_ld) {
        tp::tmem_ld16(t_row, v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0u;
      }
      for (int c = 0; c < nchunks; ++c) {
        if (do_ld) tp::tmem_ld_wait();
        float f[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);
        if (do_ld && c + 1 < nchunks) tp::tmem_ld16(t_row + (uint32_t)((c + 1) * 16), v);
        const int ch0 = n0 + c * 16;
        const float4* b4 = reinterpret_cast<const float4*>(bias_s + ch0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 bb = b4[j];
          f[4 * j + 0] = fmaf(f[4 * j + 0], alpha, bb.x);
          f[4 * j + 1] = fmaf(f[4 * j + 1], alpha, bb.y);
          f[4 * j + 2] = fmaf(f[4 * j + 2], alpha, bb.z);
          f[4 * j + 3] = fmaf(f[4 * j + 3], alpha, bb.w);
        }
        if (leaky) {  // leaky(x) = max(x, 0.1x), identical to x > 0 ? x : 0.1x
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.1f * f[j]);
        }
        if (RECT) {  // fused 2x2 max pool: x pair = lane^1, y pair = lane^16
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], __shfl_xor_sync(0xffffffffu, f[j], 1));
#pragma unroll
          for (int j = 0; j < 16; ++j)
            f[j] = fmaxf(f[j], __shfl_xor_sync(0xffffffffu, f[j], RECT_W));
        }
        if (TSTORE) {
          // 64-byte-per-row slabs (2 fp16 chunks or 1 fp32 chunk) staged with the SW64
          // pattern, then one TMA store of {slab, 32 rows}; halo rows are written as zeros
          // two slabs per warp alternate: staging the next one only waits for the store
          // issued two slabs ago (bulk_wait_read1), not for the one just issued
          constexpr int CPS = EPI == EPI_F32 || EPI == EPI_SPLIT ? 1 : 2;
          const int cs = c % CPS;
          const uint32_t slab_off = warp * 4096 + (slab & 1) * 2048;
          const uint32_t buf = tp::smem_u32(smC) + slab_off;
          if (cs == 0) {
            if (lane == 0) bulk_wait_read1();
            __syncwarp();
          }
          const uint32_t rbase = buf + lane * 64;
          const uint32_t swz = (lane >> 1) & 3;
          if (EPI == EPI_SPLIT) {  // one 64-byte row = [hi 16 | lo 16]
            uint32_t hi[8], lo[8];
            split_pairs<8>(f, hi, lo);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              hi[j] = valid ? hi[j] : 0u;
              lo[j] = valid ? lo[j] : 0u;
            }
            st_shared_v4(rbase + ((0 ^ swz) << 4), hi[0], hi[1], hi[2], hi[3]);
            st_shared_v4(rbase + ((1 ^ swz) << 4), hi[4], hi[5], hi[6], hi[7]);
            st_shared_v4(rbase + ((2 ^ swz) << 4), lo[0], lo[1], lo[2], lo[3]);
            st_shared_v4(rbase + ((3 ^ swz) << 4), lo[4], lo[5], lo[6], lo[7]);
          } else if (EPI == EPI_F32) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float a0 = valid ? f[4 * k] : 0.f, a1 = valid ? f[4 * k + 1] : 0.f;
              const float a2 = valid ? f[4 * k + 2] : 0.f, a3 = valid ? f[4 * k + 3] : 0.f;
              st_shared_v4(rbase + ((k ^ swz) << 4), __float_as_uint(a0), __float_as_uint(a1),
                           __float_as_uint(a2), __float_as_uint(a3));
            }
          } else {
            uint32_t pk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (f16) {
                __half2 h = __floats2half2_rn(f[2 * j], f[2 * j + 1]);
                pk[j] = valid ? *reinterpret_cast<uint32_t*>(&h) : 0u;
              } else {
                __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
                pk[j] = valid ? *reinterpret_cast<uint32_t*>(&h) : 0u;
              }
            }
            st_shared_v4(rbase + (((2 * cs) ^ swz) << 4), pk[0], pk[1], pk[2], pk[3]);
            st_shared_v4(rbase + (((2 * cs + 1) ^ swz) << 4), pk[4], pk[5], pk[6], pk[7]);
            if (EPI == EPI_HL8 && valid && !(p.dbg & 4)) {  // lo plane: 16 bytes per pixel
              uint32_t hh[8], ll[4];
              split_hl8(f, hh, ll);
              *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.out_lo) +
                                        (size_t)out_px * p.out_cstride + p.out_coff + ch0) =
                  make_uint4(ll[0], ll[1], ll[2], ll[3]);
            }
          }
          if (cs == CPS - 1) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && (p.dbg & 4) == 0) {
              tma_store_2d(&tmC, smC + slab_off,
                           EPI == EPI_SPLIT ? p.out_coff + 2 * ch0 : p.out_coff + ch0 - 16 * cs,
                           it.mt * 128 + (int)q * 32);
              bulk_commit();
            }
            ++slab;
          }
          continue;
        }
        if (!valid || !writer || ch0 >= p.cout || (p.dbg & 4)) continue;
        if (EPI == EPI_REORG) {  // darknet reorg: every element to its own (Y, X, C)
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            // channels c = 4m + a of one input pixel go to 4 output pixels (one per a),
            // channel base + 4m there (reorg_dest; the bases are computed once per pixel)
            const int a = j & 3, C = rg_cb[a] + 4 * ((ch0 + j) >> 2);
            const size_t px = (size_t)rg_px[a];
            const float v = f[j];
            if (p.out_lo != nullptr) {
              const size_t o = px * p.out_cstride + p.out_coff + C;
              store_hl8_1(reinterpret_cast<__half*>(p.out) + o,
                          reinterpret_cast<uint8_t*>(p.out_lo) + o, v);
            } else if (p.split) {
              __half* o = reinterpret_cast<__half*>(p.out) + px * p.out_cstride + p.out_coff +
                          32 * (C >> 4) + (C & 15);
              const __half h = __float2half_rn(v);
              o[0] = h;
              o[16] = __float2half_rn(v - __half2float(h));
            } else {
              __half* o = reinterpret_cast<__half*>(p.out) + px * p.out_cstride + p.out_coff + C;
              if (f16)
                *o = __float2half_rn(v);
              else
                *reinterpret_cast<__nv_bfloat16*>(o) = __float2bfloat16_rn(v);
            }
          }
        } else if (p.out_lo != nullptr) {  // HL8 planes (pooled direct stores)
          const size_t o = (size_t)out_px * p.out_cstride + p.out_coff + ch0;
          store_hl8(reinterpret_cast<__half*>(p.out) + o, reinterpret_cast<uint8_t*>(p.out_lo) + o, f);
        } else if (p.split) {
          store_split16(reinterpret_cast<__nv_bfloat16*>(p.out) + (size_t)out_px * p.out_cstride +
                            p.out_coff + 2 * ch0,
                        f);
        } else {  // (fp32 outputs always take the TMA-store path above)
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (f16) {
              __half2 h = __floats2half2_rn(f[2 * j], f[2 * j + 1]);
              pk[j] = *reinterpret_cast<uint32_t*>(&h);
            } else {
              __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
              pk[j] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
          const int cofs = p.out_coff + ch0;
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + (size_t)out_px * p.out_cstride + cofs;
          *reinterpret_cast<uint4*>(o) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(o + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      tp::tmem_ld_wait();
      }  // sub-tiles
      tp::tc_fence_before();
      __syncwarp();
      if (lane == 0) tp::mbar_arrive(&tempty[g]);
    }
    if (TSTORE && lane == 0) bulk_wait_all();
    if ((p.dbg & 32) && warp == 0 && lane == 0) {
      atomicAdd(&g_conv_prof[5], (unsigned long long)(clock64() - e_start));
      atomicAdd(&g_conv_prof[6], (unsigned long long)e_wait);
    }
  }

  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  if (warp == kMmaWarp) tp::tmem_dealloc(tmem_base, p.tmem_cols);
}

// ------------------------------------------------------------------ CTA-pair variant
// FLAT SW128 layers (every deep 3x3 / 1x1 conv): a 2-CTA cluster computes a 256-row x BN
// tile with tcgen05.mma.cta_group::2 (M=256). Each CTA stages its own 128 A rows and HALF
// of the B tile, so per SM the tensor core reads 4 KB + BN/2*32 B of shared memory per
// K=16 step instead of 4 KB + BN*32 B — the 1-CTA kernel is shared-memory-bound on B.
// The leader (rank 0) issues the MMAs; both CTAs' TMA loads complete on the leader's
// full barrier; MMA commits multicast to both CTAs' empty/tfull barriers; both CTAs'
// epilogue warps release the accumulator on the leader's tempty barrier.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t mapa_rank(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(tp::smem_u32(local)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, uint32_t leader_bar,
                                                 int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(tp::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_im2col_pair(void* dst, const void* tmap,
                                                     uint32_t leader_bar, int32_t c, int32_t w,
                                                     int32_t h, int32_t n, uint16_t ow,
                                                     uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::"
      "bytes [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(tp::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(leader_bar), "r"(c), "r"(w), "r"(h), "r"(n),
      "h"(ow), "h"(oh)
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_pair_f8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit_pair_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(tp::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    conv_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC,
                     const __grid_constant__ CUtensorMap tmA2,
                     const __grid_constant__ CUtensorMap tmB2, const ConvParams p) {
  constexpr int BK = 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* smA = smem;
  uint8_t* smB = smem + (size_t)S * p.a_stage_bytes;
  uint8_t* smC = smB + (size_t)S * p.b_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smC + p.stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 5);
  float* bias_s = reinterpret_cast<float*>(bars + 2 * S + 6);

  const uint32_t warp = tp::warp_id();
  const uint32_t lane = tp::lane_id();
  const uint32_t rank = cluster_rank();
  const int cout_pad = p.bn * p.n_blocks_n;
  const int half_bn = p.bn >> 1;

  if (warp == kProdWarp && lane == 0) {
    tp::tma_prefetch(&tmA);
    tp::tma_prefetch(&tmB);
    for (int s = 0; s < S; ++s) {
      tp::mbar_init(&full[s], 1);
      tp::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tp::mbar_init(&tfull[a], 1);
      tp::mbar_init(&tempty[a], 8);  // 4 epilogue warps in each CTA of the pair
    }
    tp::fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tp::smem_u32(tmem_slot)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < cout_pad; i += blockDim.x) bias_s[i] = p.bias[i];
  tp::tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised + TMEM allocated
  tp::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_img = p.n_img_dev != nullptr ? min(*p.n_img_dev, p.n_img) : p.n_img;
  const int total_px = n_img * p.img_px;
  const int m_blocks = (total_px + 255) / 256;
  const int total_tiles = m_blocks * p.n_blocks_n;
  // Tiles are dealt round-robin (cluster cid takes t = cid, cid + n_clusters, ...) in a
  // grouped raster: groups of GM M-blocks, N-block-major inside a group, so one wave of
  // clusters covers GM M-blocks x (n_clusters / GM) N-blocks. The live L2 set is then GM
  // activation blocks + a few weight slices instead of every weight slice at once (the
  // 2x-K parity plan's 38-47 MB weights otherwise thrash L2: 20x the DRAM reads).
  const int n_clusters = (int)gridDim.x >> 1, cid = (int)blockIdx.x >> 1;
  const int n_tiles = cid < total_tiles ? (total_tiles - cid + n_clusters - 1) / n_clusters : 0;
  const int GM = max(1, n_clusters / min(p.n_blocks_n, 2));
  auto tile_at = [&](int i, int& mt, int& nb) {
    const int t = cid + i * n_clusters;
    const int grp = t / (GM * p.n_blocks_n);
    const int gm = min(GM, m_blocks - grp * GM);
    const int tl = t - grp * GM * p.n_blocks_n;
    nb = tl / gm;
    mt = grp * GM + (tl - nb * gm);
  };

  if (warp == kProdWarp) {
    if (lane == 0) {
      // ============ TMA producer (both CTAs; bytes land on the leader's barrier) ============
      int s = 0;
      uint32_t ph = 0;
      const int lo = p.ksize == 3 ? -1 : 0;  // im2col window corner
      long long pr_wait = 0;
      PROF_T0(pr_start);
      for (int i = 0; i < n_tiles; ++i) {
        int mt, nb;
        tile_at(i, mt, nb);
        const int n0 = nb * p.bn;
        const PixPos f0 = pix_pos(mt * 256 + (int)rank * 128, p.res, p.img_px);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          PROF_T0(tw);
          tp::mbar_wait(&empty[s], ph ^ 1);
          PROF_ADD(pr_wait, tw);
          if (p.dbg & 16) {  // profiling: no TMA, stale operands (the leader's arrival only)
            if (rank == 0) tp::mbar_arrive(&full[s]);
            if (++s == S) {
              s = 0;
              ph ^= 1;
            }
            continue;
          }
          if (rank == 0)
            tp::mbar_arrive_expect_tx(&full[s], 2 * (p.a_stage_bytes + p.b_stage_bytes));
          const uint32_t lbar = mapa_rank(&full[s], 0);
          const int tap = kb / p.kb_per_tap;
          const int cb = kb - tap * p.kb_per_tap;
          const int ox = p.ksize == 3 ? tap % 3 : 0, oy = p.ksize == 3 ? tap / 3 : 0;
          if (cb < p.kb_hi) {
            tma_load_im2col_pair(smA + (size_t)s * p.a_stage_bytes, &tmA, lbar, cb * BK,
                                 f0.x + lo, f0.y + lo, f0.n, (uint16_t)ox, (uint16_t)oy);
            tma_load_2d_pair(smB + (size_t)s * p.b_stage_bytes, &tmB, lbar, tap * p.cin + cb * BK,
                             n0 + (int)rank * half_bn);
          } else {  // HL8 lo block: 128 e4m3 channels, same stage bytes
            const int cl = cb - p.kb_hi;
            tma_load_im2col_pair(smA + (size_t)s * p.a_stage_bytes, &tmA2, lbar, cl * 128,
                                 f0.x + lo, f0.y + lo, f0.n, (uint16_t)ox, (uint16_t)oy);
            tma_load_2d_pair(smB + (size_t)s * p.b_stage_bytes, &tmB2, lbar,
                             tap * p.cin + cl * 128, n0 + (int)rank * half_bn);
          }
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      if ((p.dbg & 32) && rank == 0) {
        atomicAdd(&g_conv_prof[0], (unsigned long long)(clock64() - pr_start));
        atomicAdd(&g_conv_prof[1], (unsigned long long)pr_wait);
        if (blockIdx.x == 0) atomicAdd(&g_conv_prof[7], 1ull);
      }
    }
  } else if (warp == kMmaWarp) {
    if (rank == 0) {
      // ============ MMA issuer: leader CTA, warp-convergent loop, one elected lane ============
      const uint64_t a_desc0 = tp::umma_desc(tp::smem_u32(smA), 16, 1024, 2);
      const uint64_t b_desc0 = tp::umma_desc(tp::smem_u32(smB), 16, 1024, 2);
      const uint32_t a_step = p.a_stage_bytes >> 4, b_step = p.b_stage_bytes >> 4;
      int s = 0;
      uint32_t ph = 0;
      uint32_t aph[2] = {0, 0};
      long long w_te = 0, w_fu = 0;
      PROF_T0(m_start);
      for (int i = 0; i < n_tiles; ++i) {
        const int acc = i & 1;
        PROF_T0(t1);
        tp::mbar_wait(&tempty[acc], aph[acc] ^ 1);
        PROF_ADD(w_te, t1);
        aph[acc] ^= 1;
        tp::tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * p.bn);
        int cbk = 0;  // K block within the tap (>= kb_hi: an HL8 lo block)
        for (int kb = 0; kb < p.num_kb; ++kb) {
          const bool lo_blk = cbk >= p.kb_hi;
          if (++cbk == p.kb_per_tap) cbk = 0;
          PROF_T0(t2);
          tp::mbar_wait(&full[s], ph);
          PROF_ADD(w_fu, t2);
          tp::tc_fence_after();
          const uint64_t ad0 = a_desc0 + (uint64_t)(s * a_step);
          const uint64_t bd0 = b_desc0 + (uint64_t)(s * b_step);
          if (tp::elect_one()) {
            if (lo_blk) {  // 128 e4m3 channels: 4 x K32 (32 bytes per row per step)
#pragma unroll
              for (int k = 0; k < 4; ++k) mma_pair_f8(d_tmem, ad0 + 2 * k, bd0 + 2 * k, p.idesc, 1);
            } else {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_pair(d_tmem, ad0 + 2 * k, bd0 + 2 * k, p.idesc, (kb | k) != 0);
            }
            commit_pair_mc(&empty[s]);  // frees the stage in both CTAs
          }
          __syncwarp();
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        if (tp::elect_one()) commit_pair_mc(&tfull[acc]);  // both CTAs' epilogues may read
        __syncwarp();
      }
      if ((p.dbg & 32) && lane == 0) {
        atomicAdd(&g_conv_prof[2], (unsigned long long)(clock64() - m_start));
        atomicAdd(&g_conv_prof[3], (unsigned long long)w_te);
        atomicAdd(&g_conv_prof[4], (unsigned long long)w_fu);
      }
    }
  } else {
    // ============ epilogue: both CTAs, own 128 rows; groups alternate accumulators ============
    const int g = (int)warp >> 2;
    const float alpha = p.alpha;
    const uint32_t q = warp & 3;
    const bool f16 = p.f16 != 0;
    const bool leaky = p.leaky != 0;
    const int nchunks = p.bn >> 4;
    const uint32_t leader_tempty[2] = {mapa_rank(&tempty[0], 0), mapa_rank(&tempty[1], 0)};
    uint32_t ph = 0;
    uint32_t slab = 0;  // TSTORE staging slabs used by this warp
    long long e_wait = 0;
    PROF_T0(e_start);
    for (int i = 0; i < n_tiles; ++i) {
      if ((i & 1) != g) continue;
      int mt, nb;
      tile_at(i, mt, nb);
      const int n0 = nb * p.bn;
      PROF_T0(t3);
      tp::mbar_wait(&tfull[g], ph);
      PROF_ADD(e_wait, t3);
      ph ^= 1;
      tp::tc_fence_after();
      const int rbase = mt * 256 + (int)rank * 128 + (int)q * 32;
      const bool valid = rbase + (int)lane < total_px;
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + (uint32_t)(g * p.bn);
      const uint32_t swz = (lane >> 1) & 3;
      uint32_t v[16];
      tp::tmem_ld16(t_row, v);
      for (int c = 0; c < nchunks; ++c) {
        tp::tmem_ld_wait();
        float f[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);
        if (c + 1 < nchunks) tp::tmem_ld16(t_row + (uint32_t)((c + 1) * 16), v);
        const int ch0 = n0 + c * 16;
        const float4* b4 = reinterpret_cast<const float4*>(bias_s + ch0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 bb = b4[j];
          f[4 * j + 0] = fmaf(f[4 * j + 0], alpha, bb.x);
          f[4 * j + 1] = fmaf(f[4 * j + 1], alpha, bb.y);
          f[4 * j + 2] = fmaf(f[4 * j + 2], alpha, bb.z);
          f[4 * j + 3] = fmaf(f[4 * j + 3], alpha, bb.w);
        }
        if (leaky) {
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.1f * f[j]);
        }
        constexpr int CPS = EPI == EPI_F32 || EPI == EPI_SPLIT ? 1 : 2;
        const int cs = c % CPS;
        const uint32_t slab_off = warp * 4096 + (slab & 1) * 2048;  // two alternating slabs
        const uint32_t rowa = tp::smem_u32(smC) + slab_off + lane * 64;
        if (cs == 0) {
          if (lane == 0) bulk_wait_read1();
          __syncwarp();
        }
        if (EPI == EPI_SPLIT) {  // one 64-byte row = [hi 16 | lo 16]
          uint32_t hi[8], lo[8];
          split_pairs<8>(f, hi, lo);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            hi[j] = valid ? hi[j] : 0u;
            lo[j] = valid ? lo[j] : 0u;
          }
          st_shared_v4(rowa + ((0 ^ swz) << 4), hi[0], hi[1], hi[2], hi[3]);
          st_shared_v4(rowa + ((1 ^ swz) << 4), hi[4], hi[5], hi[6], hi[7]);
          st_shared_v4(rowa + ((2 ^ swz) << 4), lo[0], lo[1], lo[2], lo[3]);
          st_shared_v4(rowa + ((3 ^ swz) << 4), lo[4], lo[5], lo[6], lo[7]);
        } else if (EPI == EPI_F32) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float a0 = valid ? f[4 * k] : 0.f, a1 = valid ? f[4 * k + 1] : 0.f;
            const float a2 = valid ? f[4 * k + 2] : 0.f, a3 = valid ? f[4 * k + 3] : 0.f;
            st_shared_v4(rowa + ((k ^ swz) << 4), __float_as_uint(a0), __float_as_uint(a1),
                         __float_as_uint(a2), __float_as_uint(a3));
          }
        } else {
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (f16) {
              __half2 h = __floats2half2_rn(f[2 * j], f[2 * j + 1]);
              pk[j] = valid ? *reinterpret_cast<uint32_t*>(&h) : 0u;
            } else {
              __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
              pk[j] = valid ? *reinterpret_cast<uint32_t*>(&h) : 0u;
            }
          }
          st_shared_v4(rowa + (((2 * cs) ^ swz) << 4), pk[0], pk[1], pk[2], pk[3]);
          st_shared_v4(rowa + (((2 * cs + 1) ^ swz) << 4), pk[4], pk[5], pk[6], pk[7]);
          if (EPI == EPI_HL8 && valid) {  // lo plane: 16 bytes per pixel and chunk
            uint32_t hh[8], ll[4];
            split_hl8(f, hh, ll);
            *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.out_lo) +
                                      (size_t)(rbase + (int)lane) * p.out_cstride + p.out_coff +
                                      ch0) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
          }
        }
        if (cs == CPS - 1) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmC, smC + slab_off,
                         EPI == EPI_SPLIT ? p.out_coff + 2 * ch0 : p.out_coff + ch0 - 16 * cs,
                         rbase);
            bulk_commit();
          }
          ++slab;
        }
      }
      tp::tmem_ld_wait();
      tp::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty[g]);
    }
    if (lane == 0) bulk_wait_all();
    if ((p.dbg & 32) && warp == 0 && lane == 0 && rank == 0) {
      atomicAdd(&g_conv_prof[5], (unsigned long long)(clock64() - e_start));
      atomicAdd(&g_conv_prof[6], (unsigned long long)e_wait);
    }
  }

  tp::tc_fence_before();
  cluster_sync_all();
  tp::tc_fence_after();
  if (warp == kMmaWarp)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols)
                 : "memory");
}

// ------------------------------------------------------------------ CTA-pair pooled 3x3
// Pooled 3x3 layers whose weights do not fit in shared memory (16-bit plan: layer 10;
// parity plan: layers 6 and 10, K = 1152 / 2304): a 2-CTA cluster computes a 16 x 16
// output block (each CTA one 16 x 8 half, M = 256) x N with tcgen05.mma.cta_group::2.
// One stage per (kernel column dx, 64-channel block): a halo box {64, 16, 10} whose three
// kernel rows are descriptor offsets of 16 box rows, plus the three taps' half-N weight
// slices — A is fetched 3x per tile instead of 9x (RECT tiles) and each CTA stages only
// half of B. The epilogue pools 2x2 in registers (x pair lane^1, y pair lane^16) and
// stores the pooled pixels directly (16-bit, or hi/lo pairs in the parity plan).
__device__ __forceinline__ void tma_load_4d_pair(void* dst, const void* tmap, uint32_t leader_bar,
                                                 int32_t c0, int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(tp::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

constexpr int PR_W = 16, PR_H = 8;  // one M = 128 block: 16 x 8 output pixels

// MH = M blocks per CTA (1: 16 x 8 per CTA, the pair covers 16 x 16; 2: 16 x 16 per CTA,
// one {64, 16, 18} halo box serves both blocks, so the A + B bytes each stage brings per
// MMA drop from 44 KB / 12 to 60 KB / 24 — for N = 128 the fill rate from L2, not the
// tensor pipe, bounds the MH = 1 tile). POOL: fused 2x2 max pool, else every pixel is
// stored (16-bit or hi/lo pairs).
template <int MH, bool POOL>
__global__ void __launch_bounds__(kThreads, 1)
    conv_pair_rect_kernel(const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmA2,
                          const __grid_constant__ CUtensorMap tmB2, const ConvParams p) {
  constexpr int BK = 64;
  constexpr int CH = PR_H * MH;  // output rows per CTA
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* smA = smem;
  uint8_t* smB = smem + (size_t)S * p.a_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smB + (size_t)S * p.b_stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 5);
  float* bias_s = reinterpret_cast<float*>(bars + 2 * S + 6);

  const uint32_t warp = tp::warp_id();
  const uint32_t lane = tp::lane_id();
  const uint32_t rank = cluster_rank();
  const int cout_pad = p.bn * p.n_blocks_n;
  const int half_bn = p.bn >> 1;

  if (warp == kProdWarp && lane == 0) {
    tp::tma_prefetch(&tmA);
    tp::tma_prefetch(&tmB);
    for (int s = 0; s < S; ++s) {
      tp::mbar_init(&full[s], 1);
      tp::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tp::mbar_init(&tfull[a], 1);
      tp::mbar_init(&tempty[a], 8);  // 4 epilogue warps in each CTA of the pair
    }
    tp::fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tp::smem_u32(tmem_slot)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < cout_pad; i += blockDim.x) bias_s[i] = p.bias[i];
  tp::tc_fence_before();
  cluster_sync_all();
  tp::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_img = p.n_img_dev != nullptr ? min(*p.n_img_dev, p.n_img) : p.n_img;
  const int per_img = p.tiles_x * p.tiles_y;
  const int m_blocks = n_img * per_img;
  const int total_tiles = m_blocks * p.n_blocks_n;
  const int n_clusters = (int)gridDim.x >> 1, cid = (int)blockIdx.x >> 1;
  const int n_tiles = cid < total_tiles ? (total_tiles - cid + n_clusters - 1) / n_clusters : 0;
  const int GM = max(1, n_clusters / min(p.n_blocks_n, 2));
  auto tile_at = [&](int i, int& img, int& y0, int& x0, int& nb) {
    const int t = cid + i * n_clusters;
    const int grp = t / (GM * p.n_blocks_n);
    const int gm = min(GM, m_blocks - grp * GM);
    const int tl = t - grp * GM * p.n_blocks_n;
    nb = tl / gm;
    const int mt = grp * GM + (tl - nb * gm);
    img = mt / per_img;
    const int r = mt - img * per_img;
    const int by = r / p.tiles_x;
    x0 = (r - by * p.tiles_x) * PR_W;
    y0 = by * 2 * CH + (int)rank * CH;  // this CTA's half of the pair's rows
  };

  if (warp == kProdWarp) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs; bytes land on the leader's barrier) =====
      int s = 0;
      uint32_t ph = 0;
      const uint32_t b_slice = (uint32_t)half_bn * BK * 2;
      for (int i = 0; i < n_tiles; ++i) {
        int img, y0, x0, nb;
        tile_at(i, img, y0, x0, nb);
        const int n0 = nb * p.bn;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          tp::mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0)
            tp::mbar_arrive_expect_tx(&full[s], 2 * (p.a_stage_bytes + p.b_stage_bytes));
          const uint32_t lbar = mapa_rank(&full[s], 0);
          const int dx = kb / p.kb_per_tap - 1;
          const int cb = kb - (dx + 1) * p.kb_per_tap;
          // HL8 lo block (cb >= kb_hi): 128 e4m3 channels of the lo plane, same box bytes
          const bool lo_blk = cb >= p.kb_hi;
          const int cc = lo_blk ? (cb - p.kb_hi) * 128 : cb * BK;
          tma_load_4d_pair(smA + (size_t)s * p.a_stage_bytes, lo_blk ? &tmA2 : &tmA, lbar, cc,
                           x0 + dx, y0 - 1, img);
          uint8_t* bdst = smB + (size_t)s * p.b_stage_bytes;
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
            tma_load_2d_pair(bdst + dy * b_slice, lo_blk ? &tmB2 : &tmB, lbar,
                             (dy * 3 + dx + 1) * p.cin + cc, n0 + (int)rank * half_bn);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    if (rank == 0) {
      // ===== MMA issuer: leader CTA, warp-convergent loop, one elected lane =====
      const uint64_t a_desc0 = tp::umma_desc(tp::smem_u32(smA), 16, 1024, 2);
      const uint64_t b_desc0 = tp::umma_desc(tp::smem_u32(smB), 16, 1024, 2);
      const uint32_t a_step = p.a_stage_bytes >> 4, b_step = p.b_stage_bytes >> 4;
      constexpr uint32_t a_row16 = PR_W * BK * 2 / 16;  // one box row of 16 pixels, >> 4
      const uint32_t b_slice16 = (uint32_t)half_bn * BK * 2 / 16;
      int s = 0;
      uint32_t ph = 0;
      uint32_t aph[2] = {0, 0};
      for (int i = 0; i < n_tiles; ++i) {
        const int acc = i & 1;
        tp::mbar_wait(&tempty[acc], aph[acc] ^ 1);
        aph[acc] ^= 1;
        tp::tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * MH * p.bn);
        int cbk = 0;  // K block within the kernel column (>= kb_hi: an HL8 lo block)
        for (int kb = 0; kb < p.num_kb; ++kb) {
          const bool lo_blk = cbk >= p.kb_hi;
          if (++cbk == p.kb_per_tap) cbk = 0;
          tp::mbar_wait(&full[s], ph);
          tp::tc_fence_after();
          const uint64_t ad0 = a_desc0 + (uint64_t)(s * a_step);
          const uint64_t bd0 = b_desc0 + (uint64_t)(s * b_step);
          if (tp::elect_one()) {
            if (lo_blk) {
#pragma unroll
              for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                for (int h = 0; h < MH; ++h)
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    mma_pair_f8(d_tmem + (uint32_t)(h * p.bn),
                                ad0 + (dy + PR_H * h) * a_row16 + 2 * k,
                                bd0 + dy * b_slice16 + 2 * k, p.idesc, 1);
            } else {
#pragma unroll
              for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                for (int h = 0; h < MH; ++h)  // M block h: output rows 8h .. 8h+7 of the CTA
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    mma_pair(d_tmem + (uint32_t)(h * p.bn), ad0 + (dy + PR_H * h) * a_row16 + 2 * k,
                             bd0 + dy * b_slice16 + 2 * k, p.idesc, (kb | dy | k) != 0);
            }
            commit_pair_mc(&empty[s]);
          }
          __syncwarp();
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        if (tp::elect_one()) commit_pair_mc(&tfull[acc]);
        __syncwarp();
      }
    }
  } else {
    // ===== epilogue: both CTAs, own rows; groups alternate accumulators =====
    const int g = (int)warp >> 2;
    const float alpha = p.alpha;
    const uint32_t q = warp & 3;
    const int row = (int)(q * 32 + lane);
    const bool f16 = p.f16 != 0, leaky = p.leaky != 0, spl = p.split != 0;
    const int ores = POOL ? p.res >> 1 : p.res, oimg = ores * ores;
    const int nchunks = p.bn >> 4;
    const uint32_t leader_tempty[2] = {mapa_rank(&tempty[0], 0), mapa_rank(&tempty[1], 0)};
    uint32_t ph = 0;
    for (int i = 0; i < n_tiles; ++i) {
      if ((i & 1) != g) continue;
      int img, y0, x0, nb;
      tile_at(i, img, y0, x0, nb);
      const int n0 = nb * p.bn;
      tp::mbar_wait(&tfull[g], ph);
      ph ^= 1;
      tp::tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < MH; ++h) {
        const int x = x0 + (row & (PR_W - 1)), y = y0 + PR_H * h + (row >> 4);
        const bool store = x < p.res && y < p.res && (!POOL || ((x | y) & 1) == 0);
        const int ox = POOL ? x >> 1 : x, oy = POOL ? y >> 1 : y;
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) +
                           (size_t)(img * oimg + oy * ores + ox) * p.out_cstride + p.out_coff;
        const uint32_t t_row = tmem_base + ((q * 32u) << 16) + (uint32_t)((g * MH + h) * p.bn);
        uint32_t v[16];
        tp::tmem_ld16(t_row, v);
        for (int c = 0; c < nchunks; ++c) {
          tp::tmem_ld_wait();
          float f[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);
          if (c + 1 < nchunks) tp::tmem_ld16(t_row + (uint32_t)((c + 1) * 16), v);
          if (POOL) {
            // 2x2 max first (bias and leaky are monotonic: the same value), x pair lane^1,
            // y pair lane^16
#pragma unroll
            for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], __shfl_xor_sync(0xffffffffu, f[j], 1));
#pragma unroll
            for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], __shfl_xor_sync(0xffffffffu, f[j], PR_W));
          }
          const int ch0 = n0 + c * 16;
          const float4* b4 = reinterpret_cast<const float4*>(bias_s + ch0);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 bb = b4[j];
            f[4 * j + 0] = fmaf(f[4 * j + 0], alpha, bb.x);
            f[4 * j + 1] = fmaf(f[4 * j + 1], alpha, bb.y);
            f[4 * j + 2] = fmaf(f[4 * j + 2], alpha, bb.z);
            f[4 * j + 3] = fmaf(f[4 * j + 3], alpha, bb.w);
          }
          if (leaky) {
#pragma unroll
            for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.1f * f[j]);
          }
          if (!store || ch0 >= p.cout || (p.dbg & 4)) continue;
          if (p.out_lo != nullptr) {
            const size_t oo = (size_t)(img * oimg + oy * ores + ox) * p.out_cstride + p.out_coff + ch0;
            store_hl8(reinterpret_cast<__half*>(p.out) + oo, reinterpret_cast<uint8_t*>(p.out_lo) + oo, f);
            continue;
          }
          if (spl) {
            store_split16(o + 2 * ch0, f);
            continue;
          }
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (f16) {
              __half2 hh = __floats2half2_rn(f[2 * j], f[2 * j + 1]);
              pk[j] = *reinterpret_cast<uint32_t*>(&hh);
            } else {
              __nv_bfloat162 hh = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
              pk[j] = *reinterpret_cast<uint32_t*>(&hh);
            }
          }
          *reinterpret_cast<uint4*>(o + ch0) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(o + ch0 + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
        tp::tmem_ld_wait();
      }
      tp::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty[g]);
    }
  }

  tp::tc_fence_before();
  cluster_sync_all();
  tp::tc_fence_after();
  if (warp == kMmaWarp)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols)
                 : "memory");
}

// ------------------------------------------------------------------ swapped operands, N = 128
// 3x3 layers with 128 output channels (parity plan: layers 4 and 6). With pixels as the M
// operand, every K = 16 step of a 128 x 128 MMA reads 4 KB of A + 4 KB of B from shared
// memory in its 64 cycles of math — the operand reads, not the tensor pipe, bound those
// layers (~55-78% pipe activity). Swapped, the weights are A (M = 128 output channels)
// and the pixels are B (N = 256 = a 16 x 16 output block): 4 KB + 8 KB per 128 cycles.
// One stage per (kernel column dx, 32-channel block): a halo box {32, 16, 18} of the input
// (SW64) whose three kernel rows dy are descriptor offsets of 16 box rows, plus the three
// taps' weight slices {32, 128}. The accumulator is channel-major (TMEM lane = output
// channel, column = pixel), so the epilogue stores each pixel's channels as one
// warp-contiguous 64-byte run per 16-bit plane (hi and lo planes in the parity plan) and
// pools 2 x 2 inside a thread (columns x, x+1 of rows y, y+1).
// The SW_CL CTAs of a cluster take consecutive pixel blocks and share the weights: each
// loads 1/SW_CL of every weight slice and multicasts it to all, so a stage brings 18 KB of
// pixels + 24/SW_CL KB of weights per CTA instead of 18 + 24 (the L2 -> SM fill rate,
// ~55 B/clk per SM unshared, held the MMA issuer on `full` 16-38% of the time).
constexpr int SW_BK = 32, SW_W = 16, SW_H = 16, SW_CL = 2;  // 4-CTA clusters: not all co-resident (1.7x slower)
constexpr int SW_STAGING = 8 * 2 * 2048;  // unpooled epilogue: 2 slabs of 16 px x 128 B per warp
constexpr int SW_POOL_SCRATCH = 1024;     // pooled HL8 epilogue: per-warp transpose tile
// HL8 unpooled epilogue: 2 slabs per warp of two rows (hi 2 x 1 KB + lo 2 x 512 B)
constexpr int SW_SLAB_HL8 = 3072, SW_STAGING_HL8 = 8 * 2 * SW_SLAB_HL8;

// 16 TMEM lanes x 16 columns in the mma-fragment layout: thread t holds lane t/4 (v0, v1;
// v4, v5) and lane t/4 + 8 (v2, v3; v6, v7), columns 2(t%4), 2(t%4)+1 (+8 for v4..v7)
__device__ __forceinline__ void tmem_ld_16x256b_x2(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
// four 8x8 b16 fragments stored transposed: smem row j (address from thread 8m + j for
// matrix m) receives column j of fragment m
__device__ __forceinline__ void stmatrix_x4_trans(uint32_t addr, uint32_t r0, uint32_t r1,
                                                  uint32_t r2, uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.x4.trans.m8n8.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr),
               "r"(r0), "r"(r1), "r"(r2), "r"(r3)
               : "memory");
}
// 2-D box multicast to every CTA in cta_mask (same smem offset and barrier offset in each)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const void* tmap, uint64_t* bar,
                                               int32_t c0, int32_t c1, uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(tp::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(tp::smem_u32(bar)), "r"(c0), "r"(c1), "h"(cta_mask)
      : "memory");
}
// single-CTA MMA completion arriving on the same barrier in every CTA of cta_mask
__device__ __forceinline__ void commit_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(tp::smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void* tmap, const void* smem_src, int32_t c0,
                                             int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(tp::smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// Unpooled swap epilogue with HL8 output (layer 4 of the F16F8 plan): per output row the
// warp's 32 channels x 16 pixels leave as an fp16 hi slab (16 px x 64 B, SW64, stmatrix
// .trans as in the pair path) and an e4m3 lo slab (16 px x 32 B): thread t holds channels
// t/4 and t/4 + 8 of each 16-channel half for pixels 2(t%4), +1 (+8), so 4 shuffles per
// (half, pixel group) gather channel pair (2k, 2k+1), k = t/4, into one b16 per pixel and
// a second stmatrix .trans writes each pixel's 32 lo bytes in channel order. Both slabs of
// a row are one bulk group; two rows alternate (wait_group.read 1), as the pair path.
__device__ __forceinline__ void swap_epilogue_hl8(const ConvParams& p, const CUtensorMap& tmC,
                                                  const CUtensorMap& tmC2, uint8_t* smC,
                                                  uint32_t slab0, uint32_t t_row, bool live,
                                                  int y0, int x0, int img, int nb, uint32_t q,
                                                  uint32_t lane, int ores, float alpha,
                                                  bool leaky) {
  const int m = (int)lane >> 3, j = (int)lane & 7;
  const int cq = (int)lane >> 2, tq = (int)lane & 3;
  const float* bias = p.bias;
  float bq[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    bq[h][0] = bias[nb * 128 + (int)q * 32 + 16 * h + cq];
    bq[h][1] = bias[nb * 128 + (int)q * 32 + 16 * h + cq + 8];
  }
  // destination channel pair k = cq of each half: sources = lanes holding channels 2k, 2k+1
  const int src_a = 4 * ((2 * cq) & 7) + tq, src_b = src_a + 4;
  const bool hi_e = cq >= 4;  // channels 2k >= 8 are those lanes' e = 1 values
  // TMEM loads are software-pipelined: row r+1's two 16x256b loads are in flight while row
  // r's lo bytes are exchanged and both slabs are staged and stored
  uint32_t v[16];  // [h = 0: v0..7 | h = 1: v8..15]
  if (live && y0 < ores) {
    tmem_ld_16x256b_x2(t_row, *reinterpret_cast<uint32_t(*)[8]>(v));
    tmem_ld_16x256b_x2(t_row + (16u << 16), *reinterpret_cast<uint32_t(*)[8]>(v + 8));
  }
  // rows leave in pairs: a slab holds two rows (hi [0, 2048), lo [2048, 3072)) and one
  // 2-row TMA store per plane drains it (half the store count of per-row slabs; a row
  // below the image inside a pair is staged garbage that the tensor map clips)
#pragma unroll 1
  for (int r = 0; r < SW_H; ++r) {
    if (!live || y0 + r >= ores) break;
    const int rr = r & 1;
    const uint32_t slab = slab0 + (uint32_t)((r >> 1) & 1) * SW_SLAB_HL8;
    uint32_t hs[2][2][2], lw[2][2];  // hi pairs [h][cg][e]; lo stmatrix words [h][cg]
    uint32_t lp[2][2];               // lo byte pairs of channels cq (low 16) and cq + 8 (high)
    tp::tmem_ld_wait_regs(v);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int cg = 0; cg < 2; ++cg) {
        uint32_t l2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float a = fmaf(__uint_as_float(v[8 * h + 4 * cg + 2 * e]), alpha, bq[h][e]);
          float b = fmaf(__uint_as_float(v[8 * h + 4 * cg + 2 * e + 1]), alpha, bq[h][e]);
          if (leaky) {
            a = fmaxf(a, 0.1f * a);
            b = fmaxf(b, 0.1f * b);
          }
          const __half2 hh = __floats2half2_rn(a, b);
          hs[h][cg][e] = *reinterpret_cast<const uint32_t*>(&hh);
          const float2 hf = __half22float2(hh);
          uint16_t pr;  // byte 0 = pixel 2tq, byte 1 = pixel 2tq + 1
          asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;"
              : "=h"(pr)
              : "f"((b - hf.y) * kLoScale), "f"((a - hf.x) * kLoScale));
          l2[e] = pr;
        }
        lp[h][cg] = l2[0] | (l2[1] << 16);
      }
    }
    if (r + 1 < SW_H && y0 + r + 1 < ores) {
      tmem_ld_16x256b_x2(t_row + (uint32_t)((r + 1) * 16), *reinterpret_cast<uint32_t(*)[8]>(v));
      tmem_ld_16x256b_x2(t_row + (16u << 16) + (uint32_t)((r + 1) * 16),
                         *reinterpret_cast<uint32_t(*)[8]>(v + 8));
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int cg = 0; cg < 2; ++cg) {
        // one shuffle per source lane brings both of its channels (cq, cq + 8); the
        // destination keeps the one its channel pair needs
        const uint32_t A = __shfl_sync(0xffffffffu, lp[h][cg], src_a);
        const uint32_t B = __shfl_sync(0xffffffffu, lp[h][cg], src_b);
        // (ch 2k, px) (ch 2k+1, px) (ch 2k, px+1) (ch 2k+1, px+1)
        lw[h][cg] = __byte_perm(hi_e ? A >> 16 : A, hi_e ? B >> 16 : B, 0x5140);
      }
    if (rr == 0) {
      if (lane == 0) bulk_wait_read1();  // the stores two pairs back have read this slab
      __syncwarp();
    }
    {
      // hi: matrices (h, channels 0-7 | 8-15) -> 16-byte chunk 2h + (m & 1) of the pixel's
      // 64-byte row (SW64: chunk ^ ((pixel >> 1) & 3)); one x4 per pixel group cg
#pragma unroll
      for (int cg = 0; cg < 2; ++cg) {
        const int pix = 16 * rr + 8 * cg + j;
        const uint32_t addr = slab + (uint32_t)(pix * 64) + (uint32_t)(((m ^ (pix >> 1)) & 3) * 16);
        stmatrix_x4_trans(addr, hs[0][cg][0], hs[0][cg][1], hs[1][cg][0], hs[1][cg][1]);
      }
      // lo: matrix m = (h = m >> 1, cg = m & 1): pixel 8cg + j, bytes 16h .. 16h + 15
      const int lpix = 16 * rr + 8 * (m & 1) + j;
      stmatrix_x4_trans(slab + 2048 + (uint32_t)(lpix * 32 + 16 * (m >> 1)), lw[0][0], lw[0][1],
                        lw[1][0], lw[1][1]);
    }
    if (rr == 1 || r + 1 >= SW_H || y0 + r + 1 >= ores) {  // the pair is staged: store it
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int c0 = p.out_coff + nb * 128 + (int)q * 32;
        tma_store_4d(&tmC, smC + (slab - tp::smem_u32(smC)), c0, x0, y0 + r - rr, img);
        tma_store_4d(&tmC2, smC + (slab + 2048 - tp::smem_u32(smC)), c0, x0, y0 + r - rr, img);
        bulk_commit();
      }
    }
  }
}

// ---- fused 1x1 consumer of the unpooled HL8 swap epilogue (layer 4 -> layer 5)
// Staging X (one buffer for both epilogue groups) + the resident 1x1 weights, in the
// operand layouts the unfused 1x1 kernel reads: X hi = 4 K blocks (32 channels each, warp q
// writes block q) of [128 px][64 B] SW64, X lo = 4 x [128 px][32 B] SW32; W likewise with
// 64 rows (output channels).
constexpr int FU_N = 64;                  // 1x1 output channels
constexpr uint32_t FU_XL = 32768, FU_WH = 49152, FU_WL = 65536, FU_BYTES = 73728;
constexpr int FU_SCRATCH = 3072;           // per epilogue warp: one tile row, hi 2 KB + lo 1 KB
constexpr int FU_EXTRA = 4 * 8 + FU_N * 4 + 16 + kEpiWarps * FU_SCRATCH;  // x4bar, bias, scratch

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Per tile i and pixel half hf (tile rows 8hf .. 8hf+7 = 128 pixels = TMEM columns
// [128hf, 128hf + 128) of the group's accumulator): the group's 4 warps turn layer 4's
// accumulators into its HL8 values (the same ops as swap_epilogue_hl8) and stage them in X;
// after a group barrier one thread issues the 1x1's MMAs (A = X, B = W, M = 128, N = 64)
// into the half's drained accumulator columns [128hf, 128hf + 64), in the unfused 1x1
// kernel's K order (hi channels in K16 steps, then lo channels in K32 steps: the same
// products summed in the same order, so the results are the unfused ones bit for bit).
// X use u = 2i + hf waits for use u - 1's MMAs (x4bar[(u - 1) % 4], arrived by their
// commit); uses complete in order and a group has seen its own use u - 4 complete, so every
// parity wait is within one phase. Then the 1x1's epilogue: warp q reads TMEM lanes 32q ..
// 32q + 31 (pixels) x 64 columns and stores both HL8 planes of the 1x1's output.
__device__ __forceinline__ void swap_fused_1x1(const ConvParams& p, uint32_t xs, uint32_t scr,
                                               uint64_t* x4bar, const float* bias4,
                                               const float* bias5,
                                               uint32_t tmem_base, int i, int g, uint32_t q,
                                               uint32_t lane, bool live, int y0, int x0, int img,
                                               int ores, float alpha, bool leaky) {
  const int m = (int)lane >> 3, j = (int)lane & 7;
  const int cq = (int)lane >> 2, tq = (int)lane & 3;
  float bq[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    bq[h][0] = bias4[(int)q * 32 + 16 * h + cq];
    bq[h][1] = bias4[(int)q * 32 + 16 * h + cq + 8];
  }
  const int src_a = 4 * ((2 * cq) & 7) + tq, src_b = src_a + 4;
  const bool hi_e = cq >= 4;
  const uint32_t t_row = tmem_base + ((q * 32u) << 16) + (uint32_t)(g * 256);
  const uint32_t xh = xs + q * 8192u, xl = xs + FU_XL + q * 4096u;
  // TP_CONV_DEBUG bit 32: phase cycles of warp q = 0 (g_conv_prof 0: waiting for the staging
  // buffer, 1: staging, 5: waiting for the 1x1's MMAs, 6: the 1x1's epilogue)
  const bool prof = (p.dbg & 32) && q == 0 && lane == 0;
  long long t_a = 0, t_b = 0, t_c = 0, t_d = 0, t0 = 0;
#pragma unroll 1
  for (int hf = 0; hf < 2; ++hf) {
    const int u = 2 * i + hf;
    if (prof) t0 = clock64();
    if (u > 0) tp::mbar_wait(&x4bar[(u - 1) & 3], (uint32_t)(((u - 1) >> 2) & 1));
    if (prof) {
      const long long t1 = clock64();
      t_a += t1 - t0;
      t0 = t1;
    }
    const uint32_t c0 = t_row + (uint32_t)(hf * 128);
    uint32_t v[16];
    tmem_ld_16x256b_x2(c0, *reinterpret_cast<uint32_t(*)[8]>(v));
    tmem_ld_16x256b_x2(c0 + (16u << 16), *reinterpret_cast<uint32_t(*)[8]>(v + 8));
#pragma unroll 1
    for (int r = 0; r < 8; ++r) {
      uint32_t hs[2][2][2], lw[2][2], lp[2][2];
      tp::tmem_ld_wait_regs(v);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int cg = 0; cg < 2; ++cg) {
          uint32_t l2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            float a = fmaf(__uint_as_float(v[8 * h + 4 * cg + 2 * e]), alpha, bq[h][e]);
            float b = fmaf(__uint_as_float(v[8 * h + 4 * cg + 2 * e + 1]), alpha, bq[h][e]);
            if (leaky) {
              a = fmaxf(a, 0.1f * a);
              b = fmaxf(b, 0.1f * b);
            }
            const __half2 hh = __floats2half2_rn(a, b);
            hs[h][cg][e] = *reinterpret_cast<const uint32_t*>(&hh);
            const float2 hf2 = __half22float2(hh);
            uint16_t pr;
            asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;"
                : "=h"(pr)
                : "f"((b - hf2.y) * kLoScale), "f"((a - hf2.x) * kLoScale));
            l2[e] = pr;
          }
          lp[h][cg] = l2[0] | (l2[1] << 16);
        }
      }
      if (r + 1 < 8) {
        tmem_ld_16x256b_x2(c0 + (uint32_t)((r + 1) * 16), *reinterpret_cast<uint32_t(*)[8]>(v));
        tmem_ld_16x256b_x2(c0 + (16u << 16) + (uint32_t)((r + 1) * 16),
                           *reinterpret_cast<uint32_t(*)[8]>(v + 8));
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int cg = 0; cg < 2; ++cg) {
          const uint32_t A = __shfl_sync(0xffffffffu, lp[h][cg], src_a);
          const uint32_t B = __shfl_sync(0xffffffffu, lp[h][cg], src_b);
          lw[h][cg] = __byte_perm(hi_e ? A >> 16 : A, hi_e ? B >> 16 : B, 0x5140);
        }
#pragma unroll
      for (int cg = 0; cg < 2; ++cg) {
        const int pl = 16 * r + 8 * cg + j;
        stmatrix_x4_trans(xh + (uint32_t)(pl * 64) + (uint32_t)(((m ^ (pl >> 1)) & 3) * 16),
                          hs[0][cg][0], hs[0][cg][1], hs[1][cg][0], hs[1][cg][1]);
      }
      const int lpl = 16 * r + 8 * (m & 1) + j;
      stmatrix_x4_trans(xl + (uint32_t)(lpl * 32) + (uint32_t)((((m >> 1) ^ (lpl >> 2)) & 1) * 16),
                        lw[0][0], lw[0][1], lw[1][0], lw[1][1]);
    }
    fence_proxy_async_smem();
    tp::tc_fence_before();
    named_bar_sync(1u + (uint32_t)g, 128);
    tp::tc_fence_after();
    if (prof) t_b += clock64() - t0;
    if (q == 0) {
      if (tp::elect_one()) {
        const uint32_t d = tmem_base + (uint32_t)(g * 256 + hf * 128);
        const uint32_t idesc = tp::idesc_f16kind(128, FU_N, false);
        const uint64_t xhd = tp::umma_desc(xs, 16, 512, 4);
        const uint64_t whd = tp::umma_desc(xs + FU_WH, 16, 512, 4);
        const uint64_t xld = tp::umma_desc(xs + FU_XL, 16, 256, 6);
        const uint64_t wld = tp::umma_desc(xs + FU_WL, 16, 256, 6);
#pragma unroll
        for (int kq = 0; kq < 4; ++kq)
#pragma unroll
          for (int k = 0; k < 2; ++k)
            tp::mma_bf16(d, xhd + (uint64_t)(kq * 512 + 2 * k), whd + (uint64_t)(kq * 256 + 2 * k),
                         idesc, (kq | k) != 0);
#pragma unroll
        for (int kq = 0; kq < 4; ++kq)
          mma_f8(d, xld + (uint64_t)(kq * 256), wld + (uint64_t)(kq * 128), idesc, 1);
        tp::mma_commit(&x4bar[u & 3]);
      }
      __syncwarp();
    }
  }
#pragma unroll 1
  for (int hf = 0; hf < 2; ++hf) {
    const int u = 2 * i + hf;
    if (prof) t0 = clock64();
    tp::mbar_wait(&x4bar[u & 3], (uint32_t)((u >> 2) & 1));
    if (prof) {
      const long long t1 = clock64();
      t_c += t1 - t0;
      t0 = t1;
    }
    tp::tc_fence_after();
    const uint32_t ta = tmem_base + ((q * 32u) << 16) + (uint32_t)(g * 256 + hf * 128);
    uint32_t a[4][16];
#pragma unroll
    for (int c = 0; c < 4; ++c) tp::tmem_ld16(ta + (uint32_t)(16 * c), a[c]);
    tp::tmem_ld_wait();
    uint32_t hi[4][8], lo[4][4];  // this lane's pixel: 64 fp16 + 64 e4m3 channels
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float f[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        f[e] = fmaf(__uint_as_float(a[c][e]), p.f5_alpha, bias5[16 * c + e]);
        if (p.f5_leaky) f[e] = fmaxf(f[e], 0.1f * f[e]);
      }
      split_hl8(f, hi[c], lo[c]);
    }
    // lanes 16k .. 16k+15 hold tile row 8hf + 2q + k: stage that row (hi 16 x 128 B SW128,
    // lo 16 x 64 B SW64) in the warp's scratch, then store it with every lane writing 16
    // consecutive bytes (4 pixels = 512 contiguous bytes per instruction; a lane-per-pixel
    // store touched 32 lines per instruction and held the epilogue)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      __syncwarp();
      if (((int)lane >> 4) == k) {
        const uint32_t r = lane & 15;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          st_shared_v4(scr + r * 128 + (((uint32_t)cc ^ (r & 7)) << 4), hi[cc >> 1][4 * (cc & 1)],
                       hi[cc >> 1][4 * (cc & 1) + 1], hi[cc >> 1][4 * (cc & 1) + 2],
                       hi[cc >> 1][4 * (cc & 1) + 3]);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
          st_shared_v4(scr + 2048 + r * 64 + (((uint32_t)cc ^ ((r >> 1) & 3)) << 4), lo[cc][0],
                       lo[cc][1], lo[cc][2], lo[cc][3]);
      }
      __syncwarp();
      const int y = y0 + 8 * hf + 2 * (int)q + k;
      if (!live || y >= ores) {
        if (prof && k == 1) t_d += clock64() - t0;
        continue;
      }
      const size_t row0 = ((size_t)img * ores + y) * ores;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t pr = 4 * t + (lane >> 3), cc = lane & 7;
        uint4 v;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(scr + pr * 128 + ((cc ^ (pr & 7)) << 4))
                     : "memory");
        if (x0 + (int)pr < ores)
          *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(p.f5_out) +
                                    (row0 + x0 + pr) * p.f5_cstride + 8 * cc) = v;
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const uint32_t pr = 8 * t + (lane >> 2), cc = lane & 3;
        uint4 v;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(scr + 2048 + pr * 64 + ((cc ^ ((pr >> 1) & 3)) << 4))
                     : "memory");
        if (x0 + (int)pr < ores)
          *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.f5_out_lo) +
                                    (row0 + x0 + pr) * p.f5_cstride + 16 * cc) = v;
      }
      if (prof && k == 1) t_d += clock64() - t0;
    }
  }
  if (prof) {
    atomicAdd(&g_conv_prof[0], (unsigned long long)t_a);
    atomicAdd(&g_conv_prof[1], (unsigned long long)t_b);
    atomicAdd(&g_conv_prof[5], (unsigned long long)t_c);
    atomicAdd(&g_conv_prof[6], (unsigned long long)t_d);
  }
}

template <bool POOL>
__global__ void __launch_bounds__(kThreads, 1)
    conv_swap_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmA2,
                     const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC2,
                     const ConvParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* smX = smem;                                   // pixel boxes (B operand)
  uint8_t* smW = smem + (size_t)S * p.a_stage_bytes;     // weight slices (A operand)
  uint8_t* smC = smW + (size_t)S * p.b_stage_bytes;    // unpooled: output staging slabs
  uint64_t* bars = reinterpret_cast<uint64_t*>(smC + p.stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);
  float* bias_s = reinterpret_cast<float*>(bars + 2 * S + 5);
  uint64_t* x4bar = bars + 2 * S + 5 + 64;  // fused 1x1: staging-buffer uses (after 128 biases)
  float* bias5_s = reinterpret_cast<float*>(x4bar + 4);
  // fused 1x1: per-epilogue-warp store scratch (16-byte aligned, after the 1x1's bias)
  const uint32_t fu_scr = (tp::smem_u32(bias5_s + FU_N) + 15u) & ~15u;

  const uint32_t warp = tp::warp_id();
  const uint32_t lane = tp::lane_id();
  const int cout_pad = 128 * p.n_blocks_n;
  const bool fused = !POOL && p.fuse != 0;
  if (warp == kProdWarp && lane == 0) {
    tp::tma_prefetch(&tmA);
    tp::tma_prefetch(&tmB);
    for (int i = 0; i < S; ++i) {
      tp::mbar_init(&full[i], 1);
      tp::mbar_init(&empty[i], SW_CL);  // every CTA's MMAs must have drained the stage
    }
    for (int a = 0; a < 2; ++a) {
      tp::mbar_init(&tfull[a], 1);
      tp::mbar_init(&tempty[a], 4);
    }
    if (fused)
      for (int a = 0; a < 4; ++a) tp::mbar_init(&x4bar[a], 1);
    tp::fence_mbar_init();
  }
  if (warp == kMmaWarp) tp::tmem_alloc(tmem_slot, 512);
  for (int i = threadIdx.x; i < cout_pad; i += blockDim.x) bias_s[i] = p.bias[i];
  if (fused) {
    // the 1x1's weights, resident: hi [64][128] fp16 -> 4 SW64 K blocks, lo [64][128] e4m3
    // -> 4 SW32 K blocks (16-byte chunks; chunk c of row n XORed as TMA would place it)
    const uint32_t xs = tp::smem_u32(smC);
    const uint4* wh = reinterpret_cast<const uint4*>(p.f5_w);
    const uint4* wl = reinterpret_cast<const uint4*>(p.f5_wlo);
    for (int t = threadIdx.x; t < FU_N * 16; t += blockDim.x) {
      const int n = t >> 4, c = t & 15;
      const uint4 w = wh[t];
      st_shared_v4(xs + FU_WH + (uint32_t)((c >> 2) * 4096 + n * 64 + (((c & 3) ^ ((n >> 1) & 3)) << 4)),
                   w.x, w.y, w.z, w.w);
    }
    for (int t = threadIdx.x; t < FU_N * 8; t += blockDim.x) {
      const int n = t >> 3, c = t & 7;
      const uint4 w = wl[t];
      st_shared_v4(xs + FU_WL + (uint32_t)((c >> 1) * 2048 + n * 32 + (((c & 1) ^ ((n >> 2) & 1)) << 4)),
                   w.x, w.y, w.z, w.w);
    }
    for (int t = threadIdx.x; t < FU_N; t += blockDim.x) bias5_s[t] = p.f5_bias[t];
    fence_proxy_async_smem();  // generic-proxy writes -> the MMAs' async-proxy reads
  }
  tp::tc_fence_before();
  cluster_sync_all();  // the peer's barriers are initialised before any multicast lands
  tp::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t rank = cluster_rank();

  const int n_img = p.n_img_dev != nullptr ? min(*p.n_img_dev, p.n_img) : p.n_img;
  const int per_img = p.tiles_x * p.tiles_y;
  const int total_tiles = n_img * per_img * p.n_blocks_n;
  // the CTAs of a cluster run the same number of tiles (they feed each other's weight
  // stages): tile group j of cluster c = tiles SW_CL (c + j * clusters) + rank; a CTA whose
  // tile is past the end recomputes the last tile and stores nothing
  const int n_clusters = (int)gridDim.x / SW_CL, cid = (int)blockIdx.x / SW_CL;
  const int total_groups = (total_tiles + SW_CL - 1) / SW_CL;
  const int n_tiles = cid < total_groups ? (total_groups - cid + n_clusters - 1) / n_clusters : 0;
  auto tile_at = [&](int i, int& img, int& y0, int& x0, int& nb) {
    const int t = min(SW_CL * (cid + i * n_clusters) + (int)rank, total_tiles - 1);
    const int mt = t / p.n_blocks_n;
    nb = t - mt * p.n_blocks_n;
    img = mt / per_img;
    const int r = mt - img * per_img;
    const int by = r / p.tiles_x;
    x0 = (r - by * p.tiles_x) * SW_W;
    y0 = by * SW_H;
  };

  if (warp == kProdWarp) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint32_t w_slice = 128 * SW_BK * 2;
      for (int i = 0; i < n_tiles; ++i) {
        int img, y0, x0, nb;
        tile_at(i, img, y0, x0, nb);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          tp::mbar_wait(&empty[s], ph ^ 1);
          tp::mbar_arrive_expect_tx(&full[s], p.a_stage_bytes + p.b_stage_bytes);
          const int dx = kb / p.kb_per_tap - 1;
          const int cb = kb - (dx + 1) * p.kb_per_tap;
          // HL8 lo block (cb >= kb_hi): 64 e4m3 channels (64-byte rows, same box bytes)
          const bool lo_blk = cb >= p.kb_hi;
          const int cc = lo_blk ? (cb - p.kb_hi) * 64 : cb * SW_BK;
          tma_load_4d(smX + (size_t)s * p.a_stage_bytes, lo_blk ? &tmA2 : &tmA, &full[s], cc,
                      x0 + dx, y0 - 1, img);
          // this CTA's 128 / SW_CL output channels of each tap's slice, to every CTA
          uint8_t* wdst = smW + (size_t)s * p.b_stage_bytes + rank * (w_slice / SW_CL);
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
            tma_load_2d_mc(wdst + dy * w_slice, lo_blk ? &tmB2 : &tmB, &full[s],
                           (dy * 3 + dx + 1) * p.cin + cc,
                           nb * 128 + (128 / SW_CL) * (int)rank, (uint16_t)((1 << SW_CL) - 1));
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    constexpr uint32_t row_bytes = SW_BK * 2, sbo = 8 * row_bytes;
    const uint64_t x_desc0 = tp::umma_desc(tp::smem_u32(smX), 16, sbo, 4);  // SW64
    const uint64_t w_desc0 = tp::umma_desc(tp::smem_u32(smW), 16, sbo, 4);
    const uint32_t x_step = p.a_stage_bytes >> 4, w_step = p.b_stage_bytes >> 4;
    constexpr uint32_t x_row16 = SW_W * row_bytes / 16;   // one box row of 16 pixels, >> 4
    constexpr uint32_t w_slice16 = 128 * row_bytes / 16;  // one tap's weight slice, >> 4
    int s = 0;
    uint32_t ph = 0;
    uint32_t aph[2] = {0, 0};
    long long w_te = 0, w_fu = 0;
    PROF_T0(m_start);
    for (int i = 0; i < n_tiles; ++i) {
      const int acc = i & 1;
      PROF_T0(t1);
      tp::mbar_wait(&tempty[acc], aph[acc] ^ 1);
      PROF_ADD(w_te, t1);
      aph[acc] ^= 1;
      tp::tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * 256);
      int cbk = 0;  // K block within the kernel column (>= kb_hi: an HL8 lo block)
      for (int kb = 0; kb < p.num_kb; ++kb) {
        const bool lo_blk = cbk >= p.kb_hi;
        if (++cbk == p.kb_per_tap) cbk = 0;
        PROF_T0(t2);
        tp::mbar_wait(&full[s], ph);
        PROF_ADD(w_fu, t2);
        tp::tc_fence_after();
        const uint64_t xd = x_desc0 + (uint64_t)(s * x_step);
        const uint64_t wd = w_desc0 + (uint64_t)(s * w_step);
        if (tp::elect_one()) {
          if (lo_blk) {  // 64 e4m3 channels per row: 2 x K32 (32 bytes each, as below)
#pragma unroll
            for (int dy = 0; dy < 3; ++dy)
#pragma unroll
              for (int k = 0; k < 2; ++k)
                mma_f8(d_tmem, wd + dy * w_slice16 + 2 * k, xd + dy * x_row16 + 2 * k, p.idesc, 1);
          } else {
#pragma unroll
            for (int dy = 0; dy < 3; ++dy)
#pragma unroll
              for (int k = 0; k < SW_BK / 16; ++k)
                tp::mma_bf16(d_tmem, wd + dy * w_slice16 + 2 * k, xd + dy * x_row16 + 2 * k,
                             p.idesc, (kb | dy | k) != 0);
          }
          commit_mc(&empty[s], (uint16_t)((1 << SW_CL) - 1));  // frees it for every producer
        }
        __syncwarp();
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
      if (tp::elect_one()) tp::mma_commit(&tfull[acc]);
      __syncwarp();
    }
    if ((p.dbg & 32) && lane == 0) {
      atomicAdd(&g_conv_prof[2], (unsigned long long)(clock64() - m_start));
      atomicAdd(&g_conv_prof[3], (unsigned long long)w_te);
      atomicAdd(&g_conv_prof[4], (unsigned long long)w_fu);
      if (blockIdx.x == 0) atomicAdd(&g_conv_prof[7], 1ull);
    }
  } else {
    // epilogue: group g takes tiles i % 2 == g; warp q owns output channels q*32 .. q*32+31
    const int g = (int)warp >> 2;
    const float alpha = p.alpha;
    const uint32_t q = warp & 3;
    const bool f16 = p.f16 != 0, leaky = p.leaky != 0, spl = p.split != 0;
    const int ores = POOL ? p.res >> 1 : p.res;
    uint32_t ph = 0;
    for (int i = 0; i < n_tiles; ++i) {
      if ((i & 1) != g) continue;
      int img, y0, x0, nb;
      tile_at(i, img, y0, x0, nb);
      const int co = nb * 128 + (int)(q * 32 + lane);
      // the plan requires cout == 128; a recomputed last tile (odd count) stores nothing
      const bool live = !(p.dbg & 4) && SW_CL * (cid + i * n_clusters) + (int)rank < total_tiles;
      // stored channel of co: hi/lo planes interleaved per 16 channels in the parity plan
      const int sc = p.out_coff + (spl ? 32 * (co >> 4) + (co & 15) : co);
      const float bco = bias_s[co];
      tp::mbar_wait(&tfull[g], ph);
      ph ^= 1;
      tp::tc_fence_after();
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + (uint32_t)(g * 256);
      // a warp writes one pixel's 32 channels per instruction (64 B, or 2 x 32 B hi/lo runs)
      auto put = [&](int y, int x, float v) {
        v = fmaf(v, alpha, bco);
        if (leaky) v = fmaxf(v, 0.1f * v);
        const size_t oi = ((size_t)(img * ores + y) * ores + x) * p.out_cstride + sc;
        __half* o = reinterpret_cast<__half*>(p.out) + oi;
        if (p.out_lo != nullptr) {  // HL8 planes (sc is the real channel)
          store_hl8_1(o, reinterpret_cast<uint8_t*>(p.out_lo) + oi, v);
        } else if (spl) {
          const __half h = __float2half_rn(v);
          o[0] = h;
          o[16] = __float2half_rn(v - __half2float(h));
        } else if (f16) {
          o[0] = __float2half_rn(v);
        } else {
          *reinterpret_cast<__nv_bfloat16*>(o) = __float2bfloat16_rn(v);
        }
      };
      if (POOL) {
        // TMEM loads software-pipelined: pooled row r+1's two loads are in flight while
        // row r is pooled and stored
        uint32_t a[16], b[16];
        tp::tmem_ld16(t_row, a);
        tp::tmem_ld16(t_row + 16u, b);
        for (int r = 0; r < SW_H / 2; ++r) {
          tp::tmem_ld_wait_regs(a);
          tp::tmem_ld_wait_regs(b);
          float m[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)  // 2x2 max before bias + leaky (both monotonic)
            m[j] = fmaxf(fmaxf(__uint_as_float(a[2 * j]), __uint_as_float(a[2 * j + 1])),
                         fmaxf(__uint_as_float(b[2 * j]), __uint_as_float(b[2 * j + 1])));
          if (r + 1 < SW_H / 2) {
            tp::tmem_ld16(t_row + (uint32_t)(2 * (r + 1) * 16), a);
            tp::tmem_ld16(t_row + (uint32_t)((2 * (r + 1) + 1) * 16), b);
          }
          const int oy = (y0 >> 1) + r;
          if (!live || oy >= ores) continue;
          if (p.out_lo != nullptr) {
            // HL8: the warp's 32 channels x 8 pooled pixels go through a per-warp smem tile
            // (hi [8 px][32 ch] fp16, lo [8 px][32 ch] bytes) and leave as 16-byte vectors,
            // one store per lane and plane instead of 8 scalar 2-byte / 1-byte stores per
            // lane (the scalar stores held the epilogue at ~1.4x the MMA time)
            const uint32_t scr = tp::smem_u32(smC) + warp * SW_POOL_SCRATCH;  // explicit .shared
            __syncwarp();  // the previous row's vector reads are done
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float v = fmaf(m[j], alpha, bco);
              if (leaky) v = fmaxf(v, 0.1f * v);
              const __half h = __float2half_rn(v);
              uint16_t pr;
              asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;"
                  : "=h"(pr)
                  : "f"(0.0f), "f"((v - __half2float(h)) * kLoScale));
              asm volatile("st.shared.b16 [%0], %1;" ::"r"(scr + (uint32_t)(j * 32 + lane) * 2),
                           "h"(__half_as_ushort(h))
                           : "memory");
              asm volatile("st.shared.b8 [%0], %1;" ::"r"(scr + 512u + (uint32_t)(j * 32 + lane)),
                           "h"(pr)
                           : "memory");
            }
            __syncwarp();
            const int pj = (int)lane >> 2, c8 = (int)lane & 3;
            const int ox = (x0 >> 1) + pj;
            const size_t px = (size_t)(img * ores + oy) * ores + ox;
            const int cb = p.out_coff + nb * 128 + (int)q * 32;
            uint4 hv, lv;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(hv.x), "=r"(hv.y), "=r"(hv.z), "=r"(hv.w)
                         : "r"(scr + (uint32_t)(pj * 64 + c8 * 16))
                         : "memory");
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(lv.x), "=r"(lv.y), "=r"(lv.z), "=r"(lv.w)
                         : "r"(scr + 512u + (uint32_t)(pj * 32 + (c8 & 1) * 16))
                         : "memory");
            if (ox < ores) {
              *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(p.out) + px * p.out_cstride + cb + 8 * c8) = hv;
              if (c8 < 2)
                *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.out_lo) + px * p.out_cstride + cb + 16 * c8) = lv;
            }
            continue;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int ox = (x0 >> 1) + j;
            if (ox < ores) put(oy, ox, m[j]);
          }
        }
        tp::tmem_ld_wait();
      } else {
        // unpooled (parity plan): per output row, the warp's 32 channels x 16 pixels leave
        // through a 16 x 128 B smem slab (SW128) written transposed by stmatrix, then one TMA
        // store (out-of-image pixels are clipped by the tensor map). Fragment rows =
        // channels, columns = pixels (tcgen05.ld 16x256b), so stmatrix .trans lands each
        // pixel's [hi 16 | lo 16] channel groups contiguously.
        const uint32_t slab0 = tp::smem_u32(smC) + warp * 4096;
        const int m = (int)lane >> 3, j = (int)lane & 7;  // stmatrix: matrix m, row j
        if (fused) {
          swap_fused_1x1(p, tp::smem_u32(smC), fu_scr + warp * FU_SCRATCH, x4bar, bias_s, bias5_s,
                         tmem_base, i, g, q, lane, live, y0, x0, img, ores, alpha, leaky);
          tp::tc_fence_before();
          __syncwarp();
          if (lane == 0) tp::mbar_arrive(&tempty[g]);
          continue;
        }
        if (p.out_lo != nullptr) {
          swap_epilogue_hl8(p, tmC, tmC2, smC, tp::smem_u32(smC) + warp * (2 * SW_SLAB_HL8), t_row,
                            live, y0, x0, img, nb, q, lane, ores, alpha, leaky);
          tp::tc_fence_before();
          __syncwarp();
          if (lane == 0) tp::mbar_arrive(&tempty[g]);
          continue;
        }
        const int cq = (int)lane >> 2;                     // fragment row (channel) of this thread
        float bq[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          bq[h][0] = bias_s[nb * 128 + (int)q * 32 + 16 * h + cq];
          bq[h][1] = bias_s[nb * 128 + (int)q * 32 + 16 * h + cq + 8];
        }
#pragma unroll 1
        for (int r = 0; r < SW_H; ++r) {
          // rows below the image are neither staged nor stored: a staged row without a
          // committed store would let wait_group.read 1 pass while the store two slabs back
          // is still reading
          if (!live || y0 + r >= ores) break;
          const uint32_t slab = slab0 + (uint32_t)(r & 1) * 2048;
          // TMEM -> registers -> hi/lo pairs first: this overlaps the previous row's TMA
          // store, which must finish reading its slab before the stmatrix writes below
          uint32_t hs[2][2][2], ls[2][2][2];  // [half h][pixel group cg][channel cq (+8)]
#pragma unroll
          for (int h = 0; h < 2; ++h) {  // channels 16h .. 16h+15 of the warp
            uint32_t v[8];
            tmem_ld_16x256b_x2(t_row + ((uint32_t)(16 * h) << 16) + (uint32_t)(r * 16), v);
            tp::tmem_ld_wait_regs(v);
#pragma unroll
            for (int cg = 0; cg < 2; ++cg)  // pixels 8cg .. 8cg+7
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                float a = fmaf(__uint_as_float(v[4 * cg + 2 * e]), alpha, bq[h][e]);
                float b = fmaf(__uint_as_float(v[4 * cg + 2 * e + 1]), alpha, bq[h][e]);
                if (leaky) {
                  a = fmaxf(a, 0.1f * a);
                  b = fmaxf(b, 0.1f * b);
                }
                const __half2 hh = __floats2half2_rn(a, b);
                hs[h][cg][e] = *reinterpret_cast<const uint32_t*>(&hh);
                const float2 hf = __half22float2(hh);
                const __half2 ll = __floats2half2_rn(a - hf.x, b - hf.y);
                ls[h][cg][e] = *reinterpret_cast<const uint32_t*>(&ll);
              }
          }
          if (lane == 0) bulk_wait_read1();  // the store two rows back has read this slab
          __syncwarp();
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int cg = 0; cg < 2; ++cg) {
              // matrices: 0 hi ch 0-7, 1 hi ch 8-15, 2 lo ch 0-7, 3 lo ch 8-15 of this half
              // -> 16-byte chunk 4h + m of the pixel's 128-byte row
              const int pix = 8 * cg + j;
              const uint32_t addr = slab + (uint32_t)(pix * 128) +
                                    (uint32_t)((((4 * h + m) ^ (pix & 7)) & 7) * 16);
              stmatrix_x4_trans(addr, hs[h][cg][0], hs[h][cg][1], ls[h][cg][0], ls[h][cg][1]);
            }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(&tmC, smC + (slab - tp::smem_u32(smC)),
                         p.out_coff + 64 * (nb * 4 + (int)q), x0, y0 + r, img);
            bulk_commit();
          }
        }
      }
      tp::tc_fence_before();
      __syncwarp();
      if (lane == 0) tp::mbar_arrive(&tempty[g]);
    }
  }

  if (!POOL && warp < kEpiWarps && lane == 0) bulk_wait_all();
  tp::tc_fence_before();
  cluster_sync_all();  // no CTA leaves while its peer may still signal its barriers
  tp::tc_fence_after();
  if (warp == kMmaWarp) tp::tmem_dealloc(tmem_base, 512);
}

// ------------------------------------------------------------------ layer 0, pool-in-M
// Layer 0 (3x3, 3->32, leaky, 2x2 maxpool) has K = 48 but 608^2 outputs per tile, so it
// is bound by epilogue instructions, not math. Here each M row is one POOLED output
// pixel: the four pool positions (py,px) accumulate into four TMEM accumulators.
// Input: 8-byte pixels P(u) = rgb0 of tile column u (zero halo: 1 row above / below, 2
// columns left, 4 right). A row R(k) = P(2k-2) .. P(2k+5) is 64 bytes at a 16-byte
// aligned offset, so one overlapping TMA view (k 16 B apart) serves every k. Even conv
// columns x = 2k use the first 32 bytes [P(2k-2) P(2k-1) P(2k) P(2k+1)] with weights
// [0 w-1 w0 w+1]; odd columns x = 2k+1 use the same 32 bytes with [0 0 w-1 w0] plus the
// second 32 bytes [P(2k+2) ..] with [w+1 0 0 0] — no MMA operand straddles a 32-byte
// K chunk. Both column phases of index k share R(k) (SW64, K = 32): TMA loads one box
// {32 halves, 16 k, 9 rows (stride 2)} per input row phase — 288 box rows per tile, the
// TMA row rate was this kernel's limit at 32-byte rows. Per tile (16x8 pooled = 32x16
// conv pixels): 12 MMAs (K=16: per pool row and kernel row one N=64 MMA for both column
// phases' first-chunk term + one N=32 for the odd phase's second chunk at +32 B); the epilogue
// reads 4 x 32 columns per row and does max + bias + leaky + pack.
constexpr int L0_BOX_ROWS = 9;                       // strided rows per box
constexpr int L0_BOX_BYTES = L0_BOX_ROWS * 16 * 64;  // 9216: 9 rows x 16 windows x 64 B
constexpr int L0_STAGE = 2 * L0_BOX_BYTES;           // 18432: one box per input row phase
constexpr int L0_STAGING = 8 * 2 * 4096;             // epilogue store slabs

__global__ void __launch_bounds__(kThreads, 1)
    conv_l0_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                   const ConvParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* smA = smem;
  uint8_t* smB = smem + (size_t)S * L0_STAGE;  // resident weights: 9 chunks x 1 KB
  uint8_t* smC = smB + 9 * 1024;  // output staging: 8 warps x 2 slabs x 4 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(smC + L0_STAGING);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  // 4 accumulator buffers (4 x 128 TMEM columns): epilogue group g takes tiles i % 2 == g
  // and alternates buffers i % 4, so the MMAs of its next tile run while it drains one
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + 4;
  uint64_t* bres_bar = bars + 2 * S + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 9);
  float* bias_s = reinterpret_cast<float*>(bars + 2 * S + 10);

  const uint32_t warp = tp::warp_id();
  const uint32_t lane = tp::lane_id();
  if (warp == kProdWarp && lane == 0) {
    tp::tma_prefetch(&tmA);
    tp::tma_prefetch(&tmB);
    for (int s = 0; s < S; ++s) {
      tp::mbar_init(&full[s], 1);
      tp::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 4; ++a) {
      tp::mbar_init(&tfull[a], 1);
      tp::mbar_init(&tempty[a], 4);
    }
    tp::mbar_init(bres_bar, 1);
    tp::fence_mbar_init();
  }
  if (warp == kMmaWarp) tp::tmem_alloc(tmem_slot, 512);
  for (int i = threadIdx.x; i < 32; i += blockDim.x) bias_s[i] = p.bias[i];
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_img = p.n_img_dev != nullptr ? min(*p.n_img_dev, p.n_img) : p.n_img;
  // input: the gather's padded expanded image (610^2); output: compact 304^2
  const int ores = p.res >> 1, oimg = ores * ores, hp = p.res + 2;
  const int txs = ores / 16, tys = ores / 8, per_img = txs * tys;  // 304 = 19*16 = 38*8
  const int total_tiles = n_img * per_img;
  const int per_cta = total_tiles / (int)gridDim.x, extra = total_tiles % (int)gridDim.x;
  const int t_begin = (int)blockIdx.x * per_cta + min((int)blockIdx.x, extra);
  const int n_tiles = per_cta + ((int)blockIdx.x < extra ? 1 : 0);

  if (warp == kProdWarp) {
    if (lane == 0) {
      if (n_tiles > 0) {
        tp::mbar_arrive_expect_tx(bres_bar, 9 * 1024);  // chunk dy*3 + variant
        for (int j = 0; j < 9; ++j) tp::tma_load_2d(smB + j * 1024, &tmB, bres_bar, j * 16, 0);
      }
      int s = 0;
      uint32_t ph = 0;
      long long pr_wait = 0;
      PROF_T0(pr_start);
      for (int i = 0; i < n_tiles; ++i) {
        const int t = t_begin + i;
        const int img = t / per_img, r = t - img * per_img;
        const int by = r / txs, bx = r - by * txs;
        PROF_T0(tw);
        tp::mbar_wait(&empty[s], ph ^ 1);
        PROF_ADD(pr_wait, tw);
        uint8_t* dst = smA + (size_t)s * L0_STAGE;
        if (p.dbg & 16) {  // profiling: no TMA, stale operands
          tp::mbar_arrive(&full[s]);
        } else {
          tp::mbar_arrive_expect_tx(&full[s], L0_STAGE);
#pragma unroll
          for (int f = 0; f < 2; ++f)  // input row phase; both column phases share the rows
            tma_load_3d(dst + f * L0_BOX_BYTES, &tmA, &full[s], 0, 16 * bx,
                        img * hp + 1 + 16 * by + f - 1);
        }
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
      if (p.dbg & 32) {
        atomicAdd(&g_conv_prof[0], (unsigned long long)(clock64() - pr_start));
        atomicAdd(&g_conv_prof[1], (unsigned long long)pr_wait);
        if (blockIdx.x == 0) atomicAdd(&g_conv_prof[7], 1ull);
      }
    }
  } else if (warp == kMmaWarp) {
    {
      if (n_tiles > 0) tp::mbar_wait(bres_bar, 0);  // weights load only if this CTA has tiles
      // A: SW64 rows of 64 B = R(k); B: SW32 rows of 32 B (K = 16)
      const uint64_t a_desc0 = tp::umma_desc(tp::smem_u32(smA), 16, 512, 4);
      const uint64_t b_desc0 = tp::umma_desc(tp::smem_u32(smB), 16, 256, 6);
      const uint32_t idesc64 = tp::idesc_f16kind(128, 64, p.f16 == 0);
      int s = 0;
      uint32_t ph = 0;
      uint32_t aph = 0;  // phase bit per accumulator buffer
      long long w_te = 0, w_fu = 0;
      PROF_T0(m_start);
      for (int i = 0; i < n_tiles; ++i) {
        const int acc = i & 3;
        PROF_T0(t1);
        tp::mbar_wait(&tempty[acc], ((aph >> acc) & 1) ^ 1);
        PROF_ADD(w_te, t1);
        aph ^= 1u << acc;
        PROF_T0(t2);
        tp::mbar_wait(&full[s], ph);
        PROF_ADD(w_fu, t2);
        tp::tc_fence_after();
        const uint64_t ad0 = a_desc0 + (uint64_t)(s * (L0_STAGE >> 4));
        const bool leader = tp::elect_one();
        if (leader && (p.dbg & 2)) {  // profiling: no MMAs
          tp::mma_commit(&empty[s]);
          tp::mma_commit(&tfull[acc]);
        } else if (leader) {
          // pool row py: accumulators (py, px=0) and (py, px=1) are adjacent TMEM column
          // blocks and both read R(k)'s first 32 bytes, with adjacent weight chunks (even,
          // odd-A) — one N=64 MMA; the odd column's second-chunk term is one N=32 MMA
#pragma unroll
          for (int py = 0; py < 2; ++py) {
            const uint32_t d = tmem_base + (uint32_t)(acc * 128 + py * 64);
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
              const int o = py + dy;  // input row offset + 1, in 0..3
              const int f = o & 1, start = o >> 1;
              const uint32_t w0 = (f * L0_BOX_BYTES + start * 16 * 64) >> 4;  // R(k) bytes 0..31: K 0..15
              const uint64_t bw = b_desc0 + (uint64_t)(dy * 3 * 64);
              tp::mma_bf16(d, ad0 + w0, bw, idesc64, dy != 0);
              tp::mma_bf16(d + 32, ad0 + w0 + 2, bw + 128, p.idesc, 1);  // R(k) bytes 32..63
            }
          }
          tp::mma_commit(&empty[s]);
          tp::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
      if ((p.dbg & 32) && lane == 0) {
        atomicAdd(&g_conv_prof[2], (unsigned long long)(clock64() - m_start));
        atomicAdd(&g_conv_prof[3], (unsigned long long)w_te);
        atomicAdd(&g_conv_prof[4], (unsigned long long)w_fu);
      }
    }
  } else {
    const int g = (int)warp >> 2;
    const float alpha = p.alpha;
    const uint32_t q = warp & 3;
    const bool f16 = p.f16 != 0;
    uint32_t ph = 0, nslab = 0;  // ph: phase bit per accumulator buffer
    long long e_wait = 0;
    PROF_T0(e_start);
    for (int i = 0; i < n_tiles; ++i) {
      if ((i & 1) != g) continue;
      const int acc = i & 3;
      const int t = t_begin + i;
      const int img = t / per_img, r = t - img * per_img;
      const int by = r / txs, bx = r - by * txs;
      PROF_T0(t3);
      tp::mbar_wait(&tfull[acc], (ph >> acc) & 1);
      PROF_ADD(e_wait, t3);
      ph ^= 1u << acc;
      tp::tc_fence_after();
      if (p.dbg & 1) {  // profiling: no epilogue work
        tp::tc_fence_before();
        __syncwarp();
        if (lane == 0) tp::mbar_arrive(&tempty[acc]);
        continue;
      }
      // split outputs: this warp's 32 pooled pixels (2 output rows x 16) are staged as 32
      // SW128 smem rows [hi 16 | lo 16] x 2 and written by one TMA store — per-thread
      // 16-byte stores at a 128-byte pixel pitch were LSU-bound (0.86 -> 0.44 ms per 120
      // tiles). Plain 64-byte pixels are stored directly (staging measured 13% slower).
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + (uint32_t)(acc * 128);
      const bool spl = p.split != 0 || p.out_lo != nullptr;  // staged TMA-store outputs
      const uint32_t slab = tp::smem_u32(smC) + warp * 8192 + (nslab & 1) * 4096;
      const int X = bx * 16 + (int)(lane & 15), Y = by * 8 + 2 * (int)q + (int)(lane >> 4);
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) +
                         (size_t)(img * oimg + Y * ores + X) * p.out_cstride;
      if (spl) {
        if (lane == 0) bulk_wait_read1();
        __syncwarp();
      }
      // TMEM loads software-pipelined: chunk 1's four loads are in flight while chunk 0 is
      // pooled, converted and staged
      uint32_t v0[16], v1[16], v2[16], v3[16];
      tp::tmem_ld16(t_row, v0);
      tp::tmem_ld16(t_row + 32, v1);
      tp::tmem_ld16(t_row + 64, v2);
      tp::tmem_ld16(t_row + 96, v3);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tp::tmem_ld_wait();
        float fv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          fv[j] = fmaxf(fmaxf(__uint_as_float(v0[j]), __uint_as_float(v1[j])),
                        fmaxf(__uint_as_float(v2[j]), __uint_as_float(v3[j])));
        if (c == 0) {
          tp::tmem_ld16(t_row + 16, v0);
          tp::tmem_ld16(t_row + 48, v1);
          tp::tmem_ld16(t_row + 80, v2);
          tp::tmem_ld16(t_row + 112, v3);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          // scale (alpha > 0), bias and leaky are monotonic: pooling first is the same value
          const float a = fmaf(fv[j], p.alpha, bias_s[c * 16 + j]);
          fv[j] = fmaxf(a, 0.1f * a);
        }
        if (p.split) {  // SW128 rows: 16-byte unit u at u ^ (row & 7)
          uint32_t hi[8], lo[8];
          split_pairs<8>(fv, hi, lo);
          const uint32_t rb = slab + lane * 128, sw = lane & 7;
          st_shared_v4(rb + (((4 * c + 0) ^ sw) << 4), hi[0], hi[1], hi[2], hi[3]);
          st_shared_v4(rb + (((4 * c + 1) ^ sw) << 4), hi[4], hi[5], hi[6], hi[7]);
          st_shared_v4(rb + (((4 * c + 2) ^ sw) << 4), lo[0], lo[1], lo[2], lo[3]);
          st_shared_v4(rb + (((4 * c + 3) ^ sw) << 4), lo[4], lo[5], lo[6], lo[7]);
          continue;
        }
        if (p.out_lo != nullptr) {  // HL8: staged hi rows (64 B, SW64) + lo rows (32 B, SW32)
          uint32_t hi[8], lo[4];
          split_hl8(fv, hi, lo);
          const uint32_t rh = slab + lane * 64, sh = (lane >> 1) & 3;
          st_shared_v4(rh + (((2 * c) ^ sh) << 4), hi[0], hi[1], hi[2], hi[3]);
          st_shared_v4(rh + (((2 * c + 1) ^ sh) << 4), hi[4], hi[5], hi[6], hi[7]);
          st_shared_v4(slab + 2048 + lane * 32 + ((c ^ ((lane >> 2) & 1)) << 4), lo[0], lo[1],
                       lo[2], lo[3]);
          continue;
        }
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float a = fv[2 * j], b = fv[2 * j + 1];
          if (f16) {
            __half2 h = __floats2half2_rn(a, b);
            pk[j] = *reinterpret_cast<uint32_t*>(&h);
          } else {
            __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
            pk[j] = *reinterpret_cast<uint32_t*>(&h);
          }
        }
        *reinterpret_cast<uint4*>(o + c * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(o + c * 16 + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      if (spl) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && (p.dbg & 4) == 0) {
          tma_store_3d(&tmC, smC + (slab - tp::smem_u32(smC)), 0, bx * 16,
                       img * ores + by * 8 + 2 * (int)q);
          if (p.out_lo != nullptr)
            tma_store_3d(&tmC2, smC + (slab + 2048 - tp::smem_u32(smC)), 0, bx * 16,
                         img * ores + by * 8 + 2 * (int)q);
          bulk_commit();
        }
        ++nslab;
      }
      tp::tc_fence_before();
      __syncwarp();
      if (lane == 0) tp::mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) bulk_wait_all();
    if ((p.dbg & 32) && warp == 0 && lane == 0) {
      atomicAdd(&g_conv_prof[5], (unsigned long long)(clock64() - e_start));
      atomicAdd(&g_conv_prof[6], (unsigned long long)e_wait);
    }
  }
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  if (warp == kMmaWarp) tp::tmem_dealloc(tmem_base, 512);
}

// ------------------------------------------------------------------ full-halo box kernel
// 3x3 convs whose input channels fit one K block (cin = BK = 32 or 64) and whose weights
// fit in shared memory (L2 32->64, L4/L6 64->128). One TMA box per output tile holds the
// tile plus its one-pixel halo; all nine taps are descriptor row offsets into that box
// (tcgen05 swizzle is computed from absolute smem address bits, so a K-major SW64/SW128
// operand may start on any 128/64-byte row and the 8-row group pitch may be any row
// count — tools/swz_shift_test.cu checks this numerically). Versus the FLAT path (A re-read
// once per tap, B once per tile) this cuts L2->SM fill traffic ~6x, which is what bounds
// these layers (the chip's L2 delivers ~42 B/clk/SM when every SM streams).
//   BOX_PLAIN / BOX_POOL: output tile 8 x 16 pixels (M = 128, row m = pixel (m%8, m/8)),
//     box {BK, 10, 18}; tap (dy,dx) starts at box row dy*10+dx, group pitch 10 rows.
//     BOX_POOL pools 2x2 in the epilogue (x pair lane^1, y pair lane^8).
//   BOX_POOLM: M rows are POOLED pixels (8 x 16 pooled = 16 x 32 conv pixels); the four
//     pool positions accumulate into four TMEM accumulators fed by four stride-2 parity
//     planes {BK, 9, 17}; the epilogue pools with a per-thread max (no shuffles).
enum BoxEpi { BOX_PLAIN = 0, BOX_POOL = 1, BOX_POOLM = 2 };
constexpr int BOX_TW = 8, BOX_TH = 16;
constexpr int PLANE_W = BOX_TW + 1, PLANE_H = BOX_TH + 1;  // 9 x 17 parity-plane rows

template <int BK, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    conv_box_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmA2,
                    const __grid_constant__ CUtensorMap tmB2, const ConvParams p) {
  constexpr uint32_t RB = BK * 2;  // bytes per pixel row in smem (one swizzle row)
  constexpr uint32_t LAY = BK == 64 ? 2 : 4;
  constexpr bool PM = EPI == BOX_POOLM;
  constexpr int NACC = PM ? 4 : 1;  // accumulators per tile
  // plain outputs leave through per-warp SW64 staging slabs + TMA bulk stores (coalesced);
  // scattered 16-byte stores at a 256-byte pixel pitch were LSU-bound
  constexpr bool TSTORE = EPI == BOX_PLAIN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* smA = smem;
  uint8_t* smB = smem + (size_t)S * p.a_stage_bytes;  // resident weights, 9 tap chunks
  uint8_t* smC = smB + p.bres_bytes;  // 1024-aligned: 8 warps x 2 KB staging (TSTORE)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smC + p.stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;   // one per accumulator buffer (<= 4)
  uint64_t* tempty = bars + 2 * S + 4;
  uint64_t* bres_bar = bars + 2 * S + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 9);
  float* bias_s = reinterpret_cast<float*>(bars + 2 * S + 10);

  const uint32_t warp = tp::warp_id();
  const uint32_t lane = tp::lane_id();
  const int N = p.bn;
  const int NB = p.nbuf;  // accumulator buffers: MMA runs up to NB-1 tiles ahead of epilogues
  if (warp == kProdWarp && lane == 0) {
    tp::tma_prefetch(&tmA);
    tp::tma_prefetch(&tmB);
    for (int s = 0; s < S; ++s) {
      tp::mbar_init(&full[s], 1);
      tp::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 4; ++a) {
      tp::mbar_init(&tfull[a], 1);
      tp::mbar_init(&tempty[a], 4);
    }
    tp::mbar_init(bres_bar, 1);
    tp::fence_mbar_init();
  }
  if (warp == kMmaWarp) tp::tmem_alloc(tmem_slot, p.tmem_cols);
  for (int i = threadIdx.x; i < N; i += blockDim.x) bias_s[i] = p.bias[i];
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_img = p.n_img_dev != nullptr ? min(*p.n_img_dev, p.n_img) : p.n_img;
  const int per_img = p.tiles_x * p.tiles_y;
  const int total_tiles = n_img * per_img;
  const int per_cta = total_tiles / (int)gridDim.x, extra = total_tiles % (int)gridDim.x;
  const int t_begin = (int)blockIdx.x * per_cta + min((int)blockIdx.x, extra);
  const int n_tiles = per_cta + ((int)blockIdx.x < extra ? 1 : 0);

  if (warp == kProdWarp) {
    if (lane == 0) {
      // ================= TMA producer: one box (or 4 parity planes) per tile =================
      if (n_tiles > 0) {
        tp::mbar_arrive_expect_tx(bres_bar, p.bres_bytes);
        for (int j = 0; j < p.n_bchunks; ++j) {  // chunk j = (K block j / 9, tap j % 9)
          const int cb = j / 9, tap = j - cb * 9;
          if (PM && p.lo_in && cb >= p.kb_hi)  // HL8: e4m3 lo chunks after the fp16 ones
            tp::tma_load_2d(smB + (size_t)9 * p.kb_hi * p.bchunk_bytes +
                                (size_t)(j - 9 * p.kb_hi) * (p.bchunk_bytes >> 1),
                            &tmB2, bres_bar, tap * p.cin, 0);
          else
            tp::tma_load_2d(smB + (size_t)j * p.bchunk_bytes, &tmB, bres_bar, tap * p.cin + cb * BK, 0);
        }
      }
      int s = 0;
      uint32_t ph = 0;
      int img = t_begin / per_img, r = t_begin - img * per_img;
      int by = r / p.tiles_x, bx = r - by * p.tiles_x;
      long long pr_wait = 0;
      PROF_T0(pr_start);
      const int nkb = PM ? p.num_kb : 1;
      for (int i = 0; i < n_tiles; ++i) {
       for (int cb = 0; cb < nkb; ++cb) {  // K blocks of the tile (PM with 64 channels: 2)
        PROF_T0(tw);
        tp::mbar_wait(&empty[s], ph ^ 1);
        PROF_ADD(pr_wait, tw);
        uint8_t* dst = smA + (size_t)s * p.a_stage_bytes;
        // exact box bytes (stages / planes are padded to 1 KB in smem); an HL8 lo block
        // (PM, cb >= kb_hi) has BK e4m3 channels: half the row bytes (SW32)
        const bool lo_blk = PM && p.lo_in && cb >= p.kb_hi;
        constexpr uint32_t tx = PM ? 4 * PLANE_W * PLANE_H * RB : (BOX_TW + 2) * (BOX_TH + 2) * RB;
        tp::mbar_arrive_expect_tx(&full[s], lo_blk ? tx / 2 : tx);
        if (PM) {
          // plane (ey, ex) holds input (2*X0 - ex + 2i, 2*Y0 - ey + 2j); -1 reads as 0
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int ey = b >> 1, ex = b & 1;
            tma_load_4d(dst + b * (p.a_stage_bytes >> 2), lo_blk ? &tmA2 : &tmA, &full[s],
                        lo_blk ? (cb - p.kb_hi) * BK : cb * BK, 2 * BOX_TW * bx - ex,
                        2 * BOX_TH * by - ey, img);
          }
        } else {  // tile + one-pixel halo; the halo outside the image reads as 0
          tma_load_4d(dst, &tmA, &full[s], 0, BOX_TW * bx - 1, BOX_TH * by - 1, img);
        }
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
       }
        if (++bx == p.tiles_x) {
          bx = 0;
          if (++by == p.tiles_y) {
            by = 0;
            ++img;
          }
        }
      }
      if (p.dbg & 32) {
        atomicAdd(&g_conv_prof[0], (unsigned long long)(clock64() - pr_start));
        atomicAdd(&g_conv_prof[1], (unsigned long long)pr_wait);
        if (blockIdx.x == 0) atomicAdd(&g_conv_prof[7], 1ull);
      }
    }
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer (warp-convergent, one elected lane) =================
    if (n_tiles > 0) tp::mbar_wait(bres_bar, 0);  // weights load only if this CTA has tiles
    constexpr uint32_t pitch = (PM ? PLANE_W : BOX_TW + 2) * RB;  // 8-row group pitch
    const uint64_t a_desc0 = tp::umma_desc(tp::smem_u32(smA), 16, pitch, LAY);
    const uint64_t b_desc_base = tp::umma_desc(tp::smem_u32(smB), 16, 8 * RB, LAY);
    const uint32_t a_step = p.a_stage_bytes >> 4, bch = p.bchunk_bytes >> 4;
    const uint32_t plane16 = (p.a_stage_bytes >> 2) >> 4;
    const uint32_t idesc = p.idesc;
    int s = 0;
    uint32_t ph = 0;
    uint32_t aph = 0;  // phase bit per accumulator buffer
    long long w_te = 0, w_fu = 0;
    PROF_T0(m_start);
    for (int i = 0; i < n_tiles; ++i) {
      const int acc = i & (NB - 1);
      PROF_T0(t1);
      tp::mbar_wait(&tempty[acc], ((aph >> acc) & 1) ^ 1);
      PROF_ADD(w_te, t1);
      aph ^= 1u << acc;
      const int nkb = PM ? p.num_kb : 1;
      for (int cb = 0; cb < nkb; ++cb) {
      PROF_T0(t2);
      tp::mbar_wait(&full[s], ph);
      PROF_ADD(w_fu, t2);
      tp::tc_fence_after();
      const uint64_t ad = a_desc0 + (uint64_t)(s * a_step);
      const uint32_t d0 = tmem_base + (uint32_t)(acc * NACC * N);
      const uint64_t b_desc0 = b_desc_base + (uint64_t)(cb * 9 * bch);  // this K block's taps
      const bool lo_blk = PM && p.lo_in && cb >= p.kb_hi;
      if (lo_blk) {
        // HL8 lo block: BK e4m3 channels = one K = 32 MMA per (tap, accumulator) from
        // BK-byte rows (SW32); weights = the e4m3 chunks after the 9 * kb_hi fp16 ones
        if (BK == 32 && tp::elect_one() && (p.dbg & 2) == 0) {
          constexpr uint32_t RBL = BK;
          const uint64_t adl = tp::umma_desc(tp::smem_u32(smA), 16, PLANE_W * RBL, 6) +
                               (uint64_t)(s * a_step);
          const uint32_t bchl = bch >> 1;
          const uint64_t bdl = tp::umma_desc(tp::smem_u32(smB), 16, 8 * RBL, 6) +
                               (uint64_t)(9 * p.kb_hi * bch + (cb - p.kb_hi) * 9 * bchl);
          const uint32_t idesc2 = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(2 * N) >> 3 << 17);
#pragma unroll
          for (int py = 0; py < 2; ++py) {
            const uint32_t dpair = d0 + (uint32_t)(2 * py * N);
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
              const int sy = py + dy;
#pragma unroll
              for (int o = 0; o < 4; ++o) {
                const int sx = o == 0 ? 1 : o == 1 ? 2 : o == 2 ? 0 : 3;
                const int plane = ((sy + 1) & 1) * 2 + ((sx + 1) & 1);
                const uint32_t off = plane * plane16 + (((sy >> 1) * PLANE_W + (sx >> 1)) * RBL >> 4);
                const int chunk = 3 * dy + (o < 2 ? sx - 1 : o == 2 ? 0 : 2);
                mma_f8(o == 2 ? dpair + (uint32_t)N : dpair, adl + off, bdl + chunk * bchl,
                       o < 2 ? idesc2 : idesc, 1);
              }
            }
          }
        }
      } else if (tp::elect_one() && (p.dbg & 2) == 0) {
        if (PM && (p.dbg & 64)) {  // profiling: unmerged pool-in-M (6 N-wide MMAs per row)
#pragma unroll
          for (int pp = 0; pp < NACC; ++pp) {
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
              const int dy = tap / 3, dx = tap % 3;
              const int sy = (pp >> 1) + dy, sx = (pp & 1) + dx;
              const int plane = ((sy + 1) & 1) * 2 + ((sx + 1) & 1);
              const uint32_t off = plane * plane16 + (((sy >> 1) * PLANE_W + (sx >> 1)) * RB >> 4);
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                tp::mma_bf16(d0 + (uint32_t)(pp * N), ad + off + 2 * k, b_desc0 + tap * bch + 2 * k,
                             idesc, (cb | tap | k) != 0);
            }
          }
        } else if (PM) {
          // The two x pool positions of a pooled row share input columns: sample column
          // sx = px + dx in {0..3}; sx = 1 and 2 serve (px 0, dx sx) and (px 1, dx sx-1)
          // with ONE A operand, so one N = 2N MMA against the adjacent weight chunks
          // [W(dy, sx-1); W(dy, sx)] fills both accumulators of the pair: columns [0, N) =
          // px 1, [N, 2N) = px 0 (the pooling epilogue takes a max over all four, so the
          // accumulator order is free). sx = 0 / 3 are single N MMAs. Per pooled row: 2
          // MMAs at N = 2N + 2 at N instead of 6 at N (N = 64: 224 vs 288 cycles).
          const uint32_t idesc2 = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(2 * N) >> 3 << 17);
#pragma unroll
          for (int py = 0; py < 2; ++py) {
            const uint32_t dpair = d0 + (uint32_t)(2 * py * N);  // [px 1 | px 0]
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
              const int sy = py + dy;
#pragma unroll
              for (int o = 0; o < 4; ++o) {
                const int sx = o == 0 ? 1 : o == 1 ? 2 : o == 2 ? 0 : 3;  // merged ones first
                const int plane = ((sy + 1) & 1) * 2 + ((sx + 1) & 1);
                const uint32_t off = plane * plane16 + (((sy >> 1) * PLANE_W + (sx >> 1)) * RB >> 4);
                // weights: merged -> chunks (dy, sx-1), (dy, sx); sx = 0 -> (dy, 0) into
                // px 0; sx = 3 -> (dy, 2) into px 1
                const int chunk = 3 * dy + (o < 2 ? sx - 1 : o == 2 ? 0 : 2);
                const uint32_t d = o == 2 ? dpair + (uint32_t)N : dpair;
                const uint32_t id = o < 2 ? idesc2 : idesc;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                  tp::mma_bf16(d, ad + off + 2 * k, b_desc0 + chunk * bch + 2 * k, id,
                               (cb | dy | o | k) != 0);
              }
            }
          }
        } else {
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const int dy = tap / 3, dx = tap % 3;
            const uint32_t off = (dy * (BOX_TW + 2) + dx) * RB >> 4;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tp::mma_bf16(d0, ad + off + 2 * k, b_desc0 + tap * bch + 2 * k, idesc, (tap | k) != 0);
          }
        }
      }
      if (tp::elect_one()) {
        tp::mma_commit(&empty[s]);
        if (cb == nkb - 1) tp::mma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
      }  // K blocks
    }
    if ((p.dbg & 32) && lane == 0) {
      atomicAdd(&g_conv_prof[2], (unsigned long long)(clock64() - m_start));
      atomicAdd(&g_conv_prof[3], (unsigned long long)w_te);
      atomicAdd(&g_conv_prof[4], (unsigned long long)w_fu);
    }
  } else {
    // ================= epilogue: two warpgroups alternate accumulators =================
    const int g = (int)warp >> 2;
    const float alpha = p.alpha;
    const uint32_t q = warp & 3;
    const int row = (int)(q * 32 + lane);
    const bool f16 = p.f16 != 0;
    const bool leaky = p.leaky != 0;
    const int ores = PM || EPI == BOX_POOL ? p.res >> 1 : p.res;
    const int oimg = ores * ores;
    const int nchunks = N >> 4;
    uint32_t ph = 0;  // phase bit per accumulator buffer
    uint32_t slab = 0;  // TSTORE staging slabs used by this warp
    int img = t_begin / per_img, r = t_begin - img * per_img;
    int by = r / p.tiles_x, bx = r - by * p.tiles_x;
    long long e_wait = 0;
    PROF_T0(e_start);
    for (int i = 0; i < n_tiles; ++i) {
      const int timg = img, tby = by, tbx = bx;
      if (++bx == p.tiles_x) {
        bx = 0;
        if (++by == p.tiles_y) {
          by = 0;
          ++img;
        }
      }
      if ((i & 1) != g) continue;
      const int acc = i & (NB - 1);
      PROF_T0(t3);
      tp::mbar_wait(&tfull[acc], (ph >> acc) & 1);
      PROF_ADD(e_wait, t3);
      ph ^= 1u << acc;
      tp::tc_fence_after();
      if (p.dbg & 1) {
        tp::tc_fence_before();
        __syncwarp();
        if (lane == 0) tp::mbar_arrive(&tempty[acc]);
        continue;
      }
      // this thread's pixel (conv output, or pooled output for POOLM)
      const int x = tbx * BOX_TW + (row & 7), y = tby * BOX_TH + (row >> 3);
      bool store;
      int opx;
      if (EPI == BOX_POOL) {  // both lanes of an x pair store (8 channels each)
        store = y < p.res && (y & 1) == 0;
        opx = timg * oimg + (y >> 1) * ores + (x >> 1);
      } else {
        store = y < ores;
        opx = timg * oimg + y * ores + x;
      }
      __nv_bfloat16* o =
          reinterpret_cast<__nv_bfloat16*>(p.out) + (size_t)opx * p.out_cstride + p.out_coff;
      // TSTORE: this warp's 32 pixels are 4 full rows of 8 (res % 4 == 0), all valid or not
      const bool warp_rows_valid = tby * BOX_TH + (int)q * 4 < p.res;
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + (uint32_t)(acc * NACC * N);
      // TMEM loads are software-pipelined: chunk c+1 is in flight while chunk c is
      // converted and stored (its registers are copied out before the next load).
      uint32_t v0[16], v1[16], v2[16], v3[16];
      tp::tmem_ld16(t_row, v0);
      if (PM) {
        tp::tmem_ld16(t_row + N, v1);
        tp::tmem_ld16(t_row + 2 * N, v2);
        tp::tmem_ld16(t_row + 3 * N, v3);
      }
      for (int c = 0; c < nchunks; ++c) {
        float f[16];
        tp::tmem_ld_wait();
        if (PM) {
          // bias + leaky are monotonic, so pooling first gives the same value
#pragma unroll
          for (int j = 0; j < 16; ++j)
            f[j] = fmaxf(fmaxf(__uint_as_float(v0[j]), __uint_as_float(v1[j])),
                         fmaxf(__uint_as_float(v2[j]), __uint_as_float(v3[j])));
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v0[j]);
        }
        if (c + 1 < nchunks) {
          const uint32_t tc = t_row + (uint32_t)((c + 1) * 16);
          tp::tmem_ld16(tc, v0);
          if (PM) {
            tp::tmem_ld16(tc + N, v1);
            tp::tmem_ld16(tc + 2 * N, v2);
            tp::tmem_ld16(tc + 3 * N, v3);
          }
        }
        if (EPI == BOX_POOL) {
          // 2x2 pool BEFORE bias + leaky (both monotonic: same value). After the x-pair
          // exchange (lane^1) the even lane keeps channels 0-7 and the odd lane 8-15, so
          // the y exchange (lane^8), bias, leaky, pack and store handle 8 values per lane.
          const bool odd = (lane & 1) != 0;
          float h8[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float send = odd ? f[j] : f[j + 8];
            const float mine = odd ? f[j + 8] : f[j];
            h8[j] = fmaxf(mine, __shfl_xor_sync(0xffffffffu, send, 1));
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) h8[j] = fmaxf(h8[j], __shfl_xor_sync(0xffffffffu, h8[j], 8));
          const int ch = c * 16 + (odd ? 8 : 0);
          const float4 b0 = *reinterpret_cast<const float4*>(bias_s + ch);
          const float4 b1 = *reinterpret_cast<const float4*>(bias_s + ch + 4);
          h8[0] = fmaf(h8[0], alpha, b0.x);
          h8[1] = fmaf(h8[1], alpha, b0.y);
          h8[2] = fmaf(h8[2], alpha, b0.z);
          h8[3] = fmaf(h8[3], alpha, b0.w);
          h8[4] = fmaf(h8[4], alpha, b1.x);
          h8[5] = fmaf(h8[5], alpha, b1.y);
          h8[6] = fmaf(h8[6], alpha, b1.z);
          h8[7] = fmaf(h8[7], alpha, b1.w);
          if (leaky) {
#pragma unroll
            for (int j = 0; j < 8; ++j) h8[j] = fmaxf(h8[j], 0.1f * h8[j]);
          }
          if (!store || ch >= p.cout || (p.dbg & 4)) continue;
          if (p.split) {
            uint32_t hi[4], lo[4];
            split_pairs<4>(h8, hi, lo);
            __nv_bfloat16* os = o + 2 * c * 16 + (odd ? 8 : 0);
            *reinterpret_cast<uint4*>(os) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            *reinterpret_cast<uint4*>(os + 16) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            continue;
          }
          uint32_t pk[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (f16) {
              __half2 h = __floats2half2_rn(h8[2 * j], h8[2 * j + 1]);
              pk[j] = *reinterpret_cast<uint32_t*>(&h);
            } else {
              __nv_bfloat162 h = __floats2bfloat162_rn(h8[2 * j], h8[2 * j + 1]);
              pk[j] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
          *reinterpret_cast<uint4*>(o + ch) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          continue;
        }
        const float4* b4 = reinterpret_cast<const float4*>(bias_s + c * 16);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 bb = b4[j];
          f[4 * j + 0] = fmaf(f[4 * j + 0], alpha, bb.x);
          f[4 * j + 1] = fmaf(f[4 * j + 1], alpha, bb.y);
          f[4 * j + 2] = fmaf(f[4 * j + 2], alpha, bb.z);
          f[4 * j + 3] = fmaf(f[4 * j + 3], alpha, bb.w);
        }
        if (leaky) {
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.1f * f[j]);
        }
        if (TSTORE) {
          if (!warp_rows_valid) continue;
          const bool spl = p.split != 0;  // split: one slab ([hi 16 | lo 16]) per chunk
          const int cs = spl ? 0 : (c & 1);
          const uint32_t slab_off = warp * 4096 + (slab & 1) * 2048;  // two alternating slabs
          const uint32_t buf = tp::smem_u32(smC) + slab_off;
          if (cs == 0) {
            if (lane == 0) bulk_wait_read1();
            __syncwarp();
          }
          if (spl) {
            uint32_t hi[8], lo[8];
            split_pairs<8>(f, hi, lo);
            const uint32_t rbase = buf + lane * 64, swz = (lane >> 1) & 3;
            st_shared_v4(rbase + ((0 ^ swz) << 4), hi[0], hi[1], hi[2], hi[3]);
            st_shared_v4(rbase + ((1 ^ swz) << 4), hi[4], hi[5], hi[6], hi[7]);
            st_shared_v4(rbase + ((2 ^ swz) << 4), lo[0], lo[1], lo[2], lo[3]);
            st_shared_v4(rbase + ((3 ^ swz) << 4), lo[4], lo[5], lo[6], lo[7]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && (p.dbg & 4) == 0) {
              tma_store_3d(&tmC, smC + slab_off, p.out_coff + 2 * c * 16, tbx * BOX_TW,
                           timg * p.res + tby * BOX_TH + (int)q * 4);
              bulk_commit();
            }
            ++slab;
            continue;
          }
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (f16) {
              __half2 h = __floats2half2_rn(f[2 * j], f[2 * j + 1]);
              pk[j] = *reinterpret_cast<uint32_t*>(&h);
            } else {
              __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
              pk[j] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
          const uint32_t rbase = buf + lane * 64, swz = (lane >> 1) & 3;
          st_shared_v4(rbase + (((2 * cs) ^ swz) << 4), pk[0], pk[1], pk[2], pk[3]);
          st_shared_v4(rbase + (((2 * cs + 1) ^ swz) << 4), pk[4], pk[5], pk[6], pk[7]);
          if (cs == 1) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && (p.dbg & 4) == 0) {
              tma_store_3d(&tmC, smC + slab_off, p.out_coff + (c - 1) * 16, tbx * BOX_TW,
                           timg * p.res + tby * BOX_TH + (int)q * 4);
              bulk_commit();
            }
            ++slab;
          }
          continue;
        }
        if (!store || c * 16 >= p.cout || (p.dbg & 4)) continue;
        if (p.out_lo != nullptr) {  // HL8 planes
          const size_t oo = (size_t)opx * p.out_cstride + p.out_coff + c * 16;
          store_hl8(reinterpret_cast<__half*>(p.out) + oo, reinterpret_cast<uint8_t*>(p.out_lo) + oo, f);
          continue;
        }
        if (p.split) {
          store_split16(o + 2 * c * 16, f);
          continue;
        }
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (f16) {
            __half2 h = __floats2half2_rn(f[2 * j], f[2 * j + 1]);
            pk[j] = *reinterpret_cast<uint32_t*>(&h);
          } else {
            __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
            pk[j] = *reinterpret_cast<uint32_t*>(&h);
          }
        }
        *reinterpret_cast<uint4*>(o + c * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(o + c * 16 + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      tp::tc_fence_before();
      __syncwarp();
      if (lane == 0) tp::mbar_arrive(&tempty[acc]);
    }
    if (TSTORE && lane == 0) bulk_wait_all();
    if ((p.dbg & 32) && warp == 0 && lane == 0) {
      atomicAdd(&g_conv_prof[5], (unsigned long long)(clock64() - e_start));
      atomicAdd(&g_conv_prof[6], (unsigned long long)e_wait);
    }
  }
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  if (warp == kMmaWarp) tp::tmem_dealloc(tmem_base, p.tmem_cols);
}

// 2x2/2 max pool, padded NHWC 16-bit -> padded NHWC (interior only), 8 channels/thread.
__global__ void maxpool2_kernel(const __nv_bfloat16* __restrict__ in, int n_img, int res,
                                int cstride, __nv_bfloat16* __restrict__ out,
                                const int32_t* __restrict__ n_img_dev, int f16) {
  if (n_img_dev != nullptr) n_img = min(n_img, *n_img_dev);
  const int ores = res >> 1;
  const int cg = cstride >> 3;
  const long long total = (long long)n_img * ores * ores * cg;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(i % cg);
    long long r = i / cg;
    const int x = (int)(r % ores);
    r /= ores;
    const int y = (int)(r % ores);
    const int img = (int)(r / ores);
    const __nv_bfloat16* src =
        in + (((long long)img * res + 2 * y) * res + 2 * x) * cstride + g * 8;
    uint4 a = *reinterpret_cast<const uint4*>(src);
    uint4 b = *reinterpret_cast<const uint4*>(src + cstride);
    uint4 c = *reinterpret_cast<const uint4*>(src + (long long)res * cstride);
    uint4 d = *reinterpret_cast<const uint4*>(src + (long long)res * cstride + cstride);
    uint4 m;
    if (f16) {
      const __half2* pa = reinterpret_cast<const __half2*>(&a);
      const __half2* pb = reinterpret_cast<const __half2*>(&b);
      const __half2* pc = reinterpret_cast<const __half2*>(&c);
      const __half2* pd = reinterpret_cast<const __half2*>(&d);
      __half2* pm = reinterpret_cast<__half2*>(&m);
#pragma unroll
      for (int j = 0; j < 4; ++j) pm[j] = __hmax2(__hmax2(pa[j], pb[j]), __hmax2(pc[j], pd[j]));
    } else {
      const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
      const __nv_bfloat162* pc = reinterpret_cast<const __nv_bfloat162*>(&c);
      const __nv_bfloat162* pd = reinterpret_cast<const __nv_bfloat162*>(&d);
      __nv_bfloat162* pm = reinterpret_cast<__nv_bfloat162*>(&m);
#pragma unroll
      for (int j = 0; j < 4; ++j) pm[j] = __hmax2(__hmax2(pa[j], pb[j]), __hmax2(pc[j], pd[j]));
    }
    __nv_bfloat16* dst = out + (((long long)img * ores + y) * ores + x) * cstride + g * 8;
    *reinterpret_cast<uint4*>(dst) = m;
  }
}

// 2x2/2 max pool of a split (hi/lo interleaved) tensor: each thread pools 8 channels,
// comparing the exact fp32 values hi + lo (exact: |lo| <= ulp(hi) / 2), and re-splits.
__global__ void maxpool2_split_kernel(const __half* __restrict__ in, int n_img, int res,
                                      int cstride, __half* __restrict__ out,
                                      const int32_t* __restrict__ n_img_dev) {
  if (n_img_dev != nullptr) n_img = min(n_img, *n_img_dev);
  const int ores = res >> 1;
  const int cg = cstride >> 4;  // 8-channel hi blocks: two per 32-channel group
  const long long total = (long long)n_img * ores * ores * cg;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(i % cg);
    long long r = i / cg;
    const int x = (int)(r % ores);
    r /= ores;
    const int y = (int)(r % ores);
    const int img = (int)(r / ores);
    const int coff = (g >> 1) * 32 + (g & 1) * 8;
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const __half* src = in + (((long long)img * res + 2 * y + (k >> 1)) * res + 2 * x + (k & 1)) *
                                   cstride + coff;
      const uint4 h = *reinterpret_cast<const uint4*>(src);
      const uint4 l = *reinterpret_cast<const uint4*>(src + 16);
      const __half2* ph = reinterpret_cast<const __half2*>(&h);
      const __half2* pl = reinterpret_cast<const __half2*>(&l);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 a = __half22float2(ph[j]), b = __half22float2(pl[j]);
        m[2 * j] = fmaxf(m[2 * j], a.x + b.x);
        m[2 * j + 1] = fmaxf(m[2 * j + 1], a.y + b.y);
      }
    }
    uint32_t hi[4], lo[4];
    split_pairs<4>(m, hi, lo);
    __half* dst = out + (((long long)img * ores + y) * ores + x) * cstride + coff;
    *reinterpret_cast<uint4*>(dst) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(dst + 16) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

// 2x2/2 max pool of an HL8 tensor (hi fp16 plane + e4m3 lo plane, same indexing): each
// thread pools 8 channels by their values hi + lo * 2^-TP_LO_EXP and copies the winning
// pixel's hi and lo codes (ties keep the first: the values are equal).
__device__ __forceinline__ float2 e4m3x2_to_float2(uint16_t v) {
  uint32_t h2;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(v));
  return __half22float2(*reinterpret_cast<__half2*>(&h2));
}
__global__ void maxpool2_hl8_kernel(const __half* __restrict__ in, const uint8_t* __restrict__ in_lo,
                                    int n_img, int res, int cstride, __half* __restrict__ out,
                                    uint8_t* __restrict__ out_lo,
                                    const int32_t* __restrict__ n_img_dev) {
  // one block row per output row (blockIdx.y = image * ores + y): 32-bit index math only
  // (the 64-bit grid-stride divisions of a flat index cost more than the pool itself)
  if (n_img_dev != nullptr) n_img = min(n_img, *n_img_dev);
  const int ores = res >> 1;
  const int cg = cstride >> 3;
  const int img = (int)blockIdx.y / ores, y = (int)blockIdx.y - img * ores;
  const int t = (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (img >= n_img || t >= ores * cg) return;
  {
    const int x = t / cg, g = t - x * cg;
    float best[8];
    uint16_t bh[8];
    uint8_t bl[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const long long e = (((long long)img * res + 2 * y + (k >> 1)) * res + 2 * x + (k & 1)) *
                              cstride + g * 8;
      const uint4 h = *reinterpret_cast<const uint4*>(in + e);
      const uint2 l = *reinterpret_cast<const uint2*>(in_lo + e);
      const uint16_t* hs = reinterpret_cast<const uint16_t*>(&h);
      const uint8_t* ls = reinterpret_cast<const uint8_t*>(&l);
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(hs + j));
        const float2 lf = e4m3x2_to_float2((uint16_t)(ls[j] | (ls[j + 1] << 8)));
        const float v0 = hf.x + lf.x * (1.0f / kLoScale), v1 = hf.y + lf.y * (1.0f / kLoScale);
        if (k == 0 || v0 > best[j]) {
          best[j] = v0;
          bh[j] = hs[j];
          bl[j] = ls[j];
        }
        if (k == 0 || v1 > best[j + 1]) {
          best[j + 1] = v1;
          bh[j + 1] = hs[j + 1];
          bl[j + 1] = ls[j + 1];
        }
      }
    }
    const long long o = (((long long)img * ores + y) * ores + x) * cstride + g * 8;
    uint4 ho;
    uint2 lo;
    uint16_t* hp = reinterpret_cast<uint16_t*>(&ho);
    uint8_t* lp = reinterpret_cast<uint8_t*>(&lo);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      hp[j] = bh[j];
      lp[j] = bl[j];
    }
    *reinterpret_cast<uint4*>(out + o) = ho;
    *reinterpret_cast<uint2*>(out_lo + o) = lo;
  }
}

// Darknet reorg as a gather (the YOLO plan's layer 26): layer 26 writes its plain
// [n][R][R][cin] output to a scratch buffer (TMA-store epilogue, L2-resident), then each
// thread builds 8 consecutive channels of one output pixel of [n][R/2][R/2][4 cin] from their
// sources (the inverse of reorg_dest: output (C, Y, X) at NCHW flat P reads input flat
// Q = w2 + 2R h2 + 4R^2 c2 with i = P % R, j = (P / R) % R, k = P / R^2, c2 = k % (cin/4),
// off = k / (cin/4), w2 = 2i + off % 2, h2 = 2j + off / 2) and stores them as one run —
// the scatter epilogue's 2-byte stores to 4 pixels per source pixel were LSU-bound.
// fmt: 0 plain 16-bit, 1 X2 (hi/lo interleaved per 16 channels), 2 HL8 (+ lo planes).
template <int R, int cin>  // compile-time sides: the index math is multiply-shift only
__global__ void reorg_gather_kernel(const uint16_t* __restrict__ in, const uint8_t* __restrict__ in_lo,
                                    int n_img, const int32_t* __restrict__ n_img_dev,
                                    int in_cstride, uint16_t* __restrict__ out,
                                    uint8_t* __restrict__ out_lo, int out_cstride, int fmt) {
  if (n_img_dev != nullptr) n_img = min(n_img, *n_img_dev);
  constexpr int hr = R >> 1, cout = 4 * cin, groups = cout >> 3;
  const long long total = (long long)n_img * hr * hr * groups;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(t % groups);
    const long long px = t / groups;  // output pixel: img * hr^2 + Y * hr + X
    const int img = (int)(px / (hr * hr));
    const int yx = (int)(px - (long long)img * hr * hr);
    uint32_t h[8], l[8];  // 16-bit codes (lo: e4m3 bytes for HL8)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int C = 8 * g + e;
      const int P = yx + hr * hr * C;
      const int i = P % R, j = (P / R) % R, k = P / (R * R);
      constexpr int q4 = cin >> 2;
      const int c2 = k % q4, off = k / q4;
      const int Q = (2 * i + (off & 1)) + 2 * R * (2 * j + (off >> 1)) + 4 * R * R * c2;
      const int ci = Q / (R * R), yi = (Q / R) % R, xi = Q % R;
      const size_t src = ((size_t)img * R * R + (size_t)yi * R + xi) * in_cstride;
      if (fmt == 1) {
        h[e] = in[src + 32 * (ci >> 4) + (ci & 15)];
        l[e] = in[src + 32 * (ci >> 4) + (ci & 15) + 16];
      } else {
        h[e] = in[src + ci];
        l[e] = fmt == 2 ? in_lo[src + ci] : 0;
      }
    }
    const size_t dst = (size_t)px * out_cstride;
    if (fmt == 1) {  // hi and lo 8-runs of the interleaved group
      const int c0 = 8 * g, so = 32 * (c0 >> 4) + (c0 & 15);
      *reinterpret_cast<uint4*>(out + dst + so) =
          make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
      *reinterpret_cast<uint4*>(out + dst + so + 16) =
          make_uint4(l[0] | (l[1] << 16), l[2] | (l[3] << 16), l[4] | (l[5] << 16), l[6] | (l[7] << 16));
    } else {
      *reinterpret_cast<uint4*>(out + dst + 8 * g) =
          make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
      if (fmt == 2)
        *reinterpret_cast<uint2*>(out_lo + dst + 8 * g) =
            make_uint2(l[0] | (l[1] << 8) | (l[2] << 16) | (l[3] << 24),
                       l[4] | (l[5] << 8) | (l[6] << 16) | (l[7] << 24));
    }
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                   cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn get_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(ptr);
  }
  return fn;
}

// im2col map over a compact NHWC activation {cstride, res, res, n}: `pixels` consecutive
// output pixels x `bk` channels per load; window corner `lo` (-1 = 3x3 with zero padding,
// 0 = 1x1). Out-of-bounds taps are zero-filled.
int make_tmap_im2col(CUtensorMap* tm, const void* base, int cstride, int res, int n, int bk,
                     int pixels, int lo, CUtensorMapSwizzle swz, bool f16, int esize = 2) {
  EncodeIm2colFn enc = get_im2col_fn();
  if (enc == nullptr) {
    tp_set_error("cuTensorMapEncodeIm2col unavailable (no CUDA driver?)");
    return TP_ERR_CUDA;
  }
  const cuuint64_t dims[4] = {(cuuint64_t)cstride, (cuuint64_t)res, (cuuint64_t)res,
                              (cuuint64_t)n};
  const cuuint64_t strides[3] = {(cuuint64_t)cstride * esize, (cuuint64_t)cstride * esize * res,
                                 (cuuint64_t)cstride * esize * res * res};
  const int lower[2] = {lo, lo}, upper[2] = {lo, lo};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUtensorMapDataType dt = esize == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : f16      ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                            : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUresult r = enc(tm, dt, 4,
                   const_cast<void*>(base), dims, strides, lower, upper, (cuuint32_t)bk,
                   (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    tp_set_error("cuTensorMapEncodeIm2col failed (%d): cstride %d res %d n %d", (int)r, cstride,
                 res, n);
    return TP_ERR_CUDA;
  }
  return TP_OK;
}

// rank-2..4 tiled tensor map, dims[0] contiguous (e.g. {C, W, H, N} for NHWC activations).
// esize 2 = 16-bit (f16 selects fp16 vs bf16), 4 = fp32. Out-of-bounds reads are zero.
int make_tmap(CUtensorMap* tm, const void* base, int rank, const uint64_t* dims,
              const uint32_t* box, CUtensorMapSwizzle swz, bool f16, int esize = 2,
              const uint32_t* elem_strides = nullptr,
              const cuuint64_t* byte_strides = nullptr) {  // default: dense
  EncodeTiledFn enc = get_encode_fn();
  if (enc == nullptr) {
    tp_set_error("cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
    return TP_ERR_CUDA;
  }
  cuuint64_t gdims[4], strides[3];
  cuuint32_t gbox[4], estr[4] = {1, 1, 1, 1};
  uint64_t stride = dims[0] * esize;
  for (int i = 0; i < rank; ++i) {
    gdims[i] = dims[i];
    gbox[i] = box[i];
    if (elem_strides != nullptr) estr[i] = elem_strides[i];
    if (i > 0) {
      strides[i - 1] = byte_strides != nullptr ? byte_strides[i - 1] : stride;
      stride *= dims[i];
    }
  }
  const CUtensorMapDataType dt = esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : esize == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : f16       ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUresult r = enc(tm, dt,
                   rank, const_cast<void*>(base), gdims, strides, gbox, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    tp_set_error("cuTensorMapEncodeTiled failed (%d): rank %d dims %llu,%llu box %u,%u", (int)r,
                 rank, (unsigned long long)dims[0], (unsigned long long)dims[1], box[0], box[1]);
    return TP_ERR_CUDA;
  }
  return TP_OK;
}

// SM count of the current device (cached per device: a process may drive several GPUs)
int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// The 227 KB dynamic-smem opt-in is a per-device function attribute: set it once per
// (kernel, device), thread-safely (kernels of one signature share a template
// instantiation here, so the record is keyed by the kernel's address).
template <typename Kernel>
int ensure_smem_optin(Kernel kernel) {
  static std::mutex mu;
  static std::unordered_map<const void*, uint64_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  const void* key = reinterpret_cast<const void*>(kernel);
  std::lock_guard<std::mutex> lock(mu);
  uint64_t& mask = done[key];
  if (!(mask & bit)) {
    TP_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    mask |= bit;
  }
  return TP_OK;
}

// A fully prepared layer launch (tensor maps encoded once).
struct ConvLaunch {
  int mode;
  int pair;  // CTA-pair (cta_group::2) kernel
  int l0;    // layer-0 pool-in-M kernel
  int box;   // full-halo box kernel: 0 off, else 1 + BoxEpi
  int prect; // CTA-pair pooled 3x3 kernel (conv_pair_rect_kernel)
  int swap;  // swapped-operand 3x3 kernel for 128 output channels (conv_swap_kernel)
  int box_bk;
  CUtensorMap tmA, tmB, tmC;
  CUtensorMap tmA2, tmB2;  // HL8 input: lo-plane activations and e4m3 weights
  CUtensorMap tmC2;        // swap kernel HL8 output: lo-plane store map
  ConvParams p;
  size_t smem;
};

// Activations are compact NHWC [n][res][res][cin_stride] (the conv's zero padding comes
// from TMA out-of-bounds fill), except layer 0 (cin_used == 16): its input is the gather's
// padded, horizontally expanded [n][res+2][res+2][16] image, and it must pool.
// pool != 0 fuses the 2x2 max pool; `out` is then the half-resolution buffer.
int prepare_conv(ConvLaunch* L, const void* in, int max_img, int res, int cin_stride, int cin_used,
                 const void* weight, const float* bias, int cout, int cout_pad, int ksize,
                 int leaky, void* out, int out_cstride, int out_coff, int out_fp32, int reorg,
                 int dtype, int pool, float alpha = 1.0f, const void* in_lo = nullptr,
                 const void* weight_lo = nullptr, void* out_lo = nullptr) {
  memset(L, 0, sizeof(*L));
  if (out_lo != nullptr && (dtype != TP_DTYPE_F16 || out_fp32)) {
    tp_set_error("conv: an HL8 output is an fp16 hi plane (dtype F16) + lo plane");
    return TP_ERR_ARG;
  }
  const bool f16 = dtype != TP_DTYPE_BF16;
  // TP_DTYPE_F16X2: split (hi/lo) 16-bit outputs; the fp32 head output stays fp32
  const int split = dtype == TP_DTYPE_F16X2 && !out_fp32 ? 1 : 0;
  if (cout_pad % 32 != 0 || cout > cout_pad) {
    tp_set_error("conv: bad cout/cout_pad %d/%d (cout_pad must be a multiple of 32)", cout,
                 cout_pad);
    return TP_ERR_ARG;
  }
  if (pool && (res % 2 != 0 || reorg || out_fp32)) {
    tp_set_error("conv: fused pool needs an even side and a 16-bit plain output");
    return TP_ERR_ARG;
  }
  if (!out_fp32 && (cout % 16 != 0 || out_cstride % 8 != 0 || out_coff % 8 != 0)) {
    tp_set_error("conv: 16-bit output needs 16-channel multiples");
    return TP_ERR_ARG;
  }
  if (cout_pad > kMaxBias) {
    tp_set_error("conv: cout_pad %d exceeds %d", cout_pad, kMaxBias);
    return TP_ERR_UNSUPPORTED;
  }
  const int img_px = res * res;
  if ((long long)max_img * (res + 2) * (res + 2) >= (1ll << 31)) {
    tp_set_error("conv: %d images of side %d exceed 32-bit pixel indexing", max_img, res);
    return TP_ERR_CAPACITY;
  }
  ConvParams& p = L->p;
  p.n_img = max_img;
  p.res = res;
  p.img_px = img_px;
  p.ksize = ksize;
  p.cin = cin_used;
  p.cout = cout;
  p.f16 = f16 ? 1 : 0;
  p.bias = bias;
  p.out = out;
  p.out_cstride = out_cstride;
  p.out_coff = out_coff;
  p.out_fp32 = out_fp32;
  p.leaky = leaky;
  p.reorg = reorg;
  p.split = split;
  p.alpha = alpha;
  p.out_lo = out_lo;
  p.dbg = getenv("TP_CONV_DEBUG") ? atoi(getenv("TP_CONV_DEBUG")) : 0;
  // everything else in smem: 1 KB alignment slack, bias, barriers (<= 12 stages), TMEM slot
  const int fixed = 1024 + cout_pad * 4 + (2 * 12 + 6) * 8 + 16;
  int rc;

  if (cin_used == 16) {  // layer 0: pool-in-M kernel with stride-2 TMA boxes
    if (!(ksize == 3 && pool && cout_pad == 32 && cout == 32 && res % 32 == 0)) {
      tp_set_error("conv: the 16-channel expanded input needs 3x3, 32 outputs, fused pool, "
                   "side %% 32 == 0");
      return TP_ERR_UNSUPPORTED;
    }
    const int hp = res + 2, xp = res + 6;
    {
      // 8-byte pixels P(c) = rgb0 of tile column c - 2 (rows padded by 1, columns by 2|4);
      // the kernel reads 64-byte rows [P(2k) .. P(2k+7)] = tile columns 2k-2 .. 2k+5
      // through a {32 halves, k (16 B apart: rows overlap), row} view with the SW64
      // swizzle (tools/tma_overlap_probe.cu)
      const uint64_t dims[3] = {32, (uint64_t)((xp - 8) / 2 + 1), (uint64_t)max_img * hp};
      const cuuint64_t strides[2] = {16, (cuuint64_t)xp * 8};
      const uint32_t box[3] = {32, 16, 18};
      const uint32_t estr[3] = {1, 1, 2};
      rc = make_tmap(&L->tmA, in, 3, dims, box, CU_TENSOR_MAP_SWIZZLE_64B, f16, 2, estr,
                     strides);
      if (rc) return rc;
    }
    {  // weights [32][144]: per kernel row dy, variants (even, odd first, odd second) x K 16
      const uint64_t dims[2] = {144, 32};
      const uint32_t box[2] = {16, 32};
      rc = make_tmap(&L->tmB, weight, 2, dims, box, CU_TENSOR_MAP_SWIZZLE_32B, f16);
      if (rc) return rc;
    }
    {  // output store map {stored channels, X, image rows}: box = one warp's 2 rows x 16 px
      const int ores = res / 2;
      const uint64_t dims[3] = {(uint64_t)out_cstride, (uint64_t)ores, (uint64_t)max_img * ores};
      const uint32_t box[3] = {(uint32_t)out_cstride, 16, 2};
      if (out_cstride != (split ? 64 : 32) || out_coff != 0) {
        tp_set_error("conv: layer 0 writes a dense [n][res/2][res/2][%d] output", split ? 64 : 32);
        return TP_ERR_UNSUPPORTED;
      }
      rc = make_tmap(&L->tmC, out, 3, dims, box,
                     split ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, f16);
      if (rc) return rc;
      if (out_lo != nullptr) {  // HL8 lo plane: 32-byte rows
        rc = make_tmap(&L->tmC2, out_lo, 3, dims, box, CU_TENSOR_MAP_SWIZZLE_32B, f16, 1);
        if (rc) return rc;
      }
    }
    L->l0 = 1;
    int st = (int)((227 * 1024 - fixed - 9 * 1024 - L0_STAGING) / L0_STAGE);
    if (st > 8) st = 8;
    p.stages = st;
    p.bn = 32;
    p.n_blocks_n = 1;
    p.idesc = tp::idesc_f16kind(128, 32, !f16);
    L->smem = 1024 + (size_t)st * L0_STAGE + 9 * 1024 + L0_STAGING + (2 * st + 10) * 8 + 32 * 4 + 16;
    return TP_OK;
  }

  int mode, bk;
  if (cin_used % 64 == 0) {
    mode = MODE_SW128;
    bk = 64;
  } else if (cin_used == 32) {
    mode = MODE_SW64;
    bk = 32;
  } else {
    tp_set_error("conv: unsupported cin %d", cin_used);
    return TP_ERR_UNSUPPORTED;
  }
  int bn = cout_pad;
  if (bn > 256) {
    bn = 256;
    while (cout_pad % bn != 0 || bn % 32 != 0) bn -= 32;
  }
  const int taps = ksize * ksize;
  const int ktotal = taps * cin_used;
  CUtensorMapSwizzle swz =
      mode == MODE_SW128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  // halo variant: weights (whole K x N) fit next to the A ring -> resident in smem
  const size_t bres = (size_t)cout_pad * ktotal * 2;
  const bool halo = pool && ksize == 3 && cout_pad <= 256 && bres <= 48 * 1024;
  // super-tile height: SUB x 8 rows per halo box (fewer, larger tiles for the 32/64-channel
  // layers whose per-tile fixed costs dominate); keep SUB x BN <= 256 TMEM columns
  int subt = 1;
  if (halo) {
    subt = 2;
    while (subt > 1 && (subt * cout_pad > 256 || res % (RECT_H * subt) != 0)) subt >>= 1;
  }
  if (pool) {  // RECT tiles: 4-D boxes {C, 16, rows, 1}, image borders zero-filled
    const uint64_t dims[4] = {(uint64_t)cin_stride, (uint64_t)res, (uint64_t)res,
                              (uint64_t)max_img};
    const uint32_t box[4] = {(uint32_t)bk, RECT_W,
                             halo ? (uint32_t)(RECT_H * subt + 2) : (uint32_t)RECT_H, 1};
    rc = make_tmap(&L->tmA, in, 4, dims, box, swz, f16);
  } else {  // FLAT tiles: im2col over 128 consecutive compact pixels
    rc = make_tmap_im2col(&L->tmA, in, cin_stride, res, max_img, bk, 128, ksize == 3 ? -1 : 0,
                          swz, f16);
  }
  if (rc) return rc;
  {
    const uint64_t dims[2] = {(uint64_t)ktotal, (uint64_t)cout_pad};
    const uint32_t box[2] = {(uint32_t)bk, (uint32_t)bn};
    rc = make_tmap(&L->tmB, weight, 2, dims, box, swz, f16);
  }
  if (rc) return rc;
  const bool tstore = !pool && !reorg;
  if (tstore) {  // output store tensor map: {cstride, rows}, box {64 B of channels, 32 rows}
    const uint64_t dims[2] = {(uint64_t)out_cstride, (uint64_t)max_img * img_px};
    const uint32_t box[2] = {out_fp32 ? 16u : 32u, 32u};
    rc = make_tmap(&L->tmC, out, 2, dims, box, CU_TENSOR_MAP_SWIZZLE_64B, f16, out_fp32 ? 4 : 2);
    if (rc) return rc;
  } else {
    L->tmC = L->tmA;  // unused
  }

  p.bn = bn;
  p.n_blocks_n = cout_pad / bn;
  p.kb_per_tap = cin_used / bk;
  p.num_kb = taps * p.kb_per_tap;
  p.a_stage_bytes = 128 * bk * 2;
  p.b_stage_bytes = bn * bk * 2;
  p.halo = halo ? 1 : 0;
  if (halo) {
    p.num_kb = 3 * p.kb_per_tap;  // one stage per (dx, channel block)
    p.a_stage_bytes = (RECT_H * subt + 2) * RECT_W * bk * 2;
    p.b_stage_bytes = 0;
    p.bchunk_bytes = bn * bk * 2;
    p.n_bchunks = ktotal / bk;
    p.bres_bytes = (uint32_t)bres;
  }
  p.stage_bytes = tstore ? 8 * 4096 : 0;  // 8 epilogue warps x 2 alternating 2 KB slabs
  const uint32_t stage_bytes = p.a_stage_bytes + p.b_stage_bytes;
  int stages = (int)((227 * 1024 - fixed - (int)p.bres_bytes - (int)p.stage_bytes) /
                     (int)stage_bytes);
  if (stages > 12) stages = 12;
  if (stages < 2) {
    tp_set_error("conv: stage too large");
    return TP_ERR_UNSUPPORTED;
  }
  p.stages = stages;
  p.sub = subt;
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * subt * bn)) cols <<= 1;
  p.tmem_cols = cols;
  p.idesc = tp::idesc_f16kind(128, (uint32_t)bn, !f16);
  p.rect = pool ? 1 : 0;
  p.tiles_x = (res + RECT_W - 1) / RECT_W;
  p.tiles_y = (res + RECT_H * subt - 1) / (RECT_H * subt);
  L->mode = mode;
  L->smem = 1024 + (size_t)stages * stage_bytes + p.bres_bytes + p.stage_bytes +
            (2 * stages + 6) * 8 + cout_pad * 4 + 16;
  // CTA-pair variant for FLAT SW128 layers (TP_PAIR=0 disables it): N = 256 tiles, and
  // N >= 128 for 3x3 layers / the fp32 head (measured: 1x1 layers with N < 256 are HBM-bound
  // and lose ~10-40% to the pair's coarser tiles)
  const char* pe = getenv("TP_PAIR");
  const bool pair_shape = bn == 256 || (bn >= 128 && (ksize == 3 || out_fp32));
  if (tstore && mode == MODE_SW128 && pair_shape && (pe == nullptr || atoi(pe) != 0)) {
    const uint64_t dims[2] = {(uint64_t)ktotal, (uint64_t)cout_pad};
    const uint32_t box[2] = {(uint32_t)bk, (uint32_t)(bn / 2)};
    rc = make_tmap(&L->tmB, weight, 2, dims, box, swz, f16);
    if (rc) return rc;
    L->pair = 1;
    p.b_stage_bytes = (bn / 2) * bk * 2;
    p.idesc = tp::idesc_f16kind(256, (uint32_t)bn, !f16);
    const uint32_t sb = p.a_stage_bytes + p.b_stage_bytes;
    int st = (int)((227 * 1024 - fixed - (int)p.stage_bytes) / (int)sb);
    if (st > 12) st = 12;
    p.stages = st;
    L->smem = 1024 + (size_t)st * sb + p.stage_bytes + (2 * st + 6) * 8 + cout_pad * 4 + 16;
  }
  // CTA-pair halo-box kernel for pooled 3x3 SW128 layers whose weights are not resident
  // (TP_PRECT=0 disables it, TP_PRECT_MH=1 keeps one M block per CTA; the box kernel below
  // still wins where it applies). TP_PRECT_PLAIN=1 also routes unpooled N = 128 layers
  // here: measured slower than the im2col pair kernel (parity layer 4: 0.96 vs 0.84 ms per
  // 120 tiles; its direct 16-byte stores of 4x the pooled bytes cap the epilogue)
  const char* pr = getenv("TP_PRECT");
  const char* prm = getenv("TP_PRECT_MH");
  const char* prp = getenv("TP_PRECT_PLAIN");
  const bool plain_ok = bn == 128 && prp != nullptr && atoi(prp) == 1;
  if ((pool || plain_ok) && ksize == 3 && mode == MODE_SW128 && !halo && bn >= 128 &&
      !out_fp32 && !reorg && (pr == nullptr || atoi(pr) != 0)) {
    const int mh = bn <= 128 && (prm == nullptr || atoi(prm) != 1) ? 2 : 1;
    const uint64_t adims[4] = {(uint64_t)cin_stride, (uint64_t)res, (uint64_t)res, (uint64_t)max_img};
    const uint32_t abox[4] = {(uint32_t)bk, PR_W, (uint32_t)(PR_H * mh + 2), 1};
    ConvLaunch P = *L;
    rc = make_tmap(&P.tmA, in, 4, adims, abox, swz, f16);
    if (rc) return rc;
    const uint64_t bdims[2] = {(uint64_t)ktotal, (uint64_t)cout_pad};
    const uint32_t bbox[2] = {(uint32_t)bk, (uint32_t)(bn / 2)};
    rc = make_tmap(&P.tmB, weight, 2, bdims, bbox, swz, f16);
    if (rc) return rc;
    ConvParams& q = P.p;
    q.bn = bn;
    q.n_blocks_n = cout_pad / bn;
    q.kb_per_tap = cin_used / bk;
    q.num_kb = 3 * q.kb_per_tap;
    q.a_stage_bytes = PR_W * (PR_H * mh + 2) * bk * 2;
    q.b_stage_bytes = 3 * (bn / 2) * bk * 2;
    q.bres_bytes = 0;
    q.stage_bytes = 0;
    q.halo = 0;
    q.sub = mh;
    q.rect = pool ? 1 : 0;
    q.tiles_x = (res + PR_W - 1) / PR_W;
    q.tiles_y = (res + 2 * PR_H * mh - 1) / (2 * PR_H * mh);
    uint32_t pcols = 32;
    while (pcols < (uint32_t)(2 * mh * bn)) pcols <<= 1;
    q.tmem_cols = pcols;
    q.idesc = tp::idesc_f16kind(256, (uint32_t)bn, !f16);
    const uint32_t sb = q.a_stage_bytes + q.b_stage_bytes;
    int st = (int)((227 * 1024 - fixed) / (int)sb);
    if (st > 8) st = 8;
    if (st >= 2 && pcols <= 512) {
      q.stages = st;
      P.smem = 1024 + (size_t)st * sb + (2 * st + 6) * 8 + cout_pad * 4 + 16;
      P.prect = 1;
      P.pair = 0;
      *L = P;
    }
  }
  // swapped-operand kernel for 3x3 layers with 128 output channels whose weights are not
  // resident — pooled ones, and unpooled ones of the parity plan (their hi/lo output
  // leaves through stmatrix + TMA stores). TP_SWAP=0 disables it; the box kernel below
  // still wins where it applies.
  const char* sw = getenv("TP_SWAP");
  if (ksize == 3 && cout_pad == 128 && cout == 128 && cin_used % SW_BK == 0 && !halo &&
      !out_fp32 && !reorg && (pool || split || out_lo != nullptr) &&
      (sw == nullptr || atoi(sw) != 0)) {
    ConvLaunch P = *L;
    const uint64_t xdims[4] = {(uint64_t)cin_stride, (uint64_t)res, (uint64_t)res, (uint64_t)max_img};
    const uint32_t xbox[4] = {SW_BK, SW_W, SW_H + 2, 1};
    rc = make_tmap(&P.tmA, in, 4, xdims, xbox, CU_TENSOR_MAP_SWIZZLE_64B, f16);
    if (rc) return rc;
    const uint64_t wdims[2] = {(uint64_t)ktotal, (uint64_t)cout_pad};
    const uint32_t wbox[2] = {SW_BK, 128 / SW_CL};  // each CTA of a cluster loads a share
    rc = make_tmap(&P.tmB, weight, 2, wdims, wbox, CU_TENSOR_MAP_SWIZZLE_64B, f16);
    if (rc) return rc;
    ConvParams& q = P.p;
    q.bn = 128;
    q.n_blocks_n = 1;
    q.kb_per_tap = cin_used / SW_BK;
    q.num_kb = 3 * q.kb_per_tap;
    q.a_stage_bytes = SW_W * (SW_H + 2) * SW_BK * 2;  // pixel box (MMA B operand)
    q.b_stage_bytes = 3 * 128 * SW_BK * 2;              // three weight slices (MMA A operand)
    q.bres_bytes = 0;
    q.stage_bytes = pool ? (out_lo != nullptr ? 8 * SW_POOL_SCRATCH : 0)
                    : out_lo != nullptr ? SW_STAGING_HL8 : SW_STAGING;
    q.halo = 0;
    q.sub = 1;
    q.rect = pool ? 1 : 0;
    if (!pool && out_lo != nullptr) {  // HL8: hi 16 px x 64 B (SW64) + lo 16 px x 32 B
      const uint64_t cdims[4] = {(uint64_t)out_cstride, (uint64_t)res, (uint64_t)res,
                                 (uint64_t)max_img};
      const uint32_t cbox[4] = {32, SW_W, 2, 1};  // two rows per store
      rc = make_tmap(&P.tmC, out, 4, cdims, cbox, CU_TENSOR_MAP_SWIZZLE_64B, f16);
      if (rc) return rc;
      rc = make_tmap(&P.tmC2, out_lo, 4, cdims, cbox, CU_TENSOR_MAP_SWIZZLE_NONE, f16, 1);
      if (rc) return rc;
    } else if (!pool) {  // store map {stored channels, x, y, image}, box = 16 px x 128 B of one row
      const uint64_t cdims[4] = {(uint64_t)out_cstride, (uint64_t)res, (uint64_t)res,
                                 (uint64_t)max_img};
      const uint32_t cbox[4] = {64, SW_W, 1, 1};
      rc = make_tmap(&P.tmC, out, 4, cdims, cbox, CU_TENSOR_MAP_SWIZZLE_128B, f16);
      if (rc) return rc;
    }
    q.tiles_x = (res + SW_W - 1) / SW_W;
    q.tiles_y = (res + SW_H - 1) / SW_H;
    q.tmem_cols = 512;
    q.idesc = tp::idesc_f16kind(128, 256, !f16);
    const uint32_t sb = q.a_stage_bytes + q.b_stage_bytes;
    int st = (int)((227 * 1024 - fixed - (int)q.stage_bytes) / (int)sb);
    if (st > 8) st = 8;
    if (st >= 2) {
      q.stages = st;
      P.smem = 1024 + (size_t)st * sb + q.stage_bytes + (2 * st + 6) * 8 + cout_pad * 4 + 16;
      P.swap = 1;
      P.prect = 0;
      P.pair = 0;
      *L = P;
    }
  }
  // full-halo box kernel (TP_BOX=0 disables it): 3x3, one K block, resident weights
  const char* be = getenv("TP_BOX");
  const bool box_ok = ksize == 3 && (cin_used == 32 || cin_used == 64) && cout_pad <= 256 &&
                      cout == cout_pad && !reorg && !out_fp32 && res % 8 == 0 &&
                      (in_lo == nullptr || (pool && cin_used == 32 && cout_pad <= 64)) &&
                      bres <= 160 * 1024 && (be == nullptr || atoi(be) != 0);
  // HL8 input (pool-in-M only): + 9 resident e4m3 lo chunks (half the fp16 chunk bytes)
  const size_t bres_box = in_lo != nullptr ? bres + bres / 2 : bres;
  // pool-in-M first (4 pool accumulators x 2 buffers must fit TMEM; pooled side in 8-px
  // tiles), then the shuffle-pool / plain box if its four parity planes do not fit smem
  for (int try_pm = 1; box_ok && try_pm >= 0 && !L->box; --try_pm) {
    const bool pm = try_pm && pool && cout_pad <= 64 && (res / 2) % 8 == 0;
    if (try_pm && !pm) continue;
    const int epi = pm ? BOX_POOLM : pool ? BOX_POOL : BOX_PLAIN;
    // pool-in-M with 64 input channels (the parity plan's layer 2): four 64-channel planes
    // plus the resident weights leave room for one stage only, so the planes come in two
    // 32-channel K blocks (SW64) per tile
    const int kbk = pm && cin_used == 64 &&
                    4 * ((PLANE_W * PLANE_H * 128 + 1023) & ~1023) * 2 + (int)bres > 200 * 1024
                        ? 32 : bk;
    const CUtensorMapSwizzle kswz = kbk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    const uint32_t rb = (uint32_t)kbk * 2;
    const uint32_t stage = pm ? 4 * ((PLANE_W * PLANE_H * rb + 1023) & ~1023u)
                              : ((BOX_TW + 2) * (BOX_TH + 2) * rb + 1023) & ~1023u;
    const uint32_t staging = (!pool && res % 4 == 0) ? 8 * 4096 : 0;  // 2 slabs per warp
    const int bfixed = 1024 + cout_pad * 4 + (2 * 8 + 10) * 8 + 16 + (int)staging;
    int st = (int)((227 * 1024 - bfixed - (int)bres_box) / (int)stage);
    if (st > 8) st = 8;
    const uint32_t per_tile = (pm ? 4u : 1u) * (uint32_t)cout_pad;  // TMEM columns per tile
    const int nbuf = per_tile <= 128 ? 4 : 2;
    const uint32_t need = (uint32_t)nbuf * per_tile;
    uint32_t cols = 32;
    while (cols < need) cols <<= 1;
    if (st >= 2 && cols <= 512) {
      const uint64_t dims[4] = {(uint64_t)cin_stride, (uint64_t)res, (uint64_t)res,
                                (uint64_t)max_img};
      if (pm) {
        const uint32_t box[4] = {(uint32_t)kbk, 2 * PLANE_W, 2 * PLANE_H, 1};
        const uint32_t estr[4] = {1, 2, 2, 1};
        rc = make_tmap(&L->tmA, in, 4, dims, box, kswz, f16, 2, estr);
      } else {
        const uint32_t box[4] = {(uint32_t)bk, BOX_TW + 2, BOX_TH + 2, 1};
        rc = make_tmap(&L->tmA, in, 4, dims, box, swz, f16);
      }
      if (rc) return rc;
      {
        const uint64_t dims[2] = {(uint64_t)ktotal, (uint64_t)cout_pad};
        const uint32_t box[2] = {(uint32_t)kbk, (uint32_t)cout_pad};
        rc = make_tmap(&L->tmB, weight, 2, dims, box, kswz, f16);
        if (rc) return rc;
      }
      p.bn = cout_pad;
      p.n_blocks_n = 1;
      p.a_stage_bytes = stage;
      p.b_stage_bytes = 0;
      p.bchunk_bytes = cout_pad * rb;
      p.num_kb = cin_used / kbk;        // K blocks per tile (stages per tile)
      p.n_bchunks = 9 * p.num_kb;       // resident weight chunks: [K block][tap]
      p.bres_bytes = (uint32_t)bres;
      p.stage_bytes = staging;
      p.sub = 1;
      p.rect = 0;
      p.tiles_x = (pm ? res / 2 : res) / BOX_TW;
      p.tiles_y = ((pm ? res / 2 : res) + BOX_TH - 1) / BOX_TH;
      p.idesc = tp::idesc_f16kind(128, (uint32_t)cout_pad, !f16);
      p.tmem_cols = cols;
      p.nbuf = nbuf;
      p.stages = st;
      L->box = 1 + epi;
      L->box_bk = kbk;
      L->pair = 0;
      L->prect = 0;
      L->swap = 0;
      if (staging) {  // output store map {cstride, res, rows}, box {32 ch, 8 px, 4 rows}
        const uint64_t dims[3] = {(uint64_t)out_cstride, (uint64_t)res, (uint64_t)max_img * res};
        const uint32_t box[3] = {32, BOX_TW, 4};
        rc = make_tmap(&L->tmC, out, 3, dims, box, CU_TENSOR_MAP_SWIZZLE_64B, f16);
        if (rc) return rc;
      }
      L->smem = 1024 + (size_t)st * stage + bres + staging + (2 * st + 10) * 8 + cout_pad * 4 + 16;
    }
  }
  p.kb_hi = p.kb_per_tap;
  if (in_lo != nullptr && L->box) {
    // pool-in-M box with an HL8 input (cin 32): K block 0 = the fp16 hi planes (SW64),
    // K block 1 = the e4m3 lo planes (32-byte rows, SW32) against 9 resident e4m3 chunks
    if (L->box - 1 != BOX_POOLM || L->box_bk != 32 || weight_lo == nullptr) {
      tp_set_error("conv: HL8 input of the box kernel needs pool-in-M with 32 channels");
      return TP_ERR_UNSUPPORTED;
    }
    p.lo_in = 1;
    p.kb_hi = 1;
    p.num_kb = 2;
    p.n_bchunks = 18;
    p.bres_bytes += p.bres_bytes / 2;
    L->smem += bres / 2;
    const uint64_t dims[4] = {(uint64_t)cin_stride, (uint64_t)res, (uint64_t)res, (uint64_t)max_img};
    const uint32_t box[4] = {32, 2 * PLANE_W, 2 * PLANE_H, 1};
    const uint32_t estr[4] = {1, 2, 2, 1};
    rc = make_tmap(&L->tmA2, in_lo, 4, dims, box, CU_TENSOR_MAP_SWIZZLE_32B, f16, 1, estr);
    if (rc) return rc;
    const uint64_t wdims[2] = {(uint64_t)ktotal, (uint64_t)cout_pad};
    const uint32_t wbox[2] = {32, (uint32_t)cout_pad};
    return make_tmap(&L->tmB2, weight_lo, 2, wdims, wbox, CU_TENSOR_MAP_SWIZZLE_32B, f16, 1);
  }
  if (in_lo != nullptr) {
    // HL8 input: after each tap's kb_hi fp16 blocks come cin/128 e4m3 lo blocks of the
    // same stage bytes (128 rows x 128 B); FLAT im2col (tc / pair) and pair-rect only
    // (swap kernel: 32-channel fp16 blocks + 64-channel e4m3 blocks, 64-byte rows)
    const bool flat_tc = !L->pair && !L->prect && !L->box && !L->swap && !L->l0 && !p.rect;
    if (L->swap) {
      if (cin_used % 64 != 0 || weight_lo == nullptr) {
        tp_set_error("conv: HL8 input of the swap kernel needs cin %% 64 == 0");
        return TP_ERR_UNSUPPORTED;
      }
      p.lo_in = 1;
      p.kb_hi = cin_used / SW_BK;
      p.kb_per_tap = p.kb_hi + cin_used / 64;
      p.num_kb = 3 * p.kb_per_tap;
      const uint64_t xdims[4] = {(uint64_t)cin_stride, (uint64_t)res, (uint64_t)res, (uint64_t)max_img};
      const uint32_t xbox[4] = {64, SW_W, SW_H + 2, 1};
      rc = make_tmap(&L->tmA2, in_lo, 4, xdims, xbox, CU_TENSOR_MAP_SWIZZLE_64B, f16, 1);
      if (rc) return rc;
      const uint64_t wdims[2] = {(uint64_t)ktotal, (uint64_t)cout_pad};
      const uint32_t wbox[2] = {64, 128 / SW_CL};
      return make_tmap(&L->tmB2, weight_lo, 2, wdims, wbox, CU_TENSOR_MAP_SWIZZLE_64B, f16, 1);
    }
    if (!(L->pair || L->prect || flat_tc) || cin_used % 128 != 0 || weight_lo == nullptr ||
        mode != MODE_SW128) {
      tp_set_error("conv: HL8 input needs a FLAT or pair-rect SW128 layer with cin %% 128 == 0");
      return TP_ERR_UNSUPPORTED;
    }
    p.lo_in = 1;
    p.kb_hi = cin_used / 64;
    p.kb_per_tap = p.kb_hi + cin_used / 128;
    p.num_kb = (L->prect ? 3 : taps) * p.kb_per_tap;
    if (L->prect) {
      const uint64_t adims[4] = {(uint64_t)cin_stride, (uint64_t)res, (uint64_t)res, (uint64_t)max_img};
      const uint32_t abox[4] = {128, PR_W, (uint32_t)(PR_H * p.sub + 2), 1};
      rc = make_tmap(&L->tmA2, in_lo, 4, adims, abox, CU_TENSOR_MAP_SWIZZLE_128B, f16, 1);
    } else {
      rc = make_tmap_im2col(&L->tmA2, in_lo, cin_stride, res, max_img, 128, 128,
                            ksize == 3 ? -1 : 0, CU_TENSOR_MAP_SWIZZLE_128B, f16, 1);
    }
    if (rc) return rc;
    const uint64_t wdims[2] = {(uint64_t)ktotal, (uint64_t)cout_pad};
    const uint32_t wbox[2] = {128, (uint32_t)(L->pair || L->prect ? p.bn / 2 : p.bn)};
    rc = make_tmap(&L->tmB2, weight_lo, 2, wdims, wbox, CU_TENSOR_MAP_SWIZZLE_128B, f16, 1);
    if (rc) return rc;
  } else {
    L->tmA2 = L->tmA;  // unused
    L->tmB2 = L->tmB;
  }
  return TP_OK;
}

// Fuse a 1x1 HL8 consumer (128 -> 64 channels, leaky) into an unpooled HL8 swap launch:
// the 3x3's HL8 output is staged in shared memory as the 1x1's A operand instead of being
// written to HBM, and the 1x1's MMAs + epilogue run in the same kernel (swap_fused_1x1).
int fuse_swap_1x1(ConvLaunch* L, const void* w, const void* wlo, const float* bias, float alpha,
                  void* out, void* out_lo, int out_cstride) {
  ConvParams& q = L->p;
  if (!L->swap || q.rect || q.out_lo == nullptr || q.n_blocks_n != 1 || w == nullptr ||
      wlo == nullptr || bias == nullptr || out == nullptr || out_lo == nullptr ||
      out_cstride % 16 != 0)
    return TP_ERR_UNSUPPORTED;
  const int fixed = 1024 + 128 * 4 + (2 * 12 + 6) * 8 + 16 + FU_EXTRA;
  const uint32_t sb = q.a_stage_bytes + q.b_stage_bytes;
  int st = (int)((227 * 1024 - fixed - (int)FU_BYTES) / (int)sb);
  if (st > 8) st = 8;
  if (st < 2) return TP_ERR_UNSUPPORTED;
  q.stages = st;
  q.stage_bytes = FU_BYTES;
  q.fuse = 1;
  q.f5_w = w;
  q.f5_wlo = wlo;
  q.f5_bias = bias;
  q.f5_alpha = alpha;
  q.f5_leaky = 1;
  q.f5_out = out;
  q.f5_out_lo = out_lo;
  q.f5_cstride = out_cstride;
  L->smem = 1024 + (size_t)st * sb + FU_BYTES + (2 * st + 6) * 8 + 128 * 4 + 16 + FU_EXTRA;
  return TP_OK;
}

template <int BK, int EPI>
int launch_box(const ConvLaunch& L, int n_img, const int32_t* n_img_dev, cudaStream_t st) {
  if (int rc = ensure_smem_optin(conv_box_kernel<BK, EPI>)) return rc;
  ConvParams p = L.p;
  p.n_img = n_img;
  p.n_img_dev = n_img_dev;
  const long long tiles = (long long)n_img * p.tiles_x * p.tiles_y;
  if (tiles == 0) return TP_OK;
  const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
  conv_box_kernel<BK, EPI><<<grid, kThreads, L.smem, st>>>(L.tmA, L.tmB, L.tmC, L.tmA2, L.tmB2, p);
  TP_LAUNCH_CHECK();
  return TP_OK;
}

template <int MODE, int EPI>
int launch_mode(const ConvLaunch& L, int n_img, const int32_t* n_img_dev, cudaStream_t st) {
  if (int rc = ensure_smem_optin(conv_tc_kernel<MODE, EPI>)) return rc;
  ConvParams p = L.p;
  p.n_img = n_img;
  p.n_img_dev = n_img_dev;
  const long long m_blocks = p.rect ? (long long)n_img * p.tiles_x * p.tiles_y
                                    : ((long long)n_img * p.img_px + 127) / 128;
  const long long tiles = m_blocks * p.n_blocks_n;
  if (tiles == 0) return TP_OK;
  int grid = (int)(tiles < num_sms() ? tiles : num_sms());
  conv_tc_kernel<MODE, EPI><<<grid, kThreads, L.smem, st>>>(L.tmA, L.tmB, L.tmC, L.tmA2, L.tmB2, p);
  TP_LAUNCH_CHECK();
  return TP_OK;
}

template <int EPI>
int launch_pair(const ConvLaunch& L, int n_img, const int32_t* n_img_dev, cudaStream_t st) {
  if (int rc = ensure_smem_optin(conv_pair_kernel<EPI>)) return rc;
  ConvParams p = L.p;
  p.n_img = n_img;
  p.n_img_dev = n_img_dev;
  const long long tiles = (((long long)n_img * p.img_px + 255) / 256) * p.n_blocks_n;
  if (tiles == 0) return TP_OK;
  const int max_clusters = num_sms() / 2;
  const int clusters = (int)(tiles < max_clusters ? tiles : max_clusters);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, conv_pair_kernel<EPI>, L.tmA, L.tmB, L.tmC, L.tmA2, L.tmB2, p));
  return TP_OK;
}

template <int MH, bool POOL>
int launch_pair_rect(const ConvLaunch& L, int n_img, const int32_t* n_img_dev, cudaStream_t st) {
  if (int rc = ensure_smem_optin(conv_pair_rect_kernel<MH, POOL>)) return rc;
  ConvParams p = L.p;
  p.n_img = n_img;
  p.n_img_dev = n_img_dev;
  const long long tiles = (long long)n_img * p.tiles_x * p.tiles_y * p.n_blocks_n;
  if (tiles == 0) return TP_OK;
  const int max_clusters = num_sms() / 2;
  const int clusters = (int)(tiles < max_clusters ? tiles : max_clusters);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, conv_pair_rect_kernel<MH, POOL>, L.tmA, L.tmB, L.tmA2, L.tmB2, p));
  return TP_OK;
}

template <bool POOL>
int launch_swap(const ConvLaunch& L, int n_img, const int32_t* n_img_dev, cudaStream_t st) {
  if (int rc = ensure_smem_optin(conv_swap_kernel<POOL>)) return rc;
  ConvParams p = L.p;
  p.n_img = n_img;
  p.n_img_dev = n_img_dev;
  const long long tiles = (long long)n_img * p.tiles_x * p.tiles_y * p.n_blocks_n;
  if (tiles == 0) return TP_OK;
  const long long groups = (tiles + SW_CL - 1) / SW_CL;
  const int max_clusters = num_sms() / SW_CL;
  const int clusters = (int)(groups < max_clusters ? groups : max_clusters);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(SW_CL * clusters, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = SW_CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, conv_swap_kernel<POOL>, L.tmA, L.tmB, L.tmC, L.tmA2, L.tmB2,
                                   L.tmC2, p));
  return TP_OK;
}

int run_conv(const ConvLaunch& L, int n_img, const int32_t* n_img_dev, cudaStream_t st) {
  if (n_img > L.p.n_img) {
    tp_set_error("conv: n_img %d exceeds planned %d", n_img, L.p.n_img);
    return TP_ERR_CAPACITY;
  }
  if (L.box) {
    const int epi = L.box - 1;
    if (L.box_bk == 64)
      return epi == BOX_POOLM ? launch_box<64, BOX_POOLM>(L, n_img, n_img_dev, st)
             : epi == BOX_POOL ? launch_box<64, BOX_POOL>(L, n_img, n_img_dev, st)
                               : launch_box<64, BOX_PLAIN>(L, n_img, n_img_dev, st);
    return epi == BOX_POOLM ? launch_box<32, BOX_POOLM>(L, n_img, n_img_dev, st)
           : epi == BOX_POOL ? launch_box<32, BOX_POOL>(L, n_img, n_img_dev, st)
                             : launch_box<32, BOX_PLAIN>(L, n_img, n_img_dev, st);
  }
  if (L.swap)
    return L.p.rect ? launch_swap<true>(L, n_img, n_img_dev, st)
                    : launch_swap<false>(L, n_img, n_img_dev, st);
  if (L.prect) {
    const bool pool = L.p.rect != 0;
    if (L.p.sub == 2)
      return pool ? launch_pair_rect<2, true>(L, n_img, n_img_dev, st)
                  : launch_pair_rect<2, false>(L, n_img, n_img_dev, st);
    return pool ? launch_pair_rect<1, true>(L, n_img, n_img_dev, st)
                : launch_pair_rect<1, false>(L, n_img, n_img_dev, st);
  }
  if (L.pair)
    return L.p.out_fp32 ? launch_pair<EPI_F32>(L, n_img, n_img_dev, st)
           : L.p.split  ? launch_pair<EPI_SPLIT>(L, n_img, n_img_dev, st)
           : L.p.out_lo ? launch_pair<EPI_HL8>(L, n_img, n_img_dev, st)
                        : launch_pair<EPI_PLAIN>(L, n_img, n_img_dev, st);
  if (L.l0) {
    if (int rc = ensure_smem_optin(conv_l0_kernel)) return rc;
    ConvParams p = L.p;
    p.n_img = n_img;
    p.n_img_dev = n_img_dev;
    const long long tiles = (long long)n_img * (p.res / 32) * (p.res / 16);
    if (tiles == 0) return TP_OK;
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    conv_l0_kernel<<<grid, kThreads, L.smem, st>>>(L.tmA, L.tmB, L.tmC, L.tmC2, p);
    TP_LAUNCH_CHECK();
    return TP_OK;
  }
  const int epi = L.p.rect ? EPI_POOL : L.p.reorg ? EPI_REORG : L.p.out_fp32 ? EPI_F32
                : L.p.split ? EPI_SPLIT : L.p.out_lo ? EPI_HL8 : EPI_PLAIN;
#define TP_EPI_SWITCH(M)                                                  \
  switch (epi) {                                                          \
    case EPI_POOL: return launch_mode<M, EPI_POOL>(L, n_img, n_img_dev, st);   \
    case EPI_REORG: return launch_mode<M, EPI_REORG>(L, n_img, n_img_dev, st); \
    case EPI_F32: return launch_mode<M, EPI_F32>(L, n_img, n_img_dev, st);     \
    case EPI_SPLIT: return launch_mode<M, EPI_SPLIT>(L, n_img, n_img_dev, st); \
    case EPI_HL8: return launch_mode<M, EPI_HL8>(L, n_img, n_img_dev, st);     \
    default: return launch_mode<M, EPI_PLAIN>(L, n_img, n_img_dev, st);        \
  }
  if (L.mode == MODE_SW128) {
    TP_EPI_SWITCH(MODE_SW128)
  }
  TP_EPI_SWITCH(MODE_SW64)
#undef TP_EPI_SWITCH
}

int run_pool(const void* in, int n_img, int res, int cstride, void* out, cudaStream_t st,
             const int32_t* n_img_dev, int f16, int split = 0, const void* in_lo = nullptr,
             void* out_lo = nullptr) {
  const long long total = (long long)n_img * (res / 2) * (res / 2) * (cstride / (split ? 16 : 8));
  if (total == 0) return TP_OK;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (in_lo != nullptr) {
    const dim3 grid((unsigned)(((res / 2) * (cstride / 8) + 255) / 256), (unsigned)(n_img * (res / 2)));
    maxpool2_hl8_kernel<<<grid, 256, 0, st>>>((const __half*)in, (const uint8_t*)in_lo, n_img, res,
                                              cstride, (__half*)out, (uint8_t*)out_lo, n_img_dev);
    TP_LAUNCH_CHECK();
    return TP_OK;
  }
  if (split) {
    maxpool2_split_kernel<<<(int)blocks, 256, 0, st>>>((const __half*)in, n_img, res, cstride,
                                                      (__half*)out, n_img_dev);
    TP_LAUNCH_CHECK();
    return TP_OK;
  }
  maxpool2_kernel<<<(int)blocks, 256, 0, st>>>((const __nv_bfloat16*)in, n_img, res, cstride,
                                               (__nv_bfloat16*)out, n_img_dev, f16);
  TP_LAUNCH_CHECK();
  return TP_OK;
}

// ------------------------------------------------------------------ YOLO v2-608 plan
// Layer table (darknet layer index, cin, cout, ksize, res). BN is folded into
// weights+bias by the host; layer 30 is linear (no BN, no leaky). Layer 0's weights are
// [32][144]: per kernel row, 3 variants (conv_l0_kernel comment) x 4 slots x rgb0.
struct LayerDef {
  int idx, cin, cout, k, res;
};
const LayerDef kConvs[23] = {
    {0, 16, 32, 3, 608},     {2, 32, 64, 3, 304},     {4, 64, 128, 3, 152},
    {5, 128, 64, 1, 152},    {6, 64, 128, 3, 152},    {8, 128, 256, 3, 76},
    {9, 256, 128, 1, 76},    {10, 128, 256, 3, 76},   {12, 256, 512, 3, 38},
    {13, 512, 256, 1, 38},   {14, 256, 512, 3, 38},   {15, 512, 256, 1, 38},
    {16, 256, 512, 3, 38},   {18, 512, 1024, 3, 19},  {19, 1024, 512, 1, 19},
    {20, 512, 1024, 3, 19},  {21, 1024, 512, 1, 19},  {22, 512, 1024, 3, 19},
    {23, 1024, 1024, 3, 19}, {24, 1024, 1024, 3, 19}, {26, 512, 64, 1, 38},
    {29, 1280, 1024, 3, 19}, {30, 1024, 425, 1, 19}};

// R38: layer 26's plain 38^2 x 64 output, gathered into CAT19 by reorg_gather_kernel
enum Buf {
  I608, P304, P152, A152, B152, P76, A76, B76, P38, A38, B38, E38, P19, A19, B19, C19, CAT19,
  HEAD, R38, NBUF
};
struct BufDef {
  int res, ch, bytes_per;  // bytes per element
};
constexpr BufDef kBufs[NBUF] = {{608, 4, 2},  {304, 32, 2},  {152, 64, 2},   {152, 128, 2},
                            {152, 64, 2},  {76, 128, 2},  {76, 256, 2},   {76, 128, 2},
                            {38, 256, 2},  {38, 512, 2},  {38, 256, 2},   {38, 512, 2},
                            {19, 512, 2},  {19, 1024, 2}, {19, 512, 2},   {19, 1024, 2},
                            {19, 1280, 2}, {19, 448, 4},  {38, 64, 2}};
constexpr int kHeadCstride = 448;

// Step list: conv (layer slot, in, out, channel offset, reorg, fused pool) or pool (in, out).
struct Step {
  int is_pool;
  int conv;  // index into kConvs
  int in, out, coff, reorg, fpool;
};
constexpr Step kSteps[] = {
    {0, 0, I608, P304, 0, 0, 1},  {0, 1, P304, P152, 0, 0, 1},  {0, 2, P152, A152, 0, 0, 0},
    {0, 3, A152, B152, 0, 0, 0},  {0, 4, B152, P76, 0, 0, 1},   {0, 5, P76, A76, 0, 0, 0},
    {0, 6, A76, B76, 0, 0, 0},    {0, 7, B76, P38, 0, 0, 1},    {0, 8, P38, A38, 0, 0, 0},
    {0, 9, A38, B38, 0, 0, 0},    {0, 10, B38, A38, 0, 0, 0},   {0, 11, A38, B38, 0, 0, 0},
    {0, 12, B38, E38, 0, 0, 0},   {1, -1, E38, P19, 0, 0, 0},   {0, 13, P19, A19, 0, 0, 0},
    {0, 14, A19, B19, 0, 0, 0},   {0, 15, B19, C19, 0, 0, 0},   {0, 16, C19, B19, 0, 0, 0},
    {0, 17, B19, A19, 0, 0, 0},   {0, 18, A19, C19, 0, 0, 0},   {0, 19, C19, CAT19, 256, 0, 0},
    {0, 20, E38, CAT19, 0, 1, 0}, {0, 21, CAT19, A19, 0, 0, 0}, {0, 22, A19, HEAD, 0, 0, 0}};
constexpr int kNumSteps = sizeof(kSteps) / sizeof(kSteps[0]);

// Storage format of a buffer: the F16X2 plan pairs every activation but the layer-0 slots
// (integer pixel values, exact in fp16) and the fp32 head; the F16F8 plan stores those same
// activations as HL8 planes (TP_DTYPE_F16F8).
enum BufFmt { FMT_PLAIN = 0, FMT_X2 = 1, FMT_HL8 = 2 };
int buf_fmt(int b, int dtype) {
  if (b == I608 || b == HEAD) return FMT_PLAIN;
  if (dtype == TP_DTYPE_F16X2) return FMT_X2;
  if (dtype == TP_DTYPE_F16F8) return FMT_HL8;
  return FMT_PLAIN;
}
// channels stored per pixel (hi plane for HL8)
int buf_ch(int b, int dtype) { return kBufs[b].ch * (buf_fmt(b, dtype) == FMT_X2 ? 2 : 1); }
// bytes of an HL8 buffer's e4m3 lo plane (0 for other formats)
size_t buf_lo_bytes(int b, int max_tiles, int dtype) {
  if (buf_fmt(b, dtype) != FMT_HL8) return 0;
  return (size_t)max_tiles * kBufs[b].res * kBufs[b].res * kBufs[b].ch;
}

size_t buf_bytes(int b, int max_tiles, int dtype) {
  // compact NHWC, except the layer-0 input (padded, written by the gather)
  // the layer-0 input is [610 rows][614 columns][rgb0] (tp_gather.cu): a 1-pixel zero halo
  // above / below, 2 | 4 columns left / right for the 64-byte 8-pixel windows
  if (b == I608)
    return (size_t)max_tiles * (kBufs[b].res + 2) * (kBufs[b].res + 6) * 4 * 2;
  const size_t side = kBufs[b].res;
  return (size_t)max_tiles * side * side * buf_ch(b, dtype) * kBufs[b].bytes_per;
}

}  // namespace

struct tp_yolo_net {
  int max_tiles;
  int dtype;
  void* bufs[NBUF];
  void* lo[NBUF];  // HL8 lo planes (nullptr for other formats)
  ConvLaunch convs[23];
  // F16F8 plan: step kFuseStep's 1x1 runs inside step kFuseStep - 1's swap kernel when
  // fused != 0 (the default); unfused keeps the separate launches (tp_yolo_set_fused)
  int fusable, fused;
  ConvLaunch fused_launch, plain_launch;
};
// the F16F8 plan's fused pair: step 2 (layer 4, 3x3 64 -> 128 at 152^2, conv_swap_kernel)
// feeds step 3 (layer 5, 1x1 128 -> 64), and nothing else reads step 2's output
constexpr int kFuseStep = 3;

extern "C" size_t tp_yolo_workspace_bytes(int max_tiles, int dtype) {
  size_t total = 0;
  for (int b = 0; b < NBUF; ++b) {
    total += (buf_bytes(b, max_tiles, dtype) + 1023) & ~size_t(1023);
    total += (buf_lo_bytes(b, max_tiles, dtype) + 1023) & ~size_t(1023);
  }
  return total;
}

extern "C" uint32_t tp_yolo_hl8_inputs(void) {
  uint32_t m = 0;
  for (int s = 0; s < kNumSteps; ++s)
    if (!kSteps[s].is_pool && buf_fmt(kSteps[s].in, TP_DTYPE_F16F8) == FMT_HL8)
      m |= 1u << kSteps[s].conv;
  return m;
}

extern "C" int tp_yolo_create(int max_tiles, const void* const* weights,
                              const float* const* biases, void* workspace,
                              size_t workspace_bytes, int dtype, tp_yolo_net** out) {
  return tp_yolo_create_ex(max_tiles, weights, nullptr, biases, nullptr, workspace,
                           workspace_bytes, dtype, out);
}

extern "C" int tp_yolo_create_ex(int max_tiles, const void* const* weights,
                                 const void* const* weights_lo, const float* const* biases,
                                 const float* alphas, void* workspace, size_t workspace_bytes,
                                 int dtype, tp_yolo_net** out) {
  if (max_tiles < 1 || weights == nullptr || biases == nullptr || workspace == nullptr ||
      out == nullptr) {
    tp_set_error("tp_yolo_create: bad argument");
    return TP_ERR_ARG;
  }
  if (dtype != TP_DTYPE_BF16 && dtype != TP_DTYPE_F16 && dtype != TP_DTYPE_F16X2 &&
      dtype != TP_DTYPE_F16F8) {
    tp_set_error("tp_yolo_create: bad dtype %d", dtype);
    return TP_ERR_ARG;
  }
  if (dtype == TP_DTYPE_F16F8 && (weights_lo == nullptr || alphas == nullptr)) {
    tp_set_error("tp_yolo_create: the F16F8 plan needs lo weights and accumulator scales");
    return TP_ERR_ARG;
  }
  if (workspace_bytes < tp_yolo_workspace_bytes(max_tiles, dtype)) {
    tp_set_error("tp_yolo_create: workspace too small");
    return TP_ERR_CAPACITY;
  }
  tp_yolo_net* net = new tp_yolo_net();
  net->max_tiles = max_tiles;
  net->dtype = dtype;
  uint8_t* w = reinterpret_cast<uint8_t*>(workspace);
  for (int b = 0; b < NBUF; ++b) {
    net->bufs[b] = w;
    w += (buf_bytes(b, max_tiles, dtype) + 1023) & ~size_t(1023);
    const size_t lb = buf_lo_bytes(b, max_tiles, dtype);
    net->lo[b] = lb ? w : nullptr;
    w += (lb + 1023) & ~size_t(1023);
  }
  // halos (and every never-written byte) must be zero
  cudaError_t e = cudaMemset(workspace, 0, tp_yolo_workspace_bytes(max_tiles, dtype));
  if (e != cudaSuccess) {
    delete net;
    tp_set_error("tp_yolo_create: memset: %s", cudaGetErrorString(e));
    return TP_ERR_CUDA;
  }
  for (int s = 0; s < kNumSteps; ++s) {
    const Step& st = kSteps[s];
    if (st.is_pool) continue;
    const LayerDef& L = kConvs[st.conv];
    const int cout_pad = L.cout == 425 ? kHeadCstride : L.cout;
    const bool head = (st.out == HEAD);
    // X2 input: K covers the interleaved hi/lo pairs (duplicated weights); HL8 input: hi
    // blocks + e4m3 lo blocks, accumulator scaled by alphas[conv]; layer 0 reads integer
    // pixels in both parity plans and scales its accumulators by 1/255
    const int fin = buf_fmt(st.in, dtype), fout = buf_fmt(st.out, dtype);
    const bool parity = dtype == TP_DTYPE_F16X2 || dtype == TP_DTYPE_F16F8;
    const int cin = fin == FMT_X2 && st.conv != 0 ? 2 * L.cin : L.cin;
    const int coff = fout == FMT_X2 ? 2 * st.coff : st.coff;
    const int ldt = dtype == TP_DTYPE_F16F8 ? (fout == FMT_X2 ? TP_DTYPE_F16X2 : TP_DTYPE_F16)
                                            : dtype;
    const float alpha = parity && st.conv == 0 ? 1.0f / 255.0f
                        : fin == FMT_HL8       ? alphas[st.conv]
                                               : 1.0f;
    // the reorg layer writes R38 (plain layout, TMA-store epilogue); tp_yolo_forward_range
    // gathers it into the concat buffer (reorg_gather_kernel)
    const int ob = st.reorg ? R38 : st.out;
    int rc = prepare_conv(&net->convs[st.conv], net->bufs[st.in], max_tiles, L.res,
                          buf_ch(st.in, dtype), cin, weights[st.conv], biases[st.conv], L.cout,
                          cout_pad, L.k, head ? 0 : 1, net->bufs[ob], buf_ch(ob, dtype),
                          st.reorg ? 0 : coff, head ? 1 : 0, 0, ldt, st.fpool, alpha,
                          net->lo[st.in], fin == FMT_HL8 ? weights_lo[st.conv] : nullptr,
                          net->lo[ob]);
    if (rc) {
      delete net;
      return rc;
    }
  }
  if (dtype == TP_DTYPE_F16F8) {
    const Step& a = kSteps[kFuseStep - 1];
    const Step& b = kSteps[kFuseStep];
    const LayerDef& lb = kConvs[b.conv];
    static_assert(kSteps[kFuseStep].in == kSteps[kFuseStep - 1].out, "fused pair");
    if (!a.is_pool && !b.is_pool && lb.k == 1 && lb.cin == 128 && lb.cout == FU_N && b.coff == 0 &&
        !b.reorg && !b.fpool) {
      ConvLaunch f = net->convs[a.conv];
      if (fuse_swap_1x1(&f, weights[b.conv], weights_lo[b.conv], biases[b.conv], alphas[b.conv],
                        net->bufs[b.out], net->lo[b.out], buf_ch(b.out, dtype)) == TP_OK) {
        net->plain_launch = net->convs[a.conv];
        net->fused_launch = f;
        net->convs[a.conv] = f;
        net->fusable = net->fused = 1;
      }
    }
  }
  *out = net;
  return TP_OK;
}

extern "C" int tp_yolo_set_fused(tp_yolo_net* net, int fused) {
  if (net == nullptr) {
    tp_set_error("tp_yolo_set_fused: null plan");
    return TP_ERR_ARG;
  }
  if (!net->fusable) return fused ? TP_ERR_UNSUPPORTED : TP_OK;
  net->fused = fused ? 1 : 0;
  net->convs[kSteps[kFuseStep - 1].conv] = fused ? net->fused_launch : net->plain_launch;
  return TP_OK;
}

extern "C" int tp_yolo_step_fused(tp_yolo_net* net, int step) {
  return net != nullptr && net->fused && step == kFuseStep ? 1 : 0;
}

extern "C" void* tp_yolo_input(tp_yolo_net* net) { return net ? net->bufs[I608] : nullptr; }
extern "C" const float* tp_yolo_head(tp_yolo_net* net) {
  return net ? reinterpret_cast<const float*>(net->bufs[HEAD]) : nullptr;
}
extern "C" int tp_yolo_head_cstride(void) { return kHeadCstride; }
extern "C" int tp_yolo_num_steps(void) { return kNumSteps; }

extern "C" int tp_yolo_forward_range(tp_yolo_net* net, int n_tiles, const int32_t* n_tiles_dev,
                                     int first, int last, void* stream) {
  if (net == nullptr || n_tiles < 0 || n_tiles > net->max_tiles) {
    tp_set_error("tp_yolo_forward: bad n_tiles %d", n_tiles);
    return TP_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  for (int s = first; s <= last && s < kNumSteps; ++s) {
    const Step& sp = kSteps[s];
    int rc;
    if (sp.is_pool) {
      rc = run_pool(net->bufs[sp.in], n_tiles, kBufs[sp.in].res, buf_ch(sp.in, net->dtype),
                    net->bufs[sp.out], st, n_tiles_dev, net->dtype != TP_DTYPE_BF16,
                    buf_fmt(sp.in, net->dtype) == FMT_X2, net->lo[sp.in], net->lo[sp.out]);
    } else if (net->fused && s == kFuseStep) {
      rc = TP_OK;  // ran inside step kFuseStep - 1's kernel
    } else {
      rc = run_conv(net->convs[sp.conv], n_tiles, n_tiles_dev, st);
      if (rc == TP_OK && sp.reorg) {  // layer 26 wrote R38: gather it into CAT19 [0, 256)
        const int fmt = buf_fmt(R38, net->dtype) == FMT_X2 ? 1 : buf_fmt(R38, net->dtype) == FMT_HL8 ? 2 : 0;
        const long long total = (long long)n_tiles * 19 * 19 * (4 * kBufs[R38].ch / 8);
        long long blocks = (total + 255) / 256;
        if (blocks > 148 * 8) blocks = 148 * 8;
        static_assert(kBufs[R38].res == 38 && kBufs[R38].ch == 64, "reorg_gather_kernel<38, 64>");
        if (total > 0) {
          reorg_gather_kernel<38, 64><<<(int)blocks, 256, 0, st>>>(
              (const uint16_t*)net->bufs[R38], (const uint8_t*)net->lo[R38], n_tiles, n_tiles_dev,
              buf_ch(R38, net->dtype), (uint16_t*)net->bufs[sp.out], (uint8_t*)net->lo[sp.out],
              buf_ch(sp.out, net->dtype), fmt);
          TP_LAUNCH_CHECK();
        }
      }
    }
    if (rc) return rc;
  }
  return TP_OK;
}

extern "C" int tp_yolo_forward(tp_yolo_net* net, int n_tiles, const int32_t* n_tiles_dev,
                               void* stream) {
  return tp_yolo_forward_range(net, n_tiles, n_tiles_dev, 0, kNumSteps - 1, stream);
}

// Output buffer of step `layer` (index into the step list).
extern "C" int tp_yolo_layer_output(tp_yolo_net* net, int layer, void** ptr, int* res,
                                    int* cstride) {
  if (net == nullptr || layer < 0 || layer >= kNumSteps) {
    tp_set_error("tp_yolo_layer_output: bad step %d", layer);
    return TP_ERR_ARG;
  }
  const int b = kSteps[layer].out;
  *ptr = net->bufs[b];
  *res = kBufs[b].res;
  *cstride = buf_ch(b, net->dtype);
  return TP_OK;
}

extern "C" int tp_yolo_layer_output_lo(tp_yolo_net* net, int layer, void** ptr) {
  if (net == nullptr || layer < 0 || layer >= kNumSteps || ptr == nullptr) {
    tp_set_error("tp_yolo_layer_output_lo: bad step %d", layer);
    return TP_ERR_ARG;
  }
  *ptr = net->lo[kSteps[layer].out];
  return TP_OK;
}

// Kernel chosen for conv slot `conv` of the plan: 0 conv_tc_kernel, 1 conv_pair_kernel,
// 2 conv_l0_kernel, 3 conv_box_kernel, 4 conv_pair_rect_kernel, 5 conv_swap_kernel.
extern "C" int tp_yolo_layer_kernel(tp_yolo_net* net, int conv) {
  if (net == nullptr || conv < 0 || conv >= 23) {
    tp_set_error("tp_yolo_layer_kernel: bad conv slot %d", conv);
    return -1;
  }
  const ConvLaunch& L = net->convs[conv];
  return L.box ? 3 : L.l0 ? 2 : L.pair ? 1 : L.prect ? 4 : L.swap ? 5 : 0;
}

extern "C" int tp_yolo_destroy(tp_yolo_net* net) {
  delete net;
  return TP_OK;
}

extern "C" int tp_conv(const void* in, int n_img, int res, int cin_stride, const void* weight,
                       const float* bias, int cout, int cout_pad, int ksize, int leaky, void* out,
                       int out_cstride, int out_coff, int out_fp32, int reorg, int dtype, int pool,
                       void* stream) {
  if (in == nullptr || weight == nullptr || bias == nullptr || out == nullptr || n_img < 1 ||
      (ksize != 1 && ksize != 3)) {
    tp_set_error("tp_conv: bad argument");
    return TP_ERR_ARG;
  }
  if (dtype == TP_DTYPE_F16F8) {  // HL8 lo planes exist only inside a tp_yolo_net plan
    tp_set_error("tp_conv: TP_DTYPE_F16F8 is a plan format (tp_yolo_create_ex), not a layer dtype");
    return TP_ERR_UNSUPPORTED;
  }
  ConvLaunch L;
  const float alpha = dtype == TP_DTYPE_F16X2 && cin_stride == 16 ? 1.0f / 255.0f : 1.0f;
  int rc = prepare_conv(&L, in, n_img, res, cin_stride, cin_stride, weight, bias, cout, cout_pad,
                        ksize, leaky, out, out_cstride, out_coff, out_fp32, reorg, dtype, pool,
                        alpha);
  if (rc) return rc;
  return run_conv(L, n_img, nullptr, (cudaStream_t)stream);
}

extern "C" int tp_debug_conv_counters(uint64_t* out, int n, int reset) {
  unsigned long long h[8] = {0};
  if (n > 8) n = 8;
  if (out != nullptr && n > 0) {
    if (cudaMemcpyFromSymbol(h, g_conv_prof, sizeof(h)) != cudaSuccess) {
      tp_set_error("tp_debug_conv_counters: copy failed");
      return -1;
    }
    for (int i = 0; i < n; ++i) out[i] = h[i];
  }
  if (reset) {
    unsigned long long z[8] = {0};
    if (cudaMemcpyToSymbol(g_conv_prof, z, sizeof(z)) != cudaSuccess) {
      tp_set_error("tp_debug_conv_counters: reset failed");
      return -1;
    }
  }
  return 0;
}

extern "C" int tp_maxpool2(const void* in, int n_img, int res, int cstride, int dtype,
                           void* out, void* stream) {
  const int split = dtype == TP_DTYPE_F16X2;
  if (in == nullptr || out == nullptr || (res & 1) || (cstride & (split ? 31 : 7)) ||
      dtype == TP_DTYPE_F16F8) {
    tp_set_error("tp_maxpool2: bad argument (TP_DTYPE_F16F8 pools run inside the YOLO plan)");
    return TP_ERR_ARG;
  }
  return run_pool(in, n_img, res, cstride, out, (cudaStream_t)stream, nullptr,
                  dtype != TP_DTYPE_BF16, split);
}
