// Probe: does a tiled TMA map whose dims overlap in memory ({16 halves = slots x and x+1,
// slot x 16 B apart, row}) load slots x, x+1 for each x, with and without SW32?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_overlap_probe_bin tools/tma_overlap_probe.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdio>

#include "../paper_1810_10551_b200/csrc/tp_common.cuh"

void tp_set_error(const char*, ...) {}

constexpr int W = 40, H = 6;

__global__ void probe(const __grid_constant__ CUtensorMap tm, int x0, int y0, float* out) {
  __shared__ __align__(1024) __half buf[32 * 8 * 3];
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 32 * 8 * 3; i += blockDim.x) buf[i] = __float2half(-1.0f);
  if (threadIdx.x == 0) {
    tp::mbar_init(&bar, 1);
    tp::fence_mbar_init();
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    tp::mbar_arrive_expect_tx(&bar, 32 * 8 * 3 * 2);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(tp::smem_u32(buf)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(tp::smem_u32(&bar)), "r"(0), "r"(x0), "r"(y0)
        : "memory");
  }
  tp::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 32 * 8 * 3; i += blockDim.x) out[i] = __half2float(buf[i]);
}

int main() {
  // slot (y, x) = 8 halves, value 100*y + x in element 0, 0.5 + that in element 4
  static __half h[H * W * 8];
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x)
      for (int c = 0; c < 8; ++c)
        h[(y * W + x) * 8 + c] = __float2half(c == 0 ? 100.f * y + x : (c == 4 ? 100.f * y + x + 0.5f : 0.f));
  void* d;
  cudaMalloc(&d, sizeof(h));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  float* dout;
  cudaMalloc(&dout, 32 * 8 * 3 * sizeof(float));
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  Enc enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  for (int sw = 0; sw < 2; ++sw)
    for (int es : {1, 2}) {
      // 3-D view {32 halves = slots 2k..2k+3, k (32 B apart: overlapping), row}
      CUtensorMap tm;
      cuuint64_t dims[3] = {32, W / 2 - 1, H};
      cuuint64_t strides[2] = {32, W * 16};
      cuuint32_t box[3] = {32, (cuuint32_t)(8 * es), (cuuint32_t)(3 * es)};
      cuuint32_t estr[3] = {1, (cuuint32_t)es, (cuuint32_t)es};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, d, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE,
                       sw ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("swizzle %s estride %d: encode %d\n", sw ? "64B" : "none", es, (int)r);
      if (r != CUDA_SUCCESS) continue;
      probe<<<1, 128>>>(tm, 3, 1, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("  launch error %s\n", cudaGetErrorString(e));
        return 1;
      }
      float o[32 * 8 * 3];
      cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
      // row r of 64 B (32 halves) per (y, k): halves 0, 4, ..., 28 (raw smem order)
      for (int row = 0; row < 24; ++row)
        printf("  smem row %2d: %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f\n", row,
               o[row * 32], o[row * 32 + 4], o[row * 32 + 8], o[row * 32 + 12], o[row * 32 + 16],
               o[row * 32 + 20], o[row * 32 + 24], o[row * 32 + 28]);
    }
  return 0;
}
