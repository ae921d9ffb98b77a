// Probe of TMA im2col semantics (cuTensorMapEncodeIm2col + cp.async.bulk.tensor.4d.im2col):
// which (n, y, x) pixel lands in each smem row for given corners / coordinates / offsets.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/im2col_probe_bin tools/im2col_probe.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdio>

#include "../paper_1810_10551_b200/csrc/tp_common.cuh"

void tp_set_error(const char*, ...) {}

constexpr int N = 3, H = 5, W = 5, C = 64, PIX = 32;

__global__ void probe(const __grid_constant__ CUtensorMap tm, int c0, int w0, int h0, int n0, int ow,
                      int oh, float* out) {
  __shared__ __align__(1024) __half buf[PIX * C];
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < PIX * C; i += blockDim.x) buf[i] = __float2half(-1.0f);
  if (threadIdx.x == 0) {
    tp::mbar_init(&bar, 1);
    tp::fence_mbar_init();
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    tp::mbar_arrive_expect_tx(&bar, PIX * C * 2);
    const uint16_t offw = (uint16_t)ow, offh = (uint16_t)oh;
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(tp::smem_u32(buf)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(tp::smem_u32(&bar)), "r"(c0), "r"(w0), "r"(h0),
        "r"(n0), "h"(offw), "h"(offh)
        : "memory");
  }
  tp::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < PIX; i += blockDim.x) out[i] = __half2float(buf[i * C]);
}

int main() {
  // value at (n, y, x, c=0) = 100 n + 10 y + x + 1 (0 = zero fill, -1 = not written)
  __half h[N * H * W * C];
  for (int n = 0; n < N; ++n)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        for (int c = 0; c < C; ++c)
          h[((n * H + y) * W + x) * C + c] = __float2half((float)(100 * n + 10 * y + x + 1));
  void* d;
  cudaMalloc(&d, sizeof(h));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  float* dout;
  cudaMalloc(&dout, PIX * sizeof(float));
  for (int corner : {0, 1}) {
    CUtensorMap tm;
    cuuint64_t dims[4] = {C, W, H, N};
    cuuint64_t strides[3] = {C * 2, W * C * 2, H * W * C * 2};
    int lower[2], upper[2];
    if (corner == 0) {  // pad 1, 3x3: windows start at -1 .. W-2
      lower[0] = lower[1] = -1;
      upper[0] = upper[1] = -1;
    } else {
      lower[0] = lower[1] = -1;
      upper[0] = upper[1] = -2;
    }
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeIm2col(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, d, dims, strides,
                                         lower, upper, C, PIX, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      continue;
    }
    struct Q {
      int w, h, n, ow, oh;
    } qs[] = {{0, 0, 0, 0, 0}, {-1, -1, 0, 0, 0}, {-1, -1, 0, 1, 1}, {-1, -1, 0, 2, 2},
              {2, 3, 0, 0, 0},  {-1, -1, 1, 0, 0}};
    for (const Q& q : qs) {
      probe<<<1, 128>>>(tm, 0, q.w, q.h, q.n, q.ow, q.oh, dout);
      cudaError_t e = cudaDeviceSynchronize();
      float o[PIX];
      cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
      printf("corner %d lower (%d,%d) upper (%d,%d) coords w=%d h=%d n=%d off (%d,%d) %s:", corner,
             lower[0], lower[1], upper[0], upper[1], q.w, q.h, q.n, q.ow, q.oh,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
      for (int i = 0; i < PIX; ++i) printf(" %g", o[i]);
      printf("\n");
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
