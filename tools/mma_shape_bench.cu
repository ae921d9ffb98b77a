// Micro-benchmark: cycles per tcgen05.mma.cta_group::1.kind::f16 (K = 16) for M in {64, 128}
// and N in {64, 128, 256} (and A 8-row group pitches 1024 / 1152 / 1280 / 2048 B, A starting mid swizzle atom), operands resident in shared memory (SW128 K-major), one issuing
// thread, back-to-back MMAs into one accumulator. Answers whether an M = 64 MMA (64 output
// channels as the A operand) runs at the M = 128 rate per FLOP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_shape tools/mma_shape_bench.cu
#include <cstdio>

#include "../paper_1810_10551_b200/csrc/tp_common.cuh"

void tp_set_error(const char*, ...) {}

__global__ void mma_shape(int n_mma, uint32_t m, uint32_t n, uint32_t sbo, uint32_t a_off, long long* out) {
  extern __shared__ uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    tp::mbar_init(&bar, 1);
    tp::fence_mbar_init();
  }
  if (threadIdx.x < 32) tp::tmem_alloc(&slot, 512);
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint32_t idesc = tp::idesc_f16kind(m, n, false);
    const uint64_t ad = tp::umma_desc(tp::smem_u32(base) + a_off, 16, sbo, 2);
    const uint64_t bd = tp::umma_desc(tp::smem_u32(base + 32768), 16, 1024, 2);
    __syncwarp();
    const long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      if (tp::elect_one()) tp::mma_bf16(tmem, ad, bd, idesc, i > 0);
      __syncwarp();
    }
    if (tp::elect_one()) tp::mma_commit(&bar);
    __syncwarp();
    tp::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) *out = t1 - t0;
  }
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  if (threadIdx.x < 32) tp::tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long));
  cudaFuncSetAttribute(mma_shape, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int n_mma = 4096;
  const uint32_t shapes[][4] = {{128, 64, 1024, 0}, {128, 128, 1024, 0}, {128, 256, 1024, 0},
                                 {64, 64, 1024, 0}, {64, 128, 1024, 0}, {64, 256, 1024, 0},
                                 {128, 64, 1152, 0}, {128, 128, 1152, 0}, {128, 64, 2048, 0},
                                 {128, 128, 1280, 0}, {128, 64, 1152, 128}, {128, 128, 1152, 384},
                                 {128, 64, 1152, 640}};
  for (auto& s : shapes) {
    mma_shape<<<1, 128, 80 * 1024>>>(n_mma, s[0], s[1], s[2], s[3], d);
    long long c = 0;
    cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
    const double per = (double)c / n_mma;
    const double flop_clk = 2.0 * s[0] * s[1] * 16 / per;
    printf("M=%3u N=%3u A-SBO=%4u A-start+%3u: %.1f cycles/MMA, %.0f FLOP/clk/SM (%s)\n", s[0], s[1], s[2], s[3], per, flop_clk,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
