// Micro-benchmark: cycles per tcgen05.mma.cta_group::1.kind::f16 (M=128, K=16) for
// several N, operands resident in shared memory (SW128 K-major), single issuing thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_bench tools/mma_bench.cu
#include <cstdio>

#include "../paper_1810_10551_b200/csrc/tp_common.cuh"

void tp_set_error(const char*, ...) {}

__global__ void mma_loop(int n_mma, uint32_t n, long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[8];
  __shared__ uint64_t ready;
  __shared__ uint32_t slot;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    tp::mbar_init(&bar, 1);
    for (int q = 0; q < 8; ++q) tp::mbar_init(&bar2[q], 1);
    tp::mbar_init(&ready, 1);
    tp::mbar_arrive(&ready);
    tp::fence_mbar_init();
  }
  if (threadIdx.x < 32) tp::tmem_alloc(&slot, 512);
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  const uint32_t tmem = slot;
  const bool conv = mode >= 10 && mode < 20;
  if (conv) mode -= 10;
  if ((conv || mode >= 20) ? threadIdx.x < 32 : threadIdx.x == 0) {
    const uint32_t idesc = tp::idesc_f16kind(128, n, false);
    const uint32_t a = tp::smem_u32(base), b = tp::smem_u32(base + 16384);
    long long t0 = clock64();
    const uint64_t a128 = tp::umma_desc(a, 16, 1024, 2), b128 = tp::umma_desc(b, 16, 1024, 2);
    const uint64_t a64 = tp::umma_desc(a, 16, 512, 4), b64 = tp::umma_desc(b + 4096, 16, 512, 4);
    if (mode == 0) {  // SW128, one accumulator, fixed operands
#pragma unroll 4
      for (int i = 0; i < n_mma; ++i)
        if (!conv || tp::elect_one()) tp::mma_bf16(tmem, a128 + 2 * (i & 3), b128 + 2 * (i & 3), idesc, 1);
    } else if (mode == 1) {  // SW64, one accumulator, fixed operands
#pragma unroll 4
      for (int i = 0; i < n_mma; ++i) tp::mma_bf16(tmem, a64 + 2 * (i & 1), b64 + 2 * (i & 1), idesc, 1);
    } else if (mode == 2) {  // SW64, layer-2 pattern: windows moving, 2 accumulators every 6
      for (int i = 0; i < n_mma; i += 12) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int k = 0; k < 2; ++k)
              tp::mma_bf16(tmem + j * n, a64 + (((i / 12) & 1) * 18432 + (j * 8 + dy) * 1024) / 16 + 2 * k,
                           b64 + (dy * 4096) / 16 + 2 * k, idesc, 1);
      }
    } else if (mode >= 30) {  // no-swizzle K-major, 9 taps as 16-B-shifted start addresses (30) / fixed (31)
      // A: [k-block of 8 ch][180 px][16 B], rows = pixels; M=128 = 16 rows x 8 px; SBO 160 B
      const uint32_t plane = 180 * 16;
      uint64_t an = tp::umma_desc(a, plane, 160, 0), bn = tp::umma_desc(b + 40960, 128 * 16 * 2, 128, 0);
      if (mode == 32) {  // canonical interleaved: K-adjacent cores contiguous (LBO 128), 8-row groups 256 B apart
        an = tp::umma_desc(a, 128, 256, 0);
        bn = tp::umma_desc(b + 40960, 128, 256, 0);
      } else if (mode == 33) {  // swapped roles
        an = tp::umma_desc(a, 256, 128, 0);
        bn = tp::umma_desc(b + 40960, 256, 128, 0);
      } else if (mode == 34) {  // swapped plane layout
        an = tp::umma_desc(a, 160, plane, 0);
        bn = tp::umma_desc(b + 40960, 128, 128 * 16 * 2, 0);
      }
      for (int i = 0; i < n_mma; i += 9) {
#pragma unroll
        for (int t = 0; t < 9; ++t) {
          const uint32_t off = mode == 30 ? ((t / 3) * 160 + (t % 3) * 16) >> 4 : 0;
          tp::mma_bf16(tmem, an + off, bn, idesc, 1);
        }
      }
    } else if (mode >= 20) {  // warp-convergent; one elect per 12-MMA group (20), + commit (21), + wait (22); 23: one elect for all
      if (mode == 23) {
        if (tp::elect_one()) {
          for (int i = 0; i < n_mma; i += 12) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                for (int k = 0; k < 2; ++k)
                  tp::mma_bf16(tmem + j * n, a64 + (((i / 12) & 1) * 18432 + (j * 8 + dy) * 1024) / 16 + 2 * k,
                               b64 + (dy * 4096) / 16 + 2 * k, idesc, 1);
          }
        }
        __syncwarp();
      } else {
        for (int i = 0; i < n_mma; i += 12) {
          if (tp::elect_one()) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                for (int k = 0; k < 2; ++k)
                  tp::mma_bf16(tmem + j * n, a64 + (((i / 12) & 1) * 18432 + (j * 8 + dy) * 1024) / 16 + 2 * k,
                               b64 + (dy * 4096) / 16 + 2 * k, idesc, 1);
            if (mode >= 21) tp::mma_commit(&bar2[(i / 12) & 7]);
          }
          __syncwarp();
          if (mode >= 22) tp::mbar_wait(&ready, 0);
        }
      }
    } else if (mode >= 4) {  // layer-2 pattern + per-12-MMA sync: 4 commit, 5 commit+wait(ready), 6 +fence
      for (int i = 0; i < n_mma; i += 12) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int k = 0; k < 2; ++k)
              if (!conv || tp::elect_one())
              tp::mma_bf16(tmem + j * n, a64 + (((i / 12) & 1) * 18432 + (j * 8 + dy) * 1024) / 16 + 2 * k,
                           b64 + (dy * 4096) / 16 + 2 * k, idesc, 1);
        if (!conv || tp::elect_one()) tp::mma_commit(&bar2[(i / 12) & 7]);
        __syncwarp(conv ? 0xffffffffu : 1u);
        if (mode >= 5) tp::mbar_wait(&ready, 0);
        if (mode >= 6) tp::tc_fence_after();
      }
    } else {  // SW128, alternating accumulators every MMA
#pragma unroll 4
      for (int i = 0; i < n_mma; ++i) tp::mma_bf16(tmem + (i & 1) * n, a128 + 2 * (i & 3), b128 + 2 * (i & 3), idesc, 1);
    }
    const bool cw = conv || mode >= 20;
    if (!cw || tp::elect_one()) tp::mma_commit(&bar);
    __syncwarp(cw ? 0xffffffffu : 1u);
    tp::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tp::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tp::tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int n_mma = 4096;
  cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  for (int mode : {31, 32, 33, 34})
  for (uint32_t n : {32u, 64u, 128u, 256u}) {
    
    for (int grid : {148}) {
      mma_loop<<<grid, 128, 120 * 1024>>>(n_mma, n, d, mode);
      cudaDeviceSynchronize();
      mma_loop<<<grid, 128, 120 * 1024>>>(n_mma, n, d, mode);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      double cyc = (double)h[0] / n_mma;
      printf("mode %d N=%3u grid=%3d: %.1f cycles/MMA (floor %.0f) -> %.0f%% of floor rate %s\n", mode, n, grid,
             cyc, 128.0 * n / 256.0, 100.0 * (128.0 * n / 256.0) / cyc,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
