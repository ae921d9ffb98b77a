// Numerics probe: can a SW128 K-major UMMA operand start at an arbitrary 128-byte row
// offset inside a TMA-style swizzled buffer (1024-B aligned base)? Runs one
// tcgen05.mma (M=128, N=32, K=16) per (row shift, k chunk, base_offset mode) and compares
// with a host product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/swz_shift_test_bin tools/swz_shift_test.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>

#include "../paper_1810_10551_b200/csrc/tp_common.cuh"

void tp_set_error(const char*, ...) {}

constexpr int AR = 768, BR = 32;

__device__ __host__ inline float aval(int r, int k) { return (float)(((r * 7 + k * 3) % 9) - 4); }
__device__ __host__ inline float bval(int n, int k) { return (float)(((n * 5 + k) % 7) - 3); }

// byte offset of element (row, k) in a TMA-swizzled image (SW128: 128-B rows, chunk ^= row&7;
// SW64: 64-B rows, chunk ^= (row>>1)&3), base 1024-aligned. K here spans one row.
__device__ inline uint32_t swz(int r, int k, int rb) {
  const uint32_t kb = (uint32_t)k * 2;
  const uint32_t addr = (uint32_t)r * rb + kb;
  const uint32_t chunk = (addr >> 4) & 7, x = (addr >> 7) & 7;
  return rb == 128 ? (addr & ~0x70u) | ((chunk ^ x) << 4)
                   : (addr & ~0x30u) | ((((addr >> 4) & 3) ^ ((addr >> 7) & 3)) << 4);
}

__global__ void probe(int shift, int kc, int rb, int pitch, float* out) {
  const int K = rb / 2;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* A = base;
  uint8_t* B = base + 96 * 1024;
  for (int i = threadIdx.x; i < AR * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    if (r * rb >= 96 * 1024) continue;
    *reinterpret_cast<__half*>(A + swz(r, k, rb)) = __float2half(aval(r, k));
  }
  for (int i = threadIdx.x; i < BR * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__half*>(B + swz(n, k, rb)) = __float2half(bval(n, k));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    tp::mbar_init(&bar, 1);
    tp::fence_mbar_init();
  }
  if (threadIdx.x < 32) tp::tmem_alloc(&slot, 32);
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint32_t lay = rb == 128 ? 2 : 4;
    const uint32_t a_addr = tp::smem_u32(A) + shift * rb + kc * 32;
    const uint64_t ad = tp::umma_desc(a_addr, 16, pitch * rb, lay);
    const uint64_t bd = tp::umma_desc(tp::smem_u32(B) + kc * 32, 16, 8 * rb, lay);
    if (tp::elect_one()) {
      tp::mma_bf16(tmem, ad, bd, tp::idesc_f16kind(128, 32, false), 0);
      tp::mma_commit(&bar);
    }
    __syncwarp();
  }
  tp::mbar_wait(&bar, 0);
  tp::tc_fence_after();
  const uint32_t w = threadIdx.x >> 5;
  uint32_t v[16];
  for (int c = 0; c < 2; ++c) {
    tp::tmem_ld16(tmem + ((w * 32) << 16) + c * 16, v);
    tp::tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[threadIdx.x * 32 + c * 16 + j] = __uint_as_float(v[j]);
  }
  tp::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tp::tmem_dealloc(tmem, 32);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 32 * sizeof(float));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  float h[128 * 32];
  for (int rb : {128, 64})
  for (int pitch : {8, 9, 10, 18, 34})
    for (int shift : {0, 1, 2, 3, 5, 8, 9, 10, 19}) {
      int bad_total = 0;
      for (int kc = 0; kc < rb / 32; ++kc) {
        probe<<<1, 128, 110 * 1024>>>(shift, kc, rb, pitch, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < 32; ++n) {
            float ref = 0.f;
            const int r = (m / 8) * pitch + (m % 8) + shift;  // 8-row groups at `pitch` rows
            for (int k = kc * 16; k < kc * 16 + 16; ++k) ref += aval(r, k) * bval(n, k);
            if (h[m * 32 + n] != ref) ++bad_total;
          }
      }
      printf("row %3d B pitch %2d shift %2d: %s (%d mismatches)\n", rb, pitch, shift,
             bad_total ? "WRONG" : "ok", bad_total);
    }
  return 0;
}
