// Micro-benchmark: cycles per tcgen05.ld (TMEM -> registers) for the epilogue shapes the
// conv kernels use, per warp, with 1..8 loads in flight before tcgen05.wait::ld, and with
// 1..16 warps of the CTA loading at once (all 4 TMEM lane quadrants, several warps per
// quadrant). Answers: is an epilogue bound by TMEM load latency (more loads in flight
// help) or by a per-quadrant datapath (more warps per quadrant do not)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_ld_bench tools/tmem_ld_bench.cu
#include <cstdio>

#include "../paper_1810_10551_b200/csrc/tp_common.cuh"

void tp_set_error(const char*, ...) {}

__device__ __forceinline__ void ld_16x256b_x2(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// shape 0: 32x32b.x16 (16 columns x 32 lanes, 2 KB per warp-instruction)
// shape 1: 16x256b.x2 (16 lanes x 16 columns, 1 KB per warp-instruction)
template <int SHAPE, int INFLIGHT>
__global__ void ld_loop(int iters, int active_warps, long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 0) tp::tmem_alloc(&slot, 512);
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  const uint32_t tmem = slot;
  uint32_t acc = 0;
  long long t = 0;
  if ((int)warp < active_warps) {
    const uint32_t row = tmem + (((warp & 3) * 32u) << 16) + (warp >> 2) * 64u;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (SHAPE == 0) {
        uint32_t v[INFLIGHT][16];
#pragma unroll
        for (int k = 0; k < INFLIGHT; ++k) tp::tmem_ld16(row + (uint32_t)(16 * (k & 3)), v[k]);
        tp::tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < INFLIGHT; ++k)
#pragma unroll
          for (int j = 0; j < 16; ++j) acc += v[k][j];
      } else {
        uint32_t v[INFLIGHT][8];
#pragma unroll
        for (int k = 0; k < INFLIGHT; ++k) ld_16x256b_x2(row + (uint32_t)(16 * (k & 3)), v[k]);
        tp::tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < INFLIGHT; ++k)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc += v[k][j];
      }
    }
    t = clock64() - t0;
  }
  if ((threadIdx.x & 31) == 0 && (int)warp < active_warps) out[warp] = t;
  if (acc == 0x12345678u) sink[0] = acc;
  tp::tc_fence_before();
  __syncthreads();
  tp::tc_fence_after();
  if (warp == 0) tp::tmem_dealloc(tmem, 512);
}

template <int SHAPE, int INFLIGHT>
void run(int warps) {
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 32 * sizeof(long long));
  cudaMalloc(&sink, 4);
  const int iters = 2000;
  ld_loop<SHAPE, INFLIGHT><<<1, 512>>>(iters, warps, d, sink);
  ld_loop<SHAPE, INFLIGHT><<<1, 512>>>(iters, warps, d, sink);
  long long h[32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
  const double per_ld = (double)mx / iters / INFLIGHT;
  const double bytes = SHAPE == 0 ? 2048.0 : 1024.0;
  printf("%-12s in-flight %d warps %2d: %7.1f cycles per load per warp, SM total %7.1f B/clk\n",
         SHAPE == 0 ? "32x32b.x16" : "16x256b.x2", INFLIGHT, warps, per_ld,
         bytes * warps / per_ld);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run<0, 1>(w);
    run<0, 2>(w);
    run<0, 4>(w);
    run<1, 1>(w);
    run<1, 2>(w);
    run<1, 4>(w);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
