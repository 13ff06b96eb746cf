// Does legacy mma.sync (HMMA) traffic slow tcgen05.mma on the same SM?  One CTA per SM: warp 0 issues
// N_UMMA tcgen05.mma (M=128, N=256, K=16, bf16, operands = garbage smem) and times them; warps 4..15
// optionally run dependent-free HMMA loops at the same time.
#include <cstdio>
#include <cstdint>
#include "../../paper_2605_01060_b200/csrc/common.cuh"
using namespace surge;

__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(512, 1) k(int n_umma, int hmma_iters, long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
  if (warp == 1) { tmem_alloc(&slot, 256); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 0) {
    const uint64_t ad = umma_desc_sw128(smem_u32(sm)), bd = umma_desc_sw128(smem_u32(sm + 16384));
    constexpr uint32_t idesc = umma_idesc_bf16(128, 256);
    const long long t0 = clock64();
    for (int i = 0; i < n_umma; ++i) {
      if (elect_one()) {
        tc_mma_bf16(tm, ad, bd, idesc, i != 0);
        if ((i & 63) == 63) tc_commit(&bar);
      }
      __syncwarp();
      if ((i & 63) == 63) mbar_wait(&bar, (i >> 6) & 1);
    }
    const long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    done = 1;
  } else if (warp >= 4) {
    uint32_t a[4] = {threadIdx.x, 2u, 3u, 4u};
    float d[8][4] = {};
    long long t0 = clock64();
    int it = 0;
    for (; it < hmma_iters && !done; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c) hmma(d[c], a, it, c);
    long long t1 = clock64();
    float s = 0;
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    sink[blockIdx.x * 512 + threadIdx.x] = s;
    if (lane == 0 && blockIdx.x == 0 && warp == 4) { out[1] = t1 - t0; out[2] = it; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tm, 256);
}

int main() {
  long long* o; float* s; cudaMalloc(&o, 64); cudaMalloc(&s, 148 * 512 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  long long h[3];
  const int NU = 64 * 2000;
  for (int hm : {0, 1000000}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(o, 0, 64);
      k<<<148, 512, 65536>>>(NU, hm, o, s);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, o, 24, cudaMemcpyDeviceToHost);
      printf("hmma %s: tcgen05 128x256x16: %.1f cycles/MMA (ideal 64); HMMA warps ran %lld iters in %lld cycles (%.2f HMMA/clk/SM) %s\n",
             hm ? "on " : "off", double(h[0]) / NU, h[2], h[1], h[2] ? 12.0 * 8 * h[2] / double(h[1]) : 0.0,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
