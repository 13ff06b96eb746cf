// mma.sync m16n8k16 bf16 latency (dependent chain) and throughput (8 independent chains) on sm_100a.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <int CH>
__global__ void k(float* out, long long* cyc, int iters) {
  uint32_t a[4] = {threadIdx.x, 2u, 3u, 4u};
  float d[CH][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) mma(d[c], a, i, c);
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8 * 1024);
  long long h;
  const int it = 4096;
  k<1><<<1, 32>>>(o, c, it); cudaDeviceSynchronize();
  k<1><<<1, 32>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("1 warp, dependent chain: %.1f cycles/HMMA\n", double(h) / it);
  k<8><<<1, 32>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("1 warp, 8 chains: %.2f cycles/HMMA\n", double(h) / it / 8);
  k<8><<<1, 128>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("4 warps (1/SMSP), 8 chains: %.2f cycles/HMMA per warp\n", double(h) / it / 8);
  k<8><<<1, 512>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("16 warps, 8 chains: %.2f cycles/HMMA per warp -> %.1f HMMA/clk/SM\n", double(h) / it / 8, 16.0 * it * 8 / h);
  return 0;
}
