// tcgen05.mma issue cost by shape and operand source, to size an on-tensor-core attention for the
// fused QKV kernel: is the ~77-cycle minimum per SS MMA (profiles/r01/umma_smem.log)
// a per-instruction cost, or the read-modify-write dependency on one TMEM accumulator?
//   (1) SS, M = 128, N swept, ND accumulators used round-robin (ND = 1: every MMA accumulates into
//       the same D, as a K loop does);
//   (2) TS: A (the P matrix of an attention) read from TMEM instead of shared memory;
//   (3) SS, M = 64;
//   (4) fp32x2 FMA (FFMA2) throughput per SM, 16 warps of independent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_shapes umma_shapes.cu
#include <cstdint>
#include <cstdio>

#include "../../paper_2605_01060_b200/csrc/common.cuh"
using namespace surge;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// MODE 0: SS, MODE 1: TS (A from TMEM columns [448, 456))
template <int M, int N, int ND, int MODE>
__global__ void __launch_bounds__(128, 1) kshape(int n_umma, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 1) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 0) {
    const uint64_t ad = umma_desc_sw128(smem_u32(sm)), bd = umma_desc_sw128(smem_u32(sm + 16384));
    constexpr uint32_t idesc = umma_idesc_bf16(M, N);
    const long long t0 = clock64();
    for (int i = 0; i < n_umma; ++i) {
      if (elect_one()) {
        const uint32_t d = tm + uint32_t((i % ND) * N);
        if (MODE == 0) tc_mma_bf16(d, ad + uint64_t((i & 3) * 2), bd + uint64_t((i & 3) * 2), idesc, i >= ND);
        else mma_ts(d, tm + 448 + uint32_t((i & 3) * 8) % 64, bd + uint64_t((i & 3) * 2), idesc, i >= ND);
        if ((i & 63) == 63) tc_commit(&bar);
      }
      __syncwarp();
      if ((i & 63) == 63) mbar_wait(&bar, (i >> 6) & 1);
    }
    const long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tm, 512);
}

template <int M, int N, int ND, int MODE>
void run(long long* o) {
  cudaFuncSetAttribute(kshape<M, N, ND, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int NU = 64 * 2000;
  long long h = 0;
  cudaError_t e = cudaSuccess;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(o, 0, 64);
    kshape<M, N, ND, MODE><<<148, 128, 65536>>>(NU, o);
    e = cudaDeviceSynchronize();
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
  }
  printf("%s M=%3d N=%3d ND=%d: %6.1f cycles/MMA (floor %5.1f)  %s\n", MODE ? "TS" : "SS", M, N, ND, double(h) / NU,
         double(M) * N / 256.0, cudaGetErrorString(e));
}

__global__ void __launch_bounds__(512, 1) kffma2(int iters, long long* out, float* sink) {
  f32x2 a[8], b = f2(1.0001f, 0.9999f), c = f2(1e-7f, -1e-7f);
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = f2(float(threadIdx.x + j), float(j));
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = ffma2(a[j], b, c);
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += f2lo(a[j]) + f2hi(a[j]);
  sink[blockIdx.x * 512 + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

__global__ void __launch_bounds__(512, 1) kffma(int iters, long long* out, float* sink) {
  float a[16];
  const float b = 1.0001f, c = 1e-7f;
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = float(threadIdx.x + j);
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], b, c);
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += a[j];
  sink[blockIdx.x * 512 + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  long long* o;
  float* s;
  cudaMalloc(&o, 64);
  cudaMalloc(&s, 148 * 512 * 4);
  run<128, 32, 1, 0>(o);
  run<128, 32, 4, 0>(o);
  run<128, 64, 1, 0>(o);
  run<128, 64, 4, 0>(o);
  run<128, 96, 1, 0>(o);
  run<128, 96, 4, 0>(o);
  run<128, 128, 1, 0>(o);
  run<128, 128, 2, 0>(o);
  run<128, 192, 1, 0>(o);
  run<128, 192, 2, 0>(o);
  run<128, 256, 1, 0>(o);
  run<64, 64, 1, 0>(o);
  run<64, 128, 1, 0>(o);
  run<64, 256, 1, 0>(o);
  run<128, 32, 1, 1>(o);
  run<128, 32, 4, 1>(o);
  run<128, 64, 1, 1>(o);
  run<128, 64, 4, 1>(o);
  run<128, 128, 1, 1>(o);
  run<128, 256, 1, 1>(o);
  {
    const int it = 20000;
    long long h = 0;
    kffma2<<<148, 512>>>(it, o, s);
    cudaDeviceSynchronize();
    kffma2<<<148, 512>>>(it, o, s);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("FFMA2: %.1f FMA/clk/SM (16 warps x 8 independent fp32x2 chains)\n", 512.0 * it * 16 / double(h));
    kffma<<<148, 512>>>(it, o, s);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("FFMA : %.1f FMA/clk/SM (16 warps x 16 independent chains)\n", 512.0 * it * 16 / double(h));
  }
  return 0;
}
