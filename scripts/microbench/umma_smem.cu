// Is SS-mode tcgen05.mma (A and B from shared memory) bounded by shared-memory bandwidth at the
// tile shapes libsurge uses?  One CTA per SM: warp 0 issues N_UMMA tcgen05.mma (cta_group::1,
// M = 128, K = 16, bf16, N swept; operands = garbage smem) and times them; warps 4..15 optionally
// stream ld.shared.v4 over a separate 64 KB buffer at the same time (contending smem readers, like
// an epilogue or attention phase).  If the MMA is smem-bound, its cycles per instruction track
// (A bytes + B bytes) / smem B/clk rather than the tensor floor 128 * N / 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_smem umma_smem.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_2605_01060_b200/csrc/common.cuh"
using namespace surge;

template <int N>
__global__ void __launch_bounds__(512, 1) k(int n_umma, int contend, long long* out, float* sink) {
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
    constexpr uint32_t idesc = umma_idesc_bf16(128, N);
    const long long t0 = clock64();
    for (int i = 0; i < n_umma; ++i) {
      if (elect_one()) {
        tc_mma_bf16(tm, ad + uint64_t((i & 3) * 2), bd + uint64_t((i & 3) * 2), idesc, i != 0);
        if ((i & 63) == 63) tc_commit(&bar);
      }
      __syncwarp();
      if ((i & 63) == 63) mbar_wait(&bar, (i >> 6) & 1);
    }
    const long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    done = 1;
  } else if (warp >= 4 && contend) {
    const uint8_t* buf = sm + 65536;
    uint4 acc = make_uint4(0, 0, 0, 0);
    long long t0 = clock64();
    long long bytes = 0;
    while (!done) {
#pragma unroll 8
      for (int r = 0; r < 32; ++r) {
        uint4 v;
        asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(smem_u32(buf + ((r * 384 + threadIdx.x * 16) & 65535))));
        acc.x ^= v.x; acc.y += v.y; acc.z ^= v.z; acc.w += v.w;
      }
      bytes += 32 * 16;
    }
    long long t1 = clock64();
    sink[blockIdx.x * 512 + threadIdx.x] = float(acc.x ^ acc.y ^ acc.z ^ acc.w);
    if (lane == 0 && blockIdx.x == 0 && warp == 4) { out[1] = t1 - t0; out[2] = bytes * 32 * 12; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tm, 256);
}

template <int N>
void run(long long* o, float* s) {
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 2);
  const int NU = 64 * 4000;
  for (int c : {0, 1}) {
    long long h[3] = {0, 0, 0};
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(o, 0, 64);
      k<N><<<148, 512, 65536 * 2>>>(NU, c, o, s);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, o, 24, cudaMemcpyDeviceToHost);
      if (rep == 1)
        printf("N=%3d contend=%d: %.1f cycles/MMA (tensor floor %d; smem bytes/MMA A %d + B %d -> %.1f B/clk)"
               "  contending readers %.1f B/clk  %s\n",
               N, c, double(h[0]) / NU, 128 * N / 256, 4096, 32 * N, (4096.0 + 32 * N) / (double(h[0]) / NU),
               h[1] ? double(h[2]) / double(h[1]) : 0.0, cudaGetErrorString(e));
    }
  }
}

// cta_group::2 (the shape libsurge's fused kernels use): a cluster of 2 CTAs, M = 256 (128 rows per
// CTA), each CTA holds half of B's N rows; the leader issues.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) kp(int n_umma, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool leader = cluster_ctarank() == 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 1) { tmem_alloc_pair(&slot, 256); tmem_relinquish_pair(); }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 0 && leader) {
    const uint64_t ad = umma_desc_sw128(smem_u32(sm)), bd = umma_desc_sw128(smem_u32(sm + 16384));
    constexpr uint32_t idesc = umma_idesc_bf16(256, N);
    const long long t0 = clock64();
    for (int i = 0; i < n_umma; ++i) {
      if (elect_one()) {
        tc_mma_bf16_pair(tm, ad + uint64_t((i & 3) * 2), bd + uint64_t((i & 3) * 2), idesc, i != 0);
        if ((i & 63) == 63) tc_commit_pair_mc(&bar, 0x1);
      }
      __syncwarp();
      if ((i & 63) == 63) mbar_wait(&bar, (i >> 6) & 1);
    }
    const long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) tmem_dealloc_pair(tm, 256);
}

template <int N>
void run_pair(long long* o) {
  cudaFuncSetAttribute(kp<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int NU = 64 * 4000;
  long long h[1] = {0};
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(o, 0, 64);
    kp<N><<<148, 128, 65536>>>(NU, o);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, o, 8, cudaMemcpyDeviceToHost);
    if (rep == 1)
      printf("pair M=256 N=%3d: %.1f cycles/MMA (tensor floor %d per SM; smem bytes/MMA/SM A 4096 + B %d)  %s\n", N,
             double(h[0]) / NU, N / 2, 32 * N, cudaGetErrorString(e));
  }
}

int main() {
  long long* o; float* s; cudaMalloc(&o, 64); cudaMalloc(&s, 148 * 512 * 4);
  run<64>(o, s);
  run<128>(o, s);
  run<192>(o, s);
  run<256>(o, s);
  run_pair<64>(o);
  run_pair<128>(o);
  run_pair<192>(o);
  run_pair<256>(o);
  return 0;
}
