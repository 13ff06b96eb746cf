// TMA ingest microbenchmark v2: P producer threads (warps) per CTA, each with its own S-stage ring
// of R x 64 bf16 boxes (128B swizzle).  Reports aggregate GB/s into smem (L2-resident buffer).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void tma2d(void* dst, const void* map, uint64_t* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su32(dst)), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(su32(bar)) : "memory"); }

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap m, int R, int nboxes_r, int nboxes_c, int S, int P, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int box = R * 128;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  const int w = threadIdx.x >> 5;
  if (w >= P || (threadIdx.x & 31)) return;
  uint8_t* buf = base + w * S * box;
  uint64_t* bar = (uint64_t*)(base + P * S * box) + w * S;
  for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  const int total = nboxes_r * nboxes_c;
  unsigned long long acc = 0;
  int issued = 0;
  const int stride = gridDim.x * P;
  const int me = blockIdx.x * P + w;
  for (; issued < S && issued < iters; ++issued) {
    int b = (me + issued * stride) % total;
    mbar_expect(&bar[issued % S], box);
    tma2d(buf + (issued % S) * box, &m, &bar[issued % S], (b % nboxes_c) * 64, (b / nboxes_c) * R);
  }
  for (int done = 0; done < iters; ++done) {
    int s = done % S; uint32_t ph = (done / S) & 1;
    mbar_wait(&bar[s], ph);
    acc += buf[s * box + (done & 1023)];
    if (issued < iters) {
      int b = (me + issued * stride) % total;
      mbar_expect(&bar[s], box);
      tma2d(buf + s * box, &m, &bar[s], (b % nboxes_c) * 64, (b / nboxes_c) * R);
      ++issued;
    }
  }
  sink[me] = acc;
}

int main() {
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink; cudaMalloc(&sink, 65536 * 8);
  size_t cols = 384, rows = 48ull * 1024 * 1024 / (cols * 2);
  void* p; cudaMalloc(&p, rows * cols * 2); cudaMemset(p, 1, rows * cols * 2);
  for (int R : {64, 128, 256}) {
    CUtensorMap m; cuuint64_t dims[2] = {cols, rows}; cuuint64_t str[1] = {cols * 2}; cuuint32_t box[2] = {64, (cuuint32_t)R}; cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int P : {1, 2, 4}) for (int S : {2, 4}) {
      int smem = P * S * R * 128 + 1024 + P * S * 8 + 64;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int iters = 4000 * 128 / R / P;
      k<<<sms, 128, smem>>>(m, R, rows / R, cols / 64, S, P, 50, sink);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<sms, 128, smem>>>(m, R, rows / R, cols / 64, S, P, iters, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double bytes = double(sms) * P * iters * R * 128;
      printf("box %3dx64  producers %d  stages %d : %7.1f GB/s  (%.1f B/clk/SM @1.9GHz) %s\n", R, P, S, bytes / ms / 1e6, bytes / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
