// TMA ingest microbenchmark: each persistent CTA streams 128x64 bf16 boxes (16 KB, 128B swizzle)
// of a [rows x 64*ncol] matrix through an S-stage mbarrier ring, no compute.  Reports aggregate
// bytes/s into shared memory for an L2-resident and a DRAM-sized buffer.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void tma2d(void* dst, const void* map, uint64_t* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su32(dst)), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(su32(bar)) : "memory"); }

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap m, int nboxes_r, int nboxes_c, int S, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  uint64_t* bar = (uint64_t*)(buf + S * 16384);
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int total = nboxes_r * nboxes_c;
  unsigned long long acc = 0;
  int issued = 0, done = 0;
  const int n = iters;  // boxes per CTA
  // prologue
  for (; issued < S && issued < n; ++issued) {
    int b = (blockIdx.x + issued * gridDim.x) % total;
    mbar_expect(&bar[issued % S], 16384);
    tma2d(buf + (issued % S) * 16384, &m, &bar[issued % S], (b % nboxes_c) * 64, (b / nboxes_c) * 128);
  }
  for (; done < n; ++done) {
    int s = done % S; uint32_t ph = (done / S) & 1;
    mbar_wait(&bar[s], ph);
    acc += buf[s * 16384 + (done & 1023)];
    if (issued < n) {
      int b = (blockIdx.x + issued * gridDim.x) % total;
      mbar_expect(&bar[s], 16384);
      tma2d(buf + s * 16384, &m, &bar[s], (b % nboxes_c) * 64, (b / nboxes_c) * 128);
      ++issued;
    }
  }
  sink[blockIdx.x] = acc;
}

int main() {
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink; cudaMalloc(&sink, 4096 * 8);
  for (size_t mb : {48, 2048}) {
    size_t cols = 384, rows = mb * 1024 * 1024 / (cols * 2);
    void* p; cudaMalloc(&p, rows * cols * 2); cudaMemset(p, 1, rows * cols * 2);
    CUtensorMap m; cuuint64_t dims[2] = {cols, rows}; cuuint64_t str[1] = {cols * 2}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int nbr = rows / 128, nbc = cols / 64;
    for (int S : {2, 3, 4, 6, 8, 12}) {
      for (int ctas_per_sm : {1, 2}) {
        int smem = S * 16384 + 2048;
        if (smem * ctas_per_sm > 227 * 1024) continue;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int grid = sms * ctas_per_sm; int iters = 2000;
        k<<<grid, 128, smem>>>(m, nbr, nbc, S, 50, sink);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<grid, 128, smem>>>(m, nbr, nbc, S, iters, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bytes = double(grid) * iters * 16384;
        printf("buf %5zu MB  stages %2d  ctas/SM %d : %7.1f GB/s  (%.1f B/clk/SM at 1.9GHz)  err=%s\n", mb, S, ctas_per_sm, bytes / ms / 1e6,
               bytes / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
      }
    }
    cudaFree(p);
  }
  return 0;
}
