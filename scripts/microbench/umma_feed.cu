// How fast can an SM feed 128-row x 64-column bf16 A blocks (16 KB, the QKV kernel's X k-blocks) while its
// tensor core runs a stream of M=128 N=192 K=16 MMAs (the QKV projection's shape)?  All 148 SMs run the
// same loop over an L2-resident [rows x 384] bf16 matrix (every CTA its own rows), so the L2 / crossbar
// load is that of the real kernel.
//   feed 0: TMA boxes into a 3-slot smem ring (producer thread waits full, re-issues)     -- today's A ring
//   feed 1: 4 loader warps (one per TMEM lane quadrant), each lane its row: 4 x 32-byte ld.global per
//           block into registers (two blocks in flight), then tcgen05.st into a 2-slot TMEM ring
//   mma 0: no MMAs; 1: SS MMAs (A and B from smem, 10 KB read per MMA); 2: TS MMAs (A from TMEM, B smem)
// Prints the feed's bytes per clock per SM and the MMA issue rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_feed umma_feed.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../../paper_2605_01060_b200/csrc/common.cuh"
using namespace surge;

constexpr int ROWS_PER_CTA = 128 * 64;   // 64 tiles of 128 rows per CTA (L2 resident: 148 x 6 MB... see host)
constexpr int D = 384;

__device__ __forceinline__ void ld_v8(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap tm, const uint16_t* X, int feed,
                                             int mma, int n_blocks, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                 // 3 x 16 KB A ring
  uint8_t* sB = sm + 3 * 16384;     // 144 KB B (garbage weights)
  __shared__ uint64_t full[3], empty[3], mbar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 3; ++s) { mbar_init(&full[s], feed == 0 ? 1 : 4); mbar_init(&empty[s], 1); }
    mbar_init(&mbar, 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == 2) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  const int row0 = (blockIdx.x / 6) * ROWS_PER_CTA;   // groups of six CTAs read the same rows (six slices)
  if (warp == 0) {
    // ------------------------------------------------------------------ MMA stream (until the feed ends)
    constexpr uint32_t idesc = umma_idesc_bf16(128, 192);
    const uint64_t ad = umma_desc_sw128(smem_u32(sA)), bd = umma_desc_sw128(smem_u32(sB));
    long long n = 0;
    const long long t0 = clock64();
    if (mma) {
      while (!done) {
        for (int i = 0; i < 64; ++i) {
          if (elect_one()) {
            if (mma == 1) tc_mma_bf16(tb, ad + uint64_t((i & 3) * 2), bd + uint64_t((i & 7) * 2), idesc, 1);
            else mma_ts(tb, tb + 256 + 8 * (i & 3), bd + uint64_t((i & 7) * 2), idesc, 1);
            if (i == 63) tc_commit(&mbar);
          }
          __syncwarp();
        }
        mbar_wait(&mbar, (n >> 6) & 1);
        n += 64;
      }
    }
    if (lane == 0) out[blockIdx.x * 4 + 1] = n, out[blockIdx.x * 4 + 2] = clock64() - t0;
  } else if (warp == 1 && feed == 0) {
    // ------------------------------------------------------------------ TMA ring, consumer = this thread
    if (lane == 0) {
      const long long t0 = clock64();
      for (int b = 0; b < 3 && b < n_blocks; ++b) {
        mbar_arrive_expect_tx(&full[b], 16384);
        tma_load_2d(sA + b * 16384, &tm, &full[b], (b % 6) * 64, row0 + (b / 6) * 128 % ROWS_PER_CTA);
      }
      for (int b = 0; b < n_blocks; ++b) {
        const int s = b % 3;
        mbar_wait(&full[s], (b / 3) & 1);
        const int nb = b + 3;
        if (nb < n_blocks) {
          mbar_arrive_expect_tx(&full[s], 16384);
          tma_load_2d(sA + s * 16384, &tm, &full[s], (nb % 6) * 64, row0 + ((nb / 6) * 128) % ROWS_PER_CTA);
        }
      }
      out[blockIdx.x * 4 + 0] = clock64() - t0;
      done = 1;
    }
  } else if (warp >= 4 && feed == 1) {
    // ------------------------------------------------------------------ LDG -> registers -> TMEM ring
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t tl = tb + (uint32_t(q * 32) << 16) + 256;
    const long long t0 = clock64();
    uint32_t r0[32], r1[32], r2[32];     // three blocks in flight per lane (48 KB per SM, like the A ring)
    auto load = [&](int b, uint32_t (&v)[32]) {
      if (b >= n_blocks) return;
      const uint16_t* p = X + size_t(row0 + ((b / 6) * 128) % ROWS_PER_CTA + r) * D + (b % 6) * 64;
#pragma unroll
      for (int i = 0; i < 4; ++i) ld_v8(p + 16 * i, *reinterpret_cast<uint32_t(*)[8]>(&v[8 * i]));
    };
    auto st = [&](int b, uint32_t (&v)[32]) {
#pragma unroll
      for (int i = 0; i < 4; ++i) tmem_st8(tl + 32 * (b & 1) + 8 * i, &v[8 * i]);
    };
    load(0, r0);
    load(1, r1);
    for (int b = 0; b < n_blocks; b += 3) {
      load(b + 2, r2);
      st(b, r0);
      load(b + 3, r0);
      st(b + 1, r1);
      load(b + 4, r1);
      st(b + 2, r2);
    }
    tmem_st_wait();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (q == 0 && lane == 0) {
      out[blockIdx.x * 4 + 0] = clock64() - t0;
      done = 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tb, 512);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t rows = size_t(sms / 6 + 1) * ROWS_PER_CTA;
  uint16_t* X;
  cudaMalloc(&X, rows * D * 2);
  cudaMemset(X, 0, rows * D * 2);
  long long* out;
  cudaMalloc(&out, sms * 4 * sizeof(long long));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {D, rows};
  cuuint64_t strides[1] = {D * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 3 * 16384 + 144 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("X: %zu MB; groups of 6 CTAs stream the same %d rows\n", rows * D * 2 >> 20, ROWS_PER_CTA);
  for (int feed = 0; feed < 2; ++feed)
    for (int mma = 0; mma < 3; ++mma) {
      if (feed == 0 && mma == 2) continue;
      const int nb = 6 * 64 * 2;   // 128 tiles of 6 k-blocks
      for (int rep = 0; rep < 2; ++rep) k<<<sms, 256, smem>>>(tm, X, feed, mma, nb, out);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[4 * 200];
      cudaMemcpy(h, out, sms * 4 * sizeof(long long), cudaMemcpyDeviceToHost);
      double cyc = 0, mm = 0, mcyc = 0;
      for (int b = 0; b < sms; ++b) cyc += h[4 * b], mm += h[4 * b + 1], mcyc += h[4 * b + 2];
      cyc /= sms, mm /= sms, mcyc /= sms;
      printf("feed %s mma %s: %.1f B/clk/SM feed (%.0f cyc per 96 KB tile); MMA %.1f cyc/instr (%s)\n",
             feed ? "LDG->TMEM" : "TMA->smem", mma == 0 ? "none" : mma == 1 ? "SS" : "TS", nb * 16384.0 / cyc,
             cyc / (nb / 6), mm > 0 ? mcyc / mm : 0.0, cudaGetErrorString(e));
    }
  return 0;
}
