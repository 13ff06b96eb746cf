// ln_pair.cu -- K6 / K8 for hidden sizes whose LayerNorm row does not fit one CTA's TMEM (d = 768, 1024:
// the bge-base / bge-large classes):  C = LN(A B^T + b + R) * gamma + beta.
//
// A cluster of two CTAs (cta_group::1 each) shares a 128-row M tile and splits the d output columns: CTA r
// owns columns [r d/2, (r+1) d/2) -- its accumulator (384 or 512 fp32 columns) fills its TMEM.  The row
// statistics cross the pair through distributed shared memory: after its first LN pass each epilogue warp
// writes its part's (shift, S1, S2) into both CTAs' stats arrays (st.shared::cluster) and arrives on the
// peer's mbarrier (release.cluster); every warp then merges the four parts in the same order (Chan), so
// both halves of a row are normalised with identical mean and variance.  The fp32 pre-LN rows never reach
// HBM (the separate path writes them and runs a row-LayerNorm kernel: 4 + 4 + 2 bytes per element more).
//
// Warps: 0, 2, 3 TMA producers (A box + this CTA's B rows per k-block, ring of STAGES); 1 MMA issuer; 2
// also allocates TMEM; 4..11 epilogue (epi_ln.cuh, 2 warps per lane quadrant).  Persistent over M tiles
// (tile = cluster index, stride = number of clusters).  One accumulator: the epilogue of tile t and the
// mainloop of tile t + 1 do not overlap (as in the d = 384 LN GEMM).
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "epi_ln.cuh"
#include "internal.h"

namespace surge {

namespace {

constexpr int BM = 128;
constexpr int EPI_WARPS = 8;
#ifndef LN_PAIR_RES_PREFETCH
#define LN_PAIR_RES_PREFETCH 1
#endif
constexpr int THREADS = 128 + 32 * EPI_WARPS;

// LN_PAIR_SPLIT (384 columns per CTA, i.e. d = 768): the tile's mainloop runs as two passes over K -- output
// columns [0, 128) (N = 128 MMAs) into the 128 TMEM columns the previous tile's LayerNorm does not use, then
// columns [128, 384) (N = 256) once that LayerNorm has drained -- so the first pass overlaps the previous
// tile's epilogue (the A k-blocks are streamed twice).  The 128-column region alternates between TMEM columns
// [384, 512) (even tiles) and [0, 128) (odd tiles); the epilogue reads it through epi_ln's column remap.
// Measured (bge-base, 500K texts): out-proj + LN 171.4 -> 171.6 ms, FFN2 + LN 397.5 -> 411.7 ms, so off.
// The epilogue is not what bounds the kernel (ncu: the epilogue warps wait on the accumulator, the MMA issuer
// on the ring: 64 KB per k-block per 792 MMA cycles); halving the per-CTA weight stream by multicast over two
// M tiles (LN_PAIR_MT = 2) was slower too, so it is the ring's latency, not L2 bandwidth.
// LN_PAIR_MT = 2: a cluster of 2 CL CTAs covers two 128-row M tiles; the two CTAs of the same column part
// stream the same weight rows, so each loads half of every k-block's B boxes and multicasts them to both
// (the L2 -> SM weight stream per CTA halves); a ring slot is refilled once both consumers released it.
// Measured slower (bge-base FFN2 + LN 398 -> 427 ms per 500K texts, bge-large 588 -> 646 ms, with SM clocks
// 1.43 -> 1.48 GHz: less power, the two M tiles lock-stepped), so 1.
#ifndef LN_PAIR_MT
#define LN_PAIR_MT 1
#endif
__device__ __forceinline__ void tma_load_2d_mc_hint(void* smem_dst, const void* desc, uint64_t* bar, int32_t c0,
                                                    int32_t c1, uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5, %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc1(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
#ifndef LN_PAIR_SPLIT
#define LN_PAIR_SPLIT 0
#endif
template <int BNC, int CL>   // columns per CTA (d / CL), CTAs per cluster
struct LnPairCfg {
  static constexpr bool SPLIT = LN_PAIR_SPLIT && BNC == 384 && LN_PAIR_KB == 64 && LN_PAIR_MT == 1;
  static constexpr int N_MMA = BNC <= 256 ? 1 : 2;            // 192 / 256: one MMA, 384: 2 x 192, 512: 2 x 256
  // TMEM accumulators: two when 2 BNC <= 512 columns (clusters of 3 / 4 CTAs at d = 768 / 1024), so the
  // LayerNorm epilogue of tile t overlaps the mainloop of tile t + 1
  static constexpr int ACC = (!SPLIT && 2 * BNC <= 512) ? 2 : 1;
  static constexpr int MMA_N = BNC / N_MMA;
  static constexpr int KB = LN_PAIR_KB;                       // k-block width (elements)
  static constexpr int ROWB = KB * 2;                         // bytes per row of a k-block (= swizzle span)
  static constexpr int A_STAGE = BM * ROWB;                   // 8 / 16 KB
  static constexpr int B_STAGE = (SPLIT ? 256 : BNC) * ROWB;  // 24 / 32 KB (KB 32), 48 / 64 KB (KB 64); SPLIT 32 KB
  static constexpr int B_BOX = KB == 32 ? 128 : LN_PAIR_BBOX64 ? LN_PAIR_BBOX64 : BNC / 2;   // rows per B box (model.cu maps)
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr int HEAD = 1024;
  static constexpr int STATS = 2 * 2 * CL * BM * 16;          // [tile parity][2 CL parts][128 rows] float4
  static constexpr int CONSTS = 3 * BNC * 4;                  // bias, gamma, beta of this CTA's columns
  static constexpr int FIXED = HEAD + STATS + ((CONSTS + 1023) / 1024) * 1024;
  static constexpr int STAGES = (227 * 1024 - FIXED) / STAGE;
  static constexpr int SMEM = FIXED + STAGES * STAGE;
  static_assert(STAGES >= 2, "ring");
  static_assert(!SPLIT || B_BOX == 64, "the split mainloop loads 64-row weight boxes");
};

__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// The peers' statistics: this part's (shift, S1, S2) also lands in every peer CTA's stats array (same
// smem offset) and the warp arrives on each peer's `pstats`; wait() blocks on this CTA's own `pstats`.
template <int CL>
struct PairMerge {
  static constexpr int NPM = 2 * CL;
  int off;              // 2 * cluster rank
  uint32_t stats_cta;   // this CTA's stats slot (shared::cta address)
  uint32_t bar_cta;     // this tile's pstats barrier (shared::cta address) in every CTA
  uint64_t* my_bar;
  uint32_t parity;
  int lane, rank;       // rank = column part within the row's CL CTAs
  int base = 0;         // cluster rank of the row group's part 0 (LN_PAIR_MT > 1: m_sub * CL)
  __device__ __forceinline__ int part_off() const { return off; }
  __device__ __forceinline__ void publish(int part, int row, float4 v) const {
#pragma unroll
    for (int pr = 1; pr < CL; ++pr) {
      const uint32_t peer = uint32_t(base + (rank + pr) % CL);
      asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                       mapa_shared(stats_cta + uint32_t((part * 128 + row) * 16), peer)),
                   "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                   : "memory");
    }
    __syncwarp();
    if (lane == 0)
#pragma unroll
      for (int pr = 1; pr < CL; ++pr)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                         mapa_shared(bar_cta, uint32_t(base + (rank + pr) % CL)))
                     : "memory");
  }
  __device__ __forceinline__ void wait() const { mbar_wait_acq_cluster(my_bar, parity); }
};

template <int BNC, int CL, int MT>
__global__ void __launch_bounds__(THREADS, 1)
    ln_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmR, int M, int N,
                   int K, const float* __restrict__ bias, const uint16_t* __restrict__ res,
                   const float* __restrict__ gamma, const float* __restrict__ beta, uint16_t* __restrict__ C,
                   float eps) {
  using T = LnPairCfg<BNC, CL>;
  constexpr int STAGES = T::STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);   // [STAGES]
  uint64_t* empty = full + STAGES;                      // [STAGES]
  uint64_t* tfull = empty + STAGES;                     // [ACC] accumulator complete (commit)
  uint64_t* tempty = tfull + 2;                         // [ACC] accumulator drained (8 epilogue warps); SPLIT: [2], tile % 2
  // [2] the peer's 8 epilogue warps published tile it's statistics (barrier it % 2): two barriers, so the peer
  // (which may publish tile it + 1 before this CTA waits for tile it) can never complete a phase this CTA
  // has not observed yet
  uint64_t* pstats = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pstats + 2);
  float4* stats = reinterpret_cast<float4*>(smem + T::HEAD);                  // [2][2 CL][128]
  float* s_bias = reinterpret_cast<float*>(smem + T::HEAD + T::STATS);
  float* s_gamma = s_bias + BNC;
  float* s_beta = s_gamma + BNC;
  uint8_t* sRing = smem + T::FIXED;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = int(cluster_ctarank());
  const int rank = crank % CL, m_sub = crank / CL;   // column part; M tile within the cluster's MT
  const int n0 = rank * BNC;
  // M tiles: cluster u handles tiles MT u + m_sub, u = cluster index, stride = number of clusters; with MT > 1
  // every CTA of the cluster runs the same number of units (a tile >= m_tiles is a dummy: its A rows are
  // zero-filled by TMA, its stores and residual loads masked) because they share the weight stream
  const int u0 = int(blockIdx.x) / (CL * MT), du = int(gridDim.x) / (CL * MT);
  const int m_units = ((M + BM - 1) / BM + MT - 1) / MT;
  const int m_tiles = m_units * MT;                     // loop bound on units (t = MT u + m_sub)
  const int t0 = MT * u0 + m_sub, dt = MT * du;
  uint16_t bmask = 0;                                   // CTAs sharing this CTA's weight rows
#pragma unroll
  for (int j = 0; j < MT; ++j) bmask |= uint16_t(1u << (rank + CL * j));
  const int num_kb = K / T::KB;

  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023u) != 0) __trap();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmR);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MT);                         // released by every CTA the slot's B boxes land in
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    mbar_init(&tempty[0], EPI_WARPS);
    mbar_init(&tempty[1], EPI_WARPS);
    mbar_init(&pstats[0], (CL - 1) * EPI_WARPS);
    mbar_init(&pstats[1], (CL - 1) * EPI_WARPS);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  cluster_sync();                        // both CTAs' barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 || warp == 2 || warp == 3) {
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producers
      const int p = warp == 0 ? 0 : warp - 1;
      const uint64_t pol_w = l2_policy_evict_last();
      griddep_wait();
      uint32_t c = 0;
      constexpr int NBOX = 1 + BNC / T::B_BOX;            // A + this CTA's B rows in B_BOX-row boxes
      if constexpr (T::SPLIT) {
        uint32_t box = 0;                                 // running box index (boxes go round-robin)
        for (int t = t0; t < m_tiles; t += dt)
          for (int pass = 0; pass < 2; ++pass) {
            const int nb = pass ? 4 : 2, brow = pass ? 128 : 0;   // 64-row B boxes of this pass
            for (int kb = 0; kb < num_kb; ++kb, ++c) {
              const int s = int(c % STAGES);
              const uint32_t ph = (c / STAGES) & 1;
              for (int b = 0; b <= nb; ++b, ++box) {
                if (int(box % 3) != p) continue;
                mbar_wait(&empty[s], ph ^ 1);
                if (b == 0) {
#if LN_PAIR_RES_PREFETCH
                  if (pass == 0 && K <= 1024 && kb * 64 < BNC) tma_prefetch_2d(&tmR, n0 + kb * 64, t * BM);
#endif
                  mbar_arrive_expect_tx(&full[s], uint32_t(T::A_STAGE + nb * 64 * 128));
                  tma_load_2d(sRing + s * T::STAGE, &tmA, &full[s], kb * 64, t * BM);
                } else {
                  tma_load_2d_hint(sRing + s * T::STAGE + T::A_STAGE + (b - 1) * 64 * 128, &tmB, &full[s], kb * 64,
                                   n0 + brow + (b - 1) * 64, pol_w);
                }
              }
            }
          }
      } else
      for (int t = t0; t < m_tiles; t += dt)
        for (int kb = 0; kb < num_kb; ++kb, ++c) {
          const int s = int(c % STAGES);
          const uint32_t ph = (c / STAGES) & 1;
          for (int b = 0; b < NBOX; ++b) {
            if (int((c * NBOX + b) % 3) != p) continue;
            mbar_wait(&empty[s], ph ^ 1);
            if (b == 0) {
#if LN_PAIR_RES_PREFETCH
              // warm L2 with this tile's residual rows of this CTA's columns (read, one row per lane, by the
              // LN epilogue after the mainloop): one 64-column box per k-block while they last.  Only for the
              // out-projection (K = d): bge-base out-proj + LN 179.7 -> 171.1 ms per 500K texts; with FFN2's
              // long weight stream (K = 4 d) it measured +0.7% / +2.5% (bge-base / bge-large)
              if (K <= 1024 && kb * 64 < BNC) tma_prefetch_2d(&tmR, n0 + kb * 64, t * BM);
#endif
              mbar_arrive_expect_tx(&full[s], uint32_t(T::STAGE));
              tma_load_2d(sRing + s * T::STAGE, &tmA, &full[s], kb * T::KB, t * BM);
            } else if (MT == 1) {
              tma_load_2d_hint(sRing + s * T::STAGE + T::A_STAGE + (b - 1) * T::B_BOX * T::ROWB, &tmB, &full[s],
                               kb * T::KB, n0 + (b - 1) * T::B_BOX, pol_w);
            } else if ((b - 1) % MT == m_sub) {   // this CTA's share of the B boxes, into both CTAs' rings
              tma_load_2d_mc_hint(sRing + s * T::STAGE + T::A_STAGE + (b - 1) * T::B_BOX * T::ROWB, &tmB, &full[s],
                                  kb * T::KB, n0 + (b - 1) * T::B_BOX, bmask, pol_w);
            }
          }
        }
    }
  } else if (warp == 1) {
    griddep_launch_dependents();
    // -------------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(BM, T::MMA_N);
    const uint64_t r0 = T::KB == 32 ? umma_desc_sw64(smem_u32(sRing)) : umma_desc_sw128(smem_u32(sRing));
    uint32_t c = 0;
    int it = 0;
    if constexpr (T::SPLIT) {
      constexpr uint32_t id128 = umma_idesc_bf16(BM, 128), id256 = umma_idesc_bf16(BM, 256);
      for (int t = t0; t < m_tiles; t += dt, ++it) {
        for (int pass = 0; pass < 2; ++pass) {
          // pass 0: columns [0, 128) into the region tile it - 2 used (drained by its LayerNorm); pass 1:
          // columns [128, 384) into [128, 384) once tile it - 1's LayerNorm has drained them
          const int prev = pass ? it - 1 : it - 2;
          if (prev >= 0) mbar_wait(&tempty[prev & 1], (prev >> 1) & 1);
          tc_fence_after();
          const uint32_t dcol = pass ? 128u : ((it & 1) ? 0u : 384u);
          for (int kb = 0; kb < num_kb; ++kb, ++c) {
            const int s = int(c % STAGES);
            mbar_wait(&full[s], (c / STAGES) & 1);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t ad = r0 + uint64_t((s * T::STAGE) >> 4);
              const uint64_t bd = r0 + uint64_t((s * T::STAGE + T::A_STAGE) >> 4);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc_mma_bf16(tmem_base + dcol, ad + uint64_t(k * 2), bd + uint64_t(k * 2), pass ? id256 : id128,
                            (kb | k) != 0);
              tc_commit(&empty[s]);
              if (pass == 1 && kb == num_kb - 1) tc_commit(&tfull[0]);
            }
            __syncwarp();
          }
        }
      }
    } else
    for (int t = t0; t < m_tiles; t += dt, ++it) {
      const int acc = it % T::ACC;
      const uint32_t aph = uint32_t(it / T::ACC) & 1;
      const uint32_t d0 = tmem_base + uint32_t(acc * BNC);
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < num_kb; ++kb, ++c) {
        const int s = int(c % STAGES);
        mbar_wait(&full[s], (c / STAGES) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad = r0 + uint64_t((s * T::STAGE) >> 4);
          const uint64_t bd = r0 + uint64_t((s * T::STAGE + T::A_STAGE) >> 4);
#pragma unroll
          for (int k = 0; k < T::KB / 16; ++k)
#pragma unroll
            for (int j = 0; j < T::N_MMA; ++j)
              tc_mma_bf16(d0 + j * T::MMA_N, ad + uint64_t(k * 2),
                          bd + uint64_t((j * T::MMA_N * T::ROWB + k * 32) >> 4), idesc, (kb | k) != 0);
          if (MT == 1) tc_commit(&empty[s]);
          else tc_commit_mc1(&empty[s], bmask);   // the slot is free here and in the CTA sharing its B boxes
          if (kb == num_kb - 1) tc_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    griddep_wait();
    // ------------------------------------------------------------------ epilogue (warps 4..11)
    for (int i = threadIdx.x - 128; i < BNC; i += 32 * EPI_WARPS) {
      s_bias[i] = bias[n0 + i];
      s_gamma[i] = gamma[n0 + i];
      s_beta[i] = beta[n0 + i];
    }
    asm volatile("bar.sync 5, %0;" ::"r"(32 * EPI_WARPS) : "memory");
    const int q = warp & 3, hh = (warp - 4) >> 2;
    const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16);

    int it = 0;
    for (int t = t0; t < m_tiles; t += dt, ++it) {
      const int row = t * BM + q * 32 + lane;
      const bool ok = row < M;
      float4* st = stats + (it & 1) * 2 * CL * BM;
      const PairMerge<CL> mg{2 * rank, smem_u32(st), smem_u32(&pstats[it & 1]), &pstats[it & 1],
                             uint32_t((it >> 1) & 1), lane, rank, m_sub * CL};
      const ResidualGlobal rg{res + size_t(ok ? row : 0) * N + n0};
      const int acc = it % T::ACC;
      const uint32_t aph = uint32_t(it / T::ACC) & 1;
      auto epi = [&](auto remap_lo, auto remap_base) {
        ln_epilogue<BNC, BNC / 2, true, decltype(remap_lo)::value, decltype(remap_base)::value, float, PairMerge<CL>>(
            taddr + uint32_t(acc * BNC), 0, rg, s_bias, s_gamma, s_beta, st, q, hh, lane, eps,
            [&] {
              mbar_wait(&tfull[acc], aph);
              tc_fence_after();
            },
            [&](const uint32_t (&p)[16], int col) { store_row_64B(p, lane, C, int64_t(t) * BM + q * 32, M, N, n0 + col); },
            LnNoOp{}, mg);
      };
      if (T::SPLIT && !(it & 1))   // even tiles: columns [0, 128) live at TMEM [384, 512)
        epi(std::integral_constant<uint32_t, 128u>{}, std::integral_constant<uint32_t, 384u>{});
      else
        epi(std::integral_constant<uint32_t, 0u>{}, std::integral_constant<uint32_t, 0u>{});
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[T::SPLIT ? (it & 1) : acc]);
    }
  }
  tc_fence_before();
  cluster_sync();                        // no remote stats write / arrive may target an exited CTA
  if (warp == 2) {
    __syncwarp();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int BNC, int CL>
cudaError_t launch_t(const GemmArgs& g, cudaStream_t st) {
  using T = LnPairCfg<BNC, CL>;
  constexpr int MT = LN_PAIR_MT;
  auto kern = ln_pair_kernel<BNC, CL, MT>;
  static int max_clusters = 0;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = size_t(T::SMEM);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL * MT;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (max_clusters == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
    if (e != cudaSuccess) return e;
    if (CL * MT > 8) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    cfg.gridDim = dim3(unsigned(((sms > 0 ? sms : 148) / (CL * MT)) * CL * MT));
    e = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg);
    if (e != cudaSuccess || max_clusters <= 0) return e != cudaSuccess ? e : cudaErrorLaunchOutOfResources;
  }
  const int64_t m_units = ((g.M + BM - 1) / BM + MT - 1) / MT;
  const int clusters = int(std::min<int64_t>(m_units, max_clusters));
  cfg.gridDim = dim3(unsigned(CL * MT * clusters));
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const CUtensorMap tmR = g.tmR ? *g.tmR : *g.tmA;   // residual rows (L2 prefetch only)
  return cudaLaunchKernelEx(&cfg, kern, *g.tmA, *g.tmB, tmR, int(g.M), g.N, g.K, g.bias, g.res, g.gamma, g.beta, g.C,
                            g.eps);
}

}  // namespace

bool ln_pair_supported(int d, int k) { return (d == 768 || d == 1024) && k % LN_PAIR_KB == 0 && k > 0; }

cudaError_t launch_ln_pair(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0) return cudaSuccess;
  if (!ln_pair_supported(g.N, g.K)) return cudaErrorInvalidValue;
#ifndef LN_PAIR_CL768
#define LN_PAIR_CL768 2     // out-projection (K = d): 2 CTAs x 384 columns
#endif
#ifndef LN_PAIR_CL1024
#define LN_PAIR_CL1024 2   // out-projection: 2 x 512
#endif
  // FFN2 (K = 4 d): clusters of 3 / 4 CTAs x 256 columns, which leaves TMEM for two accumulators (the LayerNorm of
  // tile t under the mainloop of tile t + 1): FFN2 + LN 392 -> 380 ms (bge-base, 500K texts), 584 -> 573 ms
  // (bge-large, 200K); the out-projection (short K) measured slower that way (169 -> 181 / 217 -> 231 ms).
#ifndef LN_PAIR_CL768_FFN2
#define LN_PAIR_CL768_FFN2 3
#endif
#ifndef LN_PAIR_CL1024_FFN2
#define LN_PAIR_CL1024_FFN2 4
#endif
  const bool ffn2 = g.K > g.N;
  if (g.N == 768)
    return ffn2 ? launch_t<768 / LN_PAIR_CL768_FFN2, LN_PAIR_CL768_FFN2>(g, st)
                : launch_t<768 / LN_PAIR_CL768, LN_PAIR_CL768>(g, st);
  return ffn2 ? launch_t<1024 / LN_PAIR_CL1024_FFN2, LN_PAIR_CL1024_FFN2>(g, st)
              : launch_t<1024 / LN_PAIR_CL1024, LN_PAIR_CL1024>(g, st);
}

}  // namespace surge
