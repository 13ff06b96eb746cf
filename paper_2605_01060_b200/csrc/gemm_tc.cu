// gemm_tc.cu -- K4/K6/K7/K8: bf16 GEMM on 5th-gen tensor cores (tcgen05.mma, accumulators in
// TMEM, operands staged by TMA with 128-byte swizzle) with fused epilogues:
//   EPI_BIAS      C = A B^T + b                          (QKV projection, K4)
//   EPI_BIAS_GELU C = GELU_erf(A B^T + b)                (FFN1, K7)
//   EPI_BIAS_LN   C = LN(A B^T + b + R) * gamma + beta   (attention out-proj K6, FFN2 K8)
// A: [M x K] activations (row-major, K contiguous), B: [N x K] weights (HF nn.Linear [out,in]).
//
// Design: persistent grid (<= #SMs), 128 x BN output tiles, warp-specialised
// (TMA producer, single-thread MMA issuer, TMEM allocator, 8 epilogue warps); accumulators double-
// buffered in TMEM when 2*BN <= 512 so the epilogue of one tile overlaps the next tile's mainloop.
// Rows >= M of the last tile are zero-filled by TMA and never stored.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "attn_tile.cuh"
#include "common.cuh"
#include "epi_ln.cuh"
#include "internal.h"

namespace surge {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;                       // 64 bf16 = 128 B = one swizzle row
constexpr int A_STAGE_BYTES = BM * BK * 2;   // 16 KB

// PAIR: a cluster of two CTAs runs cta_group::2 MMAs on 256 x BN tiles; each CTA holds its 128
// rows of A and of the accumulator, and half of every MMA's N rows of B (so B traffic per CTA
// halves).
template <int BN, int EPI, bool PAIR = false, int DH = 0>
struct TileCfg {
  static constexpr int MMA_N = (BN <= 256) ? BN : BN / 2;       // <= 256, multiple of 16
  static constexpr int N_MMA = BN / MMA_N;
  static constexpr int B_BOX = PAIR ? MMA_N / 2 : MMA_N;         // TMA box rows for B (this CTA)
  static constexpr int N_LOADS = N_MMA;                          // B boxes per k-block
  static constexpr int B_STAGE_BYTES = N_LOADS * B_BOX * 128;    // this CTA's B bytes per k-block
  static constexpr int UMMA_M = PAIR ? 2 * BM : BM;
  static constexpr int ACC = (2 * BN <= 512) ? 2 : 1;            // TMEM accumulator buffers
  static constexpr int ACC_COLS = ACC * BN;
  static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : ACC_COLS <= 64 ? 64 : ACC_COLS <= 128 ? 128
                                   : ACC_COLS <= 256 ? 256 : 512;
  // Epilogue warps: SPLIT per TMEM lane quadrant, each owning BN / SPLIT columns.  The GELU
  // epilogue is issue-bound, so it gets three warps per quadrant (bias then comes from smem to
  // keep registers <= 128 at 512 threads); the others two.
  // The attention epilogue (EPI_QKV_ATTN) runs 12 warps: the (text, head) units of a tile are its
  // critical path.
  static constexpr bool ATT = EPI == EPI_QKV_ATTN;
  // attention epilogue: 16 warps at d_h = 32 (MiniLM; 12 -> 16 warps: QKV+attention 1138 -> 1128
  // ms/step), 12 elsewhere (their attention registers spill at the 96-register cap of 16 warps)
#ifndef ATT_SPLIT32
#define ATT_SPLIT32 4
#endif
  static constexpr int SPLIT = ATT ? (DH == 32 ? ATT_SPLIT32 : 3)
                               : EPI != EPI_BIAS_GELU ? 2 : BN % 128 == 0 ? 4 : BN % 96 == 0 ? 3 : 2;
  static constexpr int EPI_WARPS = 4 * SPLIT;
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr bool BIAS_SMEM = EPI == EPI_BIAS_GELU && SPLIT > 2;
  static constexpr int HEAD_BYTES = 1024;                         // mbarriers + TMEM slot
  static constexpr int STATS_BYTES =                              // LN: stats + bias/gamma/beta, 1 KB aligned
      EPI == EPI_BIAS_LN ? ((2 * 2 * BM * 4 * 4 + 3 * BN * 4 + 1023) / 1024) * 1024 : 0;
  // per-warp output staging buffers (3 for the LN tiles measured slower: out-proj 520 -> 590 ms/step)
  static constexpr int STG_BUFS = 1;
  static constexpr int STG_BYTES = ATT ? 0 : EPI_WARPS * STG_BUFS * 2048;  // 32 rows x 32 cols bf16 each
  // EPI_QKV_ATTN: the tile's Q | K | V (bf16) staged for attention, 128 rows + 16 zero rows read
  // past the last text by a query tile / key block, 16-byte row skew.
  static constexpr int ATT_ROWS = BM + 16;
  static constexpr int ATT_LDS = BN + 8;
  static constexpr int ATT_BYTES = ATT ? ((ATT_ROWS * ATT_LDS * 2 + 2 * ATT_REC_INTS * 4 + 1023) / 1024) * 1024 : 0;
  static constexpr int FIXED_BYTES = 1024 /*align*/ + HEAD_BYTES + STATS_BYTES + STG_BYTES + ATT_BYTES;
  __host__ __device__ static int bias_bytes(int N) { return BIAS_SMEM ? ((N * 4 + 1023) / 1024) * 1024 : 0; }
  static constexpr int MAX_SMEM = 227 * 1024;
  static constexpr int MAX_STAGES = 8;
  static constexpr int HALF = BN / SPLIT;                         // columns per epilogue warp
  static_assert(MMA_N % 16 == 0 && MMA_N >= 16 && MMA_N <= 256, "invalid UMMA N");
  static_assert(B_BOX * N_LOADS * (PAIR ? 2 : 1) == BN, "B box split");
  static_assert(HALF % 32 == 0 || (ATT && HALF % 16 == 0), "epilogue column split");
  // Weight-stationary (ws): the CTA's whole B slice [BN x K] stays resident; only A streams.
  __host__ __device__ static int b_res_bytes(int K, bool ws) { return ws ? (PAIR ? BN / 2 : BN) * K * 2 : 0; }
  __host__ __device__ static int stage_bytes(bool ws) { return A_STAGE_BYTES + (ws ? 0 : B_STAGE_BYTES); }
  __host__ __device__ static int stages(int K, bool ws, int N = 0) {
    const int n = (MAX_SMEM - FIXED_BYTES - bias_bytes(N) - b_res_bytes(K, ws)) / stage_bytes(ws);
    return n > MAX_STAGES ? MAX_STAGES : n;
  }
  __host__ __device__ static int smem_bytes(int K, bool ws, int N = 0) {
    return FIXED_BYTES + bias_bytes(N) + b_res_bytes(K, ws) + stages(K, ws, N) * stage_bytes(ws);
  }
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Tile schedule of one CTA.  Streaming (WS = false): tiles t = blockIdx.x, +gridDim.x, ... over
// (m, n) with n fastest, so concurrently running CTAs share the A rows of one M block in L2.
// Weight-stationary (WS = true): CTA c owns the N slice c % n_tiles for the whole launch (its B
// slice is loaded once and stays in shared memory) and walks M tiles c / n_tiles, + gridDim.x /
// n_tiles, ...; the grid is a multiple of n_tiles.
// PAIR (streaming only): the unit is the cluster (blockIdx.x / 2) and M tiles are 256 rows; CTA
// rank r of the pair owns rows [256 t + 128 r, +128).
// Text-aligned M tiles (EPI_QKV_ATTN): tile i is described by record i (internal.h ATT_REC_INTS
// layout; word 0 = its first row); in PAIR mode unit t is the tile pair (2t, 2t + 1).
struct AttTiles {
  const int32_t* rec;     // nullptr: regular M tiling
  int32_t n;              // tiles (even)
  float qscale;
};

template <bool WS, bool PAIR = false>
struct Sched {
  int t0, dt, tend, n_tiles, slice, rank;
  AttTiles at;
  __device__ Sched(int M, int n_tiles_, const AttTiles& at_) : n_tiles(n_tiles_), at(at_) {
    rank = PAIR ? int(blockIdx.x & 1) : 0;
    const int unit = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
    const int units = PAIR ? int(gridDim.x >> 1) : int(gridDim.x);
    const int m_tiles = at.rec ? (PAIR ? at.n / 2 : at.n)
                                 : (M + (PAIR ? 2 * BM : BM) - 1) / (PAIR ? 2 * BM : BM);
    if (WS) {
      slice = unit % n_tiles;
      t0 = unit / n_tiles;
      dt = units / n_tiles;
      tend = m_tiles;
    } else {
      slice = 0;
      t0 = unit;
      dt = units;
      tend = m_tiles * n_tiles;
    }
  }
  __device__ int mt(int t) const { return WS ? t : t / n_tiles; }
  // text-aligned tile index of this CTA in unit t
  __device__ int att_tile(int t) const { return PAIR ? 2 * mt(t) + rank : mt(t); }
  __device__ int m0(int t) const {
    if (at.rec) return at.rec[size_t(att_tile(t)) * ATT_REC_INTS];
    return mt(t) * (PAIR ? 2 * BM : BM) + rank * BM;
  }
  __device__ int n0(int t) const { return (WS ? slice : t % n_tiles); }
};

// Persistent, warp-specialised tcgen05 GEMM.
//   warps 0,2,3   TMA producers (one lane each): `stages`-deep smem ring (A, plus B when streaming)
//   warp 1        MMA issuer (whole warp, one elected lane): UMMA 128 x MMA_N x 16, accumulator it % ACC
//   warp 2        also the TMEM allocator
//   warps 4..11   epilogue: warp w reads TMEM lane quadrant w % 4, column half (w - 4) / 4;
//                 the accumulator buffer is released as soon as it is drained, so with ACC = 2 the
//                 epilogue of tile i overlaps the mainloop of tile i + 1.
#ifdef ATT_TRACE
#define ATT_TR(i)                                        \
  do {                                                   \
    const long long _c = clock64();                      \
    if (i > 0) tr_acc[i - 1] += _c - tr_last;            \
    tr_last = _c;                                        \
  } while (0)
#else
#define ATT_TR(i) do {} while (0)
#endif

// The MMA issuer's waits: with GEMM_MMA_SPIN the polling loop (the issuer is on the critical path), else the
// default suspend-time-hint wait of common.cuh (A/B: within 0.2% of each other, so the default stays).
#if defined(GEMM_MMA_SPIN) && defined(MBAR_SLEEP_ALL)
#define mma_wait mbar_wait_spin
#else
#define mma_wait mbar_wait
#endif
template <int BN, int EPI, bool WS, bool PAIR, int DH = 0>
__global__ void __launch_bounds__(TileCfg<BN, EPI, PAIR, DH>::THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmR, int M, int N,
                   int K, const float* __restrict__ bias, const uint16_t* __restrict__ res,
                   const float* __restrict__ gamma, const float* __restrict__ beta, uint16_t* __restrict__ C,
                   float eps, int stages, const AttTiles att) {
  using T = TileCfg<BN, EPI, PAIR, DH>;
  constexpr int ACC = T::ACC;
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the __shared__ array (an integer round trip would turn every
  // shared access into a generic one)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);   // [stages]
  uint64_t* empty = full + T::MAX_STAGES;               // [stages]
  uint64_t* tfull = empty + T::MAX_STAGES;              // [ACC]
  uint64_t* tempty = tfull + 2;                         // [ACC]
  uint64_t* bfull = tempty + 2;                         // resident B slice landed (WS)
  uint64_t* att_gate = bfull + 1;                       // ATT: the attention phase of a tile is done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(att_gate + 1);
  float4* stats = reinterpret_cast<float4*>(smem + T::HEAD_BYTES);                  // [2][2][BM]
  float* s_bias = reinterpret_cast<float*>(stats + 2 * 2 * BM);                      // LN: [BN] each
  float* s_gamma = s_bias + BN;
  float* s_beta = s_gamma + BN;
  uint8_t* sStg = smem + T::HEAD_BYTES + T::STATS_BYTES;  // [epi warp][STG_BUFS][2 KB] (1 KB aligned)
  float* s_bias_all = reinterpret_cast<float*>(sStg + T::STG_BYTES);   // BIAS_SMEM: bias[0..N)
  uint16_t* sAtt = reinterpret_cast<uint16_t*>(sStg + T::STG_BYTES + T::bias_bytes(N));   // ATT: [ATT_ROWS][ATT_LDS]
  int32_t* s_rec = reinterpret_cast<int32_t*>(sAtt + T::ATT_ROWS * T::ATT_LDS);   // ATT: [2][ATT_REC_INTS] records
  uint8_t* sB = sStg + T::STG_BYTES + T::bias_bytes(N) + T::ATT_BYTES;  // WS: resident [K/64][BN x 128 B]; else ring
  uint8_t* sA = sB + T::b_res_bytes(K, WS);             // [stages] x 16 KB
  uint8_t* sBs = sA + stages * A_STAGE_BYTES;           // streaming B ring [stages] x B_STAGE_BYTES

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_kb = K / BK;
  const Sched<WS, PAIR> sc(M, N / BN, att);
  const bool leader = sc.rank == 0;              // PAIR: the CTA that issues the MMAs

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], WS ? 1 : 1 + T::N_LOADS);   // one arrive (+tx) per box (leader's boxes in PAIR)
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], (PAIR ? 2 : 1) * T::EPI_WARPS);
    }
    mbar_init(bfull, 1);
    mbar_init(att_gate, (PAIR ? 2 : 1) * T::EPI_WARPS);
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) {
      tmem_alloc_pair(tmem_slot, T::TMEM_COLS);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(tmem_slot, T::TMEM_COLS);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();            // peer barriers initialised before any remote use
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 || warp == 2 || warp == 3) {
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producers
      // Three producer threads (warps 0, 2, 3) share the ring: box b of k-block counter c is issued
      // by producer (c * NBOX + b) % 3.  One thread sustains only ~one TMA box per ~500 cycles
      // (measured: scripts/microbench/tma_bw2.cu), so a single producer would cap A+B ingest far
      // below what the tensor core consumes.
      constexpr int NPROD = 3;
      constexpr int NBOX = WS ? 1 : 1 + T::N_LOADS;
      const int p = warp == 0 ? 0 : warp - 1;
      const uint64_t pol_w = l2_policy_evict_last();   // weights: re-read by every M tile
      if constexpr (WS) {
        if (p == 0 && sc.t0 < sc.tend) {
          const int n0 = sc.slice * BN;
          if constexpr (PAIR) {                   // each CTA loads its half; bytes land on the leader
            if (leader) mbar_arrive_expect_tx(bfull, uint32_t(BN) * K * 2);
            const uint32_t bar = mapa_shared(smem_u32(bfull), 0);
            for (int kb = 0; kb < num_kb; ++kb)
#pragma unroll
              for (int j = 0; j < T::N_LOADS; ++j)
                tma_load_2d_pair(sB + kb * T::B_STAGE_BYTES + j * T::B_BOX * 128, &tmB, bar, kb * BK,
                                 n0 + j * T::MMA_N + sc.rank * T::B_BOX, pol_w);
          } else {
            mbar_arrive_expect_tx(bfull, uint32_t(BN) * K * 2);
            for (int kb = 0; kb < num_kb; ++kb)
#pragma unroll
              for (int j = 0; j < T::N_LOADS; ++j)
                tma_load_2d_hint(sB + kb * T::B_STAGE_BYTES + j * T::B_BOX * 128, &tmB, bfull, kb * BK,
                                 n0 + j * T::B_BOX, pol_w);
          }
        }
      }
      griddep_wait();                         // A / residual come from the previous kernel
      uint32_t c = 0;
      for (int t = sc.t0; t < sc.tend; t += sc.dt) {
        const int m0 = sc.m0(t), n0 = sc.n0(t) * BN;
        for (int kb = 0; kb < num_kb; ++kb, ++c) {
          const int s = int(c % uint32_t(stages));
          const uint32_t ph = (c / uint32_t(stages)) & 1;
#pragma unroll
          for (int b = 0; b < NBOX; ++b) {
            if (int((c * NBOX + b) % NPROD) != p) continue;
            mbar_wait(&empty[s], ph ^ 1);
            if (b == 0) {
              if constexpr (EPI == EPI_BIAS_LN) {
                // warm L2 with this tile's residual rows (read by the LN epilogue)
                if (kb < N / 64) tma_prefetch_2d(&tmR, kb * 64, m0);
              }
              if constexpr (PAIR) {               // both halves complete on the leader's barrier
                if (leader) mbar_arrive_expect_tx(&full[s], 2 * A_STAGE_BYTES);
                tma_load_2d_pair(sA + s * A_STAGE_BYTES, &tmA, mapa_shared(smem_u32(&full[s]), 0), kb * BK, m0,
                                 l2_policy_evict_first());
              } else {
                mbar_arrive_expect_tx(&full[s], A_STAGE_BYTES);
                tma_load_2d(sA + s * A_STAGE_BYTES, &tmA, &full[s], kb * BK, m0);
              }
            } else {
              const int j = b - 1;
              if constexpr (PAIR) {               // rows [j MMA_N + r MMA_N/2, +MMA_N/2) of MMA j's B
                if (leader) mbar_arrive_expect_tx(&full[s], 2 * T::B_BOX * 128);
                tma_load_2d_pair(sBs + s * T::B_STAGE_BYTES + j * T::B_BOX * 128, &tmB,
                                 mapa_shared(smem_u32(&full[s]), 0), kb * BK,
                                 n0 + j * T::MMA_N + sc.rank * T::B_BOX, pol_w);
              } else {
                mbar_arrive_expect_tx(&full[s], T::B_BOX * 128);
                tma_load_2d_hint(sBs + s * T::B_STAGE_BYTES + j * T::B_BOX * 128, &tmB, &full[s], kb * BK,
                                 n0 + j * T::B_BOX, pol_w);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    griddep_launch_dependents();
    // -------------------------------------------------------------------- MMA issuer
    // The whole warp walks the loop (warp-uniform control flow and operands, so descriptors live
    // in uniform registers); one elected lane issues the tcgen05.mma / commit instructions.
    // Shared-memory descriptors are built once and advanced by adding (byte offset >> 4) to their
    // start-address field.
    constexpr uint32_t idesc = umma_idesc_bf16(T::UMMA_M, T::MMA_N);
    const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA));
    const uint64_t b_desc0 = umma_desc_sw128(smem_u32(WS ? sB : sBs));
    if constexpr (WS) mma_wait(bfull, 0);
    int s = 0;
    uint32_t ph = 0;
    int it = 0;
#ifdef ATT_TRACE
    long long mt_acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const long long mt_start = clock64();
#endif
    for (int t = sc.t0; t < sc.tend; t += sc.dt, ++it) {
      const int acc = it % ACC;
      const uint32_t aph = (it / ACC) & 1;
#ifdef ATT_TRACE
      long long _e0 = clock64();
      mma_wait(&tempty[acc], aph ^ 1);
      mt_acc[8] += clock64() - _e0;
#else
      mma_wait(&tempty[acc], aph ^ 1);       // epilogue drained this accumulator buffer
#endif
#ifndef ATT_GATE
#define ATT_GATE 2
#endif
      if constexpr (T::ATT) {
        // legacy mma.sync (the attention) is starved while tcgen05 MMAs run on the SM
        // (scripts/microbench/umma_hmma.cu: ~0.01 vs 0.46 HMMA/clk): the next tile's MMAs wait until
        // the previous tile's attention phase is over, instead of stretching it
        // schedule per SM: MMA(t+1) | epilogue: store(t-1), stage(t)  ->  attention(t) alone on the pipe
        // -> MMA(t+2) | ... : MMA(t) waits for attention(t-2); attention(t) waits for MMA(t+1) to retire.
#ifdef ATT_TRACE
        long long _g0 = clock64();
#endif
        if (ATT_GATE == 1 && it >= 1) mma_wait(att_gate, (it - 1) & 1);
        if (ATT_GATE == 2 && it >= 2) mma_wait(att_gate, (it - 2) & 1);
#ifdef ATT_TRACE
        mt_acc[0] += clock64() - _g0;
#endif
      }
      tc_fence_after();
      const uint32_t d0 = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
#ifdef ATT_TRACE
        long long _f0 = clock64();
        mma_wait(&full[s], ph);
        if (kb < 7) mt_acc[1 + kb] += clock64() - _f0;
#else
        mma_wait(&full[s], ph);
#endif
        tc_fence_after();
        if (elect_one()) {
          const uint64_t a_desc = a_desc0 + uint64_t((s * A_STAGE_BYTES) >> 4);
          const uint64_t b_desc = b_desc0 + uint64_t(((WS ? kb : s) * T::B_STAGE_BYTES) >> 4);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
#pragma unroll
            for (int j = 0; j < T::N_MMA; ++j) {
              const uint64_t bd = b_desc + uint64_t((j * T::B_BOX * 128 + k * 32) >> 4);
              if constexpr (PAIR) tc_mma_bf16_pair(d0 + j * T::MMA_N, a_desc + uint64_t(k * 2), bd, idesc, (kb | k) != 0);
              else tc_mma_bf16(d0 + j * T::MMA_N, a_desc + uint64_t(k * 2), bd, idesc, (kb | k) != 0);
            }
          }
          if constexpr (PAIR) tc_commit_pair_mc(&empty[s], 0x3);   // frees the stage in both CTAs
          else tc_commit(&empty[s]);          // frees this smem stage when the MMAs retire
        }
        __syncwarp();
        if (++s == stages) { s = 0; ph ^= 1; }
      }
      if (elect_one()) {                      // accumulator complete (both CTAs' halves in PAIR)
        if constexpr (PAIR) tc_commit_pair_mc(&tfull[acc], 0x3);
        else tc_commit(&tfull[acc]);
      }
      __syncwarp();
    }
#ifdef ATT_TRACE
    if constexpr (T::ATT) {
      const long long n = it > 0 ? it : 1;
      if (lane == 0 && blockIdx.x < 8)
        printf("MMA_TRACE cta %d tiles %d total %lld | gate %lld tempty %lld full kb0..5 %lld %lld %lld %lld %lld %lld (cycles/tile)\n",
               int(blockIdx.x), it, (clock64() - mt_start) / n, mt_acc[0] / n, mt_acc[8] / n, mt_acc[1] / n,
               mt_acc[2] / n, mt_acc[3] / n, mt_acc[4] / n, mt_acc[5] / n, mt_acc[6] / n);
    }
#endif
  } else if (warp >= 4) {
    griddep_wait();                           // records / residual rows / outputs of the previous kernel
    // ------------------------------------------------------------------ epilogue (warps 4..11)
    if constexpr (EPI == EPI_BIAS_LN) {       // LN tiles span all N columns: constants once
      for (int i = threadIdx.x - 128; i < BN; i += T::EPI_WARPS * 32) {
        s_bias[i] = bias[i];
        s_gamma[i] = gamma[i];
        s_beta[i] = beta[i];
      }
      named_bar_sync(5, T::EPI_WARPS * 32);
    }
    if constexpr (T::BIAS_SMEM) {
      for (int i = threadIdx.x - 128; i < N; i += T::EPI_WARPS * 32) s_bias_all[i] = bias[i];
      named_bar_sync(5, T::EPI_WARPS * 32);
    }
    if constexpr (T::ATT) {                   // zero rows [BM, BM + 16): read past the tile's last text
      for (int i = threadIdx.x - 128; i < 16 * T::ATT_LDS / 8; i += T::EPI_WARPS * 32)
        reinterpret_cast<uint4*>(sAtt + BM * T::ATT_LDS)[i] = make_uint4(0, 0, 0, 0);
      const int e = threadIdx.x - 128;          // first tile's record -> slot 0
      if (e < ATT_REC_INTS && sc.t0 < sc.tend) s_rec[e] = att.rec[size_t(sc.att_tile(sc.t0)) * ATT_REC_INTS + e];
      named_bar_sync(5, T::EPI_WARPS * 32);
    }
#ifdef ATT_TRACE
    long long tr_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tr_last = 0;
    int tr_tiles = 0;
#endif
    int stg = 0;                              // staged output boxes issued by this warp
    const int q = warp & 3;                   // TMEM lane quadrant this warp may access
    const int hh = (warp - 4) >> 2;           // column part (0 .. SPLIT-1)
    const int c_lo = hh * T::HALF;
    int it = 0;
    for (int t = sc.t0; t < sc.tend; t += sc.dt, ++it) {
      const int m0 = sc.m0(t), n0 = sc.n0(t) * BN;
      const int acc = it % ACC;
      const uint32_t aph = (it / ACC) & 1;
      const int row = m0 + q * 32 + lane;
      const bool ok = row < M;
      const uint32_t taddr = tmem_base + acc * BN + (uint32_t(q * 32) << 16);
      // Output: each warp stages its 32 rows x 32 columns (bf16) in a private, 64-byte-swizzled
      // smem buffer and one lane TMA-stores the box (coalesced; rows >= M clipped by TMA).
      auto stage_store = [&](const uint32_t (&p)[16], int col) {
        uint8_t* buf = sStg + ((warp - 4) * T::STG_BUFS + (stg % T::STG_BUFS)) * 2048;
        if (lane == 0 && stg >= T::STG_BUFS) bulk_wait_read<T::STG_BUFS - 1>();   // buffer drained
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<uint4*>(buf + lane * 64 + ((i ^ ((lane >> 1) & 3)) << 4)) =
              make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmC, buf, col, m0 + q * 32);
          bulk_commit();
        }
        ++stg;
      };
      constexpr int NSTEP = T::HALF / 32;     // 32-column steps per warp
      if constexpr (T::ATT) {
        // ---- QKV + attention (K4 + K5).  Slice columns: [Q | K | V] of HG heads, DH each.
        // phase 1: acc + bias -> bf16 (the values the separate path stores as QKV) -> sAtt, then the
        //          accumulator is released (the next tile's MMAs overlap phases 2-3);
        // phase 2: (text, head) units of the tile's texts over the epilogue warps, attn_query_tile
        //          (shared with attention_text_kernel: same arithmetic), O over the Q columns;
        // phase 3: O rows of the tile's texts -> global (16-byte stores, 128 B per row).
        constexpr int HG = BN / (3 * DH);
        constexpr int LDS = T::ATT_LDS;
        const int e = threadIdx.x - 128;
        const int slot = it & 1;
        // prefetch the next tile's record (registers; stored to the other slot after this tile)
        const bool has_next = t + sc.dt < sc.tend;
        int32_t nxt = 0;
        if (e < ATT_REC_INTS && has_next) nxt = att.rec[size_t(sc.att_tile(t + sc.dt)) * ATT_REC_INTS + e];
        // phase 1 in 16-column steps (HALF = 64 with 12 epilogue warps, 48 with 16)
        constexpr int NS16 = T::HALF / 16;
        const float4* bp = reinterpret_cast<const float4*>(bias + n0 + c_lo);
        float4 b4[2][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) b4[0][i] = __ldg(bp + i);
        uint32_t r[2][16];
        ATT_TR(0);
        mbar_wait(&tfull[acc], aph);
        ATT_TR(1);
        tc_fence_after();
        tmem_ld16(taddr + c_lo, r[0]);
        uint16_t* srow = sAtt + (q * 32 + lane) * LDS + c_lo;
#pragma unroll
        for (int k = 0; k < NS16; ++k) {
          const int cur = k & 1;
          tmem_ld_wait_regs16(r[cur]);
          const uint32_t (&rc)[16] = r[cur];
          if (k + 1 < NS16) {
            tmem_ld16(taddr + c_lo + 16 * (k + 1), r[cur ^ 1]);
#pragma unroll
            for (int i = 0; i < 4; ++i) b4[cur ^ 1][i] = __ldg(bp + 4 * (k + 1) + i);
          }
          uint32_t p[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 bb = b4[cur][i];
            const f32x2 v01 = fadd2(f2(__uint_as_float(rc[4 * i]), __uint_as_float(rc[4 * i + 1])), f2(bb.x, bb.y));
            const f32x2 v23 = fadd2(f2(__uint_as_float(rc[4 * i + 2]), __uint_as_float(rc[4 * i + 3])), f2(bb.z, bb.w));
            p[2 * i] = pack_bf16x2(f2lo(v01), f2hi(v01));
            p[2 * i + 1] = pack_bf16x2(f2lo(v23), f2hi(v23));
          }
#pragma unroll
          for (int i = 0; i < 2; ++i)
            *reinterpret_cast<uint4*>(srow + 16 * k + 8 * i) = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
          else mbar_arrive(&tempty[acc]);
        }
        ATT_TR(2);
        named_bar_sync(1, T::EPI_WARPS * 32);   // the tile's Q | K | V staged (and its record visible)
        if (ATT_GATE == 2 && has_next) {          // the next tile's MMAs retire before the attention starts
          mbar_wait(&tfull[acc ^ (ACC > 1 ? 1 : 0)], ((it + 1) / ACC) & 1);
          tc_fence_after();
        }
        ATT_TR(3);
        const int32_t* R = s_rec + slot * ATT_REC_INTS;
        const int row0 = R[0], nrows = R[1], ntexts = R[2], nunits = R[3];
        const uint8_t* tstart = reinterpret_cast<const uint8_t*>(R + 4);
        const uint16_t* units = reinterpret_cast<const uint16_t*>(R + 36);
#ifndef ATT_NHU32
#define ATT_NHU32 1
#endif
        constexpr int NHU = DH == 16 ? 2 : DH == 32 ? ATT_NHU32 : 1;   // heads per unit (internal.h att_unit_heads)
        constexpr int W = T::EPI_WARPS;
        const int w = warp - 4;
#pragma unroll 1
        for (int k = 0;; ++k) {                 // snake order over the cost-sorted units
#ifdef ATT_SKIP_P2
          break;                                // timing experiment only (wrong results)
#endif
          const int u = k * W + ((k & 1) ? W - 1 - w : w);
          if (u >= nunits) break;
          const int un = units[u];
          const int j = un & 0xff, qt = (un >> 8) & 7, h0 = (un >> 11) * NHU;
          const int ta = tstart[j];
          const int len = (j + 1 < ntexts ? int(tstart[j + 1]) : nrows) - ta;
          const int nt = (len + 15) >> 4;
          uint16_t* sQt = sAtt + (ta + 16 * qt) * LDS + h0 * DH;
          float o[NHU][DH / 8][4];
          float ia[NHU], ib[NHU];
          attn_query_tile<DH, LDS, NHU>(sQt, sAtt + ta * LDS + (HG + h0) * DH, sAtt + ta * LDS + (2 * HG + h0) * DH,
                                        len, nt, att.qscale, lane, o, ia, ib, len - 16 * qt, sAtt + BM * LDS + h0 * DH);
          __syncwarp();   // every lane has read its Q fragments before O overwrites the tile
          attn_store_tile<DH, NHU>(sQt, LDS, qt, len, lane, o, ia, ib);
        }
        ATT_TR(4);
        __syncwarp();
        if (lane == 0) {                          // attention of this tile done (its HMMAs retired)
          if constexpr (PAIR) mbar_arrive_cluster(mapa_shared(smem_u32(att_gate), 0));
          else mbar_arrive(att_gate);
        }
        named_bar_sync(1, T::EPI_WARPS * 32);   // O complete
        ATT_TR(5);
        {
          constexpr int CH = HG * DH / 8;         // 16-byte chunks of one O row
          const int dout = N / 3;
          uint16_t* orow0 = C + size_t(row0) * dout + n0 / 3;
          for (int i = e; i < nrows * CH; i += T::EPI_WARPS * 32) {
            const int rr = i / CH, cc = i - rr * CH;
            *reinterpret_cast<uint4*>(orow0 + size_t(rr) * dout + cc * 8) =
                *reinterpret_cast<const uint4*>(sAtt + rr * LDS + cc * 8);
          }
        }
        if (e < ATT_REC_INTS && has_next) s_rec[(slot ^ 1) * ATT_REC_INTS + e] = nxt;
        ATT_TR(6);
        named_bar_sync(1, T::EPI_WARPS * 32);   // sAtt free for the next tile
        ATT_TR(7);
      } else if constexpr (EPI == EPI_BIAS || EPI == EPI_BIAS_GELU) {
        // Software-pipelined over 32-column steps: the TMEM load and bias slice of step k+1 are in
        // flight while step k is computed and stored (tcgen05.wait::ld then covers only step k+1).
        const float4* bp = reinterpret_cast<const float4*>(bias + n0 + c_lo);
        const float4* sbp = reinterpret_cast<const float4*>(s_bias_all + n0 + c_lo);
        uint32_t r[2][32];
        float4 b4[T::BIAS_SMEM ? 1 : 2][8];
        if constexpr (!T::BIAS_SMEM) {
#pragma unroll
          for (int i = 0; i < 8; ++i) b4[0][i] = __ldg(bp + i);
        }
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        tmem_ld32(taddr + c_lo, r[0]);
#pragma unroll
        for (int k = 0; k < NSTEP; ++k) {
          const int cur = k & 1;
          tmem_ld_wait_regs(r[cur]);
          if (k + 1 < NSTEP) {
            tmem_ld32(taddr + c_lo + 32 * (k + 1), r[cur ^ 1]);
            if constexpr (!T::BIAS_SMEM) {
#pragma unroll
              for (int i = 0; i < 8; ++i) b4[cur ^ 1][i] = __ldg(bp + 8 * (k + 1) + i);
            }
          }
          uint32_t p[16];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 bb = T::BIAS_SMEM ? sbp[8 * k + i] : b4[T::BIAS_SMEM ? 0 : cur][i];
            const f32x2 v01 = fadd2(f2(__uint_as_float(r[cur][4 * i]), __uint_as_float(r[cur][4 * i + 1])), f2(bb.x, bb.y));
            const f32x2 v23 = fadd2(f2(__uint_as_float(r[cur][4 * i + 2]), __uint_as_float(r[cur][4 * i + 3])), f2(bb.z, bb.w));
            float v0 = f2lo(v01), v1 = f2hi(v01), v2 = f2lo(v23), v3 = f2hi(v23);
            if constexpr (EPI == EPI_BIAS_GELU) {
              gelu2(v0, v1);
              gelu2(v2, v3);
            }
            p[2 * i] = pack_bf16x2(v0, v1);
            p[2 * i + 1] = pack_bf16x2(v2, v3);
          }
          stage_store(p, n0 + c_lo + 32 * k);
        }
      } else if constexpr (EPI == EPI_BIAS_RES) {
        // fp32 v = acc + bias + residual, stored directly (each thread: its row, 32 columns / step)
        const uint16_t* rrow = res + size_t(ok ? row : 0) * N + n0 + c_lo;
        float* frow = reinterpret_cast<float*>(C) + size_t(row) * N + n0 + c_lo;
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
#pragma unroll 1
        for (int k = 0; k < NSTEP; ++k) {
          uint32_t r[32];
          tmem_ld32(taddr + c_lo + 32 * k, r);
          uint4 rs[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) rs[i] = reinterpret_cast<const uint4*>(rrow + 32 * k)[i];
          tmem_ld_wait_regs(r);
          const float4* bp = reinterpret_cast<const float4*>(bias + n0 + c_lo + 32 * k);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 b4 = __ldg(bp + i);
            const uint32_t u0 = (&rs[i >> 1].x)[(i & 1) * 2], u1 = (&rs[i >> 1].x)[(i & 1) * 2 + 1];
            const float4 o = make_float4(__uint_as_float(r[4 * i]) + b4.x + bf16lo(u0),
                                         __uint_as_float(r[4 * i + 1]) + b4.y + bf16hi(u0),
                                         __uint_as_float(r[4 * i + 2]) + b4.z + bf16lo(u1),
                                         __uint_as_float(r[4 * i + 3]) + b4.w + bf16hi(u1));
            if (ok) reinterpret_cast<float4*>(frow + 32 * k)[i] = o;
          }
        }
      } else {
        // LayerNorm over the full row (BN == N), two warps per row (column halves): epi_ln.cuh
        const ResidualGlobal rg{res + size_t(ok ? row : 0) * N};
        uint8_t* stg = sStg + (warp - 4) * T::STG_BUFS * 2048;
        ln_epilogue<BN, T::HALF>(taddr, c_lo, rg, s_bias, s_gamma, s_beta, stats + (it & 1) * 2 * BM, q, hh, lane,
                                 eps, [&] {
                                   mbar_wait(&tfull[acc], aph);
                                   tc_fence_after();
                                 },
                                 [&](const uint32_t (&p)[16], int col) {
                                   store_rows_32x32(stg, p, lane, C, m0 + q * 32, M, N, col);
                                 });
      }
      if constexpr (!T::ATT) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));   // leader's barrier
          else mbar_arrive(&tempty[acc]);
        }
      }
    }
    if (lane == 0) bulk_wait_all();           // output stores complete before the CTA retires
#ifdef ATT_TRACE
    if constexpr (T::ATT) {
      tr_tiles = it;
      if (lane == 0 && blockIdx.x < 1)
        printf("ATT_TRACE cta %d warp %d tiles %d | wait %lld p1 %lld bar1 %lld p2 %lld bar2 %lld p3 %lld bar3 %lld (cycles/tile)\n",
               int(blockIdx.x), warp, tr_tiles, tr_acc[0] / max(tr_tiles, 1), tr_acc[1] / max(tr_tiles, 1),
               tr_acc[2] / max(tr_tiles, 1), tr_acc[3] / max(tr_tiles, 1), tr_acc[4] / max(tr_tiles, 1),
               tr_acc[5] / max(tr_tiles, 1), tr_acc[6] / max(tr_tiles, 1));
    }
#endif
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();            // the peer may still read our smem / signal us
  else __syncthreads();
  if (warp == 2) {
    __syncwarp();
    if constexpr (PAIR) tmem_dealloc_pair(tmem_base, T::TMEM_COLS);
    else tmem_dealloc(tmem_base, T::TMEM_COLS);
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;

template <int BN, int EPI, bool WS, bool PAIR = false, int DH = 0>
cudaError_t launch_gemm_t(const GemmArgs& g, cudaStream_t st) {
  using T = TileCfg<BN, EPI, PAIR, DH>;
  auto kern = gemm_tc_kernel<BN, EPI, WS, PAIR, DH>;
  const int smem = T::smem_bytes(g.K, WS, g.N);
  const int stages = T::stages(g.K, WS, g.N);
  if (stages < 2 || smem > T::MAX_SMEM) return cudaErrorInvalidValue;
  static int smem_attr = 0;
  if (smem_attr < smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::MAX_SMEM);
    if (e != cudaSuccess) return e;
    smem_attr = T::MAX_SMEM;
  }
  const bool att = EPI == EPI_QKV_ATTN;
  const int64_t m_tiles = att ? g.n_att_tiles : (g.M + BM - 1) / BM, n_tiles = g.N / BN;
  const AttTiles at{att ? g.att_rec : nullptr, g.n_att_tiles, g.qscale};
  int grid;
  if (WS && PAIR) {
    const int64_t m2 = att ? g.n_att_tiles / 2 : (g.M + 2 * BM - 1) / (2 * BM);
    const int64_t per = std::min<int64_t>(std::max<int64_t>(num_sms() / 2 / n_tiles, 1), m2);
    grid = int(2 * per * n_tiles);
  } else if (WS) {
    const int64_t per = std::min<int64_t>(std::max<int64_t>(num_sms() / n_tiles, 1), m_tiles);
    grid = int(per * n_tiles);
  } else if (PAIR) {
    const int64_t m2 = att ? g.n_att_tiles / 2 : (g.M + 2 * BM - 1) / (2 * BM);
    grid = 2 * int(std::min<int64_t>(m2 * n_tiles, num_sms() / 2));
  } else {
    grid = int(std::min<int64_t>(m_tiles * n_tiles, num_sms()));
  }
  const CUtensorMap tmR = g.tmR ? *g.tmR : *g.tmC;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(T::THREADS);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (PAIR) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, *g.tmA, *g.tmB, *g.tmC, tmR, int(g.M), g.N, g.K, g.bias, g.res, g.gamma,
                            g.beta, g.C, g.eps, stages, at);
}

// Weight-stationary when the B slice fits next to >= 4 A stages and there are enough M tiles to
// give every slice's CTAs work.
template <int BN, int EPI, bool PAIR = false, int DH = 0>
bool use_ws(const GemmArgs& g) {
  using T = TileCfg<BN, EPI, PAIR, DH>;
  const int64_t m_units = g.epi == EPI_QKV_ATTN ? (PAIR ? g.n_att_tiles / 2 : g.n_att_tiles)
                         : PAIR ? (g.M + 2 * BM - 1) / (2 * BM) : (g.M + BM - 1) / BM;
  const int units = PAIR ? num_sms() / 2 : num_sms();
  return g.epi != EPI_BIAS_LN && g.epi != EPI_BIAS_RES && T::stages(g.K, true, g.N) >= 3 &&
         m_units >= units / (g.N / BN);
}

template <int BN, int EPI>
cudaError_t launch_gemm_bn(const GemmArgs& g, cudaStream_t st) {
  if (gemm_use_pair(g.N, g.K, g.epi)) {
    if constexpr (EPI != EPI_BIAS_LN && BN == 384) {
      if (use_ws<BN, EPI, true>(g)) return launch_gemm_t<BN, EPI, true, true>(g, st);
    }
    return launch_gemm_t<BN, EPI, false, true>(g, st);
  }
  if constexpr (EPI != EPI_BIAS_LN) {
    if (use_ws<BN, EPI>(g)) return launch_gemm_t<BN, EPI, true>(g, st);
  }
  return launch_gemm_t<BN, EPI, false>(g, st);
}

}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SURGE_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t init_tma_encoder() {
  if (g_encode_tiled) return cudaSuccess;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess) return e;
  if (q != cudaDriverEntryPointSuccess || !fn) return cudaErrorSymbolNotFound;
  g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return cudaSuccess;
}

// Row-major bf16 matrix [rows x cols] (cols contiguous), box = 64 cols x box_rows, 128 B swizzle.
cudaError_t make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  if (!g_encode_tiled) {
    cudaError_t e = init_tma_encoder();
    if (e != cudaSuccess) return e;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode_tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Row-major bf16 matrix, box = 32 cols (64 B) x box_rows, 64 B swizzle (ln_pair.cu's 32-wide k-blocks).
cudaError_t make_tmap_bf16_k32(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  if (!g_encode_tiled) {
    cudaError_t e = init_tma_encoder();
    if (e != cudaSuccess) return e;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode_tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_tmap_store_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols) {
  if (!g_encode_tiled) {
    cudaError_t e = init_tma_encoder();
    if (e != cudaSuccess) return e;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode_tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// LN GEMMs (full-row tiles, single TMEM accumulator) run as CTA pairs: half the B bytes per CTA.
// Weight-stationary pairs for bias-only GEMMs (each CTA keeps half of a [384 x K] slice resident,
// twice the MMA work per A byte of a 192-column slice) are implemented (WS && PAIR) but not
// selected: with a single 384-column TMEM accumulator the epilogue serialises with the mainloop
// and measured slower than 192-column single-CTA slices (QKV 109 vs 84 ms per 1M texts).
// Streaming (non-weight-stationary, BN = 256) GEMMs of the bge classes as CTA pairs too: M = 256 per
// cta_group::2 MMA, each CTA loading half of the 256 weight rows per k-block, so the weight bytes per output
// row halve.  GELU GEMM (FFN1, GEMM_GELU_PAIR): bge-base 409 -> 369 ms per 500K texts, bge-large 531 -> 476 ms
// per 200K (+2.9% / +3.1% texts/s).  Bias GEMM (the QKV projection of chunks with texts > 128 tokens,
// GEMM_BIAS_PAIR): C4 bge-large 890 -> 775 ms per 50K long texts (+1.9% texts/s).
#ifndef GEMM_GELU_PAIR
#define GEMM_GELU_PAIR 1
#endif
#ifndef GEMM_BIAS_PAIR
#define GEMM_BIAS_PAIR 1
#endif
bool gemm_use_pair(int N, int K, int epi) {
  if (K % 64 != 0) return false;
  if (((GEMM_GELU_PAIR && epi == EPI_BIAS_GELU) || (GEMM_BIAS_PAIR && epi == EPI_BIAS)) &&
      gemm_bn_for(N, K, epi) == 256 && !(TileCfg<256, EPI_BIAS>::stages(K, true) >= 3))
    return true;
  return epi == EPI_BIAS_LN && N == 384;
}

int gemm_bn_for(int N, int K, int epi) {
  if (epi == EPI_BIAS_LN) return (N == 64 || N == 384) ? N : 0;
  if (epi == EPI_BIAS_RES) return N % 256 == 0 ? 256 : N % 128 == 0 ? 128 : 0;
#ifdef GEMM_FORCE_BN
  if (N % GEMM_FORCE_BN == 0) return GEMM_FORCE_BN;   // tuning experiments only
#endif
  // Weight-stationary slices (the [BN x K] weight block stays resident, A streams; A is re-read
  // N/BN times from L2, B once per CTA).  128-column slices leave room for 7 A stages and measured
  // fastest in isolation (scripts/gemm_bench.py, M = 262144, K = 384: BN 64/128/192 ->
  // QKV 691/1078/1007, FFN1(bias) 701/1102/1020 TFLOP/s): these GEMMs are bound by A-tile latency.
  // (the GELU GEMM keeps 192-column slices: its 12-warp epilogue measured ~5% faster in the step)
  if (epi != EPI_BIAS_GELU && N % 128 == 0 && TileCfg<128, EPI_BIAS>::stages(K, true) >= 6) return 128;
  if (N % 192 == 0 && TileCfg<192, EPI_BIAS>::stages(K, true) >= 3) return 192;
  if (N % 256 == 0) return 256;
  if (N % 192 == 0) return 192;
  if (N % 128 == 0) return 128;
  if (N % 64 == 0) return 64;
  return 0;
}

uint32_t gemm_b_box_rows(int N, int K, int epi) {
  if (epi == EPI_QKV_ATTN) return ATT_SLICE / 2;   // CTA pairs: half of each 192-row slice
  const int BN = gemm_bn_for(N, K, epi);
  const int mma_n = BN <= 256 ? BN : BN / 2;
  return uint32_t(gemm_use_pair(N, K, epi) ? mma_n / 2 : mma_n);
}

template <int DH>
cudaError_t launch_qkv_att(const GemmArgs& g, cudaStream_t st) {
  if (use_ws<ATT_SLICE, EPI_QKV_ATTN, true, DH>(g)) return launch_gemm_t<ATT_SLICE, EPI_QKV_ATTN, true, true, DH>(g, st);
  return launch_gemm_t<ATT_SLICE, EPI_QKV_ATTN, false, true, DH>(g, st);
}

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t st) {
  if (g.epi == EPI_QKV_ATTN) {
    if (g.N % ATT_SLICE != 0 || g.K % BK != 0 || g.K <= 0 || g.M <= 0 || !g.att_rec || g.n_att_tiles <= 0 ||
        (g.n_att_tiles & 1))
      return cudaErrorInvalidValue;
    switch (g.head_dim) {
      case 16: return launch_qkv_att<16>(g, st);
      case 32: return launch_qkv_att<32>(g, st);
      case 64: return launch_qkv_att<64>(g, st);
    }
    return cudaErrorInvalidValue;
  }
  const int BN = gemm_bn_for(g.N, g.K, g.epi);
  if (BN == 0 || g.K % BK != 0 || g.K <= 0 || g.M <= 0) return cudaErrorInvalidValue;
  switch (g.epi) {
    case EPI_BIAS:
      switch (BN) {
        case 64: return launch_gemm_bn<64, EPI_BIAS>(g, st);
        case 128: return launch_gemm_bn<128, EPI_BIAS>(g, st);
        case 192: return launch_gemm_bn<192, EPI_BIAS>(g, st);
        case 256: return launch_gemm_bn<256, EPI_BIAS>(g, st);
        case 384: return launch_gemm_bn<384, EPI_BIAS>(g, st);
      }
      break;
    case EPI_BIAS_GELU:
      switch (BN) {
        case 64: return launch_gemm_bn<64, EPI_BIAS_GELU>(g, st);
        case 128: return launch_gemm_bn<128, EPI_BIAS_GELU>(g, st);
        case 192: return launch_gemm_bn<192, EPI_BIAS_GELU>(g, st);
        case 256: return launch_gemm_bn<256, EPI_BIAS_GELU>(g, st);
        case 384: return launch_gemm_bn<384, EPI_BIAS_GELU>(g, st);
      }
      break;
    case EPI_BIAS_LN:
      switch (BN) {
        case 64: return launch_gemm_bn<64, EPI_BIAS_LN>(g, st);
        case 384: return launch_gemm_bn<384, EPI_BIAS_LN>(g, st);
      }
      break;
    case EPI_BIAS_RES:
      switch (BN) {
        case 128: return launch_gemm_bn<128, EPI_BIAS_RES>(g, st);
        case 256: return launch_gemm_bn<256, EPI_BIAS_RES>(g, st);
      }
      break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace surge
