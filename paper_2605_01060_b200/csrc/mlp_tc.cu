// mlp_tc.cu -- K7 + K8 fused: the encoder's feed-forward block as one kernel:
//   X2 = LN_o( GELU_erf(X1 W1^T + b1) W2^T + b2 + X1 )
// H = GELU(X1 W1^T + b1) never leaves the SM: per 128-row tile it is produced in ff-chunks of 128
// columns in TMEM, turned into bf16 in shared memory by the epilogue warps, and consumed there as the
// A operand of the second GEMM, whose accumulator (d columns) stays in TMEM across all chunks.
//
// Design (DESIGN.md §6 "fused MLP"): CTA pairs (cta_group::2, M = 256 rows per pair, each CTA its 128
// rows and half of every MMA's B rows), persistent over 256-row units.
//   TMEM (512 columns): Y = [0, D) second-GEMM accumulator, H = [384, 512) first-GEMM chunk.
//   smem: A = the unit's X1 rows (D/64 k-blocks of 128 x 64 bf16, 128-byte swizzle, resident for
//         the unit), Hs = one H chunk (2 k-blocks, written by the epilogue in the same swizzled
//         K-major layout the TMA would produce; it doubles as the LN output staging), a 3-stage
//         weight ring (24 KB stages: 3 W1 k-blocks or 1 W2 k-block per stage).
//   warps 0, 2, 3: TMA producers (A once per unit, the W1 / W2 ring); warp 1: MMA issuer (leader
//   CTA); warp 2 also allocates TMEM; warps 4..11: epilogue (GELU of each chunk; LN at the end).
//   MMA issue order per unit: G1(0), G1(1), G2(0), G1(2), G2(1), ..., G1(n-1), G2(n-2), G2(n-1):
//   G2(c-1) runs on the tensor pipe while the epilogue turns H(c) into Hs.
// Numerics equal the separate K7 / K8 GEMMs: H is bias + gelu2 + bf16 as EPI_BIAS_GELU; Y sums the
// same k-blocks in the same order; the LN epilogue is epi_ln.cuh (shared).
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "epi_ln.cuh"
#include "internal.h"

namespace surge {

namespace {

constexpr int MBM = 128;            // rows per CTA
constexpr int FC = 128;             // ff columns per chunk (H accumulator columns)
#ifndef MLP_RING
#define MLP_RING 4
#endif
#ifndef MLP_STG
#define MLP_STG 1                   // LN output staging buffers per epilogue warp
#endif
#ifndef MLP_A_SPLIT
#define MLP_A_SPLIT 1               // A-tile boxes issued by all three producers (0: producer 0 alone)
#endif
#ifndef MLP_LN_PIPE
#define MLP_LN_PIPE 1               // NP = 3: LN TMEM loads one step ahead too
#endif
#ifndef MLP_G0SPLIT
// d = 384 with MLP_PINGPONG: the next unit's out-projection G0 starts under this unit's final LayerNorm:
// its first 128 output columns (N = 128 MMAs) go to the idle H-chunk TMEM columns as soon as the O tile
// and the first Wo stages are in; columns 128..383 (N = 256 MMAs) follow once the LN has drained Y.
#define MLP_G0SPLIT 1
#endif
#ifndef MLP_LN_CPARAM
// LayerNorm constants (bo, gamma_a, beta_a, b2, gamma_o, beta_o) as a __grid_constant__ kernel parameter:
// uniform constant-cache loads instead of shared-memory loads in the LN epilogues (the LNs are MIO-bound)
#define MLP_LN_CPARAM 0              // 1 measured slower (tail 392 -> 403 ms per 2M texts: LDC.64 per pair)
#endif
#ifndef MLP_X1_CHASE
// SPLIT: G1 of chunk 0 starts k-block by k-block as LN0's pass 2 (interleaved columns, epi_ln.cuh) completes
// each 64-column block of X1, instead of after the whole LN0 (k-blocks 0, 1 also wait until the H columns
// holding G0's first 128 output columns have been read)
#define MLP_X1_CHASE 1
#endif
#ifndef MLP_LN_BF16
// LayerNorm constants staged in shared memory as bf16 (the weight blob's precision: the same values), half
// the shared-memory loads of the MIO-bound LN passes
#define MLP_LN_BF16 0               // 1 measured slower (tail 390 -> 398 ms per 2M texts: the unpacking costs more issue slots than the halved loads save)
#endif
#ifndef MLP_STORE_DIRECT
#define MLP_STORE_DIRECT 0          // 1: final LN output as 32-byte stores from registers (measured equal)
#endif
#ifndef MLP_PINGPONG
#define MLP_PINGPONG 1              // A tile and weight ring swap shared-memory regions every unit
#endif
#ifndef MLP_PREFETCH
#define MLP_PREFETCH 0              // L2 prefetch of the next unit's A rows (measured: no effect)
#endif
constexpr int RING = MLP_RING;      // weight ring stages
constexpr int STAGE = 24 * 1024;    // 3 W1 k-blocks (64 rows x 128 B each) or 1 W2 k-block (2 x 96 rows)
#ifndef MLP_EPI_WARPS
#define MLP_EPI_WARPS 8   // d = 384: 8 or 12 (16 measured slower: tail 2148 -> 2344 ms/step, 96-register cap)
#endif
constexpr uint32_t H_COL = 384;     // TMEM column of the H chunk

template <int D>
struct MlpConsts {   // [bo | gamma_a | beta_a | b2 | gamma_o | beta_o], D floats each
  float v[6 * D];
};

template <int D>
struct MlpCfg {
  // epilogue warps: 4 lane quadrants x NP column parts (d = 64: 8)
  static constexpr int EPI_WARPS = D == 384 ? MLP_EPI_WARPS : 8;
  static constexpr int NP = EPI_WARPS / 4;
  static constexpr int HC = FC / NP;                 // H-chunk columns per epilogue warp (NP = 3: 48, 48, 32)
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int KB1 = D / 64;                 // k-blocks of the first GEMM
  static constexpr int A_BYTES = KB1 * MBM * 128;    // resident X1 rows
  static constexpr int HS_BYTES = 2 * MBM * 128;     // one H chunk, 2 k-blocks
  static constexpr int N2 = D <= 256 ? D : D / 2;    // second-GEMM MMA N (<= 256)
  static constexpr int N2_MMAS = D / N2;
  static constexpr int B2_BOX = N2 / 2;              // rows of W2 per CTA per MMA (pair)
  static constexpr int HEAD = 1024;                  // barriers + TMEM slot
  // The LN output staging (8 warps x 2 KB), LN stats ([2 halves][128] float4, 4 KB) and b2 / gamma /
  // beta (3 D floats, copied in per unit) live in Hs, which is idle while the LN epilogue runs.
  // LN scratch (aliases Hs, which is idle during the LN): output staging [8 warps][MLP_STG][2 KB],
  // stats [2 halves][128] float4, b2 / gamma / beta
  static constexpr int LN_STG = MLP_STORE_DIRECT ? 0 : EPI_WARPS * MLP_STG * 2048;
  static constexpr int LN_SCRATCH = ((LN_STG + NP * MBM * 16 + 3 * D * 4 + 1023) / 1024) * 1024;
  static constexpr int SCRATCH = LN_SCRATCH > HS_BYTES ? LN_SCRATCH : HS_BYTES;
  // MLP_PINGPONG: two equal regions that alternate between the A tile and the weight ring, unit by
  // unit, so the next unit's A tile loads into the drained ring region as soon as the last MMA of
  // the unit retires (instead of after the final LN has read its residual from the A tile)
  static constexpr int REGION = MLP_PINGPONG ? (A_BYTES > RING * STAGE ? A_BYTES : RING * STAGE) : 0;
  static constexpr int SMEM = MLP_PINGPONG ? 1024 + HEAD + 2 * REGION + SCRATCH
                                           : 1024 + HEAD + A_BYTES + SCRATCH + RING * STAGE;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(D % 64 == 0 && D <= 384, "Y must fit TMEM next to the H chunk");
  static_assert(KB1 % 3 == 0 || KB1 == 1, "W1 k-blocks pack 3 per stage");
  static_assert(B2_BOX * 128 * N2_MMAS <= STAGE, "W2 k-block fits a stage");
};

// MLP_TL: per-unit event timeline of CTA 0 (units 10..13 of the 4th launch), buffered in global memory and
// printed at the end of the kernel (timing experiments only)
#ifdef MLP_TL
__device__ long long g_mtl_t0;
__device__ int g_mtl_launch;
__device__ long long g_mtlbuf[4][16];
enum { M_AFULL, M_G0ISS, M_Y0, M_XRES, M_X1R, M_G1_0, M_YFULL, M_AFREE, M_YEMPTY, M_XLOAD, M_N };
__device__ const char* const g_mtl_names[M_N] = {"a_full(iss)", "g0_issued", "y0_full(epi)", "xres_full(epi)",
    "x1_ready(iss)", "g1c0_issued", "y_full(epi)", "a_free(epi)", "y_empty(epi)", "x_load(prod)"};
#define MTL(ev, j) do { if (blockIdx.x == 0 && g_mtl_launch == 3 && (j) >= 10 && (j) < 14 && (threadIdx.x & 31) == 0 && \
    (threadIdx.x < 128 || (threadIdx.x >> 5) == 4)) g_mtlbuf[(j) - 10][ev] = clock64() - g_mtl_t0; } while (0)
#else
#define MTL(ev, j) do {} while (0)
#endif
#ifdef MLP_TRACE
#define MW(bar, par, slot)                      \
  do {                                          \
    const long long _t0 = clock64();            \
    mbar_wait(bar, par);                        \
    tw[slot] += clock64() - _t0;                \
  } while (0)
#elif defined(MLP_MMA_SPIN) && defined(MBAR_SLEEP_ALL)
#define MW(bar, par, slot) mbar_wait_spin(bar, par)   // the MMA issuer polls (critical path), the rest sleep
#else
#define MW(bar, par, slot) mbar_wait(bar, par)
#endif

// LN residual from the resident A tile (128-byte-swizzled K-major: k-block c / 64, row r at r * 128 B,
// 16-byte chunk j at (j ^ (r & 7)) * 16).
struct ResidualSmemA {
  const uint8_t* sA;
  int row, c_lo;   // c_lo unused (the LN epilogue passes absolute columns)
  __device__ __forceinline__ void operator()(int c, uint32_t (&rr)[16]) const {
    const uint8_t* base = sA + (c >> 6) * (MBM * 128) + row * 128;
    const int j0 = (c & 63) >> 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 v = *reinterpret_cast<const uint4*>(base + (((j0 + i) ^ (row & 7)) << 4));
      rr[4 * i] = v.x; rr[4 * i + 1] = v.y; rr[4 * i + 2] = v.z; rr[4 * i + 3] = v.w;
    }
  }
};

// Remote arrive with the default semantics (.release at .cta scope): after fence.proxy.async this
// publishes the thread's generic-proxy shared-memory writes to the leader's MMA, as CUTLASS's 2-SM
// pipelines do; .release.cluster would add a MEMBAR.ALL.GPU (measured ~1.5K cycles per chunk).
__device__ __forceinline__ void mbar_arrive_cluster_release(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Persistent CTA-pair kernel; unit u = rows [256 u, 256 u + 256), CTA rank r owns [256 u + 128 r, +128).
// OP (out-projection prologue, K6 fused too): A = O, and per unit first Y = O Wo^T (G0), then the
// LN0 epilogue writes X1 = LN_a(Y + bo + X) as bf16 into the A tile (O is dead by then), and the
// FFN runs on that X1; X1 never reaches HBM.  The final output overwrites X in place (each CTA reads
// its LN0 residual rows of X before it writes them).
template <int D, bool OP>
__global__ void __launch_bounds__(MlpCfg<D>::THREADS, 1)
    mlp_tc_kernel(const __grid_constant__ CUtensorMap tmX1, const __grid_constant__ CUtensorMap tmW1,
                  const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmWo,
                  const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmWo64,
                  const __grid_constant__ MlpConsts<D> lc, int M, int F, const float* __restrict__ b1,
                  const float* __restrict__ b2, const float* __restrict__ gamma, const float* __restrict__ beta,
                  const float* __restrict__ bo, const float* __restrict__ gamma1, const float* __restrict__ beta1,
                  const uint16_t* __restrict__ xres, uint16_t* __restrict__ out, float eps) {
  using T = MlpCfg<D>;
  constexpr int EPI_WARPS = T::EPI_WARPS, NP = T::NP, HC = T::HC;
  constexpr bool SPLIT = OP && MLP_PINGPONG && MLP_G0SPLIT && D == 384;   // G0 in column blocks 128 + 256
  constexpr bool CHASE = SPLIT && MLP_X1_CHASE && NP == 2;
  constexpr int KB1 = T::KB1;
  constexpr int S1 = KB1 == 1 ? 1 : KB1 / 3;         // ring stages per W1 chunk
  constexpr int KPS = KB1 == 1 ? 1 : 3;              // W1 k-blocks per stage
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);        // [RING]   leader: both CTAs' bytes
  uint64_t* empty = full + RING;                             // [RING]   both (multicast commit)
  uint64_t* a_full = empty + RING;                           // leader
  uint64_t* a_empty = a_full + 1;                            // both
  uint64_t* h_full = a_empty + 1;                            // both
  uint64_t* h_empty = h_full + 1;                            // leader, 2 x EPI_WARPS arrivals
  uint64_t* hs_full = h_empty + 1;                           // leader, 2 x EPI_WARPS arrivals
  uint64_t* hs_empty = hs_full + 1;                          // both
  uint64_t* y_full = hs_empty + 1;                           // both
  uint64_t* y_empty = y_full + 1;                            // leader, 2 x EPI_WARPS arrivals
  uint64_t* a_free = y_empty + 1;                            // local: LN read its residual from A
  uint64_t* y0_full = a_free + 1;                            // both (OP): G0 retired
  uint64_t* x1_ready = y0_full + 1;                          // leader (OP), 2 x EPI_WARPS: X1 in A
  uint64_t* xres_full = x1_ready + 1;                         // local (OP): X residual rows landed in A
  uint64_t* okb_free = xres_full + 1;                         // [KB1] both (OP): G0 done with O k-block kb
  uint64_t* x1kb = okb_free + KB1;                            // [KB1] leader (OP), 2 x EPI_WARPS: X1 k-block kb in A
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x1kb + KB1);
  uint8_t* const sR0 = smem + T::HEAD;                       // [KB1][128 x 128 B] (PINGPONG: region 0)
  uint8_t* sHs = sR0 + (MLP_PINGPONG ? T::REGION : T::A_BYTES);   // [2][128 x 128 B]
  float4* stats = reinterpret_cast<float4*>(sHs + T::LN_STG); // LN only
  using CT = std::conditional_t<MLP_LN_BF16 != 0, uint16_t, float>;   // LN constants in smem
  static_assert(!(MLP_LN_BF16 && MLP_LN_CPARAM), "one LN-constant path");
  CT* s_b2 = reinterpret_cast<CT*>(stats + NP * MBM);        // LN only
  CT* s_gamma = s_b2 + D;
  CT* s_beta = s_gamma + D;
  auto to_ct = [](float v) -> CT {
    if constexpr (sizeof(CT) == 2) return CT(pack_bf16x2(v, 0.f) & 0xffffu);
    else return v;
  };
  uint8_t* const sR1 = sHs + T::SCRATCH;                     // [RING][STAGE] (PINGPONG: region 1)
  // unit ui: A tile in region ui % 2, weight ring in the other (fixed roles without PINGPONG)
  auto region_a = [&](int ui) { return (MLP_PINGPONG && (ui & 1)) ? sR1 : sR0; };
  auto region_w = [&](int ui) { return (MLP_PINGPONG && (ui & 1)) ? sR0 : sR1; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = int(blockIdx.x & 1);
  const bool leader = rank == 0;
  const int unit0 = int(blockIdx.x >> 1), units = int(gridDim.x >> 1);
  const int n_units = (M + 2 * MBM - 1) / (2 * MBM);
  const int NCH = F / FC;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX1);
    tma_prefetch_desc(&tmW1);
    tma_prefetch_desc(&tmW2);
    for (int s = 0; s < RING; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    mbar_init(h_full, 1);
    mbar_init(h_empty, 2 * EPI_WARPS);
    mbar_init(hs_full, 2 * EPI_WARPS);
    mbar_init(hs_empty, 1);
    mbar_init(y_full, 1);
    mbar_init(y_empty, 2 * EPI_WARPS);
    mbar_init(a_free, EPI_WARPS);
    mbar_init(y0_full, 1);
    mbar_init(x1_ready, 2 * EPI_WARPS);
    mbar_init(xres_full, 1);
    for (int kb = 0; kb < KB1; ++kb) mbar_init(&okb_free[kb], 1);
    for (int kb = 0; kb < KB1; ++kb) mbar_init(&x1kb[kb], 2 * EPI_WARPS);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc_pair(tmem_slot, 512);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
#ifdef MLP_DEPHASE
  // timing experiment: odd pairs start MLP_DEPHASE cycles late, so the CTA pairs' LayerNorm phases (and
  // their HBM bursts: O / X tile loads, X stores) interleave with other pairs' MMA phases
  if ((unit0 & 1) != 0) {
    const long long t_end = clock64() + MLP_DEPHASE;
    while (clock64() < t_end) __nanosleep(1000);
  }
#endif

  if (warp == 0 || warp == 2 || warp == 3) {
    griddep_wait();                            // A (O or X1) and the residual rows come from the previous kernel
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producers
      // Box sequence per unit: A (KB1 boxes, after the previous unit's last G1 freed it), then per
      // chunk slot in MMA order: W1(c) stages, W2(c-1) stages.  Ring stage i is issued by producer i % 3.
      const int p = warp == 0 ? 0 : warp - 1;
      const uint64_t pol_w = l2_policy_evict_last();
      const uint32_t full_c = mapa_shared(smem_u32(full), 0);
      const uint32_t afull_c = mapa_shared(smem_u32(a_full), 0);
      uint32_t sc = 0;                                   // ring stage counter
      int ui = 0;
      uint8_t* sW = region_w(0);
      uint8_t* sA = region_a(0);
      auto ring_w1 = [&](int c) {
        for (int s2 = 0; s2 < S1; ++s2, ++sc) {
          const int s = int(sc % RING);
          const uint32_t ph = (sc / RING) & 1;
          if (int(sc % 3) != p) continue;               // stage sc is issued by producer sc % 3
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * KPS * 64 * 128);
          for (int j = 0; j < KPS; ++j)
            tma_load_2d_pair(sW + s * STAGE + j * 64 * 128, &tmW1, full_c + uint32_t(s) * 8, (s2 * KPS + j) * 64,
                             c * FC + rank * 64, pol_w);
        }
      };
      auto ring_w2 = [&](int c) {
        for (int kb = 0; kb < 2; ++kb, ++sc) {
          const int s = int(sc % RING);
          const uint32_t ph = (sc / RING) & 1;
          if (int(sc % 3) != p) continue;
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * T::N2_MMAS * T::B2_BOX * 128);
          for (int j = 0; j < T::N2_MMAS; ++j)
            tma_load_2d_pair(sW + s * STAGE + j * T::B2_BOX * 128, &tmW2, full_c + uint32_t(s) * 8, c * FC + kb * 64,
                             j * T::N2 + rank * T::B2_BOX, pol_w);
        }
      };
      auto ring_wo = [&](int kb0, int kb1) {             // OP: Wo k-blocks in the W2 stage format
        for (int kb = kb0; kb < kb1; ++kb, ++sc) {
          const int s = int(sc % RING);
          const uint32_t ph = (sc / RING) & 1;
          if (int(sc % 3) != p) continue;
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * T::N2_MMAS * T::B2_BOX * 128);
          for (int j = 0; j < T::N2_MMAS; ++j)
            tma_load_2d_pair(sW + s * STAGE + j * T::B2_BOX * 128, &tmWo, full_c + uint32_t(s) * 8, kb * 64,
                             j * T::N2 + rank * T::B2_BOX, pol_w);
        }
      };
      // SPLIT: G0's Wo stages -- cb0 (output columns 0..127, this CTA's 64 rows of each N = 128 MMA): 2 stages
      // of 3 k-blocks; cb12 (columns 128..383, this CTA's 128 rows of each N = 256 MMA): 6 stages of 1
      // k-block (16 KB of a 24 KB slot)
      auto ring_wo_split = [&]() {
        for (int i = 0; i < 2; ++i, ++sc) {
          const int s = int(sc % RING);
          const uint32_t ph = (sc / RING) & 1;
          if (int(sc % 3) != p) continue;
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * 3 * 64 * 128);
          for (int j = 0; j < 3; ++j)
            tma_load_2d_pair(sW + s * STAGE + j * 64 * 128, &tmWo64, full_c + uint32_t(s) * 8, (3 * i + j) * 64,
                             rank * 64, pol_w);
        }
        for (int kb = 0; kb < KB1; ++kb, ++sc) {
          const int s = int(sc % RING);
          const uint32_t ph = (sc / RING) & 1;
          if (int(sc % 3) != p) continue;
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * 2 * 64 * 128);
          for (int j = 0; j < 2; ++j)
            tma_load_2d_pair(sW + s * STAGE + j * 64 * 128, &tmWo64, full_c + uint32_t(s) * 8, kb * 64,
                             128 + rank * 128 + j * 64, pol_w);
        }
      };
      // A: this CTA's rows, once per unit.  Its k-blocks are split over the three producers (one
      // issuing thread completes ~one box per 500 cycles, and the load sits between the previous
      // unit's final-LN pass 1 and this unit's G0).  Box completions of producers 1 and 2 may reach
      // the leader's a_full before producer 0's arrive.expect_tx: the transiently negative tx-count
      // cannot complete the phase while that arrival is pending.
      auto load_a = [&](int u, int m0) {
        if (MLP_PINGPONG) {
          mbar_wait(y_full, (ui & 1) ^ 1);      // every MMA of the previous unit retired: its ring region is free
        } else {
          mbar_wait(a_empty, (ui & 1) ^ 1);     // MMAs done with the previous unit's A
          mbar_wait(a_free, (ui & 1) ^ 1);      // its LN has read the residual rows
        }
#ifdef MLP_NO_ALOAD   // timing experiment only (wrong results): the A tile is not reloaded
        if (leader && p == 0) mbar_arrive(a_full);
        if (true) return;
#endif
        if (leader && p == 0) mbar_arrive_expect_tx(a_full, 2u * T::A_BYTES);
        constexpr bool SPLIT_A = (OP || MLP_PINGPONG) && MLP_A_SPLIT;
        for (int kb = SPLIT_A ? p : 0; kb < KB1; kb += SPLIT_A ? 3 : 1)
          tma_load_2d_pair(sA + kb * MBM * 128, &tmX1, afull_c, kb * 64, m0, l2_policy_evict_first());
        if (p == 0) {
          // warm L2 with the next unit's rows: its A load waits for this unit's LN (residual from A)
          if (MLP_PREFETCH && u + units < n_units)
            for (int kb = 0; kb < KB1; ++kb) tma_prefetch_2d(&tmX1, kb * 64, m0 + units * 2 * MBM);
          if constexpr (OP)                              // LN0 residual rows (X), read from L2
            for (int kb = 0; kb < KB1; ++kb) tma_prefetch_2d(&tmR, kb * 64, m0);
        }
      };
      for (int u = unit0; u < n_units; u += units, ++ui) {
        const int m0 = u * 2 * MBM + rank * MBM;
        sA = region_a(ui);
        sW = region_w(ui);
        if (MLP_PINGPONG) {
          // this unit's ring region is the previous unit's A tile: free once its MMAs are done with it
          // and its final LN has read the residual rows; the A tile goes first (it needs only y_full)
          load_a(u, m0);
          mbar_wait(a_empty, (ui & 1) ^ 1);
          mbar_wait(a_free, (ui & 1) ^ 1);
          if constexpr (OP) {
            if constexpr (SPLIT) ring_wo_split();
            else ring_wo(0, KB1);
            if (p == 0) {
              for (int kb = 0; kb < KB1; ++kb) {
                mbar_wait(&okb_free[kb], ui & 1);
                if (kb == 0) {
                  MTL(M_XLOAD, ui);
                  mbar_arrive_expect_tx(xres_full, uint32_t(T::A_BYTES));
                }
                tma_load_2d(sA + kb * MBM * 128, &tmR, xres_full, kb * 64, m0);
              }
            }
          }
          for (int c = 0; c < NCH; ++c) {
            ring_w1(c);
            if (c > 0) ring_w2(c - 1);
          }
          ring_w2(NCH - 1);
          continue;
        }
        // OP: the first RING Wo stages need only ring slots freed by the previous unit's G2, so
        // every producer issues its share of them before it waits for the A tile to be released;
        // the remaining Wo stages need slots that G0 frees, i.e. after A has landed (issuing them
        // before A would deadlock: G0 waits for A).
        constexpr int WO_EARLY = (OP && MLP_A_SPLIT) ? (RING < KB1 ? RING : KB1) : 0;
        if constexpr (OP) ring_wo(0, WO_EARLY);
        if ((OP && MLP_A_SPLIT) || p == 0) load_a(u, m0);   // !OP: producer 0 alone (unchanged)
        if constexpr (OP) {
          ring_wo(WO_EARLY, KB1);
          if (p == 0) {
            // as G0 consumes O k-block by k-block, each freed k-block of the A tile takes the same columns
            // of this unit's X rows: the LN0 residual, read from smem (its load overlaps G0)
            for (int kb = 0; kb < KB1; ++kb) {
              mbar_wait(&okb_free[kb], ui & 1);
              if (kb == 0) {
                MTL(M_XLOAD, ui);
                mbar_arrive_expect_tx(xres_full, uint32_t(T::A_BYTES));
              }
              tma_load_2d(sA + kb * MBM * 128, &tmR, xres_full, kb * 64, m0);
            }
          }
        }
        for (int c = 0; c < NCH; ++c) {
          ring_w1(c);
          if (c > 0) ring_w2(c - 1);
        }
        ring_w2(NCH - 1);
      }
    }
  } else if (warp == 1 && leader) {
    griddep_launch_dependents();
    // -------------------------------------------------------------------- MMA issuer (leader)
    constexpr uint32_t idesc1 = umma_idesc_bf16(2 * MBM, FC);
    constexpr uint32_t idesc2 = umma_idesc_bf16(2 * MBM, T::N2);
    const uint64_t hs_desc0 = umma_desc_sw128(smem_u32(sHs));
    uint64_t a_desc0 = umma_desc_sw128(smem_u32(region_a(0)));
    uint64_t w_desc0 = umma_desc_sw128(smem_u32(region_w(0)));
#ifdef MLP_TRACE
    long long tw[5] = {0, 0, 0, 0, 0};
    const long long t_start = clock64();
#endif
    uint32_t sc = 0;        // ring stage counter
    uint32_t hc = 0;        // chunks issued (G1) -> h_full / h_empty phases
    uint32_t gc = 0;        // chunks issued (G2) -> hs_full / hs_empty phases
    int ui = 0;
    auto g2 = [&](int c, int uiu) {
      if (!OP && c == 0) {
        MW(y_empty, (uiu & 1) ^ 1, 0);               // LN of the previous unit drained Y
        tc_fence_after();
      }
      if (CHASE && c == 0) {
        MW(x1_ready, uiu & 1, 1);                    // LN0 has read all of Y0 (G2 overwrites Y)
        tc_fence_after();
      }
      MW(hs_full, gc & 1, 1);                        // both CTAs' Hs(c) written
      tc_fence_after();
      for (int kb = 0; kb < 2; ++kb, ++sc) {
        const int s = int(sc % RING);
        MW(&full[s], (sc / RING) & 1, 2);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad = hs_desc0 + uint64_t((kb * MBM * 128) >> 4);
          const uint64_t bd = w_desc0 + uint64_t((s * STAGE) >> 4);
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < T::N2_MMAS; ++j)
              tc_mma_bf16_pair(tmem_base + j * T::N2, ad + uint64_t(k * 2),
                               bd + uint64_t((j * T::B2_BOX * 128 + k * 32) >> 4), idesc2, (c | kb | k) != 0);
          tc_commit_pair_mc(&empty[s], 0x3);
        }
        __syncwarp();
      }
      if (elect_one()) {
        tc_commit_pair_mc(hs_empty, 0x3);               // Hs free for the next chunk
        if (c == NCH - 1) tc_commit_pair_mc(y_full, 0x3);
      }
      __syncwarp();
      ++gc;
    };
    // SPLIT: G0 column block 0 of unit j (N = 128 into the H-chunk columns): issued at the start (j = 0)
    // or right after the previous unit's last G2, i.e. under its final LayerNorm
    auto g0_cb0 = [&](int j) {
      const uint64_t ad0 = umma_desc_sw128(smem_u32(region_a(j))), wd0 = umma_desc_sw128(smem_u32(region_w(j)));
      MW(a_full, j & 1, 3);
      MTL(M_AFULL, j);
      tc_fence_after();
      for (int i = 0; i < 2; ++i, ++sc) {
        const int s = int(sc % RING);
        MW(&full[s], (sc / RING) & 1, 2);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bd0 = wd0 + uint64_t((s * STAGE) >> 4);
          for (int jj = 0; jj < 3; ++jj) {
            const int kb = 3 * i + jj;
            const uint64_t ad = ad0 + uint64_t((kb * MBM * 128) >> 4);
            const uint64_t bd = bd0 + uint64_t((jj * 64 * 128) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_bf16_pair(tmem_base + H_COL, ad + uint64_t(k * 2), bd + uint64_t(k * 2), idesc1, (kb | k) != 0);
          }
          tc_commit_pair_mc(&empty[s], 0x3);
        }
        __syncwarp();
      }
    };
    if constexpr (SPLIT)
      if (unit0 < n_units) g0_cb0(0);
    for (int u = unit0; u < n_units; u += units, ++ui) {
      a_desc0 = umma_desc_sw128(smem_u32(region_a(ui)));
      w_desc0 = umma_desc_sw128(smem_u32(region_w(ui)));
#ifdef MLP_TL
      if (ui == 0 && blockIdx.x == 0 && lane == 0) g_mtl_t0 = clock64();
#endif
      if constexpr (!SPLIT) {
        MW(a_full, ui & 1, 3);
        MTL(M_AFULL, ui);
        tc_fence_after();
      }
      if constexpr (SPLIT) {
        // G0 columns 128..383 (N = 256) into Y[128, 384): the previous unit's final LN has drained Y
        MW(y_empty, (ui & 1) ^ 1, 0);
        tc_fence_after();
        constexpr uint32_t idesc256 = umma_idesc_bf16(2 * MBM, 256);
        for (int kb = 0; kb < KB1; ++kb, ++sc) {
          const int s = int(sc % RING);
          MW(&full[s], (sc / RING) & 1, 2);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = a_desc0 + uint64_t((kb * MBM * 128) >> 4);
            const uint64_t bd = w_desc0 + uint64_t((s * STAGE) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_bf16_pair(tmem_base + 128, ad + uint64_t(k * 2), bd + uint64_t(k * 2), idesc256, (kb | k) != 0);
            tc_commit_pair_mc(&empty[s], 0x3);
            tc_commit_pair_mc(&okb_free[kb], 0x3);   // O k-block kb read by both column blocks
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit_pair_mc(y0_full, 0x3);
        __syncwarp();
        MTL(M_G0ISS, ui);
        if constexpr (!CHASE) {
          MW(x1_ready, ui & 1, 1);                    // both CTAs' X1 written into A
          MTL(M_X1R, ui);
          tc_fence_after();
        }
      } else if constexpr (OP) {
        // G0: Y = O Wo^T (the previous unit's final LN has drained Y)
        MW(y_empty, (ui & 1) ^ 1, 0);
        tc_fence_after();
        for (int kb = 0; kb < KB1; ++kb, ++sc) {
          const int s = int(sc % RING);
          MW(&full[s], (sc / RING) & 1, 2);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = a_desc0 + uint64_t((kb * MBM * 128) >> 4);
            const uint64_t bd = w_desc0 + uint64_t((s * STAGE) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int j = 0; j < T::N2_MMAS; ++j)
                tc_mma_bf16_pair(tmem_base + j * T::N2, ad + uint64_t(k * 2),
                                 bd + uint64_t((j * T::B2_BOX * 128 + k * 32) >> 4), idesc2, (kb | k) != 0);
            tc_commit_pair_mc(&empty[s], 0x3);
            tc_commit_pair_mc(&okb_free[kb], 0x3);   // O k-block kb read: X may take its place
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit_pair_mc(y0_full, 0x3);
        __syncwarp();
        MTL(M_G0ISS, ui);
        MW(x1_ready, ui & 1, 1);                      // both CTAs' X1 written into A
        MTL(M_X1R, ui);
        tc_fence_after();
      }
      for (int c = 0; c < NCH; ++c) {
        MW(h_empty, (hc & 1) ^ 1, 4);                // epilogue drained H(c-1)
        tc_fence_after();
        for (int s2 = 0; s2 < S1; ++s2, ++sc) {
          const int s = int(sc % RING);
          MW(&full[s], (sc / RING) & 1, 2);
          tc_fence_after();
          if (CHASE && c == 0) {
            // chunk 0 chases LN0's pass 2: k-block kb once X1 k-block kb (and, for kb <= 1, the H reads) is done
            for (int j = 0; j < KPS; ++j) {
              const int kb = s2 * KPS + j;
              MW(&x1kb[kb < 1 ? 1 : kb], ui & 1, 1);
              tc_fence_after();
              if (elect_one()) {
                const uint64_t ad = a_desc0 + uint64_t((kb * MBM * 128) >> 4);
                const uint64_t bd = w_desc0 + uint64_t((s * STAGE + j * 64 * 128) >> 4);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  tc_mma_bf16_pair(tmem_base + H_COL, ad + uint64_t(k * 2), bd + uint64_t(k * 2), idesc1, (kb | k) != 0);
                if (j == KPS - 1) tc_commit_pair_mc(&empty[s], 0x3);
              }
              __syncwarp();
            }
            if (s2 == 0) MTL(M_X1R, ui);
          } else {
          if (elect_one()) {
            const uint64_t bd0 = w_desc0 + uint64_t((s * STAGE) >> 4);
            for (int j = 0; j < KPS; ++j) {
              const int kb = s2 * KPS + j;
              const uint64_t ad = a_desc0 + uint64_t((kb * MBM * 128) >> 4);
              const uint64_t bd = bd0 + uint64_t((j * 64 * 128) >> 4);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc_mma_bf16_pair(tmem_base + H_COL, ad + uint64_t(k * 2), bd + uint64_t(k * 2), idesc1, (kb | k) != 0);
            }
            tc_commit_pair_mc(&empty[s], 0x3);
          }
          __syncwarp();
          }
        }
        if (elect_one()) {
          tc_commit_pair_mc(h_full, 0x3);
          if (c == NCH - 1) tc_commit_pair_mc(a_empty, 0x3);   // A free for the next unit
        }
        __syncwarp();
        if (c == 0) MTL(M_G1_0, ui);
        ++hc;
        if (c > 0) g2(c - 1, ui);
      }
      g2(NCH - 1, ui);
      if constexpr (SPLIT) {
        if (u + units < n_units) {
          MW(h_empty, (hc & 1) ^ 1, 4);              // the GELU of the last chunk drained H
          tc_fence_after();
          g0_cb0(ui + 1);
        }
      }
    }
#ifdef MLP_TRACE
    if (lane == 0 && blockIdx.x < 8)
      printf("MLP_TRACE cta %d units %d total %lld | wait y_empty %lld hs_full %lld ring %lld a_full %lld h_empty %lld\n",
             int(blockIdx.x), ui, clock64() - t_start, tw[0], tw[1], tw[2], tw[3], tw[4]);
#endif

  } else if (warp >= 4) {
    griddep_wait();
    // ------------------------------------------------------------------ epilogue (warps 4..11)
    const int q = warp & 3;                    // TMEM lane quadrant
    const int hh = (warp - 4) >> 2;            // column part (0 .. NP-1)
    const int row_l = q * 32 + lane;           // row within the CTA tile
    const uint32_t hs_full_c = mapa_shared(smem_u32(hs_full), 0);
    const uint32_t h_empty_c = mapa_shared(smem_u32(h_empty), 0);
    const uint32_t y_empty_c = mapa_shared(smem_u32(y_empty), 0);
    const uint32_t t_row = tmem_base + (uint32_t(q * 32) << 16);
    uint32_t hc = 0;
    int ui = 0;
#ifdef MLP_TRACE
    long long et[12] = {}, el = 0;
#define ETR(i) do { const long long _c = clock64(); if (i > 0) et[i - 1] += _c - el; el = _c; } while (0)
#else
#define ETR(i) do {} while (0)
#endif
    const uint32_t x1_ready_c = mapa_shared(smem_u32(x1_ready), 0);
    for (int u = unit0; u < n_units; u += units, ++ui) {
      const int m0 = u * 2 * MBM + rank * MBM;
      uint8_t* const sA = region_a(ui);
      if constexpr (OP) {
        // ---- LN0 epilogue (K6): X1 = LN_a(Y + bo + X) -> bf16 into the A tile (swizzled K-major)
        if constexpr (!MLP_LN_CPARAM) {
          constexpr int PER = (3 * D + EPI_WARPS * 32 - 1) / (EPI_WARPS * 32);
          float cv[PER];
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            const int k = threadIdx.x - 128 + i * EPI_WARPS * 32;
            cv[i] = k < D ? __ldg(bo + k) : k < 2 * D ? __ldg(gamma1 + k - D) : k < 3 * D ? __ldg(beta1 + k - 2 * D) : 0.f;
          }
#pragma unroll
          for (int i = 0; i < PER; ++i) {     // Hs idle: the previous unit's LN is done, chunk 0 not yet
            const int k = threadIdx.x - 128 + i * EPI_WARPS * 32;
            if (k < 3 * D) s_b2[k] = to_ct(cv[i]);
          }
          asm volatile("bar.sync 5, %0;" ::"r"(EPI_WARPS * 32) : "memory");
        }
        const int row = m0 + row_l;
        (void)row;
        const ResidualSmemA rg{sA, row_l, hh * (D / NP)};
        mbar_wait(xres_full, ui & 1);          // X rows in the A tile (G0 is done with O)
        MTL(M_XRES, ui);
#if defined(MLP_SKIP_LN) && (MLP_SKIP_LN & 1)   // timing experiment only (wrong results)
        mbar_wait(y0_full, ui & 1);
        tc_fence_after();
        if (false)
#endif
        const CT* c_b = MLP_LN_CPARAM ? reinterpret_cast<const CT*>(lc.v) : s_b2;
        const CT* c_g = MLP_LN_CPARAM ? reinterpret_cast<const CT*>(lc.v + D) : s_gamma;
        const CT* c_e = MLP_LN_CPARAM ? reinterpret_cast<const CT*>(lc.v + 2 * D) : s_beta;
        ln_epilogue<D, D / NP, (NP <= 2 || MLP_LN_PIPE), SPLIT ? 128u : 0u, H_COL, CT>(t_row, hh * (D / NP), rg, c_b, c_g, c_e, stats, q, hh, lane, eps,
                              [&] {
                                mbar_wait(y0_full, ui & 1);
                                MTL(M_Y0, ui);
                                tc_fence_after();
                              },
                              [&](const uint32_t (&p)[16], int col) {   // row row_l, columns col .. col+31
                                uint8_t* base = sA + (col >> 6) * (MBM * 128) + row_l * 128;
                                const int j0 = (col & 63) >> 3;
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                  *reinterpret_cast<uint4*>(base + (((j0 + i) ^ (row_l & 7)) << 4)) =
                                      make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
                                if constexpr (CHASE) {   // X1 k-block col / 64: this warp's 32 columns are in
                                  fence_proxy_async_smem();
                                  tc_fence_before();
                                  __syncwarp();
                                  if (lane == 0) mbar_arrive_cluster_release(mapa_shared(smem_u32(&x1kb[col >> 6]), 0));
                                }
                              });
        tc_fence_before();                     // Y reads done before G2(0) may accumulate into Y
        fence_proxy_async_smem();              // X1 (generic writes) -> visible to the MMA
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_release(x1_ready_c);
        asm volatile("bar.sync 5, %0;" ::"r"(EPI_WARPS * 32) : "memory");   // LN0 scratch free
      }
      // H(c) columns [col0, col0 + W) of this row: TMEM -> registers (then the accumulator is released),
      // + bias, GELU, bf16 -> Hs (k-block col / 64, 16-byte chunk (col % 64) / 8 at (chunk ^ (row & 7)))
      auto gelu_chunk = [&](auto wc, int col0, int c) {
        constexpr int W = decltype(wc)::value;
        const float4* bp = reinterpret_cast<const float4*>(b1 + c * FC + col0);
        float4 bb[W / 4];
#pragma unroll
        for (int i = 0; i < W / 4; ++i) bb[i] = __ldg(bp + i);
        uint32_t rh[W];
        ETR(0);
        mbar_wait(h_full, hc & 1);
        ETR(1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < W / 32; ++s) tmem_ld32(t_row + H_COL + col0 + 32 * s, *reinterpret_cast<uint32_t(*)[32]>(rh + 32 * s));
        if constexpr (W % 32 == 16) tmem_ld16(t_row + H_COL + col0 + W - 16, *reinterpret_cast<uint32_t(*)[16]>(rh + W - 16));
#pragma unroll
        for (int s = 0; s < W / 32; ++s) tmem_ld_wait_regs(*reinterpret_cast<uint32_t(*)[32]>(rh + 32 * s));
        if constexpr (W % 32 == 16) tmem_ld_wait_regs16(*reinterpret_cast<uint32_t(*)[16]>(rh + W - 16));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(h_empty_c);
        ETR(2);
        uint32_t pk[W / 2];
#pragma unroll
        for (int i = 0; i < W / 4; ++i) {
          float v0 = __uint_as_float(rh[4 * i]) + bb[i].x, v1 = __uint_as_float(rh[4 * i + 1]) + bb[i].y;
          float v2 = __uint_as_float(rh[4 * i + 2]) + bb[i].z, v3 = __uint_as_float(rh[4 * i + 3]) + bb[i].w;
          gelu2(v0, v1);
          gelu2(v2, v3);
          pk[2 * i] = pack_bf16x2(v0, v1);
          pk[2 * i + 1] = pack_bf16x2(v2, v3);
        }
        ETR(3);
        mbar_wait(hs_empty, (hc & 1) ^ 1);      // Hs free: G2(c-1) retired
        ETR(4);
#pragma unroll
        for (int j = 0; j < W / 8; ++j) {
          const int col = col0 + 8 * j;
          *reinterpret_cast<uint4*>(sHs + (col >> 6) * MBM * 128 + row_l * 128 + ((((col & 63) >> 3) ^ (row_l & 7)) << 4)) =
              make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
        ETR(5);
        fence_proxy_async_smem();              // generic-proxy writes -> visible to the MMA (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_release(hs_full_c);
        ETR(6);
      };
      for (int c = 0; c < NCH; ++c, ++hc) {
        if constexpr (NP == 3) {               // 128 columns over 3 warps: 48 + 48 + 32
          if (hh < 2) gelu_chunk(std::integral_constant<int, 48>{}, 48 * hh, c);
          else gelu_chunk(std::integral_constant<int, 32>{}, 96, c);
        } else {
          gelu_chunk(std::integral_constant<int, HC>{}, HC * hh, c);
        }
      }
      // ---- LN epilogue: X2 = LN(Y + b2 + X1); output staged per warp in Hs (free after G2(last))
      if constexpr (MLP_LN_CPARAM) {
        ETR(0);
        mbar_wait(y_full, ui & 1);            // Hs no longer read by the MMA
        MTL(M_YFULL, ui);
        ETR(7);
      } else {
        constexpr int PER = (3 * D + EPI_WARPS * 32 - 1) / (EPI_WARPS * 32);
        float cv[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {       // loads in flight while G2(last) finishes
          const int k = threadIdx.x - 128 + i * EPI_WARPS * 32;
          cv[i] = k < D ? __ldg(b2 + k) : k < 2 * D ? __ldg(gamma + k - D) : k < 3 * D ? __ldg(beta + k - 2 * D) : 0.f;
        }
        ETR(0);
        mbar_wait(y_full, ui & 1);            // Hs no longer read by the MMA
        MTL(M_YFULL, ui);
        ETR(7);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int k = threadIdx.x - 128 + i * EPI_WARPS * 32;
          if (k < 3 * D) s_b2[k] = to_ct(cv[i]);
        }
        asm volatile("bar.sync 5, %0;" ::"r"(EPI_WARPS * 32) : "memory");
      }
      // residual X1 = this unit's A tile, still resident (the next unit's A load waits for a_free)
      const ResidualSmemA ra{sA, row_l, hh * (D / NP)};
      uint8_t* stg0 = sHs + (warp - 4) * (MLP_STG * 2048);
#if defined(MLP_SKIP_LN) && (MLP_SKIP_LN & 2)   // timing experiment only (wrong results)
      mbar_wait(y_full, ui & 1);
      tc_fence_after();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_free);
      if (false)
#endif
      const CT* f_b = MLP_LN_CPARAM ? reinterpret_cast<const CT*>(lc.v + 3 * D) : s_b2;
      const CT* f_g = MLP_LN_CPARAM ? reinterpret_cast<const CT*>(lc.v + 4 * D) : s_gamma;
      const CT* f_e = MLP_LN_CPARAM ? reinterpret_cast<const CT*>(lc.v + 5 * D) : s_beta;
      ln_epilogue<D, D / NP, (NP <= 2 || MLP_LN_PIPE), 0u, 0u, CT>(t_row, hh * (D / NP), ra, f_b, f_g, f_e, stats, q, hh, lane, eps,
                            [&] {
                              mbar_wait(y_full, ui & 1);
                              tc_fence_after();
                            },
                            [&](const uint32_t (&p)[16], int col) {
#ifndef MLP_NO_FSTORE   // timing experiment only (wrong results)
#if MLP_STORE_DIRECT
                              store_row_64B(p, lane, out, m0 + q * 32, M, D, col);
#else
                              store_rows_32x32(stg0, p, lane, out, m0 + q * 32, M, D, col);
#endif
#else
                              if (p[0] == 0x7fffffffu && col < 0) out[0] = 0;
#endif
                            },
                            [&] {                // residual read for the last time: the A tile may take
                              __syncwarp();      // the next unit's rows while pass 2 runs
                              if (lane == 0) mbar_arrive(a_free);
                              MTL(M_AFREE, ui);
                            });
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(y_empty_c);
      MTL(M_YEMPTY, ui);
      // LN constants / stats (in Hs) consumed before the next unit's first chunk overwrites Hs
      ETR(10);
      asm volatile("bar.sync 5, %0;" ::"r"(EPI_WARPS * 32) : "memory");
      ETR(11);
    }
    if (lane == 0) bulk_wait_all();
#ifdef MLP_TRACE
    if (lane == 0 && blockIdx.x < 1)
      printf("MLP_EPI warp %d chunks %u | h_full %lld ld %lld gelu %lld hs_empty %lld write %lld fence+arrive %lld "
             "| y_full %lld consts %lld bar5a %lld LN %lld bar5b %lld | LN pass1 %lld bar %lld pass2 %lld\n", warp, hc,
             et[0], et[1], et[2], et[3], et[4], et[5], et[6], et[7], et[8], et[9], et[10],
#ifdef LN_TRACE
             g_ln_trace[warp][0], g_ln_trace[warp][1], g_ln_trace[warp][2]
#else
             0ll, 0ll, 0ll
#endif
             );
#endif
  }
  tc_fence_before();
  cluster_sync();
#ifdef MLP_TL
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (g_mtl_launch == 3)
      for (int j = 0; j < 4; ++j)
        for (int e = 0; e < M_N; ++e) printf("MTL %8lld unit %d %s\n", g_mtlbuf[j][e], 10 + j, g_mtl_names[e]);
    ++g_mtl_launch;
  }
#endif
  if (warp == 2) {
    __syncwarp();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

template <int D, bool OP>
cudaError_t launch_mlp_t(const MlpArgs& a, cudaStream_t st) {
  using T = MlpCfg<D>;
  auto kern = mlp_tc_kernel<D, OP>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t n_units = (a.M + 2 * MBM - 1) / (2 * MBM);
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int pairs = int(std::min<int64_t>(n_units, (sms > 0 ? sms : 148) / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(2 * pairs));
  cfg.blockDim = dim3(T::THREADS);
  cfg.dynamicSmemBytes = size_t(T::SMEM);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const CUtensorMap& tmWo = OP ? *a.tmWo : *a.tmW2;
  const CUtensorMap& tmR = OP ? *a.tmX : *a.tmA;
  const CUtensorMap& tmWo64 = a.tmWo64 ? *a.tmWo64 : tmWo;
  MlpConsts<D> lc{};
  if (MLP_LN_CPARAM) {
    if (!a.ln_host) return cudaErrorInvalidValue;
    for (int i = 0; i < 6 * D; ++i) lc.v[i] = a.ln_host[i];
  }
  if (OP && MLP_PINGPONG && MLP_G0SPLIT && D == 384 && !a.tmWo64) return cudaErrorInvalidValue;
  return cudaLaunchKernelEx(&cfg, kern, *a.tmA, *a.tmW1, *a.tmW2, tmWo, tmR, tmWo64, lc, int(a.M), a.F, a.b1, a.b2, a.gamma,
                            a.beta, a.bo, a.gamma1, a.beta1, a.x, a.out, a.eps);
}

}  // namespace

bool mlp_fused_supported(int d, int ffn) { return (d == 384 || d == 64) && ffn % FC == 0 && ffn > 0; }

cudaError_t launch_mlp(const MlpArgs& a, cudaStream_t st) {
  if (a.M <= 0) return cudaSuccess;
  if (!mlp_fused_supported(a.D, a.F)) return cudaErrorInvalidValue;
  const bool op = a.tmWo != nullptr;
  switch (a.D) {
    case 64: return op ? launch_mlp_t<64, true>(a, st) : launch_mlp_t<64, false>(a, st);
    case 384: return op ? launch_mlp_t<384, true>(a, st) : launch_mlp_t<384, false>(a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace surge
