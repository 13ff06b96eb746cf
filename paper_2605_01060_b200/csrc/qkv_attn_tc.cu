// qkv_attn_tc.cu -- K4 + K5 with the attention on the 5th-gen tensor cores (
// reading R10: per text, softmax(q k^T / sqrt(d_h)) v over the text's own tokens, bidirectional).
//
// One CTA per SM (cta_group::1), weight-stationary: the CTA keeps one 192-row slice of the permuted
// W_qkv ([Q | K | V] of two whole heads at d_h = 32; 144 KB) in shared memory and walks text-aligned
// 128-row tiles of X (every tile = whole texts, host-built records, internal.h AttRec).  Per tile t:
//   QKV(t)   = X_t W_slice^T                      tcgen05.mma M=128 N=192, 24 x K=16, A (X) streamed by TMA
//   staging  : + bias -> bf16; Q -> TMEM (the A operand of S, "TS" form), K and V -> smem as stored
//              (row = key, [X_h0 | X_h1], 128-byte swizzle): K is S's K-major B, V is P V's MN-major B
//   S(t,h)   = Q_h K_h^T                          M=128 N=128 (all keys of the tile) K=32, A from TMEM
//   softmax  : each row over its own text's keys only (block-diagonal mask), exp2 form with the row max
//              of the raw scores (p = 2^(s q - m q), q = log2(e)/sqrt(d_h)); P (bf16) written over S in TMEM
//   O(t,h)   = P_h V_h                            M=128 N=32 K=128 keys, A = P from TMEM
//   O / rowsum -> bf16 -> global O [T x d] (the head's 32 columns).
// QKV, S and P never leave the SM.  The attention MMAs cost ~1.5K tensor cycles per tile next to the
// 2.4K of the projection (scripts/microbench/umma_shapes.cu); with the CTA-pair kernel (gemm_tc.cu,
// EPI_QKV_ATTN) the same attention would need cta_group::2 MMAs over both CTAs' 256 keys (2x the cost),
// and its mma.sync attention cannot overlap tcgen05 on the same SM.  The layouts (TS operand: lane =
// row, column c = elements 2c, 2c+1; the K tile; V as an MN-major B operand) are checked by scripts/microbench/ts_attn_check.cu.
//
// Tensor-pipe issue order (one thread): PV(t-1, h0), PV(t-1, h1), S(t, h0), QKV(t+1)[kb 0,1], S(t, h1),
// QKV(t+1)[kb 2..5], PV(t, h0), ...: the softmax of tile t (CUDA cores) runs under QKV(t+1), the staging
// of t+1 under PV(t), the O read-out of (t, h) under the MMAs issued before S(t+1, h).
// TMEM (512 columns): [0,192) QKV accumulator; [192,224) Q bf16 (16 columns per head);
// [256 + 128 h, +128) S_h, then P_h in its first 64 columns and O_h in the next 32.
//
// Warps: 0, 2, 3 TMA producers (B slice once, the A ring); 1 MMA issuer; 2 also allocates TMEM;
// 4..15 epilogue, warp w reads TMEM lane quadrant w % 4 (rows 32 (w % 4) ..), part (w - 4) / 4:
//   part 0: Q -> TMEM, K -> smem, and the text window [ta, te) of every row (from the tile's 128-bit
//   start-of-text mask, one coalesced 128-byte load of the record) -> a shared table;
//   parts 1, 2: head h = part - 1: V_h -> registers -> smem (after PV(t-1, h) has read the previous
//   one), O of tile t-1 (TMEM -> / rowsum -> global), softmax of tile t.
// Numerics vs the mma.sync path (attn_tile.cuh): same bf16 Q/K/V/P values and softmax formula (one
// max per text: the round-1 path takes one per 32 keys, i.e. the same for texts <= 32 tokens); fp32
// accumulation order of S, P V and the row sum differs (not bit-identical; reading R21).
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace surge {

namespace {

constexpr int BM = 128;
constexpr int BN = ATT_SLICE;                  // 192
constexpr int DH = 32;
constexpr int HG = BN / (3 * DH);              // 2 heads per slice
constexpr int D = 384;                         // model dim (K of the projection)
constexpr int KB1 = D / 64;                    // 6 k-blocks
#ifndef QA_EXP16
#define QA_EXP16 0                     // softmax exponentials on f16x2 pairs (half the MUFU ops)
#endif
#ifndef QA_STAGES
#define QA_STAGES 3
#endif
// QA_MC: the six CTAs holding the six slices of W_qkv form one thread-block cluster that walks the same
// tiles; each k-block of X is loaded from L2 once per cluster (by CTA kb % 6) and multicast into all six
// A rings (a slot is refilled once all six MMA issuers have released it: multicast commits)
#ifndef QA_MC
#define QA_MC 0                        // measured slower (256 vs 233 ms per 2M texts): off
#endif
// QA_PF_MODE: the L2 prefetch of a later tile's X rows.  0: all six boxes by every CTA ahead of k-block 0's
// load; 1: box kb right after the load of k-block kb; 2: as 1, but box kb by slice kb only (each box
// prefetched once per group).  (The TMA unit serves requests in order: prefetches queued ahead of a load
// delay it.)
#ifndef QA_PF_MODE
#define QA_PF_MODE 0
#endif
constexpr int STAGES = QA_STAGES;
constexpr int A_STAGE = BM * 128;              // 16 KB: 128 rows x 64 bf16
constexpr int B_KBLK = BN * 128;               // 24 KB: 192 rows x 64 bf16
// QA_HS: head-split staging -- 8 epilogue warps, the four of head h stage Q_h, K_h and V_h of tile t
// themselves, drain O(t-1, h) and arrive on one per-head barrier (staged[h] = v_ready[h]); S(t, h) waits
// only for its own head, and no drain waits for the other head's (or a separate staging part's) work.
#ifndef QA_HS
#define QA_HS 1
#endif
// QA_DYN (with QA_HS): the MMA issuer polls while it waits (for an A stage, the accumulator, a staged head)
// and issues P V(t, h) as soon as the softmax of (t, h) is done, instead of at the start of tile t + 1
#ifndef QA_DYN
#define QA_DYN 0
#endif
#ifndef QA_LB
#define QA_LB 2                        // pieces per TMEM load batch in the long-window softmax
#endif
#ifndef QA_DYN_HINT
#define QA_DYN_HINT 200                // ns a dyn wait sleeps before it looks at the softmax barriers again
#endif
constexpr int EPI_WARPS = QA_HS ? 8 : 12;   // 12: 128 registers per thread at 512 threads
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr int HEAD = 2048;                     // barriers + TMEM slot
constexpr int OFF_B = HEAD;
constexpr int OFF_K = OFF_B + KB1 * B_KBLK;    // K tile [128 keys][128 B]: [K_h0 | K_h1] per key
constexpr int OFF_V = OFF_K + BM * 128;        // V tile [128 keys][128 B]: [V_h0 | V_h1] per key (MN-major B)
constexpr int OFF_A = OFF_V + BM * 128;
constexpr int SMEM = OFF_A + STAGES * A_STAGE;
static_assert(SMEM <= 227 * 1024, "shared memory");
constexpr uint32_t T_ACC = 0, T_Q = 192, T_S = 256;

// QA_TL: per-tile event timeline of CTA 0, tiles 40..43 of the 4th launch, buffered in global memory and
// printed at the end of the kernel (timing experiments only)
#ifdef QA_TL
__device__ long long g_tl_t0;
__device__ int g_tl_launch;
__device__ long long g_tlbuf[4][32];
__device__ int g_tl_tile;    // loop index of the producers (TL of the loads)
enum { E_QLO, E_QHI, E_STG, E_QKR, E_VR, E_S0, E_S1, E_SF0, E_SF1, E_PR0, E_PR1, E_PV0, E_PV1, E_OE0, E_OE1,
       E_KB0, E_LD0 = E_KB0 + 6, E_DR0 = E_LD0 + 6, E_DR1, E_TE, E_N };
__device__ const char* const g_tl_names[E_N] = {"qkv_lo_iss", "qkv_hi_iss", "stg_start", "qk_ready", "v_ready",
    "s0_iss", "s1_iss", "sfull0", "sfull1", "pready0", "pready1", "pv0_iss", "pv1_iss", "oempty0", "oempty1",
    "full_kb0", "full_kb1", "full_kb2", "full_kb3", "full_kb4", "full_kb5",
    "load_kb0", "load_kb1", "load_kb2", "load_kb3", "load_kb4", "load_kb5", "drained0", "drained1", "tempty"};
#define TL(ev, j) do { if (blockIdx.x == 0 && g_tl_launch == 3 && (j) >= 40 && (j) < 44 && (threadIdx.x & 31) == 0 && \
    (threadIdx.x < 128 || (threadIdx.x >> 5) % 4 == 0)) g_tlbuf[(j) - 40][ev] = clock64() - g_tl_t0; } while (0)
#else
#define TL(ev, j) do {} while (0)
#endif
// QA_TRACE: per-wait cycle counters of the MMA issuer and the epilogue parts (CTA 0 prints averages)
#ifdef QA_TRACE
#define QW(bar, par, slot)                      \
  do {                                          \
    const long long _t0 = clock64();            \
    mbar_wait(bar, par);                        \
    tw[slot] += clock64() - _t0;                \
  } while (0)
#else
#define QW(bar, par, slot) mbar_wait(bar, par)
#endif

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// TMA load of a 2-D box into the same smem offset of every CTA in `mask` (bytes completed on each CTA's
// barrier at `bar`'s offset)
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const void* desc, uint64_t* bar, int32_t c0, int32_t c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// arrive on the barrier at `bar`'s offset in every CTA of `mask` once this thread's prior MMAs completed
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// non-blocking phase test, the same answer in every lane of the warp (lane 0's)
__device__ __forceinline__ bool mbar_test_warp(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}
// wait up to ~hint ns for a phase (suspended, not spinning); the same answer in every lane (lane 0's)
__device__ __forceinline__ bool mbar_try_warp(uint64_t* bar, uint32_t parity, uint32_t hint) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(hint)
      : "memory");
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// 32-byte global store (STG.256, sm_100)
__device__ __forceinline__ void st_global_v8(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e,
                                             uint32_t f, uint32_t g, uint32_t h) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d), "r"(e),
               "r"(f), "r"(g), "r"(h)
               : "memory");
}
// byte offset of element (row, k) in a 128-byte-swizzled K-major tile of 64-element rows
__device__ __forceinline__ uint32_t sw128_off(int row, int k) {
  return uint32_t(row) * 128u + uint32_t(((k >> 3) ^ (row & 7)) << 4) + uint32_t(k & 7) * 2u;
}

// acc (32 fp32 columns of one row) + bias (shared memory) -> 16 packed bf16 pairs
__device__ __forceinline__ void bias_pack32(const uint32_t (&r)[32], const float* b, uint32_t (&p)[16]) {
  const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 bb = b4[i];
    const f32x2 v01 = fadd2(f2(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1])), f2(bb.x, bb.y));
    const f32x2 v23 = fadd2(f2(__uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3])), f2(bb.z, bb.w));
    p[2 * i] = pack_bf16x2(f2lo(v01), f2hi(v01));
    p[2 * i + 1] = pack_bf16x2(f2lo(v23), f2hi(v23));
  }
}

// softmax of (t, h) over each row's own text window [ta, te) of S_h (TMEM columns at sh; the warp's rows'
// windows lie in the 16-column pieces [p0, p1]); P (bf16) is written over S, pieces outside [p0, p1] are
// zeroed; returns the row sum of the (bf16-rounded-from) exponentials.  Ends with the TMEM stores complete
// and tcgen05.fence::before_thread_sync (the caller arrives on pready).
__device__ __forceinline__ float qa_softmax(uint32_t sh, uint64_t* sfull_h, int it, int h, int ta, int te, int p0,
                                            int p1, float qs) {
  mbar_wait(sfull_h, it & 1);
  TL(h ? E_SF1 : E_SF0, it);
  tc_fence_after();
  float l = 0.f;
  if (p1 - p0 < 4) {
    // common case: one load group of <= 4 pieces (64 columns)
    uint32_t sv[4][16];
#pragma unroll
    for (int g = 0; g < 4; ++g)
      if (p0 + g <= p1) tmem_ld16(sh + 16 * (p0 + g), sv[g]);
    tmem_ld_wait();
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int i = 0; i < 16; ++i) asm volatile("" : "+r"(sv[g][i]));
    // this row's window as a bit mask over the 64 loaded columns; scores outside it -> -inf
    // (2^(-inf) = 0 below, so P is zero there with no further test)
    const int a = ta - 16 * p0, b = te - 16 * p0;
    const uint64_t wm = te > ta ? ((b >= 64 ? ~0ull : ((1ull << b) - 1ull)) & ~((1ull << a) - 1ull)) : 0ull;
    const uint32_t wlo = uint32_t(wm), whi = uint32_t(wm >> 32);
#pragma unroll
    for (int i = 0; i < 64; ++i)      // in place: sv now holds the masked scores
      if (!((i < 32 ? (wlo >> i) : (whi >> (i - 32))) & 1u)) sv[i >> 4][i & 15] = 0xff800000u;   // -inf
#define X_(i) __uint_as_float(sv[(i) >> 4][(i) & 15])
    float mx[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) mx[i] = fmaxf(fmaxf(X_(i), X_(i + 16)), fmaxf(X_(i + 32), X_(i + 48)));
#pragma unroll
    for (int w2 = 8; w2 >= 1; w2 >>= 1)
#pragma unroll
      for (int i = 0; i < w2; ++i) mx[i] = fmaxf(mx[i], mx[i + w2]);
    const float mq = te > ta ? mx[0] * qs : 0.f;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (p0 + g > p1) break;
      float e[16];
      uint32_t pk[8];
#if QA_EXP16
      // 2^x on f16x2 pairs: one MUFU op per two scores (x rounded to f16: |dx| <= 2^-11 |x|)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t hx;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hx) : "f"(fmaf(X_(16 * g + 2 * i + 1), qs, -mq)),
            "f"(fmaf(X_(16 * g + 2 * i), qs, -mq)));
        asm("ex2.approx.f16x2 %0, %0;" : "+r"(hx));
        asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tcvt.f32.f16 %0, lo;\n\tcvt.f32.f16 %1, hi;\n\t}"
            : "=f"(e[2 * i]), "=f"(e[2 * i + 1]) : "r"(hx));
        pk[i] = pack_bf16x2(e[2 * i], e[2 * i + 1]);
      }
#else
#pragma unroll
      for (int i = 0; i < 16; ++i) e[i] = ex2_approx(fmaf(X_(16 * g + i), qs, -mq));
#pragma unroll
      for (int i = 0; i < 8; ++i) pk[i] = pack_bf16x2(e[2 * i], e[2 * i + 1]);
#endif
      tmem_st8(sh + 8 * (p0 + g), pk);      // P piece over S columns already read
#pragma unroll
      for (int w2 = 8; w2 >= 1; w2 >>= 1)
#pragma unroll
        for (int i = 0; i < w2; ++i) e[i] += e[i + w2];
      l += e[0];
    }
#undef X_
  } else {
    // long windows (> 4 pieces): the max, then exp / P, each over batches of QA_LB pieces loaded together
    // (one TMEM load wait per batch; a batch past p1 re-reads piece p1, masked).  P of batch
    // [b0, b0 + QA_LB) lands on S pieces <= (b0 + QA_LB - 1) / 2 < b0 + QA_LB, i.e. on pieces already read.
    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int b0 = p0; b0 <= p1; b0 += QA_LB) {
      uint32_t sv[QA_LB][16];
#pragma unroll
      for (int g = 0; g < QA_LB; ++g) tmem_ld16(sh + 16 * min(b0 + g, p1), sv[g]);
      tmem_ld_wait();
#pragma unroll
      for (int g = 0; g < QA_LB; ++g)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          asm volatile("" : "+r"(sv[g][i]));
          const int key = 16 * (b0 + g) + i;
          const float v = (key >= ta && key < te) ? __uint_as_float(sv[g][i]) : -INFINITY;
          m4[i & 3] = fmaxf(m4[i & 3], v);
        }
    }
    const float m = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    const float mq = te > ta ? m * qs : 0.f;
    for (int b0 = p0; b0 <= p1; b0 += QA_LB) {
      uint32_t sv[QA_LB][16];
#pragma unroll
      for (int g = 0; g < QA_LB; ++g) tmem_ld16(sh + 16 * min(b0 + g, p1), sv[g]);
      tmem_ld_wait();
#pragma unroll
      for (int g = 0; g < QA_LB; ++g) {
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          asm volatile("" : "+r"(sv[g][2 * i]), "+r"(sv[g][2 * i + 1]));
          const int key = 16 * (b0 + g) + 2 * i;
          const float e0 = (key >= ta && key < te) ? ex2_approx(fmaf(__uint_as_float(sv[g][2 * i]), qs, -mq)) : 0.f;
          const float e1 = (key + 1 >= ta && key + 1 < te) ? ex2_approx(fmaf(__uint_as_float(sv[g][2 * i + 1]), qs, -mq)) : 0.f;
          l += e0 + e1;
          pk[i] = pack_bf16x2(e0, e1);
        }
        if (b0 + g <= p1) tmem_st8(sh + 8 * (b0 + g), pk);
      }
    }
  }
  {
    const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    for (int pc = 0; pc < BM / 16; ++pc)      // zero P outside the warp's pieces
      if (pc < p0 || pc > p1) tmem_st8(sh + 8 * pc, z);
  }
  tmem_st_wait();
  tc_fence_before();
  return l;
}

__global__ void __launch_bounds__(THREADS, 1)
    qkv_attn_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const float* __restrict__ bias, const int32_t* __restrict__ rec, int n_tiles, float qscale,
                       uint16_t* __restrict__ O) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);   // [STAGES]
  uint64_t* empty = full + STAGES;                      // [STAGES]
  uint64_t* bfull = empty + STAGES;
  uint64_t* tfull = bfull + 1;       // QKV(t) retired (commit)
  uint64_t* tempty = tfull + 1;      // accumulator read by the staging (12 warps)
  uint64_t* qk_ready = tempty + 1;   // Q in TMEM, K in smem, row windows in smem (4 warps: part 0)
  uint64_t* v_ready = qk_ready + 1;  // [2] V_h in smem (4 warps: part 1 + h)
  uint64_t* sfull = v_ready + 2;     // [2] S(t, h) retired (commit)
  uint64_t* pready = sfull + 2;      // [2] P(t, h) in TMEM (4 warps: part 1 + h)
  uint64_t* ofull = pready + 2;      // [2] PV(t, h) retired (commit)
  uint64_t* oempty = ofull + 2;      // [2] O(t, h) read from TMEM (4 warps: part 1 + h)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(oempty + 2);
  float* s_bias = reinterpret_cast<float*>(smem + 256);        // [192] the slice's bias
  uint16_t* wtab = reinterpret_cast<uint16_t*>(smem + 1024);   // [2 tiles][128 rows]: ta | te << 8
  uint8_t* sB = smem + OFF_B;
  uint8_t* sK = smem + OFF_K;
  uint8_t* sV = smem + OFF_V;
  uint8_t* sA = smem + OFF_A;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int n_slices = 3 * D / BN;
  const int slice = int(blockIdx.x) % n_slices;
  const int t0 = int(blockIdx.x) / n_slices, dt = int(gridDim.x) / n_slices;
  const int n0 = slice * BN;

  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023u) != 0) __trap();   // the swizzled tiles need a 1 KB-aligned base
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], QA_MC ? n_slices : 1);
    }
    mbar_init(bfull, 1);
    mbar_init(tfull, 1);
    mbar_init(tempty, EPI_WARPS);
    mbar_init(qk_ready, 4);
    for (int h = 0; h < 2; ++h) {
      mbar_init(&v_ready[h], 4);
      mbar_init(&sfull[h], 1);
      mbar_init(&pready[h], 4);
      mbar_init(&ofull[h], 1);
      mbar_init(&oempty[h], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
#if QA_MC
  cluster_sync();                      // the peers' barriers are initialised before any multicast
#endif
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 || warp == 2 || warp == 3) {
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producers
      const int p = warp == 0 ? 0 : warp - 1;
      if (p == 0 && t0 < n_tiles) {      // the weight slice, once (two 96-row boxes per k-block)
        mbar_arrive_expect_tx(bfull, uint32_t(B_KBLK) * KB1);
        const uint64_t pol = l2_policy_evict_last();
        for (int kb = 0; kb < KB1; ++kb)
          for (int j = 0; j < 2; ++j)
            tma_load_2d_hint(sB + kb * B_KBLK + j * 96 * 128, &tmB, bfull, kb * 64, n0 + j * 96, pol);
      }
      griddep_wait();                    // X and the tile records come from the previous kernels
      uint32_t c = 0;
      const bool feeds = !QA_MC || p == 0;   // QA_MC: producer 0 alone (one box in six is its own)
#ifndef QA_PREFETCH
#define QA_PREFETCH 2                    // tiles ahead whose X rows are prefetched into L2
#endif
      if (p == 0 && (!QA_MC || slice == 0))
        for (int k = 1; k <= QA_PREFETCH; ++k)
          if (t0 + k * dt < n_tiles) {
            const int mp = __ldg(rec + size_t(t0 + k * dt) * ATT_REC_INTS);
            for (int kb = 0; kb < KB1; ++kb) tma_prefetch_2d(&tmA, kb * 64, mp);
          }
      for (int t = t0; feeds && t < n_tiles; t += dt) {
        const int m0 = __ldg(rec + size_t(t) * ATT_REC_INTS);
        const bool pf_t = QA_PREFETCH > 0 && (!QA_MC || slice == 0) && t + (QA_PREFETCH + 1) * dt < n_tiles;
        const int m_pf = pf_t ? __ldg(rec + size_t(t + (QA_PREFETCH + 1) * dt) * ATT_REC_INTS) : 0;
        if (QA_PF_MODE == 0 && pf_t && p == 0)   // the X rows of a later tile -> L2 (HBM latency off the A ring)
          for (int kb = 0; kb < KB1; ++kb) tma_prefetch_2d(&tmA, kb * 64, m_pf);
        for (int kb = 0; kb < KB1; ++kb, ++c) {
          if (!QA_MC && int(c % 3) != p) continue;
          const int s = int(c % STAGES);
#ifdef QA_SPIN
          mbar_wait(&empty[s], ((c / STAGES) & 1) ^ 1);
#else
          mbar_wait_sleep(&empty[s], ((c / STAGES) & 1) ^ 1);
#endif
          TL(E_LD0 + kb, int(c / KB1));
          mbar_arrive_expect_tx(&full[s], A_STAGE);
#if QA_MC
          // every CTA expects the box on its own barrier; CTA kb % 6 loads it for all six (a peer's bytes
          // may land before this CTA's expect_tx: the phase cannot complete before its local arrival)
          if (kb % n_slices == slice)
            tma_load_2d_mc(sA + s * A_STAGE, &tmA, &full[s], kb * 64, m0, uint16_t((1u << n_slices) - 1u));
#else
          tma_load_2d(sA + s * A_STAGE, &tmA, &full[s], kb * 64, m0);
#endif
          if (QA_PF_MODE != 0 && pf_t && (QA_PF_MODE == 1 || kb == slice)) tma_prefetch_2d(&tmA, kb * 64, m_pf);
        }
      }
    }
  } else if (warp == 1) {
    griddep_launch_dependents();
    // -------------------------------------------------------------------- MMA issuer
    // Issue order (steady state, loop index j = tile j):
    //   PV(j-1, h0), PV(j-1, h1), S(j, h0), QKV(j+1)[kb 0, 1], S(j, h1), QKV(j+1)[kb 2 .. 5]
    // so the O drain of (j-1, h) and the softmax of (j, h) on the CUDA cores each run under tensor work.
    constexpr uint32_t id_qkv = umma_idesc_bf16(BM, BN);
    constexpr uint32_t id_s = umma_idesc_bf16(BM, BM);
    constexpr uint32_t id_pv = umma_idesc_bf16(BM, DH) | (1u << 16);   // B = V MN-major (as stored)
    const uint64_t a0 = umma_desc_sw128(smem_u32(sA));
    const uint64_t b0 = umma_desc_sw128(smem_u32(sB));
    const uint64_t kd = umma_desc_sw128(smem_u32(sK));
    const uint64_t vd = umma_desc_sw128(smem_u32(sV));
    mbar_wait(bfull, 0);
#ifdef QA_TL
    if (blockIdx.x == 0 && lane == 0) g_tl_t0 = clock64();
#endif
#ifdef QA_TRACE
    long long tw[8] = {};
    const long long t_start = clock64();
#endif
    uint32_t c = 0;                      // A stages consumed
    int it = -1;                         // tile index of the loop below (-1: prologue)
    auto pv = [&](int j, int h) {        // O(j, h) = P_h V_h
      if (!QA_HS) QW(&v_ready[h], j & 1, 0);   // QA_HS: V_h(j) is staged before S(j, h) may issue
      QW(&pready[h], j & 1, 1);
      TL(h ? E_PV1 : E_PV0, j);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BM / 16; ++k)
          mma_ts(tmem_base + T_S + 128 * h + 64, tmem_base + T_S + 128 * h + 8 * k,
                 vd + uint64_t((k * 16 * 128 + h * DH * 2) >> 4), id_pv, k);   // keys 16k.., dims of head h
        tc_commit(&ofull[h]);
      }
      __syncwarp();
    };
    constexpr bool dyn = QA_HS && QA_DYN;
    bool pv_done[2] = {true, true};      // dyn: P V(it, h) issued
    auto try_pv = [&]() {                // P V(it, h) of a head whose softmax is done
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (!pv_done[h] && mbar_test_warp(&pready[h], it & 1)) {
          pv(it, h);
          pv_done[h] = true;
        }
    };
    auto wait_dyn = [&](uint64_t* bar, uint32_t par) {
      while (!mbar_try_warp(bar, par, QA_DYN_HINT)) try_pv();
    };
    auto qkv = [&](int kb_lo, int kb_hi) {
      for (int kb = kb_lo; kb < kb_hi; ++kb, ++c) {
        const int s = int(c % STAGES);
        if (dyn) wait_dyn(&full[s], (c / STAGES) & 1);
        else QW(&full[s], (c / STAGES) & 1, 3);
        TL(E_KB0 + kb, it + 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad = a0 + uint64_t((s * A_STAGE) >> 4), bd = b0 + uint64_t((kb * B_KBLK) >> 4);
#pragma unroll
          for (int k = 0; k < 4; ++k) tc_mma_bf16(tmem_base + T_ACC, ad + uint64_t(k * 2), bd + uint64_t(k * 2), id_qkv, (kb | k) != 0);
#if QA_MC
          tc_commit_mc(&empty[s], uint16_t((1u << n_slices) - 1u));   // slot s released in all six CTAs
#else
          tc_commit(&empty[s]);
#endif
          if (kb == KB1 - 1) tc_commit(tfull);
        }
        __syncwarp();
      }
      TL(kb_hi == KB1 ? E_QHI : E_QLO, it + 1);
    };
    auto sq = [&](int j, int h) {        // S(j, h) = Q_h K_h^T
      if (dyn) wait_dyn(&v_ready[h], j & 1);
      else if (QA_HS) QW(&v_ready[h], j & 1, 5);     // Q_h, K_h, V_h of tile j staged, O(j-1, h) drained
      else if (j > 0) QW(&oempty[h], (j - 1) & 1, 5);   // O(j-1, h) read out of S_h's columns
      TL(h ? E_S1 : E_S0, j);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < DH / 16; ++k)
          mma_ts(tmem_base + T_S + 128 * h, tmem_base + T_Q + (DH / 2) * h + 8 * k,
                 kd + uint64_t((h * (DH / 16) + k) * 2), id_s, k);
        tc_commit(&sfull[h]);
      }
      __syncwarp();
    };
    if (t0 < n_tiles) qkv(0, KB1);
    it = 0;
    for (int t = t0; t < n_tiles; t += dt, ++it) {
      const bool next = t + dt < n_tiles;
      if (it > 0) {
        if (!pv_done[0]) pv(it - 1, 0);
        if (!pv_done[1]) pv(it - 1, 1);
      }
      pv_done[0] = pv_done[1] = false;     // P V(it, h) pending (dyn: issued by try_pv once ready)
      if (!QA_HS) QW(qk_ready, it & 1, 4);   // staging of tile it done (Q, K, row windows; accumulator read)
      sq(it, 0);
      if (next) {
        if (dyn) wait_dyn(tempty, it & 1);
        else QW(tempty, it & 1, 2);
        tc_fence_after();
        qkv(0, 2);
      }
      sq(it, 1);
      if (next) qkv(2, KB1);
    }
    if (it > 0) {
      if (!pv_done[0]) pv(it - 1, 0);
      if (!pv_done[1]) pv(it - 1, 1);
    }
#ifdef QA_TRACE
    if (lane == 0 && blockIdx.x < 2)
      printf("QA_MMA cta %d tiles %d cyc/tile %lld | v_ready %lld pready %lld tempty %lld full %lld qk_ready %lld oempty %lld\n",
             int(blockIdx.x), it, (clock64() - t_start) / (it ? it : 1), tw[0] / (it ? it : 1), tw[1] / (it ? it : 1),
             tw[2] / (it ? it : 1), tw[3] / (it ? it : 1), tw[4] / (it ? it : 1), tw[5] / (it ? it : 1));
#endif
  } else if (warp >= 4) {
    griddep_wait();                      // records; O may still be read by the previous kernel
    // ------------------------------------------------------------------ epilogue (warps 4..15)
    const int q = warp & 3, part = (warp - 4) >> 2;
    const int r = q * 32 + lane;                          // row (= key) within the tile
    const uint32_t tl = tmem_base + (uint32_t(q * 32) << 16);
    const float* bs = s_bias;
#ifdef QA_TRACE
    long long et[8] = {}, el = clock64();
#define ETR(i) do { const long long _c = clock64(); et[i] += _c - el; el = _c; } while (0)
#else
#define ETR(i) do {} while (0)
#endif
    int it = 0;
    for (int i = threadIdx.x - 128; i < BN; i += 32 * EPI_WARPS) s_bias[i] = __ldg(bias + n0 + i);
    asm volatile("bar.sync 1, %0;" ::"r"(32 * EPI_WARPS) : "memory");
#if QA_HS
    if (true) {
      // ---------------- head h = part: per tile t, the row window [ta, te) (from the record, before the
      // accumulator is ready), Q_h -> TMEM, K_h -> smem, O(t-1, h) drained, V_h -> smem, staged[h];
      // then the O(t-1, h) stores and the softmax of (t, h)
      const int h = part;
      const uint32_t sh = tl + T_S + 128 * h;
      float l_prev = 1.f;
      int row0_prev = 0, nrows_prev = 0;
      for (int t = t0; t < n_tiles; t += dt, ++it) {
        const int32_t* R = rec + size_t(t) * ATT_REC_INTS;
        const int row0 = __ldg(R), nrows = __ldg(R + 1), ntexts = __ldg(R + 2);
        const uint32_t tsw = uint32_t(__ldg(R + 4 + lane));   // start rows of texts 4 lane .. 4 lane + 3
        uint32_t m0w = 0u, m1w = 0u, m2w = 0u, m3w = 0u;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (4 * lane + b < ntexts) {
            const uint32_t st = (tsw >> (8 * b)) & 0xffu, bit = 1u << (st & 31);
            m0w |= (st >> 5) == 0 ? bit : 0u;
            m1w |= (st >> 5) == 1 ? bit : 0u;
            m2w |= (st >> 5) == 2 ? bit : 0u;
            m3w |= (st >> 5) == 3 ? bit : 0u;
          }
        m0w = __reduce_or_sync(0xffffffffu, m0w);
        m1w = __reduce_or_sync(0xffffffffu, m1w);
        m2w = __reduce_or_sync(0xffffffffu, m2w);
        m3w = __reduce_or_sync(0xffffffffu, m3w);
        const uint64_t lo64 = (uint64_t(m1w) << 32) | m0w, hi64 = (uint64_t(m3w) << 32) | m2w;
        int ta = 0, te = 0;
        if (r < nrows) {
          const uint64_t le_lo = r >= 64 ? lo64 : (lo64 & (~0ull >> (63 - r)));
          const uint64_t le_hi = r >= 64 ? (hi64 & (~0ull >> (63 - (r - 64)))) : 0ull;
          ta = le_hi ? 64 + 63 - __clzll(le_hi) : 63 - __clzll(le_lo);   // row 0 always starts a text
          const uint64_t gt_lo = r >= 63 ? 0ull : (lo64 & (~0ull << (r + 1)));
          const uint64_t gt_hi = r >= 127 ? 0ull : r >= 63 ? (hi64 & (~0ull << (r + 1 - 64))) : hi64;
          te = gt_lo ? __ffsll(gt_lo) - 1 : gt_hi ? 64 + __ffsll(gt_hi) - 1 : nrows;
          te = te < nrows ? te : nrows;
        }
        mbar_wait_sleep(tfull, it & 1);
        TL(E_STG, it);
        tc_fence_after();
        uint32_t a[32], pk[16];
        tmem_ld32(tl + T_ACC + h * DH, a);                  // Q_h
        tmem_ld_wait_regs(a);
        bias_pack32(a, bs + h * DH, pk);
        tmem_ld32(tl + T_ACC + HG * DH + h * DH, a);        // K_h
        tmem_st16(tl + T_Q + (DH / 2) * h, pk);            // S(t-1, h) has read Q(t-1) (sfull waited)
        tmem_ld_wait_regs(a);
        bias_pack32(a, bs + HG * DH + h * DH, pk);
        tmem_ld32(tl + T_ACC + 2 * HG * DH + h * DH, a);    // V_h
#pragma unroll
        for (int j = 0; j < 4; ++j)                         // K_h: S's K-major B operand
          *reinterpret_cast<uint4*>(sK + sw128_off(r, h * DH + 8 * j)) =
              make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        tmem_ld_wait_regs(a);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
        TL(E_TE, it);
        bias_pack32(a, bs + 2 * HG * DH + h * DH, pk);
        // O(t-1, h): P V retired -> its TMEM columns (and V_h(t-1) in smem) are free
        uint32_t o[32];
        if (it > 0) {
          mbar_wait(&ofull[h], (it - 1) & 1);
          tc_fence_after();
          tmem_ld32(sh + 64, o);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)                         // V_h (row = key; the MN-major B operand of P V)
          *reinterpret_cast<uint4*>(sV + sw128_off(r, h * DH + 8 * j)) =
              make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        if (it > 0) tmem_ld_wait_regs(o);
        fence_proxy_async_smem();                           // K, V (generic writes) -> the MMAs
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&v_ready[h]);           // staged(t, h)
        TL(E_QKR, it);
        if (it > 0 && r < nrows_prev) {
          TL(h ? E_OE1 : E_OE0, it - 1);
          const float il = __frcp_rn(l_prev);               // == 1.0f / l_prev (both correctly rounded)
          uint32_t ok[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            ok[i] = pack_bf16x2(__uint_as_float(o[2 * i]) * il, __uint_as_float(o[2 * i + 1]) * il);
          uint16_t* dst = O + size_t(row0_prev + r) * D + slice * (HG * DH) + h * DH;
#pragma unroll
          for (int i = 0; i < 2; ++i)                        // two 32-byte stores: whole L2 sectors
            st_global_v8(dst + 16 * i, ok[8 * i], ok[8 * i + 1], ok[8 * i + 2], ok[8 * i + 3], ok[8 * i + 4],
                         ok[8 * i + 5], ok[8 * i + 6], ok[8 * i + 7]);
        }
        const int lo = __reduce_min_sync(0xffffffffu, te > ta ? ta : BM);
        const int hi = __reduce_max_sync(0xffffffffu, te > ta ? te : 0);
        const int p0 = lo >> 4, p1 = hi > lo ? (hi - 1) >> 4 : -1;   // pieces [p0, p1]
        const float l = qa_softmax(sh, &sfull[h], it, h, ta, te, p0, p1, qscale);
        TL(h ? E_PR1 : E_PR0, it);
        __syncwarp();
        if (lane == 0) mbar_arrive(&pready[h]);
        l_prev = te > ta ? l : 1.f;
        row0_prev = row0;
        nrows_prev = nrows;
      }
      if (it > 0) {                                          // O of the last tile
        mbar_wait(&ofull[h], (it - 1) & 1);
        tc_fence_after();
        uint32_t o[32];
        tmem_ld32(sh + 64, o);
        tmem_ld_wait_regs(o);
        if (r < nrows_prev) {
          const float il = __frcp_rn(l_prev);
          uint32_t ok[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            ok[i] = pack_bf16x2(__uint_as_float(o[2 * i]) * il, __uint_as_float(o[2 * i + 1]) * il);
          uint16_t* dst = O + size_t(row0_prev + r) * D + slice * (HG * DH) + h * DH;
#pragma unroll
          for (int i = 0; i < 2; ++i)
            st_global_v8(dst + 16 * i, ok[8 * i], ok[8 * i + 1], ok[8 * i + 2], ok[8 * i + 3], ok[8 * i + 4],
                         ok[8 * i + 5], ok[8 * i + 6], ok[8 * i + 7]);
        }
      }
    } else
#endif
    if (part == 0) {
      // ---------------- part 0: Q -> TMEM (TS operand of S), K -> smem (row = key, [K_h0 | K_h1]) and the
      // text window [ta, te) of every row of the tile -> wtab
      for (int t = t0; t < n_tiles; t += dt, ++it) {
        const int32_t* R = rec + size_t(t) * ATT_REC_INTS;
        const int nrows = __ldg(R + 1), ntexts = __ldg(R + 2);
        const uint32_t tsw = uint32_t(__ldg(R + 4 + lane));   // start rows of texts 4 lane .. 4 lane + 3
        mbar_wait_sleep(tfull, it & 1);
        TL(E_STG, it);
        tc_fence_after();
        uint32_t a0[32], a1[32], pk[16];
        tmem_ld32(tl + T_ACC, a0);
        tmem_ld32(tl + T_ACC + DH, a1);
        tmem_ld_wait_regs(a0);
        tmem_ld_wait_regs(a1);
        bias_pack32(a0, bs, pk);
        tmem_st16(tl + T_Q, pk);
        bias_pack32(a1, bs + DH, pk);
        tmem_st16(tl + T_Q + DH / 2, pk);
        tmem_ld32(tl + T_ACC + HG * DH, a0);
        tmem_ld32(tl + T_ACC + HG * DH + DH, a1);
        tmem_ld_wait_regs(a0);
        tmem_ld_wait_regs(a1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
        TL(E_TE, it);
#pragma unroll
        for (int h = 0; h < HG; ++h) {
          bias_pack32(h ? a1 : a0, bs + HG * DH + h * DH, pk);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(sK + sw128_off(r, h * DH + 8 * j)) =
                make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
        // this row's text window [ta, te) from the tile's 128-bit start-of-text mask
        uint32_t m0w = 0u, m1w = 0u, m2w = 0u, m3w = 0u;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (4 * lane + b < ntexts) {
            const uint32_t st = (tsw >> (8 * b)) & 0xffu, bit = 1u << (st & 31);
            m0w |= (st >> 5) == 0 ? bit : 0u;
            m1w |= (st >> 5) == 1 ? bit : 0u;
            m2w |= (st >> 5) == 2 ? bit : 0u;
            m3w |= (st >> 5) == 3 ? bit : 0u;
          }
        m0w = __reduce_or_sync(0xffffffffu, m0w);
        m1w = __reduce_or_sync(0xffffffffu, m1w);
        m2w = __reduce_or_sync(0xffffffffu, m2w);
        m3w = __reduce_or_sync(0xffffffffu, m3w);
        const uint64_t lo64 = (uint64_t(m1w) << 32) | m0w, hi64 = (uint64_t(m3w) << 32) | m2w;
        int ta = 0, te = 0;
        if (r < nrows) {
          const uint64_t le_lo = r >= 64 ? lo64 : (lo64 & (~0ull >> (63 - r)));
          const uint64_t le_hi = r >= 64 ? (hi64 & (~0ull >> (63 - (r - 64)))) : 0ull;
          ta = le_hi ? 64 + 63 - __clzll(le_hi) : 63 - __clzll(le_lo);   // row 0 always starts a text
          const uint64_t gt_lo = r >= 63 ? 0ull : (lo64 & (~0ull << (r + 1)));
          const uint64_t gt_hi = r >= 127 ? 0ull : r >= 63 ? (hi64 & (~0ull << (r + 1 - 64))) : hi64;
          te = gt_lo ? __ffsll(gt_lo) - 1 : gt_hi ? 64 + __ffsll(gt_hi) - 1 : nrows;
          te = te < nrows ? te : nrows;
        }
        wtab[(it & 1) * BM + r] = uint16_t(ta | (te << 8));
        fence_proxy_async_smem();                         // K (generic writes) -> the S MMA
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(qk_ready);             // also releases wtab to the softmax warps
        TL(E_QKR, it);
        ETR(1);
      }
    } else {
      // ---------------- parts 1, 2: head h = part - 1: V_h of tile t -> smem, O of tile t-1, softmax of tile t
      const int h = part - 1;
      const uint32_t sh = tl + T_S + 128 * h;
      float l_prev = 1.f;
      int row0_prev = 0, nrows_prev = 0;
      auto drain = [&](int j) {          // O(j, h): TMEM -> / rowsum -> bf16 -> global (64 B of the row)
        mbar_wait(&ofull[h], j & 1);
        tc_fence_after();
        uint32_t o[32];
        tmem_ld32(sh + 64, o);
        tmem_ld_wait_regs(o);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&oempty[h]);
        TL(h ? E_OE1 : E_OE0, j);
        if (r < nrows_prev) {
          const float il = __frcp_rn(l_prev);             // == 1.0f / l_prev (both correctly rounded)
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            pk[i] = pack_bf16x2(__uint_as_float(o[2 * i]) * il, __uint_as_float(o[2 * i + 1]) * il);
          uint16_t* dst = O + size_t(row0_prev + r) * D + slice * (HG * DH) + h * DH;
#pragma unroll
          for (int i = 0; i < 2; ++i)       // two 32-byte stores: whole L2 sectors
#ifdef QA_NOSTORE   // timing experiment only
            if (pk[i] == 0x7fc07fc0u && row0_prev < 0)
#endif
            st_global_v8(dst + 16 * i, pk[8 * i], pk[8 * i + 1], pk[8 * i + 2], pk[8 * i + 3], pk[8 * i + 4],
                         pk[8 * i + 5], pk[8 * i + 6], pk[8 * i + 7]);
        }
      };
      for (int t = t0; t < n_tiles; t += dt, ++it) {
        const int32_t* R = rec + size_t(t) * ATT_REC_INTS;
        const int row0 = __ldg(R), nrows = __ldg(R + 1);
        uint32_t vv[16];
        {
          // V_h of tile t: + bias -> bf16 pairs (written to smem once PV(t-1, h) has read V_h(t-1))
          mbar_wait(tfull, it & 1);
          tc_fence_after();
          uint32_t a[32];
          tmem_ld32(tl + T_ACC + 2 * HG * DH + h * DH, a);
          tmem_ld_wait_regs(a);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty);
          bias_pack32(a, bs + 2 * HG * DH + h * DH, vv);
        }
        // wtab of tile it (part 0).  Checked before this warp releases S_h (oempty in the drain): the next
        // phase of qk_ready needs S(it, h), so it cannot complete before this wait has seen phase it.
        mbar_wait(qk_ready, it & 1);
        const uint32_t w = wtab[(it & 1) * BM + r];
        const int ta = int(w & 0xffu), te = int(w >> 8);
        if (it > 0) drain(it - 1);
        TL(h ? E_DR1 : E_DR0, it);
#pragma unroll
        for (int j = 0; j < 4; ++j)                       // V_h (row = key; the MN-major B operand of P V)
          *reinterpret_cast<uint4*>(sV + sw128_off(r, h * DH + 8 * j)) =
              make_uint4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&v_ready[h]);
        ETR(2);
        // softmax(t, h): the warp loads the 16-column pieces covering its rows' windows
        const int lo = __reduce_min_sync(0xffffffffu, te > ta ? ta : BM);
        const int hi = __reduce_max_sync(0xffffffffu, te > ta ? te : 0);
        const int p0 = lo >> 4, p1 = hi > lo ? (hi - 1) >> 4 : -1;   // pieces [p0, p1]
        ETR(3);
        const float l = qa_softmax(sh, &sfull[h], it, h, ta, te, p0, p1, qscale);
        ETR(4);
        __syncwarp();
        if (lane == 0) mbar_arrive(&pready[h]);
        TL(h ? E_PR1 : E_PR0, it);
        ETR(5);
        l_prev = te > ta ? l : 1.f;
        row0_prev = row0;
        nrows_prev = nrows;
      }
      if (it > 0) drain(it - 1);
    }
#ifdef QA_TRACE
    if (lane == 0 && blockIdx.x == 0 && q == 0)
      printf("QA_EPI part %d tiles %d | tfull %lld stage %lld ofull/drain %lld vt/rows %lld sfull %lld softmax %lld\n",
             part, it, et[0] / (it ? it : 1), et[1] / (it ? it : 1), et[2] / (it ? it : 1), et[3] / (it ? it : 1),
             et[4] / (it ? it : 1), et[5] / (it ? it : 1));
#endif
  }
  tc_fence_before();
  __syncthreads();
#if QA_MC
  cluster_sync();                      // no peer multicasts into / arrives on this CTA's smem any more
#endif
#ifdef QA_TL
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (g_tl_launch == 3)
      for (int j = 0; j < 4; ++j)
        for (int e = 0; e < E_N; ++e) printf("TL %8lld tile %d %s\n", g_tlbuf[j][e], 40 + j, g_tl_names[e]);
    ++g_tl_launch;
  }
#endif
  if (warp == 2) {
    __syncwarp();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace

bool qkv_attn_tc_supported(int d, int heads) { return d == D && d / heads == DH; }

cudaError_t launch_qkv_attn_tc(const GemmArgs& g, cudaStream_t st) {
  if (g.epi != EPI_QKV_ATTN || g.K != D || g.N != 3 * D || g.head_dim != DH || !g.att_rec || g.n_att_tiles <= 0)
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(qkv_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  constexpr int n_slices = 3 * D / BN;
  int groups = (sms > 0 ? sms : 148) / n_slices;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = size_t(SMEM);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
#if QA_MC
  at[na].id = cudaLaunchAttributeClusterDimension;
  at[na].val.clusterDim.x = n_slices;
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
  static int max_clusters = 0;         // clusters of six co-resident (GPC boundaries), queried once
  if (max_clusters == 0) {
    cfg.gridDim = dim3(unsigned(groups * n_slices));
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&max_clusters, qkv_attn_tc_kernel, &cfg);
    if (e != cudaSuccess || max_clusters <= 0) return e != cudaSuccess ? e : cudaErrorLaunchOutOfResources;
  }
  groups = std::min(groups, max_clusters);
#endif
  const int per = int(std::max<int64_t>(1, std::min<int64_t>(groups, g.n_att_tiles)));
  cfg.gridDim = dim3(unsigned(per * n_slices));
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, qkv_attn_tc_kernel, *g.tmA, *g.tmB, g.bias, g.att_rec, int(g.n_att_tiles), g.qscale,
                            g.C);
}

}  // namespace surge
