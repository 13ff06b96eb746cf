// attn_long_tc.cu -- K5 for texts of 129..512 tokens at d_h = 64 (the bge classes' long-text workload,
// SURVEY.md §8(f) N1; reading R10: softmax(q k^T / sqrt(d_h)) v over the text's own tokens) with both
// products on the tcgen05 tensor cores.  One CTA per (text, head); the text's K and V rows of the head stay
// in shared memory (TMA boxes of 128 rows x 64 bf16 from the QKV buffer, 128-byte swizzle) while its
// 128-row query tiles go through:
//   S = Q K^T     tcgen05 M = 128, N = L (the text length rounded up to 64, <= 512: the whole row of S
//                 fits TMEM, so the softmax is exact in one pass -- no online rescaling), K = 64;
//   softmax       8 warps, two per TMEM lane quadrant, each over half of the row's columns (keys >= len
//                 masked); row max and row sum exchanged through shared memory; exp2 form with the row
//                 max, P (bf16) written over the columns of S already read (P_A at [0, L/4), P_B at
//                 [L/2, 3L/4));
//   O = P V       tcgen05 M = 128, N = 64, K = L, A = P read from TMEM, B = V as stored (MN-major);
//   O / rowsum -> bf16 -> global O (128 bytes per row), rows < len.
// TMEM: 512 columns, S in [0, L), O in [3L/4, 3L/4 + 64).  Layouts as in qkv_attn_tc.cu (checked by
// scripts/microbench/ts_attn_check.cu).  Same bf16 Q/K/V/P values and softmax formula as the mma.sync
// kernels (attn_tile.cuh); fp32 accumulation order differs (reading R21).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace surge {

namespace {

constexpr int DH = 64;
constexpr int BM = 128;
constexpr int THREADS = 320;          // warp 0 control (TMA + MMA), warp 1 TMEM, warps 2..9 softmax / O
constexpr int OFF_Q = 3072;           // after the barriers (< 256) and the max / sum exchange ([256, 2304))
// Two size classes, launched over the same text list (a CTA whose text is of the other class exits at
// once): texts of <= 256 tokens use 256 TMEM columns and 81 KB of shared memory, so two CTAs share an SM
// and hide each other's load / softmax latency; longer texts take the whole TMEM (one CTA per SM).
// 2^a, 2^b (a, b <= 0: scores minus the row max).  ATT_LONG_EXP16 (measured slower: C4 attention 1,743 -> 1,860 ms
// per 50K texts, off): one ex2.approx.f16x2 for the pair (half
// the MUFU operations; the arguments rounded to f16 move 2^x by <= 2^-11 ln2 relative near 0 -- below the
// bf16 rounding P gets anyway -- and results below 2^-24 flush to 0); otherwise two ex2.approx.f32.
#ifndef ATT_LONG_EXP16
#define ATT_LONG_EXP16 0
#endif
__device__ __forceinline__ void exp2_pair(float a, float b, float& ea, float& eb) {
#if ATT_LONG_EXP16
  uint32_t hx;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hx) : "f"(fmaxf(b, -24.f)), "f"(fmaxf(a, -24.f)));
  asm("ex2.approx.f16x2 %0, %0;" : "+r"(hx));
  asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tcvt.f32.f16 %0, lo;\n\tcvt.f32.f16 %1, hi;\n\t}"
      : "=f"(ea), "=f"(eb) : "r"(hx));
#else
  ea = ex2_approx(a);
  eb = ex2_approx(b);
#endif
}

template <int LMAX>
struct LongCfg {
  static constexpr int OFF_K = OFF_Q + 2 * BM * 128;   // two Q buffers (query tile qt: buffer qt % 2)
  static constexpr int OFF_V = OFF_K + LMAX * 128;
  static constexpr int SMEM = OFF_V + LMAX * 128;   // 99 / 163 KB
};
static_assert(OFF_Q >= 256 + 2 * 2 * BM * 4 && OFF_Q % 1024 == 0, "Q tiles after the max / sum exchange arrays");

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

template <int LMAX>
__global__ void __launch_bounds__(THREADS, LMAX <= 256 ? 2 : 1)
    attn_long_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const int32_t* __restrict__ cu,
                        const int32_t* __restrict__ d_long, int32_t tok0, int d, uint16_t* __restrict__ out,
                        float qscale) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* q_full = kv_full + 1;     // [2] per Q buffer
  uint64_t* q_empty = q_full + 2;     // [2] S(qt) retired: its Q buffer may be reloaded (commit)
  uint64_t* s_full = q_empty + 2;     // commit
  uint64_t* p_ready = s_full + 1;     // 8 softmax warps
  uint64_t* o_full = p_ready + 1;     // commit
  uint64_t* o_empty = o_full + 1;     // 4 warps (part 0) have read O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);
  float* xmax = reinterpret_cast<float*>(smem + 256);   // [2 parts][128 rows]
  float* xsum = xmax + 2 * BM;                          // [2 parts][128 rows]
  uint8_t* sQ = smem + OFF_Q;
  uint8_t* sK = smem + LongCfg<LMAX>::OFF_K;
  uint8_t* sV = smem + LongCfg<LMAX>::OFF_V;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int text = __ldg(d_long + blockIdx.x), head = int(blockIdx.y);
  const int ta = __ldg(cu + text) - tok0, len = __ldg(cu + text + 1) - __ldg(cu + text);
  const int L = (len + 63) & ~63;                       // <= 512 (the caller checks max_len)
  const int nq = (len + BM - 1) / BM;
  // texts <= 128 tokens: the mma.sync kernel (same arithmetic as the fused QKV + attention epilogue);
  // otherwise the other size class's text
  if (len <= BM || L > LMAX || (LMAX > 256 && L <= 256)) return;

  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023u) != 0) __trap();
    tma_prefetch_desc(&tmQKV);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_ready, 8);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, LMAX);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t O_COL = uint32_t(3 * L / 4);

  if (warp == 0) {
    // ------------------------------------------------------------------ control: TMA + MMA (one thread)
    if (lane == 0) {
      griddep_wait();
      const int nkv = (L + BM - 1) / BM;
      mbar_arrive_expect_tx(kv_full, uint32_t(2 * nkv * BM * 128));
      for (int j = 0; j < nkv; ++j) {
        tma_load_2d(sK + j * BM * 128, &tmQKV, kv_full, d + head * DH, ta + j * BM);
        tma_load_2d(sV + j * BM * 128, &tmQKV, kv_full, 2 * d + head * DH, ta + j * BM);
      }
      const uint64_t kd = umma_desc_sw128(smem_u32(sK)), vd = umma_desc_sw128(smem_u32(sV));
      const uint32_t id_pv = umma_idesc_bf16(BM, DH) | (1u << 16);   // B = V MN-major (as stored)
      auto load_q = [&](int qt) {                      // query tile qt -> Q buffer qt % 2
        if (qt >= 2) mbar_wait(&q_empty[qt & 1], ((qt - 2) >> 1) & 1);   // S(qt - 2) has read it
        mbar_arrive_expect_tx(&q_full[qt & 1], uint32_t(BM * 128));
        tma_load_2d(sQ + (qt & 1) * BM * 128, &tmQKV, &q_full[qt & 1], head * DH, ta + qt * BM);
      };
      load_q(0);
      for (int qt = 0; qt < nq; ++qt) {
        if (qt + 1 < nq) load_q(qt + 1);               // the next tile's Q loads under this tile's work
        const uint64_t qd = umma_desc_sw128(smem_u32(sQ + (qt & 1) * BM * 128));
        mbar_wait(&q_full[qt & 1], (qt >> 1) & 1);
        if (qt == 0) mbar_wait(kv_full, 0);
        if (qt > 0) mbar_wait(o_empty, (qt - 1) & 1);  // O(qt-1) read: S / P / O columns may be rewritten
        tc_fence_after();
        // S = Q K^T: N = L in blocks of <= 256 columns, K = 64 (4 steps)
        for (int n0 = 0; n0 < L; n0 += 256) {
          const int nn = L - n0 < 256 ? L - n0 : 256;
          const uint32_t id_s = umma_idesc_bf16(BM, uint32_t(nn));
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            tc_mma_bf16(tmem + uint32_t(n0), qd + uint64_t(k * 2), kd + uint64_t((n0 * 128) >> 4) + uint64_t(k * 2), id_s,
                        k);
        }
        tc_commit(s_full);
        tc_commit(&q_empty[qt & 1]);
        mbar_wait(p_ready, qt & 1);
        tc_fence_after();
        // O = P V: K = L keys in steps of 16; P_A (keys < L/2) at column 0, P_B at column L/2
        for (int k = 0; k < L / 16; ++k) {
          const int kk = k < L / 32 ? k : k - L / 32;
          const uint32_t pa = tmem + (k < L / 32 ? 0u : uint32_t(L / 2)) + uint32_t(8 * kk);
          mma_ts(tmem + O_COL, pa, vd + uint64_t((k * 16 * 128) >> 4), id_pv, k);
        }
        tc_commit(o_full);
      }
    }
  } else if (warp >= 2) {
    // ------------------------------------------------------------------ softmax + O (warps 2..9)
    const int q = warp & 3, hh = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const uint32_t tl = tmem + (uint32_t(q * 32) << 16);
    const int half = L / 2, c0 = hh * half;
    const float qs = qscale;
    for (int qt = 0; qt < nq; ++qt) {
      mbar_wait(s_full, qt & 1);
      tc_fence_after();
      constexpr int NB = LMAX <= 256 ? 1 : 4;         // (two CTAs per SM at LMAX 256: 96 registers)
      // the part's half row in batches of 32 NB columns (NB loads, one wait; loads clamped into the row,
      // columns past the half masked): the max, then P = 2^(s q - m q) (0 past the text), bf16, over S
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      for (int cb = 0; cb < half; cb += 32 * NB) {
        uint32_t sv[NB][32];
#pragma unroll
        for (int j = 0; j < NB; ++j) tmem_ld32(tl + uint32_t(min(c0 + cb + 32 * j, L - 32)), sv[j]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < NB; ++j)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            asm volatile("" : "+r"(sv[j][i]));
            const int c = cb + 32 * j + i;
            if (c < half && c0 + c < len) m4[i & 3] = fmaxf(m4[i & 3], __uint_as_float(sv[j][i]));
          }
      }
      float m = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      xmax[hh * BM + r] = m;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");   // the two warps of this quadrant
      m = fmaxf(m, xmax[(hh ^ 1) * BM + r]);
      const float mq = m * qs;                          // len >= 1: finite for every row of the tile
      float l = 0.f;
      for (int cb = 0; cb < half; cb += 32 * NB) {
        uint32_t sv[NB][32];
#pragma unroll
        for (int j = 0; j < NB; ++j) tmem_ld32(tl + uint32_t(min(c0 + cb + 32 * j, L - 32)), sv[j]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            asm volatile("" : "+r"(sv[j][2 * i]), "+r"(sv[j][2 * i + 1]));
            const int c = cb + 32 * j + 2 * i, key = c0 + c;
            float e0, e1;
            exp2_pair(fmaf(__uint_as_float(sv[j][2 * i]), qs, -mq), fmaf(__uint_as_float(sv[j][2 * i + 1]), qs, -mq), e0, e1);
            e0 = (c < half && key < len) ? e0 : 0.f;
            e1 = (c + 1 < half && key + 1 < len) ? e1 : 0.f;
            l += e0 + e1;
            pk[i] = pack_bf16x2(e0, e1);
          }
          // P of columns c0 + cb + 32 j.. lands on S columns c0 + (cb + 32 j) / 2.. (already read)
          if (cb + 32 * j < half) tmem_st16(tl + uint32_t(c0 + (cb + 32 * j) / 2), pk);
        }
      }
      xsum[hh * BM + r] = l;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
      if (hh == 0) {
        const float il = __frcp_rn(l + xsum[BM + r]);
        mbar_wait(o_full, qt & 1);
        tc_fence_after();
        uint32_t o[32], o2[32];
        tmem_ld32(tl + O_COL, o);
        tmem_ld32(tl + O_COL + 32, o2);
        tmem_ld_wait_regs(o);
        tmem_ld_wait_regs(o2);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_empty);
        const int row = qt * BM + r;
        if (row < len) {
          uint16_t* dst = out + size_t(ta + row) * d + head * DH;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const uint32_t (&src)[32] = h2 ? o2 : o;
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              pk[i] = pack_bf16x2(__uint_as_float(src[2 * i]) * il, __uint_as_float(src[2 * i + 1]) * il);
#pragma unroll
            for (int i = 0; i < 2; ++i)
              asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 32 * h2 + 16 * i),
                           "r"(pk[8 * i]), "r"(pk[8 * i + 1]), "r"(pk[8 * i + 2]), "r"(pk[8 * i + 3]),
                           "r"(pk[8 * i + 4]), "r"(pk[8 * i + 5]), "r"(pk[8 * i + 6]), "r"(pk[8 * i + 7])
                           : "memory");
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem, LMAX);
  }
}

// Texts of 129..256 tokens: a persistent CTA per SM works through its (text, head) items as a pipeline of
// elements e = (item, 128-row query tile), two in flight: TMEM regions of 256 columns alternate by e % 2
// (S / P / O of element e), the K/V tiles of consecutive items alternate between two shared-memory buffers
// (the next item's K/V load under the current item's work), and the single MMA thread issues S(e + 1)
// before it waits for the softmax of e to issue PV(e) -- so the softmax of one element runs under the
// tensor work (and loads) of its neighbours instead of in series with them.
constexpr int PIPE_OFF_Q = 5120;   // [2 buffers] Q tile of an element, after the max / sum exchange ([256, 4352))
constexpr int PIPE_OFF_KV = PIPE_OFF_Q + 2 * BM * 128;             // [2 buffers][K 256 rows | V 256 rows]
constexpr int PIPE_KV = 2 * 256 * 128;                             // 64 KB per buffer
constexpr int PIPE_SMEM = PIPE_OFF_KV + 2 * PIPE_KV;              // 165 KB
static_assert(PIPE_OFF_Q >= 256 + 2 * 4 * BM * 4 && PIPE_OFF_Q % 1024 == 0, "Q tiles after the exchange arrays");

__global__ void __launch_bounds__(THREADS, 1)
    attn_long_pipe_kernel(const __grid_constant__ CUtensorMap tmQKV, const int32_t* __restrict__ cu,
                          const int32_t* __restrict__ d_long, int32_t n_items, int heads, int32_t tok0, int d,
                          uint16_t* __restrict__ out, float qscale) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(smem);   // [2] per KV buffer
  uint64_t* kv_free = kv_full + 2;     // [2] commit after the item's last PV
  uint64_t* q_full = kv_free + 2;      // [2] per Q buffer (element e: buffer e % 2)
  uint64_t* q_empty = q_full + 2;      // [2] commit after S(e)
  uint64_t* s_full = q_empty + 2;      // [2] per TMEM region
  uint64_t* p_ready = s_full + 2;      // [2] 8 warps
  uint64_t* o_full = p_ready + 2;      // [2] commit
  uint64_t* o_empty = o_full + 2;      // [2] 4 warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);
  float* xmax = reinterpret_cast<float*>(smem + 256);   // [2 regions][2 parts][128]
  float* xsum = xmax + 4 * BM;                          // [2 regions][2 parts][128]
  uint8_t* sQ = smem + PIPE_OFF_Q;
  uint8_t* sKV = smem + PIPE_OFF_KV;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // item i (of this CTA's list): global item blockIdx.x + i gridDim.x, text d_long[g / heads], head g % heads;
  // only texts of 129..256 tokens are this kernel's
  auto item_of = [&](int g, int& ta, int& len, int& head) -> bool {
    const int text = __ldg(d_long + g / heads);
    head = g % heads;
    ta = __ldg(cu + text) - tok0;
    len = __ldg(cu + text + 1) - __ldg(cu + text);
    return len > BM && len <= 256;
  };
  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023u) != 0) __trap();
    tma_prefetch_desc(&tmQKV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_free[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_ready[i], 8);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      griddep_wait();
      const uint32_t id_pv = umma_idesc_bf16(BM, DH) | (1u << 16);

      // the CTA's valid items, walked twice in step: `ld` = next item whose K/V to load, `e` elements
      int g_ld = int(blockIdx.x), n_ld = 0;            // loads issued (items)
      auto load_next = [&]() -> bool {                 // K/V of the next valid item into buffer n_ld % 2
        int ta, len, head;
        for (; g_ld < n_items; g_ld += int(gridDim.x)) {
          if (!item_of(g_ld, ta, len, head)) continue;
          const int b = n_ld & 1;
          if (n_ld >= 2) mbar_wait(&kv_free[b], ((n_ld - 2) >> 1) & 1);   // item n_ld - 2's last PV retired
          uint8_t* kv = sKV + b * PIPE_KV;
          mbar_arrive_expect_tx(&kv_full[b], uint32_t(2 * 2 * BM * 128));
          for (int j = 0; j < 2; ++j) {
            tma_load_2d(kv + j * BM * 128, &tmQKV, &kv_full[b], d + head * DH, ta + j * BM);
            tma_load_2d(kv + 256 * 128 + j * BM * 128, &tmQKV, &kv_full[b], 2 * d + head * DH, ta + j * BM);
          }
          g_ld += int(gridDim.x);
          ++n_ld;
          return true;
        }
        return false;
      };
      load_next();
      load_next();
      // element e = (item n_it, query tile qt); S(e) issued one element ahead of PV(e)
      int g_it = int(blockIdx.x), n_it = -1, ta = 0, len = 0, head = 0, qt = 1, e = 0;
      auto next_elem = [&]() -> bool {                 // advance (n_it, qt) to the next element
        if (n_it >= 0 && qt + 1 < 2) {
          ++qt;
          return true;
        }
        for (; g_it < n_items; g_it += int(gridDim.x))
          if (item_of(g_it, ta, len, head)) {
            g_it += int(gridDim.x);
            ++n_it;
            qt = 0;
            return true;
          }
        return false;
      };
      struct El { int n_it, ta, len, head, qt; };
      auto load_q = [&](int ee, const El& x) {        // Q tile of element ee -> Q buffer ee % 2
        const int b = ee & 1;
        if (ee >= 2) mbar_wait(&q_empty[b], ((ee - 2) >> 1) & 1);   // S(ee - 2) has read the buffer
        mbar_arrive_expect_tx(&q_full[b], uint32_t(BM * 128));
        tma_load_2d(sQ + b * BM * 128, &tmQKV, &q_full[b], x.head * DH, x.ta + x.qt * BM);
      };
      auto issue_s = [&](int ee, const El& x) {       // S(ee) = Q K^T into TMEM region ee % 2
        const int rg = ee & 1;
        const uint64_t qd = umma_desc_sw128(smem_u32(sQ + (ee & 1) * BM * 128));
        mbar_wait(&q_full[ee & 1], (ee >> 1) & 1);
        if (x.qt == 0) mbar_wait(&kv_full[x.n_it & 1], (x.n_it >> 1) & 1);
        if (ee >= 2) mbar_wait(&o_empty[rg], ((ee - 2) >> 1) & 1);   // region's previous element drained
        tc_fence_after();
        const int L = (x.len + 63) & ~63;
        const uint64_t kd = umma_desc_sw128(smem_u32(sKV + (x.n_it & 1) * PIPE_KV));
#pragma unroll
        for (int k = 0; k < DH / 16; ++k)
          tc_mma_bf16(tmem + uint32_t(256 * rg), qd + uint64_t(k * 2), kd + uint64_t(k * 2), umma_idesc_bf16(BM, uint32_t(L)),
                      k);
        tc_commit(&s_full[rg]);
        tc_commit(&q_empty[ee & 1]);
      };
      auto issue_pv = [&](int ee, const El& x) {
        const int rg = ee & 1;
        mbar_wait(&p_ready[rg], (ee >> 1) & 1);
        tc_fence_after();
        const int L = (x.len + 63) & ~63;
        const uint64_t vd = umma_desc_sw128(smem_u32(sKV + (x.n_it & 1) * PIPE_KV + 256 * 128));
        const uint32_t base = tmem + uint32_t(256 * rg);
        for (int k = 0; k < L / 16; ++k) {
          const int kk = k < L / 32 ? k : k - L / 32;
          const uint32_t pa = base + (k < L / 32 ? 0u : uint32_t(L / 2)) + uint32_t(8 * kk);
          mma_ts(base + uint32_t(3 * L / 4), pa, vd + uint64_t((k * 16 * 128) >> 4), id_pv, k);
        }
        tc_commit(&o_full[rg]);
        if (x.qt == 1) {                               // the item's last query tile: its K/V buffer is free
          tc_commit(&kv_free[x.n_it & 1]);
          load_next();
        }
      };
      // iteration e: Q of element e + 2 loads (its buffer freed by S(e)), S(e + 1) issues, then P V(e) once
      // the softmax of e is done -- the Q load latency stays off the issue chain
      El cur{}, nxt{}, nxt2{};
      bool have = next_elem();
      if (have) {
        cur = El{n_it, ta, len, head, qt};
        load_q(0, cur);
      }
      bool more = have && next_elem();
      if (more) {
        nxt = El{n_it, ta, len, head, qt};
        load_q(1, nxt);
      }
      if (have) issue_s(0, cur);
      for (e = 0; have; ++e) {
        const bool more2 = more && next_elem();
        if (more2) {
          nxt2 = El{n_it, ta, len, head, qt};
          load_q(e + 2, nxt2);
        }
        if (more) issue_s(e + 1, nxt);
        issue_pv(e, cur);
        cur = nxt;
        nxt = nxt2;
        have = more;
        more = more2;
      }
    }
  } else if (warp >= 2) {
    // ------------------------------------------------------------------ softmax + O (warps 2..9)
    const int q = warp & 3, hh = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const float qs = qscale;
    int e = 0;
    for (int g = int(blockIdx.x); g < n_items; g += int(gridDim.x)) {
      int ta, len, head;
      if (!item_of(g, ta, len, head)) continue;
      const int L = (len + 63) & ~63, half = L / 2, c0 = hh * half;
      for (int qt = 0; qt < 2; ++qt, ++e) {
        const int rg = e & 1;
        const uint32_t tl = tmem + uint32_t(256 * rg) + (uint32_t(q * 32) << 16);
        float* xm = xmax + rg * 2 * BM;
        float* xs = xsum + rg * 2 * BM;
        mbar_wait(&s_full[rg], (e >> 1) & 1);
        tc_fence_after();
        // the warp's half row (96 or 128 columns) in two batches of 64 (two loads, one wait each; the
        // 32 columns past a 96-column half are read and masked, their P not stored): the max, then P
        constexpr int NB = 2;
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int cb = 0; cb < 128; cb += 32 * NB) {
          uint32_t sv[NB][32];
#pragma unroll
          for (int j = 0; j < NB; ++j) tmem_ld32(tl + uint32_t(c0 + cb + 32 * j), sv[j]);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < NB; ++j)
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              asm volatile("" : "+r"(sv[j][i]));
              const int c = cb + 32 * j + i;
              if (c < half && c0 + c < len) m4[i & 3] = fmaxf(m4[i & 3], __uint_as_float(sv[j][i]));
            }
        }
        float m = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        xm[hh * BM + r] = m;
        asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
        m = fmaxf(m, xm[(hh ^ 1) * BM + r]);
        const float mq = m * qs;
        float l = 0.f;
#pragma unroll
        for (int cb = 0; cb < 128; cb += 32 * NB) {
          uint32_t sv[NB][32];
#pragma unroll
          for (int j = 0; j < NB; ++j) tmem_ld32(tl + uint32_t(c0 + cb + 32 * j), sv[j]);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              asm volatile("" : "+r"(sv[j][2 * i]), "+r"(sv[j][2 * i + 1]));
              const int c = cb + 32 * j + 2 * i, key = c0 + c;
              float e0, e1;
              exp2_pair(fmaf(__uint_as_float(sv[j][2 * i]), qs, -mq), fmaf(__uint_as_float(sv[j][2 * i + 1]), qs, -mq), e0,
                        e1);
              e0 = (c < half && key < len) ? e0 : 0.f;
              e1 = (c + 1 < half && key + 1 < len) ? e1 : 0.f;
              l += e0 + e1;
              pk[i] = pack_bf16x2(e0, e1);
            }
            // P over S columns this warp has already read (c0 + (cb + 32 j) / 2 < c0 + cb + 64)
            if (cb + 32 * j < half) tmem_st16(tl + uint32_t(c0 + (cb + 32 * j) / 2), pk);
          }
        }
        xs[hh * BM + r] = l;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_ready[rg]);
        asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
        if (hh == 0) {
          const float il = __frcp_rn(l + xs[BM + r]);
          mbar_wait(&o_full[rg], (e >> 1) & 1);
          tc_fence_after();
          uint32_t o[32], o2[32];
          tmem_ld32(tl + uint32_t(3 * L / 4), o);
          tmem_ld32(tl + uint32_t(3 * L / 4 + 32), o2);
          tmem_ld_wait_regs(o);
          tmem_ld_wait_regs(o2);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&o_empty[rg]);
          const int row = qt * BM + r;
          if (row < len) {
            uint16_t* dst = out + size_t(ta + row) * d + head * DH;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const uint32_t (&src)[32] = h2 ? o2 : o;
              uint32_t pk[16];
#pragma unroll
              for (int i = 0; i < 16; ++i)
                pk[i] = pack_bf16x2(__uint_as_float(src[2 * i]) * il, __uint_as_float(src[2 * i + 1]) * il);
#pragma unroll
              for (int i = 0; i < 2; ++i)
                asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 32 * h2 + 16 * i),
                             "r"(pk[8 * i]), "r"(pk[8 * i + 1]), "r"(pk[8 * i + 2]), "r"(pk[8 * i + 3]),
                             "r"(pk[8 * i + 4]), "r"(pk[8 * i + 5]), "r"(pk[8 * i + 6]), "r"(pk[8 * i + 7])
                             : "memory");
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool attn_long_tc_supported(int head_dim) { return head_dim == DH; }

// Off by default: one (text, head) per CTA with its loads, both MMAs, the softmax and the stores in series
// measured slower than the mma.sync kernel on the C4 workload (bge-large long texts: attention 3.20 s vs
// 2.71 s per 100K texts); SURGE_ATT_LONG_TC=1 selects it.
bool attn_long_tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("SURGE_ATT_LONG_TC");
    return e && e[0] == '1';
  }();
  return on;
}

cudaError_t launch_attn_long_tc(const uint16_t* qkv, const int32_t* cu, const int32_t* d_long, int32_t n_long,
                                int32_t tok0, int32_t ntok, int heads, uint16_t* out, cudaStream_t st) {
  if (n_long <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_long_tc_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         LongCfg<256>::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_long_tc_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, LongCfg<512>::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_long_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PIPE_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int d = heads * DH;
  CUtensorMap tm;
  cudaError_t e = make_tmap_bf16(&tm, qkv, uint64_t(ntok), uint64_t(3 * d), BM);
  if (e != cudaSuccess) return e;
  const float qscale = 1.4426950408889634f / sqrtf(float(DH));
#ifndef ATT_LONG_PIPE
#define ATT_LONG_PIPE 1
#endif
  if (ATT_LONG_PIPE) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = int64_t(n_long) * heads;
    attn_long_pipe_kernel<<<unsigned(std::min<int64_t>(items, sms > 0 ? sms : 148)), THREADS, PIPE_SMEM, st>>>(
        tm, cu, d_long, int32_t(items), heads, tok0, d, out, qscale);
  } else {
    attn_long_tc_kernel<256><<<dim3(unsigned(n_long), unsigned(heads)), THREADS, LongCfg<256>::SMEM, st>>>(
        tm, cu, d_long, tok0, d, out, qscale);
  }
  attn_long_tc_kernel<512><<<dim3(unsigned(n_long), unsigned(heads)), THREADS, LongCfg<512>::SMEM, st>>>(
      tm, cu, d_long, tok0, d, out, qscale);
  return cudaGetLastError();
}

}  // namespace surge
