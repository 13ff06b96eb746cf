// attn_tile.cuh -- the per-(text, head, 16-row query tile) attention arithmetic shared by every
// kernel that runs K5 (reading R10: softmax(q k^T / sqrt(d_h)) v over the
// text's own tokens, block-diagonal, bidirectional):
//   * attention_text_kernel / attention_long_kernel (kernels.cu): QKV read from HBM;
//   * the QKV GEMM's attention epilogue (gemm_tc.cu, EPI_QKV_ATTN): QKV straight from TMEM.
// One code path means one rounding order: a text's attention output is bit-identical whichever
// kernel computes it (SuperBatch / chunk invariance).
//
// Layout: Q, K, V rows of the text in shared memory, row stride LDS bf16 elements (16-byte skew),
// the head's DH columns contiguous.  Query tiles and key blocks are 16 rows aligned to the text's
// first token; keys j >= len are masked to -inf before the online softmax (exp2 form,
// p = 2^(s qscale - m qscale) with qscale = log2(e) / sqrt(d_h) and m the running max of the raw
// scores; MUFU ex2.approx); P enters the PV product as bf16 (ATT_P_SPLIT = 1: as bf16 hi + lo parts,
// two MMAs).  Rows up to 16 * ceil(len / 16) are read, so the caller provides finite values (or
// zeros) there.
#pragma once

#include "common.cuh"

// 1: P enters P V as bf16 hi + lo parts (two MMAs, ~16 mantissa bits of P); 0: bf16 P (one MMA).
#ifndef ATT_P_SPLIT
#define ATT_P_SPLIT 0
#endif

namespace surge {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D (16x8 fp32) += A (16x16 bf16, row) * B (16x8 bf16, col)
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One step of the online softmax over NS consecutive 16-key sub-blocks (NS = 1 or 2) for NH heads
// (FIRST: the first step, where the running max is -inf, so the rescale factors are exactly 0 and
// are skipped -- the same values the general step gives).  Wider steps shorten the dependency chain
// of texts longer than 16 tokens (one max / exp / rescale round per 32 keys instead of per 16).
template <int DH, int LDS, int NH, int NS, bool FIRST>
__device__ __forceinline__ void attn_key_block(uint32_t k_addr, uint32_t v_addr, const uint32_t (&qa)[NH][DH / 16][4],
                                               int j0, int len, float qscale, float (&o)[NH][DH / 8][4],
                                               float (&ma)[NH], float (&mb)[NH], float (&la)[NH], float (&lb)[NH]) {
  constexpr uint32_t SB = 16 * LDS * 2;          // bytes between 16-row sub-blocks
  float s[NH][NS][2][4];
#pragma unroll
  for (int h = 0; h < NH; ++h)
#pragma unroll
    for (int sb = 0; sb < NS; ++sb) {
#pragma unroll
      for (int i = 0; i < 4; ++i) s[h][sb][0][i] = s[h][sb][1][i] = 0.f;
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
        uint32_t b00, b01, b10, b11;
        ldsm_x4(k_addr + sb * SB + h * DH * 2 + kk * 32, b00, b01, b10, b11);
        mma_bf16_16816(s[h][sb][0], qa[h][kk], b00, b01);
        mma_bf16_16816(s[h][sb][1], qa[h][kk], b10, b11);
      }
    }
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    // raw scores; the scale (log2(e) / sqrt(d_h) > 0) is applied inside the exponent:
    // p = 2^(s q - m q), m = running row max of the raw scores.  pa: row g, pb: row g + 8;
    // element 4 sb + 2 t + e = key j0 + 16 sb + 8 t + e.
    float pa[4 * NS], pb[4 * NS];
#pragma unroll
    for (int sb = 0; sb < NS; ++sb)
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool v = j0 + 16 * sb + 8 * t + e < len;
          pa[4 * sb + 2 * t + e] = v ? s[h][sb][t][e] : -INFINITY;
          pb[4 * sb + 2 * t + e] = v ? s[h][sb][t][2 + e] : -INFINITY;
        }
    float xa = pa[0], xb = pb[0];
#pragma unroll
    for (int i = 1; i < 4 * NS; ++i) {
      xa = fmaxf(xa, pa[i]);
      xb = fmaxf(xb, pb[i]);
    }
    xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 1));
    xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 2));
    xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 1));
    xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 2));
    const float na = FIRST ? xa : fmaxf(ma[h], xa), nb = FIRST ? xb : fmaxf(mb[h], xb);   // finite
    const float nqa = na * qscale, nqb = nb * qscale;
#pragma unroll
    for (int i = 0; i < 4 * NS; ++i) {
      pa[i] = ex2_approx(fmaf(pa[i], qscale, -nqa));   // masked: 2^-inf = 0
      pb[i] = ex2_approx(fmaf(pb[i], qscale, -nqb));
    }
    float sa = (pa[0] + pa[1]) + (pa[2] + pa[3]), sbb = (pb[0] + pb[1]) + (pb[2] + pb[3]);
    if (NS == 2) {
      sa += (pa[4] + pa[5]) + (pa[6] + pa[7]);
      sbb += (pb[4] + pb[5]) + (pb[6] + pb[7]);
    }
    if (FIRST) {
      la[h] = sa;
      lb[h] = sbb;
    } else {
      const float ca = ex2_approx(fmaf(ma[h], qscale, -nqa)), cb = ex2_approx(fmaf(mb[h], qscale, -nqb));
      la[h] = fmaf(la[h], ca, sa);
      lb[h] = fmaf(lb[h], cb, sbb);
#pragma unroll
      for (int n = 0; n < DH / 8; ++n) {
        o[h][n][0] *= ca; o[h][n][1] *= ca;
        o[h][n][2] *= cb; o[h][n][3] *= cb;
      }
    }
    ma[h] = na;
    mb[h] = nb;
#pragma unroll
    for (int sb = 0; sb < NS; ++sb) {
      const uint32_t pf[4] = {pack_bf16x2(pa[4 * sb], pa[4 * sb + 1]), pack_bf16x2(pb[4 * sb], pb[4 * sb + 1]),
                              pack_bf16x2(pa[4 * sb + 2], pa[4 * sb + 3]), pack_bf16x2(pb[4 * sb + 2], pb[4 * sb + 3])};
#if ATT_P_SPLIT
      // P = P_hi + P_lo, both bf16 (two MMAs): P V keeps ~16 mantissa bits of P
      const uint32_t pl[4] = {pack_bf16x2(pa[4 * sb] - bf16lo(pf[0]), pa[4 * sb + 1] - bf16hi(pf[0])),
                              pack_bf16x2(pb[4 * sb] - bf16lo(pf[1]), pb[4 * sb + 1] - bf16hi(pf[1])),
                              pack_bf16x2(pa[4 * sb + 2] - bf16lo(pf[2]), pa[4 * sb + 3] - bf16hi(pf[2])),
                              pack_bf16x2(pb[4 * sb + 2] - bf16lo(pf[3]), pb[4 * sb + 3] - bf16hi(pf[3]))};
#endif
#pragma unroll
      for (int n = 0; n < DH / 16; ++n) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(v_addr + sb * SB + h * DH * 2 + n * 32, b0, b1, b2, b3);
        if (FIRST && sb == 0) {   // o = 0 + P V: start the accumulators from zero inside the MMA
          o[h][2 * n][0] = o[h][2 * n][1] = o[h][2 * n][2] = o[h][2 * n][3] = 0.f;
          o[h][2 * n + 1][0] = o[h][2 * n + 1][1] = o[h][2 * n + 1][2] = o[h][2 * n + 1][3] = 0.f;
        }
        mma_bf16_16816(o[h][2 * n], pf, b0, b1);
        mma_bf16_16816(o[h][2 * n + 1], pf, b2, b3);
#if ATT_P_SPLIT
        mma_bf16_16816(o[h][2 * n], pl, b0, b1);
        mma_bf16_16816(o[h][2 * n + 1], pl, b2, b3);
#endif
      }
    }
  }
}

// One warp computes the 16 query rows [16 qt, 16 qt + 16) of one text for NH heads at once (the
// heads' arithmetic is independent and interleaved for instruction-level parallelism; each head's
// operation sequence is the single-head one, so results do not depend on NH):
//   sQt : the tile's first query row at head 0's columns; sK / sV : the text's first key row at
//   head 0's columns; head h is DH columns further right in each; len = text length,
//   nt = ceil(len / 16) key blocks; q_rows = query rows of the tile inside the text; sZ = a zero row
//   (same column base) read instead of the rows past the text, which may belong to the next text
//   whose O another warp is writing over its Q (their values would only reach discarded rows).
// Returns the unnormalised accumulators o[h] (mma C-fragment layout: row g = lane / 4 in
// o[h][n][0..1], row g + 8 in o[h][n][2..3], columns 8 n + 2 (lane % 4) + {0, 1}) and the
// reciprocal row sums ia[h] (row g), ib[h] (row g + 8): O = o * i.
template <int DH, int LDS, int NH>
__device__ __forceinline__ void attn_query_tile(const uint16_t* sQt, const uint16_t* sK, const uint16_t* sV,
                                                int len, int nt, float qscale, int lane, float (&o)[NH][DH / 8][4],
                                                float (&ia)[NH], float (&ib)[NH], int q_rows, const uint16_t* sZ) {
  const int c4 = lane & 3;
  uint32_t qa[NH][DH / 16][4];
  const int qr = (lane & 7) + ((lane >> 3) & 1) * 8;
  const uint32_t q_addr = smem_u32((qr < q_rows ? sQt + qr * LDS : sZ) + (lane >> 4) * 8);
#pragma unroll
  for (int h = 0; h < NH; ++h)
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk)
      ldsm_x4(q_addr + h * DH * 2 + kk * 32, qa[h][kk][0], qa[h][kk][1], qa[h][kk][2], qa[h][kk][3]);
  float ma[NH], mb[NH], la[NH], lb[NH];
  const uint32_t k_base = smem_u32(sK + ((lane & 7) + ((lane >> 4) & 1) * 8) * LDS + ((lane >> 3) & 1) * 8);
  const uint32_t v_base = smem_u32(sV + ((lane & 7) + ((lane >> 3) & 1) * 8) * LDS + (lane >> 4) * 8);
  // key index within the text of a thread's score element: 16 sub-block + 8 t + 2 c4 + e; valid iff < len.
  // Steps of 32 keys while more than 16 keys remain, a final step of 16 (reads stay within
  // 16 * ceil(len / 16) rows of the text, as with 16-key steps).
  if (nt >= 2) {
    attn_key_block<DH, LDS, NH, 2, true>(k_base, v_base, qa, 2 * c4, len, qscale, o, ma, mb, la, lb);
  } else {
    attn_key_block<DH, LDS, NH, 1, true>(k_base, v_base, qa, 2 * c4, len, qscale, o, ma, mb, la, lb);
  }
#pragma unroll 1
  for (int kb = 2; kb < nt; kb += 2) {
    const uint32_t off = uint32_t(kb * 16 * LDS * 2);
    if (kb + 1 < nt)
      attn_key_block<DH, LDS, NH, 2, false>(k_base + off, v_base + off, qa, 16 * kb + 2 * c4, len, qscale, o, ma, mb,
                                            la, lb);
    else
      attn_key_block<DH, LDS, NH, 1, false>(k_base + off, v_base + off, qa, 16 * kb + 2 * c4, len, qscale, o, ma, mb,
                                            la, lb);
  }
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    la[h] += __shfl_xor_sync(0xffffffffu, la[h], 1);
    la[h] += __shfl_xor_sync(0xffffffffu, la[h], 2);
    lb[h] += __shfl_xor_sync(0xffffffffu, lb[h], 1);
    lb[h] += __shfl_xor_sync(0xffffffffu, lb[h], 2);
    ia[h] = 1.0f / la[h];
    ib[h] = 1.0f / lb[h];
  }
}

// O = o * i, bf16, rows < len of the query tile written at sOt (tile row 0, head 0 columns; head h
// DH columns further right), row stride LDS_O.
template <int DH, int NH, typename RowStride>
__device__ __forceinline__ void attn_store_tile(uint16_t* sOt, RowStride lds_o, int qt, int len, int lane,
                                                const float (&o)[NH][DH / 8][4], const float (&ia)[NH],
                                                const float (&ib)[NH]) {
  const int g = lane >> 2, c4 = lane & 3;
  const int ra = 16 * qt + g, rb = ra + 8;     // rows within the text
  uint16_t* oa = sOt + g * lds_o + 2 * c4;
#pragma unroll
  for (int h = 0; h < NH; ++h)
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) {
      if (ra < len) *reinterpret_cast<uint32_t*>(oa + h * DH + n * 8) = pack_bf16x2(o[h][n][0] * ia[h], o[h][n][1] * ia[h]);
      if (rb < len)
        *reinterpret_cast<uint32_t*>(oa + 8 * lds_o + h * DH + n * 8) = pack_bf16x2(o[h][n][2] * ib[h], o[h][n][3] * ib[h]);
    }
}

}  // namespace surge
