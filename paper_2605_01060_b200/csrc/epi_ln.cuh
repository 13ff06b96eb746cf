// epi_ln.cuh -- the residual + LayerNorm GEMM epilogue (K6 / K8; reading R9:
// post-LN, biased variance, fp32 statistics), shared by the LN GEMM (gemm_tc.cu) and the fused MLP
// (mlp_tc.cu) so both round identically.
//
// The accumulator row (BN fp32 columns in TMEM, lane = row) is split over NP warps of the same lane
// quadrant q (hh = the warp's part), interleaved in 32-column steps: step k of part hh covers columns
// [32 (NP k + hh), +32), so after step k of every part the 32 NP columns [32 NP k, 32 NP (k + 1)) are done
// (the fused tail lets its next MMAs chase the LN0 output k-block by k-block).
//   pass 1: v = acc + bias + residual, written back to TMEM in place, shifted partial sums (the
//           residual slice and TMEM load of step k+1 are in flight while step k is computed; the
//           first residual slice is fetched before the accumulator is ready);
//   combine the halves (Chan's parallel variance) through smem (stats: [2 halves][128 rows]);
//   pass 2: y = (v - mean) rstd gamma + beta -> bf16, handed to store(p, column) 32 columns at a time.
#pragma once

#include "common.cuh"

namespace surge {

// Residual source: load(col, rr) fills rr[16] = the 32 bf16 residual values of columns col .. col + 31,
// packed in pairs.  It is called one step ahead of use.
struct ResidualGlobal {
  const uint16_t* rrow;   // this row, column 0
  __device__ __forceinline__ void operator()(int col, uint32_t (&rr)[16]) const {
    const uint4* p = reinterpret_cast<const uint4*>(rrow + col);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 v = p[i];
      rr[4 * i] = v.x; rr[4 * i + 1] = v.y; rr[4 * i + 2] = v.z; rr[4 * i + 3] = v.w;
    }
  }
};

#ifdef LN_TRACE
__device__ long long g_ln_trace[32][4];
#define LNT(i) do { const long long _c = clock64(); if (i > 0 && blockIdx.x == 0 && (threadIdx.x & 31) == 0) g_ln_trace[threadIdx.x >> 5][i - 1] += _c - _lt; _lt = _c; } while (0)
#else
#define LNT(i) do {} while (0)
#endif

// Coalesced store of a warp's 32 rows x 32 bf16 columns (lane = row, p = its 64 bytes): transposed
// through a 2 KB per-warp smem buffer (64-byte rows, 16-byte chunks XOR-swizzled by (row / 2) % 4,
// conflict-free both ways), then each store instruction writes 8 whole 64-byte row segments.
// Plain st.global: no wait on the TMA unit (whose queue is shared with the producers' loads).
__device__ __forceinline__ void store_rows_32x32(uint8_t* stg, const uint32_t (&p)[16], int lane, uint16_t* out,
                                                 int64_t row0, int64_t rows, int ld, int col) {
  __syncwarp();   // previous use of stg drained
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<uint4*>(stg + lane * 64 + ((i ^ ((lane >> 1) & 3)) << 4)) =
        make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
  __syncwarp();
  const int c = lane & 3;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int r = 8 * t + (lane >> 2);
    const uint4 v = *reinterpret_cast<const uint4*>(stg + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
    if (row0 + r < rows) *reinterpret_cast<uint4*>(out + size_t(row0 + r) * ld + col + 8 * c) = v;
  }
}

// The same 32 rows x 32 columns stored straight from registers: each lane writes its row's 64 bytes as
// two 32-byte stores (STG.256, whole L2 sectors) -- no shared-memory transpose.
__device__ __forceinline__ void store_row_64B(const uint32_t (&p)[16], int lane, uint16_t* out, int64_t row0,
                                              int64_t rows, int ld, int col) {
  if (row0 + lane < rows) {
    uint16_t* dst = out + size_t(row0 + lane) * ld + col;
#pragma unroll
    for (int i = 0; i < 2; ++i)
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 16 * i), "r"(p[8 * i]),
                   "r"(p[8 * i + 1]), "r"(p[8 * i + 2]), "r"(p[8 * i + 3]), "r"(p[8 * i + 4]), "r"(p[8 * i + 5]),
                   "r"(p[8 * i + 6]), "r"(p[8 * i + 7])
                   : "memory");
  }
}

// NP warps share a lane quadrant, each owning HALF = BN / NP columns (part hh).  PIPE: TMEM loads and
// residual loads one step ahead (2 register buffers); !PIPE: one buffer (for register-limited kernels).
struct LnNoOp {
  __device__ __forceinline__ void operator()() const {}
};
// Row statistics merge over the parts of one CTA (default) -- or, for a row split over a cluster of CTAs,
// a publisher that also writes this part's (shift, S1, S2) into the peer CTAs' stats array and waits for
// theirs (ln_pair.cu): part_off = index of this CTA's first part, NPM = parts in the merge.
struct LnLocalMerge {
  static constexpr int NPM = 0;   // 0: the CTA's own NP parts
  __device__ __forceinline__ int part_off() const { return 0; }
  __device__ __forceinline__ void publish(int, int, float4) const {}
  __device__ __forceinline__ void wait() const {}
};

// pass1_done() runs once the residual has been read for the last time (after pass 1).
// REMAP_LO > 0: accumulator columns [0, REMAP_LO) live at TMEM column REMAP_BASE + c instead of c (the fused
// tail's split out-projection, mlp_tc.cu MLP_G0SPLIT).
// CT = float: bias / gamma / beta as fp32 in shared memory; CT = uint16_t: as bf16 (the weight blob's own
// precision, so the same values), half the shared-memory loads (the LN passes are MIO-bound).
template <int BN, int HALF, bool PIPE = true, uint32_t REMAP_LO = 0, uint32_t REMAP_BASE = 0, typename CT = float,
          typename Merge = LnLocalMerge, typename Res, typename Ready, typename Store, typename P1 = LnNoOp,
          int NP = BN / HALF>
__device__ __forceinline__ void ln_epilogue(uint32_t taddr, int c_lo, const Res& load_res, const CT* s_bias,
                                            const CT* s_gamma, const CT* s_beta, float4* stats, int q, int hh,
                                            int lane, float eps, Ready&& wait_ready, Store&& store,
                                            P1&& pass1_done = P1{}, const Merge& merge = Merge{}) {
  constexpr int NPM = Merge::NPM > 0 ? Merge::NPM : NP;   // parts in the statistics merge
#ifdef LN_TRACE
  long long _lt = 0;
#endif
  constexpr int NSTEP = HALF / 32;
  constexpr int NB = PIPE ? 2 : 1;
  auto tcol = [](int c) { return uint32_t(c) < REMAP_LO ? REMAP_BASE + uint32_t(c) : uint32_t(c); };
  uint32_t r[NB][32];
  uint32_t rs[NB][16];
  (void)c_lo;
  auto lncol = [&](int k) { return 32 * (NP * k + hh); };   // columns of step k
  load_res(lncol(0), rs[0]);
  wait_ready();
  LNT(0);
  tmem_ld32(taddr + tcol(lncol(0)), r[0]);
  float shift = 0.f;
  f32x2 s1 = f2(0.f, 0.f), s2 = f2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < NSTEP; ++k) {
    const int cur = PIPE ? (k & 1) : 0;
    const int c = lncol(k);
    if (!PIPE && k > 0) {
      tmem_ld32(taddr + tcol(c), r[0]);
      load_res(c, rs[0]);
    }
    tmem_ld_wait_regs(r[cur]);
    if (PIPE && k + 1 < NSTEP) {
      tmem_ld32(taddr + tcol(lncol(k + 1)), r[cur ^ 1]);
      load_res(lncol(k + 1), rs[cur ^ 1]);
    }
    const uint32_t (&rr)[16] = rs[cur];
    uint4 cb[4];                                        // CT = bf16: this step's 32 bias values
    if constexpr (sizeof(CT) == 2) {
#pragma unroll
      for (int j = 0; j < 4; ++j) cb[j] = reinterpret_cast<const uint4*>(s_bias + c)[j];
    }
    auto bias2 = [&](int i) -> float2 {                 // bias of columns c + 2i, c + 2i + 1
      if constexpr (sizeof(CT) == 2) {
        const uint32_t u = (&cb[i >> 2].x)[i & 3];
        return make_float2(bf16lo(u), bf16hi(u));
      } else {
        return *reinterpret_cast<const float2*>(s_bias + c + 2 * i);
      }
    };
    if (k == 0) shift = __uint_as_float(r[cur][0]) + bias2(0).x + bf16lo(rr[0]);
    uint32_t w[32];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 bb = bias2(i);
      const f32x2 v = fadd2(fadd2(f2(__uint_as_float(r[cur][2 * i]), __uint_as_float(r[cur][2 * i + 1])),
                                  f2(bb.x, bb.y)),
                            f2(bf16lo(rr[i]), bf16hi(rr[i])));
      const f32x2 dv = fadd2(v, f2(-shift, -shift));
      s1 = fadd2(s1, dv);
      s2 = ffma2(dv, dv, s2);
      w[2 * i] = __float_as_uint(f2lo(v));
      w[2 * i + 1] = __float_as_uint(f2hi(v));
    }
    tmem_st32(taddr + tcol(c), w);
  }
  tmem_st_wait();
  pass1_done();
  LNT(1);
  const float S1 = f2lo(s1) + f2hi(s1), S2 = f2lo(s2) + f2hi(s2);
  const float4 mine = make_float4(shift, S1, S2, 0.f);
  stats[(merge.part_off() + hh) * 128 + q * 32 + lane] = mine;
  merge.publish(merge.part_off() + hh, q * 32 + lane, mine);
  asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * NP) : "memory");   // the NP warps of this quadrant
  merge.wait();
  LNT(2);
  const float nh = float(HALF);
  float mean, var;
  if constexpr (NPM == 2) {
    const float4 o = stats[(hh ^ 1) * 128 + q * 32 + lane];
    const float mean_a = shift + S1 / nh, m2_a = S2 - S1 * S1 / nh;
    const float mean_b = o.x + o.y / nh, m2_b = o.z - o.y * o.y / nh;
    const float dm = mean_a - mean_b;
    mean = 0.5f * (mean_a + mean_b);
    var = fmaxf((m2_a + m2_b + dm * dm * (nh * 0.5f)) / float(BN), 0.f);
  } else {
    // Chan's parallel merge of NPM equal-size parts, in part order (identical in every warp and CTA)
    float mp[NPM], m2p[NPM];
    float msum = 0.f;
#pragma unroll
    for (int i = 0; i < NPM; ++i) {
      const float4 o = stats[i * 128 + q * 32 + lane];
      mp[i] = o.x + o.y / nh;
      m2p[i] = o.z - o.y * o.y / nh;
      msum += mp[i];
    }
    mean = msum * (1.0f / NPM);
    float m2 = 0.f;
#pragma unroll
    for (int i = 0; i < NPM; ++i) {
      const float dm = mp[i] - mean;
      m2 += m2p[i] + nh * dm * dm;
    }
    var = fmaxf(m2 / float(NPM * HALF), 0.f);
  }
  const float rstd = rsqrtf(var + eps);
  const f32x2 k_rstd = f2(rstd, rstd), k_off = f2(-mean * rstd, -mean * rstd);
  tmem_ld32(taddr + tcol(lncol(0)), r[0]);
#pragma unroll
  for (int k = 0; k < NSTEP; ++k) {
    const int cur = PIPE ? (k & 1) : 0;
    const int c = lncol(k);
    if (!PIPE && k > 0) tmem_ld32(taddr + tcol(c), r[0]);
    tmem_ld_wait_regs(r[cur]);
    if (PIPE && k + 1 < NSTEP) tmem_ld32(taddr + tcol(lncol(k + 1)), r[cur ^ 1]);
    uint32_t p[16];
    uint4 cg[4], ce[4];
    if constexpr (sizeof(CT) == 2) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        cg[j] = reinterpret_cast<const uint4*>(s_gamma + c)[j];
        ce[j] = reinterpret_cast<const uint4*>(s_beta + c)[j];
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float2 gg, be;
      if constexpr (sizeof(CT) == 2) {
        const uint32_t ug = (&cg[i >> 2].x)[i & 3], ue = (&ce[i >> 2].x)[i & 3];
        gg = make_float2(bf16lo(ug), bf16hi(ug));
        be = make_float2(bf16lo(ue), bf16hi(ue));
      } else {
        gg = *reinterpret_cast<const float2*>(s_gamma + c + 2 * i);
        be = *reinterpret_cast<const float2*>(s_beta + c + 2 * i);
      }
      const f32x2 z = ffma2(f2(__uint_as_float(r[cur][2 * i]), __uint_as_float(r[cur][2 * i + 1])), k_rstd, k_off);
      const f32x2 y = ffma2(z, f2(gg.x, gg.y), f2(be.x, be.y));
      p[i] = pack_bf16x2(f2lo(y), f2hi(y));
    }
    store(p, c);
  }
  LNT(3);
}

}  // namespace surge
