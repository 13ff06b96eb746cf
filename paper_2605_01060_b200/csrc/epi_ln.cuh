// epi_ln.cuh -- the residual + LayerNorm GEMM epilogue (K6 / K8; reading R9:
// post-LN, biased variance, fp32 statistics), shared by the LN GEMM (gemm_tc.cu) and the fused tail
// kernel (mlp_tc.cu) so both round identically.
//
// Preloaded accumulator: before a tile's first MMA the epilogue writes bias + residual (fp32) into
// the TMEM accumulator and every MMA of the tile accumulates onto it, so the accumulator ends as
// v = bias + residual + A B^T.  The LN then only reads v -- no bias / residual traffic on its
// critical path, and the residual source (an smem tile or HBM rows) is free as soon as the preload
// is written, long before the LN runs.
//
// The accumulator row (BN fp32 columns in TMEM, lane = row) is split over NP warps of the same lane
// quadrant q, each owning columns [c_lo, c_lo + HALF), hh = which part.
//   pass 1: shifted partial sums of v (TMEM loads one step ahead);
//   combine the parts (Chan's parallel variance) through smem (stats: [NP parts][128 rows]);
//   pass 2: y = (v - mean) rstd gamma + beta -> bf16, handed to store(p, column) 32 columns at a time;
//           optionally the columns just read are rewritten with the NEXT tile's preload (pre).
#pragma once

#include "common.cuh"

namespace surge {

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

// ------------------------------------------------------------------------------ accumulator preloads
// w[0..31] = fp32 bias[c + i] + residual[c + i] for the 32 columns from c.
__device__ __forceinline__ void preload_values(const float* s_bias, int c, const uint32_t (&rs)[16], uint32_t (&w)[32]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 bb = *reinterpret_cast<const float2*>(s_bias + c + 2 * i);
    const f32x2 v = fadd2(f2(bb.x, bb.y), f2(bf16lo(rs[i]), bf16hi(rs[i])));
    w[2 * i] = __float_as_uint(f2lo(v));
    w[2 * i + 1] = __float_as_uint(f2hi(v));
  }
}

// Residual row in global memory (this row, column c_lo): rs = its 32 bf16 values of step k, packed.
__device__ __forceinline__ void load_row32(const uint16_t* row_c_lo, int k, uint32_t (&rs)[16]) {
  const uint4* p = reinterpret_cast<const uint4*>(row_c_lo + 32 * k);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 v = p[i];
    rs[4 * i] = v.x; rs[4 * i + 1] = v.y; rs[4 * i + 2] = v.z; rs[4 * i + 3] = v.w;
  }
}

// No preload in pass 2 (the accumulator is not reused, or the caller preloads it otherwise).
struct PreNone {
  static constexpr bool kActive = false;
  __device__ __forceinline__ bool on() const { return false; }
  __device__ __forceinline__ void load(int, uint32_t (&)[16]) const {}
  __device__ __forceinline__ void make(int, const uint32_t (&)[16], const uint32_t (&)[16], uint32_t (&)[32]) const {}
};

// Preload of the next tile's row: bias + residual read from global (row pointer at column c_lo;
// nullptr = no next tile).
struct PreGlobal {
  static constexpr bool kActive = true;
  const uint16_t* row;
  const float* s_bias;
  __device__ __forceinline__ bool on() const { return row != nullptr; }
  __device__ __forceinline__ void load(int k, uint32_t (&rs)[16]) const { load_row32(row, k, rs); }
  __device__ __forceinline__ void make(int c, const uint32_t (&rs)[16], const uint32_t (&)[16], uint32_t (&w)[32]) const {
    preload_values(s_bias, c, rs, w);
  }
};

// Preload from this LN's own output: the next GEMM on the same rows adds its bias to the bf16 value
// just produced (the fused tail: Y <- b2 + X1 while LN_a writes X1).
struct PreFromOutput {
  static constexpr bool kActive = true;
  const float* s_bias;
  __device__ __forceinline__ bool on() const { return true; }
  __device__ __forceinline__ void load(int, uint32_t (&)[16]) const {}
  __device__ __forceinline__ void make(int c, const uint32_t (&)[16], const uint32_t (&p)[16], uint32_t (&w)[32]) const {
    preload_values(s_bias, c, p, w);
  }
};

// Preload of a whole accumulator row part (columns [c_lo, c_lo + HALF)) from a global residual row:
// the first tile of a CTA, before any MMA.
template <int HALF>
__device__ __forceinline__ void ln_preload(uint32_t taddr, int c_lo, const uint16_t* row_c_lo, const float* s_bias) {
  constexpr int NSTEP = HALF / 32;
  uint32_t rs[2][16];
  load_row32(row_c_lo, 0, rs[0]);
#pragma unroll
  for (int k = 0; k < NSTEP; ++k) {
    if (k + 1 < NSTEP) load_row32(row_c_lo, k + 1, rs[(k + 1) & 1]);
    uint32_t w[32];
    preload_values(s_bias, c_lo + 32 * k, rs[k & 1], w);
    tmem_st32(taddr + c_lo + 32 * k, w);
  }
  tmem_st_wait();
}

// NP warps share a lane quadrant, each owning HALF = BN / NP columns (part hh).  PIPE: TMEM loads one
// step ahead (2 register buffers); !PIPE: one buffer (for register-limited kernels).
template <int BN, int HALF, bool PIPE = true, typename Ready, typename Store, typename Pre = PreNone,
          int NP = BN / HALF>
__device__ __forceinline__ void ln_epilogue(uint32_t taddr, int c_lo, const float* s_gamma, const float* s_beta,
                                            float4* stats, int q, int hh, int lane, float eps, Ready&& wait_ready,
                                            Store&& store, const Pre& pre = Pre{}) {
#ifdef LN_TRACE
  long long _lt = 0;
#endif
  constexpr int NSTEP = HALF / 32;
  constexpr int NB = PIPE ? 2 : 1;
  const bool pre_on = Pre::kActive && pre.on();
  uint32_t rn[2][16];                          // next tile's residual slices (PreGlobal), one step ahead
  if (pre_on) pre.load(0, rn[0]);              // in flight across pass 1
  uint32_t r[NB][32];
  wait_ready();
  LNT(0);
  tmem_ld32(taddr + c_lo, r[0]);
  float shift = 0.f;
  f32x2 s1 = f2(0.f, 0.f), s2 = f2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < NSTEP; ++k) {
    const int cur = PIPE ? (k & 1) : 0;
    if (!PIPE && k > 0) tmem_ld32(taddr + c_lo + 32 * k, r[0]);
    tmem_ld_wait_regs(r[cur]);
    if (PIPE && k + 1 < NSTEP) tmem_ld32(taddr + c_lo + 32 * (k + 1), r[cur ^ 1]);
    if (k == 0) shift = __uint_as_float(r[cur][0]);
    const f32x2 sh = f2(-shift, -shift);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const f32x2 dv = fadd2(f2(__uint_as_float(r[cur][2 * i]), __uint_as_float(r[cur][2 * i + 1])), sh);
      s1 = fadd2(s1, dv);
      s2 = ffma2(dv, dv, s2);
    }
  }
  LNT(1);
  const float S1 = f2lo(s1) + f2hi(s1), S2 = f2lo(s2) + f2hi(s2);
  stats[hh * 128 + q * 32 + lane] = make_float4(shift, S1, S2, 0.f);
  asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * NP) : "memory");   // the NP warps of this quadrant
  LNT(2);
  const float nh = float(HALF);
  float mean, var;
  if constexpr (NP == 2) {
    const float4 o = stats[(hh ^ 1) * 128 + q * 32 + lane];
    const float mean_a = shift + S1 / nh, m2_a = S2 - S1 * S1 / nh;
    const float mean_b = o.x + o.y / nh, m2_b = o.z - o.y * o.y / nh;
    const float dm = mean_a - mean_b;
    mean = 0.5f * (mean_a + mean_b);
    var = fmaxf((m2_a + m2_b + dm * dm * (nh * 0.5f)) / float(BN), 0.f);
  } else {
    // Chan's parallel merge of NP equal-size parts, in part order (identical in every warp)
    float mp[NP], m2p[NP];
    float msum = 0.f;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const float4 o = stats[i * 128 + q * 32 + lane];
      mp[i] = o.x + o.y / nh;
      m2p[i] = o.z - o.y * o.y / nh;
      msum += mp[i];
    }
    mean = msum * (1.0f / NP);
    float m2 = 0.f;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const float dm = mp[i] - mean;
      m2 += m2p[i] + nh * dm * dm;
    }
    var = fmaxf(m2 / float(BN), 0.f);
  }
  const float rstd = rsqrtf(var + eps);
  const f32x2 k_rstd = f2(rstd, rstd), k_off = f2(-mean * rstd, -mean * rstd);
  tmem_ld32(taddr + c_lo, r[0]);
#pragma unroll
  for (int k = 0; k < NSTEP; ++k) {
    const int cur = PIPE ? (k & 1) : 0;
    const int c = c_lo + 32 * k;
    if (!PIPE && k > 0) tmem_ld32(taddr + c, r[0]);
    tmem_ld_wait_regs(r[cur]);
    if (PIPE && k + 1 < NSTEP) tmem_ld32(taddr + c + 32, r[cur ^ 1]);
    if (pre_on && k + 1 < NSTEP) pre.load(k + 1, rn[(k + 1) & 1]);
    uint32_t p[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 gg = *reinterpret_cast<const float2*>(s_gamma + c + 2 * i);
      const float2 be = *reinterpret_cast<const float2*>(s_beta + c + 2 * i);
      const f32x2 z = ffma2(f2(__uint_as_float(r[cur][2 * i]), __uint_as_float(r[cur][2 * i + 1])), k_rstd, k_off);
      const f32x2 y = ffma2(z, f2(gg.x, gg.y), f2(be.x, be.y));
      p[i] = pack_bf16x2(f2lo(y), f2hi(y));
    }
    store(p, c);
    if (pre_on) {                              // these columns were read (wait::ld above): rewrite them
      uint32_t w[32];
      pre.make(c, rn[k & 1], p, w);
      tmem_st32(taddr + c, w);
    }
  }
  if (pre_on) tmem_st_wait();
  LNT(3);
}

}  // namespace surge
