// kernels.cu -- the non-GEMM kernels of the encoder chain (sm_100a):
//   K1 superbatch_pack : exclusive scan of text lengths -> cu_seqlens, partition row/token offsets
//   K3 embed_ln        : X[t] = LN(word[id_t] + pos[t - cu_s] + type[0])
//   K5 varlen_attention: per (text, head) softmax(Q K^T / sqrt(d_h)) V over the text's own tokens
//   K9 meanpool_l2     : e_s = v / max(||v||, 1e-12), v = mean of the text's rows
// All are HBM/L2-bound; accesses are 8- or 16-byte vectors, fp32 math, bf16 storage.
#include "attn_tile.cuh"
#include "common.cuh"
#include "internal.h"

#include <climits>
#include <type_traits>

namespace surge {

namespace {

// ------------------------------------------------------------------------------------ K1 pack
constexpr int PACK_THREADS = 1024;
constexpr int PACK_PER_THREAD = 8;

// out[0..n] = exclusive prefix sums of in[0..n), out[n] = total.  One CTA; tiles of 8192.
__device__ void block_exclusive_scan(const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ out,
                                     int32_t* s_warp, int32_t* s_carry) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) *s_carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += int64_t(PACK_THREADS) * PACK_PER_THREAD) {
    const int64_t i0 = base + int64_t(t) * PACK_PER_THREAD;
    int32_t v[PACK_PER_THREAD];
    int32_t local = 0;
#pragma unroll
    for (int k = 0; k < PACK_PER_THREAD; ++k) {
      v[k] = (i0 + k < n) ? in[i0 + k] : 0;
      local += v[k];
    }
    int32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[w] = incl;
    __syncthreads();
    if (w == 0) {
      int32_t x = s_warp[lane];
      int32_t xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += y;
      }
      s_warp[lane] = xi - x;   // exclusive warp offsets
    }
    __syncthreads();
    int32_t run = *s_carry + s_warp[w] + (incl - local);
#pragma unroll
    for (int k = 0; k < PACK_PER_THREAD; ++k) {
      if (i0 + k < n) out[i0 + k] = run;
      run += v[k];
    }
    __syncthreads();
    if (t == PACK_THREADS - 1) *s_carry = run;   // last thread holds the tile total + carry
    __syncthreads();
  }
  if (t == 0) out[n] = *s_carry;
}

__global__ void __launch_bounds__(PACK_THREADS) pack_kernel(const int32_t* __restrict__ lengths, int64_t n,
                                                            const int32_t* __restrict__ sizes, int64_t m,
                                                            int32_t* __restrict__ cu, int32_t* __restrict__ row_off,
                                                            int32_t* __restrict__ tok_off) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  block_exclusive_scan(lengths, n, cu, s_warp, &s_carry);
  if (m > 0) {
    __syncthreads();
    block_exclusive_scan(sizes, m, row_off, s_warp, &s_carry);
    __syncthreads();   // cu and row_off visible to the whole block
    for (int64_t j = threadIdx.x; j <= m; j += PACK_THREADS) tok_off[j] = cu[row_off[j]];
  }
}

// K1 for SuperBatches of more than one tile (S up to ~5.7e5 texts at a Safety flush): CTA b scans
// tile b after adding the sum of all lengths before it (read directly, coalesced: no scratch buffer,
// no inter-CTA protocol; the last CTA reads n - TILE values, a few microseconds), so the one-CTA tile
// loop (7.7 us per 8K-element tile, ~0.1 ms per C2 SuperBatch) becomes one wave of CTAs.  The
// partition offsets (m values) follow in a one-CTA kernel once cu is complete.
constexpr int PACK_TILE = PACK_THREADS * PACK_PER_THREAD;

__global__ void __launch_bounds__(PACK_THREADS) pack_scan_tiles_kernel(const int32_t* __restrict__ lengths,
                                                                       int64_t n, int32_t* __restrict__ cu) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t base = int64_t(blockIdx.x) * PACK_TILE;
  int32_t acc[4] = {0, 0, 0, 0};
  int64_t i = t;
  for (; i + 3 * PACK_THREADS < base; i += 4 * PACK_THREADS) {
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] += __ldg(lengths + i + k * PACK_THREADS);
  }
  for (; i < base; i += PACK_THREADS) acc[0] += __ldg(lengths + i);
  int32_t part = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) s_warp[w] = part;
  __syncthreads();
  if (w == 0) {
    int32_t x = s_warp[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) s_carry = x;
  }
  __syncthreads();
  // the one-tile body of block_exclusive_scan, starting from the carry
  const int64_t i0 = base + int64_t(t) * PACK_PER_THREAD;
  int32_t v[PACK_PER_THREAD];
  int32_t local = 0;
#pragma unroll
  for (int k = 0; k < PACK_PER_THREAD; ++k) {
    v[k] = (i0 + k < n) ? lengths[i0 + k] : 0;
    local += v[k];
  }
  int32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();   // s_warp reused
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    int32_t x = s_warp[lane];
    int32_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    s_warp[lane] = xi - x;
  }
  __syncthreads();
  int32_t run = s_carry + s_warp[w] + (incl - local);
#pragma unroll
  for (int k = 0; k < PACK_PER_THREAD; ++k) {
    if (i0 + k < n) cu[i0 + k] = run;
    run += v[k];
  }
  if (blockIdx.x == gridDim.x - 1 && t == PACK_THREADS - 1) cu[n] = run;   // the total
}

__global__ void __launch_bounds__(PACK_THREADS) pack_offsets_kernel(const int32_t* __restrict__ sizes, int64_t m,
                                                                    const int32_t* __restrict__ cu,
                                                                    int32_t* __restrict__ row_off,
                                                                    int32_t* __restrict__ tok_off) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  block_exclusive_scan(sizes, m, row_off, s_warp, &s_carry);
  __syncthreads();
  for (int64_t j = threadIdx.x; j <= m; j += PACK_THREADS) tok_off[j] = cu[row_off[j]];
}

// ------------------------------------------------------------------------------- K3 embed + LN
// One warp per text; lane owns columns {4*(lane + 32*i) .. +3}.
template <int D>
__global__ void __launch_bounds__(256) embed_ln_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ cu,
                                                       int64_t n_texts, int32_t tok0, const uint16_t* __restrict__ word,
                                                       const uint16_t* __restrict__ pos,
                                                       const uint16_t* __restrict__ type,
                                                       const float* __restrict__ gamma,
                                                       const float* __restrict__ beta, float eps,
                                                       uint16_t* __restrict__ x) {
  constexpr int G = D / 4;                       // 4-column groups per row
  constexpr int PER = (G + 31) / 32;
  const int64_t text = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (text >= n_texts) return;
  const int32_t a = cu[text], b = cu[text + 1];
  float g4[PER][4], b4[PER][4], ty[PER][4];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int g = lane + 32 * i;
    if (g < G) {
      const float4 gg = reinterpret_cast<const float4*>(gamma)[g];
      const float4 bb = reinterpret_cast<const float4*>(beta)[g];
      const uint2 tt = reinterpret_cast<const uint2*>(type)[g];
      g4[i][0] = gg.x; g4[i][1] = gg.y; g4[i][2] = gg.z; g4[i][3] = gg.w;
      b4[i][0] = bb.x; b4[i][1] = bb.y; b4[i][2] = bb.z; b4[i][3] = bb.w;
      ty[i][0] = bf16lo(tt.x); ty[i][1] = bf16hi(tt.x); ty[i][2] = bf16lo(tt.y); ty[i][3] = bf16hi(tt.y);
    }
  }
  // NT tokens of the text at a time: independent gather -> reduce -> store chains interleave (the
  // per-token chain is latency-bound: two L2 gathers, then two dependent warp reductions)
  auto tokens = [&](auto nt_tag, int32_t t) {
    constexpr int NT = decltype(nt_tag)::value;
    float v[NT][PER][4];
    float s[NT];
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      const int32_t id = ids[t + u];
      const uint2* wr = reinterpret_cast<const uint2*>(word + size_t(id) * D);
      const uint2* pr = reinterpret_cast<const uint2*>(pos + size_t(t + u - a) * D);
      s[u] = 0.f;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int g = lane + 32 * i;
        if (g < G) {
          const uint2 w2 = __ldg(wr + g), p2 = __ldg(pr + g);
          v[u][i][0] = bf16lo(w2.x) + bf16lo(p2.x) + ty[i][0];
          v[u][i][1] = bf16hi(w2.x) + bf16hi(p2.x) + ty[i][1];
          v[u][i][2] = bf16lo(w2.y) + bf16lo(p2.y) + ty[i][2];
          v[u][i][3] = bf16hi(w2.y) + bf16hi(p2.y) + ty[i][3];
          s[u] += v[u][i][0] + v[u][i][1] + v[u][i][2] + v[u][i][3];
        } else {
          v[u][i][0] = v[u][i][1] = v[u][i][2] = v[u][i][3] = 0.f;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      const float mean = warp_sum(s[u]) * (1.0f / D);
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int g = lane + 32 * i;
        if (g < G) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float dv = v[u][i][k] - mean;
            q += dv * dv;
          }
        }
      }
      const float rstd = rsqrtf(warp_sum(q) * (1.0f / D) + eps);
      uint2* xr = reinterpret_cast<uint2*>(x + size_t(t + u - tok0) * D);
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int g = lane + 32 * i;
        if (g < G) {
          float y[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) y[k] = (v[u][i][k] - mean) * rstd * g4[i][k] + b4[i][k];
          xr[g] = make_uint2(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]));
        }
      }
    }
  };
  int32_t t = a;
#ifndef EMB_NT
#define EMB_NT 2   // tokens per step (4: 113 registers, lower occupancy, measured slower)
#endif
  for (; t + EMB_NT <= b; t += EMB_NT) tokens(std::integral_constant<int, EMB_NT>{}, t);
  if (EMB_NT > 2 && t + 2 <= b) {
    tokens(std::integral_constant<int, 2>{}, t);
    t += 2;
  }
  if (t < b) tokens(std::integral_constant<int, 1>{}, t);
}

// K3 for d = 384 with 16-byte accesses: one warp per text, each half-warp one token at a time (two tokens per
// warp step), lane l of a half owning the 8-column groups l, l + 16, l + 32 -- every load and store
// instruction of a half-warp covers 256 contiguous bytes of a row; the row reductions are 4-step half-warp
// butterflies.  gamma, beta and the token-type row are held as packed bf16 pairs (they are bf16 values of the
// weight blob, so the packing is exact).  v = word + pos + type, mean, biased variance, as embed_ln_kernel.
// Measured slower than the 8-byte one-warp-per-token-pair kernel (11.2 vs 8.9 ms per 2M texts: 116 registers,
// two CTAs per SM instead of three; the kernel is latency-bound on its two dependent row reductions, not on
// load width), so EMB_V16 is off.
#ifndef EMB_V16
#define EMB_V16 0
#endif
template <int D>
__global__ void __launch_bounds__(256) embed_ln16_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ cu,
                                                         int64_t n_texts, int32_t tok0, const uint16_t* __restrict__ word,
                                                         const uint16_t* __restrict__ pos,
                                                         const uint16_t* __restrict__ type,
                                                         const float* __restrict__ gamma,
                                                         const float* __restrict__ beta, float eps,
                                                         uint16_t* __restrict__ x) {
  constexpr int PER = D / 128;                    // 16-byte groups per lane
  static_assert(D % 128 == 0, "d");
  const int64_t text = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, hl = lane & 15, hw = lane >> 4;
  if (text >= n_texts) return;
  const int32_t a = cu[text], b = cu[text + 1];
  uint32_t gp[PER][4], bp[PER][4], tp[PER][4];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int g = hl + 16 * i;
    const float4 g0 = reinterpret_cast<const float4*>(gamma)[2 * g], g1 = reinterpret_cast<const float4*>(gamma)[2 * g + 1];
    const float4 b0 = reinterpret_cast<const float4*>(beta)[2 * g], b1 = reinterpret_cast<const float4*>(beta)[2 * g + 1];
    gp[i][0] = pack_bf16x2(g0.x, g0.y); gp[i][1] = pack_bf16x2(g0.z, g0.w);
    gp[i][2] = pack_bf16x2(g1.x, g1.y); gp[i][3] = pack_bf16x2(g1.z, g1.w);
    bp[i][0] = pack_bf16x2(b0.x, b0.y); bp[i][1] = pack_bf16x2(b0.z, b0.w);
    bp[i][2] = pack_bf16x2(b1.x, b1.y); bp[i][3] = pack_bf16x2(b1.z, b1.w);
    const uint4 tt = reinterpret_cast<const uint4*>(type)[g];
    tp[i][0] = tt.x; tp[i][1] = tt.y; tp[i][2] = tt.z; tp[i][3] = tt.w;
  }
  for (int32_t t0 = a; t0 < b; t0 += 2) {        // warp-uniform trip count: both halves run the shuffles
    const int32_t t = t0 + hw;
    const bool ok = t < b;
    const int32_t tt = ok ? t : t0;
    const int32_t id = ids[tt];
    const uint4* wr = reinterpret_cast<const uint4*>(word + size_t(id) * D);
    const uint4* pr = reinterpret_cast<const uint4*>(pos + size_t(tt - a) * D);
    uint4 w4[PER], p4[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      w4[i] = __ldg(wr + hl + 16 * i);
      p4[i] = __ldg(pr + hl + 16 * i);
    }
    float v[PER][8];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const uint32_t wv[4] = {w4[i].x, w4[i].y, w4[i].z, w4[i].w}, pv[4] = {p4[i].x, p4[i].y, p4[i].z, p4[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[i][2 * j] = bf16lo(wv[j]) + bf16lo(pv[j]) + bf16lo(tp[i][j]);
        v[i][2 * j + 1] = bf16hi(wv[j]) + bf16hi(pv[j]) + bf16hi(tp[i][j]);
        s += v[i][2 * j] + v[i][2 * j + 1];
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s * (1.0f / D);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float dv = v[i][k] - mean;
        q += dv * dv;
      }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float rstd = rsqrtf(q * (1.0f / D) + eps);
    if (ok) {
      uint4* xr = reinterpret_cast<uint4*>(x + size_t(t - tok0) * D);
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        uint32_t o4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float y0 = (v[i][2 * j] - mean) * rstd * bf16lo(gp[i][j]) + bf16lo(bp[i][j]);
          const float y1 = (v[i][2 * j + 1] - mean) * rstd * bf16hi(gp[i][j]) + bf16hi(bp[i][j]);
          o4[j] = pack_bf16x2(y0, y1);
        }
        xr[hl + 16 * i] = make_uint4(o4[0], o4[1], o4[2], o4[3]);
      }
    }
  }
}

// ------------------------------------------------------------------------- K5 varlen attention
// One warp per (text, head).  Lane j owns query row qb+j; the text's K/V rows for this head are
// staged 32 at a time in shared memory as fp32 and read as broadcasts.  Scores of a 32-key tile
// are formed first, then one online-softmax rescale per tile (exp2 with log2(e)/sqrt(d_h) folded
// into q).
template <int DH>
struct AttCfg {
  static constexpr int WARPS = DH <= 32 ? 4 : 2;   // 2 x 32 x DH fp32 per warp in smem
};

template <int DH, int ATT_WARPS = AttCfg<DH>::WARPS>
__global__ void __launch_bounds__(ATT_WARPS * 32) attention_kernel(const uint16_t* __restrict__ qkv,
                                                                   const int32_t* __restrict__ cu, int64_t n_texts,
                                                                   int32_t tok0, int heads,
                                                                   uint16_t* __restrict__ out, float qscale,
                                                                   int32_t min_len) {
  __shared__ __align__(16) float sK[ATT_WARPS][32][DH];
  __shared__ __align__(16) float sV[ATT_WARPS][32][DH];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = int64_t(blockIdx.x) * ATT_WARPS + w;
  if (item >= n_texts * heads) return;
  const int64_t text = item / heads;
  const int h = int(item % heads);
  const int d = heads * DH, ld = 3 * d;
  const int32_t start = cu[text] - tok0;
  const int32_t len = cu[text + 1] - cu[text];
  if (len < min_len) return;   // short texts are handled by attention_text_kernel
  constexpr int V8 = DH / 8;   // 16-byte vectors per head row

  for (int qb = 0; qb < len; qb += 32) {
    const int qi = qb + lane;
    const bool qok = qi < len;
    float q[DH];
    {
      const uint4* qp = reinterpret_cast<const uint4*>(qkv + size_t(start + (qok ? qi : 0)) * ld + h * DH);
#pragma unroll
      for (int v = 0; v < V8; ++v) {
        const uint4 u = qp[v];
        const uint32_t uu[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          q[v * 8 + 2 * k] = bf16lo(uu[k]) * qscale;
          q[v * 8 + 2 * k + 1] = bf16hi(uu[k]) * qscale;
        }
      }
    }
    float o[DH];
#pragma unroll
    for (int c = 0; c < DH; ++c) o[c] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int kb = 0; kb < len; kb += 32) {
      const int nk = min(32, len - kb);
      __syncwarp();
      if (lane < nk) {
        const size_t r = size_t(start + kb + lane) * ld + h * DH;
        const uint4* kp = reinterpret_cast<const uint4*>(qkv + r + d);
        const uint4* vp = reinterpret_cast<const uint4*>(qkv + r + 2 * d);
#pragma unroll
        for (int v = 0; v < V8; ++v) {
          const uint4 ku = kp[v], vu = vp[v];
          const uint32_t kk[4] = {ku.x, ku.y, ku.z, ku.w};
          const uint32_t vv[4] = {vu.x, vu.y, vu.z, vu.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            sK[w][lane][v * 8 + 2 * k] = bf16lo(kk[k]);
            sK[w][lane][v * 8 + 2 * k + 1] = bf16hi(kk[k]);
            sV[w][lane][v * 8 + 2 * k] = bf16lo(vv[k]);
            sV[w][lane][v * 8 + 2 * k + 1] = bf16hi(vv[k]);
          }
        }
      }
      __syncwarp();
      float s[32];
      float mt = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < nk) {
          const float4* kr = reinterpret_cast<const float4*>(&sK[w][j][0]);
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < DH / 4; ++c) {
            const float4 k4 = kr[c];
            acc = fmaf(q[4 * c], k4.x, acc);
            acc = fmaf(q[4 * c + 1], k4.y, acc);
            acc = fmaf(q[4 * c + 2], k4.z, acc);
            acc = fmaf(q[4 * c + 3], k4.w, acc);
          }
          s[j] = acc;
          mt = fmaxf(mt, acc);
        } else {
          s[j] = -INFINITY;
        }
      }
      const float mnew = fmaxf(m, mt);
      const float corr = exp2f(m - mnew);   // m = -inf on the first tile -> 0
      l *= corr;
#pragma unroll
      for (int c = 0; c < DH; ++c) o[c] *= corr;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < nk) {
          const float p = exp2f(s[j] - mnew);
          l += p;
          const float4* vr = reinterpret_cast<const float4*>(&sV[w][j][0]);
#pragma unroll
          for (int c = 0; c < DH / 4; ++c) {
            const float4 v4 = vr[c];
            o[4 * c] = fmaf(p, v4.x, o[4 * c]);
            o[4 * c + 1] = fmaf(p, v4.y, o[4 * c + 1]);
            o[4 * c + 2] = fmaf(p, v4.z, o[4 * c + 2]);
            o[4 * c + 3] = fmaf(p, v4.w, o[4 * c + 3]);
          }
        }
      }
      m = mnew;
    }
    if (qok) {
      const float inv = 1.0f / l;
      uint4* op = reinterpret_cast<uint4*>(out + size_t(start + qi) * d + h * DH);
#pragma unroll
      for (int v = 0; v < V8; ++v) {
        op[v] = make_uint4(pack_bf16x2(o[v * 8 + 0] * inv, o[v * 8 + 1] * inv),
                           pack_bf16x2(o[v * 8 + 2] * inv, o[v * 8 + 3] * inv),
                           pack_bf16x2(o[v * 8 + 4] * inv, o[v * 8 + 5] * inv),
                           pack_bf16x2(o[v * 8 + 6] * inv, o[v * 8 + 7] * inv));
      }
    }
  }
}

// ------------------------------------------------- K5 (texts <= 64 tokens): tensor-core tiles
// win[w] = min{ s : cu[s] - tok0 >= 64 w } for w in [0, nwin], nwin = ceil(ntok / 64) (win[nwin] = n):
// the first text that starts in 64-token window w.  One thread per text boundary s in [0, n].
__global__ void window_index_kernel(const int32_t* __restrict__ cu, int64_t n, int32_t tok0, int32_t ntok,
                                    int32_t* __restrict__ win) {
  const int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > n) return;
  const int32_t nwin = (ntok + 63) >> 6;
  const int32_t prev = (s == 0) ? -1 : cu[s - 1] - tok0;
  const int32_t a = (s == n) ? ntok : cu[s] - tok0;
  const int32_t w_lo = (prev < 0) ? 0 : (prev >> 6) + 1;
  const int32_t w_hi = (s == n) ? nwin : (a >> 6);
  for (int32_t w = w_lo; w <= w_hi; ++w) win[w] = int32_t(s);
}

// Block-diagonal varlen attention for texts of <= ATT_SHORT tokens, text-tiled.  A CTA owns the
// texts that START in one 64-token window (their rows [R0, R1) span at most 64 + 63 tokens, so
// no halo is loaded) and a group of HG heads; Q/K/V of those rows are staged in padded shared
// memory with cp.async.  Each warp takes whole texts: per (text, head), query tiles of 16 rows
// and key blocks of 16 keys, both aligned to the text's first token, on mma.sync m16n8k16 (bf16
// in, fp32 accumulate; P split hi+lo bf16), keys masked to j < len, flash-style online softmax in
// exp2 form.  Every text's arithmetic is therefore identical wherever it sits in the stream
// (bit-exact SuperBatch invariance).  O is written over the text's own Q rows and stored with
// 16-byte coalesced stores.  A text longer than ATT_SHORT is left to attention_kernel.
constexpr int ATT_SHORT = 64;
#ifndef ATT_HEADS_PER_CTA
#define ATT_HEADS_PER_CTA 2
#endif

template <int DH, int HG>
struct TextAtt {
  static constexpr int WIN = 64;                 // window of text starts per CTA
  static constexpr int WARPS = 4;
  static constexpr int COLS = HG * DH;           // columns of one Q / K / V slice
  static constexpr int LDS = COLS + 8;           // smem row stride (bf16): 16-byte skew per row
  static constexpr int CH = COLS / 8;            // 16-byte chunks per row
  // rows staged: texts starting in the window end within WIN + L - 1 rows (L = longest short
  // text), + 16 zero rows read by the last tile
  static int rows(int max_len) {
    const int L = max_len < ATT_SHORT ? (max_len < 1 ? 1 : max_len) : ATT_SHORT;
    return WIN + L - 1 + 16;
  }
  static size_t smem(int max_len) { return size_t(3) * rows(max_len) * LDS * 2; }
};

template <int DH, int HG>
__global__ void __launch_bounds__(TextAtt<DH, HG>::WARPS * 32) attention_text_kernel(
    const uint16_t* __restrict__ qkv, const int32_t* __restrict__ cu, int32_t tok0, int32_t ntok,
    const int32_t* __restrict__ win, int heads, uint16_t* __restrict__ out, float qscale, int ROWS) {
  using A = TextAtt<DH, HG>;
  constexpr int LDS = A::LDS, CH = A::CH;
  extern __shared__ __align__(16) uint16_t att_sm[];
  uint16_t* sQ = att_sm;                         // [ROWS][LDS]  (Q, then O)
  uint16_t* sK = sQ + ROWS * LDS;
  uint16_t* sV = sK + ROWS * LDS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int d = heads * DH, ld = 3 * d;
  const int col0 = blockIdx.y * A::COLS;
  const int32_t s_a = win[blockIdx.x];
  int32_t s_b = win[blockIdx.x + 1];             // texts [s_a, s_b) start in this window
  if (s_b <= s_a) return;
  const int32_t R0 = cu[s_a] - tok0;
  // a text longer than ATT_SHORT can only be the window's last text (it ends past the next window)
  if (cu[s_b] - cu[s_b - 1] > ATT_SHORT) --s_b;
  const int32_t R1 = cu[s_b] - tok0;
  const int nr = R1 - R0;                        // <= WIN + ATT_SHORT - 1
  for (int i = tid; i < nr * CH; i += blockDim.x) {
    const int r = i / CH, c = i - r * CH;
    const uint16_t* g = qkv + size_t(R0 + r) * ld + col0 + c * 8;
    cp_async16(sQ + r * LDS + c * 8, g);
    cp_async16(sK + r * LDS + c * 8, g + d);
    cp_async16(sV + r * LDS + c * 8, g + 2 * d);
  }
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int i = tid; i < 16 * CH; i += blockDim.x) {   // tiles may read 15 rows past the last text
    const int r = nr + i / CH, c = i % CH;
    *reinterpret_cast<uint4*>(sQ + r * LDS + c * 8) = z;
    *reinterpret_cast<uint4*>(sK + r * LDS + c * 8) = z;
    *reinterpret_cast<uint4*>(sV + r * LDS + c * 8) = z;
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  // work units (text, head), round-robin over the warps
#pragma unroll 1
  for (int32_t u = warp; u < s_b - s_a; u += A::WARPS) {   // work unit: one text, all HG heads
    const int32_t txt = s_a + u;
    const int32_t ta = cu[txt] - tok0 - R0;      // smem row of the text's first token
    const int32_t len = cu[txt + 1] - cu[txt];
    const int nt = (len + 15) >> 4;              // query tiles = key blocks
#pragma unroll 1
    for (int qt = 0; qt < nt; ++qt) {
      uint16_t* sQt = sQ + (ta + 16 * qt) * LDS;
      float o[HG][DH / 8][4];
      float ia[HG], ib[HG];
      attn_query_tile<DH, LDS, HG>(sQt, sK + ta * LDS, sV + ta * LDS, len, nt, qscale, lane, o, ia, ib, len - 16 * qt,
                                   sQ + nr * LDS);
      __syncwarp();   // every lane has read its Q fragments before O overwrites the tile
      attn_store_tile<DH, HG>(sQt, LDS, qt, len, lane, o, ia, ib);
    }
  }
  __syncthreads();
  for (int i = tid; i < nr * CH; i += blockDim.x) {
    const int r = i / CH, c = i - r * CH;
    *reinterpret_cast<uint4*>(out + size_t(R0 + r) * d + col0 + c * 8) =
        *reinterpret_cast<const uint4*>(sQ + r * LDS + c * 8);
  }
}

// ------------------------------------------------- K5 (texts > ATT_SHORT tokens): one CTA per (text, head)
// The text's K and V rows for the head (<= max_position rows) stay in shared memory; query blocks of
// 128 rows (8 warps x 16) are staged in turn.  The per-row arithmetic is the text-tiled kernel's:
// 16-row query tiles and 16-key blocks aligned to the text start, mma.sync m16n8k16 with P split
// hi+lo, online softmax over the key blocks in order (so long and short texts follow one rule).
// warps per CTA of the long-text kernel's classes <= 256 tokens (> 256: 16); C4 attention per 50K texts:
// 4 warps 1,309 ms, 8 warps 1,238 ms, 12 warps 1,429 ms
#ifndef ATT_LONG_WS
#define ATT_LONG_WS 8
#endif
// W warps per CTA (query blocks of 16 W rows); the launcher splits the long texts into length classes so
// the K/V buffers (and the CTAs per SM) fit the class: (64, 128], (128, 192], (192, 256] with 8 warps,
// (256, 512] with 16 -- a 150-token text no longer takes a whole SM's shared memory sized for 512
template <int DH, int W>
struct LongAtt {
  static constexpr int WARPS = W;                // one 16-row query tile per warp
  static constexpr int QROWS = 16 * WARPS;
  static constexpr int LDS = DH + 8;
  static constexpr int CH = DH / 8;
  static int kv_rows(int max_len) { return ((max_len + 15) / 16) * 16 + 16; }
  static size_t smem(int max_len) { return size_t(2 * kv_rows(max_len) + QROWS + 16) * LDS * 2; }
};

template <int DH, int W>
__global__ void __launch_bounds__(W * 32) attention_long_kernel(
    const uint16_t* __restrict__ qkv, const int32_t* __restrict__ cu, const int32_t* __restrict__ texts,
    int32_t tok0, int heads, uint16_t* __restrict__ out, float qscale, int kv_rows, int min_handled,
    int max_handled) {
  using A = LongAtt<DH, W>;
  constexpr int LDS = A::LDS, CH = A::CH;
  extern __shared__ __align__(16) uint16_t att_sm[];
  uint16_t* sK = att_sm;                         // [kv_rows][LDS]
  uint16_t* sV = sK + kv_rows * LDS;             // [kv_rows][LDS]
  uint16_t* sQ = sV + kv_rows * LDS;             // [QROWS + 16][LDS]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t txt = texts[blockIdx.x];
  const int h = blockIdx.y;
  const int d = heads * DH, ld = 3 * d;
  const int32_t a = cu[txt] - tok0, len = cu[txt + 1] - cu[txt];
  if (len > max_handled || len <= min_handled) return;   // another length class (or the tcgen05 kernel)
  const int nt = (len + 15) >> 4;
  for (int i = tid; i < len * CH; i += blockDim.x) {
    const int r = i / CH, c = i - r * CH;
    const uint16_t* g = qkv + size_t(a + r) * ld + h * DH + c * 8;
    cp_async16(sK + r * LDS + c * 8, g + d);
    cp_async16(sV + r * LDS + c * 8, g + 2 * d);
  }
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int i = tid; i < (nt * 16 + 16 - len) * CH; i += blockDim.x) {
    const int r = len + i / CH, c = i % CH;
    *reinterpret_cast<uint4*>(sK + r * LDS + c * 8) = z;
    *reinterpret_cast<uint4*>(sV + r * LDS + c * 8) = z;
  }
#pragma unroll 1
  for (int qb0 = 0; qb0 < len; qb0 += A::QROWS) {
    const int nq = min(A::QROWS, len - qb0);
    for (int i = tid; i < nq * CH; i += blockDim.x) {
      const int r = i / CH, c = i - r * CH;
      cp_async16(sQ + r * LDS + c * 8, qkv + size_t(a + qb0 + r) * ld + h * DH + c * 8);
    }
    for (int i = tid; i < (A::QROWS + 16 - nq) * CH; i += blockDim.x) {
      const int r = nq + i / CH, c = i % CH;
      *reinterpret_cast<uint4*>(sQ + r * LDS + c * 8) = z;
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int qt = (qb0 >> 4) + warp;            // query tile within the text
    if (16 * qt < len) {
      float o[1][DH / 8][4];
      float ia[1], ib[1];
      attn_query_tile<DH, LDS, 1>(sQ + 16 * warp * LDS, sK, sV, len, nt, qscale, lane, o, ia, ib, nq - 16 * warp,
                                  sQ + A::QROWS * LDS);
      attn_store_tile<DH, 1>(out + size_t(a + 16 * qt) * d + h * DH, size_t(d), qt, len, lane, o, ia, ib);
    }
    __syncthreads();                             // sQ reused by the next query block
  }
}

// ------------------------------------------------------------------------ row LayerNorm (d > 384)
// One warp per row: fp32 v (D values, 16-byte loads) -> mean, biased variance (two passes over the
// registers), y = (v - mean) rstd gamma + beta -> bf16.
template <int D>
__global__ void __launch_bounds__(256) layernorm_kernel(const float* __restrict__ v, int64_t rows,
                                                        const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, float eps,
                                                        uint16_t* __restrict__ y) {
  constexpr int PER = D / 128;                   // float4 per lane
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float4* vr = reinterpret_cast<const float4*>(v + size_t(row) * D);
  float4 x[PER];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    x[i] = vr[lane + 32 * i];
    s += (x[i].x + x[i].y) + (x[i].z + x[i].w);
  }
  const float mean = warp_sum(s) * (1.0f / D);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const float a = x[i].x - mean, b = x[i].y - mean, c = x[i].z - mean, d = x[i].w - mean;
    q += (a * a + b * b) + (c * c + d * d);
  }
  const float rstd = rsqrtf(warp_sum(q) * (1.0f / D) + eps);
  uint2* yr = reinterpret_cast<uint2*>(y + size_t(row) * D);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int g = lane + 32 * i;
    const float4 gg = reinterpret_cast<const float4*>(gamma)[g];
    const float4 bb = reinterpret_cast<const float4*>(beta)[g];
    yr[g] = make_uint2(pack_bf16x2((x[i].x - mean) * rstd * gg.x + bb.x, (x[i].y - mean) * rstd * gg.y + bb.y),
                       pack_bf16x2((x[i].z - mean) * rstd * gg.z + bb.z, (x[i].w - mean) * rstd * gg.w + bb.w));
  }
}

// ----------------------------------------------------------------------------- K9 meanpool + L2
// CLS: [CLS] pooling (the text's first row only; bge's native pooling, execution option).
// OUTB: the unit vector is stored as bf16 (out_dtype SURGE_BF16) instead of fp32.
template <int D, bool CLS = false, bool OUTB = false>
__global__ void __launch_bounds__(256) meanpool_l2_kernel(const uint16_t* __restrict__ x,
                                                          const int32_t* __restrict__ cu, int64_t n_texts,
                                                          int32_t tok0, void* __restrict__ out) {
  constexpr int G = D / 4;
  constexpr int PER = (G + 31) / 32;
  const int64_t text = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (text >= n_texts) return;
  const int32_t a = cu[text] - tok0, b = CLS ? a + 1 : cu[text + 1] - tok0;
  float acc[PER][4];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  for (int32_t t = a; t < b; ++t) {
    const uint2* xr = reinterpret_cast<const uint2*>(x + size_t(t) * D);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int g = lane + 32 * i;
      if (g < G) {
        const uint2 u = xr[g];
        acc[i][0] += bf16lo(u.x);
        acc[i][1] += bf16hi(u.x);
        acc[i][2] += bf16lo(u.y);
        acc[i][3] += bf16hi(u.y);
      }
    }
  }
  const float inv_l = 1.0f / float(b - a);
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc[i][k] *= inv_l;
      ss += acc[i][k] * acc[i][k];
    }
  }
  const float inv = 1.0f / fmaxf(sqrtf(warp_sum(ss)), 1e-12f);
  if constexpr (OUTB) {
    uint2* orow = reinterpret_cast<uint2*>(static_cast<uint16_t*>(out) + size_t(text) * D);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int g = lane + 32 * i;
      if (g < G)
        orow[g] = make_uint2(pack_bf16x2(acc[i][0] * inv, acc[i][1] * inv), pack_bf16x2(acc[i][2] * inv, acc[i][3] * inv));
    }
  } else {
    float4* orow = reinterpret_cast<float4*>(static_cast<float*>(out) + size_t(text) * D);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int g = lane + 32 * i;
      if (g < G) orow[g] = make_float4(acc[i][0] * inv, acc[i][1] * inv, acc[i][2] * inv, acc[i][3] * inv);
    }
  }
}

__global__ void bf16_to_f32_kernel(const uint16_t* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = bf16f(in[i]);
}

// Tile records for the fused QKV + attention kernel (internal.h ATT_REC_INTS layout): one warp per
// tile; the unit list is built level by level (cost = ceil(len / 16) from 8 down to 1) with an
// exclusive warp scan of each text's unit count.
__global__ void __launch_bounds__(256) att_records_kernel(const int32_t* __restrict__ tiles, int32_t n_tiles,
                                                          const int32_t* __restrict__ cu, int32_t tok0,
                                                          int32_t n_groups, int32_t* __restrict__ rec) {
  const int32_t t = int32_t((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= n_tiles) return;
  const int32_t s_a = tiles[t], s_b = tiles[t + 1];
  const int32_t base = cu[s_a];
  int32_t* r = rec + size_t(t) * ATT_REC_INTS;
  uint8_t* start = reinterpret_cast<uint8_t*>(r + 4);
  uint16_t* units = reinterpret_cast<uint16_t*>(r + 36);
  const int n = s_b - s_a;
  for (int j = lane; j < n; j += 32) start[j] = uint8_t(cu[s_a + j] - base);
  int run = 0;
  for (int level = 8; level >= 1; --level) {
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      int cnt = 0;
      if (j < n) {
        const int a = cu[s_a + j];
        const int c = (cu[s_a + j + 1] - a + 15) >> 4;
        cnt = c == level ? c * n_groups : 0;
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      for (int q = 0; q < cnt; ++q)
        units[run + incl - cnt + q] = uint16_t(j | ((q / n_groups) << 8) | ((q % n_groups) << 11));
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  if (lane == 0) {
    r[0] = base - tok0;
    r[1] = cu[s_b] - base;
    r[2] = n;
    r[3] = run;
  }
}

inline unsigned blocks_for_warps(int64_t warps, int warps_per_block) {
  return unsigned((warps + warps_per_block - 1) / warps_per_block);
}

}  // namespace

cudaError_t launch_bf16_to_f32(const uint16_t* in, float* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  bf16_to_f32_kernel<<<unsigned((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

int pack_launch_count(int64_t n, int64_t m) { return n <= PACK_TILE ? 1 : (m > 0 ? 2 : 1); }

cudaError_t launch_pack(const int32_t* lengths, int64_t n, const int32_t* sizes, int64_t m, int32_t* cu,
                        int32_t* row_off, int32_t* tok_off, cudaStream_t st) {
  if (n <= PACK_TILE) {       // one tile: the one-CTA kernel does cu and the partition offsets
    pack_kernel<<<1, PACK_THREADS, 0, st>>>(lengths, n, sizes, m, cu, row_off, tok_off);
    return cudaGetLastError();
  }
  pack_scan_tiles_kernel<<<unsigned((n + PACK_TILE - 1) / PACK_TILE), PACK_THREADS, 0, st>>>(lengths, n, cu);
  if (m > 0) pack_offsets_kernel<<<1, PACK_THREADS, 0, st>>>(sizes, m, cu, row_off, tok_off);
  return cudaGetLastError();
}

cudaError_t launch_embed_ln(const int32_t* ids, const int32_t* cu, int64_t n_texts, int32_t tok0,
                            const uint16_t* word, const uint16_t* pos, const uint16_t* type, const float* gamma,
                            const float* beta, int d, float eps, uint16_t* x, cudaStream_t st) {
  if (n_texts <= 0) return cudaSuccess;
  const unsigned grid = blocks_for_warps(n_texts, 8);
#define SURGE_EMB(DD)                                                                                       \
  case DD:                                                                                                   \
    embed_ln_kernel<DD><<<grid, 256, 0, st>>>(ids, cu, n_texts, tok0, word, pos, type, gamma, beta, eps, x); \
    break;
  if (EMB_V16 && d == 384) {
    embed_ln16_kernel<384><<<grid, 256, 0, st>>>(ids, cu, n_texts, tok0, word, pos, type, gamma, beta, eps, x);
    return cudaGetLastError();
  }
  switch (d) {
    SURGE_EMB(64)
    SURGE_EMB(384)
    SURGE_EMB(768)
    SURGE_EMB(1024)
    default: return cudaErrorInvalidValue;
  }
#undef SURGE_EMB
  return cudaGetLastError();
}

cudaError_t launch_attention(const uint16_t* qkv, const int32_t* cu, int64_t n_texts, int32_t tok0,
                             int32_t ntok, int32_t max_len, int32_t* win, bool win_ready, int heads, int head_dim,
                             uint16_t* out, cudaStream_t st, const int32_t* d_long, int32_t n_long,
                             const int32_t* long_class_off, int* n_launched) {
  int nl_ = 0;
  if (n_texts <= 0 || ntok <= 0) return cudaSuccess;
  constexpr int HG = ATT_HEADS_PER_CTA;
  if (heads % HG) return cudaErrorInvalidValue;
  const float qscale = 1.4426950408889634f / sqrtf(float(head_dim));
  const int32_t nwin = (ntok + 63) >> 6;
  if (!win_ready)
    window_index_kernel<<<unsigned((n_texts + 1 + 255) / 256), 256, 0, st>>>(cu, n_texts, tok0, ntok, win);
  nl_ += win_ready ? 1 : 2;                           // (window index) + the short-text kernel
#define SURGE_ATT(DH)                                                                                        \
  case DH: {                                                                                                 \
    using TA = TextAtt<DH, HG>;                                                                               \
    static bool attr_##DH = false;                                                                           \
    if (!attr_##DH) {                                                                                        \
      cudaFuncSetAttribute(attention_text_kernel<DH, HG>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                           int(TA::smem(ATT_SHORT)));                                                        \
      attr_##DH = true;                                                                                      \
    }                                                                                                        \
    const dim3 grid(unsigned(nwin), unsigned(heads / HG));                                                    \
    attention_text_kernel<DH, HG><<<grid, TA::WARPS * 32, TA::smem(max_len), st>>>(                           \
        qkv, cu, tok0, ntok, win, heads, out, qscale, TA::rows(max_len));                                    \
    if (max_len > ATT_SHORT && d_long) {                                                                     \
      using LA8 = LongAtt<DH, ATT_LONG_WS>;                                                                  \
      using LA16 = LongAtt<DH, 16>;                                                                          \
      static bool lattr_##DH = false;                                                                        \
      if (!lattr_##DH) {                                                                                     \
        cudaFuncSetAttribute(attention_long_kernel<DH, ATT_LONG_WS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             int(LA8::smem(256)));                                                           \
        cudaFuncSetAttribute(attention_long_kernel<DH, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                             int(LA16::smem(512)));                                                          \
        lattr_##DH = true;                                                                                   \
      }                                                                                                      \
      if (max_len > 512) return cudaErrorInvalidValue;                                                       \
      /* texts of 65..128 tokens keep the mma.sync arithmetic of the fused QKV + attention epilogue (a     \
         text's bits must not depend on its chunk's other texts); longer ones go to tcgen05 (d_h = 64) */   \
      const bool tc_ = attn_long_tc_enabled() && attn_long_tc_supported(DH) && max_len > ATT_TILE_ROWS;     \
      if (n_long > 0 && tc_) {                                                                              \
        cudaError_t e_ = launch_attn_long_tc(qkv, cu, d_long, n_long, tok0, ntok, heads, out, st);            \
        if (e_ != cudaSuccess) return e_;                                                                    \
        nl_ += 2;                                                                                            \
      }                                                                                                      \
      const int top_ = tc_ ? ATT_TILE_ROWS : max_len;                                                        \
      for (int c_ = 0, lo_ = ATT_SHORT; n_long > 0 && lo_ < top_; ++c_) {   /* classes (lo_, hi_] */       \
        const int hi_ = c_ == 0 ? 128 : c_ == 1 ? 192 : c_ == 2 ? 256 : 512;                                \
        const int cap_ = hi_ < top_ ? hi_ : top_;                                                            \
        const int32_t* tl_ = long_class_off ? d_long + long_class_off[c_] : d_long;                          \
        const int32_t nc_ = long_class_off ? long_class_off[c_ + 1] - long_class_off[c_] : n_long;          \
        const dim3 gc_{unsigned(nc_), unsigned(heads), 1u};                                                  \
        if (nc_ > 0 && hi_ <= 256)                                                                           \
          attention_long_kernel<DH, ATT_LONG_WS><<<gc_, ATT_LONG_WS * 32, LA8::smem(cap_), st>>>(              \
              qkv, cu, tl_, tok0, heads, out, qscale, LA8::kv_rows(cap_), lo_, hi_);                           \
        else if (nc_ > 0)                                                                                    \
          attention_long_kernel<DH, 16><<<gc_, 16 * 32, LA16::smem(cap_), st>>>(                               \
              qkv, cu, tl_, tok0, heads, out, qscale, LA16::kv_rows(cap_), lo_, hi_);                          \
        nl_ += nc_ > 0 ? 1 : 0;                                                                              \
        lo_ = hi_;                                                                                           \
      }                                                                                                      \
    } else if (max_len > ATT_SHORT) {   /* list of long texts unknown: scalar per-(text, head) kernel */    \
      constexpr int W1 = AttCfg<DH>::WARPS;                                                                  \
      attention_kernel<DH><<<blocks_for_warps(n_texts * heads, W1), W1 * 32, 0, st>>>(                       \
          qkv, cu, n_texts, tok0, heads, out, qscale, ATT_SHORT + 1);                                        \
      nl_ += 1;                                                                                              \
    }                                                                                                        \
  } break;
  switch (head_dim) {
    SURGE_ATT(16)
    SURGE_ATT(32)
    SURGE_ATT(64)
    default: return cudaErrorInvalidValue;
  }
#undef SURGE_ATT
  if (n_launched) *n_launched = nl_;
  return cudaGetLastError();
}

cudaError_t launch_att_records(const int32_t* tiles, int32_t n_tiles, const int32_t* cu, int32_t tok0,
                               int32_t n_groups, int32_t* rec, cudaStream_t st) {
  if (n_tiles <= 0) return cudaSuccess;
  att_records_kernel<<<blocks_for_warps(n_tiles, 8), 256, 0, st>>>(tiles, n_tiles, cu, tok0, n_groups, rec);
  return cudaGetLastError();
}

cudaError_t launch_window_index(const int32_t* cu, int64_t n_texts, int32_t tok0, int32_t ntok, int32_t* win,
                                cudaStream_t st) {
  if (n_texts <= 0) return cudaSuccess;
  window_index_kernel<<<unsigned((n_texts + 1 + 255) / 256), 256, 0, st>>>(cu, n_texts, tok0, ntok, win);
  return cudaGetLastError();
}

cudaError_t launch_layernorm(const float* v, int64_t rows, int d, const float* gamma, const float* beta, float eps,
                             uint16_t* y, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const unsigned grid = blocks_for_warps(rows, 8);
  switch (d) {
    case 768: layernorm_kernel<768><<<grid, 256, 0, st>>>(v, rows, gamma, beta, eps, y); break;
    case 1024: layernorm_kernel<1024><<<grid, 256, 0, st>>>(v, rows, gamma, beta, eps, y); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_meanpool_l2(const uint16_t* x, const int32_t* cu, int64_t n_texts, int32_t tok0, int d,
                               void* out, cudaStream_t st, int pooling, bool out_bf16) {
  if (n_texts <= 0) return cudaSuccess;
  const unsigned grid = blocks_for_warps(n_texts, 8);
#define SURGE_POOL(DD)                                                                                          \
  case DD:                                                                                                      \
    if (out_bf16) {                                                                                             \
      if (pooling == 1) meanpool_l2_kernel<DD, true, true><<<grid, 256, 0, st>>>(x, cu, n_texts, tok0, out);    \
      else meanpool_l2_kernel<DD, false, true><<<grid, 256, 0, st>>>(x, cu, n_texts, tok0, out);                \
    } else {                                                                                                    \
      if (pooling == 1) meanpool_l2_kernel<DD, true><<<grid, 256, 0, st>>>(x, cu, n_texts, tok0, out);          \
      else meanpool_l2_kernel<DD, false><<<grid, 256, 0, st>>>(x, cu, n_texts, tok0, out);                      \
    }                                                                                                           \
    break;
  switch (d) {
    SURGE_POOL(64)
    SURGE_POOL(384)
    SURGE_POOL(768)
    SURGE_POOL(1024)
    default: return cudaErrorInvalidValue;
  }
#undef SURGE_POOL
  return cudaGetLastError();
}

}  // namespace surge
