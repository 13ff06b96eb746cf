// kernels.cu -- the non-GEMM kernels of the encoder chain (sm_100a):
//   K1 superbatch_pack : exclusive scan of text lengths -> cu_seqlens, partition row/token offsets
//   K3 embed_ln        : X[t] = LN(word[id_t] + pos[t - cu_s] + type[0])
//   K5 varlen_attention: per (text, head) softmax(Q K^T / sqrt(d_h)) V over the text's own tokens
//   K9 meanpool_l2     : e_s = v / max(||v||, 1e-12), v = mean of the text's rows
// All are HBM/L2-bound; accesses are 8- or 16-byte vectors, fp32 math, bf16 storage.
#include "common.cuh"
#include "internal.h"

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
  for (int32_t t = a; t < b; ++t) {
    const int32_t id = ids[t];
    const uint2* wr = reinterpret_cast<const uint2*>(word + size_t(id) * D);
    const uint2* pr = reinterpret_cast<const uint2*>(pos + size_t(t - a) * D);
    float v[PER][4];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int g = lane + 32 * i;
      if (g < G) {
        const uint2 w2 = __ldg(wr + g), p2 = __ldg(pr + g);
        v[i][0] = bf16lo(w2.x) + bf16lo(p2.x) + ty[i][0];
        v[i][1] = bf16hi(w2.x) + bf16hi(p2.x) + ty[i][1];
        v[i][2] = bf16lo(w2.y) + bf16lo(p2.y) + ty[i][2];
        v[i][3] = bf16hi(w2.y) + bf16hi(p2.y) + ty[i][3];
        s += v[i][0] + v[i][1] + v[i][2] + v[i][3];
      } else {
        v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0.f;
      }
    }
    const float mean = warp_sum(s) * (1.0f / D);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int g = lane + 32 * i;
      if (g < G) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float dv = v[i][k] - mean;
          q += dv * dv;
        }
      }
    }
    const float rstd = rsqrtf(warp_sum(q) * (1.0f / D) + eps);
    uint2* xr = reinterpret_cast<uint2*>(x + size_t(t - tok0) * D);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int g = lane + 32 * i;
      if (g < G) {
        float y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) y[k] = (v[i][k] - mean) * rstd * g4[i][k] + b4[i][k];
        xr[g] = make_uint2(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]));
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
  if (len < min_len) return;   // short texts are handled by attention_window_kernel
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

// ------------------------------------------------------- K5 (short texts): window attention
// win[w] = min{s : a_s >= 32 w} for w in [0, nwin], a_s = cu[s] - tok0 (a_n = T): the first
// text starting in 32-token window w.  One thread per text boundary s in [0, n].
__global__ void window_index_kernel(const int32_t* __restrict__ cu, int64_t n, int32_t tok0, int32_t ntok,
                                    int32_t* __restrict__ win) {
  const int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > n) return;
  const int32_t nwin = (ntok + 31) >> 5;
  const int32_t prev = (s == 0) ? -1 : cu[s - 1] - tok0;
  const int32_t a = (s == n) ? ntok : cu[s] - tok0;
  const int32_t w_lo = (prev < 0) ? 0 : (prev >> 5) + 1;
  const int32_t w_hi = (s == n) ? nwin : (a >> 5);
  for (int32_t w = w_lo; w <= w_hi; ++w) win[w] = int32_t(s);
}

// One warp per (32-token window, head) over the texts that START in the window and have
// length <= 32 (their rows lie in [R0, R0 + 64)).  Each lane stages the K/V head slices of its
// rows once into padded fp32 shared memory; lane = query row; online softmax over the text's own
// keys with a lazy rescale (only when the running max grows).  Longer texts: attention_kernel.
template <int DH>
struct WinCfg {
  static constexpr int WARPS = 4;
  static constexpr int LD = DH + 4;   // padded row stride (floats): distinct rows hit distinct banks
  static constexpr int SMEM = 2 * WARPS * 64 * LD * 4;
};

template <int DH, int WARPS = WinCfg<DH>::WARPS>
__global__ void __launch_bounds__(WARPS * 32) attention_window_kernel(
    const uint16_t* __restrict__ qkv, const int32_t* __restrict__ cu, int32_t tok0, int32_t ntok,
    const int32_t* __restrict__ win, int heads, uint16_t* __restrict__ out, float qscale) {
  constexpr int LD = WinCfg<DH>::LD;
  constexpr int V8 = DH / 8;
  extern __shared__ __align__(16) float att_smem[];
  float(*sK)[64][LD] = reinterpret_cast<float(*)[64][LD]>(att_smem);
  float(*sV)[64][LD] = reinterpret_cast<float(*)[64][LD]>(att_smem + WARPS * 64 * LD);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = int64_t(blockIdx.x) * WARPS + w;
  const int32_t nwin = (ntok + 31) >> 5;
  if (gw >= int64_t(nwin) * heads) return;
  const int32_t window = int32_t(gw / heads);
  const int h = int(gw % heads);
  const int32_t s_a = win[window], s_b = win[window + 1];
  const int32_t nb = s_b - s_a;                     // texts starting in this window (<= 32)
  if (nb <= 0) return;
  const int d = heads * DH, ld = 3 * d;
  const int32_t bnd = (lane < nb) ? cu[s_a + lane] - tok0 : 0x7fffffff;   // start of text s_a + lane
  const int32_t R1 = cu[s_b] - tok0;
  const int32_t R0 = __shfl_sync(0xffffffffu, bnd, 0);

  int32_t ts[2], te[2];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int32_t r = R0 + lane + 32 * p;
    int t = -1;
    for (int i = 0; i < nb; ++i) t += (__shfl_sync(0xffffffffu, bnd, i) <= r);
    const int32_t st = __shfl_sync(0xffffffffu, bnd, t < 0 ? 0 : t);
    const int32_t en_n = __shfl_sync(0xffffffffu, bnd, (t + 1) < 32 ? t + 1 : 31);
    const int32_t en = (t + 1 < nb) ? en_n : R1;
    const bool ok = (r < R1) && (en - st <= 32);
    ts[p] = ok ? st - R0 : 0;
    te[p] = ok ? en - R0 : 0;                       // empty range => row not handled here
    if (ok) {
      const size_t base = size_t(r) * ld + h * DH;
      const uint4* kp = reinterpret_cast<const uint4*>(qkv + base + d);
      const uint4* vp = reinterpret_cast<const uint4*>(qkv + base + 2 * d);
      float* kr = &sK[w][lane + 32 * p][0];
      float* vr = &sV[w][lane + 32 * p][0];
#pragma unroll
      for (int v = 0; v < V8; ++v) {
        const uint4 ku = kp[v], vu = vp[v];
        reinterpret_cast<float4*>(kr)[2 * v] = make_float4(bf16lo(ku.x), bf16hi(ku.x), bf16lo(ku.y), bf16hi(ku.y));
        reinterpret_cast<float4*>(kr)[2 * v + 1] = make_float4(bf16lo(ku.z), bf16hi(ku.z), bf16lo(ku.w), bf16hi(ku.w));
        reinterpret_cast<float4*>(vr)[2 * v] = make_float4(bf16lo(vu.x), bf16hi(vu.x), bf16lo(vu.y), bf16hi(vu.y));
        reinterpret_cast<float4*>(vr)[2 * v + 1] = make_float4(bf16lo(vu.z), bf16hi(vu.z), bf16lo(vu.w), bf16hi(vu.w));
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    if (te[p] <= ts[p]) continue;
    const int32_t r = R0 + lane + 32 * p;
    float q[DH];
    {
      const uint4* qp = reinterpret_cast<const uint4*>(qkv + size_t(r) * ld + h * DH);
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
    for (int32_t j = ts[p]; j < te[p]; ++j) {
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
      if (acc > m) {                                 // lazy rescale
        const float corr = exp2f(m - acc);
        l *= corr;
#pragma unroll
        for (int c = 0; c < DH; ++c) o[c] *= corr;
        m = acc;
      }
      const float pj = exp2f(acc - m);
      l += pj;
      const float4* vr = reinterpret_cast<const float4*>(&sV[w][j][0]);
#pragma unroll
      for (int c = 0; c < DH / 4; ++c) {
        const float4 v4 = vr[c];
        o[4 * c] = fmaf(pj, v4.x, o[4 * c]);
        o[4 * c + 1] = fmaf(pj, v4.y, o[4 * c + 1]);
        o[4 * c + 2] = fmaf(pj, v4.z, o[4 * c + 2]);
        o[4 * c + 3] = fmaf(pj, v4.w, o[4 * c + 3]);
      }
    }
    const float inv = 1.0f / l;
    uint4* op = reinterpret_cast<uint4*>(out + size_t(r) * d + h * DH);
#pragma unroll
    for (int v = 0; v < V8; ++v) {
      op[v] = make_uint4(pack_bf16x2(o[v * 8 + 0] * inv, o[v * 8 + 1] * inv),
                         pack_bf16x2(o[v * 8 + 2] * inv, o[v * 8 + 3] * inv),
                         pack_bf16x2(o[v * 8 + 4] * inv, o[v * 8 + 5] * inv),
                         pack_bf16x2(o[v * 8 + 6] * inv, o[v * 8 + 7] * inv));
    }
  }
}

// ----------------------------------------------------------------------------- K9 meanpool + L2
template <int D>
__global__ void __launch_bounds__(256) meanpool_l2_kernel(const uint16_t* __restrict__ x,
                                                          const int32_t* __restrict__ cu, int64_t n_texts,
                                                          int32_t tok0, float* __restrict__ out) {
  constexpr int G = D / 4;
  constexpr int PER = (G + 31) / 32;
  const int64_t text = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (text >= n_texts) return;
  const int32_t a = cu[text] - tok0, b = cu[text + 1] - tok0;
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
  float4* orow = reinterpret_cast<float4*>(out + size_t(text) * D);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int g = lane + 32 * i;
    if (g < G) orow[g] = make_float4(acc[i][0] * inv, acc[i][1] * inv, acc[i][2] * inv, acc[i][3] * inv);
  }
}

__global__ void bf16_to_f32_kernel(const uint16_t* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = bf16f(in[i]);
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

cudaError_t launch_pack(const int32_t* lengths, int64_t n, const int32_t* sizes, int64_t m, int32_t* cu,
                        int32_t* row_off, int32_t* tok_off, cudaStream_t st) {
  pack_kernel<<<1, PACK_THREADS, 0, st>>>(lengths, n, sizes, m, cu, row_off, tok_off);
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
                             uint16_t* out, cudaStream_t st) {
  if (n_texts <= 0) return cudaSuccess;
  const float qscale = 1.4426950408889634f / sqrtf(float(head_dim));
  const int32_t nwin = (ntok + 31) >> 5;
  if (!win_ready) {
    window_index_kernel<<<unsigned((n_texts + 1 + 255) / 256), 256, 0, st>>>(cu, n_texts, tok0, ntok, win);
  }
#define SURGE_ATT(DH)                                                                                        \
  case DH: {                                                                                                 \
    constexpr int W = WinCfg<DH>::WARPS;                                                                     \
    static bool attr_##DH = false;                                                                           \
    if (!attr_##DH) {                                                                                        \
      cudaFuncSetAttribute(attention_window_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                           WinCfg<DH>::SMEM);                                                                \
      attr_##DH = true;                                                                                      \
    }                                                                                                        \
    attention_window_kernel<DH><<<blocks_for_warps(int64_t(nwin) * heads, W), W * 32, WinCfg<DH>::SMEM, st>>>( \
        qkv, cu, tok0, ntok, win, heads, out, qscale);                                                       \
    if (max_len > 32) {                                                                                      \
      constexpr int W1 = AttCfg<DH>::WARPS;                                                                  \
      attention_kernel<DH><<<blocks_for_warps(n_texts * heads, W1), W1 * 32, 0, st>>>(qkv, cu, n_texts, tok0, \
                                                                                      heads, out, qscale, 33); \
    }                                                                                                        \
  } break;
  switch (head_dim) {
    SURGE_ATT(16)
    SURGE_ATT(32)
    SURGE_ATT(64)
    default: return cudaErrorInvalidValue;
  }
#undef SURGE_ATT
  return cudaGetLastError();
}

cudaError_t launch_window_index(const int32_t* cu, int64_t n_texts, int32_t tok0, int32_t ntok, int32_t* win,
                                cudaStream_t st) {
  if (n_texts <= 0) return cudaSuccess;
  window_index_kernel<<<unsigned((n_texts + 1 + 255) / 256), 256, 0, st>>>(cu, n_texts, tok0, ntok, win);
  return cudaGetLastError();
}

cudaError_t launch_meanpool_l2(const uint16_t* x, const int32_t* cu, int64_t n_texts, int32_t tok0, int d,
                               float* out, cudaStream_t st) {
  if (n_texts <= 0) return cudaSuccess;
  const unsigned grid = blocks_for_warps(n_texts, 8);
  switch (d) {
    case 64: meanpool_l2_kernel<64><<<grid, 256, 0, st>>>(x, cu, n_texts, tok0, out); break;
    case 384: meanpool_l2_kernel<384><<<grid, 256, 0, st>>>(x, cu, n_texts, tok0, out); break;
    case 768: meanpool_l2_kernel<768><<<grid, 256, 0, st>>>(x, cu, n_texts, tok0, out); break;
    case 1024: meanpool_l2_kernel<1024><<<grid, 256, 0, st>>>(x, cu, n_texts, tok0, out); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace surge
