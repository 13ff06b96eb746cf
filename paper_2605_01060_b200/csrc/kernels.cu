// kernels.cu -- the non-GEMM kernels of the encoder chain (sm_100a):
//   K1 superbatch_pack : exclusive scan of text lengths -> cu_seqlens, partition row/token offsets
//   K3 embed_ln        : X[t] = LN(word[id_t] + pos[t - cu_s] + type[0])
//   K5 varlen_attention: per (text, head) softmax(Q K^T / sqrt(d_h)) V over the text's own tokens
//   K9 meanpool_l2     : e_s = v / max(||v||, 1e-12), v = mean of the text's rows
// All are HBM/L2-bound; accesses are 8- or 16-byte vectors, fp32 math, bf16 storage.
#include "common.cuh"
#include "internal.h"

#include <climits>

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
  if (len < min_len) return;   // short texts are handled by attention_tile_kernel
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
// seg[t] = (first, end) token of the text containing token t (chunk-local).  One warp per text.
__global__ void seg_kernel(const int32_t* __restrict__ cu, int64_t n, int32_t tok0, int2* __restrict__ seg) {
  const int64_t text = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (text >= n) return;
  const int32_t a = cu[text] - tok0, b = cu[text + 1] - tok0;
  const int2 v = make_int2(a, b);
  for (int32_t t = a + lane; t < b; t += 32) seg[t] = v;
}

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

// Block-diagonal varlen attention for texts of <= ATT_SHORT tokens.  A CTA owns query rows
// [r0, r0 + ROWS) and a group of HG heads; it stages those Q rows and the K/V rows of every text
// that intersects them ([k0, k1), at most ROWS + 2 (L - 1) rows) in padded shared memory with
// cp.async, then each warp computes 16 query rows: S = Q K^T and O = P V on mma.sync m16n8k16
// (bf16 in, fp32 accumulate; P split hi+lo bf16), 16-key blocks aligned to text starts over the warp's texts only, with the text mask
// (key j valid for query i iff j lies in i's text), flash-style online softmax in exp2 form.
// O is staged back into the Q tile and written with 16-byte stores.  Rows of longer texts are
// left to attention_kernel.
constexpr int ATT_SHORT = 64;

template <int DH, int HG>
struct TileAtt {
  static constexpr int ROWS = 64;                // query rows per CTA
  static constexpr int WARPS = ROWS / 16;
  static constexpr int COLS = HG * DH;           // columns of one Q / K / V slice
  static constexpr int LDS = COLS + 8;           // smem row stride (bf16): 16-byte skew per row
  static constexpr int CH = COLS / 8;            // 16-byte chunks per row
  static int kcap(int max_len) {                 // K/V rows staged (+16 zero rows for the last step)
    const int L = max_len < ATT_SHORT ? (max_len < 1 ? 1 : max_len) : ATT_SHORT;
    return ((ROWS + 2 * (L - 1) + 16 + 7) / 8) * 8;
  }
  static size_t smem(int max_len) { return size_t(ROWS + 2 * kcap(max_len)) * LDS * 2; }
};

template <int DH, int HG>
__global__ void __launch_bounds__(TileAtt<DH, HG>::WARPS * 32) attention_tile_kernel(
    const uint16_t* __restrict__ qkv, const int2* __restrict__ seg, int32_t ntok, int heads,
    uint16_t* __restrict__ out, float qscale, int kcap) {
  using A = TileAtt<DH, HG>;
  constexpr int ROWS = A::ROWS, LDS = A::LDS, CH = A::CH;
  extern __shared__ __align__(16) uint16_t att_sm[];
  uint16_t* sQ = att_sm;                         // [ROWS][LDS]  (Q, then O)
  uint16_t* sK = sQ + ROWS * LDS;                // [kcap][LDS]
  uint16_t* sV = sK + kcap * LDS;                // [kcap][LDS]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int d = heads * DH, ld = 3 * d;
  const int32_t r0 = blockIdx.x * ROWS;
  const int col0 = blockIdx.y * A::COLS;
  const int32_t r_end = min(r0 + ROWS, ntok);    // query rows [r0, r_end)
  const int2 sa = seg[r0], sb = seg[r_end - 1];
  const int32_t k0 = (sa.y - sa.x <= ATT_SHORT) ? sa.x : r0;
  const int32_t k1 = (sb.y - sb.x <= ATT_SHORT) ? sb.y : r_end;
  const int nq = r_end - r0, nk = k1 - k0;

  for (int i = tid; i < nq * CH; i += blockDim.x) {
    const int r = i / CH, c = i - r * CH;
    cp_async16(sQ + r * LDS + c * 8, qkv + size_t(r0 + r) * ld + col0 + c * 8);
  }
  for (int i = tid; i < nk * CH; i += blockDim.x) {
    const int r = i / CH, c = i - r * CH;
    const uint16_t* g = qkv + size_t(k0 + r) * ld + col0 + c * 8;
    cp_async16(sK + r * LDS + c * 8, g + d);
    cp_async16(sV + r * LDS + c * 8, g + 2 * d);
  }
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int i = tid; i < 16 * CH; i += blockDim.x) {   // zero rows after the span (masked, must be finite)
    const int r = nk + i / CH, c = i % CH;
    *reinterpret_cast<uint4*>(sK + r * LDS + c * 8) = z;
    *reinterpret_cast<uint4*>(sV + r * LDS + c * 8) = z;
  }
  for (int i = tid; i < (ROWS - nq) * CH; i += blockDim.x) {
    const int r = nq + i / CH, c = i % CH;
    *reinterpret_cast<uint4*>(sQ + r * LDS + c * 8) = z;
  }
  cp_async_wait_all();
  __syncthreads();

  const int g = lane >> 2, c4 = lane & 3;
  const int32_t qr = r0 + warp * 16;             // first query row of this warp
  const int32_t ra = qr + g, rb = qr + g + 8;
  int2 ta = make_int2(0, 0), tb = make_int2(0, 0);
  if (ra < r_end) ta = seg[ra];
  if (rb < r_end) tb = seg[rb];
  const bool va = ra < r_end && ta.y - ta.x <= ATT_SHORT;
  const bool vb = rb < r_end && tb.y - tb.x <= ATT_SHORT;
  if (!va) ta = make_int2(-1, -1);   // never matches a text start: the row takes no keys
  if (!vb) tb = make_int2(-1, -1);
  int32_t kw0 = min(va ? ta.x : INT_MAX, vb ? tb.x : INT_MAX);
  int32_t kw1 = max(va ? ta.y : INT_MIN, vb ? tb.y : INT_MIN);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    kw0 = min(kw0, __shfl_xor_sync(0xffffffffu, kw0, o));
    kw1 = max(kw1, __shfl_xor_sync(0xffffffffu, kw1, o));
  }
  if (kw0 < kw1) {
    const uint32_t q_base = smem_u32(sQ + (warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + (lane >> 4) * 8);
#pragma unroll 1
    for (int h = 0; h < HG; ++h) {
      uint32_t qa[DH / 16][4];
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk)
        ldsm_x4(q_base + (h * DH + kk * 16) * 2, qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
      float o[DH / 8][4];
#pragma unroll
      for (int n = 0; n < DH / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
      float ma = -INFINITY, mb = -INFINITY, la = 0.f, lb = 0.f;
      // Key blocks are aligned to each text's first token and visited text by text, so every
      // query row sees exactly the same 16-key blocks (other texts' blocks contribute exact zeros
      // and unit rescales) wherever its text sits in the stream: bit-exact SuperBatch invariance.
      int32_t t_beg = kw0, t_end = kw0, kb = kw0;
#pragma unroll 1
      for (;;) {
        if (kb >= t_end) {                         // next text
          if (t_end >= kw1) break;
          const int2 tx = seg[t_end];
          t_beg = tx.x;
          t_end = tx.y;
          kb = t_beg;
          if (t_end - t_beg > ATT_SHORT) {         // long text: its rows belong to attention_kernel
            kb = t_end;
            continue;
          }
        }
        const int kr = kb - k0;                    // smem row of key kb
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t k_addr =
            smem_u32(sK + (kr + (lane & 7) + ((lane >> 4) & 1) * 8) * LDS + h * DH + ((lane >> 3) & 1) * 8);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          uint32_t b00, b01, b10, b11;
          ldsm_x4(k_addr + kk * 32, b00, b01, b10, b11);
          mma_bf16_16816(s0, qa[kk], b00, b01);
          mma_bf16_16816(s1, qa[kk], b10, b11);
        }
        // scale + text mask: only rows of the current text [t_beg, t_end) take keys from this block
        // (keys kb + 2c4 + {0,1} in s0, kb + 8 + 2c4 + {0,1} in s1; all >= t_beg by construction)
        const int32_t j0 = kb + 2 * c4, j1 = j0 + 1, j2 = j0 + 8, j3 = j0 + 9;
        const int32_t ea = (ta.x == t_beg) ? t_end : INT_MIN, eb = (tb.x == t_beg) ? t_end : INT_MIN;
        float pa[4], pb[4];
        pa[0] = j0 < ea ? s0[0] * qscale : -INFINITY;
        pa[1] = j1 < ea ? s0[1] * qscale : -INFINITY;
        pa[2] = j2 < ea ? s1[0] * qscale : -INFINITY;
        pa[3] = j3 < ea ? s1[1] * qscale : -INFINITY;
        pb[0] = j0 < eb ? s0[2] * qscale : -INFINITY;
        pb[1] = j1 < eb ? s0[3] * qscale : -INFINITY;
        pb[2] = j2 < eb ? s1[2] * qscale : -INFINITY;
        pb[3] = j3 < eb ? s1[3] * qscale : -INFINITY;
        float xa = fmaxf(fmaxf(pa[0], pa[1]), fmaxf(pa[2], pa[3]));
        float xb = fmaxf(fmaxf(pb[0], pb[1]), fmaxf(pb[2], pb[3]));
        xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 1));
        xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 2));
        xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 1));
        xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 2));
        const float na = fmaxf(ma, xa), nb = fmaxf(mb, xb);
        const float ua = (na == -INFINITY) ? 0.f : na, ub = (nb == -INFINITY) ? 0.f : nb;
        const float ca = exp2f(ma - ua), cb = exp2f(mb - ub);
        ma = na;
        mb = nb;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          pa[i] = exp2f(pa[i] - ua);
          pb[i] = exp2f(pb[i] - ub);
        }
        la = la * ca + (pa[0] + pa[1] + pa[2] + pa[3]);
        lb = lb * cb + (pb[0] + pb[1] + pb[2] + pb[3]);
#pragma unroll
        for (int n = 0; n < DH / 8; ++n) {
          o[n][0] *= ca; o[n][1] *= ca;
          o[n][2] *= cb; o[n][3] *= cb;
        }
        // P = P_hi + P_lo, both bf16 (two MMAs): P·V keeps ~16 mantissa bits of P
        const uint32_t pf[4] = {pack_bf16x2(pa[0], pa[1]), pack_bf16x2(pb[0], pb[1]), pack_bf16x2(pa[2], pa[3]),
                                pack_bf16x2(pb[2], pb[3])};
        const uint32_t pl[4] = {pack_bf16x2(pa[0] - bf16lo(pf[0]), pa[1] - bf16hi(pf[0])),
                                pack_bf16x2(pb[0] - bf16lo(pf[1]), pb[1] - bf16hi(pf[1])),
                                pack_bf16x2(pa[2] - bf16lo(pf[2]), pa[3] - bf16hi(pf[2])),
                                pack_bf16x2(pb[2] - bf16lo(pf[3]), pb[3] - bf16hi(pf[3]))};
        const uint32_t v_addr =
            smem_u32(sV + (kr + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + h * DH + (lane >> 4) * 8);
#pragma unroll
        for (int n = 0; n < DH / 16; ++n) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(v_addr + n * 32, b0, b1, b2, b3);
          mma_bf16_16816(o[2 * n], pf, b0, b1);
          mma_bf16_16816(o[2 * n + 1], pf, b2, b3);
          mma_bf16_16816(o[2 * n], pl, b0, b1);
          mma_bf16_16816(o[2 * n + 1], pl, b2, b3);
        }
        kb += 16;
      }
      la += __shfl_xor_sync(0xffffffffu, la, 1);
      la += __shfl_xor_sync(0xffffffffu, la, 2);
      lb += __shfl_xor_sync(0xffffffffu, lb, 1);
      lb += __shfl_xor_sync(0xffffffffu, lb, 2);
      const float ia = la > 0.f ? 1.0f / la : 0.f, ib = lb > 0.f ? 1.0f / lb : 0.f;
      __syncwarp();   // every lane has read its Q fragments of head h before they are overwritten
      uint16_t* oa = sQ + (warp * 16 + g) * LDS + h * DH + 2 * c4;
#pragma unroll
      for (int n = 0; n < DH / 8; ++n) {
        *reinterpret_cast<uint32_t*>(oa + n * 8) = pack_bf16x2(o[n][0] * ia, o[n][1] * ia);
        *reinterpret_cast<uint32_t*>(oa + 8 * LDS + n * 8) = pack_bf16x2(o[n][2] * ib, o[n][3] * ib);
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < nq * CH; i += blockDim.x) {
    const int r = i / CH, c = i - r * CH;
    const int2 t = seg[r0 + r];
    if (t.y - t.x <= ATT_SHORT)
      *reinterpret_cast<uint4*>(out + size_t(r0 + r) * d + col0 + c * 8) =
          *reinterpret_cast<const uint4*>(sQ + r * LDS + c * 8);
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
                             int32_t ntok, int32_t max_len, int32_t* seg, bool seg_ready, int heads, int head_dim,
                             uint16_t* out, cudaStream_t st) {
  if (n_texts <= 0 || ntok <= 0) return cudaSuccess;
  if (heads % 2) return cudaErrorInvalidValue;
  const float qscale = 1.4426950408889634f / sqrtf(float(head_dim));
  int2* sg = reinterpret_cast<int2*>(seg);
  if (!seg_ready) seg_kernel<<<blocks_for_warps(n_texts, 8), 256, 0, st>>>(cu, n_texts, tok0, sg);
#define SURGE_ATT(DH)                                                                                        \
  case DH: {                                                                                                 \
    using TA = TileAtt<DH, 2>;                                                                               \
    static int attr_##DH = 0;                                                                                \
    const size_t sm = TA::smem(max_len);                                                                     \
    if (attr_##DH < int(sm)) {                                                                               \
      cudaFuncSetAttribute(attention_tile_kernel<DH, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                           int(TA::smem(ATT_SHORT)));                                                        \
      attr_##DH = int(TA::smem(ATT_SHORT));                                                                  \
    }                                                                                                        \
    const dim3 grid(unsigned((ntok + TA::ROWS - 1) / TA::ROWS), unsigned(heads / 2));                        \
    attention_tile_kernel<DH, 2><<<grid, TA::WARPS * 32, sm, st>>>(qkv, sg, ntok, heads, out, qscale,        \
                                                                   TA::kcap(max_len));                       \
    if (max_len > ATT_SHORT) {                                                                               \
      constexpr int W1 = AttCfg<DH>::WARPS;                                                                  \
      attention_kernel<DH><<<blocks_for_warps(n_texts * heads, W1), W1 * 32, 0, st>>>(                       \
          qkv, cu, n_texts, tok0, heads, out, qscale, ATT_SHORT + 1);                                        \
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

cudaError_t launch_seg(const int32_t* cu, int64_t n_texts, int32_t tok0, int32_t* seg, cudaStream_t st) {
  if (n_texts <= 0) return cudaSuccess;
  seg_kernel<<<blocks_for_warps(n_texts, 8), 256, 0, st>>>(cu, n_texts, tok0, reinterpret_cast<int2*>(seg));
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
