// model.cu -- device-resident BERT-class encoder (weights + chunked encoder chain).
//
// Per chunk of whole texts (<= Workspace::cap tokens), the chain is:
//   K3 embed+LN -> L x [ K4 QKV GEMM(+bias) -> K5 varlen attention -> K6 out-proj GEMM(+bias+res+LN)
//                        -> K7 FFN1 GEMM(+bias+GELU) -> K8 FFN2 GEMM(+bias+res+LN) ] -> K9 meanpool+L2
// Activations are bf16 in HBM between kernels; all math is fp32 inside the kernels.
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.h"

namespace surge {

size_t blob_elems(const ModelShape& s) {
  const size_t d = s.d, f = s.ffn;
  size_t n = size_t(s.vocab + s.max_pos + s.type_vocab) * d + 2 * d;
  n += size_t(s.layers) * (4 * (d * d + d) + 2 * d + (f * d + f) + (d * f + d) + 2 * d);
  return n;
}

cudaError_t Workspace::alloc(const ModelShape& s, int64_t cap_tokens) {
  release();
  const size_t t = size_t(cap_tokens);
  cudaError_t e;
  if ((e = cudaMalloc(&X, t * s.d * 2)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&QKV, t * 3 * s.d * 2)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&O, t * s.d * 2)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&X1, t * s.d * 2)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&H, t * s.ffn * 2)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&win, (t / 64 + 2) * sizeof(int32_t))) != cudaSuccess) return e;
  if (!fused_ln(s.d) && (e = cudaMalloc(&V, t * s.d * 4)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&long_idx, (t / 65 + 1) * sizeof(int32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&tiles, (att_max_tiles(cap_tokens) + 1) * sizeof(int32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&att_rec, att_max_tiles(cap_tokens) * ATT_REC_INTS * sizeof(int32_t))) != cudaSuccess) return e;
  cap = cap_tokens;
  return cudaSuccess;
}

int32_t* PinnedRing::acquire(size_t n, int* slot) {
  const int j = next;
  next = (next + 1) % NS;
  if (ev[j]) cudaEventSynchronize(ev[j]);   // the slot's previous copy has run
  else if (cudaEventCreateWithFlags(&ev[j], cudaEventDisableTiming) != cudaSuccess) return nullptr;
  if (cap[j] < n) {
    if (buf[j]) cudaFreeHost(buf[j]);
    buf[j] = nullptr;
    const size_t c = n < 4096 ? 4096 : 2 * n;
    if (cudaHostAlloc(reinterpret_cast<void**>(&buf[j]), c * sizeof(int32_t), cudaHostAllocPortable) != cudaSuccess) {
      cap[j] = 0;
      return nullptr;
    }
    cap[j] = c;
  }
  *slot = j;
  return buf[j];
}

cudaError_t PinnedRing::copy(int slot, int32_t* dst, size_t n, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(dst, buf[slot], n * sizeof(int32_t), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  return cudaEventRecord(ev[slot], st);
}

cudaError_t PinnedRing::upload(int32_t* dst, const int32_t* src, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int slot = 0;
  int32_t* h = acquire(n, &slot);
  if (!h) return cudaErrorMemoryAllocation;
  std::memcpy(h, src, n * sizeof(int32_t));
  return copy(slot, dst, n, st);
}

void PinnedRing::release() {
  for (int j = 0; j < NS; ++j) {
    if (ev[j]) {
      cudaEventSynchronize(ev[j]);
      cudaEventDestroy(ev[j]);
    }
    if (buf[j]) cudaFreeHost(buf[j]);
    ev[j] = nullptr;
    buf[j] = nullptr;
    cap[j] = 0;
  }
}

void Workspace::release() {
  for (uint16_t** p : {&X, &QKV, &O, &X1, &H}) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  if (win) cudaFree(win);
  win = nullptr;
  if (V) cudaFree(V);
  V = nullptr;
  if (long_idx) cudaFree(long_idx);
  long_idx = nullptr;
  if (tiles) cudaFree(tiles);
  tiles = nullptr;
  if (att_rec) cudaFree(att_rec);
  att_rec = nullptr;
  cap = 0;
}

int32_t att_tiles_for(const int32_t* host_cu, int64_t s0, int64_t s1, std::vector<int32_t>& out) {
  int32_t n = 0;
  int64_t s = s0;
  while (s < s1) {
    if (host_cu[s + 1] - host_cu[s] > ATT_TILE_ROWS) return -1;
    out.push_back(int32_t(s));
    ++n;
    int64_t e = s + 1;
    while (e < s1 && host_cu[e + 1] - host_cu[s] <= ATT_TILE_ROWS) ++e;
    s = e;
  }
  if (n & 1) {   // empty tile: zero rows, starts at the chunk's end
    out.push_back(int32_t(s1));
    ++n;
  }
  out.push_back(int32_t(s1));
  return n;
}

DeviceModel::~DeviceModel() {
  for (void* p : allocs_) cudaFree(p);
}

cudaError_t DeviceModel::dalloc(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess) allocs_.push_back(*p);
  return e;
}

#define SURGE_TRY(x)                   \
  do {                                 \
    cudaError_t _e = (x);              \
    if (_e != cudaSuccess) return _e;  \
  } while (0)

cudaError_t DeviceModel::init(const ModelShape& s, const uint16_t* blob, bool blob_on_device, cudaStream_t st) {
  s_ = s;
  const size_t n = blob_elems(s);
  uint16_t* dblob = nullptr;
  SURGE_TRY(cudaMalloc(&dblob, n * 2));
  cudaError_t e = cudaMemcpyAsync(dblob, blob, n * 2, blob_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) { cudaFree(dblob); return e; }

  size_t off = 0;
  // copy a bf16 tensor of `cnt` elements out of the blob into its own allocation
  auto take_bf16 = [&](uint16_t** dst, size_t cnt) -> cudaError_t {
    SURGE_TRY(dalloc(reinterpret_cast<void**>(dst), cnt * 2));
    SURGE_TRY(cudaMemcpyAsync(*dst, dblob + off, cnt * 2, cudaMemcpyDeviceToDevice, st));
    off += cnt;
    return cudaSuccess;
  };
  auto take_f32 = [&](float** dst, size_t cnt) -> cudaError_t {
    SURGE_TRY(dalloc(reinterpret_cast<void**>(dst), cnt * 4));
    SURGE_TRY(launch_bf16_to_f32(dblob + off, *dst, int64_t(cnt), st));
    off += cnt;
    return cudaSuccess;
  };
  const size_t d = s.d, f = s.ffn;
  e = [&]() -> cudaError_t {
    SURGE_TRY(take_bf16(&word_, size_t(s.vocab) * d));
    SURGE_TRY(take_bf16(&pos_, size_t(s.max_pos) * d));
    SURGE_TRY(take_bf16(&type_, size_t(s.type_vocab) * d));
    SURGE_TRY(take_f32(&emb_g_, d));
    SURGE_TRY(take_f32(&emb_b_, d));
    layers_.resize(s.layers);
    for (int l = 0; l < s.layers; ++l) {
      LayerW& L = layers_[l];
      // Q, K, V weights are separated by their biases in the blob -> gather into [3d x d] / [3d]
      SURGE_TRY(dalloc(reinterpret_cast<void**>(&L.wqkv), 3 * d * d * 2));
      SURGE_TRY(dalloc(reinterpret_cast<void**>(&L.bqkv), 3 * d * 4));
      for (int j = 0; j < 3; ++j) {
        SURGE_TRY(cudaMemcpyAsync(L.wqkv + j * d * d, dblob + off, d * d * 2, cudaMemcpyDeviceToDevice, st));
        off += d * d;
        SURGE_TRY(launch_bf16_to_f32(dblob + off, L.bqkv + j * d, int64_t(d), st));
        off += d;
      }
      SURGE_TRY(take_bf16(&L.wo, d * d));
      SURGE_TRY(take_f32(&L.bo, d));
      SURGE_TRY(take_f32(&L.ln1_g, d));
      SURGE_TRY(take_f32(&L.ln1_b, d));
      SURGE_TRY(take_bf16(&L.w1, f * d));
      SURGE_TRY(take_f32(&L.b1, f));
      SURGE_TRY(take_bf16(&L.w2, d * f));
      SURGE_TRY(take_f32(&L.b2, d));
      SURGE_TRY(take_f32(&L.ln2_g, d));
      SURGE_TRY(take_f32(&L.ln2_b, d));
      SURGE_TRY(make_tmap_bf16(&L.tm_wqkv, L.wqkv, 3 * d, d, gemm_b_box_rows(int(3 * d), int(d), EPI_BIAS)));
      if (qkv_att_supported(int(d), s.heads)) {
        // head-complete slices: slice j = [Q | K | V] rows of heads j*HG .. j*HG + HG - 1
        const size_t dh = d / s.heads, hg = ATT_SLICE / (3 * dh);
        SURGE_TRY(dalloc(reinterpret_cast<void**>(&L.wqkv_att), 3 * d * d * 2));
        SURGE_TRY(dalloc(reinterpret_cast<void**>(&L.bqkv_att), 3 * d * 4));
        size_t row = 0;
        for (size_t j = 0; j < size_t(s.heads) / hg; ++j)
          for (size_t part = 0; part < 3; ++part)
            for (size_t hh = 0; hh < hg; ++hh, row += dh) {
              const size_t src = part * d + (j * hg + hh) * dh;
              SURGE_TRY(cudaMemcpyAsync(L.wqkv_att + row * d, L.wqkv + src * d, dh * d * 2, cudaMemcpyDeviceToDevice, st));
              SURGE_TRY(cudaMemcpyAsync(L.bqkv_att + row, L.bqkv + src, dh * 4, cudaMemcpyDeviceToDevice, st));
            }
        SURGE_TRY(make_tmap_bf16(&L.tm_wqkv_att, L.wqkv_att, 3 * d, d, gemm_b_box_rows(int(3 * d), int(d), EPI_QKV_ATTN)));
      }
      const int ln_epi = fused_ln(int(d)) ? EPI_BIAS_LN : EPI_BIAS_RES;
      SURGE_TRY(make_tmap_bf16(&L.tm_wo, L.wo, d, d, gemm_b_box_rows(int(d), int(d), ln_epi)));
      SURGE_TRY(make_tmap_bf16(&L.tm_w1, L.w1, f, d, gemm_b_box_rows(int(f), int(d), EPI_BIAS_GELU)));
      SURGE_TRY(make_tmap_bf16(&L.tm_w2, L.w2, d, f, gemm_b_box_rows(int(d), int(f), ln_epi)));
      if (ln_pair_supported(int(d), int(d))) {
        if (LN_PAIR_KB == 32) {          // 32-wide k-blocks, 128-row B boxes (ln_pair.cu)
          SURGE_TRY(make_tmap_bf16_k32(&L.tm_wo_p64, L.wo, d, d, 128));
          SURGE_TRY(make_tmap_bf16_k32(&L.tm_w2_p64, L.w2, d, f, 128));
        } else {
          const uint32_t bb = LN_PAIR_BBOX64 ? LN_PAIR_BBOX64 : uint32_t(d / 4);   // = the kernel's BNC / 2
          SURGE_TRY(make_tmap_bf16(&L.tm_wo_p64, L.wo, d, d, bb));
          SURGE_TRY(make_tmap_bf16(&L.tm_w2_p64, L.w2, d, f, bb));
        }
      }
      if (mlp_fused_supported(int(d), int(f))) {
        SURGE_TRY(make_tmap_bf16(&L.tm_wo_mlp, L.wo, d, d, mlp_w2_box_rows(int(d))));
        SURGE_TRY(make_tmap_bf16(&L.tm_w1_mlp, L.w1, f, d, 64));
        SURGE_TRY(make_tmap_bf16(&L.tm_wo64, L.wo, d, d, 64));
        SURGE_TRY(make_tmap_bf16(&L.tm_w2_mlp, L.w2, d, f, mlp_w2_box_rows(int(d))));
      }
    }
    return cudaSuccess;
  }();
  cudaError_t e2 = cudaStreamSynchronize(st);
  cudaFree(dblob);
  if (e != cudaSuccess) return e;
  if (off != n) return cudaErrorInvalidValue;
  if (e2 != cudaSuccess) return e2;
  // host copies of the LayerNorm constants: a kernel parameter of the fused tail (mlp_tc.cu MLP_LN_CPARAM)
  for (LayerW& L : layers_) {
    L.ln_host.resize(6 * d);
    const float* src[6] = {L.bo, L.ln1_g, L.ln1_b, L.b2, L.ln2_g, L.ln2_b};
    for (int i = 0; i < 6; ++i) SURGE_TRY(cudaMemcpy(L.ln_host.data() + i * d, src[i], d * 4, cudaMemcpyDeviceToHost));
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------------------ profiler
cudaEvent_t Profiler::take() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
void Profiler::begin(cudaStream_t st, cudaEvent_t* a) {
  *a = nullptr;
  if (!on) return;
  *a = take();
  cudaEventRecord(*a, st);
}
void Profiler::end(int kind, cudaStream_t st, cudaEvent_t a, double fl, double by) {
  if (!on || !a) return;
  cudaEvent_t b = take();
  cudaEventRecord(b, st);
  recs.push_back({kind, a, b, fl, by});
}
cudaError_t Profiler::resolve() {
  for (const Rec& r : recs) {
    float t = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return e;
    e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess) return e;
    launches[r.kind] += 1;
    ms[r.kind] += t;
    flops[r.kind] += r.fl;
    bytes[r.kind] += r.by;
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  recs.clear();
  return cudaSuccess;
}
void Profiler::clear() {
  for (const Rec& r : recs) {
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  recs.clear();
  for (int k = 0; k < KK_COUNT; ++k) {
    launches[k] = 0;
    ms[k] = flops[k] = bytes[k] = 0;
  }
}
Profiler::~Profiler() {
  for (const Rec& r : recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

cudaError_t DeviceModel::encode_chunk(Workspace& ws, const int32_t* d_ids, const int32_t* d_cu, int64_t s0,
                                      int64_t s1, int32_t tok0, int32_t ntok, void* d_out, cudaStream_t st,
                                      int64_t* launches, Profiler* prof, const int32_t* host_cu) const {
  const int64_t n = s1 - s0;
  if (n <= 0) return cudaSuccess;
  if (ntok > ws.cap) return cudaErrorInvalidValue;
  const int d = s_.d, f = s_.ffn;
  const int32_t* cu = d_cu + s0;
  CUtensorMap tmX, tmO, tmX1, tmH;            // GEMM A operands (loads)
  CUtensorMap smX, smQKV, smX1, smH;          // GEMM outputs (epilogue TMA stores)
  SURGE_TRY(make_tmap_bf16(&tmX, ws.X, ntok, d, 128));
  SURGE_TRY(make_tmap_bf16(&tmO, ws.O, ntok, d, 128));
  SURGE_TRY(make_tmap_bf16(&tmX1, ws.X1, ntok, d, 128));
  SURGE_TRY(make_tmap_bf16(&tmH, ws.H, ntok, f, 128));
  CUtensorMap tmO32, tmH32;                   // the cluster-pair LN GEMMs' A operands (LN_PAIR_KB = 32)
  const bool kb32 = LN_PAIR_KB == 32 && ln_pair_ && ln_pair_supported(d, d);
  if (kb32) {
    SURGE_TRY(make_tmap_bf16_k32(&tmO32, ws.O, ntok, d, 128));
    SURGE_TRY(make_tmap_bf16_k32(&tmH32, ws.H, ntok, f, 128));
  }
  SURGE_TRY(make_tmap_store_bf16(&smX, ws.X, ntok, d));
  SURGE_TRY(make_tmap_store_bf16(&smQKV, ws.QKV, ntok, 3 * d));
  SURGE_TRY(make_tmap_store_bf16(&smX1, ws.X1, ntok, d));
  SURGE_TRY(make_tmap_store_bf16(&smH, ws.H, ntok, f));
  const bool P = prof && prof->on;
  double sum_l2 = 0;
  int32_t max_len = s_.max_pos;     // unknown -> assume long texts may be present
  std::vector<int32_t> long_texts;    // chunk-relative indices of texts longer than 64 tokens (by length class)
  int32_t long_off[ATT_LONG_CLASSES + 1] = {0, 0, 0, 0, 0};
  // fused QKV + attention (EPI_QKV_ATTN) when every text of the chunk fits one 128-row tile
  std::vector<int32_t> tiles;
  int32_t n_tiles = -1;
  if (host_cu && att_fused_ && qkv_att_supported(s_.d, s_.heads)) {
    tiles.reserve(size_t(s1 - s0) + 4);
    n_tiles = att_tiles_for(host_cu, s0, s1, tiles);
    if (n_tiles > att_max_tiles(ntok)) return cudaErrorInvalidValue;
    if (n_tiles > 0) {
      SURGE_TRY(ws.tables.upload(ws.tiles, tiles.data(), tiles.size(), st));
      const int dh = d / s_.heads;
      SURGE_TRY(launch_att_records(ws.tiles, n_tiles, d_cu, tok0, ATT_SLICE / (3 * dh) / att_unit_heads(dh),
                                   ws.att_rec, st));
    }
  }
  const bool att_fused = n_tiles > 0;
  if (host_cu) {
    max_len = 0;
    for (int64_t i = s0; i < s1; ++i) {
      const int32_t li = host_cu[i + 1] - host_cu[i];
      max_len = li > max_len ? li : max_len;
      sum_l2 += double(li) * double(li);
      if (li > 64) long_texts.push_back(int32_t(i - s0));
    }
    if (!long_texts.empty() && !att_fused) {
      group_long_by_class(long_texts, [&](int32_t i) { return host_cu[s0 + i + 1] - host_cu[s0 + i]; }, long_off);
      SURGE_TRY(ws.tables.upload(ws.long_idx, long_texts.data(), long_texts.size(), st));
    }
  }
  const double M = ntok, D = d, F = f;
  cudaEvent_t ev = nullptr;
  int64_t k = 0;
  if (P) prof->begin(st, &ev);
  if (att_fused) ++k;   // launch_att_records
  SURGE_TRY(launch_embed_ln(d_ids, cu, n, tok0, word_, pos_, type_, emb_g_, emb_b_, d, s_.eps, ws.X, st));
  if (!att_fused) SURGE_TRY(launch_window_index(cu, n, tok0, ntok, ws.win, st));
  // algorithmic HBM bytes: the id in, the bf16 row out (the word / position rows are gathers from a
  // 23 MB / 0.4 MB table that stays in L2)
  if (P) prof->end(KK_EMBED, st, ev, 0.0, M * (4 + 2 * D));
  k += att_fused ? 1 : 2;
  const bool fused = fused_ln(d);
  for (const LayerW& L : layers_) {
    GemmArgs g{};
    g.M = ntok;
    g.eps = s_.eps;
    if (att_fused) {
      // K4 + K5 fused: O = attention(X Wqkv^T + b), QKV never leaves the SM
      g.tmA = &tmX; g.tmB = &L.tm_wqkv_att; g.tmC = &smQKV; g.N = 3 * d; g.K = d; g.epi = EPI_QKV_ATTN;
      g.bias = L.bqkv_att; g.C = ws.O;
      g.att_rec = ws.att_rec; g.n_att_tiles = n_tiles;
      g.head_dim = d / s_.heads; g.qscale = 1.4426950408889634f / sqrtf(float(d / s_.heads));
      if (P) prof->begin(st, &ev);
      if (att_tc_ && qkv_attn_tc_supported(d, s_.heads)) SURGE_TRY(launch_qkv_attn_tc(g, st));
      else SURGE_TRY(launch_gemm(g, st));
      if (P) prof->end(KK_QKV_ATTN, st, ev, 2 * M * 3 * D * D + 4 * D * sum_l2, 2 * (M * D + 3 * D * D + M * D));
      g.att_rec = nullptr; g.n_att_tiles = 0;
      k += 1;
    } else {
      // K4: QKV = X Wqkv^T + b
      g.tmA = &tmX; g.tmB = &L.tm_wqkv; g.tmC = &smQKV; g.N = 3 * d; g.K = d; g.epi = EPI_BIAS; g.bias = L.bqkv; g.C = ws.QKV;
      if (P) prof->begin(st, &ev);
      SURGE_TRY(launch_gemm(g, st));
      if (P) prof->end(KK_QKV, st, ev, 2 * M * 3 * D * D, 2 * (M * D + 3 * D * D + M * 3 * D));
      // K5: O = attention(QKV) per text
      if (P) prof->begin(st, &ev);
      int n_att = 0;
      SURGE_TRY(launch_attention(ws.QKV, cu, n, tok0, ntok, max_len, ws.win, true, s_.heads, d / s_.heads, ws.O, st,
                                 host_cu ? ws.long_idx : nullptr, int32_t(long_texts.size()),
                                 host_cu ? long_off : nullptr, &n_att));
      if (P) prof->end(KK_ATTN, st, ev, 4 * D * sum_l2, M * (3 * D * 2 + D * 2));
      k += 1 + n_att;
    }
    if (tail_fused_ && mlp_fused_ && mlp_fused_supported(d, f)) {
      // K6 + K7 + K8 fused: X = LN_o(FFN(X1) + X1), X1 = LN_a(O Wo^T + bo + X) kept on chip
      MlpArgs a{&tmO, &L.tm_w1_mlp, &L.tm_w2_mlp, &L.tm_wo_mlp, &tmX, &L.tm_wo64, ntok, d, f, L.b1, L.b2, L.ln2_g,
                L.ln2_b, L.bo, L.ln1_g, L.ln1_b, ws.X, ws.X, s_.eps};
      a.ln_host = L.ln_host.data();
      if (P) prof->begin(st, &ev);
      SURGE_TRY(launch_mlp(a, st));
      if (P) prof->end(KK_TAIL, st, ev, 2 * M * D * D + 4 * M * F * D, 2 * (D * D + 2 * F * D + 3 * M * D));
      k += 1;
      continue;
    }
    // K6: X1 = LN(O Wo^T + bo + X)
    g.tmA = &tmO; g.tmB = &L.tm_wo; g.tmC = &smX1; g.tmR = &tmX; g.N = d; g.K = d; g.epi = EPI_BIAS_LN; g.bias = L.bo; g.res = ws.X;
    g.gamma = L.ln1_g; g.beta = L.ln1_b; g.C = ws.X1;
    if (P) prof->begin(st, &ev);
    const bool pair = !fused && ln_pair_ && ln_pair_supported(d, d);
    if (fused) {
      SURGE_TRY(launch_gemm(g, st));
    } else if (pair) {
      g.tmB = &L.tm_wo_p64;
      if (kb32) g.tmA = &tmO32;
      SURGE_TRY(launch_ln_pair(g, st));
    } else {
      g.epi = EPI_BIAS_RES; g.C = reinterpret_cast<uint16_t*>(ws.V);
      SURGE_TRY(launch_gemm(g, st));
      SURGE_TRY(launch_layernorm(ws.V, ntok, d, L.ln1_g, L.ln1_b, s_.eps, ws.X1, st));
    }
    if (P) prof->end(KK_OUT_LN, st, ev, 2 * M * D * D, 2 * (M * D + D * D + 2 * M * D));
    k += (fused || pair) ? 1 : 2;
    if (mlp_fused_ && mlp_fused_supported(d, f)) {
      // K7 + K8 fused: X = LN(GELU(X1 W1^T + b1) W2^T + b2 + X1), H stays on chip
      MlpArgs a{&tmX1, &L.tm_w1_mlp, &L.tm_w2_mlp, nullptr, nullptr, nullptr, ntok, d, f, L.b1, L.b2, L.ln2_g, L.ln2_b,
                nullptr, nullptr, nullptr, nullptr, ws.X, s_.eps};
      a.ln_host = L.ln_host.data();
      if (P) prof->begin(st, &ev);
      SURGE_TRY(launch_mlp(a, st));
      if (P) prof->end(KK_MLP, st, ev, 4 * M * F * D, 2 * (2 * F * D + 2 * M * D));
      k += 1;
      continue;
    }
    // K7: H = GELU(X1 W1^T + b1)
    g.tmA = &tmX1; g.tmB = &L.tm_w1; g.tmC = &smH; g.tmR = nullptr; g.N = f; g.K = d; g.epi = EPI_BIAS_GELU; g.bias = L.b1; g.res = nullptr;
    g.gamma = g.beta = nullptr; g.C = ws.H;
    if (P) prof->begin(st, &ev);
    SURGE_TRY(launch_gemm(g, st));
    if (P) prof->end(KK_FFN1, st, ev, 2 * M * F * D, 2 * (M * D + F * D + M * F));
    // K8: X = LN(H W2^T + b2 + X1)
    g.tmA = &tmH; g.tmB = &L.tm_w2; g.tmC = &smX; g.tmR = &tmX1; g.N = d; g.K = f; g.epi = EPI_BIAS_LN; g.bias = L.b2; g.res = ws.X1;
    g.gamma = L.ln2_g; g.beta = L.ln2_b; g.C = ws.X;
    if (P) prof->begin(st, &ev);
    const bool pair2 = !fused && ln_pair_ && ln_pair_supported(d, f);
    if (fused) {
      SURGE_TRY(launch_gemm(g, st));
    } else if (pair2) {
      g.tmB = &L.tm_w2_p64;
      if (kb32) g.tmA = &tmH32;
      SURGE_TRY(launch_ln_pair(g, st));
    } else {
      g.epi = EPI_BIAS_RES; g.C = reinterpret_cast<uint16_t*>(ws.V);
      SURGE_TRY(launch_gemm(g, st));
      SURGE_TRY(launch_layernorm(ws.V, ntok, d, L.ln2_g, L.ln2_b, s_.eps, ws.X, st));
    }
    if (P) prof->end(KK_FFN2, st, ev, 2 * M * D * F, 2 * (M * F + D * F + 2 * M * D));
    k += (fused || pair2) ? 2 : 3;
  }
  if (P) prof->begin(st, &ev);
  SURGE_TRY(launch_meanpool_l2(ws.X, cu, n, tok0, d, static_cast<uint8_t*>(d_out) + size_t(s0) * d * out_elem_bytes(),
                               st, pooling_, out_bf16_));
  if (P) prof->end(KK_POOL, st, ev, 0.0, M * 2 * D + double(n) * double(out_elem_bytes()) * D);
  ++k;
  if (launches) *launches += k;
  return cudaSuccess;
}

cudaError_t DeviceModel::encode(Workspace& ws, const int32_t* d_ids, const int32_t* d_cu, const int32_t* host_cu,
                                int64_t n_texts, void* d_out, cudaStream_t st, int64_t* launches,
                                Profiler* prof) const {
  int64_t s0 = 0;
  while (s0 < n_texts) {
    int64_t s1 = s0 + 1;
    while (s1 < n_texts && int64_t(host_cu[s1 + 1]) - host_cu[s0] <= ws.cap) ++s1;
    const int32_t tok0 = host_cu[s0];
    const int32_t ntok = host_cu[s1] - tok0;
    SURGE_TRY(encode_chunk(ws, d_ids, d_cu, s0, s1, tok0, ntok, d_out, st, launches, prof, host_cu));
    s0 = s1;
  }
  return cudaSuccess;
}

}  // namespace surge
