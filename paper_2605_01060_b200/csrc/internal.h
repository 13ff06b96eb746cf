// internal.h -- declarations shared by libsurge's translation units (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace surge {

// EPI_BIAS_RES: fp32 C = A B^T + b + R (the pre-LayerNorm row, for hidden sizes whose full row
// does not fit one CTA's TMEM; launch_layernorm then normalises it).  C is float* in that case.
// EPI_QKV_ATTN: the QKV projection with K5 attention in the epilogue (DESIGN.md §6 "QKV +
// attention"): A row tiles are text-aligned (att_tiles), B = W_qkv with rows permuted so that each
// 192-row slice holds [Q | K | V] of 192 / (3 d_h) whole heads (qkv_att_perm), and the CTA writes
// the attention output O [M x N/3] instead of QKV.
enum Epilogue : int { EPI_BIAS = 0, EPI_BIAS_GELU = 1, EPI_BIAS_LN = 2, EPI_BIAS_RES = 3, EPI_QKV_ATTN = 4 };

struct GemmArgs {
  const CUtensorMap* tmA;   // A [M x K]
  const CUtensorMap* tmB;   // B [N x K]
  const CUtensorMap* tmC;   // C [M x N], store map (make_tmap_store_bf16)
  const CUtensorMap* tmR;   // residual [M x N] load map (make_tmap_bf16, box 128 rows) for L2 prefetch (LN)
  int64_t M;
  int N, K, epi;
  const float* bias;
  const uint16_t* res;      // [M x N] (EPI_BIAS_LN)
  const float* gamma;
  const float* beta;
  uint16_t* C;              // [M x N]  (EPI_QKV_ATTN: O [M x N/3])
  float eps;
  // EPI_QKV_ATTN only
  const int32_t* att_rec = nullptr;     // [n_att_tiles] tile records (AttRec layout, launch_att_records)
  int32_t n_att_tiles = 0;              // even (a CTA pair takes tiles 2u, 2u + 1)
  int32_t head_dim = 0;
  float qscale = 0.f;                   // log2(e) / sqrt(d_h)
};

// Text-aligned 128-row tiles for EPI_QKV_ATTN over texts [s0, s1) (host cu, absolute): greedy,
// each tile = the longest run of whole texts with <= 128 tokens; padded with an empty tile to an
// even count.  Appends n_tiles + 1 entries (text indices) to out; returns n_tiles, or -1 when a
// text is longer than 128 tokens (the chunk then takes the separate-attention path).
int32_t att_tiles_for(const int32_t* host_cu, int64_t s0, int64_t s1, std::vector<int32_t>& out);
constexpr int ATT_TILE_ROWS = 128;
// Tile record (int32 words): [0] row0 (chunk-relative first row), [1] nrows, [2] ntexts,
// [3] nunits; bytes [16, 144): start row of each text within the tile (uint8); bytes [144, 688):
// attention work units, uint16 (text | qt << 8 | head group << 11), qt = 16-row query tile of the
// text, sorted by cost (key blocks = ceil(len / 16)) descending.  The epilogue warps take the
// units in snake order (warp w: w, 2W-1-w, 2W+w, ...), an LPT-like balance of the tile's work.
constexpr int ATT_REC_INTS = 172;
constexpr int ATT_REC_MAX_UNITS = 272;   // (128 / 16 + ntexts <= 136 query tiles) x <= 2 head groups
// heads per work unit: 1 (head groups = heads of the slice) except d_h = 16 (4 heads per slice) -> 2
#ifndef ATT_NHU32
#define ATT_NHU32 1
#endif
inline int att_unit_heads(int dh) { return dh == 16 ? 2 : dh == 32 ? ATT_NHU32 : 1; }
// Upper bound on the tiles of a chunk of ntok tokens (two consecutive greedy tiles hold > 128 rows).
inline int64_t att_max_tiles(int64_t ntok) { return ntok / 64 + 4; }
// Device: records of tiles [0, n_tiles) from the first-text table (tiles, n_tiles + 1 entries).
cudaError_t launch_att_records(const int32_t* tiles, int32_t n_tiles, const int32_t* cu, int32_t tok0,
                               int32_t n_groups, int32_t* rec, cudaStream_t st);
constexpr int ATT_SLICE = 192;   // columns of one W_qkv slice in the fused kernel
// The fused QKV + attention path applies to head sizes whose heads tile a 192-column slice.
inline bool qkv_att_supported(int d, int heads) {
  const int dh = d / heads;
  return (dh == 16 || dh == 32 || dh == 64) && (3 * d) % ATT_SLICE == 0 && ATT_SLICE % (3 * dh) == 0;
}

cudaError_t init_tma_encoder();
// Programmatic dependent launch for the GEMM-class kernels (env SURGE_PDL=0 disables).
bool pdl_enabled();
cudaError_t make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);
cudaError_t make_tmap_bf16_k32(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);
// rows per weight (B) box of the cluster-pair LN GEMMs at 64-wide k-blocks: 64 (six / eight boxes per stage over
// the three producer threads), 32, or 0 = BNC / 2 = d / 4 (two boxes per stage).  Measured (FFN2 + LN, bge-base /
// bge-large per 500K / 200K texts): 64: 398 / 586 ms; d / 4: 403 / 622 ms; 32: 574 / 766 ms
#ifndef LN_PAIR_BBOX64
#define LN_PAIR_BBOX64 64
#endif
// k-block width of the cluster-pair LN GEMMs (ln_pair.cu): 64 (128-byte swizzle), or 32 (64-byte swizzle, twice
// the ring stages: measured slower, bge-base FFN2 + LN 382 -> 431 ms per 500K texts)
#ifndef LN_PAIR_KB
#define LN_PAIR_KB 64
#endif
// Output map for the GEMM epilogue's TMA stores: box 32 rows x 32 columns, 64-byte swizzle.
cudaError_t make_tmap_store_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols);
int gemm_bn_for(int N, int K, int epi);
bool gemm_use_pair(int N, int K, int epi);
uint32_t gemm_b_box_rows(int N, int K, int epi);   // TMA box rows of the B (weight) tensor map
cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t st);
// K4 + K5 with the attention on tcgen05 (qkv_attn_tc.cu): one CTA per SM, S = Q K^T and O = P V as
// tensor-core MMAs with Q and P read from TMEM.  d = 384, d_h = 32 (MiniLM class); same arguments as
// the EPI_QKV_ATTN GEMM (text-aligned tile records, permuted W_qkv with 96-row TMA boxes).
bool qkv_attn_tc_supported(int d, int heads);
// K6 / K8 with the LayerNorm fused for d in {768, 1024} (ln_pair.cu): a cluster of two CTAs splits the row,
// statistics exchanged through distributed shared memory.  B = the weight with 64-row TMA boxes.
bool ln_pair_supported(int d, int k);
// K5 for texts of 65..512 tokens at d_h = 64 on tcgen05 (attn_long_tc.cu): one CTA per (text, head), K / V
// of the text resident, S row in TMEM; texts > 128 tokens, off by default (env SURGE_ATT_LONG_TC=1).
bool attn_long_tc_supported(int head_dim);
bool attn_long_tc_enabled();
cudaError_t launch_attn_long_tc(const uint16_t* qkv, const int32_t* cu, const int32_t* d_long, int32_t n_long,
                                int32_t tok0, int32_t ntok, int heads, uint16_t* out, cudaStream_t st);
cudaError_t launch_ln_pair(const GemmArgs& g, cudaStream_t st);
cudaError_t launch_qkv_attn_tc(const GemmArgs& g, cudaStream_t st);
// LN GEMMs fuse the LayerNorm into the epilogue when the full row fits one CTA's TMEM (d in {64, 384});
// otherwise they write fp32 pre-LN rows (EPI_BIAS_RES) and launch_layernorm finishes them.
inline bool fused_ln(int d) { return d == 64 || d == 384; }

// K7 + K8 fused (mlp_tc.cu): X = LN(GELU(X1 W1^T + b1) W2^T + b2 + X1) * gamma + beta, H kept on chip.
struct MlpArgs {
  const CUtensorMap* tmA;    // A [M x D] load map, box 128 rows: X1, or O when tmWo is set
  const CUtensorMap* tmW1;   // W1 [F x D], box 64 rows
  const CUtensorMap* tmW2;   // W2 [D x F], box mlp_w2_box_rows(D)
  const CUtensorMap* tmWo;   // nullptr, or Wo [D x D] (box mlp_w2_box_rows(D)): K6 fused as a prologue
  const CUtensorMap* tmX;    // X [M x D] load map (L2 prefetch of the K6 residual rows), when tmWo is set
  const CUtensorMap* tmWo64 = nullptr;   // Wo [D x D], box 64 rows (d = 384: the split out-projection)
  int64_t M;
  int D, F;
  const float *b1, *b2, *gamma, *beta;       // FFN biases, LN_o
  const float *bo, *gamma1, *beta1;          // K6: out-proj bias, LN_a (when tmWo is set)
  const uint16_t* x;         // X (K6 residual rows; when tmWo is set)
  uint16_t* out;             // X [M x D] output (in place over x when tmWo is set)
  float eps;
  const float* ln_host = nullptr;        // host copy [bo | gamma_a | beta_a | b2 | gamma_o | beta_o] (6 D)
};
bool mlp_fused_supported(int d, int ffn);
inline uint32_t mlp_w2_box_rows(int d) { return uint32_t(d <= 256 ? d / 2 : d / 4); }
cudaError_t launch_mlp(const MlpArgs& a, cudaStream_t st);

// K1: cu[0..n], row_off[0..m], tok_off[0..m] (one CTA up to one 8K-element tile; beyond, one CTA per
// tile for cu, then a one-CTA kernel for the partition offsets)
int pack_launch_count(int64_t n, int64_t m);   // kernels launch_pack issues
cudaError_t launch_pack(const int32_t* lengths, int64_t n, const int32_t* sizes, int64_t m, int32_t* cu,
                        int32_t* row_off, int32_t* tok_off, cudaStream_t st);
// K3: tokens of texts [0, n_texts) described by cu (absolute offsets), activations indexed cu[i]-tok0
cudaError_t launch_embed_ln(const int32_t* ids, const int32_t* cu, int64_t n_texts, int32_t tok0,
                            const uint16_t* word, const uint16_t* pos, const uint16_t* type, const float* gamma,
                            const float* beta, int d, float eps, uint16_t* x, cudaStream_t st);
// K5: text-tiled tensor-core kernel for texts of <= 64 tokens (+ per-(text, head) kernel when
// max_len > 64).  win: int32[ntok/64 + 2] scratch = first text starting in each 64-token window;
// win_ready = already filled by launch_window_index for this chunk.
cudaError_t launch_window_index(const int32_t* cu, int64_t n_texts, int32_t tok0, int32_t ntok, int32_t* win,
                                cudaStream_t st);
cudaError_t launch_attention(const uint16_t* qkv, const int32_t* cu, int64_t n_texts, int32_t tok0,
                             int32_t ntok, int32_t max_len, int32_t* win, bool win_ready, int heads, int head_dim,
                             uint16_t* out, cudaStream_t st, const int32_t* d_long = nullptr, int32_t n_long = 0,
                             const int32_t* long_class_off = nullptr, int* n_launched = nullptr);
// d_long: device int32[n_long], indices (relative to cu) of the texts longer than 64 tokens;
// nullptr = unknown (all texts are scanned by the scalar per-(text, head) kernel).
// long_class_off (host, ATT_LONG_CLASSES + 1 entries, optional): d_long is grouped by length class
// (attn_long_class) and class c is d_long[off[c], off[c + 1]) -- each class is launched over exactly its
// texts; without it every class launch covers all of d_long and CTAs of other classes exit at once.
// n_launched (optional): kernels launched.
constexpr int ATT_LONG_CLASSES = 4;   // (64, 128], (128, 192], (192, 256], (256, 512]
inline int attn_long_class(int32_t len) { return len <= 128 ? 0 : len <= 192 ? 1 : len <= 256 ? 2 : 3; }
// Stable counting sort of text indices by length class; off[0..ATT_LONG_CLASSES] = class offsets.
template <typename LenOf>
inline void group_long_by_class(std::vector<int32_t>& idx, LenOf len_of, int32_t (&off)[ATT_LONG_CLASSES + 1]) {
  int32_t cnt[ATT_LONG_CLASSES] = {0, 0, 0, 0};
  for (int32_t i : idx) ++cnt[attn_long_class(len_of(i))];
  off[0] = 0;
  for (int c = 0; c < ATT_LONG_CLASSES; ++c) off[c + 1] = off[c] + cnt[c];
  std::vector<int32_t> out(idx.size());
  int32_t pos[ATT_LONG_CLASSES];
  for (int c = 0; c < ATT_LONG_CLASSES; ++c) pos[c] = off[c];
  for (int32_t i : idx) out[size_t(pos[attn_long_class(len_of(i))]++)] = i;
  idx.swap(out);
}
// Row LayerNorm: y[r] = LN(v[r]) * gamma + beta, v fp32 [rows x d] -> bf16 (d in {768, 1024}).
cudaError_t launch_layernorm(const float* v, int64_t rows, int d, const float* gamma, const float* beta, float eps,
                             uint16_t* y, cudaStream_t st);
// K9
// pooling: 0 mean, 1 [CLS]; out: float [n x d], or bf16 bits [n x d] when out_bf16
cudaError_t launch_meanpool_l2(const uint16_t* x, const int32_t* cu, int64_t n_texts, int32_t tok0, int d,
                               void* out, cudaStream_t st, int pooling = 0, bool out_bf16 = false);

cudaError_t launch_bf16_to_f32(const uint16_t* in, float* out, int64_t n, cudaStream_t st);

// --------------------------------------------------------------------- per-kernel-class timing
enum KernelKind : int {
  KK_EMBED = 0, KK_QKV = 1, KK_ATTN = 2, KK_OUT_LN = 3, KK_FFN1 = 4, KK_FFN2 = 5, KK_POOL = 6, KK_PACK = 7,
  KK_QKV_ATTN = 8, KK_MLP = 9, KK_TAIL = 10, KK_COUNT = 11
};

// Records a CUDA event pair around launches of each kind (only when enabled).  Not thread-safe:
// one Profiler per launching thread/stream.
struct Profiler {
  bool on = false;
  struct Rec {
    int kind;
    cudaEvent_t a, b;
    double fl, by;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  int64_t launches[KK_COUNT] = {};
  double ms[KK_COUNT] = {}, flops[KK_COUNT] = {}, bytes[KK_COUNT] = {};
  cudaEvent_t take();
  void begin(cudaStream_t st, cudaEvent_t* a);
  void end(int kind, cudaStream_t st, cudaEvent_t a, double fl, double by);
  cudaError_t resolve();   // sync-free if the events completed; call after stream sync
  void clear();
  ~Profiler();
};

// ------------------------------------------------------------------------------ device model
struct ModelShape {
  int vocab, max_pos, type_vocab, d, layers, heads, ffn;
  float eps;
};

struct LayerW {
  uint16_t *wqkv, *wo, *w1, *w2;      // bf16 [3d x d], [d x d], [ff x d], [d x ff]
  float *bqkv, *bo, *ln1_g, *ln1_b, *b1, *b2, *ln2_g, *ln2_b;
  CUtensorMap tm_wqkv, tm_wo, tm_w1, tm_w2;
  CUtensorMap tm_wo_mlp, tm_w1_mlp, tm_w2_mlp;   // fused tail (mlp_tc.cu) views of Wo / W1 / W2
  CUtensorMap tm_wo64;                            // Wo, 64-row boxes (split out-projection in the tail)
  CUtensorMap tm_wo_p64, tm_w2_p64;               // d in {768, 1024}: Wo / W2 with 64-row boxes (ln_pair.cu)
  std::vector<float> ln_host;                     // host [bo | ln1_g | ln1_b | b2 | ln2_g | ln2_b] (tail kernel parameter)
  uint16_t* wqkv_att = nullptr;       // W_qkv rows permuted into head-complete 192-row slices
  float* bqkv_att = nullptr;
  CUtensorMap tm_wqkv_att;
};

// Small host tables (tile starts, text indices, piece sizes) copied to the device per chunk or per
// SuperBatch.  A cudaMemcpyAsync from pageable memory synchronises the stream before it starts, which
// would stall the launching thread until the queued kernels finish; these tables are staged in a ring
// of pinned buffers instead, each slot guarded by an event recorded after its copy.
struct PinnedRing {
  static constexpr int NS = 8;
  int32_t* buf[NS] = {};
  size_t cap[NS] = {};
  cudaEvent_t ev[NS] = {};
  int next = 0;
  // A pinned slot of >= n int32 whose previous copy has completed; nullptr on allocation failure.
  int32_t* acquire(size_t n, int* slot);
  // Copy n int32 from slot to dst on st and guard the slot until the copy has run.
  cudaError_t copy(int slot, int32_t* dst, size_t n, cudaStream_t st);
  // acquire + memcpy from src + copy
  cudaError_t upload(int32_t* dst, const int32_t* src, size_t n, cudaStream_t st);
  void release();
  ~PinnedRing() { release(); }
};

// Activation workspace for one chunk of <= cap tokens (bf16): X, QKV, O, X1, H.
struct Workspace {
  PinnedRing tables;        // host -> device staging of the per-chunk tables
  int64_t cap = 0;
  uint16_t *X = nullptr, *QKV = nullptr, *O = nullptr, *X1 = nullptr, *H = nullptr;
  float* V = nullptr;       // fp32 pre-LayerNorm rows (hidden sizes without the fused LN epilogue)
  int32_t* long_idx = nullptr;   // texts of the chunk longer than 64 tokens, cap/65 + 1 entries
  int32_t* win = nullptr;   // attention: first text of each 64-token window, cap/64 + 2 entries
  int32_t* tiles = nullptr; // EPI_QKV_ATTN first text of each tile of the current chunk
  int32_t* att_rec = nullptr;   // EPI_QKV_ATTN tile records of the current chunk
  cudaError_t alloc(const ModelShape& s, int64_t cap_tokens);
  void release();
  ~Workspace() { release(); }
};

// Owns the encoder weights on one device and runs the encoder chain (K3, K4-K8, K5, K9).
class DeviceModel {
 public:
  DeviceModel() = default;
  ~DeviceModel();
  // blob: HF-order bf16 weights (host or device pointer), layout of include/surge.h.
  cudaError_t init(const ModelShape& s, const uint16_t* blob, bool blob_on_device, cudaStream_t st);
  // Texts [s0, s1) of a packed stream: d_ids/d_cu absolute (cu[i] = first token of text i),
  // activations chunk-local (token t at row t - tok0); writes d_out rows [s0, s1) (fp32 [n x d]).
  // host_cu (optional, absolute, indexed like d_cu) is only read when prof is enabled.
  cudaError_t encode_chunk(Workspace& ws, const int32_t* d_ids, const int32_t* d_cu, int64_t s0, int64_t s1,
                           int32_t tok0, int32_t ntok, void* d_out, cudaStream_t st, int64_t* launches,
                           Profiler* prof = nullptr, const int32_t* host_cu = nullptr) const;
  // All texts [0, n): cuts chunks of <= ws.cap tokens at text boundaries using host_cu.
  cudaError_t encode(Workspace& ws, const int32_t* d_ids, const int32_t* d_cu, const int32_t* host_cu,
                     int64_t n_texts, void* d_out, cudaStream_t st, int64_t* launches,
                     Profiler* prof = nullptr) const;
  const ModelShape& shape() const { return s_; }
  const uint16_t* word() const { return word_; }
  const uint16_t* pos() const { return pos_; }
  const uint16_t* type() const { return type_; }
  const float* emb_g() const { return emb_g_; }
  const float* emb_b() const { return emb_b_; }
  // fused QKV + attention kernel on/off (on by default; off = separate K4 GEMM + K5 kernels)
  void set_att_fused(bool on) { att_fused_ = on; }
  void set_att_tc(bool on) { att_tc_ = on; }
  void set_ln_pair(bool on) { ln_pair_ = on; }
  bool att_fused() const { return att_fused_; }
  // fused MLP kernel on/off (on by default; off = separate K7 GELU GEMM + K8 LN GEMM)
  void set_mlp_fused(bool on) { mlp_fused_ = on; }
  // out-projection + LN fused into the MLP kernel as a prologue (on by default; needs mlp fused)
  void set_tail_fused(bool on) { tail_fused_ = on; }
  // pooling: 0 = masked mean over all tokens (reading R6, default), 1 = [CLS] (bge's native)
  void set_pooling(int p) { pooling_ = p; }
  // output element type: false = float32 (default), true = bf16
  void set_out_bf16(bool b) { out_bf16_ = b; }
  size_t out_elem_bytes() const { return out_bf16_ ? 2 : 4; }

 private:
  ModelShape s_{};
  bool att_fused_ = true;
  bool att_tc_ = false;       // fused QKV + attention on tcgen05 where supported (qkv_attn_tc.cu)
  bool ln_pair_ = true;       // d in {768, 1024}: LN GEMMs as cluster pairs (ln_pair.cu) instead of fp32 rows + LN kernel
  bool mlp_fused_ = true;
  bool tail_fused_ = true;
  int pooling_ = 0;
  bool out_bf16_ = false;
  std::vector<void*> allocs_;
  uint16_t *word_ = nullptr, *pos_ = nullptr, *type_ = nullptr;
  float *emb_g_ = nullptr, *emb_b_ = nullptr;
  std::vector<LayerW> layers_;
  cudaError_t dalloc(void** p, size_t bytes);
};

// Elements in the HF-order weight blob for shape s.
size_t blob_elems(const ModelShape& s);

}  // namespace surge
