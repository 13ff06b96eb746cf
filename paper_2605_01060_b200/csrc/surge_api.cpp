// surge_api.cpp -- libsurge host runtime behind the C ABI of include/surge.h.
//
//   submit (producer thread) --copy--> pinned staging of the open SuperBatch
//        |  AddPartition (Alg.1): total += n; >= b_max Safety / >= b_min Efficiency -> seal
//        v
//   sealed SuperBatch --LPT plan (world > 1)--> worker thread (one per handle / GPU)
//        H2D ids+lengths (copy stream) -> K1 pack -> chunks: encoder chain (compute stream)
//        -> per chunk D2H of the finished rows into the SuperBatch's pinned output (copy stream)
//        -> host callback: pieces whose last row landed become pollable (TTFO)
//   poll / release (any thread): zero-copy views E[start:end] into the pinned output
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types and prototypes only: libnccl.so.2 is opened at run time (nccl_api())
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing unless a profiler is attached

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/surge.h"
#include "internal.h"

using Clock = std::chrono::steady_clock;

namespace surge {
struct Ctx;
namespace {

constexpr int REASON_EFFICIENCY = 0, REASON_SAFETY = 1, REASON_END = 2;

// NVTX range for the host runtime's timeline (nsys / ncu --nvtx): seal (Flush), per-SuperBatch
// enqueue on the worker, per-chunk encode.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Alg.1 AddPartition decision after `total += n`: Safety first, then Efficiency.
inline int alg1_decide(int64_t total, int64_t b_min, int64_t b_max) {
  if (total >= b_max) return REASON_SAFETY;
  if (total >= b_min) return REASON_EFFICIENCY;
  return -1;
}

// One AddPartition under a B_max policy (include/surge.h SURGE_BMAX_*), as steps over the arriving
// partition's rows: append rows [row0, row0 + rows) to the open SuperBatch, or seal it (Flush).
// `total` = texts already buffered (< b_min between calls).
struct AggStep {
  bool seal;
  int64_t row0, rows;
  int reason;
};

void plan_add(int64_t total, int64_t n, int64_t b_min, int64_t b_max, int policy, std::vector<AggStep>& out) {
  out.clear();
  if (policy == SURGE_BMAX_SPLIT) {          // fill to exactly b_max, flush, continue
    int64_t row0 = 0;
    while (total + (n - row0) >= b_max) {
      const int64_t take = b_max - total;
      out.push_back({false, row0, take, 0});
      out.push_back({true, 0, 0, REASON_SAFETY});
      row0 += take;
      total = 0;
    }
    if (row0 < n) {
      out.push_back({false, row0, n - row0, 0});
      if (total + (n - row0) >= b_min) out.push_back({true, 0, 0, REASON_EFFICIENCY});
    }
    return;
  }
  if (policy == SURGE_BMAX_PREFLUSH && total > 0 && total + n > b_max) {   // P:304 / P:308
    out.push_back({true, 0, 0, REASON_SAFETY});
    total = 0;
  }
  out.push_back({false, 0, n, 0});           // P:275-276 append, total += n
  const int r = alg1_decide(total + n, b_min, b_max);
  if (r >= 0) out.push_back({true, 0, 0, r});
}

double secs(Clock::time_point a, Clock::time_point b) { return std::chrono::duration<double>(b - a).count(); }

struct PinnedBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct LptPiece {
  int64_t first_row, n_rows, member, tokens;
  int32_t rank;
};

// LPT plan, the rule documented in include/surge.h (surge_lpt_plan).
void lpt_plan(const int32_t* lengths, int64_t n_texts, const int64_t* sizes, int64_t m, int world,
              std::vector<LptPiece>& out) {
  out.clear();
  int64_t row = 0;
  if (world <= 1) {
    for (int64_t j = 0; j < m; ++j) {
      int64_t tok = 0;
      for (int64_t i = row; i < row + sizes[j]; ++i) tok += lengths[i];
      out.push_back({row, sizes[j], j, tok, 0});
      row += sizes[j];
    }
    return;
  }
  int64_t T = 0;
  for (int64_t i = 0; i < n_texts; ++i) T += lengths[i];
  const int64_t U = (T + 8 * int64_t(world) - 1) / (8 * int64_t(world));
  for (int64_t j = 0; j < m; ++j) {
    int64_t first = row, tok = 0;
    const int64_t end = row + sizes[j];
    for (int64_t i = row; i < end; ++i) {
      const int64_t l = lengths[i];
      if (tok > 0 && tok + l > U) {
        out.push_back({first, i - first, j, tok, -1});
        first = i;
        tok = 0;
      }
      tok += l;
    }
    if (end > first) out.push_back({first, end - first, j, tok, -1});
    row = end;
  }
  std::vector<size_t> order(out.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    if (out[a].tokens != out[b].tokens) return out[a].tokens > out[b].tokens;
    return out[a].first_row < out[b].first_row;
  });
  std::vector<int64_t> load(world, 0);
  for (size_t idx : order) {
    int best = 0;
    for (int r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    out[idx].rank = best;
    load[best] += out[idx].tokens;
  }
}

struct SuperBatch {
  int64_t index = 0;
  int reason = 0;
  std::vector<uint64_t> keys;
  std::vector<int64_t> sizes;                // texts of each member
  std::vector<int64_t> row0, part_rows;      // member = rows [row0, row0 + size) of a partition of part_rows
  std::vector<int64_t> text_off, tok_off;   // per member, within the staging buffer
  int64_t n_texts = 0, n_tokens = 0;
  PinnedBuf stage;                           // ids [n_tokens] then lengths [n_texts] (int32)
  // rank-local share
  std::vector<LptPiece> pieces;              // this rank's pieces, global-row order
  std::vector<int64_t> piece_local_row;      // first row of piece p in the rank-local stream
  int64_t local_texts = 0, local_tokens = 0;
  PinnedBuf out;                             // float [local_texts x d]
  int64_t delivered_pieces = 0;              // pushed to the ready queue
  int64_t released_pieces = 0;
  std::vector<uint8_t> piece_state;          // per piece: 0 in flight/ready, 1 polled, 2 released
  bool done = false;                         // all local rows on the host
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  double encode_ms = -1.0;
};

struct Ready {
  SuperBatch* sb;       // nullptr for n_k = 0 partitions
  int64_t piece;        // index into sb->pieces
  uint64_t key;
};

// NCCL, resolved with dlopen on first use (K11: the one-time weight broadcast).  In a process that
// already loaded NCCL (e.g. through torch.distributed) dlopen returns that library; libsurge itself
// has no link-time NCCL dependency, so it loads and runs single-GPU without it.
struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      a.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return a;
    }
    a.get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(lib, "ncclCommInitRank"));
    a.broadcast = reinterpret_cast<decltype(&ncclBroadcast)>(dlsym(lib, "ncclBroadcast"));
    a.comm_destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(lib, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(lib, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.broadcast && a.comm_destroy && a.error_string;
    if (!a.ok) a.why = "libnccl.so.2 lacks an expected symbol";
    return a;
  }();
  return api;
}

struct ChunkDone {
  Ctx* ctx;
  SuperBatch* sb;
  int64_t row_end;      // rank-local rows [0, row_end) have landed
  bool last;
};

}  // namespace

struct Ctx {
  surge_config cfg{};
  ModelShape shape{};
  int device = 0;
  DeviceModel model;
  Workspace ws;                      // worker-thread workspace
  Workspace ws_api;                  // surge_encode_packed workspace
  cudaStream_t s_comp = nullptr, s_h2d = nullptr, s_d2h = nullptr;
  // device buffers (2 input slots, 2 output chunk buffers)
  int32_t* d_ids[2] = {nullptr, nullptr};
  int32_t* d_len[2] = {nullptr, nullptr};
  int32_t* d_cu[2] = {nullptr, nullptr};
  int32_t* d_sizes[2] = {nullptr, nullptr};
  int32_t* d_rowoff[2] = {nullptr, nullptr};
  int32_t* d_tokoff[2] = {nullptr, nullptr};
  size_t cap_ids[2] = {0, 0}, cap_texts[2] = {0, 0}, cap_pieces[2] = {0, 0};
  size_t cap_cu[2] = {0, 0}, cap_ro[2] = {0, 0}, cap_to[2] = {0, 0};
  cudaEvent_t slot_free[2] = {nullptr, nullptr};   // compute finished with input slot
  uint8_t* d_E[2] = {nullptr, nullptr};           // pooled rows of a chunk (out_dtype elements)
  cudaEvent_t e_free[2] = {nullptr, nullptr};      // D2H finished reading chunk buffer
  cudaEvent_t e_ready[2] = {nullptr, nullptr};     // chunk rows written
  int64_t chunk_counter = 0;
  int64_t slot_counter = 0;
  // api-path scratch
  int32_t* api_cu = nullptr;
  size_t api_cu_cap = 0;
  std::vector<int32_t> api_host_cu;
  std::mutex api_mu;
  // api-path gather scratch (world_size > 1)
  int32_t *api_ids = nullptr, *api_len = nullptr, *api_sizes = nullptr, *api_ro = nullptr, *api_to = nullptr;
  uint8_t* api_out = nullptr;
  size_t api_ids_cap = 0, api_len_cap = 0, api_sizes_cap = 0, api_ro_cap = 0, api_to_cap = 0, api_out_cap = 0;
  // per-kernel-class timing
  std::mutex prof_mu;
  Profiler prof;       // worker stream
  Profiler prof_api;   // device-level entry points

  // ---- aggregator state (producer thread)
  std::vector<uint64_t> buf_keys;
  std::vector<int64_t> buf_sizes, buf_text_off, buf_tok_off, buf_row0, buf_part_rows;
  std::vector<AggStep> plan;
  int64_t total = 0, total_tokens = 0;
  PinnedBuf stage;                   // open SuperBatch staging
  std::vector<int32_t> stage_len_tmp;  // lengths of the open SuperBatch (host, pageable)
  std::unordered_set<uint64_t> seen;
  bool finished = false;

  // ---- shared state (guarded by mu)
  std::mutex mu;
  std::condition_variable cv_ready, cv_work, cv_space;
  std::deque<SuperBatch*> work;
  std::deque<Ready> ready;
  std::vector<std::unique_ptr<SuperBatch>> sbs;
  std::vector<PinnedBuf> stage_pool, out_pool;
  int64_t inflight_sbs = 0, inflight_texts = 0, pending_pieces = 0;
  bool shutdown = false;
  int poisoned = 0;
  uint64_t generation = 0;           // incremented by surge_reset: tokens of an older stream are rejected
  std::string err;
  std::thread worker;
  ncclComm_t nccl = nullptr;         // surge_create_replicated: the world's communicator (K11)

  // ---- stats
  surge_stats st{};
  Clock::time_point t_first_submit{};
  bool have_first_submit = false;
  bool have_ttfo = false;
  std::atomic<int64_t> launches{0};

  void set_error(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    std::lock_guard<std::mutex> g(mu);
    if (!poisoned && code == SURGE_E_CUDA) poisoned = code;
    err = buf;
  }
};

namespace {

#define CUDA_OR_FAIL(ctx, expr)                                                                  \
  do {                                                                                            \
    cudaError_t _e = (expr);                                                                      \
    if (_e != cudaSuccess) {                                                                      \
      (ctx)->set_error(SURGE_E_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));           \
      return SURGE_E_CUDA;                                                                        \
    }                                                                                             \
  } while (0)

template <typename T>
cudaError_t ensure_dev(T** p, size_t& cap, size_t n) {
  if (cap >= n && *p) return cudaSuccess;
  size_t ncap = std::max(n, cap * 2);
  ncap = std::max<size_t>(ncap, 1024);
  if (*p) cudaFree(*p);
  *p = nullptr;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), ncap * sizeof(T));
  cap = e == cudaSuccess ? ncap : 0;
  return e;
}

// Pinned buffers are never freed on the hot path (cudaFreeHost can stall the submitting thread
// behind the device's queued work, and page-locking is slow): a buffer that must grow is replaced by
// the best-fitting pooled buffer or a fresh allocation (25% headroom), and the old one returns to the
// pool.  `mu` guards the pool (the CUDA callback and surge_release push into it).
bool grow_pinned(PinnedBuf& b, size_t bytes, size_t keep, std::vector<PinnedBuf>& pool, std::mutex& mu) {
  if (b.cap >= bytes && b.p) return true;
  PinnedBuf nb{};
  {
    std::lock_guard<std::mutex> g(mu);
    int best = -1;
    for (int i = 0; i < int(pool.size()); ++i)
      if (pool[i].cap >= bytes && (best < 0 || pool[i].cap < pool[best].cap)) best = i;
    if (best >= 0) {
      nb = pool[best];
      pool.erase(pool.begin() + best);
    }
  }
  if (!nb.p) {
    const size_t cap = std::max<size_t>(bytes + bytes / 4, size_t(1) << 20);
    if (cudaHostAlloc(&nb.p, cap, cudaHostAllocPortable) != cudaSuccess) return false;
    nb.cap = cap;
  }
  if (b.p) {
    if (keep) std::memcpy(nb.p, b.p, keep);
    std::lock_guard<std::mutex> g(mu);
    pool.push_back(b);
  }
  b = nb;
  return true;
}

PinnedBuf take_from_pool(std::vector<PinnedBuf>& pool, size_t bytes) {
  // best fit among buffers that are large enough, else the largest (will be grown)
  int best = -1;
  for (int i = 0; i < int(pool.size()); ++i) {
    if (pool[i].cap >= bytes && (best < 0 || pool[i].cap < pool[best].cap)) best = i;
  }
  if (best < 0) {   // none large enough: grow the largest (least growth)
    for (int i = 0; i < int(pool.size()); ++i)
      if (best < 0 || pool[i].cap > pool[best].cap) best = i;
  }
  if (best < 0) return PinnedBuf{};
  PinnedBuf b = pool[best];
  pool.erase(pool.begin() + best);
  return b;
}

void CUDART_CB on_chunk_done(void* arg) {
  std::unique_ptr<ChunkDone> cd(static_cast<ChunkDone*>(arg));
  Ctx* c = cd->ctx;
  SuperBatch* sb = cd->sb;
  std::lock_guard<std::mutex> g(c->mu);
  int64_t newly = 0;
  while (sb->delivered_pieces < int64_t(sb->pieces.size())) {
    const int64_t p = sb->delivered_pieces;
    if (sb->piece_local_row[p] + sb->pieces[p].n_rows > cd->row_end) break;
    c->ready.push_back(Ready{sb, p, sb->keys[sb->pieces[p].member]});
    ++sb->delivered_pieces;
    ++newly;
  }
  if (newly && !c->have_ttfo && c->have_first_submit) {
    c->have_ttfo = true;
    c->st.ttfo_s = secs(c->t_first_submit, Clock::now());
  }
  if (cd->last) {
    sb->done = true;
    c->inflight_sbs -= 1;
    c->inflight_texts -= sb->n_texts;
    // staging is no longer needed once the rows landed
    if (sb->stage.p) {
      c->stage_pool.push_back(sb->stage);
      sb->stage = PinnedBuf{};
    }
    c->cv_space.notify_all();
  }
  if (newly) c->cv_ready.notify_all();
}

// Encode one sealed SuperBatch on the worker thread (asynchronously enqueued on the streams).
int process_superbatch(Ctx* c, SuperBatch* sb) {
  NvtxRange nvtx_sb("surge.superbatch");
  const int d = c->shape.d;
  if (sb->local_texts == 0) {
    std::lock_guard<std::mutex> g(c->mu);
    sb->done = true;
    c->inflight_sbs -= 1;
    c->inflight_texts -= sb->n_texts;
    if (sb->stage.p) {
      c->stage_pool.push_back(sb->stage);
      sb->stage = PinnedBuf{};
    }
    c->cv_space.notify_all();
    return 0;
  }
  const int slot = int(c->slot_counter++ & 1);
  const int32_t* s_ids = static_cast<const int32_t*>(sb->stage.p);
  const int32_t* s_len = s_ids + sb->n_tokens;
  // rank-local stream: pieces in global-row order
  const int64_t LT = sb->local_tokens, LS = sb->local_texts, NP = int64_t(sb->pieces.size());
  CUDA_OR_FAIL(c, cudaSetDevice(c->device));
  CUDA_OR_FAIL(c, cudaStreamWaitEvent(c->s_h2d, c->slot_free[slot], 0));
  CUDA_OR_FAIL(c, ensure_dev(&c->d_ids[slot], c->cap_ids[slot], size_t(LT)));
  CUDA_OR_FAIL(c, ensure_dev(&c->d_len[slot], c->cap_texts[slot], size_t(LS)));
  CUDA_OR_FAIL(c, ensure_dev(&c->d_cu[slot], c->cap_cu[slot], size_t(LS + 1)));
  CUDA_OR_FAIL(c, ensure_dev(&c->d_sizes[slot], c->cap_pieces[slot], size_t(NP + 1)));
  CUDA_OR_FAIL(c, ensure_dev(&c->d_rowoff[slot], c->cap_ro[slot], size_t(NP + 1)));
  CUDA_OR_FAIL(c, ensure_dev(&c->d_tokoff[slot], c->cap_to[slot], size_t(NP + 1)));

  // host-side: local lengths, piece sizes, host cu (for chunk cuts)
  std::vector<int32_t> host_cu(static_cast<size_t>(LS + 1));
  std::vector<int32_t> piece_sizes(static_cast<size_t>(NP));
  host_cu[0] = 0;
  {
    int64_t r = 0;
    for (int64_t p = 0; p < NP; ++p) {
      const LptPiece& pc = sb->pieces[p];
      piece_sizes[p] = int32_t(pc.n_rows);
      for (int64_t i = 0; i < pc.n_rows; ++i, ++r) host_cu[r + 1] = host_cu[r] + s_len[pc.first_row + i];
    }
  }
  // H2D: one copy per piece (world == 1: one piece per member, contiguous -> merge runs)
  {
    int64_t lrow = 0, ltok = 0;
    int64_t p = 0;
    while (p < NP) {
      // merge consecutive pieces that are contiguous in the staging buffer
      int64_t q = p + 1;
      while (q < NP && sb->pieces[q].first_row == sb->pieces[q - 1].first_row + sb->pieces[q - 1].n_rows) ++q;
      const int64_t r0 = sb->pieces[p].first_row;
      const int64_t r1 = sb->pieces[q - 1].first_row + sb->pieces[q - 1].n_rows;
      // global token offset of row r0 within the staging buffer
      int64_t t0 = 0;
      {
        const LptPiece& pc = sb->pieces[p];
        t0 = sb->tok_off[pc.member];
        for (int64_t i = sb->text_off[pc.member]; i < r0; ++i) t0 += s_len[i];
      }
      int64_t ntok = 0;
      for (int64_t i = r0; i < r1; ++i) ntok += s_len[i];
      CUDA_OR_FAIL(c, cudaMemcpyAsync(c->d_ids[slot] + ltok, s_ids + t0, size_t(ntok) * 4, cudaMemcpyHostToDevice,
                                      c->s_h2d));
      CUDA_OR_FAIL(c, cudaMemcpyAsync(c->d_len[slot] + lrow, s_len + r0, size_t(r1 - r0) * 4,
                                      cudaMemcpyHostToDevice, c->s_h2d));
      lrow += r1 - r0;
      ltok += ntok;
      p = q;
    }
  }
  // piece sizes through the pinned ring (a pageable source would synchronise s_h2d)
  CUDA_OR_FAIL(c, c->ws.tables.upload(c->d_sizes[slot], piece_sizes.data(), size_t(NP), c->s_h2d));
  cudaEvent_t h2d_done;
  CUDA_OR_FAIL(c, cudaEventCreateWithFlags(&h2d_done, cudaEventDisableTiming));
  CUDA_OR_FAIL(c, cudaEventRecord(h2d_done, c->s_h2d));
  CUDA_OR_FAIL(c, cudaStreamWaitEvent(c->s_comp, h2d_done, 0));
  CUDA_OR_FAIL(c, cudaEventDestroy(h2d_done));

  CUDA_OR_FAIL(c, cudaEventRecord(sb->ev_begin, c->s_comp));
  {
    std::lock_guard<std::mutex> pg(c->prof_mu);
    cudaEvent_t ev = nullptr;
    c->prof.begin(c->s_comp, &ev);
    CUDA_OR_FAIL(c, launch_pack(c->d_len[slot], LS, c->d_sizes[slot], NP, c->d_cu[slot], c->d_rowoff[slot],
                                c->d_tokoff[slot], c->s_comp));
    c->prof.end(KK_PACK, c->s_comp, ev, 0.0, 8.0 * double(LS) + 12.0 * double(NP));
  }
  c->launches += pack_launch_count(LS, NP);
  // chunks
  int64_t s0 = 0;
  const int64_t cap = c->ws.cap;
  while (s0 < LS) {
    int64_t s1 = s0 + 1;
    while (s1 < LS && int64_t(host_cu[s1 + 1]) - host_cu[s0] <= cap) ++s1;
    NvtxRange nvtx_chunk("surge.chunk");
    const int b = int(c->chunk_counter++ & 1);
    CUDA_OR_FAIL(c, cudaStreamWaitEvent(c->s_comp, c->e_free[b], 0));
    int64_t nl = 0;
    // encode into d_E[b] rows [0, s1-s0): pass d_out shifted so that row s0 maps to d_E[b][0]
    const size_t eb = c->model.out_elem_bytes();
    uint8_t* dout = c->d_E[b] - size_t(s0) * d * eb;
    cudaError_t e;
    {
      std::lock_guard<std::mutex> pg(c->prof_mu);
      e = c->model.encode_chunk(c->ws, c->d_ids[slot], c->d_cu[slot], s0, s1, host_cu[s0],
                                host_cu[s1] - host_cu[s0], dout, c->s_comp, &nl, &c->prof, host_cu.data());
    }
    if (e != cudaSuccess) {
      c->set_error(SURGE_E_CUDA, "encode_chunk failed: %s", cudaGetErrorString(e));
      return SURGE_E_CUDA;
    }
    c->launches += nl;
    CUDA_OR_FAIL(c, cudaEventRecord(c->e_ready[b], c->s_comp));
    const bool last = (s1 == LS);
    if (last) {
      CUDA_OR_FAIL(c, cudaEventRecord(sb->ev_end, c->s_comp));
      CUDA_OR_FAIL(c, cudaEventRecord(c->slot_free[slot], c->s_comp));
    }
    CUDA_OR_FAIL(c, cudaStreamWaitEvent(c->s_d2h, c->e_ready[b], 0));
    CUDA_OR_FAIL(c, cudaMemcpyAsync(static_cast<uint8_t*>(sb->out.p) + size_t(s0) * d * eb, c->d_E[b], size_t(s1 - s0) * d * eb,
                                    cudaMemcpyDeviceToHost, c->s_d2h));
    CUDA_OR_FAIL(c, cudaEventRecord(c->e_free[b], c->s_d2h));
    ChunkDone* cd = new ChunkDone{c, sb, s1, last};
    cudaError_t e2 = cudaLaunchHostFunc(c->s_d2h, on_chunk_done, cd);
    if (e2 != cudaSuccess) {
      delete cd;
      c->set_error(SURGE_E_CUDA, "cudaLaunchHostFunc failed: %s", cudaGetErrorString(e2));
      return SURGE_E_CUDA;
    }
    s0 = s1;
  }
  return 0;
}

void worker_main(Ctx* c) {
  cudaSetDevice(c->device);
  for (;;) {
    SuperBatch* sb = nullptr;
    {
      std::unique_lock<std::mutex> g(c->mu);
      c->cv_work.wait(g, [&] { return c->shutdown || !c->work.empty(); });
      if (c->work.empty()) return;
      sb = c->work.front();
      c->work.pop_front();
      if (c->poisoned) continue;
    }
    if (process_superbatch(c, sb) != 0) {
      std::lock_guard<std::mutex> g(c->mu);
      c->cv_ready.notify_all();
      c->cv_space.notify_all();
    }
  }
}

// Seal the open SuperBatch (Flush) and hand it to the worker.
int seal(Ctx* c, int reason) {
  NvtxRange nvtx_seal("surge.seal");
  auto sbp = std::make_unique<SuperBatch>();
  SuperBatch* sb = sbp.get();
  sb->reason = reason;
  sb->keys.swap(c->buf_keys);
  sb->sizes.swap(c->buf_sizes);
  sb->row0.swap(c->buf_row0);
  sb->part_rows.swap(c->buf_part_rows);
  sb->text_off.swap(c->buf_text_off);
  sb->tok_off.swap(c->buf_tok_off);
  sb->n_texts = c->total;
  sb->n_tokens = c->total_tokens;
  // append lengths after the ids in the staging buffer (ids occupy [0, n_tokens))
  const size_t need = size_t(sb->n_tokens + sb->n_texts) * 4;
  if (!grow_pinned(c->stage, need, size_t(sb->n_tokens) * 4, c->stage_pool, c->mu)) {
    c->set_error(SURGE_E_OOM, "pinned staging allocation of %zu bytes failed", need);
    return SURGE_E_OOM;
  }
  int32_t* s_ids = static_cast<int32_t*>(c->stage.p);
  std::memcpy(s_ids + sb->n_tokens, c->stage_len_tmp.data(), size_t(sb->n_texts) * 4);
  c->stage_len_tmp.clear();
  sb->stage = c->stage;
  const int32_t* s_len = s_ids + sb->n_tokens;
  // LPT plan; keep this rank's pieces
  std::vector<LptPiece> all;
  lpt_plan(s_len, sb->n_texts, sb->sizes.data(), int64_t(sb->sizes.size()), c->cfg.world_size, all);
  int64_t lrow = 0;
  for (const LptPiece& p : all) {
    if (p.rank != c->cfg.rank) continue;
    sb->pieces.push_back(p);
    sb->piece_local_row.push_back(lrow);
    lrow += p.n_rows;
    sb->local_tokens += p.tokens;
  }
  sb->local_texts = lrow;
  sb->piece_state.assign(sb->pieces.size(), 0);
  cudaEventCreate(&sb->ev_begin);
  cudaEventCreate(&sb->ev_end);
  {
    std::lock_guard<std::mutex> g(c->mu);
    sb->index = int64_t(c->sbs.size());
    sb->out = PinnedBuf{};
  }
  if (!grow_pinned(sb->out, size_t(std::max<int64_t>(sb->local_texts, 1)) * c->shape.d * c->model.out_elem_bytes(), 0,
                   c->out_pool, c->mu)) {
    c->set_error(SURGE_E_OOM, "pinned output allocation failed");
    return SURGE_E_OOM;
  }
  // next staging buffer
  {
    std::lock_guard<std::mutex> g(c->mu);
    c->stage = take_from_pool(c->stage_pool, size_t(sb->n_tokens + sb->n_texts) * 4);
    c->st.superbatches += 1;
    if (reason == REASON_SAFETY) c->st.safety_flushes += 1;
    if (reason == REASON_EFFICIENCY) c->st.efficiency_flushes += 1;
    c->st.local_texts += sb->local_texts;
    c->st.local_tokens += sb->local_tokens;
    c->inflight_sbs += 1;
    c->inflight_texts += sb->n_texts;
    c->pending_pieces += int64_t(sb->pieces.size());
    c->st.peak_inflight_texts = std::max(c->st.peak_inflight_texts, c->inflight_texts);
    c->sbs.push_back(std::move(sbp));
    c->work.push_back(sb);
  }
  c->cv_work.notify_one();
  c->total = 0;
  c->total_tokens = 0;
  return 0;
}

int check_handle(Ctx* c) {
  if (!c) return SURGE_E_INVALID_ARG;
  std::lock_guard<std::mutex> g(c->mu);
  return c->poisoned ? c->poisoned : 0;
}

}  // namespace
}  // namespace surge

using surge::Ctx;

struct surge_ctx : Ctx {};

extern "C" {

const char* surge_version(void) { return "libsurge 0.1 (sm_100a)"; }

surge_status surge_create(const surge_config* cfg, const uint16_t* weights, size_t n_weights, surge_handle* out) {
  using namespace surge;
  if (!cfg || !weights || !out) return SURGE_E_INVALID_ARG;
  *out = nullptr;
  const auto t0 = Clock::now();
  const surge_config& k = *cfg;
  if (k.b_min <= 0 || k.b_max <= k.b_min) return SURGE_E_INVALID_ARG;
  if (k.hidden <= 0 || k.heads <= 0 || k.hidden % k.heads || k.layers <= 0 || k.ffn <= 0 || k.vocab_size <= 0 ||
      k.max_position <= 0 || k.type_vocab_size <= 0)
    return SURGE_E_INVALID_ARG;
  const int dh = k.hidden / k.heads;
  if (!(k.hidden == 64 || k.hidden == 384 || k.hidden == 768 || k.hidden == 1024) ||
      !(dh == 16 || dh == 32 || dh == 64) || k.ffn % 64 != 0 || k.heads % 2 != 0)
    return SURGE_E_INVALID_ARG;
  if (k.world_size < 1 || k.rank < 0 || k.rank >= k.world_size) return SURGE_E_INVALID_ARG;
  if (k.out_dtype != SURGE_F32 && k.out_dtype != SURGE_BF16) return SURGE_E_INVALID_ARG;
  if (k.bmax_policy < SURGE_BMAX_LABEL || k.bmax_policy > SURGE_BMAX_PREFLUSH) return SURGE_E_INVALID_ARG;
  ModelShape s{k.vocab_size, k.max_position, k.type_vocab_size, k.hidden, k.layers, k.heads, k.ffn, k.ln_eps};
  if (n_weights != blob_elems(s)) return SURGE_E_INVALID_ARG;

  auto c = std::make_unique<surge_ctx>();
  c->cfg = k;
  c->shape = s;
  c->model.set_out_bf16(k.out_dtype == SURGE_BF16);
  c->device = k.device;
  if (c->cfg.chunk_tokens <= 0) c->cfg.chunk_tokens = 524288;   // sweep: 131K 2.91M, 262K 3.00M, 524K 3.04M, 1M 3.06M texts/s (TTFO 7 / 9 / 16 / 28 ms)
  c->cfg.chunk_tokens = std::max(c->cfg.chunk_tokens, k.max_position);
  if (c->cfg.max_inflight <= 0) c->cfg.max_inflight = 2;
  c->st.ttfo_s = -1.0;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= k.device || k.device < 0) return SURGE_E_CUDA;
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, k.device) != cudaSuccess || prop.major != 10) return SURGE_E_CUDA;
  Ctx* C = c.get();
  auto fail = [&](cudaError_t e) -> surge_status {
    (void)e;
    return SURGE_E_CUDA;
  };
  cudaError_t e;
  if ((e = cudaSetDevice(k.device)) != cudaSuccess) return fail(e);
  if ((e = init_tma_encoder()) != cudaSuccess) return fail(e);
  if ((e = cudaStreamCreateWithFlags(&C->s_comp, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  if ((e = cudaStreamCreateWithFlags(&C->s_h2d, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  if ((e = cudaStreamCreateWithFlags(&C->s_d2h, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  if ((e = C->model.init(s, weights, k.weights_on_device != 0, C->s_comp)) != cudaSuccess) return fail(e);
  if ((e = C->ws.alloc(s, C->cfg.chunk_tokens)) != cudaSuccess) return SURGE_E_OOM;
  for (int b = 0; b < 2; ++b) {
    if ((e = cudaMalloc(&C->d_E[b], size_t(C->cfg.chunk_tokens) * s.d * C->model.out_elem_bytes())) != cudaSuccess)
      return SURGE_E_OOM;
    if ((e = cudaEventCreateWithFlags(&C->e_free[b], cudaEventDisableTiming)) != cudaSuccess) return fail(e);
    if ((e = cudaEventCreateWithFlags(&C->e_ready[b], cudaEventDisableTiming)) != cudaSuccess) return fail(e);
    if ((e = cudaEventCreateWithFlags(&C->slot_free[b], cudaEventDisableTiming)) != cudaSuccess) return fail(e);
    cudaEventRecord(C->e_free[b], C->s_d2h);
    cudaEventRecord(C->slot_free[b], C->s_comp);
  }
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(e);
  C->worker = std::thread(surge::worker_main, C);
  C->st.init_s = secs(t0, Clock::now());
  *out = c.release();
  return SURGE_OK;
}

surge_status surge_nccl_unique_id(uint8_t* id) {
  using namespace surge;
  if (!id) return SURGE_E_INVALID_ARG;
  const NcclApi& a = nccl_api();
  if (!a.ok) return SURGE_E_NCCL;
  ncclUniqueId u;
  if (a.get_unique_id(&u) != ncclSuccess) return SURGE_E_NCCL;
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return SURGE_OK;
}

surge_status surge_create_replicated(const surge_config* cfg, const uint8_t* nccl_id, const uint16_t* weights,
                                     size_t n_weights, surge_handle* out) {
  using namespace surge;
  if (!cfg || !nccl_id || !out || (cfg->rank == 0 && !weights)) return SURGE_E_INVALID_ARG;
  *out = nullptr;
  const surge_config& k = *cfg;
  if (k.world_size < 1 || k.rank < 0 || k.rank >= k.world_size) return SURGE_E_INVALID_ARG;
  ModelShape s{k.vocab_size, k.max_position, k.type_vocab_size, k.hidden, k.layers, k.heads, k.ffn, k.ln_eps};
  if (k.hidden <= 0 || k.ffn <= 0 || k.layers <= 0 || k.vocab_size <= 0 || n_weights != blob_elems(s))
    return SURGE_E_INVALID_ARG;
  const NcclApi& a = nccl_api();
  if (!a.ok) return SURGE_E_NCCL;
  const auto t0 = Clock::now();
  if (cudaSetDevice(k.device) != cudaSuccess) return SURGE_E_CUDA;
  ncclUniqueId u;
  std::memcpy(u.internal, nccl_id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  if (a.comm_init_rank(&comm, k.world_size, u, k.rank) != ncclSuccess) return SURGE_E_NCCL;
  uint16_t* blob = nullptr;
  cudaStream_t st = nullptr;
  surge_status rc = SURGE_OK;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&blob, n_weights * 2) != cudaSuccess) {
    rc = SURGE_E_OOM;
  } else {
    if (k.rank == 0 &&
        cudaMemcpyAsync(blob, weights, n_weights * 2, k.weights_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                        st) != cudaSuccess)
      rc = SURGE_E_CUDA;
    // K11: one broadcast of the bf16 blob from rank 0 over NVLink / NVSwitch (bytes: NCCL has no 16-bit int type)
    if (rc == SURGE_OK && a.broadcast(blob, blob, n_weights * 2, ncclUint8, 0, comm, st) != ncclSuccess) rc = SURGE_E_NCCL;
    if (rc == SURGE_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = SURGE_E_CUDA;
  }
  if (rc == SURGE_OK) {
    surge_config c2 = k;
    c2.weights_on_device = 1;
    rc = surge_create(&c2, blob, n_weights, out);
  }
  if (blob) cudaFree(blob);
  if (st) cudaStreamDestroy(st);
  if (rc != SURGE_OK) {
    a.comm_destroy(comm);
    return rc;
  }
  (*out)->nccl = comm;
  (*out)->cfg.weights_on_device = k.weights_on_device;
  (*out)->st.init_s = secs(t0, Clock::now());
  return SURGE_OK;
}

surge_status surge_submit_partition(surge_handle h, uint64_t partition_id, const int32_t* token_ids,
                                    const int32_t* lengths, int64_t n_texts) {
  using namespace surge;
  Ctx* c = h;
  if (int r = check_handle(c)) return surge_status(r);
  if (n_texts < 0 || (n_texts > 0 && (!lengths || !token_ids))) return SURGE_E_INVALID_ARG;
  if (c->finished) return SURGE_E_STATE;
  if (c->seen.count(partition_id)) return SURGE_E_DUPLICATE_ID;
  // validate lengths and ids
  int64_t ntok = 0;
  const int32_t maxp = c->cfg.max_position;
  for (int64_t i = 0; i < n_texts; ++i) {
    const int32_t l = lengths[i];
    if (l < 1 || l > maxp) return SURGE_E_TOO_LONG;
    ntok += l;
  }
  if (c->total_tokens + ntok >= (int64_t(1) << 31)) {   // int32 token offsets of one SuperBatch
    std::lock_guard<std::mutex> g(c->mu);
    c->err = "surge_submit_partition: the open SuperBatch would reach 2^31 tokens";
    return SURGE_E_INVALID_ARG;
  }
  {
    const uint32_t V = uint32_t(c->cfg.vocab_size);
    uint32_t bad = 0;
    for (int64_t i = 0; i < ntok; ++i) bad |= uint32_t(uint32_t(token_ids[i]) >= V);
    if (bad) return SURGE_E_TOKEN_ID;
  }
  // the add as Alg.1 steps under the B_max policy (appends and seals)
  plan_add(c->total, n_texts, c->cfg.b_min, c->cfg.b_max, c->cfg.bmax_policy, c->plan);
  // backpressure: a seal needs a free pipeline slot (nonblocking: refuse before consuming anything)
  const bool will_seal = n_texts > 0 && std::any_of(c->plan.begin(), c->plan.end(), [](const AggStep& s) { return s.seal; });
  if (will_seal && c->cfg.nonblocking_submit) {
    std::lock_guard<std::mutex> g(c->mu);
    if (c->inflight_sbs >= c->cfg.max_inflight) return SURGE_E_AGAIN;
  }
  if (!c->have_first_submit) {
    std::lock_guard<std::mutex> g(c->mu);
    c->have_first_submit = true;
    c->t_first_submit = Clock::now();
  }
  c->seen.insert(partition_id);
  {
    std::lock_guard<std::mutex> g(c->mu);
    c->st.texts += n_texts;
    c->st.tokens += ntok;
    c->st.max_partition_seen = std::max(c->st.max_partition_seen, n_texts);
  }
  if (n_texts == 0) {
    if (c->cfg.rank == 0) {
      std::lock_guard<std::mutex> g(c->mu);
      c->ready.push_back(Ready{nullptr, 0, partition_id});
      c->cv_ready.notify_all();
    }
    return SURGE_OK;
  }
  int64_t tok_row = 0, tok_at = 0;   // token offset (within the partition) of row tok_row
  for (const AggStep& step : c->plan) {
    if (step.seal) {
      {
        std::unique_lock<std::mutex> g(c->mu);
        c->cv_space.wait(g, [&] { return c->inflight_sbs < c->cfg.max_inflight || c->poisoned; });
        if (c->poisoned) return surge_status(c->poisoned);
      }
      if (int r = seal(c, step.reason)) return surge_status(r);
      continue;
    }
    // copy(texts) of rows [row0, row0 + rows) into pinned staging (Alg.1)
    while (tok_row < step.row0) tok_at += lengths[tok_row++];
    int64_t pt = 0;
    for (int64_t i = step.row0; i < step.row0 + step.rows; ++i) pt += lengths[i];
    if (!grow_pinned(c->stage, size_t(c->total_tokens + pt) * 4, size_t(c->total_tokens) * 4, c->stage_pool, c->mu)) {
      c->set_error(SURGE_E_OOM, "pinned staging allocation failed");
      return SURGE_E_OOM;
    }
    std::memcpy(static_cast<int32_t*>(c->stage.p) + c->total_tokens, token_ids + tok_at, size_t(pt) * 4);
    c->stage_len_tmp.insert(c->stage_len_tmp.end(), lengths + step.row0, lengths + step.row0 + step.rows);
    c->buf_keys.push_back(partition_id);
    c->buf_sizes.push_back(step.rows);
    c->buf_row0.push_back(step.row0);
    c->buf_part_rows.push_back(n_texts);
    c->buf_text_off.push_back(c->total);
    c->buf_tok_off.push_back(c->total_tokens);
    c->total += step.rows;               // total <- total + |texts|
    c->total_tokens += pt;
    tok_at += pt;
    tok_row = step.row0 + step.rows;
    std::lock_guard<std::mutex> g(c->mu);
    c->st.peak_buffered_texts = std::max(c->st.peak_buffered_texts, c->total);
    c->st.peak_buffered_bytes = std::max(c->st.peak_buffered_bytes, (c->total_tokens + c->total) * 4);
  }
  return SURGE_OK;
}

surge_status surge_finish(surge_handle h) {
  using namespace surge;
  Ctx* c = h;
  if (int r = check_handle(c)) return surge_status(r);
  if (c->finished) return SURGE_E_STATE;
  c->finished = true;
  if (c->total > 0) {
    {
      std::unique_lock<std::mutex> g(c->mu);
      c->cv_space.wait(g, [&] { return c->inflight_sbs < c->cfg.max_inflight || c->poisoned; });
      if (c->poisoned) return surge_status(c->poisoned);
    }
    return surge_status(seal(c, REASON_END));
  }
  return SURGE_OK;
}

surge_status surge_poll_flushed(surge_handle h, surge_flushed* out, int64_t max_items, int32_t timeout_ms,
                                int64_t* n_out) {
  using namespace surge;
  Ctx* c = h;
  if (!c || !n_out || (max_items > 0 && !out)) return SURGE_E_INVALID_ARG;
  *n_out = 0;
  std::unique_lock<std::mutex> g(c->mu);
  auto has = [&] { return !c->ready.empty() || c->poisoned; };
  if (!has() && timeout_ms != 0) {
    if (timeout_ms < 0)
      c->cv_ready.wait(g, has);
    else
      c->cv_ready.wait_for(g, std::chrono::milliseconds(timeout_ms), has);
  }
  if (c->ready.empty() && c->poisoned) return surge_status(c->poisoned);
  int64_t n = 0;
  while (n < max_items && !c->ready.empty()) {
    Ready r = c->ready.front();
    c->ready.pop_front();
    surge_flushed& f = out[n++];
    f.partition_id = r.key;
    f.d = c->shape.d;
    f.dtype = c->cfg.out_dtype;
    if (!r.sb) {
      f.row_begin = 0;
      f.n_rows = 0;
      f.partition_rows = 0;
      f.data = nullptr;
      f.superbatch = -1;
      f.token = 0;
      continue;
    }
    const LptPiece& p = r.sb->pieces[r.piece];
    f.row_begin = r.sb->row0[p.member] + (p.first_row - r.sb->text_off[p.member]);
    f.n_rows = p.n_rows;
    f.partition_rows = r.sb->part_rows[p.member];
    f.data = static_cast<const uint8_t*>(r.sb->out.p) +
             size_t(r.sb->piece_local_row[r.piece]) * c->shape.d * c->model.out_elem_bytes();
    f.superbatch = r.sb->index;
    // token: stream generation (16 bits) | SuperBatch index (28 bits) | piece (20 bits)
    f.token = ((c->generation & 0xffff) << 48) | (uint64_t(r.sb->index) << 20) | uint64_t(r.piece);
    r.sb->piece_state[r.piece] = 1;
    c->pending_pieces -= 1;
  }
  *n_out = n;
  return SURGE_OK;
}

surge_status surge_release(surge_handle h, const surge_flushed* rec) {
  using namespace surge;
  Ctx* c = h;
  if (!c || !rec) return SURGE_E_INVALID_ARG;
  if (rec->superbatch < 0) return SURGE_OK;
  std::lock_guard<std::mutex> g(c->mu);
  const uint64_t gen = rec->token >> 48, sbi = (rec->token >> 20) & ((uint64_t(1) << 28) - 1),
                 piece = rec->token & ((uint64_t(1) << 20) - 1);
  if (gen != (c->generation & 0xffff) || int64_t(sbi) != rec->superbatch || rec->superbatch >= int64_t(c->sbs.size())) {
    c->err = "surge_release: record is not from the current stream";
    return SURGE_E_INVALID_ARG;
  }
  SuperBatch* sb = c->sbs[rec->superbatch].get();
  if (piece >= sb->piece_state.size() || sb->piece_state[piece] != 1) {
    c->err = sb && piece < sb->piece_state.size() && sb->piece_state[piece] == 2 ? "surge_release: piece released twice"
                                                                                   : "surge_release: piece not polled";
    return SURGE_E_INVALID_ARG;
  }
  sb->piece_state[piece] = 2;
  sb->released_pieces += 1;
  if (sb->done && sb->released_pieces == int64_t(sb->pieces.size()) && sb->out.p) {
    c->out_pool.push_back(sb->out);
    sb->out = PinnedBuf{};
  }
  return SURGE_OK;
}

surge_status surge_pending(surge_handle h, int64_t* n_pending) {
  using namespace surge;
  Ctx* c = h;
  if (!c || !n_pending) return SURGE_E_INVALID_ARG;
  std::lock_guard<std::mutex> g(c->mu);
  *n_pending = c->pending_pieces;
  return c->poisoned ? surge_status(c->poisoned) : SURGE_OK;
}

surge_status surge_reset(surge_handle h) {
  using namespace surge;
  Ctx* c = h;
  if (int r = check_handle(c)) return surge_status(r);
  std::lock_guard<std::mutex> g(c->mu);
  if (!c->finished || c->inflight_sbs != 0 || c->pending_pieces != 0 || !c->ready.empty()) return SURGE_E_STATE;
  for (auto& sbp : c->sbs)   // every polled view must have been released: the buffers are reused
    if (sbp->released_pieces != int64_t(sbp->pieces.size())) {
      c->err = "surge_reset: polled pieces not yet released";
      return SURGE_E_STATE;
    }
  for (auto& sbp : c->sbs) {
    if (sbp->out.p) c->out_pool.push_back(sbp->out);
    if (sbp->stage.p) c->stage_pool.push_back(sbp->stage);
    if (sbp->ev_begin) cudaEventDestroy(sbp->ev_begin);
    if (sbp->ev_end) cudaEventDestroy(sbp->ev_end);
  }
  c->sbs.clear();
  c->seen.clear();
  c->generation += 1;
  c->finished = false;
  c->total = c->total_tokens = 0;
  c->have_first_submit = false;
  c->have_ttfo = false;
  const double init_s = c->st.init_s;
  c->st = surge_stats{};
  c->st.init_s = init_s;
  c->st.ttfo_s = -1.0;
  c->launches = 0;
  return SURGE_OK;
}

surge_status surge_get_stats(surge_handle h, surge_stats* out) {
  using namespace surge;
  Ctx* c = h;
  if (!c || !out) return SURGE_E_INVALID_ARG;
  std::lock_guard<std::mutex> g(c->mu);
  double tot = 0;
  for (auto& sbp : c->sbs) {
    SuperBatch* sb = sbp.get();
    if (sb->done && sb->encode_ms < 0 && sb->local_texts > 0) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, sb->ev_begin, sb->ev_end) == cudaSuccess) sb->encode_ms = ms;
    }
    if (sb->encode_ms > 0) tot += sb->encode_ms;
  }
  *out = c->st;
  out->encode_ms_total = tot;
  out->kernel_launches = c->launches.load();
  return c->poisoned ? surge_status(c->poisoned) : SURGE_OK;
}

surge_status surge_get_superbatch(surge_handle h, int64_t index, surge_superbatch_info* out) {
  using namespace surge;
  Ctx* c = h;
  if (!c || !out) return SURGE_E_INVALID_ARG;
  std::lock_guard<std::mutex> g(c->mu);
  if (index < 0 || index >= int64_t(c->sbs.size())) return SURGE_E_INVALID_ARG;
  SuperBatch* sb = c->sbs[index].get();
  if (sb->done && sb->encode_ms < 0 && sb->local_texts > 0) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, sb->ev_begin, sb->ev_end) == cudaSuccess) sb->encode_ms = ms;
  }
  out->index = sb->index;
  out->reason = sb->reason;
  out->n_members = int32_t(sb->keys.size());
  out->n_texts = sb->n_texts;
  out->n_tokens = sb->n_tokens;
  out->local_texts = sb->local_texts;
  out->local_tokens = sb->local_tokens;
  out->local_pieces = int32_t(sb->pieces.size());
  out->done = sb->done ? 1 : 0;
  out->encode_ms = sb->encode_ms;
  return SURGE_OK;
}

surge_status surge_get_superbatch_members(surge_handle h, int64_t index, uint64_t* ids, int64_t capacity,
                                          int64_t* n_out) {
  using namespace surge;
  Ctx* c = h;
  if (!c || !n_out) return SURGE_E_INVALID_ARG;
  std::lock_guard<std::mutex> g(c->mu);
  if (index < 0 || index >= int64_t(c->sbs.size())) return SURGE_E_INVALID_ARG;
  SuperBatch* sb = c->sbs[index].get();
  *n_out = int64_t(sb->keys.size());
  if (capacity < *n_out || (capacity > 0 && !ids)) return SURGE_E_INVALID_ARG;
  std::memcpy(ids, sb->keys.data(), sb->keys.size() * 8);
  return SURGE_OK;
}

const char* surge_last_error(surge_handle h) {
  if (!h) return "";
  std::lock_guard<std::mutex> g(h->mu);
  return h->err.c_str();
}

void surge_destroy(surge_handle h) {
  using namespace surge;
  if (!h) return;
  Ctx* c = h;
  {
    std::lock_guard<std::mutex> g(c->mu);
    c->shutdown = true;
  }
  c->cv_work.notify_all();
  if (c->worker.joinable()) c->worker.join();
  cudaSetDevice(c->device);
  for (cudaStream_t s : {c->s_comp, c->s_h2d, c->s_d2h})
    if (s) cudaStreamSynchronize(s);
  for (auto& sbp : c->sbs) {
    if (sbp->out.p) cudaFreeHost(sbp->out.p);
    if (sbp->stage.p) cudaFreeHost(sbp->stage.p);
    if (sbp->ev_begin) cudaEventDestroy(sbp->ev_begin);
    if (sbp->ev_end) cudaEventDestroy(sbp->ev_end);
  }
  for (auto& b : c->out_pool) cudaFreeHost(b.p);
  for (auto& b : c->stage_pool) cudaFreeHost(b.p);
  if (c->stage.p) cudaFreeHost(c->stage.p);
  for (int b = 0; b < 2; ++b) {
    for (void* p : {(void*)c->d_ids[b], (void*)c->d_len[b], (void*)c->d_cu[b], (void*)c->d_sizes[b],
                    (void*)c->d_rowoff[b], (void*)c->d_tokoff[b], (void*)c->d_E[b]})
      if (p) cudaFree(p);
    for (cudaEvent_t ev : {c->e_free[b], c->e_ready[b], c->slot_free[b]})
      if (ev) cudaEventDestroy(ev);
  }
  for (void* p : {(void*)c->api_cu, (void*)c->api_ids, (void*)c->api_len, (void*)c->api_sizes, (void*)c->api_ro,
                  (void*)c->api_to, (void*)c->api_out})
    if (p) cudaFree(p);
  for (cudaStream_t s : {c->s_comp, c->s_h2d, c->s_d2h})
    if (s) cudaStreamDestroy(s);
  if (c->nccl) nccl_api().comm_destroy(c->nccl);
  delete static_cast<surge_ctx*>(c);
}

// ------------------------------------------------------------------------------- device-level
surge_status surge_encode_packed(surge_handle h, const int32_t* d_ids, const int32_t* d_lengths,
                                 const int32_t* h_lengths, int64_t n_texts, void* d_out, void* stream) {
  using namespace surge;
  Ctx* c = h;
  if (int r = check_handle(c)) return surge_status(r);
  if (n_texts < 0 || (n_texts > 0 && (!d_ids || !d_lengths || !h_lengths || !d_out))) return SURGE_E_INVALID_ARG;
  if (n_texts == 0) return SURGE_OK;
  std::lock_guard<std::mutex> g(c->api_mu);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_OR_FAIL(c, cudaSetDevice(c->device));
  if (c->ws_api.cap == 0) CUDA_OR_FAIL(c, c->ws_api.alloc(c->shape, c->cfg.chunk_tokens));
  c->api_host_cu.resize(size_t(n_texts + 1));
  int64_t t = 0;
  c->api_host_cu[0] = 0;
  for (int64_t i = 0; i < n_texts; ++i) {
    const int32_t l = h_lengths[i];
    if (l < 1 || l > c->cfg.max_position) return SURGE_E_TOO_LONG;
    t += l;
    if (t >= (int64_t(1) << 31)) return SURGE_E_INVALID_ARG;
    c->api_host_cu[i + 1] = int32_t(t);
  }
  CUDA_OR_FAIL(c, ensure_dev(&c->api_cu, c->api_cu_cap, size_t(n_texts + 1)));
  std::lock_guard<std::mutex> pg(c->prof_mu);
  cudaEvent_t ev = nullptr;
  c->prof_api.begin(st, &ev);
  CUDA_OR_FAIL(c, launch_pack(d_lengths, n_texts, nullptr, 0, c->api_cu, nullptr, nullptr, st));
  c->prof_api.end(KK_PACK, st, ev, 0.0, 8.0 * double(n_texts));
  int64_t nl = pack_launch_count(n_texts, 0);
  CUDA_OR_FAIL(c, c->model.encode(c->ws_api, d_ids, c->api_cu, c->api_host_cu.data(), n_texts, d_out, st, &nl,
                                  &c->prof_api));
  c->launches += nl;
  return SURGE_OK;
}

surge_status surge_encode_superbatch(surge_handle h, const int32_t* d_ids, const int32_t* d_lengths,
                                     const int32_t* h_lengths, int64_t n_texts, const int64_t* h_sizes,
                                     int64_t n_members, void* d_out, void* stream) {
  using namespace surge;
  Ctx* c = h;
  if (int r = check_handle(c)) return surge_status(r);
  if (n_texts < 0 || n_members < 0) return SURGE_E_INVALID_ARG;
  if (n_texts > 0 && (!d_ids || !d_lengths || !h_lengths || !d_out || !h_sizes)) return SURGE_E_INVALID_ARG;
  if (n_texts == 0) return SURGE_OK;
  int64_t ssum = 0;
  for (int64_t j = 0; j < n_members; ++j) {
    if (h_sizes[j] < 0) return SURGE_E_INVALID_ARG;
    ssum += h_sizes[j];
  }
  if (ssum != n_texts) return SURGE_E_INVALID_ARG;
  std::lock_guard<std::mutex> g(c->api_mu);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int d = c->shape.d;
  CUDA_OR_FAIL(c, cudaSetDevice(c->device));
  if (c->ws_api.cap == 0) CUDA_OR_FAIL(c, c->ws_api.alloc(c->shape, c->cfg.chunk_tokens));
  // global token offsets (host), validation
  std::vector<int64_t> gtok(static_cast<size_t>(n_texts + 1));
  gtok[0] = 0;
  for (int64_t i = 0; i < n_texts; ++i) {
    const int32_t l = h_lengths[i];
    if (l < 1 || l > c->cfg.max_position) return SURGE_E_TOO_LONG;
    gtok[i + 1] = gtok[i] + l;
  }
  // K2: LPT plan, this rank's pieces
  std::vector<LptPiece> all, mine;
  lpt_plan(h_lengths, n_texts, h_sizes, n_members, c->cfg.world_size, all);
  for (const LptPiece& p : all)
    if (p.rank == c->cfg.rank) mine.push_back(p);
  int64_t LS = 0;
  for (const LptPiece& p : mine) LS += p.n_rows;
  if (LS == 0) return SURGE_OK;
  const bool direct = (c->cfg.world_size == 1);
  const int64_t NP = int64_t(mine.size());
  // local host cu + piece sizes
  std::vector<int32_t> host_cu(static_cast<size_t>(LS + 1));
  std::vector<int32_t> psz(static_cast<size_t>(NP));
  host_cu[0] = 0;
  {
    int64_t r = 0;
    for (int64_t p = 0; p < NP; ++p) {
      psz[p] = int32_t(mine[p].n_rows);
      for (int64_t i = 0; i < mine[p].n_rows; ++i, ++r) {
        const int64_t t = int64_t(host_cu[r]) + h_lengths[mine[p].first_row + i];
        if (t >= (int64_t(1) << 31)) return SURGE_E_INVALID_ARG;
        host_cu[r + 1] = int32_t(t);
      }
    }
  }
  const int32_t* ids = d_ids;
  const int32_t* lens = d_lengths;
  void* out = d_out;
  const size_t eb = c->model.out_elem_bytes();
  CUDA_OR_FAIL(c, ensure_dev(&c->api_cu, c->api_cu_cap, size_t(LS + 1)));
  CUDA_OR_FAIL(c, ensure_dev(&c->api_sizes, c->api_sizes_cap, size_t(NP + 1)));
  CUDA_OR_FAIL(c, ensure_dev(&c->api_ro, c->api_ro_cap, size_t(NP + 1)));
  CUDA_OR_FAIL(c, ensure_dev(&c->api_to, c->api_to_cap, size_t(NP + 1)));
  CUDA_OR_FAIL(c, c->ws_api.tables.upload(c->api_sizes, psz.data(), size_t(NP), st));
  if (!direct) {
    // gather this rank's pieces into contiguous local buffers (device-to-device)
    CUDA_OR_FAIL(c, ensure_dev(&c->api_ids, c->api_ids_cap, size_t(host_cu[LS])));
    CUDA_OR_FAIL(c, ensure_dev(&c->api_len, c->api_len_cap, size_t(LS)));
    CUDA_OR_FAIL(c, ensure_dev(&c->api_out, c->api_out_cap, size_t(LS) * d * eb));
    int64_t r = 0;
    for (const LptPiece& p : mine) {
      const int64_t t0 = gtok[p.first_row], t1 = gtok[p.first_row + p.n_rows];
      CUDA_OR_FAIL(c, cudaMemcpyAsync(c->api_ids + host_cu[r], d_ids + t0, size_t(t1 - t0) * 4,
                                      cudaMemcpyDeviceToDevice, st));
      CUDA_OR_FAIL(c, cudaMemcpyAsync(c->api_len + r, d_lengths + p.first_row, size_t(p.n_rows) * 4,
                                      cudaMemcpyDeviceToDevice, st));
      r += p.n_rows;
    }
    ids = c->api_ids;
    lens = c->api_len;
    out = c->api_out;
  }
  std::lock_guard<std::mutex> pg(c->prof_mu);
  cudaEvent_t ev = nullptr;
  c->prof_api.begin(st, &ev);
  CUDA_OR_FAIL(c, launch_pack(lens, LS, c->api_sizes, NP, c->api_cu, c->api_ro, c->api_to, st));
  c->prof_api.end(KK_PACK, st, ev, 0.0, 8.0 * double(LS) + 12.0 * double(NP));
  int64_t nl = pack_launch_count(LS, NP);
  CUDA_OR_FAIL(c, c->model.encode(c->ws_api, ids, c->api_cu, host_cu.data(), LS, out, st, &nl, &c->prof_api));
  c->launches += nl;
  if (!direct) {
    int64_t r = 0;
    for (const LptPiece& p : mine) {   // scatter rows to their SuperBatch positions
      CUDA_OR_FAIL(c, cudaMemcpyAsync(static_cast<uint8_t*>(d_out) + size_t(p.first_row) * d * eb,
                                      c->api_out + size_t(r) * d * eb, size_t(p.n_rows) * d * eb,
                                      cudaMemcpyDeviceToDevice, st));
      r += p.n_rows;
    }
  }
  return SURGE_OK;
}

surge_status surge_aggregate(const int64_t* sizes, int64_t n_partitions, int64_t b_min, int64_t b_max,
                             int64_t capacity, int64_t* sb_first, int32_t* sb_reason, int64_t* n_superbatches,
                             int64_t* peak_buffered) {
  using namespace surge;
  if (!n_superbatches || n_partitions < 0 || b_min <= 0 || b_max <= b_min || (n_partitions > 0 && !sizes))
    return SURGE_E_INVALID_ARG;
  int64_t total = 0, peak = 0, F = 0, first = 0;
  bool open = false;
  auto emit = [&](int64_t end, int reason) -> bool {
    if (F >= capacity) return false;
    if (sb_first) sb_first[F] = first;
    if (sb_reason) sb_reason[F] = reason;
    ++F;
    first = end;
    if (sb_first) sb_first[F] = end;
    return true;
  };
  for (int64_t k = 0; k < n_partitions; ++k) {
    const int64_t n = sizes[k];
    if (n < 0) return SURGE_E_INVALID_ARG;
    if (n == 0) continue;                 // completes immediately, never buffered
    open = true;
    total += n;                           // total <- total + |texts|
    peak = std::max(peak, total);
    const int reason = alg1_decide(total, b_min, b_max);
    if (reason >= 0) {
      if (!emit(k + 1, reason)) return SURGE_E_INVALID_ARG;
      total = 0;
      open = false;
    }
  }
  if (open && total > 0 && !emit(n_partitions, REASON_END)) return SURGE_E_INVALID_ARG;
  if (sb_first && F > 0) sb_first[F] = n_partitions;   // trailing empty partitions join the last range
  *n_superbatches = F;
  if (peak_buffered) *peak_buffered = peak;
  return SURGE_OK;
}

surge_status surge_aggregate_ex(const int64_t* sizes, int64_t n_partitions, int64_t b_min, int64_t b_max,
                                int32_t policy, int64_t member_capacity, int64_t* m_partition, int64_t* m_row0,
                                int64_t* m_rows, int64_t sb_capacity, int64_t* sb_first, int32_t* sb_reason,
                                int64_t* n_superbatches, int64_t* n_members, int64_t* peak_buffered) {
  using namespace surge;
  if (!n_superbatches || !n_members || n_partitions < 0 || b_min <= 0 || b_max <= b_min ||
      (n_partitions > 0 && !sizes) || policy < SURGE_BMAX_LABEL || policy > SURGE_BMAX_PREFLUSH)
    return SURGE_E_INVALID_ARG;
  std::vector<AggStep> plan;
  int64_t total = 0, peak = 0, F = 0, M = 0;
  auto seal_sb = [&](int reason) -> bool {
    if (F >= sb_capacity) return false;
    if (sb_reason) sb_reason[F] = reason;
    ++F;
    if (sb_first) sb_first[F] = M;
    total = 0;
    return true;
  };
  if (sb_first && sb_capacity >= 0) sb_first[0] = 0;
  for (int64_t k = 0; k < n_partitions; ++k) {
    const int64_t n = sizes[k];
    if (n < 0) return SURGE_E_INVALID_ARG;
    if (n == 0) continue;                 // completes immediately, never buffered
    plan_add(total, n, b_min, b_max, policy, plan);
    for (const AggStep& st : plan) {
      if (st.seal) {
        if (!seal_sb(st.reason)) return SURGE_E_INVALID_ARG;
        continue;
      }
      if (M >= member_capacity) return SURGE_E_INVALID_ARG;
      if (m_partition) m_partition[M] = k;
      if (m_row0) m_row0[M] = st.row0;
      if (m_rows) m_rows[M] = st.rows;
      ++M;
      total += st.rows;                   // total <- total + |texts|
      peak = std::max(peak, total);
    }
  }
  if (total > 0 && !seal_sb(REASON_END)) return SURGE_E_INVALID_ARG;   // Alg.1 final Flush
  *n_superbatches = F;
  *n_members = M;
  if (peak_buffered) *peak_buffered = peak;
  return SURGE_OK;
}

surge_status surge_set_option(surge_handle h, int32_t option, int64_t value) {
  using namespace surge;
  Ctx* c = h;
  if (int r = check_handle(c)) return surge_status(r);
  switch (option) {
    case SURGE_OPT_ATT_FUSED:
      if (value != 0 && value != 1) return SURGE_E_INVALID_ARG;
      c->model.set_att_fused(value != 0);
      return SURGE_OK;
    case SURGE_OPT_LN_PAIR:
      if (value != 0 && value != 1) return SURGE_E_INVALID_ARG;
      c->model.set_ln_pair(value != 0);
      return SURGE_OK;
    case SURGE_OPT_ATT_TC:
      if (value != 0 && value != 1) return SURGE_E_INVALID_ARG;
      c->model.set_att_tc(value != 0);
      return SURGE_OK;
    case SURGE_OPT_MLP_FUSED:
      if (value != 0 && value != 1) return SURGE_E_INVALID_ARG;
      c->model.set_mlp_fused(value != 0);
      return SURGE_OK;
    case SURGE_OPT_TAIL_FUSED:
      if (value != 0 && value != 1) return SURGE_E_INVALID_ARG;
      c->model.set_tail_fused(value != 0);
      return SURGE_OK;
    case SURGE_OPT_POOLING:
      if (value != SURGE_POOL_MEAN && value != SURGE_POOL_CLS) return SURGE_E_INVALID_ARG;
      c->model.set_pooling(int(value));
      return SURGE_OK;
  }
  return SURGE_E_INVALID_ARG;
}

surge_status surge_profile_enable(surge_handle h, int32_t on) {
  using namespace surge;
  Ctx* c = h;
  if (int r = check_handle(c)) return surge_status(r);
  std::lock_guard<std::mutex> pg(c->prof_mu);
  c->prof.clear();
  c->prof_api.clear();
  c->prof.on = c->prof_api.on = (on != 0);
  return SURGE_OK;
}

surge_status surge_profile_read(surge_handle h, surge_kernel_profile* out, int32_t capacity, int32_t* n_out) {
  using namespace surge;
  Ctx* c = h;
  if (!c || !n_out || (capacity > 0 && !out)) return SURGE_E_INVALID_ARG;
  std::lock_guard<std::mutex> pg(c->prof_mu);
  CUDA_OR_FAIL(c, c->prof.resolve());
  CUDA_OR_FAIL(c, c->prof_api.resolve());
  int32_t n = 0;
  for (int k = 0; k < KK_COUNT && n < capacity; ++k) {
    out[n].kind = k;
    out[n].launches = c->prof.launches[k] + c->prof_api.launches[k];
    out[n].total_ms = c->prof.ms[k] + c->prof_api.ms[k];
    out[n].flops = c->prof.flops[k] + c->prof_api.flops[k];
    out[n].bytes = c->prof.bytes[k] + c->prof_api.bytes[k];
    ++n;
  }
  *n_out = n;
  return SURGE_OK;
}

surge_status surge_op_pack(const int32_t* d_lengths, int64_t n_texts, const int32_t* d_sizes, int64_t n_members,
                           int32_t* d_cu, int32_t* d_row_off, int32_t* d_tok_off, void* stream) {
  if (n_texts < 0 || n_members < 0 || !d_cu || (n_texts > 0 && !d_lengths)) return SURGE_E_INVALID_ARG;
  if (n_members > 0 && (!d_sizes || !d_row_off || !d_tok_off)) return SURGE_E_INVALID_ARG;
  cudaError_t e = surge::launch_pack(d_lengths, n_texts, d_sizes, n_members, d_cu, d_row_off, d_tok_off,
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SURGE_OK : SURGE_E_CUDA;
}

surge_status surge_op_embed_ln(surge_handle h, const int32_t* d_ids, const int32_t* d_cu, int64_t n_texts,
                               uint16_t* d_x, void* stream) {
  using namespace surge;
  Ctx* c = h;
  if (int r = check_handle(c)) return surge_status(r);
  const DeviceModel& m = c->model;
  cudaError_t e = launch_embed_ln(d_ids, d_cu, n_texts, 0, m.word(), m.pos(), m.type(), m.emb_g(), m.emb_b(),
                                  c->shape.d, c->shape.eps, d_x, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SURGE_OK : SURGE_E_CUDA;
}

surge_status surge_op_gemm(const uint16_t* d_a, const uint16_t* d_b, const float* d_bias, const uint16_t* d_res,
                           const float* d_gamma, const float* d_beta, uint16_t* d_c, int64_t M, int32_t N, int32_t K,
                           int32_t epi, float ln_eps, void* stream) {
  using namespace surge;
  if (!d_a || !d_b || !d_bias || !d_c || M <= 0 || N <= 0 || K <= 0 || epi < 0 || epi > 3) return SURGE_E_INVALID_ARG;
  if (epi == EPI_BIAS_LN && (!d_res || !d_gamma || !d_beta)) return SURGE_E_INVALID_ARG;
  if (epi == EPI_BIAS_RES && !d_res) return SURGE_E_INVALID_ARG;
  const int BN = gemm_bn_for(N, K, epi);
  if (BN == 0 || K % 64 != 0) return SURGE_E_INVALID_ARG;
  if (init_tma_encoder() != cudaSuccess) return SURGE_E_CUDA;
  CUtensorMap ta, tb;
  if (make_tmap_bf16(&ta, d_a, uint64_t(M), uint64_t(K), 128) != cudaSuccess) return SURGE_E_CUDA;
  if (make_tmap_bf16(&tb, d_b, uint64_t(N), uint64_t(K), gemm_b_box_rows(N, K, epi)) != cudaSuccess) return SURGE_E_CUDA;
  CUtensorMap tc;
  if (make_tmap_store_bf16(&tc, d_c, uint64_t(M), uint64_t(N)) != cudaSuccess) return SURGE_E_CUDA;
  CUtensorMap tr;
  if (make_tmap_bf16(&tr, epi == EPI_BIAS_LN ? d_res : d_c, uint64_t(M), uint64_t(N), 128) != cudaSuccess)
    return SURGE_E_CUDA;
  GemmArgs g{&ta, &tb, &tc, &tr, M, N, K, epi, d_bias, d_res, d_gamma, d_beta, d_c, ln_eps};
  cudaError_t e = launch_gemm(g, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SURGE_OK : SURGE_E_CUDA;
}

surge_status surge_op_layernorm(const float* d_v, int64_t rows, int32_t d, const float* d_gamma, const float* d_beta,
                                float ln_eps, uint16_t* d_y, void* stream) {
  if (!d_v || !d_gamma || !d_beta || !d_y || rows < 0) return SURGE_E_INVALID_ARG;
  cudaError_t e = surge::launch_layernorm(d_v, rows, d, d_gamma, d_beta, ln_eps, d_y, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SURGE_OK : SURGE_E_CUDA;
}

surge_status surge_op_attention(const uint16_t* d_qkv, const int32_t* d_cu, int64_t n_texts, int32_t heads,
                                int32_t head_dim, uint16_t* d_out, void* stream) {
  if (!d_qkv || !d_cu || !d_out || n_texts < 0 || heads <= 0) return SURGE_E_INVALID_ARG;
  if (n_texts == 0) return SURGE_OK;
  // test entry point: read cu back to find the token count and the longest text (synchronous)
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<int32_t> hcu(static_cast<size_t>(n_texts + 1));
  if (cudaMemcpyAsync(hcu.data(), d_cu, hcu.size() * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return SURGE_E_CUDA;
  int32_t max_len = 0;
  for (int64_t i = 0; i < n_texts; ++i) max_len = std::max(max_len, hcu[i + 1] - hcu[i]);
  const int32_t ntok = hcu[n_texts] - hcu[0];
  std::vector<int32_t> lng;
  for (int64_t i = 0; i < n_texts; ++i)
    if (hcu[i + 1] - hcu[i] > 64) lng.push_back(int32_t(i));
  int32_t off[surge::ATT_LONG_CLASSES + 1];
  surge::group_long_by_class(lng, [&](int32_t i) { return hcu[size_t(i) + 1] - hcu[size_t(i)]; }, off);
  int32_t* win = nullptr;
  int32_t* dl = nullptr;
  if (cudaMalloc(&win, (size_t(ntok) / 64 + 2) * 4) != cudaSuccess) return SURGE_E_OOM;
  if (cudaMalloc(&dl, (lng.size() + 1) * 4) != cudaSuccess) { cudaFree(win); return SURGE_E_OOM; }
  cudaError_t e = cudaMemcpy(dl, lng.data(), lng.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = surge::launch_attention(d_qkv, d_cu, n_texts, hcu[0], ntok, max_len, win, false, heads, head_dim, d_out, st,
                                dl, int32_t(lng.size()), off);
  cudaError_t e2 = cudaStreamSynchronize(st);
  cudaFree(win);
  cudaFree(dl);
  return (e == cudaSuccess && e2 == cudaSuccess) ? SURGE_OK : SURGE_E_CUDA;
}

surge_status surge_op_meanpool_l2(const uint16_t* d_x, const int32_t* d_cu, int64_t n_texts, int32_t d, float* d_out,
                                  void* stream) {
  if (!d_x || !d_cu || !d_out || n_texts < 0) return SURGE_E_INVALID_ARG;
  cudaError_t e = surge::launch_meanpool_l2(d_x, d_cu, n_texts, 0, d, d_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SURGE_OK : SURGE_E_CUDA;
}

surge_status surge_lpt_plan(const int32_t* h_lengths, int64_t n_texts, const int64_t* h_sizes, int64_t n_members,
                            int32_t world, int64_t capacity, int64_t* first_row, int64_t* n_rows, int64_t* member,
                            int64_t* tokens, int32_t* rank, int64_t* n_pieces) {
  using namespace surge;
  if (!n_pieces || world < 1 || n_texts < 0 || n_members < 0) return SURGE_E_INVALID_ARG;
  if ((n_texts > 0 && !h_lengths) || (n_members > 0 && !h_sizes)) return SURGE_E_INVALID_ARG;
  int64_t s = 0;
  for (int64_t j = 0; j < n_members; ++j) {
    if (h_sizes[j] < 0) return SURGE_E_INVALID_ARG;
    s += h_sizes[j];
  }
  if (s != n_texts) return SURGE_E_INVALID_ARG;
  std::vector<LptPiece> out;
  lpt_plan(h_lengths, n_texts, h_sizes, n_members, world, out);
  *n_pieces = int64_t(out.size());
  if (capacity < *n_pieces) return SURGE_E_INVALID_ARG;
  for (size_t i = 0; i < out.size(); ++i) {
    if (first_row) first_row[i] = out[i].first_row;
    if (n_rows) n_rows[i] = out[i].n_rows;
    if (member) member[i] = out[i].member;
    if (tokens) tokens[i] = out[i].tokens;
    if (rank) rank[i] = out[i].rank;
  }
  return SURGE_OK;
}

}  // extern "C"
