/*
 * surge.h -- C ABI of libsurge: the data-parallel hot path of SURGE (arxiv 2605.01060)
 * on NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (LaTeX source), "S:n" = SPEC.md line n.
 *
 * The path:  partitions arrive in key order -> SuperBatch aggregation under
 * the two-threshold policy (Alg.1 AddPartition) -> on a flush, the buffered texts are
 * packed without padding into one varlen token stream (Flush) -> ONE encode of the
 * whole SuperBatch: BERT-class encoder forward, masked mean-pool, L2 normalisation
 * -> per-partition slices E[start:end] handed back as soon as they land.
 *
 * Problem statement: input = partitions {(k_i, T_i)}, sum n_i = N; output = a map
 * k_i -> E_i in R^{n_i x d}.  This ABI takes pre-tokenised texts (token ids); tokenisation is
 * out of scope.
 *
 * Conventions
 *   - Every function returns surge_status (0 = OK, < 0 = error) unless noted.
 *   - After a CUDA error the handle is POISONED: every later call returns SURGE_E_CUDA;
 *     surge_last_error() gives the text.  Nothing ever falls back to a CPU path: if the CUDA
 *     device or the sm_100a kernels are unavailable, surge_create fails with SURGE_E_CUDA.
 *   - Threading: ONE producer thread calls submit/finish/reset; poll/release/stats may be
 *     called from any thread (internally synchronised).
 *   - Pointers documented as "device" are CUDA device pointers on cfg.device; "host" pointers
 *     are ordinary (pageable or pinned) host memory.  `stream` arguments are cudaStream_t cast
 *     to void* (NULL = the legacy default stream).
 */
#ifndef SURGE_H_
#define SURGE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SURGE_OK = 0,
  SURGE_E_INVALID_ARG = -1,   /* bad pointer / size / config value                              */
  SURGE_E_DUPLICATE_ID = -2,  /* partition id already submitted (keys unique + grouped)  */
  SURGE_E_STATE = -3,         /* call not valid in the current state (e.g. submit after finish) */
  SURGE_E_TOO_LONG = -4,      /* a text length outside [1, max_position] (no silent truncation) */
  SURGE_E_OOM = -5,           /* device or pinned-host allocation failed                        */
  SURGE_E_CUDA = -6,          /* CUDA runtime/driver error, or no sm_100 device (poisons)       */
  SURGE_E_NCCL = -7,          /* NCCL unavailable or an NCCL call failed (surge_create_replicated) */
  SURGE_E_AGAIN = -8,         /* non-blocking submit would block (backpressure)                 */
  SURGE_E_TOKEN_ID = -9       /* a token id outside [0, vocab_size)                             */
} surge_status;

typedef struct surge_ctx* surge_handle;

/*
 * What B_max does (surge_config.bmax_policy; readings R2/R3/R23):
 *   SURGE_BMAX_LABEL    literal Alg.1: total >= b_max labels the flush Safety; a partition
 *                       is never split and flushes together with the buffer (default).
 *   SURGE_BMAX_SPLIT    P:1271 "splitting the oversized partition across consecutive SuperBatches":
 *                       the arriving partition's texts fill the buffer up to exactly b_max, which
 *                       flushes (Safety); the rest continues into the next SuperBatches.  Every
 *                       SuperBatch holds <= b_max texts (the Lemma's S <= B_max); a partition
 *                       may come back as several pieces (row_begin), possibly from several SuperBatches.
 *   SURGE_BMAX_PREFLUSH P:304 / P:308: before adding a partition that would push the buffer past b_max
 *                       the buffer flushes (Safety); a partition of > b_max texts is then emitted as
 *                       its own SuperBatch.  S <= b_max unless one oversized partition is alone.
 */
#define SURGE_BMAX_LABEL 0
#define SURGE_BMAX_SPLIT 1
#define SURGE_BMAX_PREFLUSH 2

/* Output element types (surge_config.out_dtype, surge_flushed.dtype). */
#define SURGE_F32 0    /* float32 unit vectors: the paper's output (pa.float32()), default */
#define SURGE_BF16 1   /* bf16 bit patterns (uint16): half the D2H / host bytes per text           */

/*
 * Encoder configuration (BERT class) + aggregation policy.
 *   Encoder classes (reading #12): MiniLM-L6 class 30522/512/2, d=384, L=6, H=12,
 *   ffn=1536; bge-base class d=768, L=12, H=12, ffn=3072; bge-large class d=1024, L=24, H=16,
 *   ffn=4096; toy (C1) vocab 1024, max_pos 64, d=64, L=2, H=4, ffn=256.
 *   Supported on the sm_100a path in this build: hidden in {64, 384, 768, 1024}, head_dim in
 *   {16, 32, 64}, an even number of heads, ffn a multiple of 64 (others return SURGE_E_INVALID_ARG
 *   at create).  hidden 64/384 fuse LayerNorm into the GEMM epilogue; 768/1024 use an fp32
 *   pre-LN pass + a row LayerNorm kernel.
 *   Thresholds: b_min = efficiency trigger, b_max = memory-safety trigger, texts,
 *   0 < b_min < b_max.
 *   Sharding: the process encodes only the LPT pieces of every SuperBatch assigned to `rank`
 *   out of `world_size` (north star).  Every rank must be fed the
 *   same partition stream; world_size = 1 encodes everything.  (SURVEY.md §8(b) sketches a
 *   single-process `num_gpus`; this library runs one process per GPU, so each handle names its
 *   own rank and device instead, and world_size plays the role of num_gpus.)
 */
typedef struct {
  int32_t vocab_size, max_position, type_vocab_size;
  int32_t hidden, layers, heads, ffn;
  float ln_eps;                 /* LayerNorm epsilon, 1e-12 for BERT                            */
  int64_t b_min, b_max;         /* two-threshold policy, texts                                  */
  int32_t rank, world_size;     /* LPT shard owned by this process; 0, 1 for single GPU         */
  int32_t device;               /* CUDA device ordinal                                          */
  int32_t chunk_tokens;         /* tokens per encode chunk; 0 = auto (524288)                   */
  int32_t max_inflight;         /* SuperBatches queued/encoding before submit blocks; 0 = 2      */
  int32_t nonblocking_submit;   /* 1: submit returns SURGE_E_AGAIN instead of blocking           */
  int32_t weights_on_device;    /* 1: `weights` passed to surge_create is a device pointer       */
  int32_t out_dtype;            /* SURGE_F32 (default) or SURGE_BF16: element type of every output
                                   row (streaming pieces and the device-level d_out buffers)      */
  int32_t bmax_policy;          /* SURGE_BMAX_LABEL (default), SURGE_BMAX_SPLIT, SURGE_BMAX_PREFLUSH */
} surge_config;

/*
 * Weight blob: bf16 bit patterns (uint16), HF BERT tensor order, each tensor row-major,
 * concatenated without padding (d = hidden, f = ffn, V = vocab_size, Pm = max_position):
 *   word_embeddings [V,d], position_embeddings [Pm,d], token_type_embeddings [type_vocab,d],
 *   embeddings.LayerNorm weight [d], bias [d],
 *   then per layer l = 0..L-1:
 *     query.weight [d,d], query.bias [d], key.weight [d,d], key.bias [d],
 *     value.weight [d,d], value.bias [d], attention.output.dense.weight [d,d], .bias [d],
 *     attention.output.LayerNorm weight [d], bias [d],
 *     intermediate.dense.weight [f,d], .bias [f], output.dense.weight [d,f], .bias [d],
 *     output.LayerNorm weight [d], bias [d].
 * Linear weights are [out, in] (y = x W^T + b).  n_weights must equal the total element count.
 * Ownership: copied at create; the caller keeps (and may free) its buffer.
 */
surge_status surge_create(const surge_config* cfg, const uint16_t* weights, size_t n_weights,
                          surge_handle* out);

/*
 * Multi-GPU creation (north star: "weights are replicated once via an NCCL broadcast"; SURVEY.md
 * §8(e) K11).  One process per GPU; all cfg.world_size ranks call surge_create_replicated
 * concurrently with the same 128-byte NCCL unique id (obtained once by rank 0 through
 * surge_nccl_unique_id and handed to the other ranks by the caller, e.g. over its process group).
 * The library opens an NCCL communicator over the world, broadcasts the weight blob from rank 0
 * (one ncclBroadcast over NVLink / NVSwitch; `weights` is read on rank 0 only and may be NULL
 * elsewhere; host or device per cfg.weights_on_device), then builds the handle as surge_create.
 * The communicator lives until surge_destroy.  No per-SuperBatch collective follows: every rank
 * encodes its own LPT pieces and returns them itself.
 * Errors: SURGE_E_NCCL (libnccl.so.2 unavailable, or an NCCL call failed), else as surge_create.
 */
surge_status surge_nccl_unique_id(uint8_t* id /* [128] out */);
surge_status surge_create_replicated(const surge_config* cfg, const uint8_t* nccl_id, const uint16_t* weights,
                                     size_t n_weights, surge_handle* out);

/*
 * AddPartition (Alg.1).  token_ids: host, sum(lengths) int32 ids in [0, vocab),
 * the n_texts texts concatenated; lengths: host, n_texts int32 values in [1, max_position],
 * each INCLUDING [CLS]/[SEP].  Both are copied before return (Alg.1 `copy(texts)`).
 * If the running total reaches b_max (Safety) or b_min (Efficiency) the SuperBatch is sealed
 * and handed to the device pipeline asynchronously (one encode per SuperBatch).
 * n_texts == 0 is accepted: the partition completes immediately with 0 rows (rank 0 only).
 * Errors: SURGE_E_DUPLICATE_ID (id seen before), SURGE_E_TOO_LONG, SURGE_E_TOKEN_ID,
 * SURGE_E_STATE (after finish), SURGE_E_AGAIN (nonblocking_submit and the pipeline is full;
 * nothing was consumed), SURGE_E_INVALID_ARG (also when the open SuperBatch would reach 2^31
 * tokens: device token offsets are int32; nothing was consumed).
 */
surge_status surge_submit_partition(surge_handle h, uint64_t partition_id,
                                    const int32_t* token_ids, const int32_t* lengths,
                                    int64_t n_texts);

/* End of stream: Alg.1 final Flush of the residual buffer; no flush if empty. */
surge_status surge_finish(surge_handle h);

/*
 * A completed output piece.  For world_size == 1 every partition yields exactly one record
 * with row_begin = 0 and n_rows = partition_rows.  For world_size > 1 a partition may be split
 * into LPT pieces encoded on different ranks; each rank returns its own pieces, and the union
 * over ranks covers every row of every partition exactly once.
 *   data: host, pinned, library-owned, row-major n_rows x d unit vectors of element type `dtype`
 *         (SURGE_F32 float32 per P:406, or SURGE_BF16; rows in submission order).  Read-only; valid
 *         until surge_release(h, rec) (the buffer lifetime rule of P:413) or surge_destroy.
 */
typedef struct {
  uint64_t partition_id;
  int64_t row_begin;        /* first row of this piece within the partition        */
  int64_t n_rows;           /* rows in this piece                                   */
  int64_t partition_rows;   /* n_k of the whole partition                           */
  int32_t d;                /* embedding dimension (= hidden)                        */
  int32_t dtype;            /* SURGE_F32 or SURGE_BF16 (the handle's out_dtype)      */
  const void* data;
  int64_t superbatch;       /* index of the SuperBatch that encoded it (-1: n_k = 0) */
  uint64_t token;           /* opaque, for surge_release                            */
} surge_flushed;

/*
 * Pop up to max_items completed pieces, in completion order.  Waits up to timeout_ms
 * (0 = do not wait, < 0 = wait forever) for at least one.  *n_out = number returned; returns
 * SURGE_OK with *n_out == 0 on timeout.
 */
surge_status surge_poll_flushed(surge_handle h, surge_flushed* out, int64_t max_items,
                                int32_t timeout_ms, int64_t* n_out);

/* Return a polled piece's buffer to the library's pinned pool.  Each polled record is released
 * exactly once: a record that was not polled from the current stream (before the last
 * surge_reset), or one released twice, returns SURGE_E_INVALID_ARG and changes nothing. */
surge_status surge_release(surge_handle h, const surge_flushed* rec);

/* Pieces sealed into SuperBatches but not yet returned by poll (0 => everything delivered). */
surge_status surge_pending(surge_handle h, int64_t* n_pending);

/* After finish, once every piece was polled AND released: start a new stream (keeps weights and
 * pools; the released buffers are reused).  SURGE_E_STATE otherwise. */
surge_status surge_reset(surge_handle h);

typedef struct {
  int64_t superbatches;          /* F: encoder invocations (one per SuperBatch, reading #17)    */
  int64_t safety_flushes;        /* flushes fired by the b_max branch                           */
  int64_t efficiency_flushes;
  int64_t texts, tokens;         /* submitted                                                   */
  int64_t local_texts, local_tokens;   /* encoded by this rank                                  */
  int64_t peak_buffered_texts;   /* aggregator buffer peak; Lemma: <= b_min - 1 + max n_k       */
  int64_t peak_buffered_bytes;   /* staging bytes (ids + lengths) of the open SuperBatch, peak   */
  int64_t peak_inflight_texts;   /* sealed-but-not-delivered texts, peak                        */
  int64_t max_partition_seen;    /* max n_k submitted so far                                    */
  int64_t kernel_launches;       /* CUDA kernels launched by this handle                        */
  double ttfo_s;                 /* first submit -> first piece available to poll (-1: none)     */
  double init_s;                 /* surge_create wall time                                      */
  double encode_ms_total;        /* sum of per-SuperBatch device time (CUDA events)             */
} surge_stats;

surge_status surge_get_stats(surge_handle h, surge_stats* out);

/* Per-SuperBatch record (flush log). reason: 0 efficiency, 1 safety, 2 end of stream. */
typedef struct {
  int64_t index;
  int32_t reason;
  int32_t n_members;
  int64_t n_texts, n_tokens;          /* whole SuperBatch                                      */
  int64_t local_texts, local_tokens;  /* this rank's LPT share                                 */
  int32_t local_pieces;
  int32_t done;                       /* 1 when every local piece has landed on the host       */
  double encode_ms;                   /* device time of pack + encode + pool (CUDA events)     */
} surge_superbatch_info;

surge_status surge_get_superbatch(surge_handle h, int64_t index, surge_superbatch_info* out);
/* Member partition ids of SuperBatch `index`, in arrival order (bounds order). */
surge_status surge_get_superbatch_members(surge_handle h, int64_t index, uint64_t* ids,
                                          int64_t capacity, int64_t* n_out);

const char* surge_last_error(surge_handle h);   /* never NULL; "" when no error; h may be NULL */
void surge_destroy(surge_handle h);             /* drains the pipeline and frees everything    */

/* ---------------------------------------------------------------------------------------------
 * Device-level entry points (inputs already resident in HBM).  These run the same sm_100a
 * kernels the streaming path uses; the tests and bench.py call them through the Python binding.
 * ------------------------------------------------------------------------------------------- */

/*
 * Encode one packed SuperBatch (or any run of whole texts) that is already on the device:
 *   d_ids     device int32[sum(lengths)]  token ids, texts concatenated (varlen, no padding)
 *   d_lengths device int32[n_texts]        text lengths
 *   h_lengths host   int32[n_texts]        the same lengths (host copy, used to cut chunks)
 *   d_out     device [n_texts * d]         unit-norm embeddings, row i = text i, element type
 *                                          cfg.out_dtype (float32, or bf16 bits)
 * Runs K1 pack -> per chunk: K3 embed+LN -> L x (QKV GEMM, varlen attention, out-proj+res+LN,
 * FFN1+GELU, FFN2+res+LN) -> K9 mean-pool+L2, enqueued on `stream`; returns without syncing.
 */
surge_status surge_encode_packed(surge_handle h, const int32_t* d_ids, const int32_t* d_lengths,
                                 const int32_t* h_lengths, int64_t n_texts, void* d_out,
                                 void* stream);

/*
 * K1 SuperBatch packer (Flush `bounds`), device in/out:
 *   d_lengths int32[n_texts], d_sizes int32[n_members] (n_k of each member, arrival order)
 *   -> d_cu int32[n_texts+1] (cu[0]=0, cu[i+1]=cu[i]+len_i),
 *      d_row_off int32[n_members+1], d_tok_off int32[n_members+1].
 * Requires sum(lengths) < 2^31.
 */
surge_status surge_op_pack(const int32_t* d_lengths, int64_t n_texts, const int32_t* d_sizes,
                           int64_t n_members, int32_t* d_cu, int32_t* d_row_off,
                           int32_t* d_tok_off, void* stream);

/* K3: X[t] = LN_e(word[id_t] + pos[t - cu[s]] + type[0]), device bf16 out [n_tokens x d]. */
surge_status surge_op_embed_ln(surge_handle h, const int32_t* d_ids, const int32_t* d_cu,
                               int64_t n_texts, uint16_t* d_x, void* stream);

/*
 * tcgen05 GEMM with fused epilogue, device pointers, bf16 bit patterns as uint16:
 *   C[M x N] = epi(A[M x K] * B[N x K]^T + bias[N])
 *   epi = 0: identity; 1: exact GELU; 2: LayerNorm(. + R[M x N]) * gamma[N] + beta[N] (N = full row);
 *   epi = 3: . + R[M x N] written as FLOAT32 (d_c is then a float* [M x N]): the pre-LayerNorm rows
 *            of hidden sizes whose row does not fit the fused epilogue (finish with surge_op_layernorm).
 * bias/gamma/beta: float32[N].  Supported: K % 64 == 0; N per epilogue as the encoder needs
 * (epi 0/1: N % 64 == 0; epi 2: N in {64, 384}; epi 3: N % 128 == 0); any M >= 1.
 */
surge_status surge_op_gemm(const uint16_t* d_a, const uint16_t* d_b, const float* d_bias,
                           const uint16_t* d_res, const float* d_gamma, const float* d_beta,
                           uint16_t* d_c, int64_t M, int32_t N, int32_t K, int32_t epi,
                           float ln_eps, void* stream);

/* Row LayerNorm (post-LN of BERT, eps ln_eps, biased variance): v float32 [rows x d] -> bf16 y,
 * y = (v - mean) / sqrt(var + eps) * gamma + beta; d in {768, 1024}.  Device pointers. */
surge_status surge_op_layernorm(const float* d_v, int64_t rows, int32_t d, const float* d_gamma, const float* d_beta,
                                float ln_eps, uint16_t* d_y, void* stream);

/* K5: varlen attention, qkv bf16 [T x 3*heads*head_dim] (Q | K | V), out bf16 [T x heads*head_dim]. */
surge_status surge_op_attention(const uint16_t* d_qkv, const int32_t* d_cu, int64_t n_texts,
                                int32_t heads, int32_t head_dim, uint16_t* d_out, void* stream);

/* K9: e_s = v/max(||v||,1e-12), v = mean over the text's rows of X (bf16 [T x d]) -> float32 [n x d]. */
surge_status surge_op_meanpool_l2(const uint16_t* d_x, const int32_t* d_cu, int64_t n_texts,
                                  int32_t d, float* d_out, void* stream);

/*
 * LPT shard plan of one SuperBatch (host-only, pure function; north star / DESIGN.md):
 * pieces <= ceil(T/(8G)) tokens cut at text boundaries, sorted (tokens desc, first_row asc),
 * each to the rank with min (load, rank).  world == 1: one piece per member.
 *   h_lengths int32[n_texts], h_sizes int64[n_members]  -> up to `capacity` pieces written in
 *   global-row order: first_row, n_rows, member, tokens, rank (int64 each array).
 * *n_pieces = number of pieces (SURGE_E_INVALID_ARG if capacity is too small).
 */
surge_status surge_lpt_plan(const int32_t* h_lengths, int64_t n_texts, const int64_t* h_sizes,
                            int64_t n_members, int32_t world, int64_t capacity,
                            int64_t* first_row, int64_t* n_rows, int64_t* member,
                            int64_t* tokens, int32_t* rank, int64_t* n_pieces);

/*
 * Alg.1 AddPartition/Flush decisions as a pure host function (the same aggregator the streaming
 * path runs): partitions of `sizes` (int64[n_partitions], arrival order) -> SuperBatches.
 *   sb_first int64[capacity+1]: SuperBatch j = partitions [sb_first[j], sb_first[j+1])
 *   sb_reason int32[capacity]:  0 efficiency, 1 safety, 2 end of stream (final residual)
 * Zero-size partitions are skipped (they complete immediately) but stay inside the ranges.
 * *n_superbatches = count F; *peak_buffered = max buffered texts (Lemma P:477-487).
 */
surge_status surge_aggregate(const int64_t* sizes, int64_t n_partitions, int64_t b_min, int64_t b_max,
                             int64_t capacity, int64_t* sb_first, int32_t* sb_reason,
                             int64_t* n_superbatches, int64_t* peak_buffered);

/*
 * Alg.1 under a B_max policy as a pure host function (the aggregator the streaming path runs):
 * partitions of `sizes` (arrival order) -> SuperBatches of members, a member being a partition or,
 * under SURGE_BMAX_SPLIT, a contiguous piece of one.
 *   member j: m_partition[j] (index into sizes), m_row0[j] (first row within the partition),
 *             m_rows[j] (texts); members are listed SuperBatch by SuperBatch, in stream order.
 *   SuperBatch i = members [sb_first[i], sb_first[i+1]), reason sb_reason[i] (0 efficiency,
 *             1 safety, 2 end of stream); sb_first has n_superbatches + 1 entries.
 * Zero-size partitions never enter a SuperBatch.  SURGE_E_INVALID_ARG if a capacity is too small.
 */
surge_status surge_aggregate_ex(const int64_t* sizes, int64_t n_partitions, int64_t b_min, int64_t b_max,
                                int32_t policy, int64_t member_capacity, int64_t* m_partition, int64_t* m_row0,
                                int64_t* m_rows, int64_t sb_capacity, int64_t* sb_first, int32_t* sb_reason,
                                int64_t* n_superbatches, int64_t* n_members, int64_t* peak_buffered);

/*
 * One SuperBatch, device-resident (the step surge_submit_partition's pipeline runs per flush):
 *   d_ids     device int32[sum(lengths)], the SuperBatch's texts concatenated (Flush allTexts)
 *   d_lengths device int32[n_texts];  h_lengths host int32[n_texts] (same values, cuts chunks)
 *   h_sizes   host int64[n_members], texts of each member in arrival order (bounds; a
 *             member may be a piece of a partition, see surge_aggregate_ex)
 *   d_out     device [n_texts * d] (cfg.out_dtype): rows of THIS rank's LPT pieces are written at their
 *             SuperBatch row positions (all rows when world_size == 1); other rows are untouched.
 * K2 LPT plan (world_size > 1) -> gather of the rank's pieces -> K1 pack -> encoder chunks ->
 * K9 pool -> scatter of the rank's rows into d_out (device-to-device), on `stream`.
 */
surge_status surge_encode_superbatch(surge_handle h, const int32_t* d_ids, const int32_t* d_lengths,
                                     const int32_t* h_lengths, int64_t n_texts, const int64_t* h_sizes,
                                     int64_t n_members, void* d_out, void* stream);

/*
 * Per-kernel-class device timing (CUDA events around every launch, on the launching stream).
 * Enable before a timed region, read after synchronising.  Classes: 0 embed_ln, 1 gemm_qkv,
 * 2 attention, 3 gemm_out_ln, 4 gemm_ffn1_gelu, 5 gemm_ffn2_ln, 6 meanpool_l2, 7 pack,
 * 8 gemm_qkv_attn (K4 + K5 fused), 9 gemm_mlp (K7 + K8 fused), 10 gemm_tail (K6 + K7 + K8 fused).
 *   flops/bytes: ALGORITHMIC work of the launches (2*M*N*K for GEMMs; 4*d*sum(l^2) attention
 *   flops; minimal HBM bytes in+out for every class), summed over launches.
 */
typedef struct {
  int32_t kind;
  int64_t launches;
  double total_ms;
  double flops;
  double bytes;
} surge_kernel_profile;

/*
 * Execution options (not part of the paper's method; they select between equivalent kernel paths).
 *   SURGE_OPT_ATT_FUSED (default 1): 1 = K4 QKV GEMM and K5 attention run as one kernel
 *     (attention in the GEMM epilogue, QKV never written to HBM) for chunks whose texts are all
 *     <= 128 tokens; 0 = separate K4 GEMM + K5 attention kernels everywhere.  Both paths compute
 *     bit-identical embeddings (shared attention arithmetic).
 * Call only while the handle is idle (no SuperBatch in flight).  Unknown option -> SURGE_E_INVALID_ARG.
 */
#define SURGE_OPT_ATT_FUSED 1
/*   SURGE_OPT_MLP_FUSED (default 1): 1 = K7 FFN1 + GELU and K8 FFN2 + residual + LN run as one kernel
 *     (H kept on chip; hidden size 384 or 64); 0 = two GEMM kernels.  Bit-identical results. */
#define SURGE_OPT_MLP_FUSED 2
/*   SURGE_OPT_TAIL_FUSED (default 1; effective with SURGE_OPT_MLP_FUSED): K6 out-projection +
 *     residual + LN also runs inside the fused MLP kernel (X1 kept on chip).  Bit-identical. */
#define SURGE_OPT_TAIL_FUSED 3
/*   SURGE_OPT_POOLING (default SURGE_POOL_MEAN): SURGE_POOL_MEAN = masked mean over all tokens of
 *     the text incl. [CLS]/[SEP] (all-MiniLM-L6-v2 convention, reading R6);
 *     SURGE_POOL_CLS = the [CLS] token's hidden state (bge's native pooling).
 *     Either is followed by L2 normalisation.  Changes the embeddings, not the schedule. */
#define SURGE_OPT_POOLING 4
#define SURGE_POOL_MEAN 0
#define SURGE_POOL_CLS 1
/*   SURGE_OPT_ATT_TC (default 0; effective with SURGE_OPT_ATT_FUSED, hidden size 384, d_h = 32): the
 *     fused QKV + attention kernel computes S = Q K^T and O = P V on the tcgen05 tensor cores (Q and
 *     P read from tensor memory; one CTA per SM); 0 = the CTA-pair kernel whose attention runs on
 *     mma.sync in the GEMM epilogue.  Same bf16 Q/K/V/P values and softmax formula; the fp32
 *     accumulation order differs, so the two agree to rounding (not bit for bit). */
#define SURGE_OPT_ATT_TC 5
/*   SURGE_OPT_LN_PAIR (default 1; hidden size 768 or 1024): the out-projection and FFN2 GEMMs fuse their
 *     residual + LayerNorm, a cluster of two CTAs splitting each row and exchanging the row statistics
 *     through distributed shared memory; 0 = fp32 pre-LN rows to HBM + a row-LayerNorm kernel.  The fp32
 *     summation order of the statistics differs between the two (agreement to rounding). */
#define SURGE_OPT_LN_PAIR 6
surge_status surge_set_option(surge_handle h, int32_t option, int64_t value);

surge_status surge_profile_enable(surge_handle h, int32_t on);   /* on: clears counters */
surge_status surge_profile_read(surge_handle h, surge_kernel_profile* out, int32_t capacity,
                                int32_t* n_out);

/* Library version string (never NULL). */
const char* surge_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SURGE_H_ */
