"""Thin ctypes binding of libsurge (include/surge.h).  Argument marshalling only.

Every function here has the name of the C entry point it calls; every step of the path runs
inside libsurge.so (sm_100a kernels + the C++ host runtime).  There is no fallback: importing
this module raises ImportError if libsurge.so has not been built, and surge_create raises
SurgeError(SURGE_E_CUDA) without an sm_100 GPU.

Device pointers may be passed as ints or as torch CUDA tensors (their data_ptr()); host arrays
are numpy arrays.  torch is used only by callers for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import threading
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SURGE_LIB: alternative build of the same library (tuning experiments, scripts/); default in-tree
LIB_PATH = os.environ.get("SURGE_LIB") or os.path.join(_HERE, "libsurge.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libsurge.so not built at {LIB_PATH}: run __graft_entry__.build() "
                      "(python paper_2605_01060_b200/build.py)")
lib = C.CDLL(LIB_PATH)

SURGE_OK, SURGE_E_INVALID_ARG, SURGE_E_DUPLICATE_ID, SURGE_E_STATE = 0, -1, -2, -3
SURGE_E_TOO_LONG, SURGE_E_OOM, SURGE_E_CUDA, SURGE_E_NCCL, SURGE_E_AGAIN, SURGE_E_TOKEN_ID = -4, -5, -6, -7, -8, -9
STATUS_NAMES = {0: "SURGE_OK", -1: "SURGE_E_INVALID_ARG", -2: "SURGE_E_DUPLICATE_ID", -3: "SURGE_E_STATE",
                -4: "SURGE_E_TOO_LONG", -5: "SURGE_E_OOM", -6: "SURGE_E_CUDA", -7: "SURGE_E_NCCL",
                -8: "SURGE_E_AGAIN", -9: "SURGE_E_TOKEN_ID"}
EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_LN = 0, 1, 2
REASONS = {0: "efficiency", 1: "safety", 2: "end_of_stream"}


class SurgeError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class surge_config(C.Structure):
    _fields_ = [("vocab_size", C.c_int32), ("max_position", C.c_int32), ("type_vocab_size", C.c_int32),
                ("hidden", C.c_int32), ("layers", C.c_int32), ("heads", C.c_int32), ("ffn", C.c_int32),
                ("ln_eps", C.c_float), ("b_min", C.c_int64), ("b_max", C.c_int64),
                ("rank", C.c_int32), ("world_size", C.c_int32), ("device", C.c_int32),
                ("chunk_tokens", C.c_int32), ("max_inflight", C.c_int32), ("nonblocking_submit", C.c_int32),
                ("weights_on_device", C.c_int32), ("out_dtype", C.c_int32), ("bmax_policy", C.c_int32)]


class surge_flushed(C.Structure):
    _fields_ = [("partition_id", C.c_uint64), ("row_begin", C.c_int64), ("n_rows", C.c_int64),
                ("partition_rows", C.c_int64), ("d", C.c_int32), ("dtype", C.c_int32),
                ("data", C.c_void_p), ("superbatch", C.c_int64), ("token", C.c_uint64)]


class surge_stats(C.Structure):
    _fields_ = [("superbatches", C.c_int64), ("safety_flushes", C.c_int64), ("efficiency_flushes", C.c_int64),
                ("texts", C.c_int64), ("tokens", C.c_int64), ("local_texts", C.c_int64),
                ("local_tokens", C.c_int64), ("peak_buffered_texts", C.c_int64),
                ("peak_buffered_bytes", C.c_int64), ("peak_inflight_texts", C.c_int64),
                ("max_partition_seen", C.c_int64), ("kernel_launches", C.c_int64), ("ttfo_s", C.c_double),
                ("init_s", C.c_double), ("encode_ms_total", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class surge_kernel_profile(C.Structure):
    _fields_ = [("kind", C.c_int32), ("launches", C.c_int64), ("total_ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


KERNEL_KINDS = ("embed_ln", "gemm_qkv", "attention", "gemm_out_ln", "gemm_ffn1_gelu", "gemm_ffn2_ln",
                "meanpool_l2", "pack", "gemm_qkv_attn", "gemm_mlp", "gemm_tail")
SURGE_OPT_ATT_FUSED = 1
SURGE_OPT_MLP_FUSED = 2
SURGE_OPT_TAIL_FUSED = 3
SURGE_OPT_POOLING = 4
SURGE_OPT_ATT_TC = 5
SURGE_OPT_LN_PAIR = 6
SURGE_POOL_MEAN, SURGE_POOL_CLS = 0, 1
SURGE_F32, SURGE_BF16 = 0, 1
SURGE_BMAX_LABEL, SURGE_BMAX_SPLIT, SURGE_BMAX_PREFLUSH = 0, 1, 2
BMAX_POLICIES = {"label": 0, "split": 1, "preflush": 2}


class surge_superbatch_info(C.Structure):
    _fields_ = [("index", C.c_int64), ("reason", C.c_int32), ("n_members", C.c_int32), ("n_texts", C.c_int64),
                ("n_tokens", C.c_int64), ("local_texts", C.c_int64), ("local_tokens", C.c_int64),
                ("local_pieces", C.c_int32), ("done", C.c_int32), ("encode_ms", C.c_double)]


_p = C.c_void_p
_i32p, _i64p, _u16p, _f32p, _u64p = (C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_uint16),
                                     C.POINTER(C.c_float), C.POINTER(C.c_uint64))
_SIGS = {
    "surge_version": (C.c_char_p, []),
    "surge_create": (C.c_int, [C.POINTER(surge_config), _p, C.c_size_t, C.POINTER(_p)]),
    "surge_nccl_unique_id": (C.c_int, [_p]),
    "surge_create_replicated": (C.c_int, [C.POINTER(surge_config), _p, _p, C.c_size_t, C.POINTER(_p)]),
    "surge_submit_partition": (C.c_int, [_p, C.c_uint64, _p, _p, C.c_int64]),
    "surge_finish": (C.c_int, [_p]),
    "surge_poll_flushed": (C.c_int, [_p, C.POINTER(surge_flushed), C.c_int64, C.c_int32, _i64p]),
    "surge_release": (C.c_int, [_p, C.POINTER(surge_flushed)]),
    "surge_pending": (C.c_int, [_p, _i64p]),
    "surge_reset": (C.c_int, [_p]),
    "surge_get_stats": (C.c_int, [_p, C.POINTER(surge_stats)]),
    "surge_get_superbatch": (C.c_int, [_p, C.c_int64, C.POINTER(surge_superbatch_info)]),
    "surge_get_superbatch_members": (C.c_int, [_p, C.c_int64, _p, C.c_int64, _i64p]),
    "surge_last_error": (C.c_char_p, [_p]),
    "surge_destroy": (None, [_p]),
    "surge_encode_packed": (C.c_int, [_p, _p, _p, _p, C.c_int64, _p, _p]),
    "surge_op_pack": (C.c_int, [_p, C.c_int64, _p, C.c_int64, _p, _p, _p, _p]),
    "surge_op_embed_ln": (C.c_int, [_p, _p, _p, C.c_int64, _p, _p]),
    "surge_op_gemm": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                C.c_float, _p]),
    "surge_op_attention": (C.c_int, [_p, _p, C.c_int64, C.c_int32, C.c_int32, _p, _p]),
    "surge_op_layernorm": (C.c_int, [_p, C.c_int64, C.c_int32, _p, _p, C.c_float, _p, _p]),
    "surge_op_meanpool_l2": (C.c_int, [_p, _p, C.c_int64, C.c_int32, _p, _p]),
    "surge_aggregate_ex": (C.c_int, [_p, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int64, _p, _p, _p,
                                     C.c_int64, _p, _p, _i64p, _i64p, _i64p]),
    "surge_aggregate": (C.c_int, [_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _p, _p, _i64p, _i64p]),
    "surge_encode_superbatch": (C.c_int, [_p, _p, _p, _p, C.c_int64, _p, C.c_int64, _p, _p]),
    "surge_profile_enable": (C.c_int, [_p, C.c_int32]),
    "surge_set_option": (C.c_int, [_p, C.c_int32, C.c_int64]),
    "surge_profile_read": (C.c_int, [_p, C.POINTER(surge_kernel_profile), C.c_int32, C.POINTER(C.c_int32)]),
    "surge_lpt_plan": (C.c_int, [_p, C.c_int64, _p, C.c_int64, C.c_int32, C.c_int64, _p, _p, _p, _p, _p,
                                 _i64p]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


def _ptr(x):
    """Device/host address of a torch tensor, numpy array, int or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(type(x))


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream   # torch.cuda.Stream


def _check(h, st: int, what: str = ""):
    if st != SURGE_OK:
        msg = lib.surge_last_error(h).decode() if h else ""
        raise SurgeError(st, f"{what} {msg}".strip())
    return st


def surge_version() -> str:
    return lib.surge_version().decode()


def make_config(enc, b_min: int, b_max: int, rank: int = 0, world_size: int = 1, device: int = 0,
                chunk_tokens: int = 0, max_inflight: int = 0, nonblocking_submit: int = 0,
                weights_on_device: int = 0, out_dtype: int = 0, bmax_policy: int = 0) -> surge_config:
    """surge_config from a synth.configs.EncoderConfig-like object."""
    return surge_config(enc.vocab_size, enc.max_position, enc.type_vocab_size, enc.hidden, enc.layers, enc.heads,
                        enc.ffn, enc.ln_eps, b_min, b_max, rank, world_size, device, chunk_tokens, max_inflight,
                        nonblocking_submit, weights_on_device, out_dtype, bmax_policy)


def surge_create(cfg: surge_config, weights, n_weights: int | None = None):
    """weights: numpy uint16 blob (host) or a device pointer/tensor when cfg.weights_on_device."""
    if isinstance(weights, np.ndarray):
        w = np.ascontiguousarray(weights, dtype=np.uint16)
        n = w.size
        ptr = w.ctypes.data
    else:
        ptr = _ptr(weights)
        n = n_weights if n_weights is not None else weights.numel()
    h = C.c_void_p()
    _check(None, lib.surge_create(C.byref(cfg), ptr, n, C.byref(h)), "surge_create")
    return h


def surge_nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0), to be handed to every rank of surge_create_replicated."""
    buf = (C.c_uint8 * 128)()
    _check(None, lib.surge_nccl_unique_id(buf), "surge_nccl_unique_id")
    return bytes(buf)


def surge_create_replicated(cfg: surge_config, nccl_id: bytes, weights=None, n_weights: int | None = None):
    """Every rank calls this concurrently: NCCL communicator over cfg.world_size ranks, one broadcast
    of the weight blob from rank 0 (weights: read on rank 0 only; host numpy blob or device tensor
    when cfg.weights_on_device), then the handle as surge_create."""
    idb = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
    ptr = None
    if isinstance(weights, np.ndarray):
        w = np.ascontiguousarray(weights, dtype=np.uint16)
        ptr, n = w.ctypes.data, w.size
    elif weights is not None:
        ptr, n = _ptr(weights), (n_weights if n_weights is not None else weights.numel())
    else:
        n = n_weights
    h = C.c_void_p()
    _check(None, lib.surge_create_replicated(C.byref(cfg), idb, ptr, n, C.byref(h)), "surge_create_replicated")
    return h


def surge_submit_partition(h, partition_id: int, token_ids: np.ndarray, lengths: np.ndarray) -> int:
    """Returns SURGE_OK or SURGE_E_AGAIN (non-blocking backpressure); raises on errors."""
    ids = np.ascontiguousarray(token_ids, dtype=np.int32)
    lens = np.ascontiguousarray(lengths, dtype=np.int32)
    st = lib.surge_submit_partition(h, C.c_uint64(int(partition_id)), ids.ctypes.data, lens.ctypes.data,
                                    lens.size)
    if st == SURGE_E_AGAIN:
        return st
    return _check(h, st, "surge_submit_partition")


def surge_finish(h):
    return _check(h, lib.surge_finish(h), "surge_finish")


_poll_tls = threading.local()


def surge_poll_flushed(h, max_items: int = 4096, timeout_ms: int = 0):
    """Completed pieces (copies of the records; their data stays library-owned until released).  The
    record buffer is cached per thread, so a poll costs no allocation proportional to max_items."""
    buf = getattr(_poll_tls, "buf", None)
    if buf is None or len(buf) < max_items:
        buf = _poll_tls.buf = (surge_flushed * max_items)()
    n = C.c_int64()
    _check(h, lib.surge_poll_flushed(h, buf, max_items, timeout_ms, C.byref(n)), "surge_poll_flushed")
    return [surge_flushed.from_buffer_copy(buf[i]) for i in range(n.value)]


def flushed_array(rec: surge_flushed) -> np.ndarray:
    """Zero-copy numpy view [n_rows, d] of a polled piece (valid until surge_release): float32, or
    uint16 bf16 bit patterns when the handle's out_dtype is SURGE_BF16 (see bf16_to_f32)."""
    ct, nt = (C.c_uint16, np.uint16) if rec.dtype == SURGE_BF16 else (C.c_float, np.float32)
    if rec.n_rows == 0:
        return np.zeros((0, rec.d), nt)
    return np.ctypeslib.as_array(C.cast(rec.data, C.POINTER(ct)), shape=(rec.n_rows, rec.d))


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float32 values (exact widening)."""
    return (np.asarray(a, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def surge_release(h, rec: surge_flushed):
    return _check(h, lib.surge_release(h, C.byref(rec)), "surge_release")


def surge_pending(h) -> int:
    n = C.c_int64()
    _check(h, lib.surge_pending(h, C.byref(n)), "surge_pending")
    return n.value


def surge_reset(h):
    return _check(h, lib.surge_reset(h), "surge_reset")


def surge_get_stats(h) -> dict:
    s = surge_stats()
    _check(h, lib.surge_get_stats(h, C.byref(s)), "surge_get_stats")
    return s.as_dict()


def surge_get_superbatch(h, index: int) -> dict:
    s = surge_superbatch_info()
    _check(h, lib.surge_get_superbatch(h, index, C.byref(s)), "surge_get_superbatch")
    d = {f: getattr(s, f) for f, _ in s._fields_}
    d["reason"] = REASONS[d["reason"]]
    return d


def surge_get_superbatch_members(h, index: int) -> list:
    n = C.c_int64()
    lib.surge_get_superbatch_members(h, index, None, 0, C.byref(n))
    out = np.zeros(n.value, dtype=np.uint64)
    _check(h, lib.surge_get_superbatch_members(h, index, out.ctypes.data, out.size, C.byref(n)),
           "surge_get_superbatch_members")
    return [int(x) for x in out]


def surge_last_error(h) -> str:
    return lib.surge_last_error(h).decode()


def surge_destroy(h):
    lib.surge_destroy(h)


def surge_encode_packed(h, d_ids, d_lengths, h_lengths: np.ndarray, n_texts: int, d_out, stream=None):
    hl = np.ascontiguousarray(h_lengths, dtype=np.int32)
    return _check(h, lib.surge_encode_packed(h, _ptr(d_ids), _ptr(d_lengths), hl.ctypes.data, n_texts,
                                             _ptr(d_out), _stream(stream)), "surge_encode_packed")


def surge_op_pack(d_lengths, n_texts, d_sizes, n_members, d_cu, d_row_off, d_tok_off, stream=None):
    return _check(None, lib.surge_op_pack(_ptr(d_lengths), n_texts, _ptr(d_sizes), n_members, _ptr(d_cu),
                                          _ptr(d_row_off), _ptr(d_tok_off), _stream(stream)), "surge_op_pack")


def surge_op_embed_ln(h, d_ids, d_cu, n_texts, d_x, stream=None):
    return _check(h, lib.surge_op_embed_ln(h, _ptr(d_ids), _ptr(d_cu), n_texts, _ptr(d_x), _stream(stream)),
                  "surge_op_embed_ln")


def surge_op_gemm(a, b, bias, res, gamma, beta, c, M, N, K, epi, ln_eps=1e-12, stream=None):
    return _check(None, lib.surge_op_gemm(_ptr(a), _ptr(b), _ptr(bias), _ptr(res), _ptr(gamma), _ptr(beta),
                                          _ptr(c), M, N, K, epi, ln_eps, _stream(stream)), "surge_op_gemm")


def surge_op_layernorm(v, rows, d, gamma, beta, out, ln_eps=1e-12, stream=None):
    return _check(None, lib.surge_op_layernorm(_ptr(v), rows, d, _ptr(gamma), _ptr(beta), ln_eps, _ptr(out),
                                               _stream(stream)), "surge_op_layernorm")


def surge_op_attention(qkv, cu, n_texts, heads, head_dim, out, stream=None):
    return _check(None, lib.surge_op_attention(_ptr(qkv), _ptr(cu), n_texts, heads, head_dim, _ptr(out),
                                               _stream(stream)), "surge_op_attention")


def surge_op_meanpool_l2(x, cu, n_texts, d, out, stream=None):
    return _check(None, lib.surge_op_meanpool_l2(_ptr(x), _ptr(cu), n_texts, d, _ptr(out), _stream(stream)),
                  "surge_op_meanpool_l2")


def surge_lpt_plan(lengths: np.ndarray, sizes, world: int):
    """-> dict of arrays (first_row, n_rows, member, tokens, rank) in global-row order."""
    lens = np.ascontiguousarray(lengths, dtype=np.int32)
    sz = np.ascontiguousarray(sizes, dtype=np.int64)
    cap = len(sz) + 8 * world + int(lens.size) if world > 1 else max(1, len(sz))
    cap = min(cap, int(lens.size) + len(sz) + 1)
    out = {k: np.zeros(cap, np.int64) for k in ("first_row", "n_rows", "member", "tokens")}
    out["rank"] = np.zeros(cap, np.int32)
    n = C.c_int64()
    _check(None, lib.surge_lpt_plan(lens.ctypes.data, lens.size, sz.ctypes.data, sz.size, world, cap,
                                    out["first_row"].ctypes.data, out["n_rows"].ctypes.data,
                                    out["member"].ctypes.data, out["tokens"].ctypes.data, out["rank"].ctypes.data,
                                    C.byref(n)), "surge_lpt_plan")
    return {k: v[:n.value].copy() for k, v in out.items()}


def surge_aggregate(sizes, b_min: int, b_max: int):
    """-> (list of (first, end, reason)), peak_buffered) -- Alg.1 flush decisions (host-only)."""
    sz = np.ascontiguousarray(sizes, dtype=np.int64)
    cap = max(1, sz.size)
    first = np.zeros(cap + 1, np.int64)
    reason = np.zeros(cap, np.int32)
    n, peak = C.c_int64(), C.c_int64()
    _check(None, lib.surge_aggregate(sz.ctypes.data, sz.size, b_min, b_max, cap, first.ctypes.data,
                                     reason.ctypes.data, C.byref(n), C.byref(peak)), "surge_aggregate")
    return [(int(first[j]), int(first[j + 1]), REASONS[int(reason[j])]) for j in range(n.value)], peak.value


def surge_aggregate_ex(sizes, b_min: int, b_max: int, policy: int = 0):
    """-> (list of SuperBatches [(reason, [(partition index, row0, rows), ...])], peak_buffered) --
    Alg.1 under a B_max policy (host-only)."""
    sz = np.ascontiguousarray(sizes, dtype=np.int64)
    nonzero = int((sz > 0).sum())
    total = int(sz.sum())
    scap = 2 * nonzero + total // max(b_max, 1) + 2     # SuperBatches (PREFLUSH: <= 2 per partition)
    mcap = nonzero + scap                               # members (SPLIT: <= one extra piece per seal)
    mp, mr0, mr = np.zeros(mcap, np.int64), np.zeros(mcap, np.int64), np.zeros(mcap, np.int64)
    first, reason = np.zeros(scap + 1, np.int64), np.zeros(scap, np.int32)
    F, M, peak = C.c_int64(), C.c_int64(), C.c_int64()
    _check(None, lib.surge_aggregate_ex(sz.ctypes.data, sz.size, b_min, b_max, policy, mcap, mp.ctypes.data,
                                        mr0.ctypes.data, mr.ctypes.data, scap, first.ctypes.data,
                                        reason.ctypes.data, C.byref(F), C.byref(M), C.byref(peak)),
           "surge_aggregate_ex")
    out = []
    for j in range(F.value):
        a, b = int(first[j]), int(first[j + 1])
        out.append((REASONS[int(reason[j])], [(int(mp[i]), int(mr0[i]), int(mr[i])) for i in range(a, b)]))
    return out, peak.value


def surge_encode_superbatch(h, d_ids, d_lengths, h_lengths: np.ndarray, h_sizes: np.ndarray, d_out, stream=None):
    hl = np.ascontiguousarray(h_lengths, dtype=np.int32)
    hs = np.ascontiguousarray(h_sizes, dtype=np.int64)
    return _check(h, lib.surge_encode_superbatch(h, _ptr(d_ids), _ptr(d_lengths), hl.ctypes.data, hl.size,
                                                 hs.ctypes.data, hs.size, _ptr(d_out), _stream(stream)),
                  "surge_encode_superbatch")


def surge_set_option(h, option: int, value: int):
    return _check(h, lib.surge_set_option(h, option, int(value)), "surge_set_option")


def surge_profile_enable(h, on: bool = True):
    return _check(h, lib.surge_profile_enable(h, 1 if on else 0), "surge_profile_enable")


def surge_profile_read(h) -> dict:
    buf = (surge_kernel_profile * 16)()
    n = C.c_int32()
    _check(h, lib.surge_profile_read(h, buf, 16, C.byref(n)), "surge_profile_read")
    return {KERNEL_KINDS[buf[i].kind]: {"launches": buf[i].launches, "ms": buf[i].total_ms,
                                        "flops": buf[i].flops, "bytes": buf[i].bytes} for i in range(n.value)}
