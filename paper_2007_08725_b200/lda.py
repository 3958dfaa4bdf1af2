"""Thin ctypes binding of libezlda.so (include/ezlda.h): argument marshalling only.

Every step of the hot path runs in the CUDA library; this module never computes
any part of the method and has no CPU fallback: if the library or a GPU is
missing, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EZLDA_LIB") or os.path.join(HERE, "libezlda.so")

EZLDA_W_HYBRID, EZLDA_W_ALL_DENSE, EZLDA_W_ALL_SPARSE = 0, 1, 2
EZLDA_DEBUG_NO_TAIL_ROWS, EZLDA_DEBUG_C1_LOOKUP, EZLDA_DEBUG_DPERM_ON, EZLDA_DEBUG_DPERM_OFF = 1, 2, 4, 8
EZLDA_DEBUG_NO_W_DELTA = 16
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_RANGE", 3: "E_NOMEM", 4: "E_CUDA", 5: "E_NCCL", 6: "E_STATE"}

# every symbol include/ezlda.h declares
EXPORTS = ["ezlda_create", "ezlda_iterate", "ezlda_counts", "ezlda_set_topics", "ezlda_loglik", "ezlda_stats",
           "ezlda_stats_sum", "ezlda_last_error", "ezlda_destroy", "ezlda_nccl_id_size", "ezlda_nccl_get_unique_id"]


class Options(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32), ("g", C.c_uint32), ("w_mode", C.c_uint32), ("dense_threshold", C.c_uint32),
        ("split_threshold", C.c_uint32), ("rank", C.c_int32), ("world", C.c_int32),
        ("nccl_unique_id", C.c_void_p), ("token_base", C.c_uint64), ("stream", C.c_void_p),
        ("input_on_device", C.c_uint32), ("no_phase_timing", C.c_uint32), ("doc_block_kb", C.c_uint32),
        ("exact_draws", C.c_uint32), ("sampler", C.c_uint32), ("local_group", C.c_uint64),
        ("debug_flags", C.c_uint32), ("schedule", C.c_uint32),
    ]


class CSR(C.Structure):
    _fields_ = [("row_ptr", C.POINTER(C.c_uint64)), ("col", C.POINTER(C.c_uint16)), ("val", C.POINTER(C.c_int32)),
                ("nnz", C.c_uint64), ("rows", C.c_uint32)]


class IterStats(C.Structure):
    _fields_ = [
        ("iteration", C.c_uint32), ("ms_total", C.c_double), ("ms_wordprep", C.c_double),
        ("ms_docpass", C.c_double), ("ms_sample", C.c_double), ("ms_allreduce", C.c_double),
        ("n_tokens", C.c_uint64), ("skip_S", C.c_uint64), ("skip_final", C.c_uint64), ("sampled", C.c_uint64),
        ("active_runs", C.c_uint64), ("drow_words", C.c_uint64), ("d_nnz", C.c_uint64),
        ("model_bytes", C.c_double), ("model_bytes_sample", C.c_double), ("model_bytes_docpass", C.c_double),
        ("kernel_launches", C.c_uint64), ("exact_redraws", C.c_uint64), ("exchange_bytes", C.c_double),
        ("ms_sampler_kernel", C.c_double),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class EzLDAError(RuntimeError):
    pass


_lib = None


def load() -> C.CDLL:
    """Load the in-tree libezlda.so (built by __graft_entry__.build()); raise if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EzLDAError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.ezlda_create.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_double, C.c_double, C.c_uint64, P(Options), P(C.c_void_p)]
        L.ezlda_iterate.argtypes = [C.c_void_p, C.c_uint32]
        L.ezlda_counts.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, P(CSR), P(CSR)]
        L.ezlda_set_topics.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32]
        L.ezlda_loglik.argtypes = [C.c_void_p, P(C.c_double)]
        L.ezlda_stats.argtypes = [C.c_void_p, P(IterStats)]
        L.ezlda_stats_sum.argtypes = [C.c_void_p, P(IterStats), C.c_int]
        L.ezlda_last_error.argtypes = [C.c_void_p]
        L.ezlda_last_error.restype = C.c_char_p
        L.ezlda_destroy.argtypes = [C.c_void_p]
        L.ezlda_destroy.restype = None
        L.ezlda_nccl_id_size.restype = C.c_size_t
        L.ezlda_nccl_get_unique_id.argtypes = [C.c_void_p]
        for name in ("ezlda_create", "ezlda_iterate", "ezlda_counts", "ezlda_set_topics", "ezlda_loglik",
                     "ezlda_stats", "ezlda_stats_sum", "ezlda_nccl_get_unique_id"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _addr(a) -> int:
    """Host (numpy) or device (torch) buffer address."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())


def nccl_unique_id() -> bytes:
    L = load()
    n = L.ezlda_nccl_id_size()
    buf = C.create_string_buffer(n)
    rc = L.ezlda_nccl_get_unique_id(buf)
    if rc:
        raise EzLDAError(f"ezlda_nccl_get_unique_id: {STATUS.get(rc, rc)}")
    return buf.raw


class EzLDA:
    """One shard of the corpus on the current CUDA device (ezlda_create ... ezlda_destroy).

    word_ids / doc_ids: uint32 numpy arrays (host) or int32/uint32 torch CUDA tensors
    (device; then input_on_device is set automatically)."""

    def __init__(self, word_ids, doc_ids, n_docs: int, V: int, K: int, alpha: float | None = None,
                 beta: float = 0.01, seed: int = 1, g: int = 0, w_mode: int = EZLDA_W_HYBRID,
                 dense_threshold: int = 0, split_threshold: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, token_base: int = 0, stream: int | None = None,
                 phase_timing: bool = True, doc_block_kb: int = 0, exact_draws: bool = False,
                 local_group: int = 0, sampler: int = 3, debug_flags: int = 0, schedule: int = 0):
        L = load()
        self._h = None
        on_dev = bool(getattr(word_ids, "is_cuda", False))
        if isinstance(word_ids, np.ndarray) or isinstance(word_ids, (list, tuple)):
            word_ids = np.ascontiguousarray(word_ids, dtype=np.uint32)
            doc_ids = np.ascontiguousarray(doc_ids, dtype=np.uint32)
        self.N = int(word_ids.shape[0])
        self.n_docs, self.V, self.K = int(n_docs), int(V), int(K)
        self.alpha = (50.0 / K if K else 0.0) if alpha is None else float(alpha)  # K = 0: E_INVALID
        self.beta = float(beta)
        o = Options()
        o.struct_size = C.sizeof(Options)
        o.g, o.w_mode, o.dense_threshold, o.split_threshold = g, w_mode, dense_threshold, split_threshold
        o.rank, o.world = rank, world
        self._nccl_id = C.create_string_buffer(nccl_id, len(nccl_id)) if nccl_id else None
        o.nccl_unique_id = C.cast(self._nccl_id, C.c_void_p) if nccl_id else None
        o.token_base = token_base
        o.stream = stream
        o.input_on_device = 1 if on_dev else 0
        o.no_phase_timing = 0 if phase_timing else 1
        o.doc_block_kb = doc_block_kb
        o.exact_draws = 1 if exact_draws else 0
        o.local_group = local_group
        o.sampler = sampler  # 3: three-branch (default), 2: two-branch ESCA baseline mode
        o.debug_flags = debug_flags  # EZLDA_DEBUG_* test hooks (rarely taken paths; same topics)
        o.schedule = schedule  # 0 per-iteration active items, 1 static list, 2 no balancing (ablation)
        h = C.c_void_p()
        rc = L.ezlda_create(_addr(word_ids), _addr(doc_ids), self.N, self.n_docs, self.V, self.K, self.alpha,
                            self.beta, seed, C.byref(o), C.byref(h))
        if rc:
            msg = L.ezlda_last_error(None)
            raise EzLDAError(f"ezlda_create: {STATUS.get(rc, rc)}: {msg.decode() if msg else ''}")
        self._h = h

    def _check(self, rc: int, what: str):
        if rc:
            msg = load().ezlda_last_error(self._h)
            raise EzLDAError(f"{what}: {STATUS.get(rc, rc)}: {msg.decode() if msg else ''}")

    def close(self):
        if self._h is not None:
            load().ezlda_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def iterate(self, n: int = 1) -> None:
        self._check(load().ezlda_iterate(self._h, n), "ezlda_iterate")

    def topics(self, out=None):
        """Topics in input order: numpy uint16 (host) or a caller-given buffer (host or device)."""
        z = np.empty(self.N, dtype=np.uint16) if out is None else out
        self._check(load().ezlda_counts(self._h, _addr(z), None, None, None), "ezlda_counts")
        return z

    def n_k(self) -> np.ndarray:
        nk = np.empty(self.K, dtype=np.int32)
        self._check(load().ezlda_counts(self._h, None, nk.ctypes.data, None, None), "ezlda_counts")
        return nk

    def _csr(self, which: str):
        q = CSR()
        args = [None, None, None, None]
        args[2 if which == "W" else 3] = C.byref(q)
        self._check(load().ezlda_counts(self._h, *args), "ezlda_counts")
        rows = q.rows
        rp = np.zeros(rows + 1, dtype=np.uint64)
        col = np.zeros(max(q.nnz, 1), dtype=np.uint16)
        val = np.zeros(max(q.nnz, 1), dtype=np.int32)
        q2 = CSR(rp.ctypes.data_as(C.POINTER(C.c_uint64)), col.ctypes.data_as(C.POINTER(C.c_uint16)),
                 val.ctypes.data_as(C.POINTER(C.c_int32)), q.nnz, 0)
        args[2 if which == "W" else 3] = C.byref(q2)
        self._check(load().ezlda_counts(self._h, *args), "ezlda_counts")
        return rp, col[: q2.nnz], val[: q2.nnz]

    def W_csr(self):
        return self._csr("W")

    def D_csr(self):
        return self._csr("D")

    @staticmethod
    def csr_to_dense(rp, col, val, K: int) -> np.ndarray:
        rows = len(rp) - 1
        out = np.zeros((rows, K), dtype=np.int32)
        r = np.repeat(np.arange(rows), np.diff(rp.astype(np.int64)))
        out[r, col.astype(np.int64)] = val
        return out

    def set_topics(self, topics, iterations_done: int) -> None:
        z = np.ascontiguousarray(topics, dtype=np.uint16) if isinstance(topics, np.ndarray) else topics
        self._check(load().ezlda_set_topics(self._h, _addr(z), iterations_done), "ezlda_set_topics")

    def loglik(self) -> float:
        out = C.c_double()
        self._check(load().ezlda_loglik(self._h, C.byref(out)), "ezlda_loglik")
        return out.value

    def stats(self) -> dict:
        st = IterStats()
        self._check(load().ezlda_stats(self._h, C.byref(st)), "ezlda_stats")
        return st.as_dict()

    def stats_sum(self, reset: bool = True) -> dict:
        """Sums over the iterations since the last reset; 'iteration' = how many."""
        st = IterStats()
        self._check(load().ezlda_stats_sum(self._h, C.byref(st), 1 if reset else 0), "ezlda_stats_sum")
        return st.as_dict()


def partition_docs(doc_lengths: np.ndarray, P: int) -> list[int]:
    """Contiguous doc ranges balanced by tokens (doc-partitioned multi-GPU).
    Returns P+1 doc boundaries."""
    cum = np.concatenate([[0], np.cumsum(np.asarray(doc_lengths, dtype=np.int64))])
    bounds = [0]
    for r in range(1, P):
        bounds.append(int(np.searchsorted(cum, cum[-1] * r / P)))
    bounds.append(len(doc_lengths))
    return bounds
