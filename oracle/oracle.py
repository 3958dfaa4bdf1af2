"""ctypes wrapper of the CPU oracle (oracle/ezlda_oracle.c).

TEST INFRASTRUCTURE ONLY: may be imported by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs -- never by the product
package paper_2007_08725_b200/.  The oracle is a plain fp64 C implementation of
SURVEY.md 8(c); see ezlda_oracle.h for what each function follows in the paper.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ezlda_oracle.c")
LIB = os.path.join(HERE, "libezlda_oracle.so")
LIB_OMP = os.path.join(HERE, "libezlda_oracle_omp.so")  # the same source with -fopenmp (all-core timing)


def build(force: bool = False, omp: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -ffp-contract=off: no FMA contraction); omp=True builds
    the OpenMP variant (words split over threads; identical results)."""
    lib = LIB_OMP if omp else LIB
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < max(
        os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "ezlda_oracle.h"))
    ):
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-Wall", *(["-fopenmp"] if omp else []), "-o", lib, SRC, "-lm"]
        subprocess.check_call(cmd)
    return lib


class DrawDetail(C.Structure):
    _fields_ = [
        ("K_sel", C.c_uint32 * 4), ("a", C.c_double * 4), ("C", C.c_uint32 * 4), ("L", C.c_uint32),
        ("M", C.c_double), ("S_est", C.c_double), ("Qp", C.c_double), ("thr", C.c_double),
        ("Sp", C.c_double), ("Z", C.c_double), ("x", C.c_double), ("branch", C.c_int),
        ("topic", C.c_uint32),
    ]

    def as_dict(self) -> dict:
        return {
            "K_sel": list(self.K_sel), "a": list(self.a), "C": list(self.C), "L": self.L,
            "M": self.M, "S_est": self.S_est, "Qp": self.Qp, "thr": self.thr, "Sp": self.Sp,
            "Z": self.Z, "x": self.x, "branch": self.branch, "topic": self.topic,
        }


_lib = None
_libs = {}


def lib(omp: bool = False):
    """The oracle library (omp=True: the OpenMP build, loaded side by side)."""
    global _lib
    if omp:
        if "omp" not in _libs:
            build(omp=True)
            _libs["omp"] = _declare(C.CDLL(LIB_OMP))
        return _libs["omp"]
    if _lib is None:
        build()
        _lib = _declare(C.CDLL(LIB))
    return _lib


def _declare(L):
    P = C.POINTER
    L.ezlda_oracle_philox4x32_10.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
    L.ezlda_oracle_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
    L.ezlda_oracle_uniform.restype = C.c_double
    L.ezlda_oracle_init_topic.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32]
    L.ezlda_oracle_init_topic.restype = C.c_uint32
    L.ezlda_oracle_draw_three_branch.argtypes = [P(C.c_int32), P(C.c_double), C.c_uint32, C.c_double,
                                                 C.c_uint32, C.c_double, P(DrawDetail)]
    L.ezlda_oracle_draw_grid.argtypes = [P(C.c_int32), P(C.c_double), C.c_uint32, C.c_double, C.c_uint32,
                                         P(C.c_double), C.c_uint64, P(C.c_uint32), P(C.c_int32)]
    L.ezlda_oracle_what.argtypes = [C.c_void_p, C.c_uint32, P(C.c_int32), P(C.c_int32), P(C.c_double)]
    L.ezlda_oracle_draw_two_branch.argtypes = [P(C.c_int32), P(C.c_double), C.c_uint32, C.c_double,
                                               C.c_double, P(C.c_double), P(C.c_double), P(C.c_double),
                                               P(C.c_double), P(C.c_double)]
    L.ezlda_oracle_draw_two_branch.restype = C.c_uint32
    L.ezlda_oracle_what_row.argtypes = [P(C.c_int32), P(C.c_int32), C.c_uint32, C.c_uint32, C.c_double,
                                        P(C.c_double)]
    L.ezlda_oracle_what_row.restype = None
    L.ezlda_oracle_set_sampler.argtypes = [C.c_void_p, C.c_uint32]
    L.ezlda_oracle_set_sampler.restype = C.c_int
    L.ezlda_oracle_inverted_index.argtypes = [P(C.c_uint32), P(C.c_uint32), C.c_uint64, C.c_uint32,
                                              P(C.c_uint64), P(C.c_uint64)]
    L.ezlda_oracle_create.argtypes = [P(C.c_uint32), P(C.c_uint32), C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_uint32, C.c_double, C.c_double, C.c_uint64, C.c_uint32,
                                      C.c_uint64, P(C.c_void_p)]
    L.ezlda_oracle_destroy.argtypes = [C.c_void_p]
    L.ezlda_oracle_token_index.argtypes = [C.c_void_p, P(C.c_uint64)]
    L.ezlda_oracle_set_topics.argtypes = [C.c_void_p, P(C.c_uint16), C.c_uint32]
    L.ezlda_oracle_topics.argtypes = [C.c_void_p, P(C.c_uint16)]
    L.ezlda_oracle_iterations.argtypes = [C.c_void_p]
    L.ezlda_oracle_iterations.restype = C.c_uint32
    L.ezlda_oracle_iterate.argtypes = [C.c_void_p, C.c_uint32, P(C.c_int32), P(C.c_int32)]
    L.ezlda_oracle_counts.argtypes = [C.c_void_p, P(C.c_int32), P(C.c_int32), P(C.c_int32)]
    L.ezlda_oracle_loglik.argtypes = [C.c_void_p, C.c_int, P(C.c_int32), P(C.c_int32), P(C.c_double),
                                      P(C.c_double)]
    L.ezlda_oracle_last_stats.argtypes = [C.c_void_p, P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]
    return L


def _ptr(a: np.ndarray | None, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def philox4x32_10(ctr, key) -> list[int]:
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().ezlda_oracle_philox4x32_10(c, k, o)
    return list(o)


def uniform(seed: int, iteration: int, t_g: int) -> float:
    return lib().ezlda_oracle_uniform(seed, iteration, t_g)


def init_topic(seed: int, t_g: int, K: int) -> int:
    return lib().ezlda_oracle_init_topic(seed, t_g, K)


def draw_three_branch(Drow, What, alpha: float, g: int, u: float) -> dict:
    D = np.ascontiguousarray(Drow, dtype=np.int32)
    Wh = np.ascontiguousarray(What, dtype=np.float64)
    det = DrawDetail()
    rc = lib().ezlda_oracle_draw_three_branch(_ptr(D, C.c_int32), _ptr(Wh, C.c_double), len(D), alpha, g, u,
                                              C.byref(det))
    if rc:
        raise ValueError(f"ezlda_oracle_draw_three_branch rc={rc}")
    return det.as_dict()


def draw_grid(Drow, What, alpha: float, g: int, u) -> tuple[np.ndarray, np.ndarray]:
    D = np.ascontiguousarray(Drow, dtype=np.int32)
    Wh = np.ascontiguousarray(What, dtype=np.float64)
    uu = np.ascontiguousarray(u, dtype=np.float64)
    topics = np.zeros(len(uu), dtype=np.uint32)
    branch = np.zeros(len(uu), dtype=np.int32)
    rc = lib().ezlda_oracle_draw_grid(_ptr(D, C.c_int32), _ptr(Wh, C.c_double), len(D), alpha, g,
                                      _ptr(uu, C.c_double), len(uu), _ptr(topics, C.c_uint32),
                                      _ptr(branch, C.c_int32))
    if rc:
        raise ValueError(f"ezlda_oracle_draw_grid rc={rc}")
    return topics, branch


def what_row(W_row, n_k, V: int, beta: float) -> np.ndarray:
    """What[v][.] = (W[v][.] + beta) / (n_k + V beta) from a count row (Eq 1-2)."""
    Wr = np.ascontiguousarray(W_row, dtype=np.int32)
    nk = np.ascontiguousarray(n_k, dtype=np.int32)
    row = np.zeros(len(Wr))
    lib().ezlda_oracle_what_row(_ptr(Wr, C.c_int32), _ptr(nk, C.c_int32), len(Wr), V, beta, _ptr(row, C.c_double))
    return row


def draw_two_branch(Drow, What, alpha: float, u: float) -> dict:
    D = np.ascontiguousarray(Drow, dtype=np.int32)
    Wh = np.ascontiguousarray(What, dtype=np.float64)
    K = len(D)
    S, Q, up = C.c_double(), C.c_double(), C.c_double()
    Sp = np.zeros(K)
    Qp = np.zeros(K)
    topic = lib().ezlda_oracle_draw_two_branch(_ptr(D, C.c_int32), _ptr(Wh, C.c_double), K, alpha, u,
                                               C.byref(S), C.byref(Q), C.byref(up), _ptr(Sp, C.c_double),
                                               _ptr(Qp, C.c_double))
    return {"topic": topic, "S": S.value, "Q": Q.value, "uprime": up.value, "S_prefix": Sp, "Q_prefix": Qp}


def inverted_index(word_ids, doc_ids, n_docs: int):
    w = np.ascontiguousarray(word_ids, dtype=np.uint32)
    d = np.ascontiguousarray(doc_ids, dtype=np.uint32)
    ofs = np.zeros(n_docs + 1, dtype=np.uint64)
    pos = np.zeros(len(w), dtype=np.uint64)
    lib().ezlda_oracle_inverted_index(_ptr(w, C.c_uint32), _ptr(d, C.c_uint32), len(w), n_docs,
                                      _ptr(ofs, C.c_uint64), _ptr(pos, C.c_uint64))
    return ofs, pos


class OracleLDA:
    """The plain CPU chain: create / iterate / topics / counts / loglik."""

    def __init__(self, word_ids, doc_ids, n_docs: int, V: int, K: int, alpha: float | None = None,
                 beta: float = 0.01, seed: int = 1, g: int = 2, token_base: int = 0, branches: int = 3,
                 omp: bool = False):
        self._L = lib(omp)  # omp: the OpenMP build (all host cores), identical results
        self.word = np.ascontiguousarray(word_ids, dtype=np.uint32)
        self.doc = np.ascontiguousarray(doc_ids, dtype=np.uint32)
        self.N = len(self.word)
        self.n_docs, self.V, self.K = n_docs, V, K
        self.alpha = 50.0 / K if alpha is None else alpha
        self.beta = beta
        h = C.c_void_p()
        rc = self._L.ezlda_oracle_create(_ptr(self.word, C.c_uint32), _ptr(self.doc, C.c_uint32), self.N, n_docs,
                                       V, K, self.alpha, beta, seed, g, token_base, C.byref(h))
        if rc:
            raise ValueError(f"ezlda_oracle_create rc={rc}")
        self._h = h
        if self._L.ezlda_oracle_set_sampler(h, branches):
            raise ValueError("branches must be 2 or 3")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and getattr(self, "_L", None) is not None:
            self._L.ezlda_oracle_destroy(h)
            self._h = None

    @property
    def iterations(self) -> int:
        return self._L.ezlda_oracle_iterations(self._h)

    def token_index(self) -> np.ndarray:
        out = np.zeros(self.N, dtype=np.uint64)
        self._L.ezlda_oracle_token_index(self._h, _ptr(out, C.c_uint64))
        return out

    def what(self, v: int, W_global=None, nk_global=None) -> np.ndarray:
        Wg = None if W_global is None else np.ascontiguousarray(W_global, dtype=np.int32)
        ng = None if nk_global is None else np.ascontiguousarray(nk_global, dtype=np.int32)
        row = np.zeros(self.K)
        if self._L.ezlda_oracle_what(self._h, v, _ptr(Wg, C.c_int32), _ptr(ng, C.c_int32), _ptr(row, C.c_double)):
            raise ValueError("word out of range")
        return row

    def set_topics(self, topics, iterations_done: int) -> None:
        z = np.ascontiguousarray(topics, dtype=np.uint16)
        if self._L.ezlda_oracle_set_topics(self._h, _ptr(z, C.c_uint16), iterations_done):
            raise ValueError("topic out of range")

    def topics(self) -> np.ndarray:
        z = np.zeros(self.N, dtype=np.uint16)
        self._L.ezlda_oracle_topics(self._h, _ptr(z, C.c_uint16))
        return z

    def iterate(self, n: int = 1, W_global=None, nk_global=None) -> None:
        Wg = None if W_global is None else np.ascontiguousarray(W_global, dtype=np.int32)
        ng = None if nk_global is None else np.ascontiguousarray(nk_global, dtype=np.int32)
        rc = self._L.ezlda_oracle_iterate(self._h, n, _ptr(Wg, C.c_int32), _ptr(ng, C.c_int32))
        if rc:
            raise RuntimeError(f"ezlda_oracle_iterate rc={rc}")

    def counts(self):
        D = np.zeros((self.n_docs, self.K), dtype=np.int32)
        W = np.zeros((self.V, self.K), dtype=np.int32)
        nk = np.zeros(self.K, dtype=np.int32)
        self._L.ezlda_oracle_counts(self._h, _ptr(D, C.c_int32), _ptr(W, C.c_int32), _ptr(nk, C.c_int32))
        return D, W, nk

    def loglik(self, method: int = 1, W_global=None, nk_global=None, return_sum: bool = False):
        Wg = None if W_global is None else np.ascontiguousarray(W_global, dtype=np.int32)
        ng = None if nk_global is None else np.ascontiguousarray(nk_global, dtype=np.int32)
        out, s = C.c_double(), C.c_double()
        rc = self._L.ezlda_oracle_loglik(self._h, method, _ptr(Wg, C.c_int32), _ptr(ng, C.c_int32), C.byref(out),
                                       C.byref(s))
        if rc:
            raise RuntimeError(f"ezlda_oracle_loglik rc={rc}")
        return (out.value, s.value) if return_sum else out.value

    def last_stats(self) -> dict:
        a, b = C.c_uint64(), C.c_uint64()
        hist = (C.c_uint64 * 4)()
        self._L.ezlda_oracle_last_stats(self._h, C.byref(a), C.byref(b), hist)
        return {"skip_S": a.value, "skip_final": b.value, "branch_hist": list(hist)}
