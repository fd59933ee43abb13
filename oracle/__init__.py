"""Plain CPU oracle of Sinnamon (arXiv 2301.10622) — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` / ``--impl reference``
legs may import this package.  It shares no code with the CUDA path
(``paper_2301_10622_b200``) and never imports it.

``sinn_oracle.c`` follows Alg. 5, Alg. 6, Alg. 7,
Alg. 3 and the deletion protocol step by step, accumulating in
fp64; ``analysis.py`` holds the paper's closed forms (Eq. at).
Pins: tests/test_oracle_pins.py (O1-O12).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, EINVAL, ENOMEM, EEXIST, ENOTFOUND = 0, 1, 2, 3, 4
UPPER_ONLY = 1
SKETCH_BF16 = 2  # F3 (R21): bfloat16 sketch cells, U rounded up, L rounded down
NO_ID = 0xFFFFFFFF

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U32 = ctypes.c_uint32


def build(force: bool = False) -> str:
    """Compile sinn_oracle.c into oracle/liboracle.so (in-tree; plain gcc, no CUDA)."""
    src = os.path.join(_HERE, "sinn_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-shared", "-fPIC",
                               "-pthread", src, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            sig = {
                "orc_create": (_P, [_I32, _I32, _I32, _P, _U32]),
                "orc_destroy": (None, [_P]),
                "orc_insert": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P]),
                "orc_delete": (ctypes.c_int, [_P, _I64, _P]),
                "orc_decode": (ctypes.c_float, [_P, _U32, _I32, ctypes.c_int]),
                "orc_find_largest": (_I64, [_P, _P, _I64, _I64, _P, _P]),
                "orc_score": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P]),
                "orc_score_budget": (ctypes.c_int, [_P, _I64, _P, _P, _I32, _P, _P]),
                "orc_exact_dot": (ctypes.c_double, [_P, _U32, _I64, _P, _P]),
                "orc_cap": (_I64, [_P]),
                "orc_live_count": (_I64, [_P]),
                "orc_search": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P,
                                              ctypes.c_int]),
                "orc_search_budget": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P,
                                                     _P, ctypes.c_int]),
                "orc_search_filtered": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _I64, _P,
                                                       _P, ctypes.c_int]),
                "orc_exact": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I32, _P, _P, ctypes.c_int]),
                "orc_export_sketch": (ctypes.c_int, [_P, _I64, _P, _P, _P]),
                "orc_postings_len": (_I64, [_P, _I32]),
                "orc_export_postings": (ctypes.c_int, [_P, _I32, _P]),
                "orc_is_live": (ctypes.c_int, [_P, _U32]),
                "orc_raw_nnz": (_I32, [_P, _U32]),
                "orc_raw_row": (ctypes.c_int, [_P, _U32, _P, _P]),
                "orc_sketch_row": (None, [_I32, _I32, _P, _I64, _P, _P, _P, _P]),
                "orc_bf16_up": (ctypes.c_float, [ctypes.c_float]),
                "orc_bf16_down": (ctypes.c_float, [ctypes.c_float]),
            }
            for name, (res, args) in sig.items():
                f = getattr(lib, name)
                f.restype = res
                f.argtypes = args
            _lib = lib
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def default_threads() -> int:
    return os.cpu_count() or 1


class OracleIndex:
    """Sinnamon index on the CPU: I (ordered sets), U/L sketches (fp32), raw store S, live set."""

    def __init__(self, n: int, m: int, h: int, table, upper_only: bool = False, bf16: bool = False):
        self._lib = _load()
        self.n, self.m, self.h, self.upper_only, self.bf16 = n, m, h, upper_only, bf16
        self._table = _c(table, np.int32)
        if self._table.size != n * h:
            raise ValueError("table must hold n*h entries")
        flags = (UPPER_ONLY if upper_only else 0) | (SKETCH_BF16 if bf16 else 0)
        self._h = self._lib.orc_create(n, m, h, _p(self._table), flags)
        if not self._h:
            raise ValueError("invalid (n, m, h, table)")

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.orc_destroy(self._h)
            self._h = None

    # -- mutation --------------------------------------------------------------------------------
    def insert(self, indptr, indices, values, ids) -> int:
        indptr, indices = _c(indptr, np.int64), _c(indices, np.int32)
        values, ids = _c(values, np.float32), _c(ids, np.uint32)
        return self._lib.orc_insert(self._h, ids.size, _p(indptr), _p(indices), _p(values), _p(ids))

    def delete(self, ids) -> int:
        ids = _c(ids, np.uint32)
        return self._lib.orc_delete(self._h, ids.size, _p(ids))

    # -- queries ---------------------------------------------------------------------------------
    def search(self, qptr, qidx, qval, k: int, kprime: int, rerank: bool = True, nthreads: int | None = None,
               with_candidates: bool = False, max_terms: int = 0):
        """Alg. 6 + 7 per query; max_terms > 0 = the anytime budget as a term count (R20)."""
        qptr, qidx, qval = _c(qptr, np.int64), _c(qidx, np.int32), _c(qval, np.float32)
        nq = qptr.size - 1
        ids = np.empty(nq * k, np.uint32)
        sc = np.empty(nq * k, np.float64)
        cid = csc = cms = None
        if with_candidates:
            cid = np.empty(nq * kprime, np.uint32)
            csc = np.empty(nq * kprime, np.float64)
            cms = np.empty(nq * kprime, np.float64)
        st = self._lib.orc_search_budget(self._h, nq, _p(qptr), _p(qidx), _p(qval), k, kprime, int(rerank),
                                         int(max_terms), _p(ids), _p(sc), _p(cid), _p(csc), _p(cms),
                                         nthreads or default_threads())
        if st:
            raise ValueError(f"orc_search status {st}")
        out = (ids.reshape(nq, k), sc.reshape(nq, k))
        if with_candidates:
            out = out + (cid.reshape(nq, kprime), csc.reshape(nq, kprime), cms.reshape(nq, kprime))
        return out

    def search_filtered(self, qptr, qidx, qval, k: int, kprime: int, allow_words, rerank: bool = True,
                        max_terms: int = 0, nthreads: int | None = None):
        """Constrained search (Eq. 3): only documents whose bit is set in allow_words (uint32 bitmap)."""
        qptr, qidx, qval = _c(qptr, np.int64), _c(qidx, np.int32), _c(qval, np.float32)
        allow = _c(allow_words, np.uint32)
        nq = qptr.size - 1
        ids = np.empty(nq * k, np.uint32)
        sc = np.empty(nq * k, np.float64)
        st = self._lib.orc_search_filtered(self._h, nq, _p(qptr), _p(qidx), _p(qval), k, kprime, int(rerank),
                                           int(max_terms), _p(allow), allow.size, _p(ids), _p(sc),
                                           nthreads or default_threads())
        if st:
            raise ValueError(f"orc_search_filtered status {st}")
        return ids.reshape(nq, k), sc.reshape(nq, k)

    def exact(self, qptr, qidx, qval, k: int, nthreads: int | None = None):
        qptr, qidx, qval = _c(qptr, np.int64), _c(qidx, np.int32), _c(qval, np.float32)
        nq = qptr.size - 1
        ids = np.empty(nq * k, np.uint32)
        sc = np.empty(nq * k, np.float64)
        st = self._lib.orc_exact(self._h, nq, _p(qptr), _p(qidx), _p(qval), k, _p(ids), _p(sc),
                                 nthreads or default_threads())
        if st:
            raise ValueError(f"orc_exact status {st}")
        return ids.reshape(nq, k), sc.reshape(nq, k)

    def scores(self, qidx, qval, max_terms: int = 0):
        """Alg. 6 scores of one query for every column (vacant = -inf) and the term mass sum|q_j e_ij|;
        max_terms > 0: only the first max_terms terms by descending |q_j| (anytime budget, R20)."""
        qidx, qval = _c(qidx, np.int32), _c(qval, np.float32)
        cap = self.cap
        s = np.empty(max(cap, 1), np.float64)[:cap]
        ms = np.empty(max(cap, 1), np.float64)[:cap]
        self._lib.orc_score_budget(self._h, qidx.size, _p(qidx), _p(qval), int(max_terms), _p(s), _p(ms))
        return s, ms

    def decode(self, i: int, j: int, positive: bool) -> float:
        return float(self._lib.orc_decode(self._h, i, j, int(positive)))

    def exact_dot(self, i: int, qidx, qval) -> float:
        qidx, qval = _c(qidx, np.int32), _c(qval, np.float32)
        return float(self._lib.orc_exact_dot(self._h, i, qidx.size, _p(qidx), _p(qval)))

    # -- inspection ------------------------------------------------------------------------------
    @property
    def cap(self) -> int:
        return int(self._lib.orc_cap(self._h))

    @property
    def live_count(self) -> int:
        return int(self._lib.orc_live_count(self._h))

    def is_live(self, i: int) -> bool:
        return bool(self._lib.orc_is_live(self._h, i))

    def sketch(self, ids):
        ids = _c(ids, np.uint32)
        U = np.empty((ids.size, self.m), np.float32)
        L = None if self.upper_only else np.empty((ids.size, self.m), np.float32)
        st = self._lib.orc_export_sketch(self._h, ids.size, _p(ids), _p(U), _p(L))
        if st:
            raise ValueError(f"orc_export_sketch status {st}")
        return U, L

    def postings(self, j: int) -> np.ndarray:
        n = int(self._lib.orc_postings_len(self._h, j))
        out = np.empty(max(n, 1), np.uint32)[:n]
        self._lib.orc_export_postings(self._h, j, _p(out))
        return out

    def raw_row(self, i: int):
        nnz = int(self._lib.orc_raw_nnz(self._h, i))
        idx = np.empty(max(nnz, 1), np.int32)[:nnz]
        val = np.empty(max(nnz, 1), np.float32)[:nnz]
        self._lib.orc_raw_row(self._h, i, _p(idx), _p(val))
        return idx, val


def find_largest(scores, ids, k: int):
    """Alg. 3 FindLargest over (score, id) pairs scanned in the given order: best first."""
    scores, ids = _c(scores, np.float64), _c(ids, np.uint32)
    oi = np.empty(max(k, 1), np.uint32)
    os_ = np.empty(max(k, 1), np.float64)
    r = _load().orc_find_largest(_p(scores), _p(ids), scores.size, k, _p(oi), _p(os_))
    return oi[:r], os_[:r]


def sketch_row(m: int, h: int, table, idx, val, lower: bool = True):
    """Alg. 5 lines 3-7 for a single vector: (u, l) with -inf/+inf in untouched cells."""
    table, idx, val = _c(table, np.int32), _c(idx, np.int32), _c(val, np.float32)
    u = np.empty(m, np.float32)
    l = np.empty(m, np.float32) if lower else None
    _load().orc_sketch_row(m, h, _p(table), idx.size, _p(idx), _p(val), _p(u), _p(l))
    return u, l


def bf16_up(x: float) -> float:
    """Smallest bfloat16 >= x (R21), as a float32 value."""
    return float(_load().orc_bf16_up(float(x)))


def bf16_down(x: float) -> float:
    """Largest bfloat16 <= x (R21), as a float32 value."""
    return float(_load().orc_bf16_down(float(x)))
