"""Seeded synthetic inputs for the five BASELINE.json configs (and small test configs).

Test/bench infrastructure shared by the oracle and the CUDA path; it holds none of
Sinnamon's arithmetic.  Rows come from a counter-based generator (datagen/gen.c):
row r of a stream is a pure function of (seed, stream, r), so any document can be
regenerated on its own.  Recipe and the readings behind it: DESIGN.md "Input recipe"
(BASELINE.json "configs").
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsinngen.so")
_lock = threading.Lock()
_lib = None

# streams of one config's seed (independent streams for docs, queries, table, deletes)
STREAM_DOCS, STREAM_QUERIES, STREAM_TABLE, STREAM_DELETES = 1, 2, 3, 4

NNZ_FIXED, NNZ_UNIFORM, NNZ_POISSON, NNZ_LOGNORMAL = 0, 1, 2, 3
COORD_UNIFORM, COORD_ZIPF = 0, 1
VAL_NORMAL, VAL_LOGNORMAL, VAL_LAPLACE, VAL_UNIFORM = 0, 1, 2, 3


class _Spec(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("nnz_kind", ctypes.c_int32), ("nnz_a", ctypes.c_double), ("nnz_b", ctypes.c_double),
        ("nnz_lo", ctypes.c_int32), ("nnz_hi", ctypes.c_int32), ("coord_kind", ctypes.c_int32),
        ("zipf_s", ctypes.c_double), ("val_kind", ctypes.c_int32), ("val_a", ctypes.c_double), ("val_b", ctypes.c_double),
    ]


@dataclasses.dataclass(frozen=True)
class VecSpec:
    n: int
    nnz_kind: int
    nnz_a: float
    nnz_b: float = 0.0
    nnz_lo: int = 0
    nnz_hi: int = 1 << 30
    coord_kind: int = COORD_UNIFORM
    zipf_s: float = 0.0
    val_kind: int = VAL_NORMAL
    val_a: float = 0.0
    val_b: float = 1.0

    def c(self) -> _Spec:
        return _Spec(self.n, self.nnz_kind, self.nnz_a, self.nnz_b, self.nnz_lo, self.nnz_hi,
                     self.coord_kind, self.zipf_s, self.val_kind, self.val_a, self.val_b)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    N: int                 # documents
    n: int                 # dimensionality
    doc: VecSpec
    query: VecSpec
    m: int                 # sketch cells per side
    h: int                 # random mappings
    upper_only: bool       # Sinnamon+ 
    nq: int                # queries in total
    batch: int             # queries per search batch
    k: int
    kprime: int
    rerank: bool
    seed: int
    insert_batch: int = 100_000


def _lognormal_mu(mean: float, sigma: float) -> float:
    return float(np.log(mean) - sigma * sigma / 2.0)


def _configs() -> dict[str, Config]:
    c: dict[str, Config] = {}
    # config 1 (BASELINE.json configs[0]) — Tiny
    c["tiny"] = Config(
        "tiny", 10_000, 1_000,
        VecSpec(1_000, NNZ_UNIFORM, 20, 60, 20, 60),
        VecSpec(1_000, NNZ_FIXED, 10, 0, 10, 10),
        m=64, h=2, upper_only=False, nq=100, batch=100, k=10, kprime=100, rerank=True, seed=20230125 + 1)
    # config 2 (configs[1]) — 1M docs, uniform coordinates
    c["c2"] = Config(
        "c2", 1_000_000, 30_000,
        VecSpec(30_000, NNZ_POISSON, 120.0, 0, 0),
        VecSpec(30_000, NNZ_POISSON, 40.0, 0, 1),
        m=128, h=2, upper_only=False, nq=1024, batch=1024, k=10, kprime=500, rerank=True, seed=20230125 + 2)
    # config 3 (configs[2]) — 8.8M docs, Zipf(1.1), log-normal values, Sinnamon+ (upper only)
    c["c3"] = Config(
        "c3", 8_800_000, 30_522,
        VecSpec(30_522, NNZ_LOGNORMAL, _lognormal_mu(120.0, 0.5), 0.5, 5, 600, COORD_ZIPF, 1.1, VAL_LOGNORMAL, 0.0, 1.0),
        VecSpec(30_522, NNZ_POISSON, 43.0, 0, 1, 1 << 30, COORD_ZIPF, 1.1, VAL_LOGNORMAL, 0.0, 1.0),
        m=64, h=1, upper_only=True, nq=4096, batch=1024, k=10, kprime=1000, rerank=True, seed=20230125 + 3)
    # config 4 (configs[3]) — streaming, config-2 distribution grown 0 -> 4M
    c["c4"] = dataclasses.replace(c["c2"], name="c4", N=4_000_000, seed=20230125 + 4)
    # config 5 (configs[4]) — 4M docs, n=100K, Zipf(0.8), Laplace values, h=3
    c["c5"] = Config(
        "c5", 4_000_000, 100_000,
        VecSpec(100_000, NNZ_POISSON, 250.0, 0, 0, 1 << 30, COORD_ZIPF, 0.8, VAL_LAPLACE, 0.0, 1.0),
        VecSpec(100_000, NNZ_POISSON, 100.0, 0, 1, 1 << 30, COORD_ZIPF, 0.8, VAL_LAPLACE, 0.0, 1.0),
        m=256, h=3, upper_only=False, nq=1024, batch=1024, k=100, kprime=2000, rerank=True, seed=20230125 + 5)
    # scaled-down variants used by parity tests (same laws, oracle-friendly sizes)
    c["c2s"] = dataclasses.replace(c["c2"], name="c2s", N=60_000, nq=64, batch=64, insert_batch=25_000)
    c["c3s"] = dataclasses.replace(c["c3"], name="c3s", N=40_000, nq=48, batch=48, insert_batch=16_000)
    c["c5s"] = dataclasses.replace(c["c5"], name="c5s", N=20_000, nq=32, batch=32, insert_batch=8_000)
    c["c4s"] = dataclasses.replace(c["c2"], name="c4s", N=30_000, nq=32, batch=32, insert_batch=5_000,
                                   seed=20230125 + 4)
    return c


CONFIGS = _configs()


def build(force: bool = False) -> str:
    """Compile gen.c into datagen/libsinngen.so (in-tree)."""
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", src, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.gen_count.restype = ctypes.c_int64
            lib.gen_count.argtypes = [ctypes.POINTER(_Spec), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_void_p]
            lib.gen_fill.restype = ctypes.c_int
            lib.gen_fill.argtypes = [ctypes.POINTER(_Spec), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
            lib.gen_table.restype = None
            lib.gen_table.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_void_p]
            lib.gen_choose.restype = None
            lib.gen_choose.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                       ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
            _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def rows(spec: VecSpec, seed: int, stream: int, start: int, count: int, nthreads: int | None = None):
    """CSR rows [start, start+count) of (spec, seed, stream): (indptr int64[count+1], indices int32, values float32)."""
    lib = _load()
    cs = spec.c()
    indptr = np.empty(count + 1, dtype=np.int64)
    total = lib.gen_count(ctypes.byref(cs), seed, stream, start, count, _ptr(indptr))
    indices = np.empty(max(total, 1), dtype=np.int32)[:total]
    values = np.empty(max(total, 1), dtype=np.float32)[:total]
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    lib.gen_fill(ctypes.byref(cs), seed, stream, start, count, _ptr(indptr), _ptr(indices), _ptr(values), nthreads)
    return indptr, indices, values


def docs(cfg: Config, start: int, count: int, nthreads: int | None = None):
    return rows(cfg.doc, cfg.seed, STREAM_DOCS, start, count, nthreads)


def queries(cfg: Config, start: int, count: int, nthreads: int | None = None):
    return rows(cfg.query, cfg.seed, STREAM_QUERIES, start, count, nthreads)


def hash_table(cfg: Config) -> np.ndarray:
    return table(cfg.n, cfg.h, cfg.m, cfg.seed)


def table(n: int, h: int, m: int, seed: int) -> np.ndarray:
    """n*h bucket ids, uniform over [0, m): flat row-major [j][o]."""
    out = np.empty(n * h, dtype=np.int32)
    _load().gen_table(n, h, m, seed, STREAM_TABLE, _ptr(out))
    return out


def choose(pool: np.ndarray, count: int, seed: int, row: int, stream: int = STREAM_DELETES) -> np.ndarray:
    """`count` distinct elements of `pool` (uint32), uniformly without replacement, seeded by (seed, stream, row)."""
    pool = np.ascontiguousarray(pool, dtype=np.uint32)
    count = min(count, pool.size)
    out = np.empty(max(count, 1), dtype=np.uint32)[:count]
    _load().gen_choose(_ptr(pool), pool.size, count, seed, stream, row, _ptr(out))
    return out
