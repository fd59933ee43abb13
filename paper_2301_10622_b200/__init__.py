"""B200-native Sinnamon (arXiv 2301.10622): Python binding of libsinn.so (include/sinn.h).

Argument marshalling only — every step of insert / delete / search runs in the library's
CUDA kernels for sm_100a.  There is no CPU fallback: if libsinn.so is missing or cannot be
loaded the import of the binding fails loudly (build it with ``python -m
paper_2301_10622_b200._build`` or ``__graft_entry__.build()``).

Device entry points take torch CUDA tensors (the caller's stream is torch's current stream);
``*_host`` entry points take numpy arrays and copy inside the C call.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._build import SO as _SO_PATH

OK, EINVAL, ENOMEM, EEXIST, ENOTFOUND, ECUDA, EPOISONED, EAGAIN = 0, 1, 2, 3, 4, 5, 6, 7
UPPER_ONLY = 1
SKETCH_BF16 = 2  # bfloat16 sketch cells, U rounded up, L rounded down (F3, R21)
BITMAP_CONTAINERS = 4  # Roaring-style (term, 32-bit document mask) containers for dense tile lists (F3)
SEARCH_NOSYNC = 1
NO_ID = 0xFFFFFFFF
MAX_KPRIME = 16384

_STATUS = {0: "SINN_OK", 1: "SINN_EINVAL", 2: "SINN_ENOMEM", 3: "SINN_EEXIST", 4: "SINN_ENOTFOUND", 5: "SINN_ECUDA",
           6: "SINN_EPOISONED", 7: "SINN_EAGAIN"}

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U32 = ctypes.c_uint32
_ST = ctypes.c_int32

# name -> (restype, argtypes): mirrors include/sinn.h one to one
SIGNATURES = {
    "sinn_version": (ctypes.c_char_p, []),
    "sinn_create": (_ST, [_I32, _I32, _I32, _P, _U32, _P, ctypes.POINTER(_P)]),
    "sinn_destroy": (_ST, [_P]),
    "sinn_insert": (_ST, [_P, _I64, _P, _P, _P, _P, _P]),
    "sinn_insert_host": (_ST, [_P, _I64, _P, _P, _P, _P, _P]),
    "sinn_reserve": (_ST, [_P, _I64, _I64, _P]),
    "sinn_delete": (_ST, [_P, _I64, _P, _P]),
    "sinn_delete_host": (_ST, [_P, _I64, _P, _P]),
    "sinn_search": (_ST, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _P, _P, _U32, _P]),
    "sinn_search_host": (_ST, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _P, _P, _P]),
    "sinn_search_stage1": (_ST, [_P, _I64, _P, _P, _P, _I32, _P, _P, _P]),
    "sinn_search_exact": (_ST, [_P, _I64, _P, _P, _P, _I32, _P, _P, _P]),
    "sinn_search_masked": (_ST, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _P, _I64, _I32, _P, _P, _P, _U32, _P]),
    "sinn_search_anytime": (_ST, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _U32, _P]),
    "sinn_search_filtered": (_ST, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _P, _I64, _P, _P, _U32, _P]),
    "sinn_search_stage1_gather": (_ST, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _P, _P, _P]),
    "sinn_rerank": (_ST, [_P, _I64, _P, _P, _P, _I32, _P, _U32, _U32, _I32, _P, _P, _P]),
    "sinn_merge_topk": (_ST, [_I64, _I32, _I32, _P, _P, _U32, _P, _I32, _P, _P, _P]),
    "sinn_sync": (_ST, [_P, _P]),
    "sinn_last_error": (ctypes.c_char_p, [_P]),
    "sinn_export_sketch": (_ST, [_P, _I64, _P, _P, _P, _P]),
    "sinn_export_postings": (_ST, [_P, _I32, _P, _I64, ctypes.POINTER(_I64), _P]),
    "sinn_decode": (_ST, [_P, _I64, _P, _P, _P, _P, _P]),
    "sinn_stats": (_ST, [_P, _P]),
    "sinn_profile": (_ST, [_P, _I32]),
    "sinn_profile_read": (_ST, [_P, _P, _P]),
}

NUM_PHASES = 12
PHASES = ("init", "score", "select", "rerank", "final", "validate", "sketch", "postings", "raw", "delete", "prep")


class Profile(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * NUM_PHASES), ("calls", ctypes.c_int64 * NUM_PHASES),
                ("launches", ctypes.c_int64 * NUM_PHASES)]


class Stats(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in
                ("live", "capacity", "postings", "raw_entries", "bytes_postings", "bytes_sketch", "bytes_raw",
                 "bytes_workspace", "containers", "container_postings", "sample_stride", "sample_rows_kept")]


class SinnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libsinn.so (in-tree).  Raises if it is missing: there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO_PATH):
            raise ImportError(f"{_SO_PATH} is missing: build it first (python -m paper_2301_10622_b200._build)")
        L = ctypes.CDLL(_SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def version() -> str:
    return lib().sinn_version().decode()


def _np(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _stream(stream):
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def _dptr(t, dtype):
    """Device pointer of a contiguous torch CUDA tensor of the given dtype."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("device entry points take torch CUDA tensors (use the *_host methods for numpy)")
    if t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"expected a contiguous {dtype} tensor, got {t.dtype}")
    return t.data_ptr()


class Index:
    """A Sinnamon index on the current CUDA device (owns its device memory)."""

    def __init__(self, n: int, m: int, h: int, hash_table, upper_only: bool = False, stream=None,
                 bf16: bool = False, containers: bool = False):
        self._lib = lib()
        self.n, self.m, self.h, self.upper_only, self.bf16 = n, m, h, upper_only, bf16
        self.containers = containers
        table = _np(hash_table, np.int32)
        if table.size != n * h:
            raise ValueError("hash_table must hold n*h entries")
        h_out = _P()
        flags = (UPPER_ONLY if upper_only else 0) | (SKETCH_BF16 if bf16 else 0) | \
            (BITMAP_CONTAINERS if containers else 0)
        st = self._lib.sinn_create(n, m, h, table.ctypes.data, flags, _stream(stream),
                                   ctypes.byref(h_out))
        if st:
            raise SinnError(st, "sinn_create failed")
        self._h = h_out.value

    def close(self):
        if getattr(self, "_h", None):
            self._lib.sinn_destroy(self._h)
            self._h = None

    __del__ = close

    def _check(self, st: int):
        if st:
            raise SinnError(st, self._lib.sinn_last_error(self._h).decode())

    def status_of(self, fn, *args) -> int:
        """Raw status of a call (for tests of the error protocol)."""
        return fn(self._h, *args)

    # ---------------------------------------------------------------- device (torch) entry points
    def insert(self, indptr, indices, values, ids, stream=None) -> None:
        import torch
        self._check(self._lib.sinn_insert(self._h, ids.numel(), _dptr(indptr, torch.int64), _dptr(indices, torch.int32),
                                          _dptr(values, torch.float32), _dptr(ids, torch.int32), _stream(stream)))

    def reserve(self, max_docs: int, postings: int, stream=None) -> None:
        """Reserve capacity for ids < max_docs and `postings` stored entries (bulk loads)."""
        self._check(self._lib.sinn_reserve(self._h, int(max_docs), int(postings), _stream(stream)))

    def delete(self, ids, stream=None) -> None:
        import torch
        self._check(self._lib.sinn_delete(self._h, ids.numel(), _dptr(ids, torch.int32), _stream(stream)))

    def search(self, q_indptr, q_indices, q_values, k: int, kprime: int, rerank: bool = True, out=None,
               sync: bool = True, stream=None):
        """Returns (ids int32 [nq, k] with -1 = SINN_NO_ID padding, scores float32 [nq, k])."""
        import torch
        nq = q_indptr.numel() - 1
        if out is None:
            out = (torch.empty((nq, k), dtype=torch.int32, device=q_indptr.device),
                   torch.empty((nq, k), dtype=torch.float32, device=q_indptr.device))
        oi, os_ = out
        self._check(self._lib.sinn_search(self._h, nq, _dptr(q_indptr, torch.int64), _dptr(q_indices, torch.int32),
                                          _dptr(q_values, torch.float32), k, kprime, int(rerank),
                                          _dptr(oi, torch.int32), _dptr(os_, torch.float32),
                                          0 if sync else SEARCH_NOSYNC, _stream(stream)))
        return oi, os_

    def search_anytime(self, q_indptr, q_indices, q_values, k: int, kprime: int, max_terms: int, rerank: bool = True,
                       stream=None):
        """sinn_search with the anytime budget: stage 1 scores each query's max_terms largest-|q_j| terms."""
        import torch
        nq = q_indptr.numel() - 1
        oi = torch.empty((nq, k), dtype=torch.int32, device=q_indptr.device)
        os_ = torch.empty((nq, k), dtype=torch.float32, device=q_indptr.device)
        self._check(self._lib.sinn_search_anytime(self._h, nq, _dptr(q_indptr, torch.int64),
                                                  _dptr(q_indices, torch.int32), _dptr(q_values, torch.float32), k,
                                                  kprime, int(rerank), int(max_terms), _dptr(oi, torch.int32),
                                                  _dptr(os_, torch.float32), 0, _stream(stream)))
        return oi, os_

    def search_filtered(self, q_indptr, q_indices, q_values, k: int, kprime: int, allow, rerank: bool = True,
                        stream=None):
        """Constrained search (Eq. 3): `allow` is a torch int32 CUDA tensor holding the uint32 column
        bitmap (bit i of word i/32 set = document i may be returned)."""
        import torch
        nq = q_indptr.numel() - 1
        oi = torch.empty((nq, k), dtype=torch.int32, device=q_indptr.device)
        os_ = torch.empty((nq, k), dtype=torch.float32, device=q_indptr.device)
        self._check(self._lib.sinn_search_filtered(self._h, nq, _dptr(q_indptr, torch.int64),
                                                   _dptr(q_indices, torch.int32), _dptr(q_values, torch.float32), k,
                                                   kprime, int(rerank), _dptr(allow, torch.int32) if allow.numel()
                                                   else None, allow.numel(), _dptr(oi, torch.int32),
                                                   _dptr(os_, torch.float32), 0, _stream(stream)))
        return oi, os_

    def search_masked(self, q_indptr, q_indices, q_values, k: int, kprime: int, masks, qmask, rerank: bool = True,
                      stream=None):
        """Constrained search with a constraint set per query (Eq. 3, F4): `masks` is a torch int32 CUDA
        tensor [nmasks, words] of uint32 column bitmaps, `qmask` int32 [nq] (mask row of each query, -1 =
        none)."""
        import torch
        nq = q_indptr.numel() - 1
        nmasks, words = (int(masks.shape[0]), int(masks.shape[1])) if masks.numel() else (0, 0)
        oi = torch.empty((nq, k), dtype=torch.int32, device=q_indptr.device)
        os_ = torch.empty((nq, k), dtype=torch.float32, device=q_indptr.device)
        self._check(self._lib.sinn_search_masked(self._h, nq, _dptr(q_indptr, torch.int64),
                                                 _dptr(q_indices, torch.int32), _dptr(q_values, torch.float32), k,
                                                 kprime, int(rerank), _dptr(masks, torch.int32) if masks.numel()
                                                 else None, words, nmasks, _dptr(qmask, torch.int32),
                                                 _dptr(oi, torch.int32), _dptr(os_, torch.float32), 0, _stream(stream)))
        return oi, os_

    def search_exact(self, q_indptr, q_indices, q_values, k: int, stream=None):
        """Exact top-k MIPS (LinScan, Alg. 2) on the GPU: (ids int32 [nq, k], scores float32 [nq, k])."""
        import torch
        nq = q_indptr.numel() - 1
        oi = torch.empty((nq, k), dtype=torch.int32, device=q_indptr.device)
        os_ = torch.empty((nq, k), dtype=torch.float32, device=q_indptr.device)
        self._check(self._lib.sinn_search_exact(self._h, nq, _dptr(q_indptr, torch.int64),
                                                _dptr(q_indices, torch.int32), _dptr(q_values, torch.float32), k,
                                                _dptr(oi, torch.int32), _dptr(os_, torch.float32), _stream(stream)))
        return oi, os_

    def sync(self, stream=None) -> None:
        self._check(self._lib.sinn_sync(self._h, _stream(stream)))

    def search_stage1(self, q_indptr, q_indices, q_values, kprime: int, stream=None):
        import torch
        nq = q_indptr.numel() - 1
        ci = torch.empty((nq, kprime), dtype=torch.int32, device=q_indptr.device)
        cs = torch.empty((nq, kprime), dtype=torch.float32, device=q_indptr.device)
        self._check(self._lib.sinn_search_stage1(self._h, nq, _dptr(q_indptr, torch.int64),
                                                 _dptr(q_indices, torch.int32), _dptr(q_values, torch.float32),
                                                 kprime, _dptr(ci, torch.int32), _dptr(cs, torch.float32),
                                                 _stream(stream)))
        return ci, cs

    def search_stage1_gather(self, q_indptr, q_indices, q_values, kprime: int, slot: int, dst_ids, dst_scores,
                             stream=None) -> None:
        """Stage 1 whose rows are stored into slot `slot` of every buffer of `dst_ids` / `dst_scores` (lists of
        W int32 / float32 CUDA tensors [W, nq, kprime]: each shard's gather buffer, peer-mapped or local)."""
        import torch
        nq, W = q_indptr.numel() - 1, len(dst_ids)
        for t in list(dst_ids) + list(dst_scores):
            if tuple(t.shape) != (W, nq, kprime):
                raise ValueError("gather buffers must be [W, nq, kprime]")
        pi = (_P * W)(*[_dptr(t, torch.int32) for t in dst_ids])
        ps = (_P * W)(*[_dptr(t, torch.float32) for t in dst_scores])
        self._check(self._lib.sinn_search_stage1_gather(self._h, nq, _dptr(q_indptr, torch.int64),
                                                        _dptr(q_indices, torch.int32), _dptr(q_values, torch.float32),
                                                        kprime, W, int(slot), pi, ps, _stream(stream)))

    def rerank(self, q_indptr, q_indices, q_values, cand_ids, k: int, id_mul: int = 1, id_add: int = 0, stream=None):
        """Exact re-rank of caller-supplied GLOBAL candidates (sinn_rerank): `cand_ids` int32 [nq, kc]; only
        the candidates this shard owns (g % id_mul == id_add, local id live) are scored.  Returns (global ids
        int32 [nq, k], exact scores float32 [nq, k])."""
        import torch
        nq, kc = int(cand_ids.shape[0]), int(cand_ids.shape[1])
        oi = torch.empty((nq, k), dtype=torch.int32, device=cand_ids.device)
        os_ = torch.empty((nq, k), dtype=torch.float32, device=cand_ids.device)
        self._check(self._lib.sinn_rerank(self._h, nq, _dptr(q_indptr, torch.int64), _dptr(q_indices, torch.int32),
                                          _dptr(q_values, torch.float32), kc, _dptr(cand_ids, torch.int32),
                                          int(id_mul), int(id_add), k, _dptr(oi, torch.int32),
                                          _dptr(os_, torch.float32), _stream(stream)))
        return oi, os_

    def export_sketch(self, ids, stream=None):
        import torch
        cnt = ids.numel()
        U = torch.empty((cnt, self.m), dtype=torch.float32, device=ids.device)
        L = None if self.upper_only else torch.empty((cnt, self.m), dtype=torch.float32, device=ids.device)
        self._check(self._lib.sinn_export_sketch(self._h, cnt, _dptr(ids, torch.int32), U.data_ptr(),
                                                 None if L is None else L.data_ptr(), _stream(stream)))
        return U, L

    def export_postings(self, term: int, stream=None):
        import torch
        ln = _I64(0)
        self._check(self._lib.sinn_export_postings(self._h, term, None, 0, ctypes.byref(ln), _stream(stream)))
        out = torch.empty(max(ln.value, 1), dtype=torch.int32, device="cuda")
        self._check(self._lib.sinn_export_postings(self._h, term, out.data_ptr(), ln.value, ctypes.byref(ln),
                                                   _stream(stream)))
        return out[:ln.value]

    def decode(self, ids, terms, positive, stream=None):
        import torch
        out = torch.empty(ids.numel(), dtype=torch.float32, device=ids.device)
        self._check(self._lib.sinn_decode(self._h, ids.numel(), _dptr(ids, torch.int32), _dptr(terms, torch.int32),
                                          _dptr(positive, torch.uint8), out.data_ptr(), _stream(stream)))
        return out

    # ---------------------------------------------------------------- host (numpy) entry points
    def insert_host(self, indptr, indices, values, ids, stream=None) -> None:
        indptr, indices, values, ids = (_np(indptr, np.int64), _np(indices, np.int32), _np(values, np.float32),
                                        _np(ids, np.uint32))
        self._check(self._lib.sinn_insert_host(self._h, ids.size, indptr.ctypes.data, indices.ctypes.data,
                                               values.ctypes.data, ids.ctypes.data, _stream(stream)))

    def delete_host(self, ids, stream=None) -> None:
        ids = _np(ids, np.uint32)
        self._check(self._lib.sinn_delete_host(self._h, ids.size, ids.ctypes.data, _stream(stream)))

    def search_host(self, q_indptr, q_indices, q_values, k: int, kprime: int, rerank: bool = True, out=None,
                    stream=None):
        """Host arrays in and out (copies inside the C call).  Returns (ids uint32 [nq,k], scores float32 [nq,k])."""
        q_indptr, q_indices, q_values = _np(q_indptr, np.int64), _np(q_indices, np.int32), _np(q_values, np.float32)
        nq = q_indptr.size - 1
        if out is None:
            out = (np.empty((nq, k), np.uint32), np.empty((nq, k), np.float32))
        oi, os_ = out
        self._check(self._lib.sinn_search_host(self._h, nq, q_indptr.ctypes.data, q_indices.ctypes.data,
                                               q_values.ctypes.data, k, kprime, int(rerank), oi.ctypes.data,
                                               os_.ctypes.data, _stream(stream)))
        return oi, os_

    def profile(self, enable: bool) -> None:
        """Start (clears totals) / stop recording CUDA events around each kernel phase."""
        self._check(self._lib.sinn_profile(self._h, int(enable)))

    def profile_read(self, stream=None) -> dict:
        """{phase: (ms, calls, kernel launches)} summed since profile(True)."""
        p = Profile()
        self._check(self._lib.sinn_profile_read(self._h, ctypes.byref(p), _stream(stream)))
        return {name: (p.ms[i], p.calls[i], p.launches[i]) for i, name in enumerate(PHASES)}

    def stats(self) -> dict:
        s = Stats()
        self._check(self._lib.sinn_stats(self._h, ctypes.byref(s)))
        return {name: getattr(s, name) for name, _ in Stats._fields_}


def merge_topk(ids, scores, kout: int, id_mul: int = 1, id_add=None, stream=None):
    """sinn_merge_topk: `ids` int32 / `scores` float32 CUDA tensors [parts, nq, kin] (an all-gather of per-shard
    lists) -> the top-kout per query by (score desc, id asc) over the union; an id of part p becomes
    id * id_mul + id_add[p].  Returns (ids int32 [nq, kout], scores float32 [nq, kout])."""
    import torch
    parts, nq, kin = (int(x) for x in ids.shape)
    add = None if id_add is None else _np(id_add, np.uint32)
    if add is not None and add.size != parts:
        raise ValueError("id_add must hold one entry per part")
    oi = torch.empty((nq, kout), dtype=torch.int32, device=ids.device)
    os_ = torch.empty((nq, kout), dtype=torch.float32, device=ids.device)
    st = lib().sinn_merge_topk(nq, parts, kin, _dptr(ids, torch.int32), _dptr(scores, torch.float32), int(id_mul),
                               None if add is None else add.ctypes.data, kout, _dptr(oi, torch.int32),
                               _dptr(os_, torch.float32), _stream(stream))
    if st:
        raise SinnError(st, "sinn_merge_topk failed")
    return oi, os_


def build(force: bool = False) -> str:
    from ._build import build as _b
    return _b(force=force)
