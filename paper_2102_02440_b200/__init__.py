"""B200-native COMPASS hot path (arXiv 2102.02440): thin ctypes binding of
``libcompass_b200.so`` (C-ABI in ``include/compass_b200.h``).

This module only marshals arguments: every step of the hot path (filter, hash,
sketch update, flush, merge, composition estimates) runs in the library's CUDA
kernels; the greedy enumerator runs in the library's host code.  PyTorch is used
for device memory and streams only.  There is no CPU fallback: if the compiled
library is missing, importing works but every call raises ``RuntimeError``.

Names follow the paper / SURVEY.md §8(b): ``sketch_create``, ``sketch_update_filtered``,
``sketch_merge``, ``estimate_join``, ``plan_greedy``.
"""
from __future__ import annotations

import ctypes
import os

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("COMPASS_LIB") or os.path.join(PKG, "libcompass_b200.so")

SK_OK, SK_EINVAL, SK_EMISMATCH, SK_EOVERFLOW, SK_ENOMEM, SK_ECUDA = range(6)
SK_INT32, SK_INT64 = 0, 1
POINT, RANGE, SUBSET = 0, 1, 2
INT64_MIN = -(1 << 63)
INT64_MAX = (1 << 63) - 1

_STATUS = {0: "SK_OK", 1: "SK_EINVAL", 2: "SK_EMISMATCH", 3: "SK_EOVERFLOW", 4: "SK_ENOMEM", 5: "SK_ECUDA"}


class SkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class sk_desc(ctypes.Structure):
    _fields_ = [("d", ctypes.c_uint32), ("ndim", ctypes.c_uint32), ("w", ctypes.c_uint32 * 3),
                ("master_seed", ctypes.c_uint64), ("edge_id", ctypes.c_char_p * 3)]


class sk_column(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_uint32), ("domain", ctypes.c_uint64)]


class sk_pred(ctypes.Structure):
    _fields_ = [("col", ctypes.c_uint32), ("kind", ctypes.c_uint32), ("lo", ctypes.c_int64), ("hi", ctypes.c_int64),
                ("set", ctypes.POINTER(ctypes.c_int64)), ("set_size", ctypes.c_uint64)]


class sk_target(ctypes.Structure):
    _fields_ = [("sketch", ctypes.c_void_p), ("key_col", ctypes.c_uint32 * 3)]


class sk_peer_push(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.POINTER(ctypes.c_void_p)), ("n_peers", ctypes.c_uint32),
                ("n", ctypes.c_uint64), ("owner_mode", ctypes.c_uint32), ("rank", ctypes.c_uint32),
                ("offset", ctypes.c_uint64), ("total", ctypes.c_uint64)]


SK_IPC_HANDLE_BYTES = 64


class sk_graph(ctypes.Structure):
    _fields_ = [("n_tables", ctypes.c_uint32), ("survivors", ctypes.POINTER(ctypes.c_int64)),
                ("n_edges", ctypes.c_uint32), ("edge_u", ctypes.POINTER(ctypes.c_uint32)),
                ("edge_v", ctypes.POINTER(ctypes.c_uint32)), ("vec_u", ctypes.POINTER(ctypes.c_void_p)),
                ("vec_v", ctypes.POINTER(ctypes.c_void_p)), ("n_mats", ctypes.c_uint32),
                ("mat_table", ctypes.POINTER(ctypes.c_uint32)), ("mat_e0", ctypes.POINTER(ctypes.c_uint32)),
                ("mat_e1", ctypes.POINTER(ctypes.c_uint32)), ("mat", ctypes.POINTER(ctypes.c_void_p))]


# every symbol include/compass_b200.h declares (checked by tests/test_abi.py)
EXPORTS = ["sketch_create", "sketch_destroy", "sketch_counters", "sketch_zero", "sketch_update_filtered",
           "sketch_merge", "sketch_wire_pack", "sketch_wire_unpack", "estimate_join", "estimate_join_exact", "estimate_subplans", "plan_greedy",
           "plan_enumerate", "exact_join_size", "sk_last_error", "sk_version", "sk_kernel_launches",
           "sketch_update_filtered_push", "sketch_peer_push", "sketch_peer_gather", "sk_ipc_alloc", "sk_ipc_free", "sk_ipc_open", "sk_ipc_close"]

# Algorithm 1 search-space settings
ENUM_GREEDY, ENUM_FULL_GREEDY, ENUM_LIMIT, ENUM_EXHAUSTIVE = range(4)
ENUM_MODES = {"greedy": ENUM_GREEDY, "full-greedy": ENUM_FULL_GREEDY, "limit": ENUM_LIMIT,
              "exhaustive": ENUM_EXHAUSTIVE}


class sk_enum_config(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("beta", ctypes.c_double), ("mode", ctypes.c_uint32),
                ("max_plans", ctypes.c_uint32), ("no_prune", ctypes.c_uint32)]


class sk_table_data(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_uint64), ("cols", ctypes.POINTER(sk_column)), ("n_cols", ctypes.c_uint32),
                ("preds", ctypes.POINTER(sk_pred)), ("n_preds", ctypes.c_uint32)]


class sk_join_data(ctypes.Structure):
    _fields_ = [("n_tables", ctypes.c_uint32), ("tables", ctypes.POINTER(sk_table_data)),
                ("n_edges", ctypes.c_uint32), ("edge_u", ctypes.POINTER(ctypes.c_uint32)),
                ("edge_v", ctypes.POINTER(ctypes.c_uint32)), ("col_u", ctypes.POINTER(ctypes.c_uint32)),
                ("col_v", ctypes.POINTER(ctypes.c_uint32)), ("key_lo", ctypes.POINTER(ctypes.c_int64)),
                ("key_domain", ctypes.POINTER(ctypes.c_uint64))]


class sk_enum_stats(ctypes.Structure):
    _fields_ = [("plans_completed", ctypes.c_uint64), ("prunes", ctypes.c_uint64),
                ("estimator_calls", ctypes.c_uint64), ("distinct_estimates", ctypes.c_uint64)]

_lib = None


def lib() -> ctypes.CDLL:
    """Load the compiled C-ABI library.  Raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: build it with __graft_entry__.build() "
                               "(the CUDA path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        st, vp, u32, u64, i64 = ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int64
        L.sketch_create.restype = st
        L.sketch_create.argtypes = [ctypes.POINTER(sk_desc), ctypes.c_int, vp, ctypes.POINTER(vp)]
        L.sketch_destroy.restype = st
        L.sketch_destroy.argtypes = [vp]
        L.sketch_counters.restype = st
        L.sketch_counters.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(u64)]
        L.sketch_zero.restype = st
        L.sketch_zero.argtypes = [vp, vp]
        L.sketch_update_filtered.restype = st
        L.sketch_update_filtered.argtypes = [ctypes.POINTER(sk_column), u32, u64, ctypes.POINTER(sk_pred), u32,
                                             ctypes.POINTER(sk_target), u32, vp, vp]
        L.sketch_merge.restype = st
        L.sketch_merge.argtypes = [vp, vp, vp]
        L.estimate_join.restype = st
        L.estimate_join.argtypes = [ctypes.POINTER(sk_graph), u64, ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double), vp]
        if hasattr(L, "sketch_wire_pack"):   # (experimental builds of older revisions lack it)
            L.sketch_wire_pack.restype = st
            L.sketch_wire_pack.argtypes = [vp, vp, u64, vp, vp]
            L.sketch_wire_unpack.restype = st
            L.sketch_wire_unpack.argtypes = [vp, vp, u64, vp]
        L.estimate_join_exact.restype = st
        L.estimate_join_exact.argtypes = [ctypes.POINTER(sk_graph), u64, ctypes.c_char_p, u32, vp]
        L.estimate_subplans.restype = st
        L.estimate_subplans.argtypes = [ctypes.POINTER(sk_graph), ctypes.POINTER(u64), u32,
                                        ctypes.POINTER(ctypes.c_double), vp]
        L.plan_greedy.restype = st
        L.plan_greedy.argtypes = [ctypes.POINTER(sk_graph), ctypes.POINTER(u32), ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double), vp]
        L.plan_enumerate.restype = st
        L.plan_enumerate.argtypes = [ctypes.POINTER(sk_graph), ctypes.POINTER(sk_enum_config), ctypes.POINTER(u32),
                                     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(sk_enum_stats), vp]
        L.exact_join_size.restype = st
        L.exact_join_size.argtypes = [ctypes.POINTER(sk_join_data), u64, ctypes.c_char_p, u32,
                                      ctypes.POINTER(ctypes.c_double), vp]
        if hasattr(L, "sketch_peer_push"):   # (experimental builds of older revisions lack it)
            L.sketch_update_filtered_push.restype = st
            L.sketch_update_filtered_push.argtypes = [ctypes.POINTER(sk_column), u32, u64, ctypes.POINTER(sk_pred), u32,
                                                      ctypes.POINTER(sk_target), u32, vp, ctypes.POINTER(sk_peer_push), vp]
            L.sketch_peer_push.restype = st
            L.sketch_peer_push.argtypes = [ctypes.POINTER(sk_peer_push), vp]
            L.sketch_peer_gather.restype = st
            L.sketch_peer_gather.argtypes = [ctypes.POINTER(sk_peer_push), vp]
            L.sk_ipc_alloc.restype = st
            L.sk_ipc_alloc.argtypes = [u64, ctypes.c_int, ctypes.POINTER(vp), ctypes.c_char_p]
            L.sk_ipc_free.restype = st
            L.sk_ipc_free.argtypes = [vp]
            L.sk_ipc_open.restype = st
            L.sk_ipc_open.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(vp)]
            L.sk_ipc_close.restype = st
            L.sk_ipc_close.argtypes = [vp]
        L.sk_last_error.restype = ctypes.c_char_p
        L.sk_last_error.argtypes = []
        L.sk_kernel_launches.restype = ctypes.c_uint64
        L.sk_kernel_launches.argtypes = []
        L.sk_version.restype = ctypes.c_char_p
        L.sk_version.argtypes = []
        _lib = L
    return _lib


def _check(status: int):
    if status != SK_OK:
        raise SkError(status, lib().sk_last_error().decode())


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Sketch:
    """A Fast-AGMS vector (ndim 1), partitioned matrix (ndim 2) or 3-D partitioned tensor
    (ndim 3) sketch whose int64 counters are a caller-owned torch tensor
    (``self.counters``); the dimensions are in canonical edge order."""

    def __init__(self, d: int, w, edge_ids, master_seed: int = 42, device=None, counters: torch.Tensor | None = None):
        w = list(w)
        edge_ids = list(edge_ids)
        assert len(w) == len(edge_ids) and len(w) in (1, 2, 3)
        self.d, self.w, self.edge_ids, self.master_seed = d, w, edge_ids, master_seed
        device = torch.device(device if device is not None else "cuda")
        if device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        shape = (d, *w)
        if counters is None:
            counters = torch.zeros(shape, dtype=torch.int64, device=device)
        assert counters.dtype == torch.int64 and counters.is_contiguous() and tuple(counters.shape) == shape
        self.counters = counters
        desc = sk_desc()
        desc.d, desc.ndim = d, len(w)
        for q in range(len(w)):
            desc.w[q] = w[q]
            desc.edge_id[q] = edge_ids[q].encode()
        desc.master_seed = master_seed
        h = ctypes.c_void_p()
        _check(lib().sketch_create(ctypes.byref(desc), counters.device.index, ctypes.c_void_p(counters.data_ptr()),
                                   ctypes.byref(h)))
        self.handle = h

    @property
    def ndim(self) -> int:
        return len(self.w)

    def zero_(self, stream=None):
        _check(lib().sketch_zero(self.handle, ctypes.c_void_p(_stream_ptr(stream))))
        return self

    def close(self):
        if getattr(self, "handle", None) and _lib is not None:
            lib().sketch_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sketch_update_filtered(columns, n_rows: int, preds, targets, survivors: torch.Tensor | None = None, stream=None,
                           domains=None, push=None):
    """One fused scan.  columns: list of int32/int64 CUDA tensors; preds: list of
    (col_index, kind, lo, hi, set_values); targets: list of (Sketch, [key col indices]);
    domains: optional per-column key-domain hints (0 = unknown); push: optional
    (src int64 CUDA tensor, [dst device pointers]) — the cross-GPU merge over peer memory
    (sketch_update_filtered_push), fused into the scan where the library can."""
    ncol = len(columns)
    cols = (sk_column * max(1, ncol))()
    for i, c in enumerate(columns):
        # device tensors, or pinned host tensors (mapped, read in place over PCIe) for key
        # columns of tables with predicates: only the survivors' keys are then transferred
        assert (c.is_cuda or c.is_pinned()) and c.dtype in (torch.int32, torch.int64) and c.is_contiguous()
        cols[i].data = c.data_ptr()
        cols[i].dtype = SK_INT64 if c.dtype == torch.int64 else SK_INT32
        cols[i].domain = int(domains[i]) if domains else 0
    keep = []
    pr = (sk_pred * max(1, len(preds)))()
    for i, p in enumerate(preds):
        p = tuple(p) + (None,) * (5 - len(p))
        pr[i].col, pr[i].kind, pr[i].lo, pr[i].hi = p[0], p[1], p[2], p[3]
        if p[1] == SUBSET:
            vals = list(p[4] or [])
            arr = (ctypes.c_int64 * max(1, len(vals)))(*vals)
            keep.append(arr)
            pr[i].set = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64))
            pr[i].set_size = len(vals)
    tg = (sk_target * max(1, len(targets)))()
    for i, (sk, keys) in enumerate(targets):
        tg[i].sketch = sk.handle
        for q, k in enumerate(keys):
            tg[i].key_col[q] = k
    sp = ctypes.c_void_p(survivors.data_ptr()) if survivors is not None else None
    if push is not None:
        pp = _peer_push_desc(push[0], push[1], push[2] if len(push) > 2 else None)
        _check(lib().sketch_update_filtered_push(cols, ncol, n_rows, pr, len(preds), tg, len(targets), sp,
                                                 ctypes.byref(pp), ctypes.c_void_p(_stream_ptr(stream))))
        return
    _check(lib().sketch_update_filtered(cols, ncol, n_rows, pr, len(preds), tg, len(targets), sp,
                                        ctypes.c_void_p(_stream_ptr(stream))))


def _peer_push_desc(src, dst_ptrs, owner=None) -> "sk_peer_push":
    """owner = (rank, offset, total): reduce-scatter mode (each element to its owner only)."""
    pp = sk_peer_push()
    if src is not None:
        assert src.dtype == torch.int64 and src.is_cuda and src.is_contiguous()
        pp.src = src.data_ptr()
        pp.n = src.numel()
    arr = (ctypes.c_void_p * max(1, len(dst_ptrs)))(*[int(p) for p in dst_ptrs])
    pp._keep = arr
    pp.dst = ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))
    pp.n_peers = len(dst_ptrs)
    if owner is not None:
        pp.owner_mode, pp.rank, pp.offset, pp.total = 1, int(owner[0]), int(owner[1]), int(owner[2])
    return pp


def sketch_peer_push(src: torch.Tensor, dst_ptrs, stream=None, owner=None):
    """Add `src` (this rank's partial slice) into every rank's merged slice (device pointers
    mapped in this process, own included), or with owner = (rank, offset, total) into the
    owning rank's only: the cross-GPU merge over peer memory."""
    pp = _peer_push_desc(src, dst_ptrs, owner)
    _check(lib().sketch_peer_push(ctypes.byref(pp), ctypes.c_void_p(_stream_ptr(stream))))


def sketch_peer_gather(dst_ptrs, rank: int, total: int, stream=None):
    """Owner-mode merge, second half: this rank's merged buffer (dst_ptrs[rank]) receives the
    ranges owned by the other ranks (dst_ptrs = every rank's merged-buffer base)."""
    pp = _peer_push_desc(None, dst_ptrs, (rank, 0, total))
    _check(lib().sketch_peer_gather(ctypes.byref(pp), ctypes.c_void_p(_stream_ptr(stream))))


class IpcBuffer:
    """A library-allocated, zeroed int64 device buffer that other processes can map (CUDA IPC):
    `.tensor` is a torch view of it, `.handle` the bytes to send to the peers."""

    def __init__(self, numel: int, device: torch.device):
        self.device = torch.device(device)
        ptr = ctypes.c_void_p()
        h = ctypes.create_string_buffer(SK_IPC_HANDLE_BYTES)
        _check(lib().sk_ipc_alloc(numel * 8, self.device.index or 0, ctypes.byref(ptr), h))
        self.ptr, self.numel, self.handle = ptr.value, numel, h.raw
        self.tensor = _tensor_at(self.ptr, numel, self.device)

    def close(self):
        if self.ptr:
            self.tensor = None
            _check(lib().sk_ipc_free(ctypes.c_void_p(self.ptr)))
            self.ptr = None


def ipc_open(handle: bytes, device: torch.device) -> int:
    """Map another process's IpcBuffer; returns its device pointer in this process."""
    ptr = ctypes.c_void_p()
    _check(lib().sk_ipc_open(handle, torch.device(device).index or 0, ctypes.byref(ptr)))
    return ptr.value


def ipc_close(ptr: int):
    _check(lib().sk_ipc_close(ctypes.c_void_p(ptr)))


def _tensor_at(ptr: int, numel: int, device: torch.device) -> torch.Tensor:
    """A torch int64 tensor over existing device memory (the library owns it)."""
    class _Arr:
        __cuda_array_interface__ = {"shape": (numel,), "typestr": "<i8", "data": (ptr, False), "version": 3,
                                    "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_Arr(), device=device)


def _columns(columns, domains=None):
    cols = (sk_column * max(1, len(columns)))()
    for i, c in enumerate(columns):
        assert c.is_cuda and c.dtype in (torch.int32, torch.int64) and c.is_contiguous()
        cols[i].data = c.data_ptr()
        cols[i].dtype = SK_INT64 if c.dtype == torch.int64 else SK_INT32
        cols[i].domain = int(domains[i]) if domains else 0
    return cols


def _preds(preds, keep):
    pr = (sk_pred * max(1, len(preds)))()
    for i, p in enumerate(preds):
        p = tuple(p) + (None,) * (5 - len(p))
        pr[i].col, pr[i].kind, pr[i].lo, pr[i].hi = p[0], p[1], p[2], p[3]
        if p[1] == SUBSET:
            vals = list(p[4] or [])
            arr = (ctypes.c_int64 * max(1, len(vals)))(*vals)
            keep.append(arr)
            pr[i].set = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64))
            pr[i].set_size = len(vals)
    return pr


def exact_join_size(tables, edges, subset_mask: int, stream=None) -> int:
    """Exact |join| of an acyclic connected sub-plan (accuracy evaluation).
    tables: list of (columns [int32/int64 CUDA tensors], preds as in sketch_update_filtered);
    edges: list of (u, v, col_u, col_v, key_lo, key_domain); subset_mask: bit t = table t."""
    keep = []
    tds = (sk_table_data * len(tables))()
    for i, (cols, preds) in enumerate(tables):
        c = _columns(cols)
        p = _preds(preds, keep)
        keep += [c, p]
        tds[i].n_rows = int(cols[0].numel()) if cols else 0
        tds[i].cols, tds[i].n_cols = ctypes.cast(c, ctypes.POINTER(sk_column)), len(cols)
        tds[i].preds, tds[i].n_preds = ctypes.cast(p, ctypes.POINTER(sk_pred)), len(preds)
    E = len(edges)
    arr = lambda t, vals: (t * max(1, E))(*vals)
    eu, ev = arr(ctypes.c_uint32, [e[0] for e in edges]), arr(ctypes.c_uint32, [e[1] for e in edges])
    cu, cv = arr(ctypes.c_uint32, [e[2] for e in edges]), arr(ctypes.c_uint32, [e[3] for e in edges])
    lo, dom = arr(ctypes.c_int64, [e[4] for e in edges]), arr(ctypes.c_uint64, [e[5] for e in edges])
    jd = sk_join_data(len(tables), tds, E, eu, ev, cu, cv, lo, dom)
    buf = ctypes.create_string_buffer(256)
    approx = ctypes.c_double()
    _check(lib().exact_join_size(ctypes.byref(jd), subset_mask, buf, 256, ctypes.byref(approx),
                                 ctypes.c_void_p(_stream_ptr(stream))))
    return int(buf.value.decode())


def sketch_merge(dst: Sketch, src: Sketch, stream=None):
    _check(lib().sketch_merge(dst.handle, src.handle, ctypes.c_void_p(_stream_ptr(stream))))


def sketch_wire_pack(counters: torch.Tensor, wire: torch.Tensor, overflow: torch.Tensor | None = None, stream=None):
    """int64 counters -> int32 wire buffer (same length), for the int32 all-reduce."""
    assert counters.dtype == torch.int64 and wire.dtype == torch.int32 and counters.numel() == wire.numel()
    assert counters.is_contiguous() and wire.is_contiguous()
    _check(lib().sketch_wire_pack(ctypes.c_void_p(counters.data_ptr()), ctypes.c_void_p(wire.data_ptr()),
                                  counters.numel(), ctypes.c_void_p(overflow.data_ptr() if overflow is not None else 0),
                                  ctypes.c_void_p(_stream_ptr(stream))))


def sketch_wire_unpack(wire: torch.Tensor, counters: torch.Tensor, stream=None):
    """int32 wire buffer -> int64 counters (same length)."""
    assert counters.dtype == torch.int64 and wire.dtype == torch.int32 and counters.numel() == wire.numel()
    assert counters.is_contiguous() and wire.is_contiguous()
    _check(lib().sketch_wire_unpack(ctypes.c_void_p(wire.data_ptr()), ctypes.c_void_p(counters.data_ptr()),
                                    counters.numel(), ctypes.c_void_p(_stream_ptr(stream))))


class JoinGraph:
    """sk_graph wrapper.  tables: list of aliases (index order = tie order);
    survivors: list of ints; edges: list of (u, v, Sketch_u, Sketch_v);
    mats: list of (table, e0, e1, Sketch) — matrices, and 3-D tensors (e0, e1 = their first
    two edges)."""

    def __init__(self, tables, survivors, edges, mats=()):
        self.tables = list(tables)
        n, E, M = len(self.tables), len(edges), len(mats)
        self._surv = (ctypes.c_int64 * max(1, n))(*[int(s) for s in survivors])
        self._eu = (ctypes.c_uint32 * max(1, E))(*[e[0] for e in edges])
        self._ev = (ctypes.c_uint32 * max(1, E))(*[e[1] for e in edges])
        self._vu = (ctypes.c_void_p * max(1, E))(*[e[2].handle.value for e in edges])
        self._vv = (ctypes.c_void_p * max(1, E))(*[e[3].handle.value for e in edges])
        self._mt = (ctypes.c_uint32 * max(1, M))(*[m[0] for m in mats])
        self._m0 = (ctypes.c_uint32 * max(1, M))(*[m[1] for m in mats])
        self._m1 = (ctypes.c_uint32 * max(1, M))(*[m[2] for m in mats])
        self._mp = (ctypes.c_void_p * max(1, M))(*[m[3].handle.value for m in mats])
        self._keep = (edges, mats)
        g = sk_graph()
        g.n_tables, g.survivors = n, self._surv
        g.n_edges, g.edge_u, g.edge_v = E, self._eu, self._ev
        g.vec_u = ctypes.cast(self._vu, ctypes.POINTER(ctypes.c_void_p))
        g.vec_v = ctypes.cast(self._vv, ctypes.POINTER(ctypes.c_void_p))
        g.n_mats, g.mat_table, g.mat_e0, g.mat_e1 = M, self._mt, self._m0, self._m1
        g.mat = ctypes.cast(self._mp, ctypes.POINTER(ctypes.c_void_p))
        self.g = g
        self.d = edges[0][2].d if edges else 1

    def mask(self, subset) -> int:
        m = 0
        for t in subset:
            m |= 1 << self.tables.index(t)
        return m

    def estimate_join(self, subset, stream=None):
        """(Est as fp64, per-row fp64 list)."""
        est = ctypes.c_double()
        rows = (ctypes.c_double * self.d)()
        _check(lib().estimate_join(ctypes.byref(self.g), self.mask(subset), ctypes.byref(est), rows,
                                   ctypes.c_void_p(_stream_ptr(stream))))
        return est.value, list(rows)

    def estimate_join_exact(self, subset, stream=None) -> list[int]:
        stride = 192
        buf = ctypes.create_string_buffer(stride * self.d)
        _check(lib().estimate_join_exact(ctypes.byref(self.g), self.mask(subset), buf, stride,
                                         ctypes.c_void_p(_stream_ptr(stream))))
        raw = buf.raw
        # a singleton's value is its exact survivor count, written once (row 0)
        rows = 1 if bin(self.mask(subset)).count("1") == 1 else self.d
        vals = [int(raw[r * stride:(r + 1) * stride].split(b"\0", 1)[0].decode()) for r in range(rows)]
        return vals * self.d if rows == 1 else vals

    def estimate_subplans(self, subsets, stream=None) -> list[float]:
        n = len(subsets)
        masks = (ctypes.c_uint64 * max(1, n))(*[self.mask(s) for s in subsets])
        est = (ctypes.c_double * max(1, n))()
        _check(lib().estimate_subplans(ctypes.byref(self.g), masks, n, est, ctypes.c_void_p(_stream_ptr(stream))))
        return list(est)[:n]

    def plan_greedy(self, stream=None):
        n = len(self.tables)
        order = (ctypes.c_uint32 * n)()
        pre = (ctypes.c_double * n)()
        cost = ctypes.c_double()
        _check(lib().plan_greedy(ctypes.byref(self.g), order, pre, ctypes.byref(cost),
                                 ctypes.c_void_p(_stream_ptr(stream))))
        return [self.tables[i] for i in order], list(pre), cost.value

    def plan_enumerate(self, mode="limit", max_plans=10, alpha=0.5, beta=0.5, prune=True, stream=None):
        """Algorithm 1: (order, per-prefix cards, cost, stats dict).
        mode: greedy | full-greedy | limit (max_plans per source) | exhaustive."""
        n = len(self.tables)
        cfg = sk_enum_config(alpha, beta, ENUM_MODES[mode], max_plans, 0 if prune else 1)
        order = (ctypes.c_uint32 * n)()
        pre = (ctypes.c_double * n)()
        cost = ctypes.c_double()
        stats = sk_enum_stats()
        _check(lib().plan_enumerate(ctypes.byref(self.g), ctypes.byref(cfg), order, pre, ctypes.byref(cost),
                                    ctypes.byref(stats), ctypes.c_void_p(_stream_ptr(stream))))
        st = {f: int(getattr(stats, f)) for f, _ in sk_enum_stats._fields_}
        return [self.tables[i] for i in order], list(pre), cost.value, st


def kernel_launches() -> int:
    return int(lib().sk_kernel_launches())


def version() -> str:
    return lib().sk_version().decode()
