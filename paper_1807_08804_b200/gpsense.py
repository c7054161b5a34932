"""Thin ctypes binding of include/gpsense.h (argument marshalling only).

Every step of filtering and joining runs in libgpsense.so's sm_100a kernels; this
module only converts Python/numpy/torch arguments into the C structs and wraps
results.  PyTorch is used for device memory views (zero-copy via
__cuda_array_interface__) and streams.  There is no CPU fallback: if the CUDA
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgpsense.so")

GPS_OK, GPS_EINVAL, GPS_EDISCONNECTED, GPS_ENOMEM, GPS_ECUDA, GPS_ENCCL, GPS_EOVERFLOW, GPS_EUNSUPPORTED = (
    0, -1, -2, -3, -4, -5, -6, -7)
GPS_ANY = -1
GPS_FREE = -1
GPS_DIRECTED, GPS_UNDIRECTED = 0, 1
GPS_REFINE_UNTIL_STABLE = 0xFFFFFFFF
GPS_PLAN_RANKING, GPS_PLAN_COMMONSENSE = 0, 1
KERNEL_CLASSES = ["check", "collect", "explore", "bitand", "ec_count", "ec_write", "scan", "join_len",
                  "join_count", "join_write", "load", "propagate", "clear"]
NK = len(KERNEL_CLASSES)
K = {name: i for i, name in enumerate(KERNEL_CLASSES)}

_STATUS = {GPS_EINVAL: "EINVAL", GPS_EDISCONNECTED: "EDISCONNECTED", GPS_ENOMEM: "ENOMEM",
           GPS_ECUDA: "ECUDA", GPS_ENCCL: "ENCCL", GPS_EOVERFLOW: "EOVERFLOW",
           GPS_EUNSUPPORTED: "EUNSUPPORTED"}


class GpsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"gps error {_STATUS.get(status, status)}: {msg}")
        self.status = status


DEV_ALLOC = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
DEV_FREE = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class CtxOpts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("nccl_comm", ctypes.c_void_p),
                ("rank", ctypes.c_int), ("world", ctypes.c_int), ("dev_alloc", DEV_ALLOC),
                ("dev_free", DEV_FREE), ("alloc_user", ctypes.c_void_p)]


class CsrDesc(ctypes.Structure):
    _fields_ = [("n_vertices", ctypes.c_uint32), ("n_arcs", ctypes.c_uint64),
                ("offsets", ctypes.c_void_p), ("targets", ctypes.c_void_p),
                ("edge_labels", ctypes.c_void_p), ("vertex_labels", ctypes.c_void_p),
                ("flags", ctypes.c_uint32)]


class QEdge(ctypes.Structure):
    _fields_ = [("src", ctypes.c_int32), ("dst", ctypes.c_int32), ("label", ctypes.c_int32)]


class QueryDesc(ctypes.Structure):
    _fields_ = [("n_vertices", ctypes.c_uint32), ("n_edges", ctypes.c_uint32),
                ("vertex_labels", ctypes.c_void_p), ("bound", ctypes.c_void_p),
                ("edges", ctypes.c_void_p)]


class MatchOpts(ctypes.Structure):
    _fields_ = [("refine_rounds", ctypes.c_uint32), ("reverse_refine", ctypes.c_int32),
                ("lowconn_threshold", ctypes.c_uint32), ("result_on_device", ctypes.c_int32),
                ("rebalance_threshold", ctypes.c_float), ("plan_mode", ctypes.c_int32),
                ("row_budget_bytes", ctypes.c_uint64)]


class Stats(ctypes.Structure):
    _fields_ = [("queries", ctypes.c_uint64), ("embeddings", ctypes.c_uint64),
                ("launches", ctypes.c_uint64), ("host_syncs", ctypes.c_uint64),
                ("k_launches", ctypes.c_uint64 * NK), ("k_bytes", ctypes.c_double * NK),
                ("k_ms", ctypes.c_double * NK), ("k_timed", ctypes.c_uint64 * NK),
                ("join_rows_max", ctypes.c_uint64), ("join_rows_total", ctypes.c_uint64)]


def _load_lib():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (nvcc, sm_100a); "
                          "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    S = ctypes.c_int
    sig = {
        "gps_default_opts": (S, [P]),
        "gps_create": (S, [P, P]),
        "gps_destroy": (S, [P]),
        "gps_load_data_graph": (S, [P, P, P]),
        "gps_free_graph": (S, [P]),
        "gps_graph_info": (S, [P, P, P, P, P]),
        "gps_match": (S, [P, P, P, P, P]),
        "gps_match_host": (S, [P, P, P, P, P, ctypes.c_uint64, P]),
        "gps_count": (S, [P, P, P, P, P]),
        "gps_result_info": (S, [P, P, P, P, P]),
        "gps_result_free": (None, [P]),
        "gps_result_free_after": (None, [P, P]),
        "gps_last_error": (ctypes.c_char_p, []),
        "gps_get_stats": (S, [P, P]),
        "gps_reset_stats": (S, [P]),
        "gps_set_profiling": (S, [P, ctypes.c_uint32]),
        "gps_debug_plan": (S, [P, P, P, P, P, P, P]),
        "gps_debug_candidates": (S, [P, P, P, P, S, P]),
        "gps_match_batch": (S, [P, P, P, ctypes.c_uint32, P, P, P]),
        "gps_count_batch": (S, [P, P, P, ctypes.c_uint32, P, P, P]),
        "gps_set_workers": (S, [P, ctypes.c_uint32]),
        "gps_set_slice": (S, [P, ctypes.c_uint32]),
        "gps_match_batch_host": (S, [P, P, P, ctypes.c_uint32, P, P, ctypes.c_uint64, P, P, P]),
        "gps_result_global_rows": (S, [P, P]),
        "gps_local_comm_create": (S, [ctypes.c_int, P]),
        "gps_shard_plan": (S, [ctypes.c_int, ctypes.c_int, P, ctypes.c_float, P, P, P]),
        "gps_load_triples": (S, [P, ctypes.c_uint32, ctypes.c_uint64, P, P, P, P, ctypes.c_uint32, P]),
        "gps_match_project": (S, [P, P, P, P, ctypes.c_uint32, P, P]),
        "gps_count_project": (S, [P, P, P, P, ctypes.c_uint32, P, P]),
        "gps_match_named": (S, [P, P, P, P, P, ctypes.c_uint32, P, P]),
        "gps_compress": (S, [P, P, ctypes.c_uint32, P, P]),
        "gps_rel_join": (S, [P, P, P, ctypes.c_uint64, P, P, ctypes.c_uint64, P]),
        "gps_rel_union": (S, [P, P, P, ctypes.c_uint64, P, P, ctypes.c_uint64, P]),
        "gps_rel_difference": (S, [P, P, P, ctypes.c_uint64, P, P, ctypes.c_uint64, P]),
        "gps_rel_closure": (S, [P, P, P, ctypes.c_uint64, ctypes.c_uint32, P, P]),
        "gps_free_compressed": (S, [P]),
        "gps_compressed_info": (S, [P, ctypes.c_uint32, P, P, P]),
        "gps_compressed_fetch": (S, [P, P, ctypes.c_uint32, P, P, P, P, P, P, P, P]),
        "gps_compressed_candidates": (S, [P, P, ctypes.c_uint32, P, P]),
        "gps_graph_attach_compressed": (S, [P, P, ctypes.c_uint32]),
        "gps_count_named": (S, [P, P, P, P, P, ctypes.c_uint32, P, P]),
        "gps_shard_recv": (S, [ctypes.c_int, ctypes.c_int, P, P, P]),
        "gps_local_comm_destroy": (S, [P]),
        "gps_create_local_rank": (S, [P, P, ctypes.c_int, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load_lib()
EXPORTED = ["gps_default_opts", "gps_create", "gps_destroy", "gps_load_data_graph", "gps_free_graph",
            "gps_graph_info", "gps_match", "gps_match_host", "gps_count", "gps_result_info",
            "gps_result_free", "gps_result_free_after", "gps_last_error", "gps_get_stats", "gps_reset_stats",
            "gps_set_profiling", "gps_debug_plan", "gps_debug_candidates", "gps_match_batch",
            "gps_count_batch", "gps_set_workers", "gps_set_slice", "gps_match_batch_host",
            "gps_result_global_rows", "gps_shard_plan", "gps_shard_recv", "gps_load_triples",
            "gps_match_project", "gps_count_project", "gps_match_named", "gps_count_named", "gps_compress", "gps_free_compressed", "gps_compressed_info",
            "gps_compressed_fetch", "gps_compressed_candidates", "gps_graph_attach_compressed", "gps_rel_join",
            "gps_rel_union", "gps_rel_difference", "gps_rel_closure", "gps_local_comm_create", "gps_local_comm_destroy", "gps_create_local_rank"]


def _check(st: int):
    if st != GPS_OK:
        raise GpsError(st, (lib.gps_last_error() or b"").decode())


def _addr(a) -> Optional[int]:
    return None if a is None else a.ctypes.data


def default_opts(**kw) -> MatchOpts:
    o = MatchOpts()
    _check(lib.gps_default_opts(ctypes.byref(o)))
    for k_, v in kw.items():
        setattr(o, k_, float(v) if k_ == "rebalance_threshold" else int(v))
    return o


def _with_device(o: MatchOpts, on_device: bool) -> MatchOpts:
    return MatchOpts(o.refine_rounds, o.reverse_refine, o.lowconn_threshold, 1 if on_device else 0,
                     o.rebalance_threshold, o.plan_mode, o.row_budget_bytes)


class _QueryArrays:
    """Keeps the numpy buffers behind a QueryDesc alive."""

    def __init__(self, q):
        if isinstance(q, dict):
            k, vl, bd, edges = q["k"], q["vlabels"], q["bound"], q["edges"]
        else:
            k, vl, bd, edges = q.k, q.vlabels, q.bound, q.edges
        self.vl = np.ascontiguousarray(np.asarray(vl, np.int32).reshape(-1))
        self.bd = np.ascontiguousarray(np.asarray(bd, np.int64).reshape(-1))
        e = np.asarray(edges, np.int32).reshape(-1, 3)
        self.e = np.ascontiguousarray(e)
        self.k = int(k)
        self.desc = QueryDesc(self.k, int(self.e.shape[0]), _addr(self.vl), _addr(self.bd),
                              _addr(self.e) if self.e.shape[0] else None)


_QDESC_DTYPE = np.dtype([("k", "<u4"), ("ne", "<u4"), ("vl", "<u8"), ("bd", "<u8"), ("e", "<u8")])
assert _QDESC_DTYPE.itemsize == ctypes.sizeof(QueryDesc)


class QueryBatch:
    """A list of queries marshalled ONCE into contiguous arrays + a gps_query array.

    Pass it instead of a list to the batch calls to keep per-call host work at a
    single library call (the descriptors stay valid while this object lives)."""

    def __init__(self, queries):
        qs = [q if not isinstance(q, dict) else _DictQuery(q) for q in queries]
        self.n = len(qs)
        ks = np.fromiter((int(q.k) for q in qs), np.int64, self.n)
        nes = np.fromiter((len(q.edges) for q in qs), np.int64, self.n)
        self.vl = np.ascontiguousarray([int(x) for q in qs for x in q.vlabels], dtype=np.int32)
        self.bd = np.ascontiguousarray([int(x) for q in qs for x in q.bound], dtype=np.int64)
        self.e = np.ascontiguousarray([int(x) for q in qs for ed in q.edges for x in ed], dtype=np.int32)
        if self.vl.shape[0] != ks.sum() or self.bd.shape[0] != ks.sum() or self.e.shape[0] != 3 * nes.sum():
            raise ValueError("query arrays do not match their sizes")
        vo = np.concatenate([[0], np.cumsum(ks)[:-1]]) if self.n else ks
        eo = np.concatenate([[0], np.cumsum(nes)[:-1]]) if self.n else nes
        d = np.zeros(max(self.n, 1), _QDESC_DTYPE)
        d["k"][: self.n] = ks
        d["ne"][: self.n] = nes
        d["vl"][: self.n] = self.vl.ctypes.data + 4 * vo if self.vl.size else 0
        d["bd"][: self.n] = self.bd.ctypes.data + 8 * vo if self.bd.size else 0
        d["e"][: self.n] = np.where(nes > 0, self.e.ctypes.data + 12 * eo, 0) if self.e.size else 0
        self.desc = d
        self.arr = ctypes.cast(ctypes.c_void_p(d.ctypes.data), ctypes.POINTER(QueryDesc))

    def __len__(self):
        return self.n


class _DictQuery:
    def __init__(self, d):
        self.k, self.vlabels, self.bound, self.edges = d["k"], d["vlabels"], d["bound"], d["edges"]


def _consumer_stream(device: int):
    try:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    except Exception:
        return None


class _DeviceRows:
    """Owner of a device gps_result; exposes __cuda_array_interface__ for torch.

    Holds the Context (the ctx owns the rows' memory and its stream orders their
    release), and frees with gps_result_free_after on the torch stream current at
    release time, so kernels still reading the rows finish before the memory is reused."""

    def __init__(self, res, rows, cols, ptr, ctx=None):
        self._res = res
        self._ctx = ctx
        self.__cuda_array_interface__ = {"shape": (int(rows), int(cols)), "typestr": "<u4",
                                         "data": (int(ptr), False), "version": 3, "strides": None,
                                         "stream": None}

    def __del__(self):
        if self._res and lib is not None:
            try:
                dev = self._ctx.device if self._ctx is not None else 0
                lib.gps_result_free_after(self._res, _consumer_stream(dev))
            except Exception:
                pass
            self._res = None
        self._ctx = None


class _HostRows:
    """Owner of a host (pinned) gps_result; exposes __array_interface__ for numpy (zero-copy)."""

    def __init__(self, res, rows, cols, ptr, ctx=None):
        self._res = res
        self._ctx = ctx   # the ctx owns the pinned rows
        self.__array_interface__ = {"shape": (int(rows), int(cols)), "typestr": "<u4",
                                    "data": (int(ptr), False), "version": 3}

    def __del__(self):
        if self._res and lib is not None:
            try:
                lib.gps_result_free(self._res)
            except Exception:
                pass
            self._res = None


class BatchResult:
    """Result handles of a gps_match_batch call; rows() is cheap, tensor(i) wraps lazily."""

    def __init__(self, ctx, res, n):
        self.ctx, self._res, self.n = ctx, res, n
        self._rows = np.zeros(n, np.uint64)
        for i in range(n):
            if res[i]:
                r = ctypes.c_uint64()
                lib.gps_result_info(res[i], ctypes.byref(r), None, None, None)
                self._rows[i] = r.value

    def rows(self) -> np.ndarray:
        return self._rows

    def tensor(self, i):
        import torch
        rows, cols, ptr, ondev = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_void_p(), ctypes.c_int()
        lib.gps_result_info(self._res[i], ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(ptr),
                            ctypes.byref(ondev))
        if rows.value == 0:
            return torch.empty((0, cols.value), dtype=torch.uint32, device=f"cuda:{self.ctx.device}")
        h = _DeviceRows(None, rows.value, cols.value, ptr.value)   # owned by this BatchResult
        t = torch.as_tensor(h, device=f"cuda:{self.ctx.device}")
        t._gps_owner = self
        return t

    def free(self):
        if self._res is not None and lib is not None:
            st = _consumer_stream(self.ctx.device)
            for i in range(self.n):
                if self._res[i]:
                    lib.gps_result_free_after(self._res[i], st)
                    self._res[i] = None
        self._res = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Graph:
    def __init__(self, ctx: "Context", handle):
        self.ctx = ctx
        self._h = handle
        n, m, nvl, lb = ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint32()
        _check(lib.gps_graph_info(handle, ctypes.byref(n), ctypes.byref(m), ctypes.byref(nvl), ctypes.byref(lb)))
        self.n, self.arcs, self.n_vlabels, self.elabel_bits = n.value, m.value, nvl.value, lb.value

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h:
            lib.gps_free_graph(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Compressed:
    """f3 multi-level compression of a Graph (gps_compress); owns its device memory."""

    def __init__(self, ctx: "Context", graph: Graph, handle, levels: int):
        self.ctx, self.graph, self._h, self.levels = ctx, graph, handle, levels

    @property
    def handle(self):
        return self._h

    def info(self, lv: int):
        """(nodes, weighted out-edges, weighted in-edges) of level lv."""
        N, eo, ei = ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib.gps_compressed_info(self._h, lv, ctypes.byref(N), ctypes.byref(eo), ctypes.byref(ei)))
        return N.value, eo.value, ei.value

    def level(self, lv: int) -> dict:
        """Level lv (1..levels) as numpy arrays: group [n], label / w_out / w_in [nodes],
        edges_out / edges_in as dict {(U, V): weight}."""
        N, eo, ei = ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib.gps_compressed_info(self._h, lv, ctypes.byref(N), ctypes.byref(eo), ctypes.byref(ei)))
        n = self.graph.n
        grp = np.zeros(n, np.uint32)
        lab, wo, wi = (np.zeros(N.value, np.uint32) for _ in range(3))
        ko, wko = np.zeros(eo.value, np.uint64), np.zeros(eo.value, np.uint32)
        ki, wki = np.zeros(ei.value, np.uint64), np.zeros(ei.value, np.uint32)
        _check(lib.gps_compressed_fetch(self.ctx._h, self._h, lv, _addr(grp), _addr(lab), _addr(wo), _addr(wi),
                                        _addr(ko), _addr(wko), _addr(ki), _addr(wki)))
        def edges(k, w):
            return {(int(x >> 32), int(x & 0xffffffff)): int(y) for x, y in zip(k.tolist(), w.tolist())}
        return {"nodes": N.value, "group": grp, "label": lab, "w_out": wo, "w_in": wi,
                "edges_out": edges(ko, wko), "edges_in": edges(ki, wki)}

    def candidates(self, lv: int, q) -> np.ndarray:
        """Expanded weighted candidates as a (k, n) bool array."""
        qa = _QueryArrays(q)
        nw = (self.graph.n + 31) // 32
        bm = np.zeros((qa.k, nw), np.uint32)
        _check(lib.gps_compressed_candidates(self.ctx._h, self._h, lv, ctypes.byref(qa.desc), _addr(bm)))
        bits = np.unpackbits(bm.view(np.uint8).reshape(qa.k, -1), axis=1, bitorder="little")
        return bits[:, :self.graph.n].astype(bool)

    def attach(self, lv: int) -> None:
        """Filters on the graph apply the weighted candidate test of level lv (0 detaches)."""
        _check(lib.gps_graph_attach_compressed(self.graph.handle, self._h if lv else None, lv))

    def free(self):
        if self._h:
            try:
                lib.gps_graph_attach_compressed(self.graph.handle, None, 0)
            except Exception:
                pass
            lib.gps_free_compressed(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def shard_plan(world: int, rank: int, pairs_all, threshold: float = 1.10):
    """gps_shard_plan: (local_targets[world+1], rebalance, total)."""
    p = np.ascontiguousarray(pairs_all, np.uint64)
    lt = np.zeros(world + 1, np.uint64)
    rb, tot = ctypes.c_int(), ctypes.c_uint64()
    _check(lib.gps_shard_plan(int(world), int(rank), ctypes.c_void_p(p.ctypes.data), float(threshold),
                              ctypes.c_void_p(lt.ctypes.data), ctypes.byref(rb), ctypes.byref(tot)))
    return lt, bool(rb.value), int(tot.value)


def shard_recv(world: int, rank: int, send_matrix):
    """gps_shard_recv: (at[world], total)."""
    m = np.ascontiguousarray(send_matrix, np.uint64).reshape(-1)
    at = np.zeros(world, np.uint64)
    tot = ctypes.c_uint64()
    _check(lib.gps_shard_recv(int(world), int(rank), ctypes.c_void_p(m.ctypes.data), ctypes.c_void_p(at.ctypes.data),
                              ctypes.byref(tot)))
    return at, int(tot.value)


class LocalComm:
    """In-process ranks on one device (tests of the row-sharded join)."""

    def __init__(self, world: int):
        h = ctypes.c_void_p()
        _check(lib.gps_local_comm_create(int(world), ctypes.byref(h)))
        self._h, self.world = h, world

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.gps_local_comm_destroy(self._h)
            self._h = None


class Context:
    """One gps_ctx: a device and a stream (default: a library-owned stream).

    nccl_comm/rank/world: row-sharded join across ranks (ProcessGroupNCCL._comm_ptr());
    local_comm/rank: in-process ranks sharing one device (tests)."""

    def __init__(self, device: int = 0, stream=None, workers: int = 0, nccl_comm=None, rank: int = 0,
                 world: int = 1, local_comm: Optional[LocalComm] = None, torch_allocator: bool = False):
        o = CtxOpts(device, None, None, int(rank), int(world))
        if torch_allocator:
            # the library's device memory comes from torch's caching allocator (gps_ctx_opts.dev_alloc)
            import torch

            def _alloc(nbytes, stream, user):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), device, int(stream or 0))
                except Exception:   # out of memory: the library reports GPS_ENOMEM
                    return None

            def _free(ptr, stream, user):
                torch.cuda.caching_allocator_delete(int(ptr))

            self._alloc_cbs = (DEV_ALLOC(_alloc), DEV_FREE(_free))   # kept alive with the ctx
            o.dev_alloc, o.dev_free = self._alloc_cbs
        if stream is not None:
            o.stream = int(getattr(stream, "cuda_stream", stream))
        if nccl_comm is not None:
            o.nccl_comm = int(nccl_comm)
        h = ctypes.c_void_p()
        if local_comm is not None:
            _check(lib.gps_create_local_rank(ctypes.byref(o), local_comm._h, int(rank), ctypes.byref(h)))
            self._comm = local_comm
        else:
            _check(lib.gps_create(ctypes.byref(o), ctypes.byref(h)))
        self._h = h
        self.device = device
        if workers:
            self.set_workers(workers)

    def set_workers(self, n: int):
        _check(lib.gps_set_workers(self._h, int(n)))

    def set_slice(self, n: int):
        _check(lib.gps_set_slice(self._h, int(n)))

    def close(self):
        if self._h:
            lib.gps_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- graph ----
    def load_graph_csr(self, n, offsets, targets, edge_labels=None, vertex_labels=None,
                       undirected=False) -> Graph:
        off = np.ascontiguousarray(offsets, np.uint64)
        tgt = np.ascontiguousarray(targets, np.uint32)
        el = None if edge_labels is None else np.ascontiguousarray(edge_labels, np.uint16)
        vl = None if vertex_labels is None else np.ascontiguousarray(vertex_labels, np.uint16)
        d = CsrDesc(int(n), int(tgt.shape[0]), _addr(off), _addr(tgt), _addr(el), _addr(vl),
                    GPS_UNDIRECTED if undirected else GPS_DIRECTED)
        h = ctypes.c_void_p()
        _check(lib.gps_load_data_graph(self._h, ctypes.byref(d), ctypes.byref(h)))
        return Graph(self, h)

    def load_graph(self, g) -> Graph:
        """From a synth.DataGraph-like object (n, to_csr(), vlab, undirected)."""
        off, tgt, el = g.to_csr()
        return self.load_graph_csr(g.n, off, tgt, el, g.vlab, g.undirected)

    def load_triples(self, n, subject, relation, obj, vertex_labels=None, undirected=False) -> Graph:
        """A knowledge base as (subject, relation, object) triples (f2)."""
        su = np.ascontiguousarray(subject, np.uint32)
        ob = np.ascontiguousarray(obj, np.uint32)
        rl = None if relation is None else np.ascontiguousarray(relation, np.uint16)
        vl = None if vertex_labels is None else np.ascontiguousarray(vertex_labels, np.uint16)
        h = ctypes.c_void_p()
        _check(lib.gps_load_triples(self._h, int(n), int(su.shape[0]), _addr(su), _addr(rl), _addr(ob), _addr(vl),
                                    GPS_UNDIRECTED if undirected else GPS_DIRECTED, ctypes.byref(h)))
        return Graph(self, h)

    def match_project(self, graph: Graph, q, project, opts: Optional[MatchOpts] = None) -> np.ndarray:
        """Distinct projections of the embeddings onto the query vertices `project` (f2, P:826,
        P:937), lexicographically sorted, as a (rows, len(project)) uint32 numpy array."""
        qa = _QueryArrays(q)
        pj = np.ascontiguousarray(project, np.int32)
        o = _with_device(opts if opts is not None else default_opts(), False)
        res = ctypes.c_void_p()
        _check(lib.gps_match_project(self._h, graph.handle, ctypes.byref(qa.desc), ctypes.byref(o), pj.shape[0],
                                     _addr(pj), ctypes.byref(res)))
        rows, cols, ptr, ondev = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_void_p(), ctypes.c_int()
        lib.gps_result_info(res, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(ptr), ctypes.byref(ondev))
        a = np.zeros((rows.value, cols.value), np.uint32)
        if rows.value:
            ctypes.memmove(a.ctypes.data, ptr.value, rows.value * cols.value * 4)
        lib.gps_result_free(res)
        return a

    def count_project(self, graph: Graph, q, project, opts: Optional[MatchOpts] = None) -> int:
        qa = _QueryArrays(q)
        pj = np.ascontiguousarray(project, np.int32)
        c = ctypes.c_uint64()
        _check(lib.gps_count_project(self._h, graph.handle, ctypes.byref(qa.desc),
                                     ctypes.byref(opts) if opts is not None else None, pj.shape[0], _addr(pj),
                                     ctypes.byref(c)))
        return int(c.value)

    # ---- f4: gSparql relation primitives ----
    def _rel_rows(self, res) -> np.ndarray:
        rows, cols, ptr, ondev = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_void_p(), ctypes.c_int()
        lib.gps_result_info(res, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(ptr), ctypes.byref(ondev))
        a = np.zeros((rows.value, 2), np.uint32)
        if rows.value:
            import torch
            t = torch.as_tensor(_DeviceRows(None, rows.value, 2, ptr.value), device=f"cuda:{self.device}")
            a = t.cpu().numpy().copy()
        lib.gps_result_free(res)
        return a

    def _rel2(self, fn, a_src, a_dst, b_src, b_dst) -> np.ndarray:
        cols = [np.ascontiguousarray(x, np.uint32) for x in (a_src, a_dst, b_src, b_dst)]
        res = ctypes.c_void_p()
        _check(fn(self._h, _addr(cols[0]), _addr(cols[1]), cols[0].shape[0], _addr(cols[2]), _addr(cols[3]),
                  cols[2].shape[0], ctypes.byref(res)))
        return self._rel_rows(res)

    def rel_join(self, r_src, r_dst, s_src, s_dst) -> np.ndarray:
        """{(x, z) : (x, y) in R, (y, z) in S} as sorted distinct (rows, 2) uint32."""
        return self._rel2(lib.gps_rel_join, r_src, r_dst, s_src, s_dst)

    def rel_union(self, a_src, a_dst, b_src, b_dst) -> np.ndarray:
        return self._rel2(lib.gps_rel_union, a_src, a_dst, b_src, b_dst)

    def rel_difference(self, a_src, a_dst, b_src, b_dst) -> np.ndarray:
        return self._rel2(lib.gps_rel_difference, a_src, a_dst, b_src, b_dst)

    def rel_closure(self, src, dst, max_rounds: int = 0):
        """Transitive closure by the recursive-rule loop: (rows, rounds)."""
        s = np.ascontiguousarray(src, np.uint32)
        d = np.ascontiguousarray(dst, np.uint32)
        res, it = ctypes.c_void_p(), ctypes.c_uint32()
        _check(lib.gps_rel_closure(self._h, _addr(s), _addr(d), s.shape[0], int(max_rounds), ctypes.byref(res),
                                   ctypes.byref(it)))
        return self._rel_rows(res), int(it.value)

    def compress(self, graph: Graph, deltas) -> "Compressed":
        """gps_compress: levels 1..len(deltas) of the f3 multi-level compression (delta = 1 only)."""
        d = np.ascontiguousarray(deltas, np.float32)
        h = ctypes.c_void_p()
        _check(lib.gps_compress(self._h, graph.handle, d.shape[0], _addr(d), ctypes.byref(h)))
        return Compressed(self, graph, h, int(d.shape[0]))

    def match_named(self, graph: Graph, q, edge_var, project=None, opts: Optional[MatchOpts] = None) -> np.ndarray:
        """Named variable edges (f2): distinct (projection, label bindings) tuples, as a
        (rows, len(project or all k) + #names) uint32 numpy array in lexicographic order."""
        qa = _QueryArrays(q)
        ev = np.ascontiguousarray(edge_var, np.int32)
        pj = np.ascontiguousarray([] if project is None else project, np.int32)
        o = _with_device(opts if opts is not None else default_opts(), False)
        res = ctypes.c_void_p()
        _check(lib.gps_match_named(self._h, graph.handle, ctypes.byref(qa.desc), ctypes.byref(o), _addr(ev),
                                   pj.shape[0], _addr(pj) if pj.shape[0] else None, ctypes.byref(res)))
        rows, cols, ptr, ondev = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_void_p(), ctypes.c_int()
        lib.gps_result_info(res, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(ptr), ctypes.byref(ondev))
        a = np.zeros((rows.value, cols.value), np.uint32)
        if rows.value:
            ctypes.memmove(a.ctypes.data, ptr.value, rows.value * cols.value * 4)
        lib.gps_result_free(res)
        return a

    def count_named(self, graph: Graph, q, edge_var, project=None, opts: Optional[MatchOpts] = None) -> int:
        qa = _QueryArrays(q)
        ev = np.ascontiguousarray(edge_var, np.int32)
        pj = np.ascontiguousarray([] if project is None else project, np.int32)
        c = ctypes.c_uint64()
        _check(lib.gps_count_named(self._h, graph.handle, ctypes.byref(qa.desc),
                                   ctypes.byref(opts) if opts is not None else None, _addr(ev), pj.shape[0],
                                   _addr(pj) if pj.shape[0] else None, ctypes.byref(c)))
        return int(c.value)

    # ---- queries ----
    def match(self, graph: Graph, q, opts: Optional[MatchOpts] = None, device: bool = True):
        """All embeddings: torch uint32 (rows, k) CUDA tensor (device=True) or numpy array."""
        qa = _QueryArrays(q)
        o = opts if opts is not None else default_opts()
        o = _with_device(o, device)
        res = ctypes.c_void_p()
        _check(lib.gps_match(self._h, graph.handle, ctypes.byref(qa.desc), ctypes.byref(o), ctypes.byref(res)))
        rows, cols, ptr, ondev = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_void_p(), ctypes.c_int()
        _check(lib.gps_result_info(res, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(ptr),
                                   ctypes.byref(ondev)))
        if device:
            import torch
            holder = _DeviceRows(res, rows.value, cols.value, ptr.value, self)
            if rows.value == 0:
                del holder
                return torch.empty((0, cols.value), dtype=torch.uint32, device=f"cuda:{self.device}")
            return torch.as_tensor(holder, device=f"cuda:{self.device}")
        try:
            n = rows.value * cols.value
            if n == 0:
                return np.zeros((0, cols.value), np.uint32)
            buf = (ctypes.c_uint32 * n).from_address(ptr.value)
            return np.frombuffer(buf, dtype=np.uint32).reshape(rows.value, cols.value).copy()
        finally:
            lib.gps_result_free(res)

    def match_shard(self, graph: Graph, q, opts: Optional[MatchOpts] = None):
        """Row-sharded join: (this rank's rows as a numpy array, global row count)."""
        qa = _QueryArrays(q)
        o = _with_device(opts if opts is not None else default_opts(), False)
        res = ctypes.c_void_p()
        _check(lib.gps_match(self._h, graph.handle, ctypes.byref(qa.desc), ctypes.byref(o), ctypes.byref(res)))
        rows, cols, ptr, ondev, glob = (ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_void_p(), ctypes.c_int(),
                                        ctypes.c_uint64())
        lib.gps_result_info(res, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(ptr), ctypes.byref(ondev))
        lib.gps_result_global_rows(res, ctypes.byref(glob))
        a = np.zeros((rows.value, cols.value), np.uint32)
        if rows.value:
            ctypes.memmove(a.ctypes.data, ptr.value, rows.value * cols.value * 4)
        lib.gps_result_free(res)
        return a, int(glob.value)

    def match_host(self, graph: Graph, q, out=None, opts: Optional[MatchOpts] = None):
        """Rows into a caller-owned host buffer (numpy uint32 or pinned torch tensor).

        Returns the (rows, k) view of `out`; raises GpsError(EOVERFLOW) if it is too small.
        """
        qa = _QueryArrays(q)
        if out is None:
            out = np.zeros((1 << 16, qa.k), np.uint32)
        if hasattr(out, "data_ptr"):
            ptr, cap = out.data_ptr(), out.numel() // qa.k
        else:
            ptr, cap = out.ctypes.data, out.size // qa.k
        rows = ctypes.c_uint64()
        o = opts if opts is not None else default_opts()
        _check(lib.gps_match_host(self._h, graph.handle, ctypes.byref(qa.desc), ctypes.byref(o),
                                  ctypes.c_void_p(ptr), cap, ctypes.byref(rows)))
        flat = out.reshape(-1) if not hasattr(out, "data_ptr") else out.view(-1)
        return flat[: rows.value * qa.k].reshape(rows.value, qa.k)

    def _batch_desc(self, queries):
        qb = queries if isinstance(queries, QueryBatch) else QueryBatch(queries)
        return [None] * qb.n, qb.arr, qb

    def match_batch(self, graph: Graph, queries, opts: Optional[MatchOpts] = None, device: bool = True):
        """All embeddings of every query, run concurrently by the library's worker pool.

        Returns a list of torch uint32 (rows, k) CUDA tensors (zero-copy), or of
        numpy arrays copied to host by the library when device=False."""
        import torch
        qas, arr, _qb = self._batch_desc(queries)
        n = len(qas)
        res = (ctypes.c_void_p * max(n, 1))()
        st = np.zeros(max(n, 1), np.int32)
        o = opts if opts is not None else default_opts()
        o = _with_device(o, device)
        rc = lib.gps_match_batch(self._h, graph.handle, arr, n, ctypes.byref(o), res,
                                 ctypes.c_void_p(st.ctypes.data))
        out = []
        for i in range(n):
            if not res[i]:
                continue
            rows, cols, ptr, ondev = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_void_p(), ctypes.c_int()
            lib.gps_result_info(res[i], ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(ptr), ctypes.byref(ondev))
            if not device:
                if rows.value == 0:
                    lib.gps_result_free(ctypes.c_void_p(res[i]))
                    out.append(np.zeros((0, cols.value), np.uint32))
                else:   # zero-copy view of the library's pinned host rows
                    out.append(np.asarray(_HostRows(ctypes.c_void_p(res[i]), rows.value, cols.value, ptr.value,
                                                    self)))
                continue
            holder = _DeviceRows(ctypes.c_void_p(res[i]), rows.value, cols.value, ptr.value, self)
            if rows.value == 0:
                del holder
                out.append(torch.empty((0, cols.value), dtype=torch.uint32, device=f"cuda:{self.device}"))
            else:
                out.append(torch.as_tensor(holder, device=f"cuda:{self.device}"))
        _check(rc)
        return out

    def match_batch_raw(self, graph: Graph, queries, opts: Optional[MatchOpts] = None) -> "BatchResult":
        """Like match_batch but returns a BatchResult (row counts + lazily wrapped tensors)."""
        qas, arr, _qb = self._batch_desc(queries)
        n = len(qas)
        res = (ctypes.c_void_p * max(n, 1))()
        o = opts if opts is not None else default_opts()
        o = _with_device(o, True)
        rc = lib.gps_match_batch(self._h, graph.handle, arr, n, ctypes.byref(o), res, None)
        br = BatchResult(self, res, n)
        _check(rc)
        return br

    def match_batch_host(self, graph: Graph, queries, out, opts: Optional[MatchOpts] = None):
        """All embeddings copied by the library into ONE host buffer `out` (numpy uint32 or a
        pinned torch tensor).  Returns (offsets, rows) numpy arrays (word offsets into out)."""
        qas, arr, _qb = self._batch_desc(queries)
        n = len(qas)
        offs = np.zeros(max(n, 1), np.uint64)
        rows = np.zeros(max(n, 1), np.uint64)
        ptr, cap = (out.data_ptr(), out.numel()) if hasattr(out, "data_ptr") else (out.ctypes.data, out.size)
        _check(lib.gps_match_batch_host(self._h, graph.handle, arr, n,
                                        ctypes.byref(opts) if opts is not None else None, ctypes.c_void_p(ptr),
                                        cap, ctypes.c_void_p(offs.ctypes.data), ctypes.c_void_p(rows.ctypes.data),
                                        None))
        return offs[:n], rows[:n]

    def count_batch(self, graph: Graph, queries, opts: Optional[MatchOpts] = None, statuses: bool = False):
        """Counts of every query (numpy u64).  statuses=True: return (counts, per-query
        statuses) instead of raising when some queries fail."""
        qas, arr, _qb = self._batch_desc(queries)
        n = len(qas)
        counts = np.zeros(max(n, 1), np.uint64)
        st = np.zeros(max(n, 1), np.int32)
        rc = lib.gps_count_batch(self._h, graph.handle, arr, n, ctypes.byref(opts) if opts is not None else None,
                                 ctypes.c_void_p(counts.ctypes.data), ctypes.c_void_p(st.ctypes.data))
        if statuses:
            return counts[:n], st[:n]
        _check(rc)
        return counts[:n]

    def count(self, graph: Graph, q, opts: Optional[MatchOpts] = None) -> int:
        qa = _QueryArrays(q)
        c = ctypes.c_uint64()
        _check(lib.gps_count(self._h, graph.handle, ctypes.byref(qa.desc),
                             ctypes.byref(opts) if opts is not None else None, ctypes.byref(c)))
        return int(c.value)

    # ---- introspection ----
    def plan(self, graph: Graph, q, opts: Optional[MatchOpts] = None):
        qa = _QueryArrays(q)
        order = np.zeros(32, np.int32)
        n = ctypes.c_uint32()
        rank = np.zeros(64, np.uint64)
        _check(lib.gps_debug_plan(self._h, graph.handle, ctypes.byref(qa.desc),
                                  ctypes.byref(opts) if opts is not None else None,
                                  ctypes.c_void_p(order.ctypes.data), ctypes.byref(n),
                                  ctypes.c_void_p(rank.ctypes.data)))
        return order[: n.value].tolist(), [(int(rank[2 * u]), int(rank[2 * u + 1])) for u in range(qa.k)]

    def candidates(self, graph: Graph, q, stage: int, opts: Optional[MatchOpts] = None) -> np.ndarray:
        """Candidate bitmaps after stage 0/1/2 as a (k, n) bool array."""
        qa = _QueryArrays(q)
        nw = (graph.n + 31) // 32
        buf = np.zeros((qa.k, nw), np.uint32)
        _check(lib.gps_debug_candidates(self._h, graph.handle, ctypes.byref(qa.desc),
                                        ctypes.byref(opts) if opts is not None else None, int(stage),
                                        ctypes.c_void_p(buf.ctypes.data)))
        bits = np.unpackbits(buf.view(np.uint8).reshape(qa.k, -1), axis=1, bitorder="little")
        return bits[:, : graph.n].astype(bool)

    def stats(self) -> dict:
        s = Stats()
        _check(lib.gps_get_stats(self._h, ctypes.byref(s)))
        return {"queries": s.queries, "embeddings": s.embeddings, "launches": s.launches,
                "host_syncs": s.host_syncs, "join_rows_max": s.join_rows_max,
                "join_rows_total": s.join_rows_total,
                "kernels": {name: {"launches": s.k_launches[i], "bytes": s.k_bytes[i], "ms": s.k_ms[i],
                                   "timed": s.k_timed[i]} for i, name in enumerate(KERNEL_CLASSES)}}

    def reset_stats(self):
        _check(lib.gps_reset_stats(self._h))

    def set_profiling(self, classes):
        mask = 0
        for c in classes:
            mask |= 1 << (K[c] if isinstance(c, str) else int(c))
        _check(lib.gps_set_profiling(self._h, mask))
