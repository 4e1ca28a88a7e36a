"""paper_2602_21247_b200 — B200-native PiPNN build hot path (arxiv 2602.21247).

Thin ctypes binding over libpipnn.so (include/pipnn.h). Argument marshalling only: every step of the path
runs in the library's sm_100a kernels; torch provides device memory and streams. There is no CPU fallback:
importing this package without the built library raises ImportError.

Python names mirror the C ABI: pipnn_partition, pipnn_leaf_pick, pipnn_sketch, hashprune_insert,
pipnn_final_prune, pipnn_build, pipnn_workspace_size.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpipnn.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libpipnn.so not built ({LIB_PATH}); run `python paper_2602_21247_b200/_build.py` "
                      "(or __graft_entry__.build()) — there is no CPU fallback")

_lib = C.CDLL(LIB_PATH)

PIPNN_OK, PIPNN_EINVAL, PIPNN_ECAPACITY, PIPNN_EWORKSPACE, PIPNN_ECUDA, PIPNN_EUNSUPPORTED = range(6)
U8, F32 = 0, 1
L2, MIPS = 0, 1


class PipnnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"pipnn status {status}: {msg}")
        self.status = status


class Points(C.Structure):
    _fields_ = [("data", C.c_void_p), ("n", C.c_int64), ("d", C.c_int32), ("ld", C.c_int32), ("dtype", C.c_int32),
                ("metric", C.c_int32)]


class PartitionParams(C.Structure):
    _fields_ = [("c_max", C.c_int32), ("c_min", C.c_int32), ("p_samp_num", C.c_int32), ("p_samp_den", C.c_int32),
                ("leader_cap", C.c_int32), ("fanout", C.c_int32 * 4), ("n_fanout", C.c_int32),
                ("replicas", C.c_int32), ("seed", C.c_uint64)]


class PickParams(C.Structure):
    _fields_ = [("k", C.c_int32), ("quant", C.c_int32)]


class HashPruneParams(C.Structure):
    _fields_ = [("m", C.c_int32), ("l_max", C.c_int32), ("seed", C.c_uint64)]


class PruneParams(C.Structure):
    _fields_ = [("R", C.c_int32), ("alpha_num", C.c_int32), ("alpha_den", C.c_int32), ("final_prune", C.c_int32)]


class SearchParams(C.Structure):
    _fields_ = [("L", C.c_int32), ("k", C.c_int32), ("exclude_self", C.c_int32)]


class BuildBuffers(C.Structure):
    _fields_ = [("leaf_off", C.c_void_p), ("leaf_ids", C.c_void_p), ("cols", C.c_void_p), ("dist", C.c_void_p),
                ("sketch", C.c_void_p), ("slots", C.c_void_p), ("count", C.c_void_p)]


class BuildParams(C.Structure):
    _fields_ = [("part", PartitionParams), ("pick", PickParams), ("hp", HashPruneParams), ("prune", PruneParams)]


class Stats(C.Structure):
    _fields_ = [("n_leaves", C.c_int64), ("n_instances", C.c_int64), ("n_edges", C.c_int64), ("max_leaf", C.c_int64),
                ("leaf_pairs", C.c_int64), ("depth", C.c_int32), ("ms_prep", C.c_float),
                ("ms_partition", C.c_float), ("ms_leaf", C.c_float), ("ms_hashprune", C.c_float),
                ("ms_final", C.c_float), ("ms_total", C.c_float), ("ms_leaf_tiles", C.c_float)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_P = C.POINTER
_vp = C.c_void_p
_lib.pipnn_last_error.restype = C.c_char_p
_lib.pipnn_abi_version.restype = C.c_int32
_lib.pipnn_required_workspace.restype = C.c_size_t
_lib.pipnn_launch_count.restype = C.c_uint64
_lib.pipnn_workspace_size.argtypes = [_P(Points), _P(BuildParams), _P(C.c_size_t)]
_lib.pipnn_partition.argtypes = [_P(Points), _P(PartitionParams), _vp, C.c_size_t, _vp, C.c_int64, _vp, C.c_int64,
                                 _P(C.c_int64), _P(C.c_int64), _vp]
_lib.pipnn_leaf_pick.argtypes = [_P(Points), _vp, _vp, C.c_int64, C.c_int64, _P(PickParams), _vp, _vp, _vp,
                                 C.c_size_t, _vp]
_lib.pipnn_sketch.argtypes = [_P(Points), _P(HashPruneParams), _vp, _vp, C.c_size_t, _vp]
_lib.pipnn_device_error.argtypes = [_vp, _vp]
_lib.hashprune_insert.argtypes = [_P(HashPruneParams), C.c_int64, _vp, C.c_int32, _vp, _vp, _vp, _vp, _vp, C.c_int64,
                                  _vp, C.c_size_t, _vp]
_lib.pipnn_final_prune.argtypes = [_P(Points), _P(HashPruneParams), _vp, _vp, _P(PruneParams), _vp, _vp, _vp,
                                   C.c_size_t, _vp]
_lib.pipnn_build.argtypes = [_P(Points), _P(BuildParams), _vp, C.c_size_t, _vp, _vp, _P(C.c_int64), _P(Stats), _vp]
_lib.pipnn_search.argtypes = [_P(Points), _vp, _vp, _vp, C.c_int64, C.c_int64, C.c_uint32, _P(SearchParams), _vp, _vp,
                              _vp, _vp, C.c_size_t, _vp]
_lib.pipnn_debug_build_buffers.argtypes = [_P(Points), _P(BuildParams), _vp, C.c_size_t, _P(BuildBuffers)]
for _f in ("pipnn_debug_build_buffers", "pipnn_workspace_size", "pipnn_partition", "pipnn_leaf_pick", "pipnn_sketch", "pipnn_device_error",
           "hashprune_insert", "pipnn_final_prune", "pipnn_build", "pipnn_search"):
    getattr(_lib, _f).restype = C.c_int

EXPORTS = ("pipnn_last_error", "pipnn_abi_version", "pipnn_required_workspace", "pipnn_launch_count", "pipnn_workspace_size",
           "pipnn_partition", "pipnn_leaf_pick", "pipnn_sketch", "pipnn_device_error", "hashprune_insert",
           "pipnn_final_prune", "pipnn_build", "pipnn_search", "pipnn_debug_build_buffers")


def lib():
    return _lib


def pipnn_launch_count() -> int:
    return _lib.pipnn_launch_count()


def _check(rc: int):
    if rc != PIPNN_OK:
        raise PipnnError(rc, _lib.pipnn_last_error().decode())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def points(X: torch.Tensor, metric: str = "l2") -> Points:
    """Describe a device tensor [n, d] (uint8 or float32, row stride X.stride(0)) as pipnn_points."""
    if not X.is_cuda:
        raise ValueError("X must be a CUDA tensor")
    if X.dim() != 2 or X.stride(1) != 1:
        raise ValueError("X must be [n, d] with unit column stride")
    dt = {torch.uint8: U8, torch.float32: F32}.get(X.dtype)
    if dt is None:
        raise TypeError("X must be uint8 or float32")
    return Points(X.data_ptr(), X.shape[0], X.shape[1], X.stride(0), dt, MIPS if metric == "mips" else L2)


def partition_params(c_max=1024, c_min=100, p_samp=None, leader_cap=1000, fanout: Sequence[int] = (2,), replicas=1,
                     seed=0x5EED) -> PartitionParams:
    p = PartitionParams()
    p.c_max, p.c_min = c_max, c_min
    num, den = p_samp if p_samp is not None else (2, c_max)
    p.p_samp_num, p.p_samp_den = num, den
    p.leader_cap = leader_cap
    fo = list(fanout)
    for i, f in enumerate(fo):
        p.fanout[i] = f
    p.n_fanout = len(fo)
    p.replicas = replicas
    p.seed = seed
    return p


def build_params(c_max=1024, c_min=100, p_samp=None, leader_cap=1000, fanout=(2,), replicas=1, k=8, m=12, l_max=128,
                 R=64, alpha=(6, 5), final_prune=1, seed=0x5EED, quant=0) -> BuildParams:
    bp = BuildParams()
    bp.part = partition_params(c_max, c_min, p_samp, leader_cap, fanout, replicas, seed)
    bp.pick.k = k
    bp.pick.quant = quant
    bp.hp.m, bp.hp.l_max, bp.hp.seed = m, l_max, seed
    bp.prune.R, bp.prune.alpha_num, bp.prune.alpha_den, bp.prune.final_prune = R, alpha[0], alpha[1], final_prune
    return bp


def build_params_from(p: dict) -> BuildParams:
    """From a synth.Config.params() dict."""
    return build_params(c_max=p["c_max"], c_min=p["c_min"], p_samp=(p["p_num"], p["p_den"]),
                        leader_cap=p["leader_cap"], fanout=p["fanout"], replicas=p["replicas"], k=p["k"], m=p["m"],
                        l_max=p["l_max"], R=p["R"], alpha=(p["alpha_num"], p["alpha_den"]),
                        final_prune=p["final_prune"], seed=p["seed"], quant=p.get("quant", 0))


def _workspace(call, device) -> torch.Tensor:
    """Two-call size query: call(None, 0) -> PIPNN_EWORKSPACE, then allocate the reported size."""
    rc = call(C.c_void_p(0), 0)
    if rc == PIPNN_OK:
        return torch.empty(0, dtype=torch.uint8, device=device)
    if rc != PIPNN_EWORKSPACE:
        _check(rc)
    need = _lib.pipnn_required_workspace()
    return torch.empty(need, dtype=torch.uint8, device=device)


def pipnn_workspace_size(X: torch.Tensor, params: BuildParams, metric="l2") -> int:
    pts = points(X, metric)
    n = C.c_size_t(0)
    _check(_lib.pipnn_workspace_size(C.byref(pts), C.byref(params), C.byref(n)))
    return n.value


def pipnn_device_error(ws: torch.Tensor, stream=None):
    _check(_lib.pipnn_device_error(_ptr(ws), _stream(stream)))


def pipnn_partition(X: torch.Tensor, params: PartitionParams, metric="l2", stream=None):
    """Alg. 5 -> (leaf_off int64[n_leaves+1], leaf_ids int32[I] (uint32 ids), both on the device)."""
    pts = points(X, metric)
    prod = 1
    for i in range(params.n_fanout):
        prod *= params.fanout[i]
    cap = X.shape[0] * prod * params.replicas
    off = torch.empty(cap + 1, dtype=torch.int64, device=X.device)
    ids = torch.empty(cap, dtype=torch.int32, device=X.device)
    nl, ni = C.c_int64(0), C.c_int64(0)
    st = _stream(stream)

    def call(ws, nbytes):
        return _lib.pipnn_partition(C.byref(pts), C.byref(params), ws, nbytes, _ptr(off), cap + 1, _ptr(ids), cap,
                                    C.byref(nl), C.byref(ni), st)

    ws = _workspace(call, X.device)
    _check(call(_ptr(ws), ws.numel()))
    return off[: nl.value + 1], ids[: ni.value]


def pipnn_leaf_pick(X: torch.Tensor, leaf_off: torch.Tensor, leaf_ids: torch.Tensor, k: int, metric="l2",
                    stream=None, check=True, quant=0):
    """Leaf building -> (nbr int32[I, k] (uint32 ids, -1 = none), dist float32[I, k])."""
    pts = points(X, metric)
    nl = leaf_off.numel() - 1
    I = leaf_ids.numel()
    nbr = torch.empty((I, k), dtype=torch.int32, device=X.device)
    dist = torch.empty((I, k), dtype=torch.float32, device=X.device)
    pp = PickParams(k, quant)
    st = _stream(stream)

    def call(ws, nbytes):
        return _lib.pipnn_leaf_pick(C.byref(pts), _ptr(leaf_off), _ptr(leaf_ids), nl, I, C.byref(pp), _ptr(nbr),
                                    _ptr(dist), ws, nbytes, st)

    ws = _workspace(call, X.device)
    _check(call(_ptr(ws), ws.numel()))
    if check:
        pipnn_device_error(ws, stream)
    return nbr, dist


def pipnn_sketch(X: torch.Tensor, m=12, seed=0x5EED, metric="l2", stream=None):
    pts = points(X, metric)
    hp = HashPruneParams(m, 1, seed)
    S = torch.empty((X.shape[0], m), dtype=torch.int32 if X.dtype == torch.uint8 else torch.float32, device=X.device)
    st = _stream(stream)

    def call(ws, nbytes):
        return _lib.pipnn_sketch(C.byref(pts), C.byref(hp), _ptr(S), ws, nbytes, st)

    ws = _workspace(call, X.device)
    _check(call(_ptr(ws), ws.numel()))
    pipnn_device_error(ws, stream)
    return S


def new_reservoirs(n: int, l_max: int, device="cuda"):
    slots = torch.full((n, l_max), -1, dtype=torch.int64, device=device)  # all-ones bytes = UINT64_MAX
    count = torch.zeros(n, dtype=torch.int32, device=device)
    return slots, count


def hashprune_insert(S: torch.Tensor, slots: torch.Tensor, count: torch.Tensor, owner: torch.Tensor,
                     cand: torch.Tensor, dist: torch.Tensor, m=12, stream=None):
    """Alg. 3 over an edge batch (in place on slots/count)."""
    n, l_max = slots.shape
    hp = HashPruneParams(m, l_max, 0)
    E = owner.numel()
    st = _stream(stream)
    skd = U8 if S.dtype == torch.int32 else F32

    def call(ws, nbytes):
        return _lib.hashprune_insert(C.byref(hp), n, _ptr(S), skd, _ptr(slots), _ptr(count), _ptr(owner),
                                     _ptr(cand), _ptr(dist), E, ws, nbytes, st)

    ws = _workspace(call, slots.device)
    _check(call(_ptr(ws), ws.numel()))
    pipnn_device_error(ws, stream)
    return slots, count


def pipnn_final_prune(X: torch.Tensor, slots: torch.Tensor, count: torch.Tensor, R=64, alpha=(6, 5), final_prune=1,
                      metric="l2", stream=None):
    pts = points(X, metric)
    n, l_max = slots.shape
    hp = HashPruneParams(12, l_max, 0)
    pr = PruneParams(R, alpha[0], alpha[1], final_prune)
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=X.device)
    col_idx = torch.empty(max(1, n * R), dtype=torch.int32, device=X.device)
    st = _stream(stream)

    def call(ws, nbytes):
        return _lib.pipnn_final_prune(C.byref(pts), C.byref(hp), _ptr(slots), _ptr(count), C.byref(pr),
                                      _ptr(row_ptr), _ptr(col_idx), ws, nbytes, st)

    ws = _workspace(call, X.device)
    _check(call(_ptr(ws), ws.numel()))
    pipnn_device_error(ws, stream)
    return row_ptr, col_idx


def pipnn_search(X: torch.Tensor, row_ptr: torch.Tensor, col_idx: torch.Tensor, Q: torch.Tensor, entry: int,
                 L: int = 64, k: int = 10, metric="l2", stream=None, count_cmps: bool = False, exclude_self=False):
    """Batched beam search (Alg. 1) of the queries Q [nq, d] (X's dtype, on the device) on the graph (row_ptr,
    col_idx) from `entry` -> (ids int32 [nq, k] (uint32 ids, -1 past the beam), dist float32 [nq, k], n_cmps)."""
    pts = points(X, metric)
    if Q.dtype != X.dtype or Q.dim() != 2 or Q.stride(1) != 1 or not Q.is_cuda:
        raise ValueError("Q must be a CUDA [nq, d] tensor of X's dtype with unit column stride")
    nq = Q.shape[0]
    sp = SearchParams(L, k, 1 if exclude_self else 0)
    ids = torch.empty((nq, k), dtype=torch.int32, device=X.device)
    dist = torch.empty((nq, k), dtype=torch.float32, device=X.device)
    cmps = torch.zeros(1, dtype=torch.int64, device=X.device) if count_cmps else None
    st = _stream(stream)

    def call(ws, nbytes):
        return _lib.pipnn_search(C.byref(pts), _ptr(row_ptr), _ptr(col_idx), _ptr(Q), Q.stride(0), nq, int(entry),
                                 C.byref(sp), _ptr(ids), _ptr(dist), _ptr(cmps), ws, nbytes, st)

    ws = _workspace(call, X.device)
    _check(call(_ptr(ws), ws.numel()))
    pipnn_device_error(ws, stream)
    return ids, dist, (int(cmps.item()) if cmps is not None else None)


def knn_graph(X: torch.Tensor, row_ptr: torch.Tensor, col_idx: torch.Tensor, entry: int, k: int = 10, L: int = 64,
              metric="l2", stream=None):
    """The k-NN-graph task: every base point queried on its own index, itself left out ->
    (ids int32 [n, k], dist float32 [n, k])."""
    ids, dist, _ = pipnn_search(X, row_ptr, col_idx, X, entry, L, k, metric, stream, exclude_self=True)
    return ids, dist


@dataclass
class BuildOut:
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    n_edges: int
    stats: dict


class Builder:
    """Holds the workspace and output buffers of repeated pipnn_build calls on same-shaped inputs."""

    def __init__(self, X: torch.Tensor, params: BuildParams, metric="l2"):
        self.params = params
        self.metric = metric
        self.ws_bytes = pipnn_workspace_size(X, params, metric)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=X.device)
        n = X.shape[0]
        self.row_ptr = torch.empty(n + 1, dtype=torch.int64, device=X.device)
        self.col_idx = torch.empty(n * params.prune.R, dtype=torch.int32, device=X.device)

    def __call__(self, X: torch.Tensor, stream=None) -> BuildOut:
        pts = points(X, self.metric)
        ne = C.c_int64(0)
        stats = Stats()
        _check(_lib.pipnn_build(C.byref(pts), C.byref(self.params), _ptr(self.ws), self.ws_bytes, _ptr(self.row_ptr),
                                _ptr(self.col_idx), C.byref(ne), C.byref(stats), _stream(stream)))
        return BuildOut(self.row_ptr, self.col_idx[: ne.value], ne.value, stats.as_dict())


    def debug_buffers(self, X: torch.Tensor, stats: dict) -> dict:
        """The last build's intermediate artefacts (pipnn_debug_build_buffers) as tensor views of the workspace:
        leaf_off, leaf_ids, cols (int16 bits of u16 local columns, [I, k]), dist [I, k], sketch [n, m],
        slots (int64 bits of u64) [n, l_max], count [n]."""
        pts = points(X, self.metric)
        b = BuildBuffers()
        _check(_lib.pipnn_debug_build_buffers(C.byref(pts), C.byref(self.params), _ptr(self.ws), self.ws_bytes,
                                              C.byref(b)))
        base = self.ws.data_ptr()
        n, k = X.shape[0], self.params.pick.k
        nl, ni = stats["n_leaves"], stats["n_instances"]
        m, lm = self.params.hp.m, self.params.hp.l_max

        def view(ptr, count, dtype):
            esz = torch.empty(0, dtype=dtype).element_size()
            off = ptr - base
            return self.ws[off: off + count * esz].view(dtype)

        skd = torch.int32 if X.dtype == torch.uint8 else torch.float32
        return {"leaf_off": view(b.leaf_off, nl + 1, torch.int64), "leaf_ids": view(b.leaf_ids, ni, torch.int32),
                "cols": view(b.cols, ni * k, torch.int16).view(ni, k), "dist": view(b.dist, ni * k, torch.float32).view(ni, k),
                "sketch": view(b.sketch, n * m, skd).view(n, m), "slots": view(b.slots, n * lm, torch.int64).view(n, lm),
                "count": view(b.count, n, torch.int32)}


def pipnn_build(X: torch.Tensor, params: BuildParams, metric="l2", stream=None) -> BuildOut:
    """Alg. 4 end to end -> degree-bounded CSR graph (row_ptr int64[n+1], col_idx int32[E])."""
    return Builder(X, params, metric)(X, stream)
