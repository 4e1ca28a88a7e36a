"""CPU ORACLE for the PiPNN build hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may import this
package. It is a plain, slow, obviously-correct implementation of what the paper computes
(oracle/pipnn_oracle.cpp, each function citing PAPER.md/SPEC.md), independent of the CUDA path: the two
share no code; only `synth` (seeded input generators) serves both.

Parity pins: every entry point here is pinned by tests/test_oracle_*.py to values the paper/SPEC fix,
closed forms, brute force or invariants. The exact float graph on the
synthetic configs is "parity unpinned" in absolute terms (no paper number exists for it); only
oracle-relative parity and invariants apply there.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "pipnn_oracle.cpp")


def build_so(force: bool = False) -> str:
    """Compile the oracle (g++ -O2 -fopenmp). Building the checker is not using it."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c++17", "-o", _SO, _SRC])
    return _SO


class Points(C.Structure):
    _fields_ = [("data", C.c_void_p), ("n", C.c_int64), ("d", C.c_int32), ("dtype", C.c_int32),
                ("metric", C.c_int32), ("mode", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("c_max", C.c_int32), ("c_min", C.c_int32), ("p_num", C.c_int32), ("p_den", C.c_int32),
                ("leader_cap", C.c_int32), ("fanout", C.c_int32 * 4), ("n_fanout", C.c_int32),
                ("replicas", C.c_int32), ("k", C.c_int32), ("m", C.c_int32), ("l_max", C.c_int32),
                ("R", C.c_int32), ("alpha_num", C.c_int32), ("alpha_den", C.c_int32), ("final_prune", C.c_int32),
                ("seed", C.c_uint64)]


class Result(C.Structure):
    _fields_ = [("n_leaves", C.c_int64), ("n_instances", C.c_int64), ("leaf_off", C.POINTER(C.c_int64)),
                ("leaf_ids", C.POINTER(C.c_uint32)), ("k", C.c_int32), ("nbr", C.POINTER(C.c_uint32)),
                ("dist", C.POINTER(C.c_double)), ("l_max", C.c_int32), ("slots", C.POINTER(C.c_uint64)),
                ("count", C.POINTER(C.c_uint32)), ("n_streamed", C.c_int64), ("row_ptr", C.POINTER(C.c_int64)),
                ("col_idx", C.POINTER(C.c_uint32)), ("depth", C.c_int32), ("check_failed", C.c_int32),
                ("t_partition", C.c_double), ("t_leaf", C.c_double), ("t_hashprune", C.c_double),
                ("t_final", C.c_double), ("t_total", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build_so())
        L = _lib
        P = C.POINTER
        L.or_num_threads.restype = C.c_int
        L.or_set_threads.argtypes = [C.c_int]
        L.or_hyperplanes.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_void_p]
        L.or_sketch.argtypes = [P(Points), C.c_void_p, C.c_int32, C.c_void_p]
        L.or_residual_hash.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        L.or_residual_hash.restype = C.c_int32
        L.or_dist.argtypes = [P(Points), C.c_int64, C.c_int64]
        L.or_dist.restype = C.c_double
        L.or_dist_okey.argtypes = [C.c_double]
        L.or_dist_okey.restype = C.c_uint16
        L.or_mix.argtypes = [C.c_uint64, C.c_uint64]
        L.or_mix.restype = C.c_uint64
        L.or_merge_plan.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
        L.or_merge_plan.restype = C.c_int
        L.or_partition.argtypes = [P(Points), P(Params)]
        L.or_partition.restype = P(Result)
        L.or_build.argtypes = [P(Points), P(Params)]
        L.or_build.restype = P(Result)
        L.or_free.argtypes = [P(Result)]
        L.or_leaf_pick.argtypes = [P(Points), C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        L.or_hashprune.argtypes = [C.c_int64, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_int64, C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p]
        L.or_hashprune_list.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_void_p, C.c_void_p]
        L.or_hashprune_list.restype = C.c_int32
        L.or_final_prune.argtypes = [P(Points), C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_void_p, C.c_void_p]
        L.or_robust_prune.argtypes = [P(Points), C.c_uint32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_void_p]
        L.or_robust_prune.restype = C.c_int32
        L.or_brute_knn.argtypes = [P(Points), C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        L.or_entry_point.argtypes = [P(Points)]
        L.or_entry_point.restype = C.c_int64
        L.or_beam_search.argtypes = [P(Points), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32,
                                     C.c_int32, C.c_void_p, P(C.c_int64)]
    return _lib


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class Dataset:
    """Points + measure + float mode ('bf16' = GPU semantics, 'exact' = paper-faithful fp64 on fp32)."""

    def __init__(self, X: np.ndarray, metric: str = "l2", mode: str = "bf16"):
        X = np.ascontiguousarray(X)
        if X.dtype not in (np.uint8, np.float32):
            raise TypeError("dtype must be uint8 or float32")
        if X.dtype == np.uint8 and metric == "mips":
            raise ValueError("uint8 + MIPS is not supported (S:27)")
        self.X = X
        self.metric = metric
        self.mode = mode
        self.s = Points(X.ctypes.data, X.shape[0], X.shape[1], 0 if X.dtype == np.uint8 else 1,
                        1 if metric == "mips" else 0, 1 if mode == "bf16" else 0)

    @property
    def n(self):
        return self.X.shape[0]

    @property
    def d(self):
        return self.X.shape[1]


def make_params(p: dict) -> Params:
    P = Params()
    for key in ("c_max", "c_min", "p_num", "p_den", "leader_cap", "replicas", "k", "m", "l_max", "R", "alpha_num",
                "alpha_den", "final_prune"):
        setattr(P, key, int(p[key]))
    fo = list(p["fanout"])
    assert 1 <= len(fo) <= 4
    for i, f in enumerate(fo):
        P.fanout[i] = int(f)
    P.n_fanout = len(fo)
    P.seed = int(p["seed"])
    return P


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def num_threads() -> int:
    return lib().or_num_threads()


def set_threads(t: int):
    lib().or_set_threads(t)


def hyperplanes(m: int, d: int, seed: int) -> np.ndarray:
    H = np.zeros((m, d), dtype=np.int8)
    lib().or_hyperplanes(m, d, seed, _ptr(H))
    return H


def sketch(ds: Dataset, H: np.ndarray) -> np.ndarray:
    H = np.ascontiguousarray(H, dtype=np.int8)
    m = H.shape[0]
    out = np.zeros((ds.n, m), dtype=np.int32 if ds.X.dtype == np.uint8 else np.float32)
    lib().or_sketch(C.byref(ds.s), _ptr(H), m, _ptr(out))
    return out


def dist(ds: Dataset, a: int, b: int) -> float:
    return lib().or_dist(C.byref(ds.s), a, b)


def dist_okey(D: float) -> int:
    return lib().or_dist_okey(D)


def mix(a: int, b: int) -> int:
    return lib().or_mix(a, b)


def merge_plan(sizes, keys, ids, c_min: int, c_max: int):
    """Merge rule of small sibling groups (reading R15): output-group index of each input group."""
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    out = np.zeros(len(sizes), dtype=np.int32)
    ng = lib().or_merge_plan(_ptr(sizes), _ptr(keys), _ptr(ids), len(sizes), c_min, c_max, _ptr(out))
    return out, ng


def residual_hash(su: np.ndarray, sv: np.ndarray) -> int:
    su = np.ascontiguousarray(su, dtype=np.float64)
    sv = np.ascontiguousarray(sv, dtype=np.float64)
    return lib().or_residual_hash(_ptr(su), _ptr(sv), su.shape[0])


def partition(ds: Dataset, params: dict):
    """Alg. 5 -> (leaf_off int64[nl+1], leaf_ids uint32[I], depth)."""
    P = make_params(params)
    r = lib().or_partition(C.byref(ds.s), C.byref(P))
    try:
        res = r.contents
        off = _arr(res.leaf_off, res.n_leaves + 1, np.int64)
        ids = _arr(res.leaf_ids, res.n_instances, np.uint32)
        return off, ids, res.depth
    finally:
        lib().or_free(r)


def leaf_pick(ds: Dataset, leaf_off: np.ndarray, leaf_ids: np.ndarray, k: int):
    """Bidirected-k-NN candidate lists: (nbr uint32[I,k], dist float64[I,k]) ascending by (D, id)."""
    leaf_off = np.ascontiguousarray(leaf_off, dtype=np.int64)
    leaf_ids = np.ascontiguousarray(leaf_ids, dtype=np.uint32)
    I = int(leaf_off[-1])
    nbr = np.zeros((I, k), dtype=np.uint32)
    dd = np.zeros((I, k), dtype=np.float64)
    lib().or_leaf_pick(C.byref(ds.s), _ptr(leaf_off), _ptr(leaf_ids), len(leaf_off) - 1, k, _ptr(nbr), _ptr(dd))
    return nbr, dd


def bidirected_edges(leaf_ids: np.ndarray, nbr: np.ndarray, dist_: np.ndarray):
    """(owner, cand, dist) of every directed edge a candidate list implies."""
    I, k = nbr.shape
    src = np.repeat(leaf_ids.astype(np.uint32), k)
    dst = nbr.reshape(-1)
    dd = dist_.reshape(-1)
    ok = dst != 0xFFFFFFFF
    src, dst, dd = src[ok], dst[ok], dd[ok]
    owner = np.concatenate([src, dst])
    cand = np.concatenate([dst, src])
    return owner.astype(np.uint32), cand.astype(np.uint32), np.concatenate([dd, dd]).astype(np.float64)


def hashprune(n: int, S: np.ndarray, l_max: int, owner, cand, dist_, perm_seed: int = 1, init=None):
    """Alg. 3 per owner (streaming over a seeded shuffle, asserted equal to the characterization).
    Returns (slots uint64[n, l_max] sorted by hash, UINT64_MAX padded; count uint32[n]; ok)."""
    S = np.ascontiguousarray(S)
    is_int = 1 if S.dtype == np.int32 else 0
    m = S.shape[1]
    if init is None:
        slots = np.full((n, l_max), np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
        count = np.zeros(n, dtype=np.uint32)
    else:
        slots, count = init[0].copy(), init[1].copy()
    owner = np.ascontiguousarray(owner, dtype=np.uint32)
    cand = np.ascontiguousarray(cand, dtype=np.uint32)
    dist_ = np.ascontiguousarray(dist_, dtype=np.float64)
    rc = lib().or_hashprune(n, _ptr(S), is_int, m, l_max, _ptr(owner), _ptr(cand), _ptr(dist_), len(owner), perm_seed,
                            0 if init is None else 1, _ptr(slots), _ptr(count))
    return slots, count, rc == 0


def hashprune_list(hashes, dists, ids, l_max: int, mode: str = "stream"):
    hashes = np.ascontiguousarray(hashes, dtype=np.uint32)
    dists = np.ascontiguousarray(dists, dtype=np.float64)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    out_ids = np.zeros(max(1, len(ids)), dtype=np.uint32)
    out_h = np.zeros(max(1, len(ids)), dtype=np.uint32)
    k = lib().or_hashprune_list(_ptr(hashes), _ptr(dists), _ptr(ids), len(ids), l_max, 0 if mode == "stream" else 1,
                                _ptr(out_ids), _ptr(out_h))
    return out_ids[:k].copy(), out_h[:k].copy()


def final_prune(ds: Dataset, slots, count, R: int, alpha=(6, 5), final: int = 1):
    """Final RobustPrune per point (lazy, asserted equal to eager) -> CSR (row_ptr int64, col_idx uint32, ok)."""
    slots = np.ascontiguousarray(slots, dtype=np.uint64)
    count = np.ascontiguousarray(count, dtype=np.uint32)
    n, l_max = slots.shape
    rp = np.zeros(n + 1, dtype=np.int64)
    ci = np.zeros(max(1, n * R), dtype=np.uint32)
    rc = lib().or_final_prune(C.byref(ds.s), _ptr(slots), _ptr(count), l_max, R, alpha[0], alpha[1], final, _ptr(rp),
                              _ptr(ci))
    return rp, ci[: rp[-1]].copy(), rc == 0


def robust_prune(ds: Dataset, x: int, cands, R: int, alpha=(6, 5), lazy: bool = True):
    cands = np.ascontiguousarray(cands, dtype=np.uint32)
    out = np.zeros(max(1, len(cands)), dtype=np.uint32)
    k = lib().or_robust_prune(C.byref(ds.s), x, _ptr(cands), len(cands), R, alpha[0], alpha[1], 1 if lazy else 0,
                              _ptr(out))
    return out[:k].copy()


class BuildResult:
    pass


def build(ds: Dataset, params: dict) -> BuildResult:
    """Alg. 4 end to end; returns every intermediate artefact plus stage timings (seconds)."""
    P = make_params(params)
    r = lib().or_build(C.byref(ds.s), C.byref(P))
    try:
        res = r.contents
        out = BuildResult()
        out.leaf_off = _arr(res.leaf_off, res.n_leaves + 1, np.int64)
        out.leaf_ids = _arr(res.leaf_ids, res.n_instances, np.uint32)
        I, k = res.n_instances, res.k
        out.nbr = _arr(res.nbr, I * k, np.uint32).reshape(I, k)
        out.dist = _arr(res.dist, I * k, np.float64).reshape(I, k)
        n, lm = ds.n, res.l_max
        out.slots = _arr(res.slots, n * lm, np.uint64).reshape(n, lm)
        out.count = _arr(res.count, n, np.uint32)
        out.n_streamed = res.n_streamed
        out.row_ptr = _arr(res.row_ptr, n + 1, np.int64)
        out.col_idx = _arr(res.col_idx, int(out.row_ptr[-1]), np.uint32)
        out.depth = res.depth
        out.check_failed = res.check_failed
        out.times = dict(partition=res.t_partition, leaf=res.t_leaf, hashprune=res.t_hashprune, final=res.t_final,
                         total=res.t_total)
        return out
    finally:
        lib().or_free(r)


# ------------------------------------------------------------------ evaluation harness (not the method)
def brute_knn(ds: Dataset, Q: np.ndarray, k: int):
    Q = np.ascontiguousarray(Q, dtype=ds.X.dtype)
    ids = np.zeros((Q.shape[0], k), dtype=np.uint32)
    dd = np.zeros((Q.shape[0], k), dtype=np.float64)
    lib().or_brute_knn(C.byref(ds.s), _ptr(Q), Q.shape[0], k, _ptr(ids), _ptr(dd))
    return ids, dd


def entry_point(ds: Dataset) -> int:
    return lib().or_entry_point(C.byref(ds.s))


def beam_search(ds: Dataset, row_ptr, col_idx, Q: np.ndarray, entry: int, L: int, k: int = 10):
    Q = np.ascontiguousarray(Q, dtype=ds.X.dtype)
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.uint32)
    if col_idx.size == 0:
        col_idx = np.zeros(1, dtype=np.uint32)
    ids = np.zeros((Q.shape[0], k), dtype=np.uint32)
    cmps = C.c_int64(0)
    lib().or_beam_search(C.byref(ds.s), _ptr(row_ptr), _ptr(col_idx), _ptr(Q), Q.shape[0], entry, L, k, _ptr(ids),
                         C.byref(cmps))
    return ids, cmps.value


def recall_at(results: np.ndarray, truth: np.ndarray, k: int = 10, kp: int = 10) -> np.ndarray:
    """Def. 2: per-query |top-k truth ∩ first-k' results| / k."""
    out = np.zeros(results.shape[0])
    for i in range(results.shape[0]):
        out[i] = len(set(truth[i, :k].tolist()) & set(results[i, :kp].tolist())) / k
    return out
