"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs 1-5).

This module holds NO arithmetic of the PiPNN method: it only draws data and queries and lists the build
hyper-parameters of each config. Both the CPU oracle (tests) and the CUDA path (tests, bench.py) take
their inputs from here, which is the only thing the two sides share.

The paper's datasets (BigANN, DEEP, Text2Image, ... PAPER.md:587-606, 1044) are not in this container;
these generators stand in for them by shape, element type, metric and rough value range (DESIGN.md
"Input recipe"). Seeds: data 0, queries 1, build 0x5EED (reading R31).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

BUILD_SEED = 0x5EED


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    dtype: str  # "u8" | "f32"
    metric: str  # "l2" | "mips"
    n_centres: int
    c_max: int
    c_min: int = 100
    fanout: tuple = (2,)
    replicas: int = 1
    k: int = 8
    m: int = 12
    l_max: int = 128
    R: int = 64
    alpha_num: int = 6
    alpha_den: int = 5
    leader_cap: int = 1000
    final_prune: int = 1
    n_queries: int = 1000
    seed: int = BUILD_SEED
    unit_norm: bool = False  # DEEP-shaped: every vector L2-normalised

    @property
    def p_samp(self) -> tuple:
        """P_samp = 2/C_max as an exact rational (reading R10)."""
        return (2, self.c_max)

    def params(self) -> dict:
        num, den = self.p_samp
        return dict(c_max=self.c_max, c_min=self.c_min, p_num=num, p_den=den, leader_cap=self.leader_cap,
                    fanout=tuple(self.fanout), replicas=self.replicas, k=self.k, m=self.m, l_max=self.l_max,
                    R=self.R, alpha_num=self.alpha_num, alpha_den=self.alpha_den, final_prune=self.final_prune,
                    seed=self.seed)

    def scaled(self, n: int, n_centres: Optional[int] = None, n_queries: Optional[int] = None, **kw) -> "Config":
        """Same generator and parameters at a smaller n (parity-test sizes)."""
        nc = n_centres if n_centres is not None else max(1, int(round(self.n_centres * n / self.n)))
        return dataclasses.replace(self, name=f"{self.name}@{n}", n=n, n_centres=nc,
                                   n_queries=n_queries if n_queries is not None else self.n_queries, **kw)


# BASELINE.json configs (index 0..4 = C1..C5)
C1 = Config("C1", n=10_000, d=128, dtype="f32", metric="l2", n_centres=100, c_max=1024, n_queries=1000)
C2 = Config("C2", n=1_000_000, d=128, dtype="u8", metric="l2", n_centres=10_000, c_max=1024, n_queries=10_000)
C3 = Config("C3", n=1_000_000, d=96, dtype="f32", metric="l2", n_centres=10_000, c_max=1024, n_queries=10_000,
            unit_norm=True)
C4 = Config("C4", n=1_000_000, d=200, dtype="f32", metric="mips", n_centres=5_000, c_max=1024, fanout=(3,), k=10,
            l_max=160, n_queries=10_000)
C5 = Config("C5", n=50_000_000, d=128, dtype="u8", metric="l2", n_centres=100_000, c_max=2048, l_max=96, R=32,
            n_queries=10_000)
# SURVEY §8(f) NEXT-3, the paper's overlap knobs on the C2 workload: a
# two-level fanout [10, 3] and two replicas (bench variants, not BASELINE configs)
C2_F103 = dataclasses.replace(C2, name="C2-f10x3", fanout=(10, 3))
C2_R2 = dataclasses.replace(C2, name="C2-rep2", replicas=2)
CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5, "C2-f10x3": C2_F103, "C2-rep2": C2_R2}


def _mixture_f32(rng: np.random.Generator, n: int, d: int, centres: np.ndarray, sigma: float) -> np.ndarray:
    # point i belongs to cluster i mod #centres (clusters as even as possible)
    idx = np.arange(n) % centres.shape[0]
    x = centres[idx].astype(np.float32)
    x += (sigma * rng.standard_normal((n, d), dtype=np.float32))
    return x


def gen_points(cfg: Config, seed: int = 0) -> np.ndarray:
    """Base vectors of a config, [n, d] uint8 or float32, C-contiguous."""
    rng = np.random.default_rng(seed)
    n, d = cfg.n, cfg.d
    if cfg.dtype == "u8":
        # BIGANN-shaped: centres ~ U[0,255]^d, x = clip(round(c + 20 N(0,I)), 0, 255). The noise of each block
        # of 2^18 rows comes from its own stream (SeedSequence([seed, block])), so blocks are drawn in parallel
        # threads (50M x 128 for C5 in seconds) and any prefix of rows is independent of n.
        centres = rng.uniform(0.0, 255.0, size=(cfg.n_centres, d)).astype(np.float32)
        out = np.empty((n, d), dtype=np.uint8)
        step = 1 << 18

        def block(s):
            e = min(n, s + step)
            brng = np.random.default_rng(np.random.SeedSequence([seed, s // step]))
            idx = np.arange(s, e) % cfg.n_centres
            x = centres[idx]
            x += 20.0 * brng.standard_normal((e - s, d), dtype=np.float32)
            np.rint(x, out=x)
            np.clip(x, 0, 255, out=x)
            out[s:e] = x.astype(np.uint8)

        starts = list(range(0, n, step))
        if len(starts) > 1:
            import concurrent.futures as cf
            import os

            with cf.ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4)) as ex:
                list(ex.map(block, starts))
        else:
            block(0)
        return out
    centres = rng.standard_normal((cfg.n_centres, d), dtype=np.float32)
    if cfg.metric == "mips":
        # Text2Image-shaped: direction = normalise(c + 0.3 N), norm ~ LogNormal(0, 0.25)
        x = _mixture_f32(rng, n, d, centres, 0.3)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        x *= rng.lognormal(0.0, 0.25, size=(n, 1)).astype(np.float32)
        return np.ascontiguousarray(x, dtype=np.float32)
    x = _mixture_f32(rng, n, d, centres, 0.3)
    if cfg.unit_norm:
        x /= np.linalg.norm(x, axis=1, keepdims=True)  # DEEP-shaped: unit norm
    return np.ascontiguousarray(x, dtype=np.float32)


def gen_queries(cfg: Config, seed: int = 1, n_queries: Optional[int] = None) -> np.ndarray:
    """Held-out queries. Same mixture (new draws); C4: centres shifted by 0.5 N(0,I), normalised (OOD)."""
    nq = cfg.n_queries if n_queries is None else n_queries
    data_rng = np.random.default_rng(0)
    rng = np.random.default_rng(seed)
    d = cfg.d
    if cfg.dtype == "u8":
        centres = data_rng.uniform(0.0, 255.0, size=(cfg.n_centres, d)).astype(np.float32)
        idx = rng.integers(0, cfg.n_centres, size=nq)
        x = centres[idx] + 20.0 * rng.standard_normal((nq, d), dtype=np.float32)
        return np.clip(np.rint(x), 0, 255).astype(np.uint8)
    centres = data_rng.standard_normal((cfg.n_centres, d), dtype=np.float32)
    idx = rng.integers(0, cfg.n_centres, size=nq)
    if cfg.metric == "mips":
        c = centres[idx] + 0.5 * rng.standard_normal((nq, d), dtype=np.float32)
        x = c + 0.3 * rng.standard_normal((nq, d), dtype=np.float32)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        return np.ascontiguousarray(x, dtype=np.float32)
    x = centres[idx] + 0.3 * rng.standard_normal((nq, d), dtype=np.float32)
    if cfg.unit_norm:
        x /= np.linalg.norm(x, axis=1, keepdims=True)
    return np.ascontiguousarray(x, dtype=np.float32)


def gen_uniform(n: int, d: int, dtype: str, seed: int = 0) -> np.ndarray:
    """Unstructured inputs for edge-case tests."""
    rng = np.random.default_rng(seed)
    if dtype == "u8":
        return rng.integers(0, 256, size=(n, d), dtype=np.uint8)
    return rng.standard_normal((n, d), dtype=np.float32)
