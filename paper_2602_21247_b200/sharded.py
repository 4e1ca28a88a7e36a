"""Multi-GPU sharded PiPNN build: one process per GPU over torch.distributed (NCCL
between GPUs; gloo works for the host logic on CPU). Every compute step runs in libpipnn's kernels through the C ABI;
this module only plans the shards and moves data with collectives.

  1. X is replicated on every rank (§8(e): the final prune needs candidate rows; 1B uint8 points fit per GPU).
  2. Rank 0 runs the partition (Alg. 5) and broadcasts the LeafSet (one broadcast of the CSR).
  3. Leaves are dealt to ranks as contiguous ranges balanced by the leaf distance work sum |b|^2; each rank
     runs the leaf pick on its range.
  4. Owners are sharded by contiguous id ranges. Each rank turns its candidate lists into the bidirected edges
     (p -> q and q -> p with the same D, R18) and routes every edge to its owner's rank with
     one all_to_all — the path's only exchange step.
  5. Each rank merges its owners' reservoirs (Alg. 3 via hashprune_insert: its result is history independent,
     P:306-308 / P:1125-1129, so the order in which edges arrive does not matter) and final-prunes them
     (P:568-570). Its CSR rows are the rows of its id range; the shards concatenate into the whole graph.

Because the leaves are the same as a single-GPU build's and Alg. 3's result does not depend on the edge order, the
sharded graph is identical to pipnn_build's (bit for bit on uint8 data; tests/test_gpu_sharded.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import torch

from . import (BuildParams, hashprune_insert, new_reservoirs, pipnn_final_prune, pipnn_leaf_pick, pipnn_partition,
               pipnn_sketch)


# ------------------------------------------------------------------ shard plans (host logic, device-agnostic)
def owner_bounds(n: int, world: int) -> List[int]:
    """Contiguous owner id ranges: rank r owns [b[r], b[r+1])."""
    chunk = -(-n // world)
    return [min(n, r * chunk) for r in range(world + 1)]


def leaf_ranges(leaf_off: torch.Tensor, world: int) -> List[int]:
    """Leaf index boundaries b[0..world] splitting the leaves into contiguous ranges of about equal sum |b|^2."""
    s = (leaf_off[1:] - leaf_off[:-1]).to(torch.float64)
    cost = torch.cumsum(s * s, 0)
    nl = cost.numel()
    if nl == 0:
        return [0] * (world + 1)
    total = float(cost[-1])
    targets = torch.tensor([total * r / world for r in range(1, world)], dtype=torch.float64, device=cost.device)
    cuts = torch.searchsorted(cost, targets, right=True).tolist() if world > 1 else []
    return [0] + [int(min(nl, c)) for c in cuts] + [nl]


def bidirected_edges(leaf_ids: torch.Tensor, nbr: torch.Tensor, dist: torch.Tensor):
    """(owner, cand, D) of every directed edge the candidate lists imply: p -> q and q -> p with the same D."""
    k = nbr.shape[1]
    p = leaf_ids.view(-1, 1).expand(-1, k).reshape(-1)
    q = nbr.reshape(-1)
    d = dist.reshape(-1)
    ok = q != -1  # UINT32_MAX marks a missing pick
    p, q, d = p[ok], q[ok], d[ok]
    return torch.cat([p, q]), torch.cat([q, p]), torch.cat([d, d])


def route_edges(owner: torch.Tensor, cand: torch.Tensor, dist: torch.Tensor, bounds: Sequence[int],
                exchange: Callable[[torch.Tensor, List[int]], torch.Tensor]):
    """Send every edge to the rank owning its owner id; `exchange(rows, send_counts)` is an all_to_all of the packed
    [E, 3] int32 rows (owner, cand, D bits) and returns the rows this rank receives."""
    world = len(bounds) - 1
    b = torch.tensor(bounds[1:-1], dtype=owner.dtype, device=owner.device)
    dest = torch.bucketize(owner, b, right=True) if world > 1 else torch.zeros_like(owner)
    order = torch.argsort(dest, stable=True)
    counts = torch.bincount(dest, minlength=world).tolist()
    rows = torch.stack([owner, cand, dist.view(torch.int32)], 1)[order].contiguous()
    got = exchange(rows, counts)
    return got[:, 0].contiguous(), got[:, 1].contiguous(), got[:, 2].contiguous().view(torch.float32)


def nccl_exchange(group=None) -> Callable[[torch.Tensor, List[int]], torch.Tensor]:
    """all_to_all of packed edge rows over torch.distributed (counts first, then the rows)."""
    import torch.distributed as dist

    def ex(rows: torch.Tensor, counts: List[int]) -> torch.Tensor:
        world = dist.get_world_size(group)
        sc = torch.tensor(counts, dtype=torch.int64, device=rows.device)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=group)
        recv_counts = rc.tolist()
        out = torch.empty((sum(recv_counts), rows.shape[1]), dtype=rows.dtype, device=rows.device)
        dist.all_to_all_single(out, rows, recv_counts, counts, group=group)
        return out

    return ex


# ------------------------------------------------------------------ the sharded build
@dataclass
class ShardOut:
    base: int            # first owner id of this rank's rows
    row_ptr: torch.Tensor  # int64 [n_local + 1], rebased to 0
    col_idx: torch.Tensor  # int32 (uint32 ids) [row_ptr[-1]]
    stats: dict


def _broadcast_leafset(leaf_off, leaf_ids, device, group):
    import torch.distributed as dist

    sizes = torch.tensor([leaf_off.numel(), leaf_ids.numel()] if leaf_off is not None else [0, 0], dtype=torch.int64,
                         device=device)
    dist.broadcast(sizes, 0, group=group)
    if leaf_off is None:
        leaf_off = torch.empty(int(sizes[0]), dtype=torch.int64, device=device)
        leaf_ids = torch.empty(int(sizes[1]), dtype=torch.int32, device=device)
    dist.broadcast(leaf_off, 0, group=group)
    dist.broadcast(leaf_ids, 0, group=group)
    return leaf_off, leaf_ids


def shard_edges(X: torch.Tensor, params: BuildParams, leaf_off: torch.Tensor, leaf_ids: torch.Tensor, rank: int,
                world: int, metric: str = "l2"):
    """Step 3: the leaf pick on this rank's leaf range -> its bidirected edges (owner, cand, D)."""
    lr = leaf_ranges(leaf_off, world)
    b0, b1 = lr[rank], lr[rank + 1]
    i0, i1 = int(leaf_off[b0]), int(leaf_off[b1])
    if b1 == b0:
        e = torch.empty(0, dtype=torch.int32, device=X.device)
        return e, e, torch.empty(0, dtype=torch.float32, device=X.device), {"leaves": 0, "instances": 0}
    my_off = (leaf_off[b0:b1 + 1] - i0).contiguous()
    my_ids = leaf_ids[i0:i1]
    nbr, dist = pipnn_leaf_pick(X, my_off, my_ids, params.pick.k, metric, quant=params.pick.quant)
    owner, cand, d = bidirected_edges(my_ids, nbr, dist)
    return owner, cand, d, {"leaves": b1 - b0, "instances": i1 - i0}


def shard_finish(X: torch.Tensor, params: BuildParams, owner: torch.Tensor, cand: torch.Tensor, d: torch.Tensor,
                 rank: int, world: int, metric: str = "l2", S: Optional[torch.Tensor] = None) -> ShardOut:
    """Step 5: this rank's owners' reservoirs (Alg. 3) from the edges routed to it, the final prune, its CSR rows."""
    n = X.shape[0]
    if S is None:
        S = pipnn_sketch(X, params.hp.m, params.hp.seed, metric)
    slots, count = new_reservoirs(n, params.hp.l_max, X.device)
    if owner.numel():
        hashprune_insert(S, slots, count, owner, cand, d, m=params.hp.m)
    pr = params.prune
    rp, ci = pipnn_final_prune(X, slots, count, pr.R, (pr.alpha_num, pr.alpha_den), pr.final_prune, metric)
    bounds = owner_bounds(n, world)
    lo, hi = bounds[rank], bounds[rank + 1]
    r0, r1 = int(rp[lo]), int(rp[hi])
    return ShardOut(lo, (rp[lo:hi + 1] - r0).contiguous(), ci[r0:r1], {"edges_in": int(owner.numel())})


def shard_step(X: torch.Tensor, params: BuildParams, leaf_off: torch.Tensor, leaf_ids: torch.Tensor, rank: int,
               world: int, exchange, metric: str = "l2") -> ShardOut:
    """Steps 3-5 for rank `rank` of `world`, given the LeafSet (identical on every rank) and an edge exchange."""
    owner, cand, d, st = shard_edges(X, params, leaf_off, leaf_ids, rank, world, metric)
    owner, cand, d = route_edges(owner, cand, d, owner_bounds(X.shape[0], world), exchange)
    out = shard_finish(X, params, owner, cand, d, rank, world, metric)
    out.stats.update(st)
    return out


def virtual_sharded_build(X: torch.Tensor, params: BuildParams, world: int, metric: str = "l2") -> List[ShardOut]:
    """The same decomposition run rank after rank in one process (no collective): every rank's edges are formed,
    then each rank receives, in source-rank order, the edges of its owners (what the all_to_all delivers). Used to
    check on one GPU that the sharded plan reproduces pipnn_build."""
    off, ids = pipnn_partition(X, params.part, metric)
    bounds = owner_bounds(X.shape[0], world)
    sent = []
    for r in range(world):
        owner, cand, d, _ = shard_edges(X, params, off, ids, r, world, metric)
        sent.append((owner, cand, d))
    S = pipnn_sketch(X, params.hp.m, params.hp.seed, metric)
    out = []
    for r in range(world):
        lo, hi = bounds[r], bounds[r + 1]
        parts = [[], [], []]
        for owner, cand, d in sent:
            m = (owner >= lo) & (owner < hi)
            parts[0].append(owner[m])
            parts[1].append(cand[m])
            parts[2].append(d[m])
        out.append(shard_finish(X, params, torch.cat(parts[0]), torch.cat(parts[1]), torch.cat(parts[2]), r, world,
                                metric, S))
    return out


def sharded_build(X: torch.Tensor, params: BuildParams, metric: str = "l2", group=None) -> ShardOut:
    """The sharded build on this process's rank (torch.distributed initialised; X on this rank's GPU)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    off = ids = None
    if rank == 0:
        off, ids = pipnn_partition(X, params.part, metric)
    off, ids = _broadcast_leafset(off, ids, X.device, group)
    return shard_step(X, params, off, ids, rank, world, nccl_exchange(group), metric)


def concat_shards(shards: Sequence[ShardOut]):
    """The whole CSR from the shards of ranks 0..W-1 (in rank order)."""
    rps, cis, base = [], [], 0
    for sh in shards:
        rps.append(sh.row_ptr[(1 if rps else 0):] + base)
        cis.append(sh.col_idx)
        base += int(sh.row_ptr[-1])
    return torch.cat(rps), torch.cat(cis)
