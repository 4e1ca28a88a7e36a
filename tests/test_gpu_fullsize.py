"""Parity at BASELINE.json's full size (C2: 1,000,000 x 128 uint8, the configuration bench.py times), on what
the oracle can compute at that size: the whole partition (bit-exact leaf sets), and for a seeded sample of
points the full chain — the oracle's picks in every leaf holding the point, its HashPrune
reservoir (Alg. 3) and final RobustPrune — against the GPU build's CSR row (bit-exact);
plus properties of the whole graph that hold at any size."""
import time

import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def P():
    import paper_2602_21247_b200 as P

    return P


def canon(off, ids):
    return sorted(tuple(ids[off[i]:off[i + 1]].tolist()) for i in range(len(off) - 1))


def oracle_row(ds, X, S, off, ids, inst_leaf, u, p):
    """The oracle's CSR row of point u: candidates streamed to u from its leaves, reservoir, lazy prune."""
    k, l_max, R = p["k"], p["l_max"], p["R"]
    cand_ids, cand_d = [], []
    for b in inst_leaf[u]:
        lo, hi = off[b], off[b + 1]
        lid = ids[lo:hi]
        nbr, dd = O.leaf_pick(ds, np.array([0, hi - lo], dtype=np.int64), lid, k)
        me = int(np.nonzero(lid == u)[0][0])
        for t in range(k):  # forward u -> q
            if nbr[me, t] != 0xFFFFFFFF:
                cand_ids.append(int(nbr[me, t]))
                cand_d.append(float(dd[me, t]))
        rows, cols = np.nonzero(nbr == u)  # reverse p -> u (same D)
        for r_, c_ in zip(rows, cols):
            cand_ids.append(int(lid[r_]))
            cand_d.append(float(dd[r_, c_]))
    hashes = [O.residual_hash(S[u], S[v]) for v in cand_ids]
    res_ids, _ = O.hashprune_list(hashes, cand_d, cand_ids, l_max, mode="stream")
    return O.robust_prune(ds, u, res_ids, R, (p["alpha_num"], p["alpha_den"]), lazy=True)


def test_c2_full_size_partition_and_sampled_build():
    cfg = synth.C2
    X = synth.gen_points(cfg)
    p = cfg.params()
    ds = O.Dataset(X)
    t0 = time.time()
    off, ids, depth = O.partition(ds, p)
    t_part = time.time() - t0
    Xt = torch.from_numpy(X).cuda()
    pp = P().partition_params(c_max=p["c_max"], c_min=p["c_min"], p_samp=(p["p_num"], p["p_den"]),
                              fanout=p["fanout"], replicas=p["replicas"], seed=p["seed"])
    goff, gids = P().pipnn_partition(Xt, pp)
    goff, gids = goff.cpu().numpy(), gids.cpu().numpy().view(np.uint32)
    assert canon(goff, gids) == canon(off, ids)  # the whole partition, bit-exact

    out = P().pipnn_build(Xt, P().build_params_from(p), metric="l2")
    torch.cuda.synchronize()
    rp, ci = out.row_ptr.cpu().numpy(), out.col_idx.cpu().numpy().view(np.uint32)
    n = cfg.n
    # properties of the whole graph
    deg = np.diff(rp)
    assert rp[0] == 0 and rp[-1] == len(ci) and deg.max() <= p["R"] and deg.min() >= 0
    assert ci.max() < n
    src = np.repeat(np.arange(n, dtype=np.uint32), deg)
    assert not np.any(src == ci)  # no self loops
    sizes = np.diff(off)
    assert out.stats["n_edges"] == 2 * int(np.minimum(p["k"], sizes - 1).clip(min=0).dot(sizes))  # R26

    # sampled points: the oracle's full chain, bit-exact against the GPU row
    H = O.hyperplanes(p["m"], cfg.d, p["seed"])
    S = O.sketch(ds, H)
    inst_leaf = {}
    leaf_of_pos = np.repeat(np.arange(len(off) - 1), sizes)
    rng = np.random.default_rng(2026)
    sample = rng.choice(n, size=150, replace=False)
    want = set(int(u) for u in sample)
    pos = np.nonzero(np.isin(ids, sample))[0]
    for q in pos:
        inst_leaf.setdefault(int(ids[q]), []).append(int(leaf_of_pos[q]))
    t0 = time.time()
    bad = []
    for u in sorted(want):
        ref = oracle_row(ds, X, S, off, ids, inst_leaf, u, p)
        got = ci[rp[u]:rp[u + 1]]
        if not np.array_equal(got, ref):
            bad.append(u)
    assert not bad, f"{len(bad)} of {len(want)} sampled rows differ (first: {bad[:5]})"
    print(f"oracle partition {t_part:.1f} s, sampled chain {time.time() - t0:.1f} s, depth {depth}")


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_float_full_size_partition_and_sampled_leaves(name):
    """C3 (1M x 96, L2, unit norm) and C4 (1M x 200, MIPS, fanout 3): the GPU partition against the oracle's
    (invariants; leaf sets identical except near-tie assignments), and the leaf picks of a seeded sample of the
    oracle's leaves under the §8(c) float tolerances."""
    from tests.helpers import check_candidate_lists_float

    cfg = synth.CONFIGS[name]
    X = synth.gen_points(cfg)
    p = cfg.params()
    ds = O.Dataset(X, metric=cfg.metric, mode="bf16")
    off, ids, _ = O.partition(ds, p)
    Xt = torch.from_numpy(X).cuda()
    pp = P().partition_params(c_max=cfg.c_max, fanout=cfg.fanout, seed=cfg.seed)
    goff, gids = P().pipnn_partition(Xt, pp, metric=cfg.metric)
    goff, gids = goff.cpu().numpy(), gids.cpu().numpy().view(np.uint32)
    assert np.diff(goff).max() <= cfg.c_max
    mult = np.bincount(gids, minlength=len(X))
    assert mult.min() >= 1 and mult.max() <= int(np.prod(cfg.fanout))
    a, b = set(canon(goff, gids)), set(canon(off, ids))
    assert len(a & b) >= 0.9 * max(len(a), len(b)), (len(a & b), len(a), len(b))
    rng = np.random.default_rng(7)
    pick = np.sort(rng.choice(len(off) - 1, size=40, replace=False))
    soff = np.concatenate([[0], np.cumsum(np.diff(off)[pick])]).astype(np.int64)
    sids = np.concatenate([ids[off[b]:off[b + 1]] for b in pick]).astype(np.uint32)
    nbr, dist = P().pipnn_leaf_pick(Xt, torch.from_numpy(soff).cuda(), torch.from_numpy(sids.view(np.int32)).cuda(),
                                    cfg.k, cfg.metric)
    torch.cuda.synchronize()
    nbr, dist = nbr.cpu().numpy().view(np.uint32), dist.cpu().numpy()
    onbr, odist = O.leaf_pick(ds, soff, sids, cfg.k)
    ndiff, rows = check_candidate_lists_float(X, cfg.metric, sids, nbr, dist, onbr, odist, cfg.k)
    assert ndiff <= 0.01 * rows, (ndiff, rows)
