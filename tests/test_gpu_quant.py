"""NEXT-2 ("quantized GEMM operations"): the float L2 leaf pick through per-leaf int8-quantised
distances on the int8 tensor cores, re-ranked with the exact bf16-input distances. Returned distances are exact
(within the float tolerance of the bf16-mode oracle); the quantised pre-selection can only miss true neighbours —
every row's picks are exact k-nearest among a superset choice, so each differing pick is no nearer than the oracle's
k-th; and the built graph's recall stays within 0.5 points of the exact path's (paired)."""
import numpy as np
import pytest

import oracle as O
import synth
from tests.helpers import UINT32_MAX, bf16_round, dist_tol, exact_dist

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def P():
    import paper_2602_21247_b200 as P

    return P


@pytest.mark.parametrize("name,n", [("C1", 10000), ("C3", 30000)])
def test_quant_leaf_pick_distances_exact_and_near_complete(name, n):
    cfg = synth.CONFIGS[name]
    cfg = cfg.scaled(n) if cfg.n != n else cfg
    X = synth.gen_points(cfg)
    Xd = torch.from_numpy(X).cuda()
    pp = P().partition_params(c_max=cfg.c_max, fanout=cfg.fanout, seed=cfg.seed)
    off, ids = P().pipnn_partition(Xd, pp)
    nbr, dist = P().pipnn_leaf_pick(Xd, off, ids, cfg.k, quant=1)
    nbr_e, _ = P().pipnn_leaf_pick(Xd, off, ids, cfg.k, quant=0)
    torch.cuda.synchronize()
    offh, idsh = off.cpu().numpy(), ids.cpu().numpy().view(np.uint32)
    g = nbr.cpu().numpy().view(np.uint32)
    gd = dist.cpu().numpy().astype(np.float64)
    onbr, odist = O.leaf_pick(O.Dataset(X, mode="bf16"), offh, idsh, cfg.k)
    Xq = bf16_round(X)
    nrm = (Xq ** 2).sum(1)
    I = len(idsh)
    pid = np.repeat(idsh.astype(np.int64), cfg.k).reshape(I, cfg.k)
    valid = g != UINT32_MAX
    assert np.array_equal(valid.sum(1), (onbr != UINT32_MAX).sum(1))
    q = np.where(valid, g, 0).astype(np.int64)
    Dex = exact_dist(Xq, pid, q, "l2")
    assert (np.abs(gd - Dex)[valid] <= dist_tol(Dex, nrm[pid], nrm[q])[valid]).all()  # exact re-ranked D
    assert (np.diff(np.where(valid, gd, np.inf), axis=1) >= 0).all()  # ascending
    same = (g == onbr).all(1)
    kth = np.where(valid, odist, -np.inf).max(1)
    for r in np.nonzero(~same)[0]:
        for v, d in zip(g[r][valid[r]], gd[r][valid[r]]):
            if v not in set(onbr[r].tolist()):  # a replacement is never nearer than the exact k-th
                assert d >= kth[r] - dist_tol(np.array([kth[r]]), nrm[pid[r, 0]], nrm[v])[0] * 2
    agree = same.mean()
    print(f"{name}: rows identical to the exact pick {agree:.4f}, exact-path (bf16 MMA) rows identical "
          f"{(nbr_e.cpu().numpy().view(np.uint32) == onbr).all(1).mean():.4f}")
    assert agree >= 0.95


@pytest.mark.parametrize("name,n", [("C1", 10000), ("C3", 20000)])
def test_quant_build_recall_parity(name, n):
    from tests.test_gpu_build import paired_recall

    cfg = synth.CONFIGS[name]
    cfg = cfg.scaled(n, n_queries=1000) if cfg.n != n else cfg
    X = synth.gen_points(cfg)
    Q = synth.gen_queries(cfg, n_queries=1000)
    Xd = torch.from_numpy(X).cuda()
    p = cfg.params()
    outs = []
    for quant in (0, 1):
        p["quant"] = quant
        o = P().pipnn_build(Xd, P().build_params_from(p), metric=cfg.metric)
        outs.append((o.row_ptr.cpu().numpy(), o.col_idx.cpu().numpy().view(np.uint32)))
    rows = paired_recall(X, Q, cfg.metric, outs[1], outs[0])
    for L, rq, re, d, se in rows:
        print(f"{name} L={L}: quant {rq:.4f} exact {re:.4f} paired {d:+.4f} (SE {se:.4f})")
        assert abs(d) <= 0.005, (L, rq, re, d, se)


def test_quant_rejects_mips():
    X = torch.from_numpy(synth.gen_points(synth.C4.scaled(3000))).cuda()
    bp = P().build_params_from({**synth.C4.params(), "quant": 1})
    with pytest.raises(P().PipnnError):
        P().pipnn_build(X, bp, metric="mips")
