"""End-to-end parity of pipnn_build (Alg. 4) against the oracle build on the same seeded inputs.
uint8: the CSR graph is bit-exact. float: final-graph recall@10 within 0.5 points (paired, same queries,
same entry point, same CPU beam search) at every L of the sweep (north_star)."""
import numpy as np
import pytest

import oracle as O
import synth
from tests.helpers import UINT32_MAX, check_candidate_lists_float, check_prune_lists_float

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

L_SWEEP = (10, 16, 32, 64, 128)


def P():
    import paper_2602_21247_b200 as P

    return P


def gpu_build(X, params, metric):
    out = P().pipnn_build(torch.from_numpy(X).cuda(), P().build_params_from(params), metric=metric)
    torch.cuda.synchronize()
    return out.row_ptr.cpu().numpy(), out.col_idx.cpu().numpy().view(np.uint32), out.stats


@pytest.mark.parametrize("n,c_max,fanout,l_max", [(20000, 1024, (2,), 128), (50000, 1024, (2,), 128),
                                                  (20000, 256, (3,), 128), (20000, 1024, (2,), 8),
                                                  (20000, 512, (2,), 24)])
def test_build_u8_bit_exact(n, c_max, fanout, l_max):
    # l_max = 8 / 24: reservoirs overflow, so the eviction rule of Alg. 3 runs in the build's merge
    cfg = synth.C2.scaled(n)
    X = synth.gen_points(cfg)
    p = cfg.params()
    p.update(c_max=c_max, p_den=c_max, fanout=fanout, c_min=min(100, c_max // 4), l_max=l_max)
    rp, ci, stats = gpu_build(X, p, "l2")
    ref = O.build(O.Dataset(X), p)
    assert ref.check_failed == 0
    assert stats["n_instances"] == len(ref.leaf_ids) and stats["n_leaves"] == len(ref.leaf_off) - 1
    assert stats["n_edges"] == ref.n_streamed
    assert np.array_equal(rp, ref.row_ptr)
    assert np.array_equal(ci, ref.col_idx)


@pytest.mark.parametrize("cfg", [synth.C5.scaled(200_000), synth.C2_F103.scaled(20_000), synth.C2_R2.scaled(50_000)],
                         ids=["C5-params-200k", "fanout-10x3", "replicas-2"])
def test_build_u8_bit_exact_headline_params_and_overlap_knobs(cfg):
    # C5's parameters (C_max 2048, P_samp 1/1024, l_max 96, R 32; BASELINE.json configs[4]) on a 200k sample
    # of its generator, and the paper's overlap knobs: fanout [10, 3] (30 leaves per
    # point, hub-heavy reservoirs: the table merge) and two replicas
    X = synth.gen_points(cfg)
    p = cfg.params()
    rp, ci, stats = gpu_build(X, p, "l2")
    ref = O.build(O.Dataset(X), p)
    assert ref.check_failed == 0
    assert stats["n_instances"] == len(ref.leaf_ids) and stats["n_leaves"] == len(ref.leaf_off) - 1
    assert stats["n_edges"] == ref.n_streamed
    assert np.array_equal(rp, ref.row_ptr)
    assert np.array_equal(ci, ref.col_idx)


@pytest.mark.parametrize("name,n", [("C2", 200_000), ("C3", 50_000), ("C4", 50_000)])
def test_build_deterministic(name, n):
    # run twice (the same workspace, then a fresh one): byte-identical graphs (SURVEY §4 layer 5)
    cfg = synth.CONFIGS[name].scaled(n)
    Xd = torch.from_numpy(synth.gen_points(cfg)).cuda()
    bp = P().build_params_from(cfg.params())
    b1 = P().Builder(Xd, bp, metric=cfg.metric)
    o1 = b1(Xd)
    g1 = (o1.row_ptr.cpu().numpy().copy(), o1.col_idx.cpu().numpy().copy())
    o2 = b1(Xd)
    o3 = P().Builder(Xd, bp, metric=cfg.metric)(Xd)
    for o in (o2, o3):
        assert np.array_equal(o.row_ptr.cpu().numpy(), g1[0]) and np.array_equal(o.col_idx.cpu().numpy(), g1[1])


@pytest.mark.parametrize("name,n", [("C1", 10000), ("C3", 20000), ("C4", 20000)])
def test_build_float_stage_parity(name, n):
    """The float build path stage by stage (pipnn_debug_build_buffers): its leaf picks against the oracle's
    picks on the same leaves (distances within 1e-3 relative, sets equal but at near-ties), its HashPrune
    reservoirs bit-exact against the oracle's Alg. 3 over the build's own candidate lists, and its final prune
    against the oracle's on the build's reservoirs (lists equal but at near-ties)."""
    cfg = synth.CONFIGS[name]
    cfg = cfg.scaled(n) if cfg.n != n else cfg
    X = synth.gen_points(cfg)
    Xd = torch.from_numpy(X).cuda()
    p = cfg.params()
    b = P().Builder(Xd, P().build_params_from(p), metric=cfg.metric)
    out = b(Xd)
    torch.cuda.synchronize()
    bufs = {kk: v.cpu().numpy() for kk, v in b.debug_buffers(Xd, out.stats).items()}
    off, ids = bufs["leaf_off"], bufs["leaf_ids"].view(np.uint32)
    k = cfg.k
    ds = O.Dataset(X, metric=cfg.metric, mode="bf16")
    # (a3, a4) picks on the build's own leaves
    sizes = np.diff(off)
    start = np.repeat(off[:-1], sizes)
    cols = bufs["cols"].view(np.uint16).astype(np.int64)
    valid = cols != 0xFFFF
    nbr_g = np.where(valid, ids[np.where(valid, start[:, None] + cols, 0)], UINT32_MAX).astype(np.uint32)
    dist_g = bufs["dist"]
    nbr_o, dist_o = O.leaf_pick(ds, off, ids, k)
    ndiff, I = check_candidate_lists_float(X, cfg.metric, ids, nbr_g, dist_g, nbr_o, dist_o, k)
    assert ndiff <= 0.01 * I, ndiff
    # (a0) sketches bit-exact; (a5, a6) reservoirs bit-exact given the build's candidate lists
    S = O.sketch(ds, O.hyperplanes(cfg.m, cfg.d, cfg.seed))
    assert np.array_equal(bufs["sketch"].view(np.uint32), S.view(np.uint32))
    own, cand, dd = O.bidirected_edges(ids, nbr_g, dist_g.astype(np.float64))
    slots_o, count_o, ok = O.hashprune(len(X), S, cfg.l_max, own, cand, dd)
    assert ok
    cnt_g = bufs["count"].view(np.uint32)
    assert np.array_equal(cnt_g, count_o)
    # (inside the build a reservoir is a set: compare each owner's occupied slots sorted)
    mask = np.arange(cfg.l_max)[None, :] < count_o[:, None]
    slots_g = np.where(mask, bufs["slots"].view(np.uint64), np.uint64(0xFFFFFFFFFFFFFFFF))
    assert np.array_equal(np.sort(slots_g, axis=1), slots_o)
    # (a7, a8) final prune on the build's reservoirs
    rp_o, ci_o, _ = O.final_prune(ds, slots_o, count_o, cfg.R)
    rp_g, ci_g = out.row_ptr.cpu().numpy(), out.col_idx.cpu().numpy().view(np.uint32)
    nd, _ = check_prune_lists_float(X, cfg.metric, slots_o, count_o, rp_g, ci_g, rp_o, ci_o)
    assert nd <= 0.01 * len(X), nd


def paired_recall(X, Q, metric, g1, g2):
    ds = O.Dataset(X, metric=metric, mode="exact")
    truth, _ = O.brute_knn(ds, Q, 10)
    e = O.entry_point(ds)
    rows = []
    for L in L_SWEEP:
        r1, _ = O.beam_search(ds, g1[0], g1[1], Q, e, L, 10)
        r2, _ = O.beam_search(ds, g2[0], g2[1], Q, e, L, 10)
        a, b = O.recall_at(r1, truth), O.recall_at(r2, truth)
        diff = a - b
        rows.append((L, a.mean(), b.mean(), diff.mean(), diff.std(ddof=1) / np.sqrt(len(diff))))
    return rows


@pytest.mark.parametrize("name,n", [("C1", 10000), ("C3", 20000), ("C4", 20000)])
def test_build_float_recall_parity(name, n):
    cfg = synth.CONFIGS[name]
    cfg = cfg.scaled(n, n_queries=1000) if cfg.n != n else cfg
    X = synth.gen_points(cfg)
    Q = synth.gen_queries(cfg, n_queries=1000)
    p = cfg.params()
    rp, ci, _ = gpu_build(X, p, cfg.metric)
    assert np.diff(rp).max() <= cfg.R
    ref = O.build(O.Dataset(X, metric=cfg.metric, mode="bf16"), p)
    rows = paired_recall(X, Q, cfg.metric, (rp, ci), (ref.row_ptr, ref.col_idx))
    for L, rg, ro, d, se in rows:
        print(f"{name} L={L}: gpu {rg:.4f} oracle {ro:.4f} paired diff {d:+.4f} (SE {se:.4f})")
        assert abs(d) <= 0.005, (L, rg, ro, d, se)
    # the oracle graph itself is a usable index (not two degenerate graphs agreeing): recall floor at L = 128
    assert rows[-1][2] >= 0.8, rows[-1]
    assert np.diff(ref.row_ptr).mean() >= 8
    ov = np.mean([len(set(ci[rp[u]:rp[u + 1]]) & set(ref.col_idx[ref.row_ptr[u]:ref.row_ptr[u + 1]]))
                  / max(1, ref.row_ptr[u + 1] - ref.row_ptr[u]) for u in range(len(X))])
    print(f"{name}: mean edge overlap {ov:.4f}")
