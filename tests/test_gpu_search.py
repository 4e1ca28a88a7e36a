"""GPU batched beam search (pipnn_search, Alg. 1) against the oracle harness's
beam search (same (D, id) beam order, same add-only-unseen rule S:398-399, same entry point) on the oracle's
own graph. uint8: identical result lists and distance-evaluation counts (exact integer distances). float: the
GPU computes fp32 distances, the oracle fp64, so lists agree up to near-ties — recall within 0.5 points."""
import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def P():
    import paper_2602_21247_b200 as P

    return P


def run(X, rp, ci, Q, entry, L, k, metric):
    ids, dist, cmps = P().pipnn_search(torch.from_numpy(X).cuda(), torch.from_numpy(rp.astype(np.int64)).cuda(),
                                       torch.from_numpy(ci.view(np.int32)).cuda(), torch.from_numpy(Q).cuda(),
                                       entry, L, k, metric, count_cmps=True)
    torch.cuda.synchronize()
    return ids.cpu().numpy().view(np.uint32), dist.cpu().numpy(), cmps


@pytest.mark.parametrize("n,L,k", [(20000, 10, 10), (20000, 64, 10), (20000, 128, 10), (5000, 256, 5)])
def test_search_u8_bit_exact(n, L, k):
    cfg = synth.C2.scaled(n)
    X = synth.gen_points(cfg)
    Q = synth.gen_queries(cfg, n_queries=300)
    ds = O.Dataset(X)
    ref = O.build(ds, cfg.params())
    e = O.entry_point(ds)
    oids, ocmps = O.beam_search(ds, ref.row_ptr, ref.col_idx, Q, e, L, k)
    ids, dist, cmps = run(X, ref.row_ptr, ref.col_idx, Q, e, L, k, "l2")
    assert np.array_equal(ids, oids)
    assert cmps == ocmps
    ok = ids != 0xFFFFFFFF
    exact = ((X[ids[ok]].astype(np.int64) - np.repeat(Q, k, 0).reshape(len(Q), k, -1)[ok].astype(np.int64)) ** 2).sum(1)
    assert np.array_equal(dist[ok].astype(np.int64), exact)


@pytest.mark.parametrize("name,n", [("C1", 10000), ("C3", 20000), ("C4", 20000)])
def test_search_float_recall_parity(name, n):
    cfg = synth.CONFIGS[name]
    cfg = cfg.scaled(n) if cfg.n != n else cfg
    X = synth.gen_points(cfg)
    Q = synth.gen_queries(cfg, n_queries=500)
    ds = O.Dataset(X, metric=cfg.metric, mode="bf16")
    ref = O.build(ds, cfg.params())
    dse = O.Dataset(X, metric=cfg.metric, mode="exact")
    e = O.entry_point(dse)
    truth, _ = O.brute_knn(dse, Q, 10)
    for L in (16, 64):
        oids, _ = O.beam_search(dse, ref.row_ptr, ref.col_idx, Q, e, L, 10)
        ids, _, _ = run(X, ref.row_ptr, ref.col_idx, Q, e, L, 10, cfg.metric)
        a, b = O.recall_at(ids, truth).mean(), O.recall_at(oids, truth).mean()
        assert abs(a - b) <= 0.005, (L, a, b)
        assert (ids == oids).all(axis=1).mean() >= 0.95  # identical lists except near-ties


def test_search_edge_cases():
    cfg = synth.C2.scaled(3000)
    X = synth.gen_points(cfg)
    ds = O.Dataset(X)
    ref = O.build(ds, cfg.params())
    Q = X[:50].copy()  # queries that are base points: their own id comes first at distance 0
    ids, dist, _ = run(X, ref.row_ptr, ref.col_idx, Q, 0, 32, 1, "l2")
    oids, _ = O.beam_search(ds, ref.row_ptr, ref.col_idx, Q, 0, 32, 1)
    assert np.array_equal(ids, oids)
    # an empty graph: the beam is the entry point alone, the rest UINT32_MAX
    rp0 = np.zeros(len(X) + 1, dtype=np.int64)
    ci0 = np.zeros(1, dtype=np.uint32)
    ids, dist, cmps = run(X, rp0, ci0, Q[:3], 7, 8, 4, "l2")
    assert (ids[:, 0] == 7).all() and (ids[:, 1:] == 0xFFFFFFFF).all() and cmps == 3
    with pytest.raises(Exception):
        run(X, ref.row_ptr, ref.col_idx, Q, 0, 300, 10, "l2")  # L > 256


def test_knn_graph_task_u8_bit_exact():
    # the k-NN-graph task: every base point queried on the index, itself left out; against the
    # oracle harness's beam search with k + 1 and the point itself dropped
    cfg = synth.C2.scaled(6000)
    X = synth.gen_points(cfg)
    ds = O.Dataset(X)
    ref = O.build(ds, cfg.params())
    e = O.entry_point(ds)
    k, L = 10, 32
    oids, _ = O.beam_search(ds, ref.row_ptr, ref.col_idx, X, e, L, L)
    want = np.full((len(X), k), 0xFFFFFFFF, dtype=np.uint32)
    for i in range(len(X)):
        row = [v for v in oids[i] if v != i and v != 0xFFFFFFFF][:k]
        want[i, :len(row)] = row
    ids, dist = P().knn_graph(torch.from_numpy(X).cuda(), torch.from_numpy(ref.row_ptr.astype(np.int64)).cuda(),
                              torch.from_numpy(ref.col_idx.view(np.int32)).cuda(), e, k, L)
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), want)


@pytest.mark.parametrize("deg", [300, 1000])
def test_search_high_degree_rows(deg):
    # rows longer than the kernel's 256-entry candidate buffer are merged in steps of 256 (top-L composes):
    # identical result lists to the oracle harness for any out-degree (include/pipnn.h). The distance count can
    # only grow: a neighbour that was in the beam when the row started but was pushed out by an earlier step of
    # the same row is evaluated again (the harness still holds it in its untruncated beam).
    cfg = synth.C2.scaled(3000)
    X = synth.gen_points(cfg)
    rng = np.random.default_rng(deg)
    n = len(X)
    rows = [np.sort(rng.choice(np.delete(np.arange(n), u), size=deg if u % 3 == 0 else 20, replace=False))
            for u in range(n)]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    ci = np.concatenate(rows).astype(np.uint32)
    Q = synth.gen_queries(cfg, n_queries=100)
    ds = O.Dataset(X)
    for L in (16, 64):
        oids, ocmps = O.beam_search(ds, rp, ci, Q, 0, L, 10)
        ids, _, cmps = run(X, rp, ci, Q, 0, L, 10, "l2")
        assert np.array_equal(ids, oids) and ocmps <= cmps <= 1.01 * ocmps
