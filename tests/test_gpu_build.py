"""End-to-end parity of pipnn_build (Alg. 4) against the oracle build on the same seeded inputs.
uint8: the CSR graph is bit-exact. float: final-graph recall@10 within 0.5 points (paired, same queries,
same entry point, same CPU beam search) at every L of the sweep (north_star)."""
import numpy as np
import pytest

import oracle as O
import synth

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
    ov = np.mean([len(set(ci[rp[u]:rp[u + 1]]) & set(ref.col_idx[ref.row_ptr[u]:ref.row_ptr[u + 1]]))
                  / max(1, ref.row_ptr[u + 1] - ref.row_ptr[u]) for u in range(len(X))])
    print(f"{name}: mean edge overlap {ov:.4f}")
