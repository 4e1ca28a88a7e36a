"""GPU parity of pipnn_leaf_pick (K5: tcgen05 distance tiles + fused top-k) against the CPU oracle, both fed
the same (oracle) leaves. uint8: bit-exact ids and distances. float: SURVEY §8(c) tolerances."""
import numpy as np
import pytest

import oracle as O
import synth
from tests.helpers import UINT32_MAX, check_candidate_lists_float

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def P():
    import paper_2602_21247_b200 as P

    return P


def run_gpu(X, metric, off, ids, k):
    Xt = torch.from_numpy(X).cuda()
    nbr, dist = P().pipnn_leaf_pick(Xt, torch.from_numpy(off).cuda(), torch.from_numpy(ids.view(np.int32)).cuda(), k,
                                    metric)
    torch.cuda.synchronize()
    return nbr.cpu().numpy().view(np.uint32), dist.cpu().numpy()


def random_leaves(n, sizes, seed=0):
    rng = np.random.default_rng(seed)
    leaves = [np.sort(rng.choice(n, size=s, replace=False)).astype(np.uint32) for s in sizes]
    off = np.concatenate([[0], np.cumsum([len(l) for l in leaves])]).astype(np.int64)
    return off, np.concatenate(leaves)


EDGE_SIZES = [1, 2, 3, 8, 9, 16, 17, 31, 32, 33, 127, 128, 129, 255, 256, 257, 300, 511, 512, 1000, 1024, 1500,
              2048, 4096]


@pytest.mark.parametrize("k", [1, 3, 8, 10, 15])
def test_leaf_pick_u8_edge_sizes_bit_exact(k):
    X = synth.gen_uniform(6000, 128, "u8", seed=3)
    X = (X // 16).astype(np.uint8)  # coarse values -> many exact distance ties (id tie-break)
    off, ids = random_leaves(len(X), EDGE_SIZES, seed=k)
    nbr, dist = run_gpu(X, "l2", off, ids, k)
    onbr, odist = O.leaf_pick(O.Dataset(X), off, ids, k)
    assert np.array_equal(nbr, onbr)
    ok = onbr != UINT32_MAX
    assert np.array_equal(dist[ok].astype(np.float64), odist[ok])
    assert np.isinf(dist[~ok]).all()


@pytest.mark.parametrize("d", [100, 128, 200])
def test_leaf_pick_u8_other_dims(d):
    X = synth.gen_uniform(3000, d, "u8", seed=d)
    off, ids = random_leaves(len(X), [5, 130, 700, 1024], seed=1)
    nbr, dist = run_gpu(X, "l2", off, ids, 8)
    onbr, odist = O.leaf_pick(O.Dataset(X), off, ids, 8)
    assert np.array_equal(nbr, onbr)
    ok = onbr != UINT32_MAX
    assert np.array_equal(dist[ok].astype(np.float64), odist[ok])


@pytest.mark.parametrize("name,n", [("C2", 20000)])
def test_leaf_pick_u8_config_leaves(name, n):
    cfg = synth.CONFIGS[name].scaled(n)
    X = synth.gen_points(cfg)
    ds = O.Dataset(X)
    off, ids, _ = O.partition(ds, cfg.params())
    nbr, dist = run_gpu(X, "l2", off, ids, cfg.k)
    onbr, odist = O.leaf_pick(ds, off, ids, cfg.k)
    assert np.array_equal(nbr, onbr)
    ok = onbr != UINT32_MAX
    assert np.array_equal(dist[ok].astype(np.float64), odist[ok])


@pytest.mark.parametrize("name,n", [("C1", 10000), ("C3", 20000), ("C4", 20000)])
def test_leaf_pick_float_config_leaves(name, n):
    cfg = synth.CONFIGS[name]
    if cfg.n != n:
        cfg = cfg.scaled(n)
    X = synth.gen_points(cfg)
    ds = O.Dataset(X, metric=cfg.metric, mode="bf16")
    off, ids, _ = O.partition(ds, cfg.params())
    nbr, dist = run_gpu(X, cfg.metric, off, ids, cfg.k)
    onbr, odist = O.leaf_pick(ds, off, ids, cfg.k)
    ndiff, rows = check_candidate_lists_float(X, cfg.metric, ids, nbr, dist, onbr, odist, cfg.k)
    assert ndiff <= 0.01 * rows, (ndiff, rows)


@pytest.mark.parametrize("metric,d,k", [("l2", 96, 8), ("mips", 200, 8), ("l2", 240, 8), ("l2", 7, 8), ("l2", 96, 3),
                                        ("mips", 200, 3), ("l2", 128, 4), ("mips", 96, 12)])
def test_leaf_pick_float_edge_sizes(metric, d, k):
    # k = 3, 4, 12 run list lengths below their instantiation's capacity (-inf sentinel slots)
    X = synth.gen_uniform(6000, d, "f32", seed=d)
    off, ids = random_leaves(len(X), EDGE_SIZES, seed=2)
    nbr, dist = run_gpu(X, metric, off, ids, k)
    onbr, odist = O.leaf_pick(O.Dataset(X, metric=metric, mode="bf16"), off, ids, k)
    ndiff, rows = check_candidate_lists_float(X, metric, ids, nbr, dist, onbr, odist, k)
    assert ndiff <= 0.01 * rows, (ndiff, rows)


def test_leaf_pick_rejects_k16():
    X = torch.zeros((10, 8), dtype=torch.uint8, device="cuda")
    off = torch.tensor([0, 10], dtype=torch.int64, device="cuda")
    ids = torch.arange(10, dtype=torch.int32, device="cuda")
    with pytest.raises(P().PipnnError):
        P().pipnn_leaf_pick(X, off, ids, 16)


def test_leaf_pick_u8_large_distances_bit_exact():
    # d = 512 with coordinates in {0, 255}: squared distances and ranking keys exceed 2^24 (not exact in fp32),
    # so any float detour in the integer path would show up as a wrong pick or distance
    rng = np.random.default_rng(11)
    X = (rng.integers(0, 2, size=(3000, 512)) * 255).astype(np.uint8)
    off, ids = random_leaves(len(X), [5, 130, 700, 1024], seed=4)
    nbr, dist = run_gpu(X, "l2", off, ids, 8)
    onbr, odist = O.leaf_pick(O.Dataset(X), off, ids, 8)
    assert odist[onbr != UINT32_MAX].max() > 2 ** 24
    assert np.array_equal(nbr, onbr)
    ok = onbr != UINT32_MAX
    # the ABI's dist is float32: the exact integer D rounded to nearest (pipnn.h)
    assert np.array_equal(dist[ok], odist[ok].astype(np.float32))


def test_leaf_pick_u8_wide_norm_range_bit_exact():
    # leaves whose squared norms span up to ~8e6 next to narrow ones (ranking keys ||y||^2 - 2 x.y over a wide
    # range, with near-zero rows): picks and distances stay exact
    rng = np.random.default_rng(21)
    narrow = np.clip(rng.normal(128, 20, size=(2000, 128)).round(), 0, 255).astype(np.uint8)
    scale = rng.uniform(0.0, 1.0, size=(2000, 1))
    wide = np.clip((scale * rng.integers(0, 256, size=(2000, 128))).round(), 0, 255).astype(np.uint8)
    X = np.concatenate([narrow, wide])
    nrm = (X.astype(np.int64) ** 2).sum(1)
    leaves = []
    for lo, hi, size in [(0, 2000, 1024), (0, 2000, 300), (2000, 4000, 1024), (2000, 4000, 129), (0, 4000, 700)]:
        leaves.append(np.sort(rng.choice(np.arange(lo, hi), size=size, replace=False)).astype(np.uint32))
    off = np.concatenate([[0], np.cumsum([len(l) for l in leaves])]).astype(np.int64)
    ids = np.concatenate(leaves)
    spans = [nrm[l].max() - nrm[l].min() for l in leaves]
    assert min(spans) < 2e6 < max(spans)  # narrow and wide leaves
    nbr, dist = run_gpu(X, "l2", off, ids, 8)
    onbr, odist = O.leaf_pick(O.Dataset(X), off, ids, 8)
    assert np.array_equal(nbr, onbr)
    ok = onbr != UINT32_MAX
    assert np.array_equal(dist[ok], odist[ok].astype(np.float32))
