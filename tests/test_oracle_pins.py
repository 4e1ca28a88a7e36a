"""Pins of the CPU oracle to things other than itself (paper/SPEC worked examples, closed forms, textbook
values, brute force, invariants). CPU only. Each test names the passage it pins."""
import itertools
import math

import numpy as np
import pytest

import oracle as O
import synth


def ds_of(rows, dtype=np.float32, metric="l2", mode="exact"):
    return O.Dataset(np.array(rows, dtype=dtype), metric=metric, mode=mode)


# ---------------------------------------------------------------- O0 dissimilarity
def test_dist_spec_examples():
    assert O.dist(ds_of([[1, 2], [1, 2]]), 0, 1) == 0.0
    assert O.dist(ds_of([[0, 0], [3, 4]]), 0, 1) == 25.0  # S:43 (3-4-5)
    assert O.dist(ds_of([[0, 0], [3, 4]], np.uint8), 0, 1) == 25.0
    assert O.dist(ds_of([[1, 0], [2, 5]], metric="mips"), 0, 1) == -2.0


def test_dist_closed_forms_u8():
    # constant vectors: ||a1 - b1||^2 = d (a-b)^2, exact for every pair of byte values
    d = 128
    for a, b in [(0, 255), (255, 0), (17, 200), (128, 127), (3, 3)]:
        ds = ds_of([[a] * d, [b] * d], np.uint8)
        assert O.dist(ds, 0, 1) == d * (a - b) ** 2
        assert O.dist(ds, 1, 0) == O.dist(ds, 0, 1)  # symmetry S:66


def test_dist_closed_forms_float():
    d = 200
    e = np.eye(d, dtype=np.float32)
    ds = O.Dataset(e[:3].copy(), "l2", "exact")
    assert O.dist(ds, 0, 1) == 2.0  # orthonormal: ||e_i - e_j||^2 = 2
    dm = O.Dataset(e[:3].copy(), "mips", "exact")
    assert O.dist(dm, 0, 1) == 0.0 and O.dist(dm, 0, 0) == -1.0
    # scaling by powers of two scales L2 by 4^s exactly
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, d)).astype(np.float32)
    D1 = O.dist(O.Dataset(x, "l2", "exact"), 0, 1)
    D2 = O.dist(O.Dataset(x * 4, "l2", "exact"), 0, 1)
    assert D2 == 16 * D1


def test_bf16_mode_rounds_inputs():
    # 1 + 2^-8 lies halfway between bf16 neighbours 1 and 1+2^-7 -> RNE to even -> 1.0
    x = np.array([[1.0 + 2 ** -8], [0.0]], dtype=np.float32)
    assert O.dist(O.Dataset(x, "l2", "bf16"), 0, 1) == 1.0
    assert O.dist(O.Dataset(x, "l2", "exact"), 0, 1) == pytest.approx((1 + 2 ** -8) ** 2, rel=0, abs=0)
    # 1 + 3*2^-8 is halfway between 1+2^-7 (odd) and 1+2^-6 (even) -> 1+2^-6
    y = np.array([[1.0 + 3 * 2 ** -8], [0.0]], dtype=np.float32)
    assert O.dist(O.Dataset(y, "l2", "bf16"), 0, 1) == (1 + 2 ** -6) ** 2


def test_okey_orders_like_values():
    # okey(bf16(.)) is monotone in the value; textbook bf16 encodings of +-1, 0
    assert O.dist_okey(1.0) == 0x3F80 ^ 0x8000
    assert O.dist_okey(-1.0) == 0xBF80 ^ 0xFFFF
    assert O.dist_okey(-0.0) == O.dist_okey(0.0) == 0x8000  # -0 canonicalised (R5)
    vals = np.sort(np.random.default_rng(0).standard_normal(2000) * 1e3)
    keys = [O.dist_okey(float(v)) for v in vals]
    assert all(a <= b for a, b in zip(keys, keys[1:]))


# ---------------------------------------------------------------- O1 randomness (docs/DETERMINISM.md)
def test_splitmix64_reference_vector():
    # SplitMix64 seeded with 0 yields 0xE220A8397B1DCDAF, then 0x6E789E6AA1B965F4 (Steele/Lea/Flood, Vigna)
    # mix(a, b) = sm(a ^ sm(b)); sm(x) is the output for state x: mix(0, g) with sm(g) = ... use sm via mix(x, y)
    # with sm(b) chosen so that a ^ sm(b) = 0: not directly reachable, so pin the composition instead:
    sm0 = 0xE220A8397B1DCDAF
    # mix(sm0, 0) = sm(sm0 ^ sm(0)) = sm(0) = sm0
    assert O.mix(sm0, 0) == sm0
    # mix(sm0 ^ 0x9E3779B97F4A7C15, 0) = sm(gamma) = second SplitMix64(0) output
    assert O.mix(sm0 ^ 0x9E3779B97F4A7C15, 0) == 0x6E789E6AA1B965F4


def test_hyperplanes_irwin_hall_moments():
    # H_ij = sum of 4 iid (2u-31), u ~ U{0..31}: range [-124,124], mean 0, var 4*(4*(32^2-1)/12) = 1364
    H = O.hyperplanes(64, 512, 7).astype(np.int64)
    assert H.min() >= -124 and H.max() <= 124
    assert abs(H.mean()) < 3 * math.sqrt(1364 / H.size)
    assert abs(H.var() - 1364) < 0.05 * 1364
    assert (np.abs(H) % 2 == 0).all()  # sum of four odd numbers is even
    assert not np.array_equal(H, O.hyperplanes(64, 512, 8))


# ---------------------------------------------------------------- O2 sketches + residual hash (Eq. 1)
def test_residual_hash_spec_examples():
    # c = p -> all ones
    s = np.array([3.0, -1.0, 0.0, 7.0])
    assert O.residual_hash(s, s) == 0b1111
    # d=2, p=origin, H=I, c=(1,-1): sketches are coordinates -> bits (1,0)
    assert O.residual_hash(np.array([0.0, 0.0]), np.array([1.0, -1.0])) == 0b01


def test_sketch_hash_equals_direct_residual_hash_u8():
    # sketch-difference hash == sign(H.(c-p)) computed directly (numpy int64 matmul), exact on u8
    X = synth.gen_uniform(300, 128, "u8", seed=5)
    ds = O.Dataset(X)
    H = O.hyperplanes(12, 128, 11)
    S = O.sketch(ds, H)
    assert S.dtype == np.int32
    np.testing.assert_array_equal(S.astype(np.int64), X.astype(np.int64) @ H.T.astype(np.int64))
    rng = np.random.default_rng(1)
    for _ in range(500):
        p, c = rng.integers(0, 300, 2)
        direct = (H.astype(np.int64) @ (X[c].astype(np.int64) - X[p].astype(np.int64))) >= 0
        want = sum(1 << i for i in range(12) if direct[i])
        assert O.residual_hash(S[p].astype(np.float64), S[c].astype(np.float64)) == want


def test_sketch_float_bf16_mode():
    X = synth.gen_uniform(50, 96, "f32", seed=2)
    H = O.hyperplanes(12, 96, 3)
    S = O.sketch(O.Dataset(X, mode="bf16"), H)
    Xb = O.Dataset(X, mode="bf16")  # values rounded to bf16 (RNE): reproduce with numpy bit ops
    u = X.view(np.uint32).astype(np.uint64)
    ub = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    xb = ub.astype(np.uint32).view(np.float32).astype(np.float64)
    ref = (xb @ H.T.astype(np.float64)).astype(np.float32)
    np.testing.assert_allclose(S, ref, rtol=1e-6, atol=1e-3)
    del Xb


def test_collision_probability_per_bit():
    # P:317 / S:268: P[one bit differs] = theta/pi for random hyperplanes through the origin. Checked on
    # dense random unit vectors (the integer Irwin-Hall generator, R7), 3 standard errors.
    d, m = 128, 4000
    H = O.hyperplanes(m, d, 99).astype(np.float64)
    rng = np.random.default_rng(4)
    for theta_deg in (10, 45, 90, 135):
        th = math.radians(theta_deg)
        a = rng.standard_normal(d); a /= np.linalg.norm(a)
        b = rng.standard_normal(d); b -= a * (a @ b); b /= np.linalg.norm(b)
        v = math.cos(th) * a + math.sin(th) * b
        diff = np.mean((H @ a >= 0) != (H @ v >= 0))
        p = th / math.pi
        assert abs(diff - p) < 3 * math.sqrt(p * (1 - p) / m) + 1e-9, (theta_deg, diff, p)


# ---------------------------------------------------------------- O3 partition (Alg. 5)
def params(**kw):
    p = synth.C1.params()
    p.update(kw)
    if "c_max" in kw and "p_den" not in kw:
        p["p_den"] = kw["c_max"]  # P_samp = 2/C_max (reading R10)
    return p


def test_partition_base_case_single_leaf():
    # n <= C_max -> one leaf with all ids
    X = synth.gen_uniform(500, 16, "f32")
    off, ids, depth = O.partition(O.Dataset(X), params(c_max=1024))
    assert len(off) == 2 and np.array_equal(ids, np.arange(500)) and depth == 0


def test_merge_spec_examples():
    keys = np.array([5, 3], dtype=np.uint64)
    g, ng = O.merge_plan([50, 60], keys, [0, 1], 100, 1024)  # [50,60] -> one group of 110
    assert ng == 1 and g[0] == g[1] == 0
    g, ng = O.merge_plan([1000, 50], keys, [0, 1], 100, 1024)  # 1050 > C_max -> unchanged
    assert ng == 2 and g[0] != g[1]
    g, ng = O.merge_plan([0, 500, 40], [1, 2, 3], [0, 1, 2], 100, 1024)  # leftover absorbed by a big group
    assert g[0] == -1 and g[1] == g[2]


def _same(g, a, b):
    return g[a] == g[b]


def test_merge_bins_close_in_key_order():
    """R15: small groups are taken in (key, id) order and a bin closes once the SUM of its sizes
    reaches C_min. Hand-derived: sizes [30, 40, 50, 20], C_min 60."""
    s = [30, 40, 50, 20]
    # key order 1, 3, 0, 2 -> sizes 40, 20 | 30, 50 -> bins {1, 3} (60) and {0, 2} (80)
    g, ng = O.merge_plan(s, np.array([3, 1, 4, 2], np.uint64), [0, 1, 2, 3], 60, 1000)
    assert ng == 2 and _same(g, 1, 3) and _same(g, 0, 2) and not _same(g, 0, 1)
    # identity order -> 30, 40 | 50, 20 -> bins {0, 1} (70) and {2, 3} (70)
    g, ng = O.merge_plan(s, np.array([1, 2, 3, 4], np.uint64), [0, 1, 2, 3], 60, 1000)
    assert ng == 2 and _same(g, 0, 1) and _same(g, 2, 3) and not _same(g, 0, 2)
    # equal keys: the id breaks the tie (ids 3, 1, 4, 2 reproduce the first order)
    g, ng = O.merge_plan(s, np.array([7, 7, 7, 7], np.uint64), [3, 1, 4, 2], 60, 1000)
    assert ng == 2 and _same(g, 1, 3) and _same(g, 0, 2) and not _same(g, 0, 1)


def test_merge_leftover_joins_first_closed_bin():
    """R15: a leftover (the small groups after the last closed bin) joins the FIRST closed bin."""
    g, ng = O.merge_plan([40, 30, 10], np.array([1, 2, 3], np.uint64), [0, 1, 2], 60, 1000)
    assert ng == 1 and _same(g, 0, 1) and _same(g, 0, 2)
    # bins {0, 1} (70) and {2, 3} (65) close; the leftover {4} joins {0, 1}
    g, ng = O.merge_plan([40, 30, 35, 30, 10], np.array([1, 2, 3, 4, 5], np.uint64), [0, 1, 2, 3, 4], 60, 1000)
    assert ng == 2 and _same(g, 4, 0) and _same(g, 0, 1) and _same(g, 2, 3) and not _same(g, 4, 2)


def test_merge_leftover_without_bins_joins_smallest_fitting_big():
    """R15: with no closed bin the leftover joins the smallest Big group whose size + leftover sum <= C_max (ties
    by key), else stands alone (a group below C_min survives only if every merge would exceed C_max)."""
    sizes = [500, 300, 300, 20, 15]  # Big: 0, 1, 2 (>= C_min 100); small 3, 4 (sum 35 < C_min: no bin closes)
    keys = np.array([9, 5, 2, 1, 1], np.uint64)
    g, ng = O.merge_plan(sizes, keys, [0, 1, 2, 3, 4], 100, 400)  # 500 + 35 > 400; 300s fit; key 2 < 5
    assert ng == 3 and _same(g, 3, 4) and _same(g, 3, 2) and not _same(g, 3, 1) and not _same(g, 3, 0)
    g, ng = O.merge_plan(sizes, keys, [0, 1, 2, 3, 4], 100, 320)  # 300 + 35 > 320: the leftover stands alone
    assert ng == 4 and _same(g, 3, 4) and len({g[0], g[1], g[2], g[3]}) == 4
    g, ng = O.merge_plan([300, 200, 20], np.array([1, 2, 3], np.uint64), [0, 1, 2], 100, 400)  # smallest fitting Big
    assert ng == 2 and _same(g, 2, 1) and not _same(g, 2, 0)


def test_merge_survival_invariant_fuzz():
    """an output group below C_min survives only if it is the only group or merging it with any other
    output group would exceed C_max; every merged group is a union of whole input groups with at most one Big."""
    rng = np.random.default_rng(1)
    for _ in range(300):
        c_max = int(rng.integers(30, 3000))
        c_min = int(rng.integers(1, max(2, (c_max - 1) // 3)))
        ng = int(rng.integers(1, 40))
        sizes = np.where(rng.random(ng) < 0.6, rng.integers(1, c_min + 1, ng), rng.integers(c_min, 2 * c_max, ng))
        keys = rng.integers(0, 2 ** 63, ng, dtype=np.uint64)
        g, n_out = O.merge_plan(sizes, keys, np.arange(ng), c_min, c_max)
        tot = np.array([sizes[g == t].sum() for t in range(n_out)])
        for t in range(n_out):
            assert (sizes[g == t] >= c_min).sum() <= 1
            if tot[t] < c_min and n_out > 1:
                assert all(tot[t] + tot[u] > c_max for u in range(n_out) if u != t)


def test_merge_bounds_fuzz():
    rng = np.random.default_rng(0)
    for _ in range(300):
        c_max = int(rng.integers(30, 3000))
        c_min = int(rng.integers(1, max(2, (c_max - 1) // 3)))
        ng = int(rng.integers(1, 40))
        sizes = np.where(rng.random(ng) < 0.6, rng.integers(0, c_min, ng), rng.integers(c_min, 2 * c_max, ng))
        keys = rng.integers(0, 2 ** 63, ng, dtype=np.uint64)
        g, n_out = O.merge_plan(sizes, keys, np.arange(ng), c_min, c_max)
        for t in range(n_out):
            members = np.where(g == t)[0]
            total = sizes[members].sum()
            if len(members) > 1:  # merged groups never exceed C_max
                assert total <= c_max
        assert (g[sizes == 0] == -1).all() and (g[sizes > 0] >= 0).all()


def brute_assign(X, L, f):
    """Nearest f leaders by (D, leader id) via full sort (brute force)."""
    D = ((X[:, None, :].astype(np.float64) - X[L][None, :, :].astype(np.float64)) ** 2).sum(-1)
    order = np.lexsort((np.broadcast_to(L, D.shape), D), axis=1)
    return order[:, :f]


def test_partition_depth0_matches_brute_force():
    # Alg. 5 lines 2-9 on a tiny input with no merge and no recursion: the leaves must be exactly the
    # groups of the f=2 nearest of the l = ceil(2n/C_max) leaders with the smallest mix(K0, id).
    n, c_max = 240, 200
    p = params(c_max=c_max, c_min=10, fanout=(2,))
    l = max(2, -(-2 * n // c_max))
    K0 = O.mix(O.mix(p["seed"], 0x5041525449544E31), 0)
    pri = sorted((O.mix(K0, i), i) for i in range(n))
    L = np.array(sorted(i for _, i in pri[:l]))
    for seed in range(100):  # first seeded input on which no group merges or recurses (precondition)
        X = np.random.default_rng(seed).integers(0, 256, size=(n, 8), dtype=np.uint8)
        a = brute_assign(X, L, 2)
        groups = [sorted(np.where((a == j).any(1))[0].tolist()) for j in range(l)]
        if all(c_max >= len(g) >= 10 for g in groups):
            break
    else:
        pytest.fail("no input satisfied the precondition")
    off, ids, depth = O.partition(O.Dataset(X), p)
    leaves = sorted(ids[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1))
    assert leaves == sorted(groups) and depth == 0


@pytest.mark.parametrize("cfg,fan,reps", [("u8", (2,), 1), ("f32", (3,), 1), ("f32", (4, 2), 2)])
def test_partition_invariants(cfg, fan, reps):
    # leaf <= C_max; every id in >= replicas and <= prod(fanout)*replicas leaves;
    # ids ascending and unique within a leaf.
    X = synth.gen_points(synth.C2.scaled(6000, n_centres=60)) if cfg == "u8" else synth.gen_points(
        synth.C1.scaled(6000, n_centres=60))
    p = params(c_max=256, c_min=40, fanout=fan, replicas=reps)
    off, ids, depth = O.partition(O.Dataset(X), p)
    sizes = np.diff(off)
    assert sizes.max() <= 256 and sizes.min() >= 1
    mult = np.bincount(ids, minlength=len(X))
    assert mult.min() >= reps and mult.max() <= int(np.prod(fan)) * reps
    for i in range(len(off) - 1):
        leaf = ids[off[i]:off[i + 1]]
        assert (np.diff(leaf.astype(np.int64)) > 0).all()
    assert depth <= 2 * math.ceil(math.log(6000) / math.log(max(2, 2 * 6000 / 256))) + 4


def test_partition_duplicates_guard():
    # all-identical points cannot separate: the guard splits into ceil(n/C_max) chunks
    X = np.zeros((1000, 8), dtype=np.uint8)
    off, ids, depth = O.partition(O.Dataset(X), params(c_max=128, c_min=10, fanout=(2,)))
    assert np.diff(off).max() <= 128
    assert set(ids.tolist()) == set(range(1000))


def test_partition_deterministic_across_threads():
    X = synth.gen_points(synth.C1.scaled(5000, n_centres=50))
    p = params(c_max=256, c_min=40)
    O.set_threads(1)
    a = O.partition(O.Dataset(X), p)
    O.set_threads(8)
    b = O.partition(O.Dataset(X), p)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ---------------------------------------------------------------- O4 leaf pick
def test_leaf_pick_collinear_example():
    # points 0,1,3 on a line, k=1: N(0)={1}, N(1)={0}, N(3)={1}; bidirected edges
    ds = ds_of([[0.0], [1.0], [3.0]])
    nbr, dd = O.leaf_pick(ds, np.array([0, 3]), np.array([0, 1, 2], np.uint32), 1)
    assert nbr[:, 0].tolist() == [1, 0, 1] and dd[:, 0].tolist() == [1.0, 1.0, 4.0]
    own, cand, _ = O.bidirected_edges(np.array([0, 1, 2], np.uint32), nbr, dd)
    assert set(zip(own.tolist(), cand.tolist())) == {(0, 1), (1, 0), (2, 1), (1, 2)}


@pytest.mark.parametrize("dtype,metric", [("u8", "l2"), ("f32", "l2"), ("f32", "mips")])
def test_leaf_pick_single_leaf_is_exact_knn(dtype, metric):
    # one leaf holding all points: forward picks = exact k-NN by full sort with id tie-break (north_star)
    n, d, k = 300, 24, 8
    X = synth.gen_uniform(n, d, dtype, seed=9)
    if dtype == "u8":
        X = (X // 32).astype(np.uint8)  # many exact ties -> exercises the id tie-break
    ds = O.Dataset(X, metric=metric, mode="exact")
    nbr, dd = O.leaf_pick(ds, np.array([0, n]), np.arange(n, dtype=np.uint32), k)
    Xd = X.astype(np.float64)
    D = -(Xd @ Xd.T) if metric == "mips" else ((Xd[:, None] - Xd[None]) ** 2).sum(-1)
    for i in range(n):
        row = [(D[i, j], j) for j in range(n) if j != i]
        row.sort()
        assert nbr[i].tolist() == [j for _, j in row[:k]]
        np.testing.assert_allclose(dd[i], [v for v, _ in row[:k]], rtol=1e-12, atol=1e-9)


def test_leaf_pick_small_leaves_clamp():
    # |b| <= k: pick |b|-1 and pad; singleton leaves emit nothing
    ds = ds_of([[0.0], [1.0], [5.0]])
    nbr, dd = O.leaf_pick(ds, np.array([0, 1, 3]), np.array([2, 0, 1], np.uint32), 4)
    assert nbr[0].tolist() == [0xFFFFFFFF] * 4 and math.isinf(dd[0, 0])
    assert nbr[1].tolist()[:2] == [1, 0xFFFFFFFF] and nbr[2].tolist()[:2] == [0, 0xFFFFFFFF]


# ---------------------------------------------------------------- O5 HashPrune (Alg. 3, Supp. G)
def test_hashprune_spec_examples():
    ids, _ = O.hashprune_list([1, 2, 3], [1.0, 2.0, 3.0], [1, 2, 3], 2)
    assert sorted(ids.tolist()) == [1, 2]
    # a(X,5) b(Y,1) c(Z,2) d(X,10), l_max=2 -> {b,c} in all 24 orders
    items = [(0, 5.0, 10), (1, 1.0, 11), (2, 2.0, 12), (0, 10.0, 13)]
    for perm in itertools.permutations(items):
        h, dd, i = zip(*perm)
        ids, _ = O.hashprune_list(h, dd, i, 2, "stream")
        assert sorted(ids.tolist()) == [11, 12]


def test_hashprune_history_independence_fuzz():
    # streaming in 20 random orders == characterization (bucket minima, then l_max closest),
    # coarse distances so bf16 ties are frequent (the id tie-break matters, R4)
    rng = np.random.default_rng(0)
    for trial in range(200):
        nc = int(rng.integers(1, 300))
        lmax = int(rng.choice([1, 2, 4, 16, 64]))
        h = rng.integers(0, int(rng.choice([2, 8, 64, 4096])), nc)
        dd = rng.integers(0, 20, nc).astype(np.float64) * 0.25
        ids = rng.integers(0, 1000, nc)
        ref, refh = O.hashprune_list(h, dd, ids, lmax, "char")
        # closed-form check of the characterization itself (numpy, independent of the oracle)
        best = {}
        for hh, d_, i in zip(h, dd, ids):
            key = (O.dist_okey(d_), int(i))
            if hh not in best or key < best[hh][0]:
                best[hh] = (key, int(i))
        keep = sorted(best.items(), key=lambda kv: kv[1][0])[:lmax]
        assert sorted((int(k), v[1]) for k, v in keep) == sorted(zip(refh.tolist(), ref.tolist()))
        for _ in range(20):
            p = rng.permutation(nc)
            got, goth = O.hashprune_list(h[p], dd[p], ids[p], lmax, "stream")
            assert got.tolist() == ref.tolist() and goth.tolist() == refh.tolist()


def test_hashprune_fig2_geometry():
    # P:336-399 Fig. 2: p at the origin; c1 (50deg,.45) c2 (160deg,.85) c3 (340deg,.65); c' (175deg,.55).
    # Coarse hyperplanes (y-sign, x-sign): c' collides with and evicts the farther c2 -> {c1,c3,c'}.
    # A finer set adds a hyperplane (normal at 77.5deg) separating c2 and c' -> all four retained.
    pol = {"c1": (50, .45), "c2": (160, .85), "c3": (340, .65), "cp": (175, .55)}
    names = list(pol)
    P = np.array([[r * math.cos(math.radians(a)), r * math.sin(math.radians(a))] for a, r in pol.values()])
    for Hs, want in [([(0, 1), (1, 0)], {"c1", "c3", "cp"}),
                     ([(0, 1), (1, 0), (math.cos(math.radians(77.5)), math.sin(math.radians(77.5)))],
                      {"c1", "c2", "c3", "cp"})]:
        H = np.array(Hs)
        S = P @ H.T
        hashes = [O.residual_hash(np.zeros(len(Hs)), S[i]) for i in range(4)]
        dd = (P ** 2).sum(1)
        ids, _ = O.hashprune_list(hashes, dd, np.arange(4), 128, "stream")
        assert {names[i] for i in ids} == want


def test_hashprune_owner_level_invariants_and_composition():
    # Dataset-level Alg. 3 over a bidirected edge multiset: size <= l_max, one slot per hash, slots sorted
    # by hash, every kept item was streamed, and A|B batched composition equals one pass (Supp. G lemma).
    cfg = synth.C2.scaled(3000, n_centres=30)
    X = synth.gen_points(cfg)
    ds = O.Dataset(X)
    off, ids, _ = O.partition(ds, params(c_max=256, c_min=40))
    nbr, dd = O.leaf_pick(ds, off, ids, 8)
    own, cand, dist_ = O.bidirected_edges(ids, nbr, dd)
    S = O.sketch(ds, O.hyperplanes(12, X.shape[1], 1))
    for lmax in (8, 128):
        slots, count, ok = O.hashprune(len(X), S, lmax, own, cand, dist_)
        assert ok
        assert (count <= lmax).all()
        streamed = set(zip(own.tolist(), cand.tolist()))
        for u in range(0, len(X), 7):
            sl = slots[u, :count[u]]
            hs = (sl >> np.uint64(48)).astype(np.int64)
            assert (np.diff(hs) > 0).all()
            assert (slots[u, count[u]:] == np.uint64(0xFFFFFFFFFFFFFFFF)).all()
            for v in (sl & np.uint64(0xFFFFFFFF)).astype(np.int64):
                assert (u, v) in streamed
        cut = len(own) // 3
        perm = np.random.default_rng(2).permutation(len(own))
        a, b = perm[:cut], perm[cut:]
        s1, c1, ok1 = O.hashprune(len(X), S, lmax, own[a], cand[a], dist_[a])
        s2, c2, ok2 = O.hashprune(len(X), S, lmax, own[b], cand[b], dist_[b], init=(s1, c1))
        assert ok1 and ok2 and np.array_equal(s2, slots) and np.array_equal(c2, count)


# ---------------------------------------------------------------- O6 RobustPrune (Alg. 2)
def test_robust_prune_spec_examples():
    ds = ds_of([[0.0], [1.0], [2.0], [3.0]])
    assert O.robust_prune(ds, 0, [1, 2, 3], 64, (1, 1), lazy=False).tolist() == [1]
    assert O.robust_prune(ds, 0, [1, 2, 3], 64, (1, 1), lazy=True).tolist() == [1]
    assert O.robust_prune(ds, 0, [2], 64).tolist() == [2]
    assert O.robust_prune(ds, 0, [3, 1, 2], 1).tolist() == [1]  # S:305 R=1 -> nearest
    assert O.robust_prune(ds, 0, [], 64).tolist() == []
    # alpha -> infinity behaves like "no pruning fires": the R nearest
    assert O.robust_prune(ds, 0, [3, 1, 2], 2, (10 ** 9, 1)).tolist() == [1, 2]


def test_robust_prune_eager_equals_lazy_and_diversity():
    # eager == lazy on random instances; output <= R; for admitted y before z: alpha*D(y,z) >= D(p,z)
    rng = np.random.default_rng(5)
    for trial in range(300):
        n = int(rng.integers(2, 60))
        X = rng.integers(0, 16, size=(n, 3)).astype(np.uint8)
        ds = O.Dataset(X)
        cands = rng.choice(np.arange(1, n), size=int(rng.integers(0, n - 1)), replace=False)
        R = int(rng.integers(1, 10))
        lazy = O.robust_prune(ds, 0, cands, R, (6, 5), True)
        eager = O.robust_prune(ds, 0, cands, R, (6, 5), False)
        assert lazy.tolist() == eager.tolist() and len(lazy) <= R
        Xd = X.astype(np.int64)
        for i, y in enumerate(lazy):
            for z in lazy[i + 1:]:
                assert 6 * ((Xd[y] - Xd[z]) ** 2).sum() >= 5 * ((Xd[0] - Xd[z]) ** 2).sum()


def _slot(hash16, bf16_bits, vid):
    # reservoir slot layout of SURVEY §8(b): hash(16) | okey(bf16 dist)(16) | id(32); for a positive bf16 value
    # okey(b) = b ^ 0x8000 (the sign bit set), written out by hand here
    return (hash16 << 48) | ((bf16_bits ^ 0x8000) << 32) | vid


def test_final_prune_zero_keeps_first_R_by_key():
    # final_prune = 0 keeps the first R reservoir entries by (stored bf16 distance, id). Hand-built
    # reservoir of point 0: dists 3.0 (0x4040), 1.0 (0x3F80), 2.0 (0x4000), 1.0 (0x3F80) for ids 7, 9, 4, 2,
    # stored in hash order -> (1.0, 2), (1.0, 9), (2.0, 4), (3.0, 7).
    X = np.zeros((10, 4), dtype=np.uint8)
    ds = O.Dataset(X)
    slots = np.full((10, 8), np.iinfo(np.uint64).max, dtype=np.uint64)
    count = np.zeros(10, dtype=np.uint32)
    row = [_slot(1, 0x4040, 7), _slot(3, 0x3F80, 9), _slot(5, 0x4000, 4), _slot(9, 0x3F80, 2)]
    slots[0, :4] = np.array(row, dtype=np.uint64)
    count[0] = 4
    for R, want in [(3, [2, 9, 4]), (1, [2]), (8, [2, 9, 4, 7])]:
        rp, ci, ok = O.final_prune(ds, slots, count, R, final=0)
        assert ok and rp.tolist() == [0] + [len(want)] * 10 and ci.tolist() == want


# MIPS final prune (R22, changed): candidates in the (-<u,c>, id) order, the alpha test on the angular
# dissimilarity 1 - cos. Hand-computed 2-D example, u = (1, 0):
#   a = (2, 0)  -<u,a> = -2, angle 0      b = (1, 1)  -<u,b> = -1, 1 - cos = 1 - 1/sqrt2 = 0.2929
#   c = (0.9, 0.1)  -<u,c> = -0.9, 1 - cos(u,c) = 1 - 0.9/0.90554 = 0.00612   e = (0, 3)  -<u,e> = 0, 1 - cos = 1
# order a, b, c, e. b: 1.2 (1 - cos(a,b)) = 0.3515 >= 0.2929 -> kept. c: 1.2 * 0.00612 (a is parallel to u)
# >= 0.00612, and 1 - cos(b,c) = 1 - 1/(sqrt2 * 0.90554) = 0.2191 -> kept. e: 1.2 (1 - cos(b,e)) =
# 1.2 * 0.2929 = 0.3515 < 1 -> pruned by b. Result [a, b, c]. (The signed rule 6 D(y,c) < 5 D(u,c) on
# D = -<.,.> prunes b by a: -12 < -5; that is the collapse R22 fixes.)
def test_robust_prune_mips_angular_hand_example():
    ds = ds_of([[1, 0], [2, 0], [1, 1], [0.9, 0.1], [0, 3]], metric="mips", mode="exact")
    for lazy in (True, False):
        assert O.robust_prune(ds, 0, [4, 3, 2, 1], 64, (6, 5), lazy).tolist() == [1, 2, 3]
        assert O.robust_prune(ds, 0, [4, 3, 2, 1], 2, (6, 5), lazy).tolist() == [1, 2]
    # a zero-norm candidate z: cos taken as 0 (1 - cos = 1), so a (1 - cos(a,z) = 1, 1.2 >= 1) cannot prune it
    dz = ds_of([[1, 0], [2, 0], [0, 0]], metric="mips", mode="exact")
    assert O.robust_prune(dz, 0, [2, 1], 64, (6, 5)).tolist() == [1, 2]


def test_robust_prune_mips_unit_norm_equals_l2():
    # closed form: for unit vectors ||a - b||^2 = 2 (1 - <a,b>), so the (-<u,.>, id) order is the L2 order and
    # alpha * (1 - cos) tests are the L2 tests halved: the MIPS prune must equal the (SPEC-pinned) L2 prune.
    # Entries +-1/4 in d = 16 make every norm exactly 1 and every value exact in fp64 (ties included).
    rng = np.random.default_rng(11)
    for trial in range(200):
        n = int(rng.integers(2, 40))
        X = (rng.integers(0, 2, size=(n, 16)) * 0.5 - 0.25).astype(np.float32)
        dm, dl = O.Dataset(X, "mips", "exact"), O.Dataset(X, "l2", "exact")
        cands = rng.choice(np.arange(1, n), size=int(rng.integers(0, n - 1)), replace=False)
        R = int(rng.integers(1, 12))
        for lazy in (True, False):
            assert O.robust_prune(dm, 0, cands, R, (6, 5), lazy).tolist() == \
                O.robust_prune(dl, 0, cands, R, (6, 5), lazy).tolist()


def test_build_mips_graph_is_navigable():
    # C4-shaped (Text2Image) sample: the final prune keeps a usable out-degree and the graph reaches the
    # exact neighbours (P:1044 reports PiPNN's highest maximum recall on the MIPS Text2Image set). Under the
    # signed-value reading the mean out-degree was 1.09 and recall@10 0.23 at L = 128 on this sample.
    cfg = synth.C4.scaled(20000, n_queries=300)
    X, Q = synth.gen_points(cfg), synth.gen_queries(cfg)
    ds = O.Dataset(X, metric="mips", mode="bf16")
    r = O.build(ds, cfg.params())
    assert r.check_failed == 0
    deg = np.diff(r.row_ptr)
    assert deg.mean() >= 10 and deg.max() <= cfg.R
    truth, _ = O.brute_knn(ds, Q, 10)
    res, _ = O.beam_search(ds, r.row_ptr, r.col_idx, Q, O.entry_point(ds), 128, 10)
    assert O.recall_at(res, truth).mean() >= 0.9


# ---------------------------------------------------------------- pipeline (Alg. 4)
def test_build_n3():
    # n=3, C_max >= 3, k=2: one leaf, bidirected 2-NN connects all pairs, every out-degree 2
    X = np.array([[0, 0], [10, 0], [5, 9]], dtype=np.uint8)  # near-equilateral: no alpha-pruning fires
    r = O.build(O.Dataset(X), params(k=2))
    assert np.diff(r.row_ptr).tolist() == [2, 2, 2] and r.check_failed == 0


@pytest.mark.parametrize("dtype", ["u8", "f32"])
def test_build_invariants(dtype):
    cfg = (synth.C2 if dtype == "u8" else synth.C1).scaled(4000, n_centres=40)
    X = synth.gen_points(cfg)
    p = params(c_max=256, c_min=40, R=32, l_max=64)
    r = O.build(O.Dataset(X), p)
    assert r.check_failed == 0  # streaming == characterization, eager == lazy for every point
    sizes = np.diff(r.leaf_off)
    # streamed-edge count = 2 * sum_b |b| * min(k, |b|-1)  (P:1111 generalised, R26)
    assert r.n_streamed == int(2 * (sizes * np.minimum(p["k"], sizes - 1)).sum())
    deg = np.diff(r.row_ptr)
    assert deg.max() <= p["R"]
    # edge provenance, no self-loops / duplicates
    co = set()
    for i in range(len(r.leaf_off) - 1):
        leaf = r.leaf_ids[r.leaf_off[i]:r.leaf_off[i + 1]].tolist()
        co.update((a, b) for a in leaf for b in leaf)
    for u in range(len(X)):
        nb = r.col_idx[r.row_ptr[u]:r.row_ptr[u + 1]].tolist()
        assert u not in nb and len(set(nb)) == len(nb)
        assert all((u, v) in co for v in nb)


def test_build_deterministic_across_threads():
    X = synth.gen_points(synth.C1.scaled(3000, n_centres=30))
    p = params(c_max=256, c_min=40)
    O.set_threads(1)
    a = O.build(O.Dataset(X), p)
    O.set_threads(8)
    b = O.build(O.Dataset(X), p)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)


# ---------------------------------------------------------------- evaluation harness pins
def test_brute_knn_and_recall():
    X = synth.gen_uniform(400, 16, "f32", seed=1)
    ds = O.Dataset(X, mode="exact")
    ids, _ = O.brute_knn(ds, X[:20], 10)
    assert (ids[:, 0] == np.arange(20)).all()  # query equal to a point -> rank 1
    t = np.arange(10)[None].repeat(3, 0)
    assert O.recall_at(t, t).tolist() == [1.0] * 3
    assert O.recall_at(t + 10, t).tolist() == [0.0] * 3
    half = t.copy(); half[:, 5:] += 100
    assert O.recall_at(half, t).tolist() == [0.5] * 3


def test_beam_search_path_graph():
    # path graph 0-1-2-3 on x=0,1,2,3, start 0, q=3.1, L=1 -> {3}
    ds = ds_of([[0.0], [1.0], [2.0], [3.0]])
    rp = np.array([0, 1, 3, 5, 6]); ci = np.array([1, 0, 2, 1, 3, 2], np.uint32)
    ids, cmps = O.beam_search(ds, rp, ci, np.array([[3.1]], np.float32), 0, 1, 1)
    assert ids[0, 0] == 3


def test_beam_search_complete_graph_recall_one():
    X = synth.gen_uniform(60, 8, "f32", seed=2)
    n = len(X)
    rp = np.arange(0, n * (n - 1) + 1, n - 1)
    ci = np.array([v for u in range(n) for v in range(n) if v != u], np.uint32)
    ds = O.Dataset(X, mode="exact")
    Q = synth.gen_uniform(30, 8, "f32", seed=3)
    truth, _ = O.brute_knn(ds, Q, 10)
    res, _ = O.beam_search(ds, rp, ci, Q, 0, 10, 10)
    assert O.recall_at(res, truth).mean() == 1.0


@pytest.mark.slow
def test_recall_quality_bar():
    # S:537 scale-free quality bar (stand-in for Fig. 5): 100K x 64 clustered, default parameters, 10@10 >=
    # 0.95 at some L <= 100. Defaults as SPEC states them: fanout [10, 3] ("10 on the top
    # level, 3 on the second"), k = 2, l_max = 64, R = 64, alpha = 1.2.
    cfg = synth.Config("S537", n=100_000, d=64, dtype="f32", metric="l2", n_centres=1000, c_max=1024,
                       fanout=(10, 3), k=2, l_max=64, n_queries=1000)
    X = synth.gen_points(cfg)
    Q = synth.gen_queries(cfg)
    ds = O.Dataset(X, mode="exact")
    r = O.build(ds, cfg.params())
    truth, _ = O.brute_knn(ds, Q, 10)
    e = O.entry_point(ds)
    res, _ = O.beam_search(ds, r.row_ptr, r.col_idx, Q, e, 100, 10)
    assert O.recall_at(res, truth).mean() >= 0.95
    assert np.diff(r.row_ptr).max() <= 64  # degree cap
