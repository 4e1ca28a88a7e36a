"""Shared comparison helpers for the GPU-vs-oracle parity tests (tolerances per SURVEY §8(c))."""
import numpy as np

UINT32_MAX = 0xFFFFFFFF


def bf16_round(X: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (RNE) -> fp64, the inputs of the float path (reading R19)."""
    u = X.astype(np.float32).view(np.uint32).astype(np.uint64)
    ub = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return ub.astype(np.uint32).view(np.float32).astype(np.float64)


def exact_dist(Xq: np.ndarray, i: np.ndarray, j: np.ndarray, metric: str) -> np.ndarray:
    """D(i, j) in fp64 on the given (already rounded) coordinates, direct form."""
    a, b = Xq[i], Xq[j]
    if metric == "mips":
        return -(a * b).sum(-1)
    return ((a - b) ** 2).sum(-1)


def dist_tol(D: np.ndarray, ni: np.ndarray, nj: np.ndarray) -> np.ndarray:
    """|D_gpu - D_oracle| <= 1e-3 |D| + 1e-6 (||x||^2 + ||y||^2)  (north_star 1e-3 relative + cancellation term)."""
    return 1e-3 * np.abs(D) + 1e-6 * (ni + nj)


def check_candidate_lists_float(X, metric, leaf_ids, nbr_g, dist_g, nbr_o, dist_o, k):
    """Float parity of candidate lists (SURVEY §8(c) tolerances):
    * every GPU distance matches the exact bf16-input distance of the same pair within tolerance;
    * per row, the symmetric difference of the id sets only holds ids whose oracle D is within tolerance
      of the row's k-th oracle distance (near-ties).  Returns (n_rows_differing, n_rows)."""
    Xq = bf16_round(X)
    nrm = (Xq ** 2).sum(1)
    I = nbr_g.shape[0]
    pid = np.repeat(leaf_ids.astype(np.int64), k).reshape(I, k)
    valid_g = nbr_g != UINT32_MAX
    valid_o = nbr_o != UINT32_MAX
    assert np.array_equal(valid_g.sum(1), valid_o.sum(1)), "different pick counts"
    q = np.where(valid_g, nbr_g, 0).astype(np.int64)
    Dex = exact_dist(Xq, pid, q, metric)
    tol = dist_tol(Dex, nrm[pid], nrm[q])
    err = np.abs(dist_g.astype(np.float64) - Dex)
    bad = valid_g & (err > tol)
    assert not bad.any(), f"{bad.sum()} GPU distances out of tolerance, max err {err[bad].max()}"
    ndiff = 0
    for r in range(I):
        sg = set(nbr_g[r][valid_g[r]].tolist())
        so = set(nbr_o[r][valid_o[r]].tolist())
        if sg == so:
            continue
        ndiff += 1
        cnt = valid_o[r].sum()
        kth = dist_o[r][cnt - 1]
        p = int(leaf_ids[r])
        for v in sg ^ so:
            Dv = exact_dist(Xq, np.array([p]), np.array([v]), metric)[0]
            t = dist_tol(np.array([kth]), nrm[p], nrm[v])[0] * 2
            assert abs(Dv - kth) <= t, f"row {r}: id {v} differs but D={Dv} is not a near-tie of kth={kth}"
    return ndiff, I


def prune_dissim(Xq: np.ndarray, a: np.ndarray, b: np.ndarray, metric: str) -> np.ndarray:
    """The final prune's alpha-test dissimilarity D' in fp64 (R22): D for L2, 1 - cos for MIPS."""
    if metric != "mips":
        return exact_dist(Xq, a, b, metric)
    dot = (Xq[a] * Xq[b]).sum(-1)
    na, nb = np.sqrt((Xq[a] ** 2).sum(-1)), np.sqrt((Xq[b] ** 2).sum(-1))
    den = na * nb
    return np.where(den > 0, 1.0 - dot / np.where(den > 0, den, 1.0), 1.0)


def check_prune_lists_float(X, metric, slots, count, rp_g, ci_g, rp_o, ci_o, alpha=(6, 5), rel=1e-4):
    """Float parity of the final prune: the GPU's admission lists equal the oracle's (same order)
    for every point except those whose decision chain holds a near-tie: two candidates whose order keys D(u,.)
    differ by <= rel (relative, plus a cancellation term), or an alpha test an*D'(y,c) vs ad*D'(u,c) whose two
    sides differ by <= rel. Returns (n_differing, n)."""
    Xq = bf16_round(X)
    nrm = (Xq ** 2).sum(1)
    an, ad = alpha
    n = len(rp_g) - 1
    ndiff = 0
    for u in range(n):
        g = ci_g[rp_g[u]:rp_g[u + 1]].tolist()
        o = ci_o[rp_o[u]:rp_o[u + 1]].tolist()
        if g == o:
            continue
        ndiff += 1
        c = (slots[u, :count[u]] & 0xFFFFFFFF).astype(np.int64)
        uu = np.full(len(c), u, dtype=np.int64)
        Du = exact_dist(Xq, uu, c, metric)
        scale = (nrm[u] + nrm[c]) if metric != "mips" else np.sqrt(nrm[u] * nrm[c])
        tolD = rel * np.abs(Du) + 1e-6 * scale
        Ds = np.sort(Du)
        order_tie = np.any(np.diff(Ds) <= tolD.max())
        Pu = prune_dissim(Xq, uu, c, metric)
        ii, jj = np.meshgrid(np.arange(len(c)), np.arange(len(c)), indexing="ij")
        Pyc = prune_dissim(Xq, c[ii.ravel()], c[jj.ravel()], metric).reshape(len(c), len(c))
        # cancellation scale of the fp32 Gram-based values: the norms involved (L2), 1 (angular, in [0, 2])
        S = 1.0 if metric == "mips" else (nrm[c][:, None] + nrm[c][None, :] + nrm[u])
        lhs, rhs = an * Pyc, ad * Pu[None, :]
        tol = rel * (np.abs(lhs) + np.abs(rhs)) + 1e-6 * (an + ad) * S
        alpha_tie = np.any((np.abs(lhs - rhs) <= tol) & (ii != jj))
        assert order_tie or alpha_tie, f"point {u}: lists differ without a near-tie ({g} vs {o})"
    return ndiff, n


def leaders_of_root(n: int, num: int, den: int, leader_cap: int, seed: int, replica: int = 0) -> np.ndarray:
    """Depth-0 leaders of Alg. 5 per docs/DETERMINISM.md: the l ids with the smallest (mix(K0, x), x),
    K0 = mix(mix(seed, DOM_PART), r), l = min(leader_cap, max(2, ceil(num*n/den)), n); ascending ids."""
    import oracle as O

    DOM_PART = 0x5041525449544E31
    K0 = O.mix(O.mix(seed, DOM_PART), replica)
    l = min(leader_cap, max(2, -(-num * n // den)), n)
    pri = np.array([O.mix(K0, x) for x in range(n)], dtype=np.uint64)
    order = np.lexsort((np.arange(n), pri))
    return np.sort(order[:l])


def check_single_level_partition_float(X, metric, leaders, fanout, goff, gids, rel=1e-3):
    """A one-level partition (every depth-0 group <= C_max, no merging): each point's leaves on the GPU are the
    groups of its f nearest leaders by (D, leader id); where they differ from the exact fp64 (bf16-input)
    choice, every differing leader lies within tolerance of the f-th/(f+1)-th nearest leader distance
    (SURVEY §8(c) "leaf assignment"). Returns the number of points whose leader set differs."""
    Xq = bf16_round(X)
    nrm = (Xq ** 2).sum(1)
    n = len(X)
    Ld = np.stack([exact_dist(Xq, np.arange(n), np.full(n, l), metric) for l in leaders], 1)  # [n, l]
    ordr = np.lexsort((np.broadcast_to(leaders, Ld.shape), Ld), axis=1)
    exact_sets = [set(leaders[ordr[i, :fanout]].tolist()) for i in range(n)]
    # label the GPU leaves with distinct leaders, greedily by overlap with the exact groups (two leaders of one
    # tight cluster can have identical groups, so labels must be assigned one-to-one)
    trip = []
    for b in range(len(goff) - 1):
        votes = {}
        for x in gids[goff[b]:goff[b + 1]].tolist():
            for l in exact_sets[x]:
                votes[l] = votes.get(l, 0) + 1
        trip += [(-v, b, l) for l, v in votes.items()]
    lab_of, used = {}, set()
    for _, b, l in sorted(trip):
        if b not in lab_of and l not in used:
            lab_of[b] = l
            used.add(l)
    assert len(lab_of) == len(goff) - 1, "unlabelled leaves"
    member_of = {}
    for b in range(len(goff) - 1):
        for x in gids[goff[b]:goff[b + 1]].tolist():
            member_of.setdefault(x, set()).add(lab_of[b])
    ndiff = 0
    for x in range(n):
        g = member_of.get(x, set())
        if g == exact_sets[x]:
            continue
        ndiff += 1
        assert len(g) == fanout, f"point {x} in {len(g)} leaves"
        row = Ld[x]
        srt = np.sort(row)
        kth = srt[fanout - 1]
        for l in g ^ exact_sets[x]:
            Dl = row[np.searchsorted(leaders, l)]
            tol = 2 * (rel * abs(kth) + 1e-6 * (nrm[x] + nrm[l]))
            assert abs(Dl - kth) <= tol, f"point {x}: leader {l} D={Dl} is not a near-tie of the f-th {kth}"
    return ndiff
