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
