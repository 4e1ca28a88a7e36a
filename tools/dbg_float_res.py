"""Debug: where do the float build's reservoirs differ from the oracle's Alg. 3 over the build's own lists?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, synth
import paper_2602_21247_b200 as P
from tests.helpers import UINT32_MAX
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = synth.CONFIGS[name]; n = 10000 if name == "C1" else 20000
cfg = cfg.scaled(n) if cfg.n != n else cfg
X = synth.gen_points(cfg); Xd = torch.from_numpy(X).cuda(); p = cfg.params()
b = P.Builder(Xd, P.build_params_from(p), metric=cfg.metric); out = b(Xd); torch.cuda.synchronize()
bufs = {kk: v.cpu().numpy() for kk, v in b.debug_buffers(Xd, out.stats).items()}
off, ids = bufs["leaf_off"], bufs["leaf_ids"].view(np.uint32)
sizes = np.diff(off); start = np.repeat(off[:-1], sizes)
cols = bufs["cols"].view(np.uint16).astype(np.int64); valid = cols != 0xFFFF
nbr_g = np.where(valid, ids[np.where(valid, start[:, None] + cols, 0)], UINT32_MAX).astype(np.uint32)
dist_g = bufs["dist"]
ds = O.Dataset(X, metric=cfg.metric, mode="bf16")
S = O.sketch(ds, O.hyperplanes(cfg.m, cfg.d, cfg.seed))
own, cand, dd = O.bidirected_edges(ids, nbr_g, dist_g.astype(np.float64))
so, co, ok = O.hashprune(len(X), S, cfg.l_max, own, cand, dd)
sg, cg = bufs["slots"].view(np.uint64), bufs["count"].view(np.uint32)
bad = [u for u in range(len(X)) if not np.array_equal(sg[u, :co[u]], so[u, :co[u]])]
print("differing owners", len(bad), "of", len(X))
def dec(s): return (int(s >> 48), hex(int((s >> 32) & 0xFFFF)), int(s & 0xFFFFFFFF))
for u in bad[:3]:
    g = set(sg[u, :co[u]].tolist()); o = set(so[u, :co[u]].tolist())
    print("u", u, "gpu-only", [dec(x) for x in sorted(g - o)], "oracle-only", [dec(x) for x in sorted(o - g)])
    m = own == u
    for v in set(int(x & 0xFFFFFFFF) for x in (g ^ o)):
        sel = m & (cand == v)
        print("   edges to", v, dd[sel])
for u in bad[:2]:
    print(u, co[u], "edges", int((own == u).sum()))
    print(" gpu", [dec(x) for x in sg[u, :co[u]]][:12])
    print(" ora", [dec(x) for x in so[u, :co[u]]][:12])
    d = np.nonzero(sg[u, :co[u]] != so[u, :co[u]])[0]
    print(" diff positions", d[:10])
