"""Whole-config leaf-pick parity: pipnn_leaf_pick on a config's GPU partition vs the oracle's picks on the same
leaves (uint8: bit-exact). python tools/check_leaf_full.py C2"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, synth
import paper_2602_21247_b200 as P
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
if len(sys.argv) > 2:
    cfg = cfg.scaled(int(sys.argv[2]), n_centres=cfg.n_centres)
Xh = synth.gen_points(cfg)
X = torch.from_numpy(Xh).cuda()
pp = P.partition_params(c_max=cfg.c_max, c_min=cfg.c_min, p_samp=cfg.p_samp, fanout=cfg.fanout, seed=cfg.seed)
off, ids = P.pipnn_partition(X, pp)
nbr, dist = P.pipnn_leaf_pick(X, off, ids, cfg.k)
torch.cuda.synchronize()
offh, idsh = off.cpu().numpy(), ids.cpu().numpy().view(np.uint32)
t = time.time()
onbr, odist = O.leaf_pick(O.Dataset(Xh), offh, idsh, cfg.k)
g = nbr.cpu().numpy().view(np.uint32)
bad = np.nonzero((g != onbr).any(1))[0]
dd = dist.cpu().numpy().astype(np.float64)
okd = np.isinf(odist) & np.isinf(dd) | (odist == dd)
print(cfg.name, "instances", len(g), "differing rows", len(bad), "dist mismatches", int((~okd).sum()), "oracle s", round(time.time() - t, 1))
for r in bad[:5]:
    print(" row", r, "gpu", g[r].tolist(), "oracle", onbr[r].tolist())
