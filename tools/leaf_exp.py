"""Leaf-kernel experiment: time pipnn_leaf_pick on the C2 leaves with PIPNN_DEBUG_EPI = 0 / 1 / 2."""
import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth
import paper_2602_21247_b200 as P
cfg = synth.C2
X = torch.from_numpy(synth.gen_points(cfg)).cuda()
pp = P.partition_params(c_max=cfg.c_max, fanout=cfg.fanout, seed=cfg.seed)
off, ids = P.pipnn_partition(X, pp)
for dbg in ["0", "1", "2", "0"]:
    os.environ["PIPNN_DEBUG_EPI"] = dbg
    for rep in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        nbr, dist = P.pipnn_leaf_pick(X, off, ids, cfg.k)
        e1.record(); torch.cuda.synchronize()
    print("dbg", dbg, "leaf_pick ms (gather + kernel)", round(e0.elapsed_time(e1), 3), flush=True)
