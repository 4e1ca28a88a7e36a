import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth
import paper_2602_21247_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
cfg = synth.CONFIGS["C3"].scaled(n) if n != 1000000 else synth.CONFIGS["C3"]
X = torch.from_numpy(synth.gen_points(cfg)).cuda()
params = P.build_params_from(cfg.params())
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    try:
        out = P.pipnn_build(X, params, metric=cfg.metric)
        torch.cuda.synchronize()
        print(i, "ok", out.n_edges, out.stats["n_leaves"], flush=True)
    except Exception as e:
        print(i, "FAIL", e, flush=True)
        break
