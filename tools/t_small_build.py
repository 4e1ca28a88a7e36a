import time, sys
t0=time.time()
import torch, numpy as np
sys.path.insert(0,'/root/repo')
import synth, paper_2602_21247_b200 as P
print("import", time.time()-t0, flush=True)
cfg = synth.C2.scaled(4000, n_centres=40)
X = synth.gen_points(cfg)
params = cfg.params(); params.update(c_max=256, p_den=256, c_min=40, R=32, l_max=64)
Xd = torch.from_numpy(X).cuda(); torch.cuda.synchronize()
print("data", time.time()-t0, flush=True)
out = P.pipnn_build(Xd, P.build_params_from(params)); torch.cuda.synchronize()
print("build", time.time()-t0, out.n_edges, flush=True)
