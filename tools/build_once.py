"""One pipnn_build of a config (default C2), for ncu captures: python tools/build_once.py [CFG]"""
import sys
import torch
sys.path.insert(0, '/root/repo')
import synth
import paper_2602_21247_b200 as P
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
X = torch.from_numpy(synth.gen_points(cfg)).cuda()
b = P.Builder(X, P.build_params_from(cfg.params()), metric=cfg.metric)
b(X)
torch.cuda.synchronize()
print("ok")
