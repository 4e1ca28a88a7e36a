"""Two pipnn_builds of a config (the second one timed, warm): python tools/build_twice.py [CFG]"""
import sys, time
import torch
sys.path.insert(0, '/root/repo')
import synth
import paper_2602_21247_b200 as P
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
X = torch.from_numpy(synth.gen_points(cfg)).cuda()
b = P.Builder(X, P.build_params_from(cfg.params()), metric=cfg.metric)
b(X)
torch.cuda.synchronize()
print("---- second build", file=sys.stderr, flush=True)
t0 = time.time()
b(X)
torch.cuda.synchronize()
print("ok %.1f ms" % (1e3 * (time.time() - t0)))
