"""Kernel timeline of one pipnn_build (torch.profiler / CUPTI): per-kernel GPU time and the idle gaps between
consecutive kernels on the device, grouped by build stage. python tools/timeline.py [CFG]"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth
import paper_2602_21247_b200 as P
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
X = torch.from_numpy(synth.gen_points(cfg)).cuda()
b = P.Builder(X, P.build_params_from(cfg.params()), metric=cfg.metric)
for _ in range(3):
    b(X)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    b(X)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev])
t0 = ks[0][0]
busy = sum(e - s for s, e, _ in ks)
span = ks[-1][1] - t0
print(f"kernels+copies {len(ks)}, span {span/1e3:.3f} ms, busy {busy/1e3:.3f} ms, idle {(span-busy)/1e3:.3f} ms")
gaps = []
for (s0, e0, n0), (s1, e1, n1) in zip(ks, ks[1:]):
    g = s1 - e0
    if g > 5:
        gaps.append((g, n0[:50], n1[:50], (e0 - t0) / 1e3))
gaps.sort(reverse=True)
for g, a, b_, at in gaps[:25]:
    print(f"  gap {g:7.1f} us at {at:7.3f} ms: {a} -> {b_}")
agg = {}
for s, e, n in ks:
    k = n.split('(')[0][:60]
    agg[k] = agg.get(k, 0) + (e - s)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:20]:
    print(f"  {v/1e3:8.3f} ms  {k}")
if os.environ.get("TL_SEQ"):
    lim = float(os.environ["TL_SEQ"])
    for s, e, n in ks:
        if (s - t0) / 1e3 > lim:
            break
        print(f"  {(s - t0)/1e3:7.3f} +{(e - s):7.1f} us  {n[:70]}")
