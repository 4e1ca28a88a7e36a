"""Partition experiment: time pipnn_partition on a config (CFG, default C2) for each PIPNN_DEBUG_EPI value on the
command line; bit 64 prints the dist_topk wait profile summed over the partition's launches."""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth
import paper_2602_21247_b200 as P
cfg = getattr(synth, os.environ.get("CFG", "C2"))
X = torch.from_numpy(synth.gen_points(cfg)).cuda()
pp = P.partition_params(c_max=cfg.c_max, fanout=cfg.fanout, seed=cfg.seed)
for dbg in (sys.argv[1:] or ["0", "64"]):
    os.environ["PIPNN_DEBUG_EPI"] = dbg
    ts = []
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        off, ids = P.pipnn_partition(X, pp, metric=cfg.metric)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    line = f"dbg {dbg} partition ms min {min(ts):.3f} med {sorted(ts)[2]:.3f}"
    if int(dbg) & 64:
        buf = (ctypes.c_ulonglong * 16)()
        P._lib.pipnn_debug_dt_prof(buf)
        v = [b / 5 / 148 for b in buf]
        line += (f" | dist_topk per SM: epi total {v[9]:.0f} wait {v[8]:.0f} out {v[11]:.0f}, mma wait acc {v[5]:.0f},"
                 f" appends/row {buf[15] / max(1, buf[3]):.2f}")
    print(line, flush=True)
