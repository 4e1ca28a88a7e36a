"""Leaf-kernel experiment: time pipnn_leaf_pick on a config's leaves under PIPNN_DEBUG_EPI (set in the environment;
the library reads it once per process). Bits 0-3: 1 = epilogue skips all tile processing, 2 = skips pass 2;
bit 64: wait profile. CFG=C3|C4|... selects the config (L2 metric)."""
import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth
import paper_2602_21247_b200 as P
cfg = getattr(synth, os.environ.get("CFG", "C2"))
X = torch.from_numpy(synth.gen_points(cfg)).cuda()
# the partition is computed without the debug knobs (read once per process by the library) and cached on disk
cache = f"/tmp/leafexp_{cfg.name}.pt"
if os.path.exists(cache):
    off, ids = (t.cuda() for t in torch.load(cache))
else:
    import subprocess
    subprocess.check_call([sys.executable, "-c", f"""
import sys, torch; sys.path.insert(0, '/root/repo'); import synth, paper_2602_21247_b200 as P
cfg = synth.{cfg.name}; X = torch.from_numpy(synth.gen_points(cfg)).cuda()
pp = P.partition_params(c_max=cfg.c_max, c_min=cfg.c_min, p_samp=cfg.p_samp, fanout=cfg.fanout, seed=cfg.seed)
off, ids = P.pipnn_partition(X, pp); torch.save((off.cpu(), ids.cpu()), '{cache}')"""],
                          env={k: v for k, v in os.environ.items() if not k.startswith("PIPNN_")})
    off, ids = (t.cuda() for t in torch.load(cache))
ref = None
for dbg in (sys.argv[1:] or [os.environ.get("PIPNN_DEBUG_EPI", "0")]):  # (the knob is read once: one value per run)
    ts = []
    for rep in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        nbr, dist = P.pipnn_leaf_pick(X, off, ids, cfg.k)
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    same = ""
    if (int(dbg) & 15) == 0:
        if ref is None: ref = nbr.clone()
        same = "same" if torch.equal(ref, nbr) else "DIFFERENT"
    h = int((nbr.to(torch.int64) * torch.arange(1, nbr.numel() + 1, device=nbr.device).view(nbr.shape)).sum().item())
    if int(dbg) & 64:
        import ctypes
        buf = (ctypes.c_ulonglong * 16)()
        P._lib.pipnn_debug_dt_prof(buf)
        v = [b / 5 / 148 for b in buf]  # per launch, per SM (producer/MMA: one lane each of 2 pipelines)
        print("  mma: tile issue (excl. ring waits) %.0f, item head %.0f | epi: pass-2 appends per row %.2f" % (v[12], v[13], buf[15] / max(1, buf[3])))
        print("  prod: wait A %.0f, wait ring-empty %.0f, total %.0f | mma: wait A %.0f, wait acc-empty %.0f, "
              "wait ring-full %.0f, total %.0f | epi: wait acc-full %.0f, output %.0f, total %.0f, tiles %.0f (cycles/SM/launch)"
              % (v[0], v[1], v[2], v[4], v[5], v[6], v[7], v[8], v[11], v[9], v[10]))
    print("P1", os.environ.get("PIPNN_P1", "-"), "hash", h % 1000003, "dbg", dbg, "leaf_pick ms (gather + kernel) min %.3f med %.3f" % (min(ts), sorted(ts)[2]), same, flush=True)
