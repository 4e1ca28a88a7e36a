"""Leaf-size statistics of a config's partition (GPU): tile and byte counts the leaf kernel works on."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2602_21247_b200 as P
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
X = torch.from_numpy(synth.gen_points(cfg)).cuda()
pp = P.partition_params(c_max=cfg.c_max, c_min=cfg.c_min, p_samp=cfg.p_samp, fanout=cfg.fanout, replicas=cfg.replicas,
                        seed=cfg.seed)
off, ids = P.pipnn_partition(X, pp, metric=cfg.metric)
s = np.diff(off.cpu().numpy())
T = -(-s // 128)
print(cfg.name, "leaves", len(s), "I", s.sum(), "mean", s.mean().round(1), "size-weighted", (s * s).sum() / s.sum())
print(" quantiles", np.percentile(s, [1, 10, 50, 90, 99]).round(), "max", s.max())
print(" sum s^2", (s.astype(np.float64) ** 2).sum(), "row blocks", T.sum(), "tiles T^2", (T * T).sum(),
      "pass-1 tiles", (T * np.minimum(T, 3)).sum())
padded = (T * 128 * (-(-s // 32) * 32)).sum()
print(" padded elements (pass 2)", padded, "ratio to s^2", padded / (s.astype(np.float64) ** 2).sum())
for lim in (512, 1024, 1536, 1792, 2048):
    print(f"  instances in leaves <= {lim}: {s[s <= lim].sum() / s.sum():.3f}")
