import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O, synth
import paper_2602_21247_b200 as P
from tests.helpers import check_candidate_lists_float
from tests.test_gpu_leaf_pick import random_leaves, EDGE_SIZES

for metric, d in [("mips", 200), ("l2", 200), ("mips", 96)]:
    for k in [1, 2, 3, 4, 5]:
        X = synth.gen_uniform(6000, d, "f32", seed=d)
        off, ids = random_leaves(len(X), [5, 40, 100, 300, 1000], seed=2)
        nbr, dist = P.pipnn_leaf_pick(torch.from_numpy(X).cuda(), torch.from_numpy(off).cuda(),
                                      torch.from_numpy(ids.view(np.int32)).cuda(), k, metric)
        nbr = nbr.cpu().numpy().view(np.uint32); dist = dist.cpu().numpy()
        onbr, odist = O.leaf_pick(O.Dataset(X, metric=metric, mode="bf16"), off, ids, k)
        bad = (nbr == 0xFFFFFFFF) != (onbr == 0xFFFFFFFF)
        print(metric, d, k, "missing", bad.sum(), "rows differ", (nbr != onbr).any(1).sum(), flush=True)
cfg = synth.CONFIGS["C4"].scaled(20000)
X = synth.gen_points(cfg)
for fan in [(1,), (2,), (3,), (4,)]:
    pp = P.partition_params(c_max=cfg.c_max, fanout=fan, seed=cfg.seed)
    try:
        goff, gids = P.pipnn_partition(torch.from_numpy(X).cuda(), pp, metric="mips")
        print("partition mips fanout", fan, "ok", len(goff) - 1)
    except Exception as e:
        print("partition mips fanout", fan, "FAIL", e)
    try:
        goff, gids = P.pipnn_partition(torch.from_numpy(X).cuda(), pp, metric="l2")
        print("partition l2 fanout", fan, "ok", len(goff) - 1)
    except Exception as e:
        print("partition l2 fanout", fan, "FAIL", e)
