"""Pipelined build + copies: per-build GPU time (events) and host time of each build call."""
import sys, time, torch
sys.path.insert(0, '/root/repo')
import synth, paper_2602_21247_b200 as P
cfg = synth.CONFIGS["C2"]
X = synth.gen_points(cfg)
Xh = torch.from_numpy(X).pin_memory()
Xd = Xh.cuda(); Xd2 = torch.empty_like(Xd)
params = P.build_params_from(cfg.params())
b1 = P.Builder(Xd, params); b2 = P.Builder(Xd, params)
for _ in range(3): b1(Xd); b2(Xd)
rp_h = torch.empty(cfg.n + 1, dtype=torch.int64).pin_memory()
ci_h = torch.empty(cfg.n * cfg.R, dtype=torch.int32).pin_memory()
stream = torch.cuda.current_stream(); cs = torch.cuda.Stream()
for mode in ("nocopy", "h2d_only", "d2h_only", "both"):
    K = 6
    bufs = [(Xd, b1), (Xd2, b2)]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    ev_b = [torch.cuda.Event() for _ in range(K)]
    ev_h = [torch.cuda.Event() for _ in range(K)]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    host = []
    for i in range(K):
        xd, b = bufs[i % 2]
        if mode in ("h2d_only", "both") and i + 1 < K:
            with torch.cuda.stream(cs):
                if i >= 1: cs.wait_event(ev_b[i - 1])
                bufs[(i + 1) % 2][0].copy_(Xh, non_blocking=True)
                ev_h[i + 1].record(cs)
        if i > 0 and mode in ("h2d_only", "both"):
            stream.wait_event(ev_h[i])
        h0 = time.perf_counter()
        evs[i][0].record(stream); o = b(xd); evs[i][1].record(stream); ev_b[i].record(stream)
        host.append((time.perf_counter() - h0) * 1e3)
        if mode in ("d2h_only", "both"):
            with torch.cuda.stream(cs):
                cs.wait_event(ev_b[i]); ci_h[: o.n_edges].copy_(o.col_idx, non_blocking=True)
    torch.cuda.synchronize(); wall = (time.perf_counter() - t0) * 1e3
    print(mode, "wall/step %.2f" % (wall / K), "build ms", [round(a.elapsed_time(b_), 2) for a, b_ in evs], "host ms", [round(h, 2) for h in host])
