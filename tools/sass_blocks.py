"""Per-block instruction/stall shares of one kernel from `ncu -i rep --page source --csv --print-source sass`:
python tools/sass_blocks.py file.csv [kernel-substring] [min-share]"""
import csv
import sys
from collections import Counter


def sections(path):
    rows = list(csv.reader(open(path)))
    out, cur, name = [], None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            name = r[1]
            continue
        if r and r[0] == "Address":
            cur = (name, r, [])
            out.append(cur)
            continue
        if cur and len(r) == len(cur[1]):
            cur[2].append(r)
    return out


def main(path, sub="", thr=0.01):
    for name, h, data in sections(path):
        if sub not in (name or ""):
            continue
        ix = {n: i for i, n in enumerate(h)}
        ie = [int(r[ix["Instructions Executed"]] or 0) for r in data]
        sm = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
        tot, ts = sum(ie), sum(sm)
        print(f"== {name[:90]}\n   warp instructions {tot}, stall samples {ts}")
        start = 0
        for i in range(1, len(data) + 1):
            if i == len(data) or ie[i] != ie[start]:
                w, s = sum(ie[start:i]), sum(sm[start:i])
                if w > thr * tot or s > 2 * thr * ts:
                    ops = Counter()
                    for k in range(start, i):
                        src = data[k][ix["Source"]].split()
                        op = src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "")
                        ops[op.split(".")[0]] += 1
                    print(f"   {start:5d}-{i:5d} exec {ie[start]:9d} inst {100 * w / tot:5.1f}% stall {100 * s / max(1, ts):5.1f}%"
                          f"  {ops.most_common(6)}")
                start = i


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", float(sys.argv[3]) if len(sys.argv) > 3 else 0.01)
