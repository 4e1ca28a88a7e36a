"""Hot SASS regions from `ncu -i rep --page source --csv --print-source sass`: python tools/sass_hot.py f.csv [N]
Prints instruction-executed share per block of consecutive addresses and the top instructions by stall samples."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ai, si, ie, samp, ti = (h.index("Address"), h.index("Source"), h.index("Instructions Executed"),
                            h.index("Warp Stall Sampling (All Samples)"), h.index("Thread Instructions Executed"))
    data = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        try:
            data.append((r[ai], r[si], int(r[ie] or 0), int(r[samp] or 0), int(r[ti] or 0)))
        except ValueError:
            pass
    tot_i = sum(d[2] for d in data)
    tot_s = sum(d[3] for d in data)
    print(f"instructions executed {tot_i}, stall samples {tot_s}")
    # windows of 16 instructions
    win = []
    for k in range(0, len(data), 16):
        w = data[k:k + 16]
        win.append((sum(x[2] for x in w), sum(x[3] for x in w), w[0][0], w[0][1]))
    for wi in sorted(win, key=lambda x: -x[1])[:int(top) // 2]:
        print(f"  win @{wi[2]} inst {100 * wi[0] / tot_i:5.1f}%  samples {100 * wi[1] / max(1, tot_s):5.1f}%  {wi[3][:60]}")
    print("top instructions by samples:")
    for d in sorted(data, key=lambda x: -x[3])[:int(top)]:
        print(f"  {d[0]} {100 * d[3] / max(1, tot_s):5.1f}% inst={d[2]:>10d} thr/inst={d[4] / max(1, d[2]):5.1f}  {d[1][:70]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
