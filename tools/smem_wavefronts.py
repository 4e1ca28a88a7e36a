"""Shared-memory wavefronts by opcode (actual vs ideal = bank-conflict excess) from
`ncu -i rep --page source --csv --print-source sass`: python tools/smem_wavefronts.py file.csv [top]"""
import csv
import sys
from collections import Counter


def main(path, top=12):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    si, wi, wid, ie = (h.index('Source'), h.index('L1 Wavefronts Shared'), h.index('L1 Wavefronts Shared Ideal'),
                       h.index('Instructions Executed'))
    wf, ideal, ex = Counter(), Counter(), Counter()
    per = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        op = [o for o in r[si].split() if not o.startswith('@')]
        if not op:
            continue
        o = op[0].split('.')[0]
        try:
            w, i, e = int(r[wi] or 0), int(r[wid] or 0), int(r[ie] or 0)
        except ValueError:
            continue
        wf[o] += w
        ideal[o] += i
        ex[o] += e
        if w:
            per.append((w - i, w, i, e, r[0][-5:], r[si].strip()[:60]))
    tot = sum(wf.values())
    print(rows[0][1][:90])
    print(f"shared wavefronts {tot}, ideal {sum(ideal.values())}")
    for o, v in wf.most_common(8):
        print(f"  {o:8s} {v:>14d} {100 * v / max(1, tot):5.1f}%  ideal {ideal[o]:>14d}  executed {ex[o]}")
    print("top instructions by excess wavefronts:")
    for x in sorted(per, reverse=True)[:int(top)]:
        print(f"  excess {x[0]:>12d} actual {x[1]:>12d} ideal {x[2]:>12d} exec {x[3]:>11d} @{x[4]} {x[5]}")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
