"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]
    ki, vi, mi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
            continue
        name = r[ki].split('(')[0][:60]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(',', ''))
    tot = sum(v[1] for v in agg.values())
    lines = [f"launches {sum(v[0] for v in agg.values())}  total {tot / 1e6:.3f} ms (ncu: cold-cache, serialised)"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:60s} {v[0]:6d} {v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}%  avg {v[1] / v[0] / 1e3:9.1f} us")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
