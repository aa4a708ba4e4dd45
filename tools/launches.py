"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys


def summarize(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, vi, mi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
            continue
        agg[r[ki][:90]][0] += 1
        agg[r[ki][:90]][1] += float(r[vi].replace(',', ''))
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v[1] / tot * 100:6.2f}% {v[0]:6d} {v[1] / v[0] / 1e3:9.2f}us  {k}")
    out.append(f"total {sum(v[0] for v in agg.values())} launches, {tot / 1e6:.3f} ms")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25))
