"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, mean duration and share of the total."""
import collections
import csv
import sys


def summarise(path, skip_names=()):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("<unnamed>::", "")
        if any(s in name for s in skip_names):
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] == "ns" else (v * 1000 if r[ui] == "ms" else v)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':70s} {'launches':>8s} {'mean us':>10s} {'share':>7s}"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{n[:70]:70s} {c:8d} {t / c:10.1f} {t / tot:7.3f}")
    out.append(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], skip_names=sys.argv[2:]))
