"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import collections
import csv
import sys


def summarize(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0][:90]
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot:.2f} ms total (serialised, cold-cache)"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        lines.append(f"{v[1]:10.3f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:5d}  {k}")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarize(p))
        print()
