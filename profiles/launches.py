"""Summarise an ncu --metrics gpu__time_duration.sum launch CSV: per-kernel
totals over the last `--last` fraction of launches (skips warm-up reps)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            h = r
            start = i + 1
            break
    else:
        raise SystemExit(f"no launches in {path}: {rows[:2]}")
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9}
    return [(r[ki].split("(")[0], float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
            for r in rows[start:] if len(r) > vi]  # nanoseconds


if __name__ == "__main__":
    data = load(sys.argv[1])
    frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    tail = data[int(len(data) * (1 - frac)):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in tail:
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v for _, v in tail)
    print(f"launches {len(tail)}  total {tot / 1e3:.1f} us")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        print(f"{t / 1e3:10.1f} us {100 * t / tot:5.1f}%  n={c:5d}  {k[:90]}")
