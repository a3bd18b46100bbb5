"""Aggregate an ncu launch list (gpu__time_duration.sum CSV) by kernel over one training step:
the launches between the 1st and 2nd (or given) occurrences of a marker kernel (development aid)."""
import collections
import csv
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(r[ui], v)
        out.append((r[ki], v))
    return out


def main(path, marker="nchw_to_nhwc", which=0):
    ks = load(path)
    starts = [i for i, (k, _) in enumerate(ks) if marker in k]
    a = starts[which]
    b = starts[which + 1] if which + 1 < len(starts) else len(ks)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, t in ks[a:b]:
        agg[k.split("(")[0][:70]][0] += 1
        agg[k.split("(")[0][:70]][1] += t
    tot = sum(t for _, t in ks[a:b])
    print(f"{b - a} launches, {tot / 1e3:.2f} ms serialized")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
        print(f"{t / 1e3:8.3f} ms {100 * t / tot:5.1f}%  n={n:4d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3] or []), *(int(v) for v in sys.argv[3:4]))
