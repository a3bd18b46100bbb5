"""Per conv launch: measured time vs a roofline floor max(FLOPs / 1.6 PF, bytes / 6.0 TB/s),
summed by (kind, resolution) -- where the step loses time (development aid)."""
import collections
import sys

sys.path.insert(0, ".")
from tools.launch_report import conv_schedule, load  # noqa: E402


def main(path, which=1):
    ks = load(path)
    starts = [i for i, (k, _) in enumerate(ks) if "nchw_to_nhwc" in k]
    step = ks[starts[which]:starts[which + 1] if which + 1 < len(starts) else len(ks)]
    names = conv_schedule()
    cl = [(k, t) for k, t in step if "conv_" in k and "kernel" in k]
    rows = []
    for (kind, o, h, fl, by), (k, t) in zip(names, cl):
        tmin = max(fl / 1.6e15, by / 6.0e12) * 1e6
        rows.append((t - tmin, t, tmin, kind, o.out, o.cin, o.cout, o.k, h, k))
    rows.sort(reverse=True)
    print("conv launches %d, total %.2f ms, lost %.2f ms" % (len(rows), sum(r[1] for r in rows) / 1e3,
                                                          sum(r[0] for r in rows) / 1e3))
    by = collections.defaultdict(lambda: [0.0, 0.0])
    for r in rows:
        by[(r[3], r[8])][0] += r[0]
        by[(r[3], r[8])][1] += r[1]
    for k, v in sorted(by.items(), key=lambda x: -x[1][0]):
        print(f"{k[0]:5s} h{k[1]:5d}  lost {v[0]:8.1f} us of {v[1]:8.1f} us")
    for r in rows[:25]:
        print("lost %7.1f t %7.1f min %7.1f %s %-22s %4d->%4d k%d h%d  %s" % r)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
