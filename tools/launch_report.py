"""Summarise an ncu launch list (gpu__time_duration.sum) of bench.py: one step, by kernel,
and per conv launch with algorithmic TF/s (development aid; profiles/ keeps the outputs)."""
import collections
import csv
import re
import sys

sys.path.insert(0, ".")


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    return [(re.sub(r"\(.*", "", r[ki]).replace("void ", ""), float(r[vi].replace(",", "")) / 1e3)
            for r in rows[h + 1:] if len(r) > vi]


def conv_schedule():
    """The step's tcgen05 conv launches in launch order as (pass, op, h, FLOPs, bytes): fprop in op
    order, then wgrad / dgrad per backward step.  A conv over a nearest upsampling runs its forward
    as one launch per output phase, its wgrad as one 1x1 launch and its dgrad as one strided launch,
    all at the low resolution (engine.py up_fprop / up_wgrad / up_dgrad); FLOPs are executed ones."""
    from paper_1810_01993_b200.engine import Plan
    from paper_1810_01993_b200.models import DeepLabConfig, build
    from paper_1810_01993_b200.nhwc import upsampled_fprop_phases
    g, p, head, loss = build(DeepLabConfig(), 0)
    pl = Plan(g, {k: v.shape for k, v in p.items()}, (2, 16, 1152, 768), loss, head)

    def up_of(o):
        u = pl.producer.get(o.ins[0])
        return u if (u is not None and u.kind == "up" and u.mode == "nearest" and o.k % 2 == 1 and o.dil == 1
                     and not o.res and o.cout % 8 == 0) else None

    out = []
    for o in (o for o in pl.ops if o.kind == "conv"):
        n, _, h, w = pl.shapes[o.out]
        u = up_of(o)
        if u is None:
            out.append(("fprop", o, h, 2 * o.k * o.k * o.cin * o.cout * n * h * w,
                        n * h * w * (o.cin + o.cout) * 2))
            continue
        f, lo = u.factor, n * h * w // (u.factor * u.factor)
        for _, _, ka, kb, _, _, _ in upsampled_fprop_phases(o.k, f):
            out.append(("fprop", o, h, 2 * ka * kb * o.cin * o.cout * lo, lo * (o.cin + o.cout) * 2))
    for st in pl.backward_program:
        o = st["op"]
        if o.kind != "conv" or (o.k == 1 and o.cout < 8):   # head: wgrad + dgrad in head_backward
            continue
        n, _, h, w = pl.shapes[o.out]
        u = up_of(o)
        if u is None:
            out.append(("wgrad", o, h, 2 * o.k * o.k * o.cin * o.cout * n * h * w,
                        n * h * w * (o.cin + o.cout) * 2))
            if st["dx"] is not None:
                out.append(("dgrad", o, h, 2 * o.k * o.k * o.cin * o.cout * n * h * w,
                            n * h * w * (2 * o.cin + o.cout) * 2))
        else:
            f, lo = u.factor, n * h * w // (u.factor * u.factor)
            kk = o.k + f - 1
            out.append(("wgrad", o, h // f, 2 * o.k * o.k * o.cin * o.cout * lo, lo * (o.cin + o.k * o.k * o.cout) * 2))
            out.append(("dgrad", o, h // f, 2 * kk * kk * o.cin * o.cout * lo, (n * h * w * o.cout + 2 * lo * o.cin) * 2))
    return out


def main(path, which=1):
    ks = load(path)
    starts = [i for i, (k, _) in enumerate(ks) if "nchw_to_nhwc" in k]
    a = starts[which]
    b = starts[which + 1] if which + 1 < len(starts) else len(ks)
    step = ks[a:b]
    tot = sum(t for _, t in step)
    print(f"step: {len(step)} launches, {tot / 1e3:.2f} ms serialized (cold, under ncu)")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, t in step:
        agg[k][0] += 1
        agg[k][1] += t
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / 1e3:8.3f} ms {100 * t / tot:5.1f}%  n={n:4d}  {k}")
    names = conv_schedule()
    conv_launches = [(k, t) for k, t in step if k.startswith("b2::conv_")]
    print(f"\nconv launches {len(conv_launches)} (expected {len(names)})")
    rows = []
    for (kind, o, h, fl, _), (k, t) in zip(names, conv_launches):
        rows.append((t, kind, o.out, o.cin, o.cout, o.k, o.dil, h, fl / (t * 1e-6) / 1e12, k))
    tot_c = sum(r[0] for r in rows)
    print(f"conv total {tot_c / 1e3:.2f} ms")
    for r in sorted(rows, key=lambda r: -r[0])[:40]:
        print(f"{r[0]:8.1f} us {r[1]:5s} {r[2]:22s} {r[3]:4d}->{r[4]:4d} k{r[5]} d{r[6]:2d} h{r[7]:4d} "
              f"{r[8]:7.1f} TF/s  {r[9]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
