"""Parity tables for DESIGN.md §7 (run on a GPU box; writes gpurun_out/parity_report.{txt,json}).

A. config 2 (2 x 16 x 1152 x 768): every conv launch of the bf16 step vs float64 on the same bf16
   operands (tests/prodshape.py), and the bf16 step's loss / logits / per-tensor gradients vs the
   fp32 engine at the same shape.
B. config 1 (1 x 16 x 288 x 192), bf16: per-tensor gradient error of the GPU vs the oracle (the
   reference's fp32 step restated, oracle/deskdl_port.py) next to the error of an ideal
   bf16-storage implementation (oracle/bf16_emulation.py) vs the same oracle; count over 2e-2.
C. config 1, fp32 engine: max per-tensor error vs the float64 oracle with and without the GPU's
   relu decisions imposed, and the number of relu flips.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import prodshape  # noqa: E402
from oracle import deskdl_port as O  # noqa: E402
from paper_1810_01993_b200.loss import ClassWeights  # noqa: E402
from paper_1810_01993_b200.models import DeepLabConfig  # noqa: E402
from paper_1810_01993_b200.net import DeepLabV3Plus  # noqa: E402
from paper_1810_01993_b200.scenes import SceneConfig, make_scene, scene_rng  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def part_a(out, lines):
    x, lab = prodshape.config2_batch()
    cw = ClassWeights((0.982, 0.017, 0.001)).vector()
    net = DeepLabV3Plus(DeepLabConfig(), seed=0)
    eng, loss, logits = prodshape.run_step(net, x, lab, cw)
    rows = prodshape.Checker(net, eng, x, lab, cw, seed=1).run()
    lines.append("A. config 2 (2x16x1152x768): every conv launch vs float64 on the same bf16 operands")
    lines.append("   metric max|a-b|/max|b| over samples (48 pixels x all channels; 24 (tap,ci,co) weight entries")
    lines.append("   summed over all N*H*W pixels)")
    worst = {}
    for kind, name, path, shape, err in rows:
        lines.append(f"   {kind:9s} {name:28s} {err:9.2e}  {str(tuple(shape)):22s} {path}")
        worst[kind] = max(worst.get(kind, 0.0), err)
    lines.append("   worst per kind: " + ", ".join(f"{k} {v:.2e}" for k, v in sorted(worst.items())))
    out["config2_launches"] = [dict(kind=k, name=n, path=p, shape=list(s), err=e) for k, n, p, s, e in rows]
    out["config2_launch_worst"] = worst
    g16 = net.backward(net.forward_loss(x, lab, cw)[2])
    net32 = DeepLabV3Plus(DeepLabConfig(), seed=0, precision="fp32")
    loss32, logits32, tape32 = net32.forward_loss(x, lab, cw)
    g32 = net32.backward(tape32)
    a, b = logits.double(), logits32.double()
    lerr = float((a - b).abs().max() / b.abs().max())
    agree = float((a.argmax(1) == b.argmax(1)).double().mean())
    tab = prodshape.grad_table(g16, g32, net.param_order)
    errs = np.array([e for _, e in tab])
    lines.append("")
    lines.append(f"A2. config 2 bf16 step vs the fp32 engine: loss {loss:.6f} vs {loss32:.6f} "
                 f"(rel {abs(loss - loss32) / abs(loss32):.2e}); logits rel {lerr:.2e}; argmax agreement {agree:.6f}")
    lines.append(f"    per-tensor gradient error (130 tensors): median {np.median(errs):.2e}, p90 "
                 f"{np.percentile(errs, 90):.2e}, max {errs.max():.2e}; over 2e-2: {int((errs > 2e-2).sum())}")
    for k, e in sorted(tab, key=lambda t: -t[1])[:10]:
        lines.append(f"      {k:28s} {e:.2e}")
    out["config2_vs_fp32"] = dict(loss_bf16=loss, loss_fp32=loss32, logits_rel=lerr, argmax_agree=agree,
                                  grad_errs=dict(tab))


def part_b(out, lines):
    from oracle.bf16_emulation import emulated_grads
    net = DeepLabV3Plus(DeepLabConfig(), seed=0)
    f, lab = make_scene(SceneConfig(channels=16, height=288, width=192), scene_rng(0, 0, 0))
    x, labels = f[None], lab[None]
    cw = O.class_weights((0.982, 0.017, 0.001))
    loss_ref, logits_ref, grads_ref, _ = O.train_step(net.graph, net.params, net.param_order, x, labels, cw,
                                                     net.loss_name, net.logits_name)
    _, emu = emulated_grads(net.graph, net.params, x, labels, cw, net.loss_name)
    loss, logits, tape = net.forward_loss(x, labels, cw)
    grads = net.backward(tape)
    gpu = {k: rel(grads[k], grads_ref[k]) for k in net.param_order}
    em = {k: rel(emu[k], grads_ref[k]) for k in net.param_order}
    ge, ee = np.array(list(gpu.values())), np.array(list(em.values()))
    ratio = ge / np.maximum(ee, 1e-30)
    lines.append("")
    lines.append("B. config 1 (1x16x288x192) bf16: per-tensor gradient error vs the oracle (fp32 reference step)")
    lines.append(f"   loss {loss:.6f} vs {loss_ref:.6f} (rel {abs(loss - loss_ref) / abs(loss_ref):.2e}); logits rel "
                 f"{rel(logits.cpu().numpy(), logits_ref):.2e}")
    lines.append(f"   GPU:       median {np.median(ge):.2e}  p90 {np.percentile(ge, 90):.2e}  max {ge.max():.2e}  "
                 f"over 2e-2: {int((ge > 2e-2).sum())}/{len(ge)}")
    lines.append(f"   bf16 emu:  median {np.median(ee):.2e}  p90 {np.percentile(ee, 90):.2e}  max {ee.max():.2e}  "
                 f"over 2e-2: {int((ee > 2e-2).sum())}/{len(ee)}")
    lines.append(f"   GPU / emu: median {np.median(ratio):.2f}  max {ratio.max():.2f}  tensors > 2x: "
                 f"{int((ratio > 2).sum())}")
    lines.append("   tensor                        GPU err   emu err   ratio")
    for k in net.param_order:
        lines.append(f"   {k:28s} {gpu[k]:9.2e} {em[k]:9.2e} {gpu[k] / max(em[k], 1e-30):6.2f}")
    out["config1_bf16"] = dict(gpu=gpu, emu=em, loss=loss, loss_ref=loss_ref)


def part_c(out, lines):
    net = DeepLabV3Plus(DeepLabConfig(), seed=0, precision="fp32")
    f, lab = make_scene(SceneConfig(channels=16, height=288, width=192), scene_rng(0, 0, 0))
    x, labels = f[None], lab[None]
    cw = O.class_weights((0.982, 0.017, 0.001))
    loss, logits, tape = net.forward_loss(x, labels, cw)
    eng = tape.engine
    grads = net.backward(tape)
    p64 = {k: v.astype(np.float64) for k, v in net.params.items()}
    masks, flips, total = {}, 0, 0
    _, free = O.run_forward(net.graph, dict(p64, x=x.astype(np.float64), labels=labels,
                                              class_weights=cw.astype(np.float64)))
    for nd in net.graph.nodes:
        if nd.kind == "relu":
            m = eng.v(nd.name).tensor().float().cpu().numpy().transpose(0, 3, 1, 2) > 0
            masks[nd.name] = m
            flips += int((m != (free.values[nd.name] > 0)).sum())
            total += m.size
    res = {}
    for tag, rm in (("unmatched", None), ("matched", masks)):
        lr, lg, gr, _ = O.train_step(net.graph, p64, net.param_order, x.astype(np.float64), labels,
                                     cw.astype(np.float64), net.loss_name, net.logits_name, relu_masks=rm)
        e = {k: rel(grads[k], gr[k]) for k in net.param_order}
        res[tag] = dict(loss_rel=abs(loss - lr) / abs(lr), logits_rel=rel(logits.cpu().numpy(), lg),
                        grad_max=max(e.values()), grad_median=float(np.median(list(e.values()))),
                        over_1e3=int(sum(v > 1e-3 for v in e.values())),
                        worst=sorted(e.items(), key=lambda t: -t[1])[:5])
    lines.append("")
    lines.append(f"C. config 1 fp32 engine vs float64 oracle: {flips} relu flips of {total} relu outputs")
    for tag, r in res.items():
        lines.append(f"   {tag:9s}: loss rel {r['loss_rel']:.2e}, logits rel {r['logits_rel']:.2e}, grad max "
                     f"{r['grad_max']:.2e}, median {r['grad_median']:.2e}, tensors over 1e-3: {r['over_1e3']}")
        for k, v in r["worst"]:
            lines.append(f"      {k:28s} {v:.2e}")
    out["config1_fp32"] = dict(flips=flips, relu_outputs=total, **res)


def main():
    torch.cuda.set_device(0)
    out, lines = {}, []
    parts = sys.argv[1:] or ["a", "b", "c"]
    for p in parts:
        {"a": part_a, "b": part_b, "c": part_c}[p](out, lines)
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_report.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "gpurun_out", "parity_report.json"), "w") as fh:
        json.dump(out, fh, indent=1, default=str)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
