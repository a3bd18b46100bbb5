"""Compare every GPU activation / activation-gradient buffer with the CPU bf16 emulation."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle.bf16_emulation as E  # noqa: E402
from paper_1810_01993_b200.loss import ClassWeights  # noqa: E402
from paper_1810_01993_b200.models import deeplab_small  # noqa: E402
from paper_1810_01993_b200.net import DeepLabV3Plus  # noqa: E402

d = np.load(os.path.join("tests/golden", "deeplab_small.npz"))
net = DeepLabV3Plus(deeplab_small(), seed=5)
cw = ClassWeights((0.982, 0.017, 0.001)).vector()

# emulation with retained intermediates
store = {}
orig = E.RoundGrad.apply


def run_keep(graph, params, x, labels, cw, loss_name):
    P = {k: torch.tensor(v, requires_grad=True) for k, v in params.items()}
    vals = {"x": torch.tensor(x), "labels": torch.tensor(labels.astype(np.int64)), "class_weights": torch.tensor(cw)}
    vals.update(P)
    cons = graph.consumers()
    F = torch.nn.functional
    for nd in graph.nodes:
        ins = [vals[s] for s in nd.inputs]
        k, a = nd.kind, nd.attrs
        if k == "conv2d":
            w = ins[1].to(torch.bfloat16).float()
            xin = ins[0].to(torch.bfloat16).float() if nd.inputs[0] == "x" else ins[0]
            out = F.conv2d(xin, w, padding=(a["kh"] - 1) * a["dilation"] // 2, dilation=a["dilation"])
        elif k == "bias_add":
            out = ins[0] + ins[1].view(1, -1, 1, 1)
        elif k == "relu":
            out = torch.relu(ins[0])
        elif k == "elementwise":
            out = ins[0] + ins[1]
        elif k == "concat":
            out = torch.cat(ins, 1)
        elif k == "avgpool":
            out = F.avg_pool2d(ins[0], a["window"])
        elif k == "upsample":
            out = ins[0].repeat_interleave(a["factor"], 2).repeat_interleave(a["factor"], 3)
        elif k == "softmax_ce":
            z, lab = ins[0], ins[1]
            wy = ins[2][lab]
            nll = -torch.log_softmax(z, 1).gather(1, lab[:, None])[:, 0]
            n = z.shape[0]
            out = ((wy * nll).reshape(n, -1).sum(1) / wy.reshape(n, -1).sum(1)).mean()
        boundary = k in ("relu", "avgpool", "upsample") or (
            k in ("bias_add", "elementwise") and not any(c.kind in ("elementwise", "relu") for c in cons[nd.name])
            and nd.name != loss_name)
        if boundary and k != "softmax_ce":
            out = E.RoundGrad.apply(out)
            out.retain_grad()
            store[nd.name] = out
        vals[nd.name] = out
    vals[loss_name].backward()


run_keep(net.graph, net.params, d["x"], d["labels"], cw, net.loss_name)
loss, logits, tape = net.forward_loss(d["x"], d["labels"], cw)
net.backward(tape)
eng = tape.engine


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


for op in eng.plan.ops:
    t = op.out
    if t not in store or op.kind == "ce":
        continue
    act = eng.v(t).tensor().float().permute(0, 3, 1, 2).cpu().numpy()
    ea = store[t].detach().numpy()
    line = f"{t:24s} act {rel(act, ea):.2e}"
    if t in eng.plan.live and store[t].grad is not None:
        g = eng.gv(t).tensor().float().permute(0, 3, 1, 2).cpu().numpy()
        eg = store[t].grad.numpy()
        if eng.plan.producer[t].kind != "conv" or eng.plan.producer[t].relu or t.endswith(("pool", "up")):
            eg = eg * (ea > 0)   # GPU stores gradients of relu-derived tensors already masked
        line += f"  grad {rel(g, eg):.2e}  |g| {np.abs(eg).max():.2e}"
    print(line)
