"""TEST INFRASTRUCTURE ONLY — CPU emulation of the GPU path's bf16 rounding points.

Runs an op graph with torch autograd in fp32, rounding to bf16 exactly where the
GPU engine stores tensors: conv weights, every fused-op output activation, and
every stored activation gradient.  Compares per-tensor gradient error with an
exact fp32 run, to tell inherent bf16 error from kernel bugs.  The GPU
parity tests require the GPU's error against the reference to be no worse
than this ideal bf16-storage implementation's (tests/test_gpu_model.py).
"""
import numpy as np
import torch
import torch.nn.functional as F


HALF = torch.bfloat16   # the 16-bit storage type being emulated (torch.float16 for the fp16 build)
LOSS_SCALE = 1.0


def set_half(dtype, loss_scale=1.0):
    """Emulate another 16-bit storage type (and its static loss scale)."""
    global HALF, LOSS_SCALE
    HALF, LOSS_SCALE = dtype, float(loss_scale)


class RoundGrad(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return x.to(HALF).float()

    @staticmethod
    def backward(ctx, g):
        return g.to(HALF).float()


def run(graph, params, x, labels, cw, loss_name, emulate, stored=None):
    """stored: names of the tensors the GPU engine stores in bf16 (its fused-op outputs, e.g.
    {o.out for o in engine.Plan(...).ops}); None = the conv-bias-add-relu chain rule below."""
    P = {k: torch.tensor(v, requires_grad=True) for k, v in params.items()}
    vals = {"x": torch.tensor(x), "labels": torch.tensor(labels.astype(np.int64)), "class_weights": torch.tensor(cw)}
    vals.update(P)
    cons = graph.consumers()
    for nd in graph.nodes:
        ins = [vals[s] for s in nd.inputs]
        k, a = nd.kind, nd.attrs
        if k == "conv2d":
            w = ins[1].to(HALF).float() if emulate else ins[1]
            xin = ins[0].to(HALF).float() if (emulate and nd.inputs[0] == "x") else ins[0]
            pad = (a["kh"] - 1) * a["dilation"] // 2
            out = F.conv2d(xin, w, padding=pad, dilation=a["dilation"])
        elif k == "bias_add":
            out = ins[0] + ins[1].view(1, -1, 1, 1)
        elif k == "relu":
            out = torch.relu(ins[0])
        elif k == "elementwise" and a["fn"] == "add":
            out = ins[0] + ins[1]
        elif k == "elementwise" and a["fn"] == "mul":
            out = ins[0] * ins[1]
        elif k == "elementwise":
            out = ins[0] * float(a.get("alpha", 1.0))
        elif k == "matmul":   # parameters are read from the fp32 master by the GPU's matmul
            out = ins[0] @ ins[1]
        elif k == "concat":
            out = torch.cat(ins, 1)
        elif k == "avgpool":
            out = F.avg_pool2d(ins[0], a["window"])
        elif k == "upsample":
            out = ins[0].repeat_interleave(a["factor"], 2).repeat_interleave(a["factor"], 3)
        elif k == "upsample_bilinear":
            out = F.interpolate(ins[0], scale_factor=a["factor"], mode="bilinear", align_corners=False)
        elif k == "batchnorm":
            out = F.batch_norm(ins[0], None, None, ins[1], ins[2], training=True, eps=a["eps"])
        elif k == "softmax_ce":
            z = ins[0]
            lab = ins[1]
            wy = ins[2][lab]
            logp = torch.log_softmax(z, 1)
            nll = -logp.gather(1, lab[:, None])[:, 0]
            n = z.shape[0]
            out = ((wy * nll).reshape(n, -1).sum(1) / wy.reshape(n, -1).sum(1)).mean()
        else:
            raise AssertionError(k)
        # fused-op boundary = where the GPU stores a bf16 tensor (and its bf16 gradient)
        if stored is not None:
            boundary = nd.name in stored
        else:
            boundary = k in ("relu", "avgpool", "upsample", "upsample_bilinear") or (
                k in ("bias_add", "elementwise", "batchnorm")
                and not any(c.kind in ("elementwise", "relu") for c in cons[nd.name]) and nd.name != loss_name)
        if emulate and boundary and k != "softmax_ce":
            out = RoundGrad.apply(out)
        vals[nd.name] = out
    loss = vals[loss_name]
    (loss * LOSS_SCALE).backward()   # the fp16 build's static loss scale (gradients stored scaled)
    if LOSS_SCALE != 1.0:
        for v in P.values():
            v.grad /= LOSS_SCALE
    run.last_values = vals
    return float(loss.detach()), {k: v.grad.numpy() for k, v in P.items()}




def emulated_grads(graph, params, x, labels, cw, loss_name, stored=None):
    """(loss, grads) with bf16 storage rounding at the GPU engine's fused-op boundaries."""
    return run(graph, params, x, labels, cw, loss_name, True, stored)


def emulated_step(graph, params, x, labels, cw, loss_name, logits_name):
    """(loss, logits, grads) of the bf16-storage emulation."""
    loss, grads = run(graph, params, x, labels, cw, loss_name, True)
    return loss, run.last_values[logits_name].detach().numpy(), grads
