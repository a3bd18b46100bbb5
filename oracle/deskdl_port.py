"""NumPy restatement of the reference's training-step arithmetic (TEST ORACLE).

Follows pkg/src/deskdl (paths below are relative to that directory):
  conv kernels       model/_kernels_py.py:18-83   (same padding, im2col + GEMM, tap GEMMs)
  tape executor      model/ops.py:29-213          (forward rules, VJP rules, fan-out sums)
  weighted CE        model/loss.py:18-93          (per-sample weight normalisation)
  LARC / SGD         optimizer.py:48-101
  FLOP rules         flops.py:56-112
  step statistics    harness/stats.py:58-79
The executor accepts any graph object with `.inputs` (name -> role) and
`.nodes` (objects with name/kind/inputs/attrs), i.e. both the reference's
OpGraph and paper_1810_01993_b200.graph.OpGraph.
"""

from __future__ import annotations

import math

import numpy as np


# ---------------------------------------------------------------- convolution (_kernels_py.py)

def same_pads(k: int, dilation: int):
    """TF 'same' split: total (k-1)*d, before = total // 2 (_kernels_py.py:18-21)."""
    total = (k - 1) * dilation
    return total // 2, total - total // 2


def _padded(x, kh, kw, d):
    (t, b), (l, r) = same_pads(kh, d), same_pads(kw, d)
    if t == b == l == r == 0:
        return x
    return np.pad(x, ((0, 0), (0, 0), (t, b), (l, r)))


def _patches(xp, kh, kw, d, h, w):
    """im2col matrix [N*H*W, Cin*Kh*Kw], channel-major then tap (_kernels_py.py:32-41)."""
    n, c = xp.shape[:2]
    taps = [xp[:, :, i * d:i * d + h, j * d:j * d + w] for i in range(kh) for j in range(kw)]
    cols = np.stack(taps, axis=2).reshape(n, c, kh, kw, h, w)
    return np.ascontiguousarray(cols.transpose(0, 4, 5, 1, 2, 3)).reshape(n * h * w, c * kh * kw)


def conv2d_forward(x, w, stride=1, dilation=1):
    """Returns (y, cols); y = cols @ W^T reshaped to NCHW (_kernels_py.py:44-55)."""
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    n, cin, h, wd = x.shape
    cout, cin_w, kh, kw = w.shape
    if cin != cin_w:
        raise ValueError(f"conv2d: input channels {cin} != weight channels {cin_w}")
    cols = _patches(_padded(x, kh, kw, dilation), kh, kw, dilation, h, wd)
    y = cols @ w.reshape(cout, -1).T
    return np.ascontiguousarray(y.reshape(n, h, wd, cout).transpose(0, 3, 1, 2)), cols


def conv2d_backward_weights(cols, dy, w_shape, dilation=1):
    """dW = dy^T @ cols (_kernels_py.py:58-62)."""
    cout = w_shape[0]
    return (dy.transpose(0, 2, 3, 1).reshape(-1, cout).T @ cols).reshape(w_shape)


def conv2d_backward_input(dy, w, x_shape, stride=1, dilation=1):
    """Per-tap GEMMs accumulated at the tap offsets of a padded buffer (_kernels_py.py:65-83)."""
    if stride != 1:
        raise NotImplementedError("execution kernels support stride 1 only")
    n, cin, h, wd = x_shape
    cout, _, kh, kw = w.shape
    (t, _), (l, _) = same_pads(kh, dilation), same_pads(kw, dilation)
    d = dilation
    acc = np.zeros((n, cin, h + (kh - 1) * d, wd + (kw - 1) * d), dtype=dy.dtype)
    g = dy.transpose(0, 2, 3, 1).reshape(-1, cout)
    for i in range(kh):
        for j in range(kw):
            part = (g @ w[:, :, i, j]).reshape(n, h, wd, cin).transpose(0, 3, 1, 2)
            acc[:, :, i * d:i * d + h, j * d:j * d + wd] += part
    return np.ascontiguousarray(acc[:, :, t:t + h, l:l + wd])


def conv2d_loops(x, w, dilation=1):
    """Direct float64 loops, the reference tests' oracle (pkg/tests/reference.py:11-43)."""
    x = np.asarray(x, np.float64)
    w = np.asarray(w, np.float64)
    n, cin, h, wd = x.shape
    cout, _, kh, kw = w.shape
    pt = ((kh - 1) * dilation) // 2
    pl = ((kw - 1) * dilation) // 2
    out = np.zeros((n, cout, h, wd))
    for i in range(kh):
        for j in range(kw):
            for oy in range(h):
                iy = oy - pt + i * dilation
                if not 0 <= iy < h:
                    continue
                for ox in range(wd):
                    ix = ox - pl + j * dilation
                    if 0 <= ix < wd:
                        out[:, :, oy, ox] += x[:, :, iy, ix] @ w[:, :, i, j].T
    return out


# ---------------------------------------------------------------- weighted CE (loss.py)

def class_weights(frequencies, dtype=np.float32):
    """Inverse square-root class weights, computed in float64 (loss.py:18-40)."""
    f = np.asarray(frequencies, dtype=np.float64)
    if f.size < 2 or np.any(f <= 0) or abs(f.sum() - 1.0) > 1e-6:
        raise ValueError(f"bad class frequencies {frequencies}")
    return (1.0 / np.sqrt(f)).astype(dtype)


def weighted_ce_loss(logits, labels, weights):
    """(loss, dlogits) with per-sample weight normalisation (loss.py:47-93)."""
    logits = np.asarray(logits)
    c = logits.shape[1]
    w = np.asarray(weights, dtype=logits.dtype)
    if w.shape != (c,) or np.any(w <= 0):
        raise ValueError("class weights must be a positive vector of length C")
    lab = np.asarray(labels)
    if lab.shape != logits.shape[:1] + logits.shape[2:]:
        raise ValueError("labels shape does not match logits")
    lab = lab.astype(np.int64)
    if lab.size and (lab.min() < 0 or lab.max() >= c):
        raise ValueError("labels outside [0, C)")
    z = np.moveaxis(logits, 1, -1)
    z = z - z.max(axis=-1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=-1, keepdims=True))
    n = lab.shape[0]
    wy = w[lab]
    wsum = wy.reshape(n, -1).sum(axis=1)
    nll = -np.take_along_axis(logp, lab[..., None], axis=-1)[..., 0]
    loss = float(((wy * nll).reshape(n, -1).sum(axis=1) / wsum).mean())
    p = np.exp(logp)
    onehot = np.zeros_like(p)
    np.put_along_axis(onehot, lab[..., None], 1, axis=-1)
    scale = wy / wsum.reshape((n,) + (1,) * (wy.ndim - 1)) / n
    g = (p - onehot) * scale[..., None]
    return loss, np.ascontiguousarray(np.moveaxis(g, -1, 1))


# ---------------------------------------------------------------- executor (ops.py)

class Tape:
    def __init__(self):
        self.values, self.caches, self.order = {}, {}, []


# ---------------------------------------------------------------- north-star extensions
# Training-mode batch normalisation and bilinear upsampling have no reference implementation
# (SURVEY §8(c) "parity unpinned" items); restated here from their definitions and pinned by
# finite differences in tests/test_oracle.py.

def batchnorm_forward(x, gamma, beta, eps):
    """y = gamma * (x - mean) / sqrt(var + eps) + beta, batch statistics over N, H, W (biased)."""
    axes = (0, 2, 3)
    mean = x.mean(axis=axes, keepdims=True)
    var = ((x - mean) ** 2).mean(axis=axes, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - mean) * rstd
    y = gamma.reshape(1, -1, 1, 1) * xhat + beta.reshape(1, -1, 1, 1)
    return y.astype(x.dtype), (xhat, rstd)


def batchnorm_backward(g, cache, gamma):
    xhat, rstd = cache
    axes = (0, 2, 3)
    m = g.shape[0] * g.shape[2] * g.shape[3]
    dbeta = g.sum(axis=axes)
    dgamma = (g * xhat).sum(axis=axes)
    dx = gamma.reshape(1, -1, 1, 1) * rstd * (g - dbeta.reshape(1, -1, 1, 1) / m
                                              - xhat * dgamma.reshape(1, -1, 1, 1) / m)
    return dx.astype(g.dtype), dgamma.astype(g.dtype), dbeta.astype(g.dtype)


def _bilinear_taps(n_in, f):
    """Per output index: (i0, i1, w0, w1) for half-pixel centres, source clamped at 0."""
    o = np.arange(n_in * f, dtype=np.float64)
    src = np.maximum((o + 0.5) / f - 0.5, 0.0)
    i0 = np.floor(src).astype(np.int64)
    i1 = np.minimum(i0 + 1, n_in - 1)
    w1 = src - i0
    return i0, i1, 1.0 - w1, w1


def bilinear_upsample(x, f):
    n, c, h, w = x.shape
    y0, y1, wy0, wy1 = _bilinear_taps(h, f)
    x0, x1, wx0, wx1 = _bilinear_taps(w, f)
    rows = x[:, :, y0, :] * wy0[None, None, :, None] + x[:, :, y1, :] * wy1[None, None, :, None]
    out = rows[:, :, :, x0] * wx0 + rows[:, :, :, x1] * wx1
    return out.astype(x.dtype)


def bilinear_upsample_backward(g, f, x_shape):
    n, c, h, w = x_shape
    y0, y1, wy0, wy1 = _bilinear_taps(h, f)
    x0, x1, wx0, wx1 = _bilinear_taps(w, f)
    gr = np.zeros((n, c, g.shape[2], w), dtype=np.float64)
    np.add.at(gr, (slice(None), slice(None), slice(None), x0), g * wx0)
    np.add.at(gr, (slice(None), slice(None), slice(None), x1), g * wx1)
    gx = np.zeros((n, c, h, w), dtype=np.float64)
    np.add.at(gx, (slice(None), slice(None), y0, slice(None)), gr * wy0[None, None, :, None])
    np.add.at(gx, (slice(None), slice(None), y1, slice(None)), gr * wy1[None, None, :, None])
    return gx.astype(g.dtype)


def _ancestors(graph, targets):
    want, keep = set(targets), []
    for nd in reversed(graph.nodes):
        if nd.name in want:
            keep.append(nd)
            want.update(nd.inputs)
    return keep[::-1]


def _fwd(nd, ins, relu_mask=None):
    k, a = nd.kind, nd.attrs
    if k == "conv2d":
        return conv2d_forward(ins[0], ins[1], a["stride"], a["dilation"])
    if k == "matmul":
        return ins[0] @ ins[1], None
    if k == "bias_add":
        return ins[0] + ins[1].reshape((1, -1) + (1,) * (ins[0].ndim - 2)), None
    if k == "relu":
        if relu_mask is not None:   # sign decisions imposed (flip-matched comparisons)
            return np.where(relu_mask, ins[0], 0).astype(ins[0].dtype), relu_mask
        return np.maximum(ins[0], 0), None
    if k == "concat":
        return np.concatenate(ins, axis=a["axis"]), None
    if k == "softmax_ce":
        loss, g = weighted_ce_loss(ins[0], ins[1], ins[2])
        return np.array([loss], dtype=ins[0].dtype), g
    if k == "avgpool":
        f = a["window"]
        n, c, h, w = ins[0].shape
        return ins[0].reshape(n, c, h // f, f, w // f, f).mean(axis=(3, 5)), None
    if k == "upsample":
        f = a["factor"]
        return ins[0].repeat(f, axis=2).repeat(f, axis=3), None
    if k == "batchnorm":
        return batchnorm_forward(ins[0], ins[1], ins[2], a["eps"])
    if k == "upsample_bilinear":
        return bilinear_upsample(ins[0], a["factor"]), None
    if k == "elementwise":
        fn = a["fn"]
        if fn == "add":
            return ins[0] + ins[1], None
        if fn == "mul":
            return ins[0] * ins[1], None
        return ins[0] * ins[0].dtype.type(a.get("alpha", 1.0)), None
    raise AssertionError(k)


def _bwd(nd, ins, out, cache, g, need):
    k, a = nd.kind, nd.attrs
    if k == "conv2d":
        gw = conv2d_backward_weights(cache, g, ins[1].shape, a["dilation"]) if need[1] else None
        gx = conv2d_backward_input(g, ins[1], ins[0].shape, a["stride"], a["dilation"]) \
            if need[0] else None
        return gx, gw
    if k == "matmul":
        return (g @ ins[1].T if need[0] else None,
                ins[0].reshape(-1, ins[0].shape[-1]).T @ g.reshape(-1, g.shape[-1]) if need[1] else None)
    if k == "bias_add":
        axes = tuple(i for i in range(g.ndim) if i != 1)
        return (g if need[0] else None), (g.sum(axis=axes) if need[1] else None)
    if k == "relu":
        m = (out > 0) if cache is None else cache
        return (m * g if need[0] else None,)
    if k == "concat":
        cuts = np.cumsum([x.shape[a["axis"]] for x in ins[:-1]])
        return tuple(p if q else None for p, q in zip(np.split(g, cuts, axis=a["axis"]), need))
    if k == "softmax_ce":
        return (cache * cache.dtype.type(g.reshape(-1)[0]) if need[0] else None), None, None
    if k == "avgpool":
        f = a["window"]
        return (g.repeat(f, axis=2).repeat(f, axis=3) / (f * f) if need[0] else None,)
    if k == "upsample":
        f = a["factor"]
        n, c, h, w = g.shape
        return (g.reshape(n, c, h // f, f, w // f, f).sum(axis=(3, 5)) if need[0] else None,)
    if k == "batchnorm":
        gx, gg, gb = batchnorm_backward(g, cache, ins[1])
        return (gx if need[0] else None, gg if need[1] else None, gb if need[2] else None)
    if k == "upsample_bilinear":
        return (bilinear_upsample_backward(g, a["factor"], ins[0].shape) if need[0] else None,)
    if k == "elementwise":
        fn = a["fn"]
        if fn == "add":
            return (g if need[0] else None, g if need[1] else None)
        if fn == "mul":
            return (g * ins[1] if need[0] else None, g * ins[0] if need[1] else None)
        return (g * g.dtype.type(a.get("alpha", 1.0)) if need[0] else None,)
    raise AssertionError(k)


def run_forward(graph, values, targets=None, relu_masks=None):
    """Tape forward over the ancestor closure of targets (ops.py:44-70).

    relu_masks (test use only): {relu node: boolean NCHW mask} imposes the on/off decision of
    those relus (forward and VJP), so two implementations can be compared without the relu
    sign flips that round-off at near-zero pre-activations causes."""
    if targets is None:
        targets = [nd.name for nd in graph.nodes]
    tape = Tape()
    tape.values.update({k: np.asarray(v) for k, v in values.items()})
    masks = relu_masks or {}
    for nd in _ancestors(graph, targets):
        out, cache = _fwd(nd, [tape.values[s] for s in nd.inputs], masks.get(nd.name))
        tape.values[nd.name] = out
        tape.caches[nd.name] = cache
        tape.order.append(nd)
    return {t: tape.values[t] for t in targets}, tape


def run_backward(graph, tape, seed, wrt):
    """Reverse sweep with fan-out accumulation (ops.py:73-106)."""
    live = set(wrt)
    for nd in tape.order:
        if any(s in live for s in nd.inputs):
            live.add(nd.name)
    grads = {seed: np.ones_like(tape.values[seed])}
    for nd in reversed(tape.order):
        g = grads.pop(nd.name, None)
        if g is None or nd.name not in live:
            continue
        gins = _bwd(nd, [tape.values[s] for s in nd.inputs], tape.values[nd.name],
                    tape.caches[nd.name], g, [s in live for s in nd.inputs])
        for s, gi in zip(nd.inputs, gins):
            if gi is not None:
                grads[s] = grads[s] + gi if s in grads else gi
    return {n: grads.get(n) for n in wrt}


# ---------------------------------------------------------------- optimizer (optimizer.py)

def larc_effective_lr(w, g, lr=1.0, trust=0.02, weight_decay=0.0, eps=1e-8):
    """min(trust*|w|/(|g|+wd*|w|), lr); lr when |w|==0 or denom<eps (optimizer.py:48-63)."""
    wn = float(np.linalg.norm(np.asarray(w, np.float32)))
    gn = float(np.linalg.norm(np.asarray(g, np.float32)))
    if not (math.isfinite(wn) and math.isfinite(gn)):
        raise FloatingPointError("non-finite norm in LARC")
    if wn == 0.0:
        return lr
    den = gn + weight_decay * wn
    if den < eps:
        return lr
    return min(trust * wn / den, lr)


def sgd_step(w, m, g, lr_eff, momentum=0.9, weight_decay=0.0):
    """In place: m = beta*m + g (+ wd*w); w -= f32(lr_eff)*m (optimizer.py:66-76)."""
    g = np.asarray(g, np.float32)
    m *= np.float32(momentum)
    m += g
    if weight_decay:
        m += np.float32(weight_decay) * w
    w -= np.float32(lr_eff) * m


def larc_sgd_step(w, m, g, lr=1.0, momentum=0.9, trust=0.02, weight_decay=0.0, eps=1e-8):
    r = larc_effective_lr(w, g, lr, trust, weight_decay, eps)
    sgd_step(w, m, g, r, momentum, weight_decay)
    return r


# ---------------------------------------------------------------- FLOPs and statistics

def graph_flops(graph, shapes) -> int:
    """Forward FLOPs with flops.py:56-74 rules given every node's output shape."""
    total = 0
    for nd in graph.nodes:
        out = math.prod(shapes[nd.name])
        if nd.kind == "conv2d":
            a = nd.attrs
            total += 2 * a["kh"] * a["kw"] * a["cin"] * out
        elif nd.kind in ("bias_add", "relu", "elementwise"):
            total += out
        elif nd.kind == "avgpool":
            total += nd.attrs["window"] ** 2 * out
        elif nd.kind == "softmax_ce":
            total += 5 * math.prod(shapes[nd.inputs[0]])
        elif nd.kind == "matmul":
            total += 2 * shapes[nd.inputs[0]][-1] * out
    return total


def sustained(rates_per_step, warmup=1):
    """(median, p16, p84) of the per-step rank-mean series, first `warmup` dropped (stats.py:58-79)."""
    s = np.asarray([float(np.mean(r)) for r in rates_per_step], dtype=np.float64)
    if len(s) > warmup:
        s = s[warmup:]
    return float(np.median(s)), float(np.percentile(s, 16.0)), float(np.percentile(s, 84.0))


# ---------------------------------------------------------------- one full step

def train_step(graph, params, param_order, x, labels, cw, loss_name, logits_name, opt=None,
               moms=None, relu_masks=None):
    """forward_loss + backward + per-tensor LARC (net.py:132-146, trainer.py:364-387).

    Updates params / moms in place when `opt` is given; returns (loss, logits, grads, lrs).
    """
    vals = dict(params)
    vals.update(x=x, labels=labels, class_weights=cw)
    out, tape = run_forward(graph, vals, targets=[loss_name, logits_name], relu_masks=relu_masks)
    grads = run_backward(graph, tape, loss_name, wrt=param_order)
    lrs = {}
    if opt is not None:
        for name in param_order:
            lrs[name] = larc_sgd_step(params[name], moms[name], grads[name], **opt)
    return float(out[loss_name][0]), out[logits_name], grads, lrs
