"""Production-shape launch checker (test infrastructure).

Runs the engine's real forward + backward at a given input shape (config 2: 2 x 16 x 1152 x 768)
and then checks EVERY conv launch of that step against float64 arithmetic on the same bf16
operands the launch read -- the reference's conv arithmetic (pkg/src/deskdl/model/
_kernels_py.py:44-83: same padding, TF split, stride 1, dilation) and VJP rules (ops.py:152-203)
-- on sampled pixels / channels:

* forward   y(p, :) = act(sum_taps x(p + off) W_tap + b + residual(p)) at sampled pixels, all
            output channels (a conv over a nearest upsampling reads the low-resolution input;
            the stem reads the original input);
* input     grad(R)(p, :) for every gradient buffer root R = the sum over every consumer of
  gradient  every tensor stored in R of its VJP contribution (conv dgrad over the consumer's
            stored, relu-masked output gradient; residual pass-through; avgpool / nearest
            upsample VJPs, recursing through a never-materialised upsample), compared after
            the relu mask where the engine stores masked gradients;
* weight    dW[tap, ci, co] = sum over ALL N*H*W pixels of x(p + off)[ci] * gy(p)[co] and
  gradient  db[co] = sum gy(p)[co] at sampled (tap, ci, co) -- the split-K launches and their
            fixed-order reduction at full K;
* CE        dlogits at sampled pixels from the fp32 logits (loss.py:80-92).

Returns a list of rows (kind, name, launch path, shape, metric) with the reference's metric
max|a-b| / max|b| (pkg/tests/test_kernels.py:17-19) over the samples.
"""

from __future__ import annotations

import numpy as np
import torch

F64 = torch.float64


def _rel(a, b):
    a = a.to(F64)
    b = b.to(F64)
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


class Checker:
    def __init__(self, net, eng, x_nchw: torch.Tensor, labels: torch.Tensor, cw, seed=0, pixels=48):
        self.net, self.eng, self.p = net, eng, eng.plan
        self.x_nhwc = x_nchw.permute(0, 2, 3, 1).to(torch.bfloat16).to(F64).contiguous()
        self.labels = labels
        self.cw = torch.as_tensor(np.asarray(cw, np.float64), device=eng.device)
        self.gen = torch.Generator(device="cpu").manual_seed(seed)
        self.npix = pixels
        self.users = {}
        for o in self.p.ops:
            for t in list(o.ins) + ([o.res] if o.kind in ("conv", "bn") and o.res else []):
                self.users.setdefault(t, []).append(o)
        self.rows = []

    # ------------------------------------------------------------------ operands
    def maskable(self, t):
        prod = self.p.producer.get(t)
        if prod is None or t == self.p.logits_name:
            return False
        if prod.kind in ("conv", "bn"):
            return prod.relu
        if prod.kind == "pool" or (prod.kind == "up" and prod.mode == "nearest"):
            return self.maskable(prod.ins[0])
        if prod.kind == "concat":
            return all(self.maskable(s) for s in prod.ins)
        return False

    def act(self, t, n, y, x):
        """fp64 activation of tensor t at integer pixel coordinates (zero outside the image)."""
        shp = self.p.shapes[t]
        h, w = shp[2], shp[3]
        ok = (y >= 0) & (y < h) & (x >= 0) & (x < w)
        yc, xc = y.clamp(0, h - 1), x.clamp(0, w - 1)
        if t == "x":
            v = self.x_nhwc[n, yc, xc]
        elif t in self.eng.dead_up:     # never materialised: read its nearest-upsampling source
            up = self.p.producer[t]
            return self.act(up.ins[0], n, torch.div(y, up.factor, rounding_mode="floor"),
                            torch.div(x, up.factor, rounding_mode="floor")) * ok[..., None]
        else:
            v = self.eng.v(t).tensor()[n, yc, xc].to(F64)
        return v * ok[..., None]

    def wt(self, name, exact=False):
        """Weight operand as the kernels read it: HWIO [kh*kw, cin, cout] (fp64), bf16-rounded
        (exact=True: the fp32 master, which the few-output-channel head's backward reads)."""
        off, shp = self.eng.slot[name]
        n = int(np.prod(shp))
        w = self.eng.flat_w[off:off + n]
        w = (w if exact else w.to(torch.bfloat16)).to(F64)
        if len(shp) == 4:
            co, ci, kh, kw = shp
            return w.view(kh * kw, ci, co)
        return w

    def _grad_owner(self, op):
        t = op.out
        while t in self.p.grad_alias:
            t = self.p.grad_alias[t]
        return t

    def gy_at(self, op, n, y, x):
        """Output gradient the conv's dgrad consumed at pixels: the stored gradient of op.out
        (through the projection alias), times the relu mask of the tensor it belongs to."""
        shp = self.p.shapes[op.out]
        h, w = shp[2], shp[3]
        ok = (y >= 0) & (y < h) & (x >= 0) & (x < w)
        yc, xc = y.clamp(0, h - 1), x.clamp(0, w - 1)
        g = self.eng.gv(op.out).tensor()[n, yc, xc].to(F64)
        t = self._grad_owner(op)
        if self.p.producer[t].relu:
            g = g * (self.eng.v(t).tensor()[n, yc, xc] > 0)
        return g * ok[..., None]

    def gy_plane(self, op, co):
        """[N, H, W] fp64 plane of output channel co of that gradient (wgrad operand)."""
        g = self.eng.gv(op.out).tensor()[..., co].to(F64)
        t = self._grad_owner(op)
        if self.p.producer[t].relu:
            g = g * (self.eng.v(t).tensor()[..., co] > 0)
        return g

    def act_plane(self, t, ci):
        """[N, H, W] fp64 plane of channel ci of tensor t (dead upsamples expanded)."""
        if t == "x":
            return self.x_nhwc[..., ci]
        if t in self.eng.dead_up:
            up = self.p.producer[t]
            src = self.act_plane(up.ins[0], ci)
            return src.repeat_interleave(up.factor, 1).repeat_interleave(up.factor, 2)
        return self.eng.v(t).tensor()[..., ci].to(F64)

    @staticmethod
    def shifted(plane, dy, dx):
        """out[:, y, x] = plane[:, y + dy, x + dx], zero outside."""
        n, h, w = plane.shape
        out = torch.zeros_like(plane)
        y0, y1 = max(0, -dy), min(h, h - dy)
        x0, x1 = max(0, -dx), min(w, w - dx)
        if y1 > y0 and x1 > x0:
            out[:, y0:y1, x0:x1] = plane[:, y0 + dy:y1 + dy, x0 + dx:x1 + dx]
        return out

    def sample_pixels(self, t):
        n, _, h, w = self.p.shapes[t]
        k = self.npix
        ns = torch.randint(0, n, (k,), generator=self.gen)
        ys = torch.randint(0, h, (k,), generator=self.gen)
        xs = torch.randint(0, w, (k,), generator=self.gen)
        # the four corners of image 0 exercise the "same" padding of every tap
        ns[:4] = 0
        ys[:4] = torch.tensor([0, 0, h - 1, h - 1])
        xs[:4] = torch.tensor([0, w - 1, 0, w - 1])
        dev = self.eng.device
        return ns.to(dev), ys.to(dev), xs.to(dev)

    @staticmethod
    def pads(k, d):
        return ((k - 1) * d) // 2

    def path(self, op):
        e = self.eng
        if op is e.win:
            return "stem row-window (conv_halo)"
        if op.w in e.heads:
            return "head (1x1, cout<8)"
        if op.out in e.up_fprop:
            return "conv over nearest x%d upsampling (phase fprop / strided dgrad / block-sum wgrad)" % \
                e.up_fprop[op.out].factor
        return f"{op.k}x{op.k} d{op.dil} implicit GEMM"

    # ------------------------------------------------------------------ forward
    def check_forward(self, op):
        n, ys, xs = self.sample_pixels(op.out)
        k, d = op.k, op.dil
        pt = self.pads(k, d)
        w = self.wt(op.w)
        acc = torch.zeros(len(n), op.cout, dtype=F64, device=self.eng.device)
        src = op.ins[0]
        for i in range(k):
            for j in range(k):
                xin = self.act(src, n, ys + i * d - pt, xs + j * d - pt)[:, :op.cin]
                acc += xin @ w[i * k + j]
        acc += self.wt(op.b)
        if op.res:
            acc += self.act(op.res, n, ys, xs)
        if op.relu:
            acc = acc.clamp_min(0)
        got = self.eng.v(op.out).tensor()[n, ys, xs].to(F64)
        self.rows.append(("fprop", op.out, self.path(op), self.p.shapes[op.out], _rel(got, acc)))

    # ------------------------------------------------------------------ weight gradient
    def check_wgrad(self, op, samples=24):
        k, d = op.k, op.dil
        pt = self.pads(k, d)
        taps = torch.randint(0, k * k, (samples,), generator=self.gen)
        cis = torch.randint(0, op.cin, (samples,), generator=self.gen)
        cos = torch.randint(0, op.cout, (samples,), generator=self.gen)
        off, _ = self.eng.slot[op.w]
        dw = self.eng.flat_g[off:off + k * k * op.cin * op.cout].view(k * k, op.cin, op.cout)
        got, ref = [], []
        for tap, ci, co in zip(taps.tolist(), cis.tolist(), cos.tolist()):
            i, j = divmod(tap, k)
            xs = self.shifted(self.act_plane(op.ins[0], ci), i * d - pt, j * d - pt)
            ref.append((xs * self.gy_plane(op, co)).sum())
            got.append(dw[tap, ci, co].to(F64))
        self.rows.append(("wgrad", op.w, self.path(op), (k * k, op.cin, op.cout),
                          _rel(torch.stack(got), torch.stack(ref))))
        boff, _ = self.eng.slot[op.b]
        db = self.eng.flat_g[boff:boff + op.cout].to(F64)[cos]
        dref = torch.stack([self.gy_plane(op, co).sum() for co in cos.tolist()])
        self.rows.append(("bias grad", op.b, self.path(op), (op.cout,), _rel(db, dref)))

    # ------------------------------------------------------------------ input gradients
    def contrib(self, t, n, y, x):
        """Reference d loss / d t at pixels (n, y, x): sum over t's consumers' VJPs."""
        c = self.p.chans(t)
        tot = torch.zeros(len(n), c, dtype=F64, device=self.eng.device)
        for op in self.users.get(t, []):
            if op.kind == "conv" and op.ins[0] == t:
                k, d = op.k, op.dil
                pt = self.pads(k, d)
                w = self.wt(op.w, exact=op.cout < 8)
                for i in range(k):
                    for j in range(k):   # dx(q) += gy(q - off) W_tap^T
                        tot += self.gy_at(op, n, y - i * d + pt, x - j * d + pt) @ w[i * k + j].T
            if op.kind == "conv" and op.res == t:
                tot += self.gy_at(op, n, y, x)
            elif op.kind == "add":
                tot += self.grad_of(op.out, n, y, x)
            elif op.kind == "pool":
                f = op.factor
                tot += self.grad_of(op.out, n, torch.div(y, f, rounding_mode="floor"),
                                    torch.div(x, f, rounding_mode="floor")) / (f * f)
            elif op.kind == "up" and op.mode == "nearest":
                f = op.factor
                for a in range(f):
                    for b in range(f):
                        tot += self.grad_of(op.out, n, y * f + a, x * f + b)
            elif op.kind == "concat":
                pass   # t's gradient region is (part of) the concat's: checked at the root
        return tot

    def grad_of(self, t, n, y, x):
        """Gradient of t at pixels as the consumer's VJP sees it: the stored gradient, or for a
        never-materialised upsample (or an unwritten buffer) the reference sum one level down."""
        if t in self.eng.skip_up:
            return self.contrib(t, n, y, x)
        g = self.eng.gv(t).tensor()[n, y, x].to(F64)
        if self.maskable(t):
            g = g * (self.eng.v(t).tensor()[n, y, x] > 0)
        return g

    def check_root(self, root):
        members = [t for t in self.p.view_of if self.p.gview_spec(t)[0] == root and t in self.p.live
                   and t != self.p.logits_name]
        if not members or root in self.eng.skip_up or root == "x":
            return
        n, ys, xs = self.sample_pixels(root)
        cs = self.p.grad_buffers[root][3]
        ref = torch.zeros(len(n), cs, dtype=F64, device=self.eng.device)
        mask = torch.ones(len(n), cs, dtype=torch.bool, device=self.eng.device)
        for t in members:
            if t in self.p.grad_alias:
                continue
            _, off, c = self.p.gview_spec(t)
            ref[:, off:off + c] += self.contrib(t, n, ys, xs)
            if self.maskable(t):
                mask[:, off:off + c] = self.eng.v(t).tensor()[n, ys, xs] > 0
        cr = self.p.chans(root)
        got = self.eng.grad[root][n, ys, xs].to(F64)[:, :cr] * mask[:, :cr]
        ref = ref[:, :cr] * mask[:, :cr]
        prods = sorted({self.path(o) for t in members for o in self.users.get(t, []) if o.kind == "conv"})
        self.rows.append(("dgrad", root, "; ".join(prods) or "pass-through", self.p.shapes[root], _rel(got, ref)))

    # ------------------------------------------------------------------ loss
    def check_ce(self):
        t = self.p.logits_name
        n, ys, xs = self.sample_pixels(t)
        z = self.eng.v(t).tensor()[n, ys, xs].to(F64)[:, :self.p.classes]
        nb, _, h, w = self.p.shapes[t]
        lab = self.labels.to(self.eng.device).long()
        wsum = self.cw[lab].view(nb, -1).sum(1)               # per-sample sum of w_y (loss.py:80-86)
        y = lab[n, ys, xs]
        sm = torch.softmax(z, dim=1)
        sm[torch.arange(len(n)), y] -= 1
        ref = sm * (self.cw[y] / (wsum[n] * nb))[:, None]
        got = self.eng.gv(t).tensor()[n, ys, xs].to(F64)[:, :self.p.classes]
        self.rows.append(("dlogits", t, "fused weighted CE", self.p.shapes[t], _rel(got, ref)))

    def run(self):
        for op in self.eng.convs:
            self.check_forward(op)
        self.check_ce()
        for op in self.eng.convs:
            self.check_wgrad(op)
        for root in self.p.grad_buffers:
            self.check_root(root)
        return self.rows


def run_step(net, x, labels, cw):
    """Forward + backward (no update) through the model API; returns the engine."""
    loss, logits, tape = net.forward_loss(x, labels, cw)
    net.backward(tape)
    torch.cuda.synchronize()
    return tape.engine, loss, logits


def config2_batch(seed=0):
    """Config 2's inputs: 2 make_scene tiles of 16 x 1152 x 768 (trainer.py:70-79 sample stream)."""
    from paper_1810_01993_b200.scenes import SceneConfig, generated_batch
    x, lab = generated_batch(SceneConfig(height=1152, width=768), seed, 0, 0, 2)
    return torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()


def grad_table(g_test: dict, g_ref: dict, order):
    """Per-tensor max|a-b|/max|b| rows, in parameter order."""
    return [(k, float(np.max(np.abs(g_test[k].astype(np.float64) - g_ref[k])) /
                     max(float(np.max(np.abs(g_ref[k]))), 1e-30))) for k in order]
