"""Lowering of an op graph to a static schedule of fused sm_100a launches.

The reference executes graphs node by node with a NumPy tape
(pkg/src/deskdl/model/ops.py:44-106).  Here a graph is planned once per input
shape:

* fusion      conv2d -> bias_add [-> elementwise add (residual)] [-> relu]
              becomes ONE tcgen05 implicit-GEMM launch with the bias, residual
              and relu in its epilogue; the head's bias output is written fp32.
* concat      zero-copy: producers write straight into channel slices of the
              concat buffer ("assembling layers in place");
              gradient buffers alias the same way, so the concat VJP
              (ops.py:178-182) costs nothing.
* layout      activations NHWC bf16, gradients NHWC bf16, parameters fp32 in one
              flat buffer (conv weights HWIO), bf16 packed copies per conv for
              the fprop and dgrad operands.
* backward    reverse schedule; each conv: relu VJP (in place), wgrad + bias
              grad (split-K tcgen05, straight into the flat gradient buffer),
              dgrad (tcgen05, accumulating into fan-in gradients), residual
              pass-through.  First contribution to a gradient region
              overwrites, later ones accumulate (decided at plan time).
* loss        fused weighted CE writes dlogits into the head's gradient buffer.

Every launch goes through libb2dl.so (nhwc.py); torch only allocates memory.
"""

from __future__ import annotations

import contextlib
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, nhwc
from .graph import OpGraph, infer_shapes
from .nhwc import View


def _r8(c: int) -> int:
    return (c + 7) // 8 * 8


_PITCH64 = os.environ.get("B2DL_PITCH64", "0") == "1"   # measured: no step-time change (off)


def _pitch(c: int) -> int:
    """Channel pitch of an NHWC buffer: a multiple of 8 (16-byte rows for TMA), and above 64
    channels a multiple of 64, so every 64-channel TMA box row of every pixel is one aligned
    128-byte line (e.g. the decoder's 304-channel concat: 320, no box straddling two lines)."""
    if _PITCH64 and c > 64:
        return (c + 63) // 64 * 64
    return _r8(c)


@dataclass
class Op:
    kind: str                      # conv | pool | up | concat | add | ce
    out: str
    ins: tuple
    nodes: tuple = ()
    # conv
    w: str = ""
    b: str = ""
    res: str | None = None
    relu: bool = False
    k: int = 1
    dil: int = 1
    cin: int = 0
    cout: int = 0
    # pool / upsample
    factor: int = 1
    # concat
    copy_ins: set = field(default_factory=set)
    # up: "nearest" | "bilinear"; bn: epsilon
    mode: str = "nearest"
    eps: float = 1e-5
    # scale
    alpha: float = 1.0


class Plan:
    """Static fused schedule + buffer layout for one (graph, input shape)."""

    def __init__(self, graph: OpGraph, param_shapes: dict, input_shape: tuple, loss_name: str,
                 logits_name: str):
        self.graph = graph
        self.loss_name, self.logits_name = loss_name, logits_name
        n, c, h, w = input_shape
        shapes = dict(param_shapes)
        shapes.update(x=(n, c, h, w), labels=(n, h, w))
        cls = graph.node(loss_name).attrs["classes"]
        shapes["class_weights"] = (cls,)
        self.classes = cls
        self.shapes = infer_shapes(graph, shapes)
        self.params = graph.param_names()
        self.data_inputs = [k for k, r in graph.inputs.items() if r == "data"]
        if self.data_inputs != ["x"]:
            raise NotImplementedError("engine expects exactly one data input named 'x'")
        self._fuse()
        self._place()
        self._liveness()

    # ---------------------------------------------------------------- fusion
    def _fuse(self):
        g = self.graph
        cons = g.consumers()
        idx = {nd.name: i for i, nd in enumerate(g.nodes)}
        used = set()
        ops = []
        for nd in g.nodes:
            if nd.name in used:
                continue
            if nd.kind == "conv2d":
                a = nd.attrs
                if a["stride"] != 1:
                    raise NotImplementedError("execution kernels support stride 1 only")
                if a["kh"] != a["kw"]:
                    raise NotImplementedError("square kernels only")
                chain = [nd]
                nxt = cons[nd.name]
                cur, bname = nd, ""
                if (len(nxt) == 1 and nxt[0].kind == "bias_add" and nxt[0].inputs[0] == nd.name
                        and g.inputs.get(nxt[0].inputs[1]) == "param"):
                    chain.append(nxt[0])
                    cur, bname = nxt[0], nxt[0].inputs[1]
                res = None
                relu = False
                nxt = cons[cur.name]
                if (len(nxt) == 1 and nxt[0].kind == "elementwise" and nxt[0].attrs["fn"] == "add"
                        and nxt[0].name not in used and cur.name != self.logits_name):
                    add = nxt[0]
                    other = [s for s in add.inputs if s != cur.name]
                    if len(other) == 1:
                        res = other[0]
                        chain.append(add)
                        cur = add
                        nxt = cons[cur.name]
                if (len(nxt) == 1 and nxt[0].kind == "relu" and nxt[0].name not in used
                        and cur.name != self.logits_name):
                    chain.append(nxt[0])
                    cur = nxt[0]
                    relu = True
                used.update(c.name for c in chain)
                op = Op("conv", cur.name, (nd.inputs[0],), tuple(c.name for c in chain), w=nd.inputs[1],
                        b=bname, res=res, relu=relu, k=a["kh"], dil=a["dilation"], cin=a["cin"],
                        cout=a["cout"])
                ops.append((idx[cur.name], op))
            elif nd.kind == "batchnorm":
                # training-mode batch norm, with a following residual add and relu fused into its
                # normalising pass (BN-add-relu)
                chain = [nd]
                cur = nd
                res = None
                relu = False
                nxt = cons[cur.name]
                if (len(nxt) == 1 and nxt[0].kind == "elementwise" and nxt[0].attrs["fn"] == "add"
                        and nxt[0].name not in used):
                    add = nxt[0]
                    other = [s_ for s_ in add.inputs if s_ != cur.name]
                    if len(other) == 1:
                        res = other[0]
                        chain.append(add)
                        cur = add
                        nxt = cons[cur.name]
                if len(nxt) == 1 and nxt[0].kind == "relu" and nxt[0].name not in used:
                    chain.append(nxt[0])
                    cur = nxt[0]
                    relu = True
                used.update(c.name for c in chain)
                ops.append((idx[cur.name], Op("bn", cur.name, (nd.inputs[0],), tuple(c.name for c in chain),
                                              w=nd.inputs[1], b=nd.inputs[2], res=res, relu=relu,
                                              cin=self.shapes[nd.name][1], cout=self.shapes[nd.name][1],
                                              eps=nd.attrs["eps"])))
            elif nd.kind == "upsample_bilinear":
                ops.append((idx[nd.name], Op("up", nd.name, nd.inputs, (nd.name,), factor=nd.attrs["factor"],
                                             mode="bilinear")))
            elif nd.kind == "avgpool":
                ops.append((idx[nd.name], Op("pool", nd.name, nd.inputs, (nd.name,), factor=nd.attrs["window"])))
            elif nd.kind == "upsample":
                ops.append((idx[nd.name], Op("up", nd.name, nd.inputs, (nd.name,), factor=nd.attrs["factor"])))
            elif nd.kind == "concat":
                if nd.attrs["axis"] != 1:
                    raise NotImplementedError("channel concat only")
                ops.append((idx[nd.name], Op("concat", nd.name, nd.inputs, (nd.name,))))
            elif nd.kind == "elementwise" and nd.attrs["fn"] == "add":
                ops.append((idx[nd.name], Op("add", nd.name, nd.inputs, (nd.name,))))
            # standalone lowerings (csrc/generic.cu): the op kinds outside conv-bias-relu chains
            elif nd.kind == "elementwise" and nd.attrs["fn"] == "mul":
                ops.append((idx[nd.name], Op("mul", nd.name, nd.inputs, (nd.name,))))
            elif nd.kind == "elementwise":   # scale
                ops.append((idx[nd.name], Op("scale", nd.name, nd.inputs, (nd.name,),
                                             alpha=float(nd.attrs.get("alpha", 1.0)))))
            elif nd.kind == "bias_add":
                if g.inputs.get(nd.inputs[1]) != "param":
                    raise NotImplementedError(f"{nd.name}: bias_add needs a parameter bias")
                chain = [nd]
                cur = nd
                nxt = cons[nd.name]
                relu = False
                if len(nxt) == 1 and nxt[0].kind == "relu" and nxt[0].name not in used:
                    chain.append(nxt[0])
                    cur = nxt[0]
                    relu = True
                used.update(c.name for c in chain)
                ops.append((idx[cur.name], Op("bias", cur.name, (nd.inputs[0],), tuple(c.name for c in chain),
                                              b=nd.inputs[1], relu=relu, cout=self.shapes[nd.name][1])))
            elif nd.kind == "relu":
                ops.append((idx[nd.name], Op("relu", nd.name, nd.inputs, (nd.name,))))
            elif nd.kind == "matmul":
                if g.inputs.get(nd.inputs[1]) != "param" or len(self.shapes[nd.inputs[0]]) != 4:
                    raise NotImplementedError(f"{nd.name}: matmul of a 4-D activation by a parameter only")
                ops.append((idx[nd.name], Op("matmul", nd.name, (nd.inputs[0],), (nd.name,), w=nd.inputs[1])))
            elif nd.kind == "softmax_ce":
                if nd.inputs[1:] != ("labels", "class_weights"):
                    raise NotImplementedError("softmax_ce must read the graph's labels / class_weights")
                ops.append((idx[nd.name], Op("ce", nd.name, (nd.inputs[0],), (nd.name,))))
            else:
                raise NotImplementedError(f"{nd.name}: op kind {nd.kind} has no fused lowering")
        ops.sort(key=lambda t: t[0])
        self.ops = [o for _, o in ops]
        self.producer = {o.out: o for o in self.ops}
        if self.logits_name not in self.producer or self.producer[self.logits_name].kind != "conv":
            raise NotImplementedError("logits must be produced by a conv + bias_add")

    # ---------------------------------------------------------------- buffers
    def chans(self, t):
        return self.shapes[t][1]

    def _place(self):
        owner = {}
        for op in reversed(self.ops):
            if op.kind != "concat":
                continue
            off = 0
            for s in op.ins:
                prod = self.producer.get(s)
                ok = (s not in owner and prod is not None
                      and prod.kind in ("conv", "bn", "pool", "up", "concat", "add", "bias", "relu", "mul",
                                        "scale", "matmul")
                      and s != self.logits_name and off % 8 == 0)
                if ok:
                    owner[s] = (op.out, off)
                else:
                    op.copy_ins.add(s)
                off += self.chans(s)
        self.view_of = {}
        self.buffers = {}

        def resolve(t):
            if t in self.view_of:
                return self.view_of[t]
            if t in owner:
                par, off = owner[t]
                root, poff = resolve(par)
                r = (root, poff + off)
            else:
                r = (t, 0)
            self.view_of[t] = r
            return r

        tensors = ["x"] + [o.out for o in self.ops if o.kind != "ce"]
        for t in tensors:
            root, _ = resolve(t)
            n, c, h, w = self.shapes[root]
            f32 = root == self.logits_name
            self.buffers[root] = (n, h, w, c if f32 else _pitch(c), f32)

    def view_spec(self, t):
        root, off = self.view_of[t]
        return root, off, self.chans(t)

    def gview_spec(self, t):
        """Gradient view: like the activation view, except a projection-shortcut output whose
        gradient is, by construction, the residual block's (masked) output gradient."""
        while t in self.grad_alias:
            t = self.grad_alias[t]
        return self.view_spec(t)

    # ---------------------------------------------------------------- gradients
    def _liveness(self):
        live = set(self.params)
        for op in self.ops:
            if op.kind in ("conv", "bn"):
                srcs = [op.ins[0], op.w, op.b] + ([op.res] if op.res else [])
            elif op.kind in ("bias", "matmul"):
                srcs = [op.ins[0], op.b or op.w]
            else:
                srcs = list(op.ins)
            if any(s in live for s in srcs):
                live.add(op.out)
        self.live = live
        # residual shortcuts (ops.py:197-198 passes the gradient through unchanged):
        #  * projection conv P feeding only block C's add: grad(P.out) IS grad(C.out) -> alias
        #  * identity input x: its pass-through is merged into the next dgrad writing grad(x)
        users = {}
        for op in self.ops:
            for t in list(op.ins) + ([op.res] if op.kind in ("conv", "bn") and op.res else []):
                users.setdefault(t, []).append(op)
        self.grad_alias = {}
        for op in self.ops:
            if op.kind in ("conv", "bn") and op.res:
                pr = self.producer.get(op.res)
                if (pr is not None and pr.kind in ("conv", "bn") and not pr.relu and users.get(op.res) == [op]
                        and self.view_of[op.res][0] == op.res):
                    self.grad_alias[op.res] = op.out
        self.grad_buffers = {}
        for t in live:
            if t in self.view_of:
                root = self.gview_spec(t)[0]
                n, h, w, _, _ = self.buffers[root]
                self.grad_buffers[root] = (n, h, w, _pitch(self.chans(root)))
        # static backward program: overwrite/accumulate and relu masking decided per contribution.
        # A contribution to the gradient of a "maskable" tensor (a relu output, or a pool /
        # nearest-upsample / concat of relu outputs -- all non-negative, zero exactly where every
        # underlying relu is inactive) is multiplied by (activation > 0) when it is written, so
        # the producer's relu VJP (ops.py:176-177) needs no separate pass.
        init = {root: [] for root in self.grad_buffers}
        contrib = {root: [] for root in self.grad_buffers}
        memo = {}

        def maskable(t):
            if t not in memo:
                prod = self.producer.get(t)
                if prod is None or t == self.logits_name:
                    memo[t] = False
                elif prod.kind in ("conv", "bn", "bias"):
                    memo[t] = prod.relu
                elif prod.kind == "relu":
                    memo[t] = True
                elif prod.kind == "pool" or (prod.kind == "up" and prod.mode == "nearest"):
                    memo[t] = maskable(prod.ins[0])
                elif prod.kind == "concat":
                    memo[t] = all(maskable(x) for x in prod.ins)
                else:
                    memo[t] = False
            return memo[t]

        def claim(t, masked):
            root, off, c = self.gview_spec(t)
            iv = init[root]
            lo, hi = off, off + c
            contrib[root].append((lo, hi, masked))
            covered = sum(max(0, min(hi, b) - max(lo, a)) for a, b in iv)
            if covered == 0:
                iv.append((lo, hi))
                return False
            if covered == hi - lo:
                return True
            raise NotImplementedError(f"partially initialised gradient region for {t}")

        def inited(t):
            root, off, c = self.gview_spec(t)
            return sum(max(0, min(off + c, b) - max(off, a)) for a, b in init[root]) > 0

        def unmasked_into(t):
            root, off, c = self.gview_spec(t)
            return any((not m) and min(off + c, b) > max(off, a) for a, b, m in contrib[root])

        prog = []
        pending = {}   # identity shortcut input -> block output whose gradient passes through

        def flush_pending(t):
            # a pass-through no dgrad absorbed before t's producer runs: plain masked add
            for r in [r for r in pending if r == t]:
                src = pending.pop(r)
                m = maskable(r)
                prog.append({"op": Op("add", r, (src,)), "acc": [(r, claim(r, m), m)], "passthrough": src})

        ce = [o for o in self.ops if o.kind == "ce"]
        if len(ce) != 1 or ce[0].ins[0] != self.logits_name:
            raise NotImplementedError("exactly one softmax_ce on the logits")
        claim(self.logits_name, False)                # written by the fused CE in forward
        for op in reversed(self.ops):
            if op.kind == "ce" or op.out not in self.live:
                continue
            if not inited(op.out):
                raise NotImplementedError(f"{op.out}: live tensor without gradient contributions")
            flush_pending(op.out)
            if op.kind == "conv":
                x, res = op.ins[0], op.res
                step = {"op": op, "dx": None, "dres": None, "mask_dx": False, "mask_res": False,
                        "dx_res": None, "relu_pass": op.relu and unmasked_into(op.out)}
                if x in self.live:
                    step["mask_dx"] = maskable(x)
                    gemm_dgrad = not (op.k == 1 and op.cout < 8)
                    if gemm_dgrad and x in pending:
                        step["dx_res"] = pending.pop(x)   # pass-through folded into this dgrad
                    step["dx"] = claim(x, step["mask_dx"])
                if res is not None and res in self.live and res not in self.grad_alias:
                    pending[res] = op.out
                prog.append(step)
            elif op.kind == "bn":
                x, res = op.ins[0], op.res
                step = {"op": op, "dx": None, "relu_pass": op.relu and unmasked_into(op.out)}
                if x in self.live:
                    step["dx"] = claim(x, False)     # pre-normalisation conv output: never masked
                if res is not None and res in self.live and res not in self.grad_alias:
                    pending[res] = op.out
                prog.append(step)
            elif op.kind in ("pool", "up"):
                x = op.ins[0]
                if x in self.live:
                    m = maskable(x)
                    prog.append({"op": op, "mask": m, "dx": claim(x, m)})
            elif op.kind == "concat":
                # aliased inputs share the gradient region; copied inputs get the slice added
                step = {"op": op, "copies": []}
                off = 0
                for s_ in op.ins:
                    if s_ in op.copy_ins and s_ in self.live:
                        m = maskable(s_)
                        step["copies"].append((s_, off, claim(s_, m), m))
                    off += self.chans(s_)
                prog.append(step)
            elif op.kind == "add":
                prog.append({"op": op, "acc": [(s_, claim(s_, maskable(s_)), maskable(s_))
                                               for s_ in op.ins if s_ in self.live]})
            elif op.kind == "mul":
                prog.append({"op": op, "acc": [(i, s_, claim(s_, maskable(s_)), maskable(s_))
                                               for i, s_ in enumerate(op.ins) if s_ in self.live]})
            elif op.kind in ("scale", "relu", "matmul", "bias"):
                x = op.ins[0]
                st = {"op": op, "dx": None, "mask": False,
                      "relu_pass": op.kind == "bias" and op.relu and unmasked_into(op.out)}
                if x in self.live:
                    st["mask"] = maskable(x)
                    st["dx"] = claim(x, st["mask"])
                prog.append(st)
        for r in list(pending):
            flush_pending(r)
        self.backward_program = prog
        self.relu_passes = sum(1 for st in prog if st.get("relu_pass"))


def _in_lib(fn):
    """Run an Engine method's launches on the engine's build (bf16 or fp16 storage)."""
    def wrapped(self, *a, **k):
        with _lib.use(self.half):
            return fn(self, *a, **k)
    wrapped.__name__, wrapped.__doc__ = fn.__name__, fn.__doc__
    return wrapped


def conv_event_totals(events, by_pass=False):
    """Sum (ms, FLOPs) over recorded (start, end, FLOPs, pass) conv events."""
    if not by_pass:
        return (sum(a.elapsed_time(b) for a, b, _, _ in events), sum(f for _, _, f, _ in events))
    out = {}
    for a, b, f, t in events:
        ms, fl = out.get(t, (0.0, 0))
        out[t] = (ms + a.elapsed_time(b), fl + f)
    return out


class Engine:
    """Device state + launches for one model at one input shape."""

    def __init__(self, graph: OpGraph, params: dict, param_order, input_shape, loss_name, logits_name,
                 device="cuda", precision="bf16"):
        if precision not in ("bf16", "fp16", "fp32"):
            raise ValueError(f"precision must be 'bf16', 'fp16' or 'fp32', not {precision!r}")
        # fp32: the parity mode -- fp32 NHWC buffers, fp32 HWIO weights, CUDA-core kernels
        # (b2dl.h group 3); same program, same fusion points
        self.fp32 = precision == "fp32"
        self.precision = precision
        self.device = torch.device(device)
        self.order = list(param_order)
        self.plan = Plan(graph, {k: v.shape for k, v in params.items()}, tuple(input_shape), loss_name,
                         logits_name)
        p = self.plan
        self.ws = nhwc.Workspace(self.device)
        # 16-bit storage: bf16 (libb2dl.so) or IEEE fp16 (libb2dl_f16.so, same kernels, kind::f16
        # MMAs on f16 operands; config 4's FP16); every launch of this engine goes to its build
        self.half = "fp16" if precision == "fp16" else "bf16"
        bf, f32 = (torch.float16 if precision == "fp16" else torch.bfloat16), torch.float32
        self.hdt = bf
        adt = f32 if self.fp32 else bf
        self.act = {r: torch.empty((n, h, w, c), dtype=f32 if isf else adt, device=self.device)
                    for r, (n, h, w, c, isf) in p.buffers.items()}
        self.grad = {r: torch.empty(s, dtype=adt, device=self.device) for r, s in p.grad_buffers.items()}
        # flat fp32 parameters / gradients / momentum in param order; conv weights HWIO
        self.slot = {}
        off = 0
        offsets = []
        for name in self.order:
            shp = tuple(params[name].shape)
            offsets.append(off)
            self.slot[name] = (off, shp)
            off += (int(np.prod(shp)) + 63) // 64 * 64
        offsets.append(off)
        self.numel = off
        self.flat_w = torch.zeros(off, dtype=f32, device=self.device)
        self.flat_g = torch.zeros(off, dtype=f32, device=self.device)
        self.flat_m = torch.zeros(off, dtype=f32, device=self.device)
        self.offsets = torch.tensor(offsets, dtype=torch.int64, device=self.device)
        self.convs = [o for o in p.ops if o.kind == "conv"]
        # per batch-norm op: [4][C] mean, rstd, scale, shift of the current step
        self.bn_stats = {o.out: torch.zeros(4 * o.cout, dtype=f32, device=self.device)
                         for o in p.ops if o.kind == "bn"}
        # bf16 mirror of the whole flat parameter buffer, refreshed by the LARC update itself:
        # conv kernels read it directly as their weight operand (HWIO; MN-major for fprop,
        # tap-flipped K-major for dgrad).  Only convs with cout % 8 != 0 (the 3-class head)
        # keep small packed copies.
        self.flat_wbf = torch.zeros(off, dtype=bf, device=self.device)
        self._lr_scratch = torch.zeros(len(self.order), dtype=f32, device=self.device)
        self._status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.wf, self.wd = {}, {}
        self.packed = [] if self.fp32 else [o for o in self.convs if o.cout % 8 != 0]
        for o in self.packed:
            t = o.k * o.k
            self.wf[o.w] = torch.zeros((o.cout, t, nhwc.cin_pad(o.cin)), dtype=bf, device=self.device)
            if o.ins[0] in p.live:
                self.wd[o.w] = torch.zeros((o.cin, t, nhwc.cin_pad(o.cout)), dtype=bf, device=self.device)
        # Row-window stem: when the data input feeds exactly one narrow conv (the 16-channel 7x7
        # stem), the input is stored with its horizontal padding baked in and the conv folds the
        # kw taps of a kernel row into one K run of kw*cin channels (b2dl_conv_args.window):
        # 14 64-wide K blocks instead of 49 16-wide ones.
        self.win = None
        users = [o for o in p.ops if "x" in o.ins]
        if len(users) == 1 and users[0].kind == "conv" and not self.fp32:
            o = users[0]
            if (o.k > 1 and o.dil == 1 and o.cin % 8 == 0 and 16 < o.cin * o.k <= 128 and o.cout % 8 == 0
                    and o.ins[0] == "x" and not o.res):
                n_, c_, h_, w_ = input_shape
                self.win = o
                self.xwin = torch.zeros((n_, h_, w_ + o.k - 1, c_), dtype=bf, device=self.device)
                self.wwin = torch.zeros((o.cout, o.k, nhwc.cin_pad(o.k * o.cin)), dtype=bf, device=self.device)
        # persistent split-K partial buffers (wgrad + bias column sums), reduced per bucket
        self.partials = {}
        self.segs = {}
        total, offs = 0, {}
        # few-output-channel 1x1 convs (the 3-class head): wgrad + dgrad in one pass over the input
        self.heads = set() if self.fp32 else {o.w for o in self.convs
                                              if o.k == 1 and o.cout < 8 and o.cin % 8 == 0
                                              and 256 % (o.cin // 8) == 0}
        # Conv over a nearest upsampling (DeepLab's full.c0 after the x4 full.up): the conv's input
        # gradient and the upsample's VJP are one conv over dy at LOW resolution with input stride f
        # and merged (k+f-1)^2-tap weights (b2dl_pack_upsampled_dgrad): (1 + (f-1)/k)^2 / f^2 of the
        # full-resolution dgrad's MMA work, and no full-resolution input gradient written or re-read.
        self.up_dgrad, self.wup, self.skip_up = {}, {}, set()
        if not self.fp32 and os.environ.get("B2DL_UP_DGRAD", "1") != "0":
            self._plan_up_dgrad()
        # ... and its forward per output phase from the low-resolution input with merged phase
        # weights (b2dl_pack_upsampled_fprop): 36 instead of 144 taps per 4 x 4 block for k 3, f 4
        self.up_fprop, self.wupf = {}, {}
        if not self.fp32 and os.environ.get("B2DL_UP_FPROP", "1") != "0":
            for o in self.convs:
                up = p.producer.get(o.ins[0])
                if (up is not None and up.kind == "up" and up.mode == "nearest" and 1 < up.factor <= 8
                        and o.k % 2 == 1 and o.dil == 1 and not o.res and o.cout % 8 == 0 and o.cin % 8 == 0
                        and o.out != p.logits_name and o is not self.win and o.w not in self.wf):
                    self.up_fprop[o.out] = up
                    self.wupf[o.w] = torch.zeros(nhwc.upsampled_fprop_taps(o.k, up.factor) * o.cin * o.cout,
                                                 dtype=self.hdt, device=self.device)
        # ... and its weight gradient: x_low^T (shifted f x f block sums of dy), one 1x1 wgrad at the
        # low resolution (b2dl_upsampled_wgrad_sums / _reduce).  With all three the upsampled
        # tensor itself is never formed.
        self.up_wgrad, self.gsum, self.up_layout = {}, {}, {}
        if not self.fp32 and os.environ.get("B2DL_UP_WGRAD", "1") != "0":
            for o in self.convs:
                up = self.up_fprop.get(o.out)
                if up is not None and o.k in (1, 3) and up.factor in (2, 4):
                    n_, _, h_, w_ = p.shapes[up.ins[0]]
                    self.up_wgrad[o.out] = up
                    self.gsum[o.w] = torch.empty(n_ * h_ * w_ * o.k * o.k * o.cout, dtype=self.hdt,
                                                 device=self.device)
        self.dead_up = {self.up_fprop[o].out for o in self.up_wgrad if o in self.up_dgrad}
        # Batch norm after a conv: the conv's TMA epilogue emits per-tile channel sums and sums of
        # squares of its stored output (b2dl_conv_args.bn_partial), so the BN forward is one
        # normalising pass with no statistics pass over the conv output (B2DL_BN_FUSED=0: off)
        self.bn_fused, self.bn_parts = {}, {}
        if not self.fp32 and os.environ.get("B2DL_BN_FUSED", "1") != "0":
            for o in p.ops:
                if o.kind != "bn":
                    continue
                c = p.producer.get(o.ins[0])
                if (c is not None and c.kind == "conv" and c.cout % 8 == 0 and c.cout > 16 and not c.relu
                        and not c.res and (c.cin > 16 or c is self.win)
                        and c.out not in self.up_fprop and c.out != p.logits_name and p.view_spec(c.out)[1] % 8 == 0
                        and (c.k > 1 or c.cout >= 8)):
                    self.bn_fused[c.out] = o
        # Narrow-output convs with >= 5 tap rows (the growth-32 5x5 dense layers): the row-tap fprop
        # kernel reads one tall input box per (column tap, channel block) and packed weights
        # (b2dl_conv_fprop picks it for w_packed, cout <= 64 here; B2DL_ROWTAP=0: the generic kernel)
        self.rowtap = []
        rt_min_k = int(os.environ.get("B2DL_ROWTAP_MINK", "3"))
        if not self.fp32 and os.environ.get("B2DL_ROWTAP", "1") != "0":
            for o in self.convs:
                if (o.k >= rt_min_k and o.cout <= 64 and o.cout % 8 == 0 and o.cin > 16 and o is not self.win
                        and o.out not in self.up_fprop and o.out not in self.bn_fused and o.w not in self.wf
                        and o.out != p.logits_name):
                    self.rowtap.append(o)
                    self.wf[o.w] = torch.zeros((o.cout, o.k * o.k, nhwc.cin_pad(o.cin)), dtype=bf, device=self.device)
        # ... and narrow input gradients (cin <= 128, or <= 256 over a <= 64-channel dy: the dgrad's
        # output is narrow) with >= 3 tap rows: packed dgrad weights, so b2dl_conv_fprop runs them
        # on the row-tap kernel too
        self.rowtap_dgrad = []
        rt_dg_max = int(os.environ.get("B2DL_ROWTAP_DGRAD_MAXC", "128"))
        if not self.fp32 and os.environ.get("B2DL_ROWTAP", "1") != "0":
            for o in self.convs:
                if (o.k >= rt_min_k and (o.cin <= rt_dg_max or (o.cin <= 256 and o.cout <= 64)) and o.cin % 8 == 0
                        and o.cout > 16 and o.ins[0] in p.live
                        and o is not self.win and o.w not in self.heads and o.w not in self.wd
                        and o.out not in self.up_fprop and o.out not in self.up_dgrad):
                    self.rowtap_dgrad.append(o)
                    self.wd[o.w] = torch.zeros((o.cin, o.k * o.k, nhwc.cin_pad(o.cout)), dtype=bf, device=self.device)
        # ... and its backward statistics (sum gy, sum gy * xhat) from the epilogue of the one dgrad
        # that writes d loss / d y (a single-consumer conv C; the relu mask is recomputed there from
        # the BN input), so the BN VJP is one input-gradient pass (b2dl_conv_args.bnb_partial)
        self.bnb_of, self.bnb_parts = {}, {}
        if self.bn_fused:
            users = {}
            for o in p.ops:
                for t in list(o.ins) + ([o.res] if o.kind in ("conv", "bn") and o.res else []):
                    users.setdefault(t, []).append(o)
            steps = {st["op"].out: st for st in p.backward_program if st["op"].kind == "conv"}
            for o in p.ops:
                if o.kind != "bn" or not o.relu or o.res or o.out not in p.live:
                    continue
                u = users.get(o.out, [])
                c = u[0] if len(u) == 1 else None
                st = steps.get(c.out) if c is not None else None
                if (c is not None and c.kind == "conv" and c.ins[0] == o.out and c.res != o.out and st is not None
                        and st["dx"] is False and st["mask_dx"] and not st["dx_res"] and o.cout % 8 == 0
                        and o.cout > 16
                        and p.view_spec(o.out) == (o.out, 0, o.cout) and p.gview_spec(o.out)[0] == o.out
                        and c.cout > 16 and c is not self.win and c.w not in self.heads
                        and c.out not in self.up_dgrad):
                    self.bnb_of[c.out] = o
        hparts = nhwc.head_backward_parts()
        for o in self.convs:
            if self.fp32:   # fp32 wgrad reduces its split-K partials itself, into flat_g
                continue
            if o.out in self.up_wgrad:
                lay = nhwc.upsampled_wgrad_layout(self._probe_view(self.up_wgrad[o.out].ins[0]), o.cout, o.k)
                self.up_layout[o.w] = lay
                offs[o.w] = (total,) + tuple(lay)
                total += (lay[0] + 255) // 256 * 256
                continue
            if o.w in self.heads:
                nw = hparts * o.cin * o.cout * 4
                offs[o.w] = (total, nw + hparts * o.cout * 4, hparts, hparts, nw)
                total += (offs[o.w][1] + 255) // 256 * 256
                continue
            if o is self.win:
                nbytes, wp, bp, bo = nhwc.wgrad_partials(
                    View(torch.empty(self.xwin.shape, dtype=bf, device="meta")), self._probe_view(o.out),
                    o.k, 1, 1, window=o.k)
            else:
                nbytes, wp, bp, bo = nhwc.wgrad_partials(self._probe_view(o.ins[0]), self._probe_view(o.out),
                                                         o.k, o.k, o.dil)
            offs[o.w] = (total, nbytes, wp, bp, bo)
            total += (nbytes + 255) // 256 * 256
        self.partials_buf = torch.empty(max(total, 256), dtype=torch.uint8, device=self.device)
        self.head_parts = {}
        for o in self.convs:
            if self.fp32:
                continue
            off, nbytes, wp, bp, bo = offs[o.w]
            buf = self.partials_buf[off:off + nbytes]
            self.partials[o.w] = buf
            if o.w in self.heads:
                self.head_parts[o.w] = (buf[:bo].view(torch.float32), buf[bo:].view(torch.float32))
            if o.out in self.up_wgrad:
                continue   # reduced (and permuted to HWIO) by b2dl_upsampled_wgrad_reduce
            base = buf.data_ptr()
            n_w = o.k * o.k * o.cin * o.cout
            self.segs[o.w] = (base, self.slot[o.w][0], n_w, wp, 0)
            if o.b:   # a conv without bias_add: its bias column sums are computed and dropped
                self.segs[o.b] = (base + bo, self.slot[o.b][0], o.cout, bp, 0)
        self.set_buckets([list(param_order)])
        n, c, h, w = input_shape
        self.labels = torch.zeros(n * h * w, dtype=torch.uint8, device=self.device)
        self.pred = torch.zeros(n * h * w, dtype=torch.uint8, device=self.device)
        self.class_weights = torch.ones(p.classes, dtype=f32, device=self.device)
        self.loss = torch.zeros(1, dtype=f32, device=self.device)
        self.counts = torch.zeros(n * p.classes, dtype=torch.int32, device=self.device)
        # 1 after a step whose labels were outside [0, classes) (its loss is NaN)
        self.label_status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.input_shape = tuple(input_shape)
        # fp16 storage: a static loss scale keeps the per-pixel dlogits (~1 / (N H W), 2.6e-7 at
        # 2 x 1152 x 768) out of fp16's subnormals; every weight gradient is divided by it again in
        # the update (and on export).  A power of two, so the scaling is exact.
        self.loss_scale = (float(2 ** max(0, int(np.log2(max(1.0, n * h * w / 16.0)))))
                           if self.half == "fp16" and not self.fp32 else 1.0)
        self.launches = 0
        self.conv_timing = False
        # side stream for wgrad || dgrad overlap (B2DL_CONCURRENT=0 serialises them)
        self.side = (torch.cuda.Stream(device=self.device)
                     if os.environ.get("B2DL_CONCURRENT", "1") != "0" and self.device.type == "cuda" else None)
        self.conv_events = []
        # bias-less convs: a zero bias operand and a scratch bias-gradient target
        cmax = max([o.cout for o in self.convs] + [8])
        self._zero_bias = torch.zeros(cmax, dtype=f32, device=self.device)
        self._bias_sink = torch.zeros(cmax, dtype=f32, device=self.device)
        self.load_params(params)

    def _plan_up_dgrad(self):
        p = self.plan
        users = {}
        for o in p.ops:
            for t in list(o.ins) + ([o.res] if o.kind in ("conv", "bn") and o.res else []):
                users.setdefault(t, []).append(o)
        prog = p.backward_program
        for i, st in enumerate(prog[:-1]):
            o, nxt = st["op"], prog[i + 1]
            up = nxt["op"]
            x = o.ins[0]
            # the upsample's backward step must directly follow the conv's (nothing else writes
            # grad of its input in between), and the upsampled tensor must be the conv's alone
            if (o.kind != "conv" or st["dx"] is None or st["dx_res"] or o.dil != 1 or o.cout % 8
                    or o is self.win or up.kind != "up" or up.mode != "nearest" or up.out != x
                    or not 1 < up.factor <= 8 or users.get(x) != [o] or p.view_spec(x)[0] != x):
                continue
            kk = o.k + up.factor - 1
            self.up_dgrad[o.out] = (up, nxt)
            self.skip_up.add(up.out)
            self.wup[o.w] = torch.zeros((o.cin, kk * kk, nhwc.cin_pad(o.cout)), dtype=self.hdt,
                                        device=self.device)

    def bias_of(self, op):
        """fp32 bias operand of a conv (zeros when the graph has no bias_add after it)."""
        if not op.b:
            return self._zero_bias[:op.cout]
        off, _ = self.slot[op.b]
        return self.flat_w[off:off + op.cout]

    def bias_grad_of(self, op):
        """Where a conv's bias gradient goes (a scratch sink when it has no bias parameter)."""
        if not op.b:
            return self._bias_sink[:op.cout]
        off, _ = self.slot[op.b]
        return self.flat_g[off:off + op.cout]

    def serialize(self, on: bool):
        """Run every launch on the current stream (no wgrad || dgrad or ASPP overlap): used to time
        each conv kernel on its own."""
        if on and self.side is not None:
            self._side_keep, self.side = self.side, None
        elif not on and getattr(self, "_side_keep", None) is not None:
            self.side, self._side_keep = self._side_keep, None
        self._runs = None

    def _probe_view(self, t):
        # shape-only view for layout queries (pointer-independent)
        root, off, c = self.plan.view_spec(t)
        n, h, w, cs, _ = self.plan.buffers[root]
        return View(torch.empty((n, h, w, cs), dtype=torch.bfloat16, device="meta"), off, c)

    def set_buckets(self, buckets):
        """Gradient buckets (lists of parameter names, the all-reduce granularity).  Each conv's
        split-K partials are reduced right after its wgrad, while they are still in L2 (one small
        fixed-order launch per conv); a bucket is ready once all of its parameters are."""
        self.buckets = [list(b) for b in buckets]
        self.bucket_of = {n: i for i, b in enumerate(self.buckets) for n in b}
        self.bucket_tables = [None] * len(self.buckets)
        if not hasattr(self, "conv_tables"):
            self.conv_tables = {}
            for o in self.convs:
                segs = [self.segs[n] for n in (o.w, o.b) if n in self.segs]
                if segs:
                    self.conv_tables[o.w] = (nhwc.segment_table(segs, self.device), len(segs),
                                             max(sg[2] for sg in segs))

    def _reduce_conv(self, op):
        t = self.conv_tables.get(op.w)
        if t is not None:
            table, nseg, max_n = t
            nhwc.reduce_segments(table, nseg, max_n, self.flat_g)
            self.launches += 1

    # ---------------------------------------------------------------- roofline timing
    def _event(self):
        # inside a CUDA-graph capture the event must become a graph record node (external)
        if getattr(self, "graph_events", False):
            return torch.cuda.Event(enable_timing=True, external=True)
        return torch.cuda.Event(enable_timing=True)

    def _tic(self):
        if not self.conv_timing:
            return None
        e = self._event()
        e.record()
        return e

    def _toc(self, ev, op, tag="fprop", flops=None):
        if ev is None:
            return
        e = self._event()
        e.record()
        n, _, h, w = self.plan.shapes[op.out]
        self.conv_events.append((ev, e, flops or 2 * op.k * op.k * op.cin * op.cout * n * h * w, tag))

    def conv_kernel_totals(self, by_pass=False):
        """(ms, algorithmic FLOPs) summed over the timed conv launches (fprop, dgrad, wgrad);
        by_pass: {pass: (ms, FLOPs)} instead."""
        torch.cuda.synchronize()
        out = conv_event_totals(self.conv_events, by_pass)
        self.conv_events = []
        return out

    # ---------------------------------------------------------------- views
    def v(self, t) -> View:
        root, off, c = self.plan.view_spec(t)
        return View(self.act[root], off, c)

    def gv(self, t) -> View:
        root, off, c = self.plan.gview_spec(t)
        return View(self.grad[root], off, c)

    def wslice(self, name, buf=None):
        off, shp = self.slot[name]
        return (self.flat_w if buf is None else buf)[off:off + int(np.prod(shp))]

    # ---------------------------------------------------------------- params
    @_in_lib
    def load_params(self, params: dict):
        for name in self.order:
            a = np.asarray(params[name], dtype=np.float32)
            t = torch.from_numpy(a)
            if a.ndim == 4:   # OIHW -> HWIO
                t = t.permute(2, 3, 1, 0).contiguous()
            self.wslice(name).copy_(t.reshape(-1).to(self.device))
        self.repack()

    def _export(self, buf) -> dict:
        out = {}
        for name in self.order:
            off, shp = self.slot[name]
            t = buf[off:off + int(np.prod(shp))]
            if len(shp) == 4:
                co, ci, kh, kw = shp
                t = t.view(kh, kw, ci, co).permute(3, 2, 0, 1)
            out[name] = t.reshape(shp).cpu().numpy().copy()
        return out

    def export_params(self) -> dict:
        return self._export(self.flat_w)

    def import_flat(self, buf, tensors: dict):
        """Write reference-layout (OIHW) tensors into a flat buffer (params / momentum / grads)."""
        for name in self.order:
            a = torch.from_numpy(np.ascontiguousarray(tensors[name], dtype=np.float32))
            if a.dim() == 4:   # OIHW -> HWIO
                a = a.permute(2, 3, 1, 0).contiguous()
            self.wslice(name, buf).copy_(a.reshape(-1).to(self.device))

    def export_grads(self) -> dict:
        g = self._export(self.flat_g)
        if self.loss_scale != 1.0:
            g = {k: v / np.float32(self.loss_scale) for k, v in g.items()}
        return g

    def wmaster(self, name):
        off, shp = self.slot[name]
        return self.flat_wbf[off:off + int(np.prod(shp))]

    @_in_lib
    def refresh_mirror(self):
        """bf16 mirror <- flat fp32 parameters (after loading weights from the host)."""
        if self.fp32:
            return
        nhwc.larc_update(self.flat_w, self.flat_m, self.flat_g, self.offsets, 1.0, 0.0, 1.0, 0.0, 1.0, 1.0,
                         self._lr_scratch, self._status, self.ws, mode=3, w_bf16=self.flat_wbf)
        self.launches += 1

    @_in_lib
    def repack(self, mirror=True):
        """Refresh the weight operands after an update; the LARC kernel already writes the mirror
        during training (mirror=False), leaving only the packed copies of ragged-channel convs."""
        if mirror:
            self.refresh_mirror()
        for o in self.packed:
            nhwc.pack_weights(self.wslice(o.w), o.k, o.k, o.cin, o.cout, fprop=self.wf[o.w],
                              dgrad=self.wd.get(o.w))
            self.launches += 1 + (o.w in self.wd)
        for o in self.rowtap:
            nhwc.pack_weights(self.wslice(o.w), o.k, o.k, o.cin, o.cout, fprop=self.wf[o.w])
            self.launches += 1
        for o in self.rowtap_dgrad:
            nhwc.pack_weights(self.wslice(o.w), o.k, o.k, o.cin, o.cout, dgrad=self.wd[o.w])
            self.launches += 1
        if self.win is not None:   # HWIO [k][k][cin][cout] is HWIO [k][1][k*cin][cout]
            o = self.win
            nhwc.pack_weights(self.wslice(o.w), o.k, 1, o.k * o.cin, o.cout, fprop=self.wwin)
            self.launches += 1
        for o in self.convs:
            if o.w in self.wupf:
                nhwc.pack_upsampled_fprop(self.wslice(o.w), o.k, o.cin, o.cout, self.up_fprop[o.out].factor,
                                          self.wupf[o.w])
                self.launches += 1
            if o.w in self.wup:
                up = self.up_dgrad[o.out][0]
                nhwc.pack_upsampled_dgrad(self.wslice(o.w), o.k, o.cin, o.cout, up.factor, self.wup[o.w])
                self.launches += 1

    # ---------------------------------------------------------------- inputs
    @_in_lib
    def set_batch(self, x_nchw: torch.Tensor, labels: torch.Tensor):
        """x fp32 NCHW and labels uint8 [N,H,W] already on the device."""
        if tuple(x_nchw.shape) != self.input_shape:
            raise ValueError(f"batch {tuple(x_nchw.shape)} does not match planned {self.input_shape}")
        if self.win is not None:
            nhwc.nchw_to_nhwc_halo(x_nchw.contiguous(), self.xwin, (self.win.k - 1) // 2)
        else:
            nhwc.nchw_to_nhwc(x_nchw.contiguous(), self.v("x"), dst_f32=self.fp32)
        self.labels.copy_(labels.reshape(-1))
        self.launches += 1

    def set_class_weights(self, w):
        self.class_weights.copy_(torch.as_tensor(np.asarray(w, dtype=np.float32)))

    # ---------------------------------------------------------------- forward
    @_in_lib
    def forward(self):
        """Fused forward program.  Runs of convs reading the same input (the ASPP branches) are
        spread over the main and side streams so their tail waves overlap."""
        forks, side_ops, joins = self._side_runs()
        for idx, op in enumerate(self.plan.ops):
            if idx in forks:
                ev = torch.cuda.Event()
                ev.record()
                self.side.wait_event(ev)
            if idx in side_ops:
                with torch.cuda.stream(self.side):
                    self._fwd_op(op)
            else:
                self._fwd_op(op)
            if idx in joins:   # end of the run: the main stream waits for the side stream's ops
                ev = torch.cuda.Event()
                ev.record(self.side)
                torch.cuda.current_stream().wait_event(ev)

    def _side_runs(self):
        """(fork indices, side-stream op indices, join indices): runs of >= 2 consecutive bf16
        convs with the same input and no residual operand (outputs are distinct buffers or concat
        slices) alternate between the main and the side stream."""
        if getattr(self, "_runs", None) is not None:
            return self._runs
        forks, side, joins = set(), set(), set()
        ops = self.plan.ops
        if self.side is not None and not self.fp32:
            i = 0
            while i < len(ops):
                j = i
                while (j + 1 < len(ops) and ops[i].kind == "conv" and ops[j + 1].kind == "conv"
                       and ops[j + 1].ins[0] == ops[i].ins[0] and not ops[i].res and not ops[j + 1].res
                       and ops[i] is not self.win):
                    j += 1
                if j > i:
                    forks.add(i)
                    side.update(k for k in range(i, j + 1) if (k - i) % 2 == 1)
                    joins.add(j)
                i = j + 1
        self._runs = (forks, side, joins)
        return self._runs

    def _fwd_op(self, op):
        p = self.plan
        if op.kind == "conv" and self.fp32:
            ev = self._tic()
            nhwc.f32_conv(self.v(op.ins[0]), self.wslice(op.w), op.cout, op.k, op.k, op.dil, self.v(op.out),
                          bias=self.bias_of(op),
                          residual=self.v(op.res) if op.res else None, relu=op.relu)
            self._toc(ev, op)
        elif op.kind == "conv" and op.out in self.up_fprop:
            up = self.up_fprop[op.out]
            n, _, h, w = self.plan.shapes[up.ins[0]]
            ev = self._tic()
            nhwc.upsampled_fprop(self.v(up.ins[0]), self.wupf[op.w], op.cin, op.cout, op.k, up.factor, self.v(op.out),
                                 bias=self.bias_of(op), relu=op.relu)
            taps = nhwc.upsampled_fprop_taps(op.k, up.factor)
            self._toc(ev, op, flops=2 * taps * op.cin * op.cout * n * h * w)
            self.launches += up.factor * up.factor - 1
        elif op.kind == "conv":
            out = op.out
            ev = self._tic()
            wsrc = dict(w_packed=self.wf[op.w]) if op.w in self.wf else dict(
                w_packed=None, w_master=self.wmaster(op.w), w_mode=1)
            xin, kw = self.v(op.ins[0]), op.k
            if op is self.win:
                wsrc = dict(w_packed=self.wwin, window=op.k)
                xin, kw = View(self.xwin), 1
            kwargs = dict(cout=op.cout, kh=op.k, kw=kw, dilation=op.dil, y=self.v(out), **wsrc, bias=self.bias_of(op),
                          residual=self.v(op.res) if op.res else None, relu=op.relu, y_f32=(out == p.logits_name))
            if out in self.bn_fused:
                if out not in self.bn_parts:   # sized on the first (eager) step, before any capture
                    tiles = nhwc.conv_fprop(xin, bn_rows_only=True, **kwargs)   # statistics rows
                    self.bn_parts[out] = (torch.empty(tiles * 2 * op.cout, dtype=torch.float32, device=self.device),
                                          tiles)
                kwargs["bn_partial"] = self.bn_parts[out][0]
            nhwc.conv_fprop(xin, **kwargs)
            self._toc(ev, op)
        elif op.kind == "bn" and op.ins[0] in self.bn_parts:
            part, tiles = self.bn_parts[op.ins[0]]
            nhwc.bn_forward_partials(part, tiles, self.v(op.ins[0]), self.wslice(op.w), self.wslice(op.b), op.eps,
                                     self.v(op.out), self.bn_stats[op.out], self.ws,
                                     residual=self.v(op.res) if op.res else None, relu=op.relu)
            self.launches += 2
        elif op.kind == "bn":
            nhwc.bn_forward(self.v(op.ins[0]), self.wslice(op.w), self.wslice(op.b), op.eps, self.v(op.out),
                            self.bn_stats[op.out], self.ws, residual=self.v(op.res) if op.res else None,
                            relu=op.relu)
            self.launches += 2
        elif op.kind == "up" and op.mode == "bilinear":
            nhwc.bilinear_fwd(self.v(op.ins[0]), self.v(op.out), op.factor)
        elif op.kind == "pool":
            (nhwc.f32_avgpool_fwd if self.fp32 else nhwc.avgpool_fwd)(self.v(op.ins[0]), self.v(op.out),
                                                                      op.factor)
        elif op.kind == "up" and op.out in self.dead_up:
            return   # its only consumer reads the low-resolution input directly (fwd, dgrad, wgrad)
        elif op.kind == "up":
            (nhwc.f32_upsample_fwd if self.fp32 else nhwc.upsample_fwd)(self.v(op.ins[0]), self.v(op.out),
                                                                        op.factor)
        elif op.kind == "concat":
            off = 0
            for s in op.ins:
                if s in op.copy_ins:
                    root, coff, c = p.view_spec(op.out)
                    self._add(self.v(s), View(self.act[root], coff + off, self.plan.chans(s)),
                              accumulate=False)
                    self.launches += 1
                off += self.plan.chans(s)
            return
        elif op.kind == "add":
            a, b = op.ins
            self._add(self.v(a), self.v(op.out), accumulate=False)
            self._add(self.v(b), self.v(op.out), accumulate=True)
            self.launches += 1
        elif op.kind == "bias":
            nhwc.ewise(self.v(op.ins[0]), self.v(op.out), bias=self.wslice(op.b), relu=op.relu, f32=self.fp32)
        elif op.kind == "relu":
            nhwc.ewise(self.v(op.ins[0]), self.v(op.out), relu=True, f32=self.fp32)
        elif op.kind == "mul":
            nhwc.ewise(self.v(op.ins[0]), self.v(op.out), x1=self.v(op.ins[1]), f32=self.fp32)
        elif op.kind == "scale":
            nhwc.ewise(self.v(op.ins[0]), self.v(op.out), alpha=op.alpha, f32=self.fp32)
        elif op.kind == "matmul":
            nhwc.matmul_w(self.v(op.ins[0]), self.wslice(op.w), self.v(op.out), f32=self.fp32)
        elif op.kind == "ce":
            nhwc.wce(self.v(op.ins[0]), self.labels, self.class_weights, self.loss, self.counts,
                     self.gv(op.ins[0]), self.pred, self.ws, dlogits_f32=self.fp32, status=self.label_status,
                     dlogits_scale=self.loss_scale)
            self.launches += 2   # histogram + loss/dlogits + final fold (3 with the +1 below)
        self.launches += 1

    # ---------------------------------------------------------------- backward
    def _reduce_bucket(self, i):
        t = self.bucket_tables[i]
        if t is not None:
            table, nseg, max_n = t
            nhwc.reduce_segments(table, nseg, max_n, self.flat_g)
            self.launches += 1

    def _param_done(self, names, pending, on_bucket_ready):
        """Count parameters whose gradients are enqueued; fire each bucket that completes.

        A bucket's gradients are written from BOTH compute streams (most wgrads and their split-K
        reductions run on the side stream, the stem's / batch norm's on the main stream, and
        side-stream wgrads trail main-stream dgrads across layers), so the all-reduce must not be
        issued from whichever stream happens to be current: it is issued from a bucket stream that
        first waits on both, which orders the collective after every write into the bucket (the
        reference reduces a tensor only once it is final, trainer.py:222-241) without making the
        compute streams wait on each other."""
        for name in names:
            if not name:
                continue
            i = self.bucket_of[name]
            pending[i] -= 1
            if pending[i] != 0:
                continue
            self._reduce_bucket(i)
            if on_bucket_ready is None:
                continue
            if self.side is None or os.environ.get("B2DL_BUCKET_JOIN", "1") == "0":
                on_bucket_ready(i)   # B2DL_BUCKET_JOIN=0: the unjoined issue (negative control only)
                continue
            bs = self._bucket_stream()
            for s in (torch.cuda.current_stream(), self.side):
                ev = torch.cuda.Event()
                ev.record(s)
                bs.wait_event(ev)
            with torch.cuda.stream(bs):
                on_bucket_ready(i)

    def _bucket_stream(self):
        if getattr(self, "_bstream", None) is None:
            self._bstream = torch.cuda.Stream(device=self.device)
        return self._bstream

    def _stress_side(self, op):
        """Test knob (B2DL_STRESS_SIDE_US): delay the side stream before the wgrads of the
        convs named by B2DL_STRESS_CONVS (prefix match), so a collective that is not ordered after
        them would read stale gradients."""
        us = int(os.environ.get("B2DL_STRESS_SIDE_US", "0"))
        if us <= 0:
            return
        pref = os.environ.get("B2DL_STRESS_CONVS", "s0.")
        if any(op.w.startswith(p) for p in pref.split(",")):
            torch.cuda._sleep(int(us * 1900))   # ~1.9 cycles per ns at the boost clock

    @_in_lib
    def backward(self, on_bucket_ready=None):
        """Fill flat_g with d loss / d params (param layout HWIO for conv weights).

        `on_bucket_ready(i)` fires as soon as bucket i's gradients are final (enqueued),
        so the trainer can start that bucket's all-reduce while backward continues."""
        pending = [len(b) for b in self.buckets]
        for st in self.plan.backward_program:
            op = st["op"]
            if op.kind == "conv" and self.fp32:
                gy = self.gv(op.out)
                if st["relu_pass"]:
                    nhwc.f32_relu_mask(gy, self.v(op.out))
                    self.launches += 1
                ev = self._tic()
                nhwc.f32_conv_wgrad(self.v(op.ins[0]), gy, op.k, op.k, op.dil, self.wslice(op.w, self.flat_g),
                                    self.ws, bias_grad=self.bias_grad_of(op))
                self._toc(ev, op, "wgrad")
                self.launches += 3
                self._param_done((op.w, op.b), pending, on_bucket_ready)
                if st["dx"] is not None:
                    ev = self._tic()
                    nhwc.f32_conv_dgrad(gy, self.wslice(op.w), op.cin, op.k, op.k, op.dil, self.gv(op.ins[0]),
                                        accumulate=st["dx"], mask=self.v(op.ins[0]) if st["mask_dx"] else None,
                                        residual=self.gv(st["dx_res"]) if st["dx_res"] else None)
                    self._toc(ev, op, "dgrad")
                    self.launches += 1
            elif op.kind == "conv":
                gy = self.gv(op.out)
                if st["relu_pass"]:
                    nhwc.relu_mask(gy, self.v(op.out))
                    self.launches += 1
                # wgrad and dgrad of a conv are independent (both only read dy): the wgrad (+ its
                # split-K reduction and the bucket's all-reduce start) runs on a side stream so the
                # two persistent kernels fill each other's tail waves; they join before the next op
                gemm_dgrad = (st["dx"] is not None and op.w not in self.heads and not (op.k == 1 and op.cout < 8))
                side = self.side if (gemm_dgrad and self.side is not None) else None
                if side is not None:
                    fork = torch.cuda.Event()
                    fork.record()
                    side.wait_event(fork)
                with (torch.cuda.stream(side) if side is not None else contextlib.nullcontext()):
                    if side is not None:
                        self._stress_side(op)
                    ev = self._tic()
                    # wgrad GEMM with the bias column sums folded in; split-K partials stay in the
                    # conv's partial buffer and are reduced right after it (fixed order, L2-hot)
                    if op.w in self.heads:
                        dwp, dbp = self.head_parts[op.w]
                        nhwc.head_backward(gy, self.wslice(op.w), self.v(op.ins[0]),
                                           self.gv(op.ins[0]) if st["dx"] is not None else None, dwp, dbp,
                                           accumulate=bool(st["dx"]), mask_dx=bool(st["mask_dx"]))
                    elif op is self.win:
                        nhwc.conv_wgrad_deferred(View(self.xwin), gy, op.k, 1, 1, self.partials[op.w],
                                                 window=op.k)
                    elif op.out in self.up_wgrad:
                        up = self.up_wgrad[op.out]
                        w_off, _ = self.slot[op.w]
                        nhwc.upsampled_wgrad(self.v(up.ins[0]), gy, op.k, up.factor, self.gsum[op.w],
                                             self.partials[op.w], self.up_layout[op.w],
                                             self.flat_g[w_off:w_off + op.k * op.k * op.cin * op.cout],
                                             self.bias_grad_of(op))
                        n, _, h, w = self.plan.shapes[up.ins[0]]
                        self.launches += 2
                        wflops = 2 * op.k * op.k * op.cin * op.cout * n * h * w
                    else:
                        nhwc.conv_wgrad_deferred(self.v(op.ins[0]), gy, op.k, op.k, op.dil, self.partials[op.w])
                    self._toc(ev, op, "wgrad", flops=wflops if op.out in self.up_wgrad else None)
                    self.launches += 1
                    self._reduce_conv(op)
                    self._param_done((op.w, op.b), pending, on_bucket_ready)
                if op.w in self.heads:
                    pass   # input gradient already produced by head_backward
                elif st["dx"] is not None and op.k == 1 and op.cout < 8:
                    # e.g. the 3-class head: a memory-bound channel expansion, not a GEMM
                    nhwc.dgrad_1x1_small(gy, self.wslice(op.w), self.gv(op.ins[0]), accumulate=st["dx"],
                                         mask=self.v(op.ins[0]) if st["mask_dx"] else None)
                    self.launches += 1
                elif op.out in self.up_dgrad:
                    # dgrad + the upsample's VJP in one strided low-resolution conv (executed FLOPs)
                    up, ust = self.up_dgrad[op.out]
                    f, kk = up.factor, op.k + up.factor - 1
                    n, _, h, w = self.plan.shapes[up.ins[0]]
                    ev = self._tic()
                    nhwc.upsampled_dgrad(gy, self.wup[op.w], op.cin, op.k, f, self.gv(up.ins[0]),
                                         accumulate=ust["dx"], mask=self.v(up.ins[0]) if ust["mask"] else None)
                    self._toc(ev, op, "dgrad", flops=2 * kk * kk * op.cin * op.cout * n * h * w)
                    self.launches += 1
                elif st["dx"] is not None:
                    ev = self._tic()
                    wsrc = dict(w_dgrad=self.wd[op.w]) if op.w in self.wd else dict(
                        w_dgrad=None, w_master=self.wmaster(op.w))
                    kw = dict(cin=op.cin, kh=op.k, kw=op.k, dilation=op.dil, dx=self.gv(op.ins[0]), **wsrc,
                              accumulate=st["dx"], mask=self.v(op.ins[0]) if st["mask_dx"] else None,
                              residual=self.gv(st["dx_res"]) if st["dx_res"] else None)
                    bn = self.bnb_of.get(op.out)
                    if bn is not None:   # dx = d loss / d (BN output): BN backward statistics in the epilogue
                        kw.update(mask=self.v(bn.ins[0]), bnb_stats=self.bn_stats[bn.out])
                        if bn.out not in self.bnb_parts:   # sized on the first (eager) step
                            rows = 4 * nhwc.conv_dgrad(gy, bn_rows_only=True, **kw)
                            self.bnb_parts[bn.out] = (torch.empty(rows * 2 * bn.cout, dtype=torch.float32,
                                                                  device=self.device), rows)
                        kw["bnb_partial"] = self.bnb_parts[bn.out][0]
                    nhwc.conv_dgrad(gy, **kw)
                    self._toc(ev, op, "dgrad")
                    self.launches += 1
                # no per-layer join: gradient buffers are never reused within a step (one per
                # activation root) and backward never writes grad(op.out) again, so the side
                # stream's wgrads may trail the main stream's dgrads; they join at the end

            elif op.kind == "bn":
                gy = self.gv(op.out)
                if st["relu_pass"]:
                    (nhwc.f32_relu_mask if self.fp32 else nhwc.relu_mask)(gy, self.v(op.out))
                    self.launches += 1
                g_off, _ = self.slot[op.w]
                b_off, _ = self.slot[op.b]
                if op.out in self.bnb_parts:   # statistics came with the consumer's dgrad
                    part, rows = self.bnb_parts[op.out]
                    nhwc.bn_backward_partials(part, rows, self.v(op.ins[0]), gy, self.wslice(op.w),
                                              self.bn_stats[op.out], self.flat_g[g_off:g_off + op.cout],
                                              self.flat_g[b_off:b_off + op.cout],
                                              self.gv(op.ins[0]) if st["dx"] is not None else None, self.ws,
                                              accumulate=bool(st["dx"]))
                    self.launches += 2
                else:
                    nhwc.bn_backward(self.v(op.ins[0]), gy, self.wslice(op.w), self.bn_stats[op.out],
                                     self.flat_g[g_off:g_off + op.cout], self.flat_g[b_off:b_off + op.cout],
                                     self.gv(op.ins[0]) if st["dx"] is not None else None, self.ws,
                                     accumulate=bool(st["dx"]))
                    self.launches += 3
                self._param_done((op.w, op.b), pending, on_bucket_ready)
            elif op.kind == "up" and op.mode == "bilinear":
                nhwc.bilinear_bwd(self.gv(op.out), self.gv(op.ins[0]), op.factor, accumulate=st["dx"],
                                  mask=self.v(op.ins[0]) if st["mask"] else None, ws=self.ws)
                self.launches += 1
            elif op.kind == "pool":
                (nhwc.f32_avgpool_bwd if self.fp32 else nhwc.avgpool_bwd)(
                    self.gv(op.out), self.gv(op.ins[0]), op.factor, accumulate=st["dx"],
                    mask=self.v(op.ins[0]) if st["mask"] else None)
                self.launches += 1
            elif op.kind == "up" and op.out in self.skip_up:
                pass   # folded into the consuming conv's dgrad
            elif op.kind == "up":
                (nhwc.f32_upsample_bwd if self.fp32 else nhwc.upsample_bwd)(
                    self.gv(op.out), self.gv(op.ins[0]), op.factor, accumulate=st["dx"],
                    mask=self.v(op.ins[0]) if st["mask"] else None)
                self.launches += 1
            elif op.kind == "concat":
                root, coff, _ = self.plan.view_spec(op.out)
                for s, off, acc, m in st["copies"]:
                    self._add(View(self.grad[root], coff + off, self.plan.chans(s)), self.gv(s), accumulate=acc,
                              mask=self.v(s) if m else None)
                    self.launches += 1
            elif op.kind in ("bias", "relu", "mul", "scale", "matmul"):
                self._bwd_generic(st, pending, on_bucket_ready)
            elif op.kind == "add":
                src = st.get("passthrough", op.out)
                for s, acc, m in st["acc"]:
                    self._add(self.gv(src), self.gv(s), accumulate=acc, mask=self.v(s) if m else None)
                    self.launches += 1
        if self.side is not None and not self.fp32:   # all wgrads (and their reductions) done
            ev = torch.cuda.Event()
            ev.record(self.side)
            torch.cuda.current_stream().wait_event(ev)
        if getattr(self, "_bstream", None) is not None:   # rejoin the bucket stream (graph capture)
            ev = torch.cuda.Event()
            ev.record(self._bstream)
            torch.cuda.current_stream().wait_event(ev)

    def _bwd_generic(self, st, pending, on_bucket_ready):
        """VJPs of the standalone lowerings (ops.py:166-177, 195-202) on the main stream."""
        op, f32 = st["op"], self.fp32
        gy = self.gv(op.out)
        x = op.ins[0]
        mask_x = self.v(x) if st.get("mask") else None
        if op.kind == "bias":
            if st["relu_pass"]:
                (nhwc.f32_relu_mask if f32 else nhwc.relu_mask)(gy, self.v(op.out))
            nhwc.channel_sum(gy, self.wslice(op.b, self.flat_g), f32=f32)
            self._param_done((op.b,), pending, on_bucket_ready)
            if st["dx"] is not None:
                nhwc.ewise(gy, self.gv(x), mask=mask_x, accumulate=st["dx"], f32=f32)
        elif op.kind == "relu" and st["dx"] is not None:
            # (relu(x) > 0) == (x > 0): the output is the mask for both the relu VJP and x's own mask
            nhwc.ewise(gy, self.gv(x), mask=self.v(op.out), accumulate=st["dx"], f32=f32)
        elif op.kind == "scale" and st["dx"] is not None:
            nhwc.ewise(gy, self.gv(x), alpha=op.alpha, mask=mask_x, accumulate=st["dx"], f32=f32)
        elif op.kind == "mul":
            for i, s_, acc, m in st["acc"]:
                nhwc.ewise(gy, self.gv(s_), x1=self.v(op.ins[1 - i]), mask=self.v(s_) if m else None,
                           accumulate=acc, f32=f32)
        elif op.kind == "matmul":
            nhwc.matmul_w_grad(self.v(x), gy, self.wslice(op.w, self.flat_g), f32=f32)
            self._param_done((op.w,), pending, on_bucket_ready)
            if st["dx"] is not None:
                nhwc.matmul_w(gy, self.wslice(op.w), self.gv(x), trans=True, mask=mask_x, accumulate=st["dx"],
                              f32=f32)
        self.launches += 2

    def _add(self, x, y, accumulate=False, mask=None):
        (nhwc.f32_add if self.fp32 else nhwc.add)(x, y, accumulate=accumulate, mask=mask)

    @_in_lib
    def logits_nchw(self) -> torch.Tensor:
        n, c, h, w = self.plan.shapes[self.plan.logits_name]
        out = torch.empty((n, c, h, w), dtype=torch.float32, device=self.device)
        nhwc.nhwc_to_nchw(self.v(self.plan.logits_name), out, src_f32=True)
        return out

    def predictions(self) -> torch.Tensor:
        n, _, h, w = self.input_shape
        return self.pred.view(n, h, w)
