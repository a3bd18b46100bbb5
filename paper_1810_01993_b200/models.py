"""Model definitions as op graphs built from the reference's op kinds.

Two families, both expressed only with ops the reference executor implements
(conv2d any dilation, bias_add, relu, elementwise add, concat, avgpool,
nearest upsample, softmax_ce), so the reference (or its restatement under
oracle/) can run the identical graph for parity ("tier A"):

* MiniDenseNet — the reference's own network (pkg/src/deskdl/model/net.py:83-112),
  the Tiramisu / FC-DenseNet variant of config 4.
* DeepLabV3Plus — ResNet-50 bottleneck encoder at output stride 8 (stage 3
  dilation 2, stage 4 dilation 4), ASPP with 1x1 + 3x3 at dilations 12/18/24,
  decoder with a 48-channel low-level projection, x4 upsample to full
  resolution followed by 3x3x256 convolutions and a 1x1 head.  Strided convs
  do not exist in the reference's execution kernels (_kernels_py.py:46-47),
  so downsampling is average pooling, as the reference's own network does.

Initialisation follows net.py:58-71: He-uniform U(+-sqrt(6/(cin*k*k))) drawn
from numpy's default_rng(seed) in build order, zero biases.  Without batch
normalisation a deep residual stack explodes at He init, so the last conv of
every residual branch is scaled by `res_scale` (a documented deviation,
DESIGN.md).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .graph import OpGraph

GROWTH_CHOICES = (16, 32)


@dataclass(frozen=True)
class NetConfig:
    """MiniDenseNet hyper-parameters (reference net.py:23-41).

    Extensions for config 4 (the paper's Tiramisu): `block_layers` may be
    a tuple with one entry per down level plus the bottleneck (the up path mirrors the down path),
    and `kernel` sets the dense-layer convolution size (the reference is uniform 3x3)."""
    channels_in: int = 16
    growth: int = 16
    block_layers: object = 2
    levels: int = 2
    classes: int = 3
    kernel: int = 3

    def __post_init__(self):
        if self.growth not in GROWTH_CHOICES:
            raise ValueError(f"growth must be one of {GROWTH_CHOICES}")
        layers = self.block_layers if isinstance(self.block_layers, tuple) else (self.block_layers,)
        if self.channels_in < 1 or min(layers) < 1 or self.classes < 2 or self.kernel < 1 or self.kernel % 2 == 0:
            raise ValueError("bad network configuration")
        if self.levels < 0:
            raise ValueError("levels must be non-negative")
        if isinstance(self.block_layers, tuple) and len(self.block_layers) != self.levels + 1:
            raise ValueError("block_layers tuple needs one entry per level plus the bottleneck")

    def layers_at(self, level: int) -> int:
        """Dense-block depth at down level `level` (== levels: the bottleneck)."""
        if isinstance(self.block_layers, tuple):
            return self.block_layers[level]
        return self.block_layers

    @property
    def downsample_factor(self) -> int:
        return 2 ** self.levels


@dataclass(frozen=True)
class DeepLabConfig:
    channels_in: int = 16
    classes: int = 3
    stem_kernel: int = 7
    stem_channels: int = 64
    stem_pool: int = 4
    blocks: tuple = (3, 4, 6, 3)
    widths: tuple = (64, 128, 256, 512)
    expansion: int = 4
    dilations: tuple = (1, 1, 2, 4)
    pool_before: tuple = (False, True, False, False)
    aspp_channels: int = 256
    aspp_dilations: tuple = (12, 18, 24)
    lowlevel_channels: int = 48
    decoder_channels: int = 256
    full_res_convs: int = 3
    res_scale: float = 0.1
    # north-star variant: batch norm after every conv but the head, and
    # bilinear instead of nearest upsampling in the decoder
    batchnorm: bool = False
    bilinear: bool = False

    @property
    def downsample_factor(self) -> int:
        f = self.stem_pool
        for p in self.pool_before:
            f *= 2 if p else 1
        return f

    @property
    def decoder_up(self) -> int:
        """Upsample factor from the ASPP map to the low-level (stage 1) map."""
        f = 1
        for p in self.pool_before[1:]:
            f *= 2 if p else 1
        return f


def deeplab_small(**kw) -> DeepLabConfig:
    """Narrow, shallow DeepLabV3+ with the full topology, for CPU-oracle parity."""
    base = dict(stem_kernel=7, stem_channels=16, blocks=(1, 1, 2, 1), widths=(16, 16, 32, 32),
                expansion=2, aspp_channels=32, aspp_dilations=(2, 3, 4), lowlevel_channels=16,
                decoder_channels=32, full_res_convs=1)
    base.update(kw)
    return DeepLabConfig(**base)


class _Builder:
    """Adds conv (+bias, +relu) blocks with He-uniform weights in build order."""

    def __init__(self, graph: OpGraph, rng):
        self.g = graph
        self.rng = rng
        self.params = {}
        self.conv_meta = {}

    def conv(self, x, name, cin, cout, k=3, dilation=1, act=True, scale=1.0, bn=False):
        g = self.g
        wname = g.add_input(f"{name}.w", role="param")
        bname = g.add_input(f"{name}.b", role="param")
        limit = np.sqrt(6.0 / (cin * k * k))
        w = self.rng.uniform(-limit, limit, size=(cout, cin, k, k)).astype(np.float32)
        if scale != 1.0:
            w = (w * np.float32(scale)).astype(np.float32)
        self.params[wname] = w
        self.params[bname] = np.zeros(cout, dtype=np.float32)
        out = g.conv2d(x, wname, f"{name}.conv", kh=k, kw=k, cin=cin, cout=cout,
                       dilation=dilation)
        out = g.bias_add(out, bname, f"{name}.bias")
        if bn:   # training-mode batch norm; scale 1, shift 0 at init
            gname = g.add_input(f"{name}.gamma", role="param")
            bename = g.add_input(f"{name}.beta", role="param")
            self.params[gname] = np.ones(cout, dtype=np.float32)
            self.params[bename] = np.zeros(cout, dtype=np.float32)
            out = g.batchnorm(out, gname, bename, f"{name}.bn")
        if act:
            out = g.relu(out, f"{name}.relu")
        return out


def _io(g: OpGraph):
    x = g.add_input("x", role="data")
    g.add_input("labels", role="aux")
    g.add_input("class_weights", role="aux")
    return x


def tiramisu_config4(**kw) -> NetConfig:
    """Config 4, frozen: the paper's Tiramisu / FC-DenseNet at the reference's op set -- 5
    resolution levels (4 pooling steps), dense blocks of (2, 2, 2, 4) layers down + 5 in the
    bottleneck (mirrored up), growth 32, 5x5 dense-layer convs."""
    base = dict(channels_in=16, growth=32, block_layers=(2, 2, 2, 4, 5), levels=4, kernel=5)
    base.update(kw)
    return NetConfig(**base)


def build_minidensenet(cfg: NetConfig, seed: int = 0, graph_cls=OpGraph):
    """Graph + params of the reference network (net.py:83-112).  `graph_cls` may be the
    reference's own deskdl.graph.OpGraph (same builder API) to run the graph on deskdl."""
    g = graph_cls()
    b = _Builder(g, np.random.default_rng(seed))
    x = _io(g)
    k = cfg.growth

    def dense(inp, name, cin, nlayers):
        feats, ch = inp, cin
        for j in range(nlayers):
            fresh = b.conv(feats, f"{name}.l{j}", ch, k, k=cfg.kernel)
            feats = g.concat([feats, fresh], f"{name}.cat{j}")
            ch += k
        return feats, ch

    cur = b.conv(x, "stem", cfg.channels_in, k)
    ch = k
    skips = []
    for lvl in range(cfg.levels):
        cur, ch = dense(cur, f"down{lvl}", ch, cfg.layers_at(lvl))
        skips.append((cur, ch))
        cur = g.avgpool(cur, f"pool{lvl}", window=2)
    cur, ch = dense(cur, "mid", ch, cfg.layers_at(cfg.levels))
    for lvl in reversed(range(cfg.levels)):
        skip, sch = skips[lvl]
        cur = g.upsample(cur, f"up{lvl}.grow", factor=2)
        cur = g.concat([cur, skip], f"up{lvl}.cat")
        cur = b.conv(cur, f"up{lvl}.squeeze", ch + sch, sch, k=1)
        ch = sch
        cur, ch = dense(cur, f"up{lvl}", ch, cfg.layers_at(lvl))
    head = b.conv(cur, "head", ch, cfg.classes, k=1, act=False)
    loss = g.softmax_ce(head, "labels", "class_weights", "loss", classes=cfg.classes)
    return g, b.params, head, loss


def build_deeplab(cfg: DeepLabConfig, seed: int = 0, graph_cls=OpGraph):
    """Graph + params of the DeepLabV3+ (OS8) used for the headline benchmark.  With
    graph_cls=deskdl.graph.OpGraph the reference-op variant builds as a graph the reference's own
    executor runs (batch norm / bilinear need this package's OpGraph)."""
    g = graph_cls()
    b = _Builder(g, np.random.default_rng(seed))
    x = _io(g)

    bn = cfg.batchnorm

    def bottleneck(inp, name, cin, mid, cout, dil):
        a = b.conv(inp, f"{name}.a", cin, mid, k=1, bn=bn)
        m = b.conv(a, f"{name}.b", mid, mid, k=3, dilation=dil, bn=bn)
        c = b.conv(m, f"{name}.c", mid, cout, k=1, act=False, scale=cfg.res_scale, bn=bn)
        sc = inp if cin == cout else b.conv(inp, f"{name}.proj", cin, cout, k=1, act=False, bn=bn)
        s = g.elementwise([c, sc], f"{name}.add", fn="add")
        return g.relu(s, f"{name}.relu")

    cur = b.conv(x, "stem", cfg.channels_in, cfg.stem_channels, k=cfg.stem_kernel, bn=bn)
    cur = g.avgpool(cur, "stem.pool", window=cfg.stem_pool)
    ch = cfg.stem_channels
    low, low_ch = None, None
    for s, nblk in enumerate(cfg.blocks):
        if cfg.pool_before[s]:
            cur = g.avgpool(cur, f"s{s}.pool", window=2)
        width = cfg.widths[s]
        out_ch = width * cfg.expansion
        for j in range(nblk):
            cur = bottleneck(cur, f"s{s}.b{j}", ch, width, out_ch, cfg.dilations[s])
            ch = out_ch
        if s == 0:
            low, low_ch = cur, ch
    a = cfg.aspp_channels
    branches = [b.conv(cur, "aspp.c1x1", ch, a, k=1, bn=bn)]
    for d in cfg.aspp_dilations:
        branches.append(b.conv(cur, f"aspp.d{d}", ch, a, k=3, dilation=d, bn=bn))
    cur = g.concat(branches, "aspp.cat")
    cur = b.conv(cur, "aspp.proj", a * len(branches), a, k=1, bn=bn)
    up = g.upsample_bilinear if cfg.bilinear else g.upsample
    cur = up(cur, "dec.up", factor=cfg.decoder_up)
    ll = b.conv(low, "dec.low", low_ch, cfg.lowlevel_channels, k=1, bn=bn)
    cur = g.concat([cur, ll], "dec.cat")
    dch = cfg.decoder_channels
    cur = b.conv(cur, "dec.c0", a + cfg.lowlevel_channels, dch, k=3, bn=bn)
    cur = b.conv(cur, "dec.c1", dch, dch, k=3, bn=bn)
    cur = up(cur, "full.up", factor=cfg.stem_pool)
    for i in range(cfg.full_res_convs):
        cur = b.conv(cur, f"full.c{i}", dch, dch, k=3, bn=bn)
    head = b.conv(cur, "head", dch, cfg.classes, k=1, act=False)
    loss = g.softmax_ce(head, "labels", "class_weights", "loss", classes=cfg.classes)
    return g, b.params, head, loss


def build(cfg, seed: int = 0):
    if isinstance(cfg, NetConfig):
        return build_minidensenet(cfg, seed)
    if isinstance(cfg, DeepLabConfig):
        return build_deeplab(cfg, seed)
    raise TypeError(f"unknown model config {type(cfg).__name__}")
