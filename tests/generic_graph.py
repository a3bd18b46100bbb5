"""A graph exercising every reference op kind outside the conv-bias-relu chains of the two model
families: standalone bias_add (+ relu), standalone relu, elementwise mul / scale, matmul over the
width axis (ops.py:120-148), a bias-less conv, channel concat and avgpool (test infrastructure)."""

import numpy as np

from paper_1810_01993_b200.graph import OpGraph


def build(seed=0, cin=8, h=16, w=16):
    rng = np.random.default_rng(seed)
    g = OpGraph()
    g.add_input("x", role="data")
    g.add_input("labels", role="aux")
    g.add_input("class_weights", role="aux")
    p = {}

    def param(name, shape, scale):
        g.add_input(name, role="param")
        p[name] = (rng.uniform(-1, 1, size=shape) * scale).astype(np.float32)
        return name

    c = 16
    g.conv2d("x", param("c1.w", (c, cin, 3, 3), (6 / (cin * 9)) ** 0.5), "c1.conv", kh=3, kw=3, cin=cin, cout=c)
    g.bias_add("c1.conv", param("c1.b", (c,), 0.1), "c1.bias")
    g.relu("c1.bias", "c1.relu")
    # width-axis matmul by a parameter, standalone bias + relu, scale, mul with the skip
    g.matmul("c1.relu", param("mm.B", (w, w), (3 / w) ** 0.5), "mm")
    g.bias_add("mm", param("mm.b", (c,), 0.1), "mm.bias")
    g.relu("mm.bias", "mm.relu")
    g.elementwise(["mm.relu"], "sc", fn="scale", alpha=0.5)
    g.elementwise(["sc", "c1.relu"], "mul", fn="mul")
    g.elementwise(["mul", "c1.relu"], "mul2", fn="add")
    g.relu("mul2", "mul.relu")          # standalone relu (after an add that no conv absorbs)
    # bias-less conv (relu fused into it)
    g.conv2d("mul.relu", param("c2.w", (c, c, 1, 1), (6 / c) ** 0.5), "c2.conv", kh=1, kw=1, cin=c, cout=c)
    g.relu("c2.conv", "c2.relu")
    g.concat(["c2.relu", "c1.relu"], "cat")
    g.conv2d("cat", param("head.w", (3, 2 * c, 1, 1), (6 / (2 * c)) ** 0.5), "head.conv", kh=1, kw=1, cin=2 * c,
             cout=3)
    g.bias_add("head.conv", param("head.b", (3,), 0.0), "head")
    g.softmax_ce("head", "labels", "class_weights", "loss", classes=3)
    return g, p, "head", "loss"


def build_wide(seed=0, cin=8, h=16, w=16):
    """Width-changing matmul path: x -> conv -> relu -> matmul (w -> 2w) -> scale -> conv ->
    matmul (2w -> w) -> head."""
    rng = np.random.default_rng(seed)
    g = OpGraph()
    g.add_input("x", role="data")
    g.add_input("labels", role="aux")
    g.add_input("class_weights", role="aux")
    p = {}

    def param(name, shape, scale):
        g.add_input(name, role="param")
        p[name] = (rng.uniform(-1, 1, size=shape) * scale).astype(np.float32)
        return name

    c = 16
    g.conv2d("x", param("c1.w", (c, cin, 3, 3), (6 / (cin * 9)) ** 0.5), "c1.conv", kh=3, kw=3, cin=cin, cout=c)
    g.bias_add("c1.conv", param("c1.b", (c,), 0.1), "c1.bias")
    g.relu("c1.bias", "c1.relu")
    g.matmul("c1.relu", param("up.B", (w, 2 * w), (3 / w) ** 0.5), "up")
    g.elementwise(["up"], "up.sc", fn="scale", alpha=1.5)
    g.conv2d("up.sc", param("c2.w", (c, c, 3, 3), (6 / (c * 9)) ** 0.5), "c2.conv", kh=3, kw=3, cin=c, cout=c)
    g.bias_add("c2.conv", param("c2.b", (c,), 0.1), "c2.bias")
    g.relu("c2.bias", "c2.relu")
    g.matmul("c2.relu", param("down.B", (2 * w, w), (1.5 / w) ** 0.5), "down")
    g.conv2d("down", param("head.w", (3, c, 1, 1), (6 / c) ** 0.5), "head.conv", kh=1, kw=1, cin=c, cout=3)
    g.bias_add("head.conv", param("head.b", (3,), 0.0), "head")
    g.softmax_ce("head", "labels", "class_weights", "loss", classes=3)
    return g, p, "head", "loss"
