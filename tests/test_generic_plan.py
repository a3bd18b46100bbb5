"""The engine's static plan lowers every reference op kind (CPU: planning needs no GPU)."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import generic_graph  # noqa: E402
from paper_1810_01993_b200.engine import Plan  # noqa: E402


def test_plan_lowers_standalone_ops():
    for build in (generic_graph.build, generic_graph.build_wide):
        g, p, logits, loss = build()
        plan = Plan(g, {k: v.shape for k, v in p.items()}, (2, 8, 16, 16), loss, logits)
        kinds = {o.kind for o in plan.ops}
        assert {"conv", "matmul", "ce"} <= kinds
        # every parameter's gradient is produced by some backward step
        produced = set()
        for st in plan.backward_program:
            o = st["op"]
            produced.update(n for n in (o.w, o.b) if n)
        assert produced == set(p), set(p) ^ produced
    g, p, logits, loss = generic_graph.build()
    plan = Plan(g, {k: v.shape for k, v in p.items()}, (2, 8, 16, 16), loss, logits)
    kinds = [o.kind for o in plan.ops]
    for k in ("bias", "relu", "mul", "scale", "matmul", "concat"):
        assert k in kinds, (k, kinds)
    conv2 = [o for o in plan.ops if o.kind == "conv" and o.w == "c2.w"][0]
    assert conv2.b == "" and conv2.relu        # bias-less conv, relu fused into its epilogue
    bias = [o for o in plan.ops if o.kind == "bias"][0]
    assert bias.relu and bias.out == "mm.relu"  # bias_add + relu fused into one stream
