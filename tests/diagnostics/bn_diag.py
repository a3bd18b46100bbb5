"""Per-tensor gradient errors of the batch-norm DeepLab (bf16 GPU and the bf16-storage emulation,
both vs float64) -- development aid."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import deskdl_port as O  # noqa: E402
from oracle.bf16_emulation import emulated_step  # noqa: E402
sys.path.insert(0, "tests")
from test_gpu_norm import _batch, _bn_net, rel  # noqa: E402

net = _bn_net(sys.argv[1] if len(sys.argv) > 1 else "bf16")
x, labels = _batch()
cw = O.class_weights((0.982, 0.017, 0.001))
p64 = {k: v.astype(np.float64) for k, v in net.params.items()}
l64, lg64, g64, _ = O.train_step(net.graph, p64, net.param_order, x.astype(np.float64), labels, cw.astype(np.float64),
                                 net.loss_name, net.logits_name)
el, elg, eg = emulated_step(net.graph, net.params, x, labels, cw, net.loss_name, net.logits_name)
loss, logits, tape = net.forward_loss(x, labels, cw)
gg = net.backward(tape)
print("loss ref %.6f gpu %.6f emu %.6f" % (l64, loss, el))
print("logits gpu %.3e emu %.3e" % (rel(logits.cpu().numpy(), lg64), rel(elg, lg64)))
for k in net.param_order:
    print("%-22s |ref| %.2e  gpu %.3e  emu %.3e" % (k, np.max(np.abs(g64[k])), rel(gg[k], g64[k]), rel(eg[k], g64[k])))
