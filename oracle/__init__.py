"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's hot path.

This package is the parity oracle for the B200 kernels.  It restates, in
NumPy, the algorithms of the reference package `deskdl` on the training-step
path (convolution kernels, tape executor, weighted CE, LARC/SGD, FLOP rules,
synthetic scenes).  Each function cites the reference file:line it follows.

Pinning: tests/test_oracle.py checks this restatement against golden vectors
produced by the reference itself (tests/golden/make_golden.py imports deskdl
from /root/reference in the build container and commits .npz fixtures).

Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline / reference
arm may import this package.  The product (paper_1810_01993_b200) never does.
"""
