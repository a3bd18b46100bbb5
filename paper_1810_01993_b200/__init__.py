"""B200-native (sm_100a) data-parallel DeepLabv3+ / FC-DenseNet training step.

Drop-in for the hot path of the reference package `deskdl`
(pkg/src/deskdl/harness/trainer.py:370-387): model / loss / optimizer /
train-step API on the host, tcgen05 tensor-core kernels in libb2dl.so behind a
C ABI (include/b2dl.h).  Every compute module imports `_lib`, which loads the
native library or raises: there is no CPU fallback.
"""

__version__ = "0.1.0"
