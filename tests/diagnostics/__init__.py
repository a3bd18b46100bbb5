"""Diagnostics run by hand on a GPU box (test infrastructure: they read the oracle).  Not
collected by pytest (no test_ functions); run from the repo root, e.g.
`python tests/diagnostics/fp32_flips.py`."""
