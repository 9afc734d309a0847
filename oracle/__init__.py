"""CPU oracle for the complex-Winograd F(4x4,3x3) int8 convolution with
integer filter-precision scaling (arXiv 1901.01965).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import,
call, link or execute anything under ``oracle/``.  The product path
(``paper_1901_01965_b200``) never imports it and shares no code with it.

Parity status per function:
  direct_conv                  pinned (torch.nn.functional.conv2d in float64)
  wino_conv, scaling off       pinned (== direct_conv exactly; Im Y == 0)
  filter/input/output tiles    pinned (identity 16*correlation, conjugate layout)
  scale_factor / codes         pinned (brute force over all (n, p); Table 1)
  filter_transform selection   pinned (per-OFM independence, maximal grid
                               factor, A5 magnitude, A16; tests/test_oracle_selection.py)
  reverse_factor               pinned (exhaustive over q; relative-error bound)
  wino_conv, scaling on        pinned by invariants, the power-of-two special
                               case (exact) and, in general, the error bound
                               derived from its three roundings against direct
                               convolution (test_oracle_selection.py); the
                               static-error POPULATION of P:376 is unstated
                               (A21): that figure alone is reported, unpinned
"""
from .oracle import *  # noqa: F401,F403
