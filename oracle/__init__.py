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
  reverse_factor               pinned (exhaustive over q; relative-error bound)
  wino_conv, scaling on        pinned only by invariants and the power-of-two
                               special case; general values: parity unpinned
                               beyond those invariants (A21/A17)
"""
from .oracle import *  # noqa: F401,F403
