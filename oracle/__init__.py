"""CPU oracle for the quadsim hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package (``paper_2509_10247_b200``) never
imports it: its GPU path fails loudly when the CUDA library is missing.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference
(``/root/reference/pkg/src/quadsim``, importable in the dev container) and
commits its outputs as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks this restatement against every fixture (fp64, ~1e-12).
"""

from oracle.quadsim_oracle import *  # noqa: F401,F403
