"""CPU oracle for the MLWE PCMM / Rhombus PCMv path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_2601_18511_b200`` never
imports it (tests/test_boundary.py enforces that).

Parity status: PARITY UNPINNED at the integer level (see he_oracle.c header and
DESIGN.md §3); layout (bitrev.py) and float semantics (clear_pcmm) are pinned by
the golden fixtures under tests/golden/.
"""

from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
