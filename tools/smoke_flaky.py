"""Run __graft_entry__.smoke() with the StC assertion instrumented: on a mismatch print which words differ.
GPU tool (investigating an intermittent smoke failure)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

_orig = np.array_equal
state = {}


def _eq(a, b, *args, **kw):
    r = _orig(a, b, *args, **kw)
    if not r and getattr(a, "shape", None) == getattr(b, "shape", None) and a.ndim == 2:
        d = np.argwhere(a != b)
        print(f"MISMATCH shape {a.shape}: {len(d)} words differ; rows {sorted(set(d[:, 0].tolist()))[:4]}, "
              f"cols {d[:8, 1].tolist()} ... got {a[tuple(d[0])]} want {b[tuple(d[0])]}", flush=True)
    return r


np.array_equal = _eq
import __graft_entry__ as g

try:
    g.smoke()
    print("SMOKE OK")
except AssertionError as e:
    print("SMOKE FAIL", e)
