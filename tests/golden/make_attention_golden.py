"""Golden PC-attention values from the reference: hesim's attention_demo inputs (seeded) and its clear
oracle clear_pc_attention, for tests/test_gpu_attention.py.  Run in the build container."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hesim import SimParams, SlotContext  # noqa: E402
from hesim.packing import pack_sheared, unpack_matrix  # noqa: E402
from hesim.pipeline import clear_pc_attention, rope_columns, rope_packed  # noqa: E402

out = {}
for d, seed in ((8, 0), (16, 1), (64, 2)):
    rng = np.random.default_rng(seed)
    scale = 1.0 / np.sqrt(d)
    k_pub = rope_columns(rng.standard_normal((d, d)) * scale, np.arange(d))   # attention_demo's draws
    v_pub = rng.standard_normal((d, d)) * scale
    q = rng.standard_normal((d, d)) * scale
    positions = d + np.arange(d)
    out[f"d{d}_q"], out[f"d{d}_k"], out[f"d{d}_v"] = q, k_pub, v_pub
    out[f"d{d}_out"] = clear_pc_attention(q, k_pub, v_pub, positions)
    ctx = SlotContext(SimParams(slot_count=max(64, d * d)))
    out[f"d{d}_rope2"] = unpack_matrix(rope_packed(ctx, pack_sheared(ctx, q, 2), positions).payload.slots, d)
np.savez(Path(__file__).with_name("attention_golden.npz"), **out)
print("wrote", sorted(out))
