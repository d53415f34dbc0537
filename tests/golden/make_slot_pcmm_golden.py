"""Golden values for the slot-domain PCMM from the reference's own kernel: hesim
pcmm_bsgs / pcmm_depth1 on d x d matrices (d = 16 on 256 slots: BASELINE config 1's toy; d = 8 on 256
slots with tiling), shear powers 0 and 2.  Run in the build container (needs /root/reference):
    python tests/golden/make_slot_pcmm_golden.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hesim import SimParams, SlotContext, make_pcmm_plan, pack_sheared, pcmm_bsgs, pcmm_depth1  # noqa: E402
from hesim.packing import unpack_matrix  # noqa: E402

out = {}
for d, shear in ((16, 0), (16, 2), (8, 1)):
    rng = np.random.default_rng(100 * d + shear)
    W = rng.uniform(-1, 1, (d, d)) / np.sqrt(d)
    B = rng.uniform(-1, 1, (d, d))
    ctx = SlotContext(SimParams(slot_count=256))
    plan = make_pcmm_plan(ctx, W, shear_power=shear)
    r = pcmm_bsgs(ctx, plan, pack_sheared(ctx, B, shear + 1))
    key = f"d{d}_l{shear}"
    out[key + "_W"] = W
    out[key + "_B"] = B
    out[key + "_hesim_bsgs"] = unpack_matrix(r.payload.slots, d)
    out[key + "_split"] = np.array([plan.split.baby, plan.split.giant])
    out[key + "_hesim_depth1"] = unpack_matrix(pcmm_depth1(ctx, plan, pack_sheared(ctx, B, shear + 1)).payload.slots, d)
np.savez(Path(__file__).with_name("slot_pcmm_golden.npz"), **out)
print("wrote", sorted(out))
