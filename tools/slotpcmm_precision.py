"""Slot-domain PCMM precision at N = 2^16 (d x d in the slots) against the plan's precision options: eager /
lazy ModDown and the weight / operand scale split pt_shift.  GPU tool."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import (HeContext, HeParams, clear_slot_pcmm, decrypt_packed, encrypt_packed,
                                   make_slot_pcmm_plan, pcmm_slot_bsgs, slot_pcmm_keygen)

ctx = HeContext(HeParams.llama(), rng="seeded")
sk = ctx.keygen(1)
for d in (128, 64):
    rng = np.random.default_rng(d)
    W = rng.uniform(-1, 1, (d, d)) / math.sqrt(d)
    B = rng.uniform(-1, 1, (d, d))
    ref = clear_slot_pcmm(W, B, 0)
    for lazy in (False, True):
        for t in (0, 2, 3, 4, 5, 6):
            if not lazy and t > 0:
                continue
            try:
                plan = make_slot_pcmm_plan(ctx, W, shear_power=0, pt_shift=t, lazy=lazy)
            except Exception as exc:
                print(f"d={d} lazy={lazy} t={t}: {exc}")
                continue
            keys = slot_pcmm_keygen(ctx, sk, plan, seed=2)
            X = encrypt_packed(ctx, sk, B, 1, seed=3, scale=plan.input_scale)
            Y = pcmm_slot_bsgs(ctx, plan, keys, X)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                Y = pcmm_slot_bsgs(ctx, plan, keys, X)
            e1.record()
            torch.cuda.synchronize()
            err = np.abs(decrypt_packed(ctx, sk, Y) - ref).max()
            print(f"d={d} split {plan.split.baby}x{plan.split.giant} lazy={lazy} pt_shift={t}: "
                  f"{-math.log2(err / np.abs(ref).max()):.1f} bits, {e0.elapsed_time(e1) / 5:.3f} ms/op", flush=True)
