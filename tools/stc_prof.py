"""One warm-up + one profiled SlotToCoeffs (N = 2^16, one ct) for ncu captures.  GPU tool."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import HeContext, HeParams
from paper_2601_18511_b200.stc import encrypt_slots, make_slot_to_coeffs_plan, slot_to_coeffs, slot_to_coeffs_keygen

ctx = HeContext(HeParams.llama(), rng="seeded")
sk = ctx.keygen(1)
P = ctx.params
plan = make_slot_to_coeffs_plan(ctx)
keys = slot_to_coeffs_keygen(ctx, sk, plan, seed=2)
X = encrypt_slots(ctx, sk, np.random.default_rng(0).uniform(-1, 1, (P.mlwe_degree // 2, 6 * P.mlwe_rank)), seed=3)
slot_to_coeffs(ctx, plan, keys, X)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
slot_to_coeffs(ctx, plan, keys, X)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
