"""One warm-up + one profiled slot-domain PCMM (d = 128, N = 2^16) for ncu captures.  GPU tool."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import (HeContext, HeParams, encrypt_packed, make_slot_pcmm_plan, pcmm_slot_bsgs,
                                   slot_pcmm_keygen)

ctx = HeContext(HeParams.llama(), rng="seeded")
sk = ctx.keygen(1)
d = 128
rng = np.random.default_rng(0)
plan = make_slot_pcmm_plan(ctx, rng.uniform(-1, 1, (d, d)) / np.sqrt(d))
keys = slot_pcmm_keygen(ctx, sk, plan, seed=2)
X = encrypt_packed(ctx, sk, rng.uniform(-1, 1, (d, d)), 1, seed=3)
pcmm_slot_bsgs(ctx, plan, keys, X)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
pcmm_slot_bsgs(ctx, plan, keys, X)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
