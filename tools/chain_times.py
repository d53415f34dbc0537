"""Factorized SlotToCoeffs (chain.py) at N = 2^16: device ms per ciphertext, per-map kernel split, precision;
then the chained op (StC -> PCMM -> ring pack).  Development tool (GPU)."""
import collections
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import (HeContext, HeParams, clear_pcmm, make_mlwe_pcmm_plan, make_ring_pack_plan,
                                   pcmm_packed, ring_pack_keygen)
from paper_2601_18511_b200.chain import (encrypt_slots_at, factorized_stc_keygen, make_factorized_stc_plan,
                                         slot_to_coeffs_factorized)

P = HeParams.llama_chain()
ctx = HeContext(P, rng="seeded")
sk = ctx.keygen(7)
n_ct = int(sys.argv[1]) if len(sys.argv) > 1 else 16
A = np.random.default_rng(5).uniform(-1, 1, (P.tokens, 256 * n_ct))
plan = make_factorized_stc_plan(ctx)
keys = factorized_stc_keygen(ctx, sk, plan, seed=9)
X = encrypt_slots_at(ctx, sk, A, seed=3, scale=plan.input_scale)
for _ in range(2):
    Y = slot_to_coeffs_factorized(ctx, plan, keys, X)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    Y = slot_to_coeffs_factorized(ctx, plan, keys, X)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
err = np.abs(ctx.decrypt_acts(sk, Y) - A).max()
print(f"factorized StC: {ms:.3f} ms for {n_ct} cts = {ms / n_ct:.3f} ms/ct, {plan.rotations} rotations, "
      f"{plan.plaintexts} plaintexts, max err 2^{np.log2(err):.1f}")
from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    slot_to_coeffs_factorized(ctx, plan, keys, X)
    torch.cuda.synchronize()
tot, cnt = collections.defaultdict(float), collections.Counter()
for e in prof.events():
    if e.device_type.name == "CUDA":
        tot[e.name[:60]] += e.device_time_total
        cnt[e.name[:60]] += 1
print(f"  sum of kernels {sum(tot.values()) / 1000:.3f} ms")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {v / 1000:8.3f} ms  x{cnt[k]:5d}  {k}")
W = np.random.default_rng(6).uniform(-1, 1, (4096, 256 * n_ct)) / np.sqrt(256 * n_ct)
pp, rp, rk = make_mlwe_pcmm_plan(ctx, W), make_ring_pack_plan(ctx, 4096), ring_pack_keygen(ctx, sk, 5)
for _ in range(2):
    Z = pcmm_packed(ctx, pp, rp, rk, slot_to_coeffs_factorized(ctx, plan, keys, X))
torch.cuda.synchronize()
e0.record()
for _ in range(3):
    Z = pcmm_packed(ctx, pp, rp, rk, slot_to_coeffs_factorized(ctx, plan, keys, X))
e1.record()
torch.cuda.synchronize()
err = np.abs(ctx.decrypt_acts(sk, Z) - clear_pcmm(W, A)).max()
print(f"chained op (level 4 slots -> StC -> PCMM 4096x{256 * n_ct}x128 -> ring pack): {e0.elapsed_time(e1) / 3:.3f} ms, "
      f"max err 2^{np.log2(err):.1f}")
