"""Generate the golden fixtures under tests/golden/ from the reference package.

Run in the build container (where /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports hesim read-only and records:
  bitrev_golden.npz -- bit_reverse tables (k = 3, 7, 8, 11), rotate_bits_down(.,8),
                       byte_mix, half_reverse over their full domains; shuffle_matrix of a
                       seeded 256x256 matrix; hesim.bitrev.check_all() results.
  pcmm_toy_golden.npz -- BASELINE config 1: hesim's own slot-domain PCMM at d = 16 on
                       256 slots (pcmm_bsgs, decoded) and clear_pcmm for seeded W, M, plus
                       the pinned 2x2 example of test_matmul.py:55-65.
The GPU/CPU tests read only these files; nothing at test time touches /root/reference.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def main():
    import hesim
    from hesim import bitrev
    from hesim.packing import decode_packed

    tabs = {}
    for k in (3, 7, 8, 11):
        tabs[f"bit_reverse_{k}"] = np.array([hesim.bit_reverse(x, k) for x in range(1 << k)], dtype=np.int64)
    tabs["rotate_bits_down_8"] = np.array([bitrev.rotate_bits_down(x, 8) for x in range(256)], dtype=np.int64)
    tabs["byte_mix"] = np.array([hesim.byte_mix(x) for x in range(256)], dtype=np.int64)
    tabs["half_reverse"] = np.array([hesim.half_reverse(x) for x in range(4096)], dtype=np.int64)
    m = np.random.default_rng(0).uniform(-1, 1, (256, 256))
    tabs["shuffle_input"] = m
    tabs["shuffle_output"] = hesim.shuffle_matrix(m)
    rep = bitrev.check_all()
    tabs["check_all_names"] = np.array(list(rep.keys()))
    tabs["check_all_values"] = np.array(list(rep.values()))
    np.savez_compressed(HERE / "bitrev_golden.npz", **tabs)

    # BASELINE config 1: toy PCMM, 16-column batch, decrypt-and-compare vs plaintext matmul
    rng = np.random.default_rng(2026)
    d = 16
    W = rng.uniform(-1, 1, (d, d)) / np.sqrt(d)
    M = rng.uniform(-1, 1, (d, d))
    ctx = hesim.SlotContext(hesim.SimParams(slot_count=256))
    plan = hesim.make_pcmm_plan(ctx, W, shear_power=0)
    out = hesim.pcmm_bsgs(ctx, plan, hesim.pack_sheared(ctx, M, 1))
    ledger = ctx.ledger.snapshot()
    pin_a = np.array([[1.0, 0.0], [0.0, 2.0]])
    pin_b = np.array([[1.0, 2.0], [3.0, 4.0]])
    np.savez_compressed(
        HERE / "pcmm_toy_golden.npz",
        W=W, M=M,
        hesim_bsgs=decode_packed(out),
        hesim_clear=hesim.clear_pcmm(W, M, 0),
        hesim_level_drop=np.array(hesim.SimParams(slot_count=256).top_level - out.payload.level),
        hesim_ct_rotations=np.array(ledger["ct_rotations"]),
        pin_clear_2x2_power1=hesim.clear_pcmm(pin_a, pin_b, 1),
        pin_clear_2x2_power0=hesim.clear_pcmm(pin_a, pin_b, 0),
    )
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))


if __name__ == "__main__":
    main()
