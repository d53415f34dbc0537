"""Worker for tests/test_gpu_multirank.py: several ranks (torchrun, gloo) sharing one GPU run the
sharded MLWE PCMM and the sharded Rhombus PCMv through the real distributed code path and check
them against the one-rank results computed in-process."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist

from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, pcmm_mlwe
from paper_2601_18511_b200.rhombus import (clear_pcmv, decrypt_vector, encrypt_vector, make_rhombus_plan,
                                           pcmv_rhombus, rhombus_keygen)
from paper_2601_18511_b200.sharding import pcmm_mlwe_sharded, pcmv_rhombus_sharded, row_shards


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    P = HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    k = P.mlwe_rank
    rng = np.random.default_rng(1)
    # MLWE PCMM, row-sharded
    n_out, n_in = 1024, 512
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    sk = ctx.keygen(7)
    X = ctx.encrypt_acts(sk, A, seed=11)
    ref = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W), X)
    b0, b1 = row_shards(n_out, k, world)[rank]
    plan = make_mlwe_pcmm_plan(ctx, W[b0 * k: b1 * k])
    out_b, out_a = pcmm_mlwe_sharded(ctx, plan, X, n_out)
    assert torch.equal(out_b, ref.out_b) and torch.equal(out_a, ref.out_a), "sharded PCMM words differ"
    # the fused all-gather: every rank's kernels store into every rank's output (symmetric memory)
    from paper_2601_18511_b200.sharding import pcmm_mlwe_sharded_fused, symmetric_outputs

    sym = symmetric_outputs(ctx, n_out)
    fused = "unavailable"
    if sym is not None:
        fb, fa = pcmm_mlwe_sharded_fused(ctx, plan, X, n_out, b0 * k, sym)
        torch.cuda.synchronize()
        assert torch.equal(fb, ref.out_b) and torch.equal(fa, ref.out_a), "fused peer-store PCMM words differ"
        fused = "ok"
    # PCMM + ring packing, row-sharded (each rank packs its blocks, packed blocks all-gathered)
    from paper_2601_18511_b200 import make_ring_pack_plan, pcmm_packed, ring_pack_keygen
    from paper_2601_18511_b200.sharding import pcmm_packed_sharded

    rkeys = ring_pack_keygen(ctx, sk, seed=21)
    full_p = pcmm_packed(ctx, make_mlwe_pcmm_plan(ctx, W), make_ring_pack_plan(ctx, n_out), rkeys, X)
    Yp = pcmm_packed_sharded(ctx, plan, make_ring_pack_plan(ctx, (b1 - b0) * k), rkeys, X, n_out)
    assert torch.equal(Yp.data, full_p.data), "sharded packed output differs"
    # Rhombus PCMv, both strategies
    for (n_o, n_i, strat) in ((8192, 4096, "rows"), (4096, 8192, "cols")):
        v = rng.uniform(-1, 1, n_i)
        Wr = rng.uniform(-1, 1, (n_o, n_i)) / np.sqrt(n_i)
        keys = rhombus_keygen(ctx, sk, 99)
        x = encrypt_vector(ctx, sk, v, seed=5)
        full = pcmv_rhombus(ctx, make_rhombus_plan(ctx, Wr), keys, x)
        y = pcmv_rhombus_sharded(ctx, Wr, keys, x, strategy=strat)
        res = decrypt_vector(ctx, keys.s_up_ntt, y)
        if strat == "rows":
            assert torch.equal(y.data, full.data), "row-sharded PCMv words differ"
        else:
            assert np.abs(res - decrypt_vector(ctx, keys.s_up_ntt, full)).max() < 2 ** -18
        assert np.abs(res - clear_pcmv(Wr, v)).max() < 2 ** -13
    dist.barrier()
    if rank == 0:
        print("multirank ok", world, "fused", fused)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
