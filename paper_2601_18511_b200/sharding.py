"""Row-sharded MLWE PCMM over the GPUs of one box.

"We broadcast the total 128 x 4096 ciphertext matrix right before matrix
multiplication.  Each GPU then computes the matrix multiplication only for the
assigned partial plaintext matrix ... in a balanced manner."

Output rows of W shard in k-row blocks (one output RLWE block each); both limbs stay
on a rank, so the fused rescale stays local.  The only data-path collectives are the
input broadcast (C2) and the all-gather of the output blocks (C1); shards are padded to
equal size so one ``all_gather_into_tensor`` (NCCL on NVLink, or gloo in the CPU tests)
moves them.
"""

from __future__ import annotations

import math


def row_shards(n_out: int, k: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous split of the n_out/k output row-blocks: [(b0, b1)] per rank,
    sizes differ by at most one (the first blocks % world ranks take the extra block)."""
    if n_out % k:
        raise ValueError(f"n_out ({n_out}) must be a multiple of k = {k}")
    if world < 1:
        raise ValueError("world must be >= 1")
    blocks = n_out // k
    base, extra = divmod(blocks, world)
    spans, b0 = [], 0
    for r in range(world):
        b1 = b0 + base + (1 if r < extra else 0)
        spans.append((b0, b1))
        b0 = b1
    return spans


def shard_slots(n_out: int, k: int, world: int) -> int:
    return math.ceil((n_out // k) / world)


def broadcast_input(data, group=None, src: int = 0):
    """C2: every rank needs the whole input ciphertext batch."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(data, src=src, group=group)
    return data


def gather_row_shards(local_b, local_a, k: int, n_out: int, group=None):
    """C1: all-gather the padded per-rank output shards and trim the padding.

    local_b: [per, N] composed b' blocks of this rank (rows past its real blocks ignored)
    local_a: [per * k, N] a' rows.  Returns (out_b [n_out/k, N], out_a [n_out, N]).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local_b[: n_out // k], local_a[:n_out]
    per = local_b.shape[0]
    all_b = torch.empty((per * world,) + tuple(local_b.shape[1:]), dtype=local_b.dtype, device=local_b.device)
    all_a = torch.empty((per * world * k,) + tuple(local_a.shape[1:]), dtype=local_a.dtype, device=local_a.device)
    dist.all_gather_into_tensor(all_b, local_b.contiguous(), group=group)
    dist.all_gather_into_tensor(all_a, local_a.contiguous(), group=group)
    # every shard is padded at its end to `per` slots; keep each rank's real blocks
    spans = row_shards(n_out, k, world)
    keep_b = torch.cat([all_b[r * per: r * per + (b1 - b0)] for r, (b0, b1) in enumerate(spans)])
    keep_a = torch.cat([all_a[r * per * k: (r * per + (b1 - b0)) * k] for r, (b0, b1) in enumerate(spans)])
    return keep_b, keep_a


def symmetric_outputs(ctx, n_out: int, group=None):
    """Full-size output buffers in symmetric (peer-mappable) memory plus every rank's pointers to them,
    or None when symmetric memory is unavailable (no NVLink P2P, single rank, older torch)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    try:
        import torch.distributed._symmetric_memory as symm

        p = ctx.params
        grp = group if group is not None else dist.group.WORLD
        out_b = symm.empty((n_out // p.mlwe_rank, p.N), dtype=torch.int32, device=ctx.device)
        out_a = symm.empty((n_out, p.N), dtype=torch.int32, device=ctx.device)
        hb = symm.rendezvous(out_b, grp)
        ha = symm.rendezvous(out_a, grp)
        return out_b, out_a, list(hb.buffer_ptrs), list(ha.buffer_ptrs), hb
    except Exception:  # pragma: no cover - depends on the box
        return None


def pcmm_mlwe_sharded_fused(ctx, plan, X, n_out: int, row0: int, sym, group=None):
    """Row-sharded op with the output all-gather fused into the kernels' stores: this rank's rows
    [row0, row0 + plan.n_out) go straight into every rank's full output (symmetric memory over
    NVLink, ``sym`` from symmetric_outputs); a barrier on the symmetric handle publishes them."""
    from .pcmm import pcmm_mlwe_into_peers

    out_b, out_a, ptr_b, ptr_a, handle = sym
    broadcast_input(X.data, group)
    pcmm_mlwe_into_peers(ctx, plan, X, ptr_b, ptr_a, row0)
    handle.barrier()
    return out_b, out_a


def pcmm_mlwe_sharded(ctx, plan, X, n_out: int, group=None, out_b=None, out_a=None):
    """Run this rank's shard (``plan`` holds rows [b0*k, b1*k) of W) between the input
    broadcast and the output all-gather.  Returns the gathered (out_b, out_a)."""
    import torch
    import torch.distributed as dist

    from .context import MlweBlocks
    from .pcmm import pcmm_mlwe

    p = ctx.params
    k = p.mlwe_rank
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    per = shard_slots(n_out, k, world)
    if out_b is None:
        out_b = torch.zeros((per, p.N), dtype=torch.int32, device=ctx.device)
        out_a = torch.zeros((per * k, p.N), dtype=torch.int32, device=ctx.device)
    rows = plan.n_out
    broadcast_input(X.data, group)
    pcmm_mlwe(ctx, plan, X, out=MlweBlocks(out_b[: rows // k], out_a[:rows], level=0, n_rows=rows))
    return gather_row_shards(out_b, out_a, k, n_out, group)
