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

import ctypes
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


def _staged(t, group) -> bool:
    """gloo moves host tensors: device tensors are staged through host memory (CPU tests and
    several ranks sharing one GPU); NCCL moves device memory directly over NVLink."""
    import torch.distributed as dist

    return t.is_cuda and dist.get_backend(group) != "nccl"


def all_gather_into(out, t, group=None):
    import torch.distributed as dist

    if _staged(t, group):
        host = out.new_empty(out.shape, device="cpu")
        dist.all_gather_into_tensor(host, t.contiguous().cpu(), group=group)
        out.copy_(host)
    else:
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    return out


def broadcast_input(data, group=None, src: int = 0):
    """C2: every rank needs the whole input ciphertext batch."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if _staged(data, group):
            host = data.cpu()
            dist.broadcast(host, src=src, group=group)
            data.copy_(host)
        else:
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
    all_gather_into(all_b, local_b, group)
    all_gather_into(all_a, local_a, group)
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
        pass
    try:
        return ipc_outputs(ctx, n_out, group)
    except Exception:  # pragma: no cover - no CUDA IPC on this box
        return None


class _IpcBuffers:
    """Full-size output buffers allocated with cudaMalloc and mapped into every rank with CUDA IPC
    (cudaIpcGetMemHandle / cudaIpcOpenMemHandle, peer access over NVLink enabled lazily): the
    symmetric-memory fallback for process groups without it (e.g. gloo).  barrier() publishes the
    peer stores: device sync, then a group barrier."""

    def __init__(self, nbytes: list, device, group):
        import ctypes

        import torch
        import torch.distributed as dist

        class Handle(ctypes.Structure):  # cudaIpcMemHandle_t, passed by value
            _fields_ = [("reserved", ctypes.c_char * 64)]

        self.group = group
        self.rt = ctypes.CDLL("libcudart.so.12")
        self.rt.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
        self.rt.cudaIpcGetMemHandle.argtypes = [ctypes.POINTER(Handle), ctypes.c_void_p]
        self.rt.cudaIpcOpenMemHandle.argtypes = [ctypes.POINTER(ctypes.c_void_p), Handle, ctypes.c_uint]
        torch.cuda.set_device(device)
        self.local, self.opened = [], []
        handles = []
        for nb in nbytes:
            ptr = ctypes.c_void_p()
            if self.rt.cudaMalloc(ctypes.byref(ptr), nb):
                raise RuntimeError("cudaMalloc failed")
            self.local.append(ptr.value)
            h = Handle()
            if self.rt.cudaIpcGetMemHandle(ctypes.byref(h), ptr):
                self.rt.cudaGetLastError()
                raise RuntimeError("cudaIpcGetMemHandle failed")
            handles.append(ctypes.string_at(ctypes.addressof(h), 64))
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        every = [None] * world
        dist.all_gather_object(every, handles, group=group)
        self.ptrs = []   # ptrs[i][r]: buffer i of rank r as seen from this rank
        for i in range(len(nbytes)):
            row = []
            for r in range(world):
                if r == rank:
                    row.append(self.local[i])
                    continue
                p = ctypes.c_void_p()
                if self.rt.cudaIpcOpenMemHandle(ctypes.byref(p), Handle.from_buffer_copy(every[r][i]), 1):
                    self.rt.cudaGetLastError()
                    raise RuntimeError("cudaIpcOpenMemHandle failed")
                self.opened.append(p.value)
                row.append(p.value)
            self.ptrs.append(row)

    def barrier(self):
        import torch
        import torch.distributed as dist

        torch.cuda.synchronize()
        dist.barrier(group=self.group)

    def __del__(self):  # unmap the peers' buffers, then free our own
        try:
            self.rt.cudaIpcCloseMemHandle.argtypes = [ctypes.c_void_p]
            self.rt.cudaFree.argtypes = [ctypes.c_void_p]
            for ptr in self.opened:
                self.rt.cudaIpcCloseMemHandle(ptr)
            for ptr in self.local:
                self.rt.cudaFree(ptr)
        except Exception:
            pass


def _device_view(ptr: int, shape, device):
    """int32 torch tensor over raw device memory (kept alive by the _IpcBuffers owner)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<i4", "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_Arr(), device=device)


def ipc_outputs(ctx, n_out: int, group=None):
    import torch.distributed as dist

    p = ctx.params
    shp_b, shp_a = (n_out // p.mlwe_rank, p.N), (n_out, p.N)
    bufs = _IpcBuffers([shp_b[0] * shp_b[1] * 4, shp_a[0] * shp_a[1] * 4], ctx.device, group)
    out_b = _device_view(bufs.local[0], shp_b, ctx.device)
    out_a = _device_view(bufs.local[1], shp_a, ctx.device)
    out_b._ipc_owner = bufs   # keep the mappings alive with the views
    out_a._ipc_owner = bufs
    del dist
    return out_b, out_a, bufs.ptrs[0], bufs.ptrs[1], bufs


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


# ---------------------------------------------------------------- Rhombus PCMv over several GPUs
def rhombus_shards(n_out: int, n_in: int, n: int, world: int, strategy: str = "auto", window: int | None = None,
                   rho: int | None = None) -> list[dict]:
    """Per-rank work of the Rhombus PCMv the way PAPER.md:87 splits it.

    "cols" -- "the ciphertext is masked and each GPU is assigned 4096/8 values": the input pieces
    (window w values each) are split over the ranks, each rank runs its columns against all rows and
    the level-1 partial outputs are summed (one ciphertext sum mod q_i, then one rescale).  At
    n_in = 4096 the default window is 256, i.e. 16 pieces: 2 pieces = 512 values per rank at 8 GPUs.
    "rows" -- "broadcast the ciphertext ... split the plaintext matrix": every rank owns the leaves
    j = g + G jl of every output piece (G = the largest power of two <= world, <= w): rows
    n o + h(u w + j), n / G of each output piece, with its packing subtree; the G subtree roots are
    gathered and the top log2 G levels finish the packing -- output words identical to one GPU.
    "auto": cols when n_in fits one degree-n piece (4096x4096, 11008x4096, 14336x4096), rows
    otherwise (4096x11008, 4096x14336) -- the paper's choice.
    Returns per rank {"strategy", "cols": (c0, c1), "piece0", "groups", "group", "active"}."""
    if world < 1:
        raise ValueError("world must be >= 1")
    w = n if window is None else int(window)
    p_in = -(-n_in // w)
    if strategy == "auto":
        strategy = "cols" if n_in <= n and p_in >= world else "rows"
    if strategy not in ("rows", "cols"):
        raise ValueError(f"unknown Rhombus shard strategy {strategy!r}")
    out = []
    if strategy == "cols":
        base, extra = divmod(p_in, world)
        p0 = 0
        for r in range(world):
            p1 = p0 + base + (1 if r < extra else 0)
            c0, c1 = min(p0 * w, n_in), min(p1 * w, n_in)
            out.append({"strategy": "cols", "cols": (c0, c1), "piece0": p0, "groups": 1, "group": 0,
                        "active": c1 > c0})
            p0 = p1
        return out
    G = 1
    while G * 2 <= min(world, w):
        G *= 2
    for r in range(world):
        out.append({"strategy": "rows", "cols": (0, n_in), "piece0": 0, "groups": G, "group": r if r < G else 0,
                    "active": r < G})
    return out


def pcmv_rhombus_sharded(ctx, W, keys, x, group=None, strategy: str = "auto"):
    """Rhombus PCMv split over the ranks of `group` (rhombus_shards).  Column shards: each rank's plan
    covers its input pieces, the level-1 partial outputs (2 x 2 x N words each) are all-gathered and
    summed mod q_i with one rescale (he_rhombus_combine).  Row shards: each rank runs its leaves'
    products and packing subtree, the subtree roots (2 x p_out x 2 x n words each) are all-gathered and
    every rank finishes the top packing levels (he_rhombus_finish).  Returns the same level-0 CtVector
    on every rank."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from .rhombus import (combine_rhombus_parts, finish_rhombus_subtrees, make_rhombus_plan, pcmv_rhombus_shard,
                          pcmv_rhombus_subtree)

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    W = np.asarray(W, dtype=np.float64) if not isinstance(W, torch.Tensor) else W
    broadcast_input(x.data, group)
    n_out, n_in = int(W.shape[0]), int(W.shape[1])
    P = ctx.params
    n, N = P.rhombus_degree, P.N
    win = x.window or n
    sl = rhombus_shards(n_out, n_in, n, world, strategy, window=win)[rank]
    if sl["strategy"] == "cols":
        c0, c1 = sl["cols"]
        if sl["active"]:
            plan = make_rhombus_plan(ctx, W[:, c0:c1], window=win)
            part = pcmv_rhombus_shard(ctx, plan, keys, x, sl["piece0"], 0)
        else:
            part = torch.zeros((2, 2, N), dtype=torch.int32, device=ctx.device)
        if world > 1:
            parts = torch.empty((world, 2, 2, N), dtype=torch.int32, device=ctx.device)
            all_gather_into(parts, part[None], group)
        else:
            parts = part[None]
        return combine_rhombus_parts(ctx, parts, n_out)
    G = sl["groups"]
    plan = make_rhombus_plan(ctx, W, window=win, groups=G, group=sl["group"])
    p_out = -(-n_out // n)
    if sl["active"]:
        roots = pcmv_rhombus_subtree(ctx, plan, keys, x)
    else:
        roots = torch.zeros((2, p_out, 2, n), dtype=torch.int32, device=ctx.device)
    if world > 1:
        allr = torch.empty((world, 2, p_out, 2, n), dtype=torch.int32, device=ctx.device)
        all_gather_into(allr, roots[None], group)
        allr = allr[:G]
    else:
        allr = roots[None]
    return finish_rhombus_subtrees(ctx, plan, keys, allr)


def all_reduce_max(t, group=None):
    """MAX all-reduce (timings: the max over ranks), staged through the host for gloo."""
    import torch.distributed as dist

    if _staged(t, group):
        host = t.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.MAX, group=group)
        return host.to(t.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def pcmm_packed_sharded(ctx, plan, rp, keys, X, n_out: int, group=None):
    """Row-sharded PCMM + ring packing: this rank's plans cover output row-blocks [b0, b1) (row_shards);
    each rank packs its own blocks and the packed level-0 RLWE blocks (2 N words each, ~128x less than
    the MLWE rows) are all-gathered.  Returns CtBlocks [n_out/k, 1, 2, N] on every rank."""
    import torch
    import torch.distributed as dist

    from .context import CtBlocks
    from .ringpack import pcmm_packed

    p = ctx.params
    k = p.mlwe_rank
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    per = shard_slots(n_out, k, world)
    broadcast_input(X.data, group)
    local = torch.zeros((per, 1, 2, p.N), dtype=torch.int32, device=ctx.device)
    pcmm_packed(ctx, plan, rp, keys, X, out=local[: rp.n_out // k])
    if world == 1:
        return CtBlocks(local[: n_out // k], level=0, n_cols=n_out)
    allp = torch.empty((per * world, 1, 2, p.N), dtype=torch.int32, device=ctx.device)
    all_gather_into(allp, local, group)
    keep = torch.cat([allp[r * per: r * per + (b1 - b0)] for r, (b0, b1) in enumerate(row_shards(n_out, k, world))])
    return CtBlocks(keep, level=0, n_cols=n_out)
