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
def rhombus_shards(n_out: int, n_in: int, n: int, world: int, strategy: str = "auto") -> list[dict]:
    """Piece-aligned slices of W for the Rhombus PCMv.

    A piece is n = rhombus_degree vector elements.  "rows": split the output pieces (each rank packs
    whole output pieces -- no reduction, words identical to one GPU); "cols": split the input pieces
    (every rank packs partial sums of all output pieces -- a ciphertext sum mod q, then one rescale);
    "auto": whichever dimension has more pieces (rows on ties).  Returns per rank
    {"rows": (r0, r1), "cols": (c0, c1), "opiece0": .., "piece0": ..}; a rank with nothing to do gets
    an empty slice (r0 == r1 or c0 == c1) and contributes a zero partial."""
    if world < 1:
        raise ValueError("world must be >= 1")
    p_out, p_in = -(-n_out // n), -(-n_in // n)
    if strategy == "auto":
        strategy = "rows" if p_out >= p_in else "cols"
    if strategy not in ("rows", "cols"):
        raise ValueError(f"unknown Rhombus shard strategy {strategy!r}")
    pieces = p_out if strategy == "rows" else p_in
    base, extra = divmod(pieces, world)
    out, p0 = [], 0
    for r in range(world):
        p1 = p0 + base + (1 if r < extra else 0)
        if strategy == "rows":
            out.append({"strategy": "rows", "rows": (min(p0 * n, n_out), min(p1 * n, n_out)), "cols": (0, n_in),
                        "opiece0": p0, "piece0": 0})
        else:
            out.append({"strategy": "cols", "rows": (0, n_out), "cols": (min(p0 * n, n_in), min(p1 * n, n_in)),
                        "opiece0": 0, "piece0": p0})
        p0 = p1
    return out


def pcmv_rhombus_sharded(ctx, W, keys, x, group=None, strategy: str = "auto"):
    """Rhombus PCMv with W sliced over the ranks of `group`: each rank builds the plan of its slice,
    runs it on the (broadcast) input to a level-1 partial output, the partials are all-gathered
    (2 x 2 x N words each) and summed mod q_i with one rescale (he_rhombus_combine).  Returns the
    same level-0 CtVector on every rank."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from .rhombus import combine_rhombus_parts, make_rhombus_plan, pcmv_rhombus_shard

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    W = np.asarray(W, dtype=np.float64) if not isinstance(W, torch.Tensor) else W
    broadcast_input(x.data, group)
    n_out, n_in = int(W.shape[0]), int(W.shape[1])
    sl = rhombus_shards(n_out, n_in, ctx.params.rhombus_degree, world, strategy)[rank]
    (r0, r1), (c0, c1) = sl["rows"], sl["cols"]
    N = ctx.params.N
    if r1 > r0 and c1 > c0:
        plan = make_rhombus_plan(ctx, W[r0:r1, c0:c1])
        part = pcmv_rhombus_shard(ctx, plan, keys, x, sl["piece0"], sl["opiece0"])
    else:
        part = torch.zeros((2, 2, N), dtype=torch.int32, device=ctx.device)
    if world > 1:
        parts = torch.empty((world, 2, 2, N), dtype=torch.int32, device=ctx.device)
        all_gather_into(parts, part[None], group)
    else:
        parts = part[None]
    return combine_rhombus_parts(ctx, parts, n_out)


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
