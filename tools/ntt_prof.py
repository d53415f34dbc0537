"""Profiling driver for the K2 NTT: forward + inverse at 4096 (16 384 polys) and 2^16 (1024 polys), 268 MB each
(the bench's `ntt` block sizes).  Run under ncu (tools/gpu_nttprof.sh)."""
import sys; sys.path.insert(0, '.')
import torch
from paper_2601_18511_b200 import HeContext, HeParams, native
ctx = HeContext(HeParams.llama(), rng="seeded")
for n, batch in ((4096, 16384), (65536, 1024)):
    x = torch.randint(0, ctx.params.moduli[0], (batch, n), dtype=torch.int64, device="cuda").to(torch.int32)
    for _ in range(2):
        native.call("he_ntt_forward", ctx.handle, x.data_ptr(), n, 0, batch, n, ctx.stream())
        native.call("he_ntt_inverse", ctx.handle, x.data_ptr(), n, 0, batch, n, ctx.stream())
torch.cuda.synchronize()
