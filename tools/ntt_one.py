import sys; sys.path.insert(0, '.')
import torch
from paper_2601_18511_b200 import HeContext, HeParams, native
ctx = HeContext(HeParams.llama(), rng="seeded")
x = torch.randint(0, ctx.params.moduli[0], (1024, 65536), dtype=torch.int64, device="cuda").to(torch.int32)
for _ in range(3):
    native.call("he_ntt_forward", ctx.handle, x.data_ptr(), 65536, 0, 1024, 65536, ctx.stream())
    native.call("he_ntt_inverse", ctx.handle, x.data_ptr(), 65536, 0, 1024, 65536, ctx.stream())
torch.cuda.synchronize()
