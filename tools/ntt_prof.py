import sys; sys.path.insert(0, '.')
import torch
from paper_2601_18511_b200 import HeContext, HeParams, native
ctx = HeContext(HeParams.llama(), rng="seeded")
for n, batch in ((4096, 4096), (65536, 256)):
    x = torch.randint(0, ctx.params.moduli[0], (batch, n), dtype=torch.int64, device="cuda").to(torch.int32)
    for _ in range(2):
        native.call("he_ntt_forward", ctx.handle, x.data_ptr(), n, 0, batch, n, ctx.stream())
torch.cuda.synchronize()
