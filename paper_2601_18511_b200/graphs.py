"""CUDA-graph replay of an op on fixed buffers (the launch-bound paths: the Rhombus PCMv's ~150 and the
slot-domain PCMM's ~30 small launches per op).

    g = OpGraph(lambda: pcmv_rhombus(ctx, plan, keys, x))   # one warm-up, then capture
    g.replay()                                              # same device work, one launch
    y = g.result                                            # the captured call's return value (its buffers)

Every op of this package is capturable: all scratch is caller-provided or allocated with
cudaMallocAsync, nothing synchronises the host.  Replay re-runs the device work on the buffers the
captured call used (write new inputs into them in place); the Python-side ledger is charged once,
by the captured call, so a caller that replays k times adds k - 1 op's counts itself.
Measured (one B200): Rhombus 4096x11008 2.76 -> 2.45 ms, slot PCMM d = 128 0.45 -> 0.35 ms; the
MLWE PCMM (six long kernels) and ring packing gain ~1%.
"""

from __future__ import annotations

from .context import _torch


class OpGraph:
    def __init__(self, fn, warmup: int = 1):
        torch = _torch()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):   # warm-up off the capture (workspaces, lazily created buffers)
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.result = fn()

    def replay(self):
        self.graph.replay()
        return self.result
