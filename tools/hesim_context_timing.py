"""SURVEY §8d CPU item 2: time the reference's own slot-domain PCMM (hesim pcmm_bsgs, float
simulator) at its largest feasible sizes, for context beside the integer CPU port.  Needs the
reference package (/root/reference, this container only); writes profiles/r01/hesim_pcmm_bsgs_cpu.json."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
from hesim import (SimParams, SlotContext, clear_pcmm, make_pcmm_plan, pack_sheared, pcmm_bsgs)  # noqa: E402

out = {"what": "hesim pcmm_bsgs (reference slot simulator, float64) on d x d, slot_count = d^2, host CPU",
       "cpu_count": os.cpu_count(), "results": {}}
for d in (16, 32, 64, 128):
    ctx = SlotContext(SimParams(slot_count=d * d))
    rng = np.random.default_rng(0)
    w, b = rng.standard_normal((d, d)), rng.standard_normal((d, d))
    pm = pack_sheared(ctx, b, 1)
    t0 = time.perf_counter()
    plan = make_pcmm_plan(ctx, w, shear_power=0)
    t1 = time.perf_counter()
    r = pcmm_bsgs(ctx, plan, pm)
    t2 = time.perf_counter()
    from hesim.packing import unpack_matrix
    err = float(np.max(np.abs(unpack_matrix(r.payload.slots, d) - clear_pcmm(w, b, 0))))
    out["results"][str(d)] = {"plan_s": round(t1 - t0, 4), "pcmm_bsgs_s": round(t2 - t1, 4), "max_err": err,
                              "word_macs_equiv": d ** 3}
    print(d, out["results"][str(d)], flush=True)
Path(__file__).resolve().parents[1].joinpath("profiles/r01/hesim_pcmm_bsgs_cpu.json").write_text(
    json.dumps(out, indent=1))
