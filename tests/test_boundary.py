"""The drop-in boundary: the C-ABI library loads and exports every symbol include/he_b200.h
declares (no compute without a GPU), the host API's error/ledger contract mirrors hesim
(matmul.py:139-149, slotsim.py:31-83,192-205), and the product never reaches the oracle."""

import ast
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2601_18511_b200 as pkg
from paper_2601_18511_b200 import native
from paper_2601_18511_b200.context import CostLedger, CtBlocks, HeContext, MlweBlocks
from paper_2601_18511_b200.errors import NeedsBootstrapError
from paper_2601_18511_b200.params import HeParams, signed_digits
from paper_2601_18511_b200.pcmm import MlwePcmmPlan, _check_operand
from paper_2601_18511_b200.sharding import row_shards

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "he_b200.h").read_text()
    return set(re.findall(r"\b(he_[a-z0-9_]+)\s*\(", text))


def test_header_declares_exactly_the_bound_symbols():
    assert header_symbols() == set(native.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = native.lib()
    for name in native.EXPORTS:
        assert hasattr(L, name), name
    assert L.he_version() == 1


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(native.library_path())], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", str(native.library_path())], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05.mma kind::i8, TMA, TMEM


def test_product_package_never_imports_the_oracle():
    for py in (ROOT / "paper_2601_18511_b200").rglob("*.py"):
        tree = ast.parse(py.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert all(not a.name.startswith("oracle") for a in node.names), py
            if isinstance(node, ast.ImportFrom):
                assert not (node.module or "").startswith("oracle"), py


def test_validation_errors_before_any_launch():
    # HE_EINVAL from argument validation needs no device
    with pytest.raises(ValueError):
        native.call("he_context_create", None, None)


def test_status_mapping():
    with pytest.raises(ValueError):
        native.check(native.HE_EINVAL)
    with pytest.raises(TypeError):
        native.check(native.HE_ETYPE)
    with pytest.raises(NeedsBootstrapError):
        native.check(native.HE_ENEEDS_BOOTSTRAP)
    with pytest.raises(RuntimeError):
        native.check(native.HE_ECUDA)


class _Fake:
    def __init__(self, shape):
        self.shape = shape


def _plan(n_out=512, n_in=512):
    return MlwePcmmPlan(n_out, n_in, 2, 100, None)


def test_operand_checks_follow_reference_order():
    ctx = HeContext(HeParams.llama(), rng="seeded")
    plan = _plan()
    with pytest.raises(TypeError, match="ciphertext operand"):
        _check_operand(ctx, plan, np.zeros(3))
    with pytest.raises(ValueError, match="dim mismatch"):
        _check_operand(ctx, plan, CtBlocks(_Fake((1, 2, 2, 65536)), 1, 256))
    with pytest.raises(ValueError, match="layout mismatch"):
        _check_operand(ctx, plan, CtBlocks(_Fake((2, 2, 2, 65536)), 1, 512, layout="slots"))
    with pytest.raises(NeedsBootstrapError, match="one level"):
        _check_operand(ctx, plan, CtBlocks(_Fake((2, 2, 2, 65536)), 0, 512))
    _check_operand(ctx, plan, CtBlocks(_Fake((2, 2, 2, 65536)), 1, 512))


def test_ledger_semantics_match_hesim():
    led = CostLedger(min_level_reached=1)
    snap = led.snapshot()
    led.pc_mults += 4
    led.rescales += 1
    led.observe_level(0)
    assert led.diff(snap) == {"ct_rotations": 0, "cc_mults": 0, "pc_mults": 4, "pt_rotations": 0,
                              "pt_mults": 0, "rescales": 1, "bootstraps": 0}
    other = CostLedger(pc_mults=2, min_level_reached=0)
    led.merge(other)
    assert led.pc_mults == 6 and led.min_level_reached == 0
    assert CostLedger.from_dict(led.to_dict()) == led


def test_context_fork_merge_private_ledgers():
    ctx = HeContext(HeParams.toy(), rng="seeded")
    kids = [ctx.fork() for _ in range(3)]
    for i, c in enumerate(kids):
        c.ledger.pc_mults += i + 1
    for c in kids:
        ctx.merge(c)
    assert ctx.ledger.pc_mults == 6
    assert kids[0].params is ctx.params


def test_params_validation_and_json_roundtrip(tmp_path):
    p = HeParams.llama()
    assert p.N == 65536 and p.width == 65792 and p.tokens == 128
    assert p.ct_digits(0) == 4 and p.ct_digits(1) == 3
    f = tmp_path / "p.json"
    f.write_text(p.to_json())
    assert HeParams.from_json(f) == p
    with pytest.raises(ValueError, match="unknown"):
        HeParams.from_dict({"slot_count": 4})
    with pytest.raises(ValueError):
        HeParams(moduli=(1073479681, 1073479681))
    with pytest.raises(ValueError):
        HeParams(moduli=(1073479681, 1000003))  # not 1 mod 2N
    with pytest.raises(ValueError):
        HeParams(moduli=(2147352577, 1179649))  # >= 2^30
    assert HeParams.wide().ct_digits(1) == 4
    assert signed_digits(127) == 1 and signed_digits(128) == 2 and signed_digits(18432) == 2


def test_row_shards_balanced_and_covering():
    for n_out, world in ((4096, 1), (4096, 8), (11008, 8), (14336, 8), (11008, 3)):
        spans = row_shards(n_out, 256, world)
        assert spans[0][0] == 0 and spans[-1][1] == n_out // 256
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        sizes = [b1 - b0 for b0, b1 in spans]
        assert max(sizes) - min(sizes) <= 1


def test_public_api_exports():
    for name in ("make_mlwe_pcmm_plan", "pcmm_mlwe", "clear_pcmm", "HeContext", "HeParams", "CostLedger",
                 "NeedsBootstrapError", "byte_mix", "half_reverse", "shuffle_matrix", "bit_reverse"):
        assert hasattr(pkg, name)
