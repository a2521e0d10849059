"""CPU-side checks of the drop-in boundary: the C-ABI library exists, loads, exports exactly the
entry points include/specmoe_b200.h declares, and fails loudly (status 3) without a GPU."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    txt = open(os.path.join(ROOT, "include", "specmoe_b200.h")).read()
    return sorted(set(re.findall(r"\b(smoe_[a-z_]+)\s*\(", txt)))


def test_header_and_python_mirror_agree():
    from paper_2604_10152_b200.engine import EXPORTS
    assert sorted(EXPORTS) == declared()


def test_library_exports_every_declared_symbol():
    from paper_2604_10152_b200 import engine
    if not os.path.exists(engine.LIB_PATH):
        engine.build()
    L = engine.lib()
    for name in declared():
        assert hasattr(L, name), name


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    from paper_2604_10152_b200.engine import Engine, EngineError, ModelSpec
    with pytest.raises(EngineError) as ei:
        Engine(ModelSpec())
    assert ei.value.code == 3


def test_sm100a_code_in_library():
    """The shipped .so carries sm_100a SASS with tcgen05 MMA, TMEM loads and TMA loads."""
    import shutil
    import subprocess
    from paper_2604_10152_b200 import engine
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    if not os.path.exists(engine.LIB_PATH):
        engine.build()
    out = subprocess.run(["cuobjdump", "-sass", engine.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in out, mnem


def test_ledger_record_array_semantics():
    """RunResult.ledger is built lazily from the C result's LedgerEntry array: it must behave like the
    reference's list of (phase, step, layer, expert, bytes) tuples (len, index, iteration, equality with
    plain lists in both directions and with another Ledger)."""
    import numpy as np
    from paper_2604_10152_b200.engine import LEDGER_DTYPE, Ledger
    rec = np.zeros(3, dtype=LEDGER_DTYPE)
    rec["phase"] = [0, 1, 2]
    rec["step"] = [0, 0, 1]
    rec["layer"] = [3, 4, 5]
    rec["expert"] = [7, 1, 0]
    rec["bytes"] = [1 << 33, 5, 6]
    L = Ledger(rec.copy())
    want = [("speculation", 0, 3, 7, 1 << 33), ("verification", 0, 4, 1, 5), ("baseline-step", 1, 5, 0, 6)]
    assert len(L) == 3 and L[1] == want[1] and L[-1] == want[-1]
    assert list(L) == want and L == want and want == L and L == Ledger(rec.copy())
    assert L != want[:2] and L != Ledger(rec[:2].copy())
    assert [list(x) for x in L][0] == ["speculation", 0, 3, 7, 1 << 33]
    assert sum(b for *_, b in L) == (1 << 33) + 11
    assert Ledger() == [] and len(Ledger()) == 0
