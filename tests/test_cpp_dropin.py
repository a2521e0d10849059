"""Drop-in proof through the reference's own C++ interface: tests/cpp/caller.cpp (a client written
only against the reference headers) compiled against include/specmoe/ + libspecmoe_b200.so must
reproduce the output of the same source compiled against the reference (tests/golden/cpp_caller.json)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "caller_b200")
EXE_S = os.path.join(ROOT, "build", "caller_sampling_b200")


def build_caller(src="caller.cpp", exe=EXE):
    from paper_2604_10152_b200 import engine
    if not os.path.exists(engine.LIB_PATH):
        engine.build()
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", src), "-L" + os.path.dirname(engine.LIB_PATH),
                    "-lspecmoe_b200", "-Wl,-rpath," + os.path.dirname(engine.LIB_PATH), "-o", exe], check=True)


def test_caller_compiles_and_links_against_dropin_headers():
    build_caller()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_caller_output_matches_reference():
    build_caller()
    got = json.loads(subprocess.run([EXE], capture_output=True, text=True, check=True).stdout)
    want = json.load(open(os.path.join(ROOT, "tests", "golden", "cpp_caller.json")))
    gl, wl = np.asarray(got["forward"].pop("logits")), np.asarray(want["forward"].pop("logits"))
    assert np.max(np.abs(gl - wl)) <= 2e-5 * np.max(np.abs(wl))   # fp32 engine vs fp64 reference
    assert got == want                                             # every integer / modeled metric exact


def test_sampling_caller_compiles_against_dropin_headers():
    build_caller("caller_sampling.cpp", EXE_S)
    assert os.path.exists(EXE_S)


@pytest.mark.gpu
def test_sampling_caller_matches_reference():
    """Sampling mode (specdec.cpp:82-157): the reference's RNG consumption order is kept, so sampled
    drafts, acceptances, corrections, tokens and ledger sizes equal the reference's (fp32 engine)."""
    build_caller("caller_sampling.cpp", EXE_S)
    got = json.loads(subprocess.run([EXE_S], capture_output=True, text=True, check=True).stdout)
    want = json.load(open(os.path.join(ROOT, "tests", "golden", "cpp_caller_sampling.json")))
    for k in want:
        assert got[k] == want[k], k
