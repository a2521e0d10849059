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


@pytest.mark.gpu
def test_caller_refilling_weights_in_place_sees_new_values():
    """The device copy of a ModelWeights is keyed by its full contents, not its address: refilling the
    tensors in place between calls reaches the GPU (head x2 -> logits x2 exactly; one expert value)."""
    exe = os.path.join(ROOT, "build", "caller_mutate_b200")
    build_caller("caller_mutate.cpp", exe)
    got = json.loads(subprocess.run([exe], capture_output=True, text=True, check=True).stdout)
    assert got == {"head_scaled_exact": 1, "expert_change_seen": 1}


@pytest.mark.gpu
def test_caller_on_tcgen05_path_is_lossless():
    """The same reference-API client with SPECMOE_B200_DTYPE=bf16 (the drop-in's tcgen05 path): every
    speculative policy decodes exactly the on-demand token stream, overlap/caching decode it too, the
    error behaviour is the reference's, and the logits are within the bf16 tolerance of the reference's."""
    build_caller()
    env = dict(os.environ, SPECMOE_B200_DTYPE="bf16")
    got = json.loads(subprocess.run([EXE], capture_output=True, text=True, check=True, env=env).stdout)
    want = json.load(open(os.path.join(ROOT, "tests", "golden", "cpp_caller.json")))
    od = got["ondemand"]["tokens"]
    for k in ("specmoe_hot_temporal", "specmoe_random", "specmoe_hot_global", "overlap", "caching"):
        assert got[k]["tokens"] == od, k
    assert got["errors"] == want["errors"]
    m = got["specmoe_hot_temporal"]["metrics"]
    assert m["bytes_total"] == m["bytes_verify"]  # speculation migrates nothing
    gl, wl = np.asarray(got["forward"]["logits"]), np.asarray(want["forward"]["logits"])
    assert np.max(np.abs(gl - wl)) <= 3e-2 * np.max(np.abs(wl))
