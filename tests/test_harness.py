"""Harness (reference harness.hpp; semantics SPEC.md:443-521) through the `specmoe` CLI and the C ABI.

CPU: selftest host checks, config parsing errors, prompts (C++ == Python restatement), trace I/O and
analysis KATs.  GPU: engine selftest, sweep rows equal to the oracle's run metrics (fp32 engine),
byte-identical reruns, trace round trip against the oracle's hotness, cross-policy text hashes.
"""
import csv
import io
import json
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2604_10152_b200", "bin", "specmoe")


def cli(*args, check=False):
    if not os.path.exists(CLI):
        subprocess.run(["make", "-C", ROOT, "-s", os.path.relpath(CLI, ROOT)], check=True)
    r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)
    if check and r.returncode != 0:
        raise AssertionError(f"specmoe {' '.join(args)} -> {r.returncode}\n{r.stdout}\n{r.stderr}")
    return r


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


# ------------------------------------------------------------------ CPU
def test_selftest_host_checks():
    r = cli("selftest")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout and "all checks passed" in r.stdout


def test_config_errors_name_line_and_invariant(tmp_path):
    r = cli("run", "--config", write(tmp_path, "a.cfg", "experts = 16\nbogus = 3\n"))
    assert r.returncode == 1 and "line 2" in r.stderr and "bogus" in r.stderr
    r = cli("run", "--config", write(tmp_path, "b.cfg", "gamma = 0\n"))
    assert r.returncode == 1 and "gamma" in r.stderr
    r = cli("run", "--config", write(tmp_path, "c.cfg", "top_k = 2\nno equals sign\n"))
    assert r.returncode == 1 and "line 2" in r.stderr
    r = cli("run", "--config", write(tmp_path, "d.cfg", "batch = 1, 2\ntrace_out = /tmp/x.trace\n"))
    assert r.returncode == 1 and "single-cell" in r.stderr
    r = cli("run", "--config", str(tmp_path / "missing.cfg"))
    assert r.returncode == 1


def test_prompts_native_equal_python_restatement():
    from paper_2604_10152_b200.engine import make_prompts_native
    from paper_2604_10152_b200.prompts import make_prompts
    for seed, B, plen, V in [(0, 4, 8, 32000), (7, 3, 5, 64), (2**63 + 11, 2, 16, 1), (5, 8, 8, 102400)]:
        assert make_prompts_native(seed, B, plen, V) == make_prompts(seed, B, plen, V)
    # batch transparency (harness.hpp:58-62): prompt b depends only on (seed, b)
    assert make_prompts_native(3, 8, 8, 1000)[:2] == make_prompts_native(3, 2, 8, 1000)


def _trace_text(M, E, K, rows):
    out = [f"# specmoe-trace v1 layers={M} experts={E} top_k={K}", "step,seq,layer,experts"]
    out += [",".join(str(x) for x in r) for r in rows]
    return "\n".join(out) + "\n"


def _analyze(tmp_path, text):
    path = write(tmp_path, "t.trace", text)
    rep = str(tmp_path / "rep.csv")
    r = cli("trace", "analyze", "--in", path, "--out", rep, "--top", "3")
    return r, (list(csv.DictReader(open(rep))) if r.returncode == 0 else None)


def test_trace_skewness_kats(tmp_path):
    # uniform: 8 experts, K=2, every expert equally often -> 0.25
    rows = [(s, 0, l, (2 * s) % 8, (2 * s + 1) % 8) for s in range(400) for l in range(2)]
    r, rep = _analyze(tmp_path, _trace_text(2, 8, 2, rows))
    assert r.returncode == 0, r.stderr
    assert abs(float(r.stdout.split()[1]) - 0.25) <= 0.01
    assert len(rep) == 16 and abs(sum(float(x["fraction"]) for x in rep if x["layer"] == "0") - 1.0) < 1e-12
    # one-hot (K=1): all mass on one expert per layer -> exactly 1.0
    rows = [(s, 0, l, 3 if l == 0 else 1) for s in range(50) for l in range(2)]
    r, rep = _analyze(tmp_path, _trace_text(2, 4, 1, rows))
    assert r.returncode == 0 and float(r.stdout.split()[1]) == 1.0
    assert "layer 0 hottest 3 0 1" in r.stdout
    # hand-computed 4-expert case [7,1,1,1] -> 0.70 exactly
    rows = [(s, 0, 0, 0) for s in range(7)] + [(7 + e, 0, 0, e) for e in (1, 2, 3)]
    r, _ = _analyze(tmp_path, _trace_text(1, 4, 1, rows))
    assert r.returncode == 0 and float(r.stdout.split()[1]) == 0.7
    assert "routed_tokens 10" in r.stdout


def test_trace_malformed_rows_name_line(tmp_path):
    r, _ = _analyze(tmp_path, _trace_text(2, 4, 2, [(0, 0, 0, 1, 2), (0, 0, 1, 1, 9)]))
    assert r.returncode == 1 and "line 4" in r.stderr and "out of range" in r.stderr
    r, _ = _analyze(tmp_path, _trace_text(2, 4, 2, [(0, 0, 0, 1)]))
    assert r.returncode == 1 and "line 3" in r.stderr
    r, _ = _analyze(tmp_path, "step,seq,layer,experts\n")
    assert r.returncode == 1 and "line 1" in r.stderr


# ------------------------------------------------------------------ GPU
TOY = """# acceptance-1 toy model (SPEC.md:512)
num_layers = 4
experts = 16
top_k = 2
hidden_dim = 32
ffn_dim = 64
vocab_size = 64
gate_skew = {skew}
max_new_tokens = 24
gamma = {gamma}
n_draft = {n}
batch = {batch}
seeds = {seeds}
engine = {engine}
policy = {policy}
verbose = true
"""


def toy(tmp_path, name="toy.cfg", skew=0.0, gamma="5", n="4", batch="2", seeds="0..2", engine="specmoe",
        policy="hot_temporal", extra=""):
    return write(tmp_path, name, TOY.format(skew=skew, gamma=gamma, n=n, batch=batch, seeds=seeds, engine=engine,
                                            policy=policy) + extra)


def fnv1a64_tokens(seqs):
    h = 0xcbf29ce484222325
    for s in seqs:
        for b in struct.pack(f"<{len(s)}i", *s):
            h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.mark.gpu
def test_selftest_engine_checks():
    r = cli("selftest")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "skip engine checks" not in r.stdout and "lossless" in r.stdout and "FAIL" not in r.stdout


@pytest.mark.gpu
def test_sweep_rows_equal_oracle_metrics(tmp_path, ref):
    from oracle.oracle import ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    cfg = toy(tmp_path, gamma="3, 5", n="2, 4", batch="1, 3", seeds="0, 1")
    out = str(tmp_path / "rows.csv")
    cli("run", "--config", cfg, "--out", out, check=True)
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 2 * 2 * 2 * 2
    spec = ModelSpec(num_layers=4, experts=16, top_k=2, hidden=32, ffn=64, vocab=64)
    m = ref.build(spec)
    bpe = spec.bytes_per_expert()
    order = [(b, g, n, s) for b in (1, 3) for g in (3, 5) for n in (2, 4) for s in (0, 1)]
    for row, (b, g, n, s) in zip(rows, order):
        assert (int(row["batch"]), int(row["gamma"]), int(row["n_draft"]), int(row["seed"])) == (b, g, n, s)
        r = m.run_specmoe(RunCfg(gamma=g, n_draft=n, max_new_tokens=24, run_seed=s, bytes_per_expert=bpe,
                                 device_capacity_bytes=4 * 16 * bpe), make_prompts(s, b, 8, 64))
        mt = r.metrics
        assert row["policy"] == "hot_temporal"
        assert float(row["tau"]) == mt["tau_mean"]
        assert float(row["tokens_per_sec"]) == mt["tokens_per_sec"]
        assert int(row["bytes_total"]) == mt["bytes_total"] and int(row["bytes_spec"]) == mt["bytes_spec"] == 0
        assert int(row["bytes_verify"]) == mt["bytes_verify"]
        assert float(row["lambda"]) == mt["lambda"]
        c = mt["c_measured"]
        assert float(row["s_eq1"]) == pytest.approx(mt["tau_mean"] / (g * c + 1.0), rel=1e-15)
        assert float(row["s_eq2"]) == pytest.approx(mt["tau_mean"] / (g * c + mt["lambda"]), rel=1e-15)
        assert int(row["text_hash"]) == fnv1a64_tokens(r.tokens)


@pytest.mark.gpu
def test_results_byte_identical_across_runs_csv_and_json(tmp_path):
    cfg = toy(tmp_path, seeds="0..3")
    for fmt in ("csv", "json"):
        a, b = str(tmp_path / f"a.{fmt}"), str(tmp_path / f"b.{fmt}")
        cli("run", "--config", cfg, "--out", a, "--format", fmt, check=True)
        cli("run", "--config", cfg, "--out", b, "--format", fmt, check=True)
        assert open(a, "rb").read() == open(b, "rb").read()
    rows = json.load(open(str(tmp_path / "a.json")))
    assert len(rows) == 4 and set(rows[0]) >= {"policy", "tau", "bytes_total", "s_eq2", "text_hash"}
    for r in rows:
        assert 1.0 <= r["tau"] <= 6.0 and r["bytes_total"] == r["bytes_spec"] + r["bytes_verify"]


@pytest.mark.gpu
def test_cross_policy_and_engine_text_hash_identical(tmp_path):
    """for a fixed seed and greedy mode every policy and engine yields identical text."""
    hashes = []
    for i, (engine, policy) in enumerate([("specmoe", "random"), ("specmoe", "hot_global"), ("specmoe", "hot_temporal"),
                                          ("ondemand", "hot_temporal"), ("overlap", "hot_temporal"),
                                          ("caching", "hot_temporal")]):
        out = str(tmp_path / f"r{i}.csv")
        cli("run", "--config", toy(tmp_path, f"c{i}.cfg", skew=1.5, engine=engine, policy=policy, batch="4"),
            "--out", out, check=True)
        hashes.append([r["text_hash"] for r in csv.DictReader(open(out))])
    assert all(h == hashes[0] for h in hashes)


@pytest.mark.gpu
def test_trace_round_trip_matches_oracle_hotness(tmp_path, ref):
    from oracle.oracle import ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    tr = str(tmp_path / "run.trace")
    cfg = toy(tmp_path, engine="ondemand", seeds="5", batch="3", skew=2.0, extra=f"trace_out = {tr}\n")
    cli("run", "--config", cfg, "--out", str(tmp_path / "r.csv"), check=True)
    rep = str(tmp_path / "rep.csv")
    r = cli("trace", "analyze", "--in", tr, "--out", rep, check=True)
    spec = ModelSpec(num_layers=4, experts=16, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=2.0)
    o = ref.build(spec).run_ondemand(RunCfg(max_new_tokens=24, run_seed=5, collect_trace=True),
                                     make_prompts(5, 3, 8, 64))
    counts = np.zeros((4, 16), dtype=np.uint64)
    for x in csv.DictReader(open(rep)):
        counts[int(x["layer"]), int(x["expert"])] = int(x["count"])
    assert np.array_equal(counts, o.hotness)
    from oracle.oracle import skewness
    assert float(r.stdout.split()[1]) == pytest.approx(skewness(ref, o.hotness, len(o.trace) // 4), abs=0)


# ------------------------------------------------------------------ SPEC acceptance criteria
def _rows(tmp_path, name, **kw):
    out = str(tmp_path / f"{name}.csv")
    cli("run", "--config", toy(tmp_path, f"{name}.cfg", **kw), "--out", out, check=True)
    return list(csv.DictReader(open(out)))


@pytest.mark.gpu
def test_acceptance_4_coalescing_zero_speculation_bytes(tmp_path):
    rows = _rows(tmp_path, "a4", skew=1.5, batch="1, 8, 32", seeds="0..3")
    for r in rows:
        assert int(r["bytes_spec"]) == 0 and int(r["bytes_total"]) == int(r["bytes_verify"])


@pytest.mark.gpu
def test_acceptance_5_transfer_reduction_trend(tmp_path):
    """Skewed toy (gate_skew 1.5), B=32, 20 seeds: specmoe < caching < ondemand == overlap (mean bytes)."""
    mean = {}
    for engine in ("specmoe", "caching", "ondemand", "overlap"):
        rows = _rows(tmp_path, f"a5_{engine}", skew=1.5, batch="32", seeds="0..19", engine=engine)
        mean[engine] = np.mean([int(r["bytes_total"]) for r in rows])
        if engine == "overlap":
            per_seed_overlap = [int(r["bytes_total"]) for r in rows]
        if engine == "ondemand":
            per_seed_ondemand = [int(r["bytes_total"]) for r in rows]
    assert mean["specmoe"] < mean["caching"] < mean["ondemand"]
    assert per_seed_overlap == per_seed_ondemand


@pytest.mark.gpu
def test_acceptance_7_tau_nondecreasing_in_n(tmp_path):
    """N sweep {2,4,8,16}: mean tau over 20 seeds is non-decreasing in N (slack 0.1)."""
    rows = _rows(tmp_path, "a7", skew=1.5, n="2, 4, 8, 16", batch="4", seeds="0..19", gamma="5")
    taus = [np.mean([float(r["tau"]) for r in rows if int(r["n_draft"]) == n]) for n in (2, 4, 8, 16)]
    for a, b in zip(taus, taus[1:]):
        assert b >= a - 0.1, taus
    assert taus[-1] == 6.0  # identity limit (acceptance 2): N = E accepts every draft


@pytest.mark.gpu
def test_acceptance_6_policy_order_and_affinity(tmp_path):
    """20 seeds on a skewed toy: random <= hot_global <= hot_temporal (slack 0.05); affinity remap >= hash."""
    tau = {}
    for policy in ("random", "hot_global", "hot_temporal"):
        rows = _rows(tmp_path, f"a6_{policy}", skew=1.5, batch="8", seeds="0..19", policy=policy)
        tau[policy] = np.mean([float(r["tau"]) for r in rows])
    rows = _rows(tmp_path, "a6_hash", skew=1.5, batch="8", seeds="0..19", extra="use_affinity = false\n")
    tau_hash = np.mean([float(r["tau"]) for r in rows])
    assert tau["random"] <= tau["hot_global"] + 0.05 and tau["hot_global"] <= tau["hot_temporal"] + 0.05, tau
    assert tau["hot_temporal"] >= tau_hash - 0.05, (tau, tau_hash)
