#!/usr/bin/env python
"""bench.py -- accepted decode tokens/s of the self-assisted speculative-decoding loop on B200.

Default workload (BASELINE.json configs[1], the metric's config): Mixtral-8x7B shape
(L32 E8 K2 d4096 f14336 V32000, SwiGLU experts, bf16 weights, random init), all experts
HBM-resident, batch 64, gamma 4, N 4 draft experts, hot_temporal + affinity, greedy.
A "step" = one speculative phase over the batch: gamma restricted draft passes, one batched verify
pass over B*(gamma+1) positions, accept/rollback, hotness + re-pin + ledger.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--shape c1|c2|c4|c5] [--batch B]

N > 1 (torchrun): expert parallelism -- every rank holds E/N experts of every layer and a
replica of the dense weights, the rows of each pass are split over the ranks, and per MoE layer the
gate / down-projection epilogues exchange routed rows through NVLink peer memory (SMOE_EP_MODE=a2a:
NCCL all-to-alls instead); the global batch is fixed (strong scaling); time = max over ranks, value =
the global batch's tokens / that time.  --replicas: independent replicas instead (weak scaling).
--impl reference times the reference's own CPU implementation (oracle/_ref, compiled from
/root/reference) on the host cores.

The default C2 run adds sections to the same JSON line: the batch sweep 1-32 (the metric is quoted over
batch 1-64), the on-demand comparator, gamma=8, C1 (configs[0]: reference CPU path vs the engine on the
reference's own weights), gate_skew=2.0, C4, C2 with real attention, the C3 offloaded store (with the
on-demand, overlap and caching comparators), the SSD tier and the CPU reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "accepted decode tokens/sec, Mixtral-8x7B shape, batch 1-64; expert bytes/token"
READ_STREAM_GBPS = 7408.4  # profiles/r04_bw_probe2.txt (K=4096, 6 x 32 KB stages, 148 CTAs, tiled)
SHAPES = {
    "c1": dict(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024),
    "c2": dict(num_layers=32, experts=8, top_k=2, hidden=4096, ffn=14336, vocab=32000),
    "c4": dict(num_layers=28, experts=64, top_k=6, hidden=2048, ffn=1408, vocab=102400, moe_mask=[0] + [1] * 27),
    # Mixtral-8x22B shape: 270.6 GB of SwiGLU experts -> expert parallel over >= 2 GPUs only
    "c5": dict(num_layers=56, experts=8, top_k=2, hidden=6144, ffn=16384, vocab=32768),
}
SHAPE_NAMES = {"c1": "tiny synthetic MoE (C1)", "c2": "Mixtral-8x7B shape (C2)", "c4": "fine-grained E64 K6 (C4)",
               "c5": "Mixtral-8x22B shape (C5)"}


def args_parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=8)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--shape", default="c2", choices=sorted(SHAPES))
    p.add_argument("--expert", default="swiglu3", choices=["swiglu3", "tanh2"])
    p.add_argument("--batch", type=int, default=0, help="0: the shape's default (64; 128 for C5)")
    p.add_argument("--gamma", type=int, default=4)
    p.add_argument("--n-draft", type=int, default=0, help="0: the shape's default (4; 8 for C4, SURVEY 8)")
    p.add_argument("--e2e-tokens", type=int, default=128, help="new tokens per sequence of the e2e run (SURVEY 8d: 128)")
    p.add_argument("--skew", type=float, default=0.0, help="gate_skew of the headline model (SPEC: 0 uniform)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-threads", type=int, default=0)
    p.add_argument("--offload", action="store_true", help="headline = C3 (experts in pinned host DRAM)")
    p.add_argument("--no-offload-section", action="store_true", help="skip the C3 section of the default run")
    p.add_argument("--offload-batch", type=int, default=64)
    p.add_argument("--offload-steps", type=int, default=2)
    p.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of expert parallelism")
    p.add_argument("--no-sections", action="store_true", help="skip the batch sweep / on-demand / gamma=8 / "
                   "gate_skew=2 / C4 sections of the default C2 run")
    a = p.parse_args()
    if a.n_draft == 0:
        a.n_draft = 8 if a.shape == "c4" else 4
    if a.batch == 0:
        a.batch = 128 if a.shape == "c5" else 64
    return a


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def reduce_over_ranks(ms: float, tokens: int, sum_tokens: bool):
    """Max of the device-timed ms over ranks; tokens summed (replicas) or taken from rank 0 (expert
    parallel: every rank decodes the same global batch)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return ms, tokens
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    k = torch.tensor([float(tokens)], dtype=torch.float64, device=dev)
    if sum_tokens:
        dist.all_reduce(k, op=dist.ReduceOp.SUM)
    else:
        dist.broadcast(k, 0)
    return float(t.item()), int(k.item())


def share_nccl_id(rank: int):
    """Rank 0 creates the engine-side NCCL unique id; every rank receives it (torch.distributed)."""
    import torch.distributed as dist
    from paper_2604_10152_b200.engine import nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


# ---------------------------------------------------------------- clocks (B200_PROFILING.md)
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev, self.proc, self.path = dev, None, f"/tmp/bench_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        for r in rows:
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), r[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------------- CPU reference (oracle/_ref)
def forward_macs(s: dict, n_layers: int, mats: int) -> float:
    """Multiply-adds of one reference forward() (model.cpp:192-263) with n_layers MoE layers."""
    d, f, E, K, V = s["hidden"], s["ffn"], s["experts"], s["top_k"], s["vocab"]
    return n_layers * (d * d + d * E + K * mats * d * f) + d * V


def cpu_reference(shape: str, expert: str, gamma: int, n_draft: int, threads: int, steps: int = 1,
                  warmup: int = 0, tau: float | None = None) -> dict:
    """Time the reference's own CPU path on a bounded sample of the workload.

    Sample: a one-MoE-layer slice of the shape (full d, f, E, K, V), built by the reference's
    build_model; `threads` host threads run forward() concurrently on the shared weights; tau comes
    from one reference run_specmoe phase on the slice.  forward() is a per-layer loop, so its time is
    extrapolated to the full depth (and from the reference's 2-matrix expert to SwiGLU's 3) by its
    multiply-add count.  tokens/s = forwards/s * tau / (2*gamma + 1).  With steps > 1 the slice is built
    once and the concurrent forward is timed `warmup` + `steps` times (median of the timed ones).
    `tau`: the acceptance of the full-depth model measured by the B200 arm on the same configuration (the
    one-layer slice accepts far more drafts than 32 layers of expert substitution do); the slice's own tau
    is used only when none is given (the reference arm)."""
    from oracle.oracle import LIBS, ModelSpec as OSpec, Oracle, RunCfg as ORun
    from paper_2604_10152_b200.prompts import make_prompts
    kind = "ref" if os.path.exists(LIBS["ref"]) else "port"
    full = dict(SHAPES[shape])
    full.pop("moe_mask", None)
    slice_spec = dict(full, num_layers=1, seed=0)
    o = Oracle(kind)
    t0 = time.time()
    m = o.build(OSpec(**slice_spec))
    build_s = time.time() - t0
    prompt = make_prompts(0, 1, 8, full["vocab"])
    t1 = m.time_forward(prompt[0], threads=1, iters=1)
    for _ in range(max(0, warmup)):
        m.time_forward(prompt[0], threads=threads, iters=1)
    samples = [m.time_forward(prompt[0], threads=threads, iters=1) for _ in range(max(1, steps))]
    tp = statistics.median(samples)
    sp = m.run_specmoe(ORun(gamma=gamma, n_draft=min(n_draft, full["experts"]), max_new_tokens=gamma + 1,
                            run_seed=0), prompt)
    tau_slice = sp.metrics["tau_mean"]
    tau_used = tau if tau else tau_slice
    mats = 3 if expert == "swiglu3" else 2
    n_moe = SHAPES[shape]["num_layers"] if "moe_mask" not in SHAPES[shape] else sum(SHAPES[shape]["moe_mask"])
    scale = forward_macs(full, SHAPES[shape]["num_layers"], mats) / forward_macs(full, 1, 2)
    fwd_s_full = tp * scale  # wall of one forward per thread, full depth
    value = threads * tau_used / ((2 * gamma + 1) * fwd_s_full)
    tau_src = ("the B200 arm's measured tau at full depth" if tau else
               f"one reference run_specmoe phase on the slice (gamma {gamma})")
    return {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference" if kind == "ref" else "port",
            "sample": (f"{kind} build of a 1-MoE-layer slice of {SHAPE_NAMES[shape]} (tanh2, fp64); "
                       f"{threads} threads x 1 forward() = {tp:.3f}s (1 thread {t1:.3f}s); tau {tau_used:.3f} from "
                       f"{tau_src}; extrapolated x{scale:.1f} by forward MACs to L={n_moe} {expert}; slice build "
                       f"{build_s:.0f}s untimed"),
            "tau": tau_used, "tau_slice": tau_slice, "forward_s_slice": t1, "forward_s_full_extrapolated": t1 * scale,
            "ondemand_value": threads / fwd_s_full,
            "step_values": [threads * tau_used / ((2 * gamma + 1) * t * scale) for t in samples]}


def section_c1(gamma: int = 4, n_draft: int = 4, new_tokens: int = 32) -> dict:
    """BASELINE configs[0] side by side (SURVEY 8(d) 'C1 in full'): the tiny synthetic MoE with the
    reference's own build_model weights, B=1, greedy, run end to end by the reference's CPU path
    (oracle/_ref, one thread as written) and by the B200 engine (fp32 parity engine on the same weights --
    its token stream must equal the reference's -- and the bf16 tcgen05 engine)."""
    from oracle.oracle import LIBS, ModelSpec as OSpec, Oracle, RunCfg as ORun
    from paper_2604_10152_b200.engine import BF16, F32, Engine, ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    spec = dict(SHAPES["c1"], seed=0)
    prompts = make_prompts(0, 1, 8, spec["vocab"])
    cfg = dict(gamma=gamma, n_draft=n_draft, max_new_tokens=new_tokens, run_seed=0)
    kind = "ref" if os.path.exists(LIBS["ref"]) else "port"
    om = Oracle(kind).build(OSpec(**spec))
    out = {"workload": f"C1 tiny synthetic MoE (L4 E8 K2 d512 f1024 V1024), reference build_model weights, B=1, "
                       f"gamma={gamma}, N={n_draft}, {new_tokens} new tokens, greedy", "reference_kind": kind}
    t0 = time.perf_counter()
    rs = om.run_specmoe(ORun(**cfg), prompts)
    ref_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    ro = om.run_ondemand(ORun(**cfg), prompts)
    ref_od_s = time.perf_counter() - t0
    out["reference_cpu"] = {"spec_tokens_per_s": rs.metrics["tokens_total"] / ref_s,
                            "ondemand_tokens_per_s": ro.metrics["tokens_total"] / ref_od_s,
                            "tau": rs.metrics["tau_mean"], "cores": 1}
    for name, wt in (("b200_fp32_parity", F32), ("b200_bf16_tcgen05", BF16)):
        e = Engine(ModelSpec(**spec), weight_type=wt, max_batch=1, max_gamma=gamma).init_exact()
        e.run_specmoe(RunCfg(**cfg), prompts)  # warm-up
        t0 = time.perf_counter()
        r = e.run_specmoe(RunCfg(**cfg), prompts)
        wall = time.perf_counter() - t0
        t0 = time.perf_counter()
        od = e.run_ondemand(RunCfg(**cfg), prompts)
        od_wall = time.perf_counter() - t0
        out[name] = {"spec_tokens_per_s": r.metrics["tokens_total"] / wall,
                     "ondemand_tokens_per_s": od.metrics["tokens_total"] / od_wall,
                     "tau": r.metrics["tau_mean"], "tokens_equal_reference": r.tokens == rs.tokens,
                     "lossless": r.tokens == od.tokens,
                     "speedup_vs_reference_spec": (r.metrics["tokens_total"] / wall) / (rs.metrics["tokens_total"] / ref_s)}
        e.close()
    return out


# ---------------------------------------------------------------- the B200 arm
def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


def ncu_traffic(draft_passes: int = 4, name: str = "r02_ncu_fused_moe.json"):
    """DRAM bytes per launch of the dominant kernel from a committed ncu --set full capture (profiles/
    <name>: one draft-pass and one verify-pass launch), weighted like the step (gamma draft passes : 1
    verify pass), or None."""
    p = os.path.join(ROOT, "profiles", name)
    try:
        la = json.load(open(p))["launches"]
        d, v = la[0], la[1]
        mb = (draft_passes * (d["dram_read_MB"] + d["dram_write_MB"]) + v["dram_read_MB"] + v["dram_write_MB"])
        return mb / (draft_passes + 1) * 1e6
    except Exception:
        return None


def measure_pcie(dev: int) -> float:
    """Pinned host->device cudaMemcpyAsync bandwidth, 1 GiB, best of 10 (the migration roofline)."""
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=torch.device("cuda", dev))
    best = 0.0
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        d.copy_(h, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        best = max(best, n / (s.elapsed_time(e) * 1e-3) / 1e9)
    del h, d
    return best


def offload_section(a, dev: int, batch: int, steps: int, warmup: int, gammas=(4,)) -> dict:
    """C3: experts in pinned host DRAM, migrated over PCIe per layer during verify.  Reports accepted
    tokens/s, PCIe bytes/token, achieved H2D GB/s vs the measured pinned-copy peak, and the on-demand
    comparator (baselines.cpp:29-105) on the same engine."""
    import torch
    from paper_2604_10152_b200.engine import BF16, SWIGLU3, TANH2, Engine, ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    pcie = measure_pcie(dev)
    spec = ModelSpec(**SHAPES[a.shape], seed=0, expert_kind=SWIGLU3 if a.expert == "swiglu3" else TANH2)
    t0 = time.time()
    eng = Engine(spec, weight_type=BF16, max_batch=batch, max_gamma=max(gammas), device=dev, offload=1)
    eng.init_device(0)
    eng.build_affinity_device()
    setup_s = time.time() - t0
    prompts = make_prompts(2000, batch, 8, spec.vocab)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", dev))
    out = {"workload": f"{SHAPE_NAMES[a.shape]}, {a.expert} experts in pinned host DRAM (C3), B={batch}, N={a.n_draft}",
           "pcie_peak_gbs": pcie, "pcie_peak_source": "pinned 1 GiB cudaMemcpyAsync H2D, best of 10, measured in this run",
           "setup_s": setup_s, "gamma": {}}
    for g in gammas:
        eng.spec_begin(RunCfg(gamma=g, n_draft=a.n_draft, max_new_tokens=1 << 30), prompts)
        for _ in range(warmup):
            eng.spec_step()
        eng.counters(reset=True)
        base_bytes = eng.spec_end().metrics["h2d_expert_bytes"]
        eng.spec_begin(RunCfg(gamma=g, n_draft=a.n_draft, max_new_tokens=1 << 30), prompts)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(stream)
        tokens = 0
        for _ in range(steps):
            tokens += eng.spec_step()[0]
        ev1.record(stream)
        ev1.synchronize()
        ms = ev0.elapsed_time(ev1)
        r = eng.spec_end()
        hb, hs = r.metrics["h2d_expert_bytes"], r.metrics["h2d_s"]
        out["gamma"][str(g)] = {
            "tokens_per_s": tokens / (ms * 1e-3), "tau": r.metrics["tau_mean"], "ms_per_step": ms / steps,
            "pcie_bytes_per_token": hb / max(1, tokens), "h2d_gbs": hb / hs / 1e9 if hs else None,
            "h2d_frac_of_measured": (hb / hs / 1e9) / pcie if hs else None,
            "pcie_busy_frac": (hs * 1e3) / ms if ms else None,
            "ledger_bytes_per_token_reference_units": r.metrics["bytes_total"] / max(1, r.metrics["tokens_total"])}
        del base_bytes
    # the comparators on the same physical store (baselines.cpp:29-157): on-demand, overlap (next-layer
    # prefetch behind each layer's fetch) and caching (top ceil(0.1 E) = 1 expert per layer pinned from a
    # hot_global on-demand warm-up of 4 steps; the reference's default warm-up is 64 steps)
    ncomp = max(2, steps)
    runs = {"ondemand": lambda c: eng.run_ondemand(c, prompts), "overlap": lambda c: eng.run_overlap(c, prompts),
            "caching": lambda c: eng.run_caching(c, prompts, 0.10)}
    for name, fn in runs.items():
        r = fn(RunCfg(gamma=max(gammas), n_draft=a.n_draft, max_new_tokens=ncomp, warmup_steps=4))
        tps = r.metrics["tokens_total"] / r.metrics["gpu_s"]
        out[name] = {"tokens_per_s": tps, "ms_per_step": 1e3 * r.metrics["gpu_s"] / ncomp,
                     "pcie_bytes_per_token": r.metrics["h2d_expert_bytes"] / max(1, r.metrics["tokens_total"]),
                     "h2d_gbs": r.metrics["h2d_expert_bytes"] / r.metrics["h2d_s"] / 1e9 if r.metrics["h2d_s"] else None,
                     "pcie_busy_frac": r.metrics["h2d_s"] / r.metrics["gpu_s"] if r.metrics["gpu_s"] else None,
                     "ledger_bytes_per_token_reference_units": r.metrics["bytes_total"] / max(1, r.metrics["tokens_total"])}
        if name == "overlap":
            out[name]["prefetch_bytes"] = r.metrics["prefetch_bytes"]
            out[name]["prefetch_wasted_bytes"] = r.metrics["prefetch_wasted_bytes"]
    od_tps = out["ondemand"]["tokens_per_s"]
    od_bpt = out["ondemand"]["pcie_bytes_per_token"]
    for name in ("overlap", "caching"):
        out[name]["speedup_vs_ondemand"] = out[name]["tokens_per_s"] / od_tps
        out[name]["transfer_reduction_vs_ondemand"] = 1.0 - out[name]["pcie_bytes_per_token"] / max(1e-9, od_bpt)
    for g, v in out["gamma"].items():
        v["speedup_vs_ondemand"] = v["tokens_per_s"] / od_tps if od_tps else None
        v["transfer_reduction_vs_ondemand"] = 1.0 - v["pcie_bytes_per_token"] / max(1e-9, od_bpt)
        v["speedup_vs_best_baseline"] = v["tokens_per_s"] / max(out[n]["tokens_per_s"] for n in runs)
        v["transfer_reduction_vs_caching"] = 1.0 - v["pcie_bytes_per_token"] / max(1e-9, out["caching"]["pcie_bytes_per_token"])
    eng.close()
    return out


def spec_measure(eng, stream, cfg, prompts, steps: int, warmup: int, profile: bool = True, clocks=None) -> dict:
    """Stepped speculative phases on one engine: `warmup` untimed, `steps` timed by CUDA events on the
    engine stream (nothing else recorded in between); then, with profile, the same number of steps again
    with events around every launch (per kernel class, split by draft / verify pass)."""
    import torch
    eng.spec_begin(cfg, prompts)
    for _ in range(warmup):
        eng.spec_step()
    eng.counters(reset=True)
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    tokens = 0
    for _ in range(steps):
        tokens += eng.spec_step()[0]
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    out = {"ms": ev0.elapsed_time(ev1), "tokens": tokens, "clocks": clocks.stop() if clocks else None}
    cnt = eng.counters(reset=True)
    out["launches"] = cnt["launches"]
    out["alg_expert_bytes"] = cnt["alg_expert_bytes"]
    if profile:
        eng.profile_reset()
        ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2.record(stream)
        tp = 0
        for _ in range(steps):
            tp += eng.spec_step()[0]
        ev3.record(stream)
        ev3.synchronize()
        eng.profile_stop()
        out["ms_prof"] = ev2.elapsed_time(ev3)
        out["tokens_prof"] = tp
        out["cnt_prof"] = eng.counters()
        out["named"] = {k: eng.counter(k) for k in ("alg_expert_bytes:draft", "alg_expert_bytes:verify",
                                                     "expert_flops:draft", "expert_flops:verify")}
        eng.counters(reset=True)
        out["prof"] = {c: eng.profile_read(c) for c in (
            "expert_gemm", "expert_gemm:draft", "expert_gemm:verify", "dense_gemm", "head_gemm", "gate", "attention",
            "combine")}
    res = eng.spec_end()
    out["tau"] = res.metrics["tau_mean"]
    out["res"] = res
    return out


def expert_roofline(m: dict, pk: dict) -> dict:
    """Expert GEMM (fused MoE launch) roofline from a profiled spec_measure: algorithmic weight bytes of
    the distinct experts each pass touches / CUDA-event time of those launches, against the HBM peak;
    split by draft and verify pass, with the tensor-pipe fraction (algorithmic flops / time / bf16 peak)."""
    pr, nm = m["prof"], m["named"]
    out = {}
    for kind in ("draft", "verify"):
        t = pr[f"expert_gemm:{kind}"]
        if t["launches"] and t["ms"] > 0:
            gbs = nm[f"alg_expert_bytes:{kind}"] / (t["ms"] * 1e-3) / 1e9
            tfs = nm[f"expert_flops:{kind}"] / (t["ms"] * 1e-3) / 1e12
            out[kind] = {"launches": t["launches"], "avg_launch_us": 1e3 * t["ms"] / t["launches"],
                         "achieved_GBps": gbs, "hbm_frac": gbs / pk["hbm_gbs"], "achieved_TFLOPs": tfs,
                         "tensor_frac": tfs / pk["bf16_tflops"],
                         "flop_per_byte": nm[f"expert_flops:{kind}"] / max(1.0, nm[f"alg_expert_bytes:{kind}"])}
    t = pr["expert_gemm"]
    gbs = m["cnt_prof"]["alg_expert_bytes"] / (t["ms"] * 1e-3) / 1e9 if t["ms"] > 0 else 0.0
    out.update({"achieved_GBps": gbs, "frac": gbs / pk["hbm_gbs"], "launches": t["launches"],
                "share_of_step": t["ms"] / m["ms_prof"] if m.get("ms_prof") else None})
    return out


SHARED_DEVICE = False  # set by run_b200: N>1 ranks on fewer GPUs (host-transport test mode)


def c2_engine(a, spec, dev, max_batch, max_gamma, rank=0, world=1, ep=False, max_seq_len=0):
    from paper_2604_10152_b200.engine import BF16, Engine
    eng = Engine(spec, weight_type=BF16, max_batch=max_batch, max_gamma=max_gamma, device=dev,
                 ep_rank=rank if ep else 0, ep_world=world if ep else 1, max_seq_len=max_seq_len)
    if ep and SHARED_DEVICE:
        from paper_2604_10152_b200.engine import HostTransport, gloo_allgather
        eng.attach_host(HostTransport(gloo_allgather()))
    elif ep:
        eng.attach_nccl(share_nccl_id(rank))
    eng.init_device(0)
    eng.build_affinity_device()
    return eng


def section_sweep(eng, stream, a, spec, pk) -> dict:
    """BASELINE's metric is quoted over batch 1-64: every batch size on the headline engine."""
    from paper_2604_10152_b200.engine import RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    rows = {}
    for B in (1, 2, 4, 8, 16, 32):
        m = spec_measure(eng, stream, RunCfg(gamma=a.gamma, n_draft=a.n_draft, max_new_tokens=1 << 30),
                         make_prompts(1000, B, 8, spec.vocab), steps=4, warmup=2)
        r = expert_roofline(m, pk)
        rows[str(B)] = {"tokens_per_s": m["tokens"] / (m["ms"] * 1e-3), "ms_per_step": m["ms"] / 4, "tau": m["tau"],
                        "expert_gemm_hbm_frac": r["frac"], "expert_gemm_share_of_step": r["share_of_step"],
                        "hbm_expert_bytes_per_token": m["alg_expert_bytes"] / max(1, m["tokens"])}
    return rows


def section_ondemand(eng, a, spec, B: int, new_tokens: int = 6) -> dict:
    """The non-speculative comparator (baselines.cpp:29-105) on the same HBM-resident engine: one target
    pass per token.  HBM expert bytes/token = distinct experts touched per step (the ledger's keys: the
    reference flushes every step) x real bytes per expert."""
    from paper_2604_10152_b200.engine import RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    od = eng.run_ondemand(RunCfg(gamma=a.gamma, max_new_tokens=new_tokens), make_prompts(1000, B, 8, spec.vocab))
    bpe = eng.info()["bytes_per_expert"]
    toks = od.metrics["tokens_total"]
    return {"workload": f"on-demand greedy decode (run_ondemand), B={B}, {new_tokens} tokens per sequence",
            "tokens_per_s": toks / od.metrics["gpu_s"], "ms_per_token_step": 1e3 * od.metrics["gpu_s"] / new_tokens,
            "hbm_expert_bytes_per_token": len(od.ledger) * bpe / max(1, toks)}


def section_gamma(eng, stream, a, spec, pk, gamma: int, B: int) -> dict:
    """C2 B=64 at a deeper speculation depth: gamma=8 puts n_e = B*(gamma+1)*K/E = 144 tokens per expert in
    the verify pass, the only C2 point where the north_star's tensor-pipe target is reachable."""
    from paper_2604_10152_b200.engine import RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    m = spec_measure(eng, stream, RunCfg(gamma=gamma, n_draft=a.n_draft, max_new_tokens=1 << 30),
                     make_prompts(1000, B, 8, spec.vocab), steps=4, warmup=2)
    r = expert_roofline(m, pk)
    out = {"workload": f"C2 B={B} gamma={gamma} N={a.n_draft}", "tokens_per_s": m["tokens"] / (m["ms"] * 1e-3),
           "ms_per_step": m["ms"] / 4, "tau": m["tau"], "expert_gemm": r,
           "tensor_target": "north_star: expert GEMMs >= 60% of tcgen05 peak at batch >= 32; verify-pass AI here is "
                            f"{r.get('verify', {}).get('flop_per_byte', 0):.0f} flop/B vs the ridge "
                            f"{pk['bf16_tflops'] * 1e3 / pk['hbm_gbs']:.0f}"}
    prof = os.path.join(ROOT, "profiles", "r04_ncu_gamma8_verify.json")
    if os.path.exists(prof):
        out["ncu_verify_launch"] = json.load(open(prof)).get("launches", [None])[0]
    return out


def section_shape(a, dev, shape: str, B: int, n_draft: int, pk, skew: float = 0.0, steps: int = 4,
                  attention: bool = False) -> dict:
    """A separate engine for another config of BASELINE.json (C4 fine-grained, or C2 with gate_skew), or
    C2 with real GQA attention (Mixtral's 32 query / 8 KV heads of 128, RoPE theta 1e6, paged KV cache)
    in place of the reference's prefix-mean surrogate."""
    import torch
    from paper_2604_10152_b200.engine import SWIGLU3, ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    extra = dict(attn_heads=32, kv_heads=8, head_dim=128, rope_theta=1e6) if attention else {}
    spec = ModelSpec(**SHAPES[shape], seed=0, gate_skew=skew, expert_kind=SWIGLU3, **extra)
    eng = c2_engine(a, spec, dev, B, a.gamma, max_seq_len=256 if attention else 0)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", dev))
    m = spec_measure(eng, stream, RunCfg(gamma=a.gamma, n_draft=n_draft, max_new_tokens=1 << 30),
                     make_prompts(1000, B, 8, spec.vocab), steps=steps, warmup=3)
    r = expert_roofline(m, pk)
    eng.close()
    out = {"workload": f"{SHAPE_NAMES[shape]}, swiglu3 bf16 HBM-resident, B={B}, gamma={a.gamma}, N={n_draft}, "
                       f"gate_skew={skew}" + (", real GQA attention 32q/8kv x 128, RoPE 1e6, paged KV cache (16-token "
                                              "pages), prompts prefilled" if attention else ""), "tokens_per_s": m["tokens"] / (m["ms"] * 1e-3), "ms_per_step": m["ms"] / steps,
           "tau": m["tau"], "hbm_expert_bytes_per_token": m["alg_expert_bytes"] / max(1, m["tokens"]),
           "expert_gemm": r, "gpu_launches_per_step": m["launches"] / steps,
           "breakdown_ms_per_step": {k: v["ms"] / steps for k, v in m["prof"].items() if v["launches"]}}
    return out


def measure_disk_read(dirpath: str, gib: int = 4) -> dict:
    """Sequential O_DIRECT read bandwidth of the SSD tier's directory: a fresh file, 8 MB reads from 4
    threads (the store's own reader shape), page cache bypassed (buffered + DONTNEED where O_DIRECT is
    refused) -- the SSD tier's roofline."""
    import mmap
    import threading
    path = os.path.join(dirpath, f"smoe_diskbench_{os.getpid()}.bin")
    chunk, n = 8 << 20, (gib << 30) // (8 << 20)
    buf = mmap.mmap(-1, chunk)
    buf.write(os.urandom(1 << 20) * 8)
    flags = os.O_RDWR | os.O_CREAT | os.O_TRUNC
    try:
        fd = os.open(path, flags | os.O_DIRECT, 0o600)
        direct = True
    except OSError:
        fd = os.open(path, flags, 0o600)
        direct = False
    try:
        for i in range(n):
            os.pwritev(fd, [buf], i * chunk)
        os.fsync(fd)
        if not direct:
            os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
        nxt = [0]
        lock = threading.Lock()

        def reader():
            b = mmap.mmap(-1, chunk)
            while True:
                with lock:
                    i = nxt[0]
                    nxt[0] += 1
                if i >= n:
                    return
                os.preadv(fd, [b], i * chunk)
        t0 = time.perf_counter()
        th = [threading.Thread(target=reader) for _ in range(4)]
        [t.start() for t in th]
        [t.join() for t in th]
        dt = time.perf_counter() - t0
    finally:
        os.close(fd)
        os.unlink(path)
    return {"read_gbs": n * chunk / dt / 1e9, "o_direct": direct, "bytes": n * chunk, "dir": dirpath}


def section_ssd(a, dev: int, B: int = 64, steps: int = 2) -> dict:
    """The SSD tier (offload = 2): Mixtral-8x7B-shape experts, 4 MoE layers (11.3 GB of experts in one
    file on local storage, read with O_DIRECT through pinned staging), speculative vs on-demand."""
    import torch
    from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    d = os.environ.get("SMOE_SSD_DIR", "/tmp")
    disk = measure_disk_read(d)
    spec = ModelSpec(**dict(SHAPES["c2"], num_layers=4), seed=0, expert_kind=SWIGLU3)
    eng = Engine(spec, weight_type=BF16, max_batch=B, max_gamma=a.gamma, device=dev, offload=2)
    eng.init_device(0)
    eng.build_affinity_device()
    prompts = make_prompts(2000, B, 8, spec.vocab)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", dev))
    m = spec_measure(eng, stream, RunCfg(gamma=a.gamma, n_draft=a.n_draft, max_new_tokens=1 << 30), prompts,
                     steps=steps, warmup=1, profile=False)
    r = m["res"]
    od = eng.run_ondemand(RunCfg(gamma=a.gamma, max_new_tokens=steps), prompts)
    direct = eng.counter("ssd_direct")
    eng.close()
    hb, hs = r.metrics["h2d_expert_bytes"], r.metrics["h2d_s"]
    out = {"workload": f"Mixtral-8x7B-shape experts, 4 MoE layers (11.3 GB), SSD tier in {d}, B={B}, gamma={a.gamma}, "
                       f"N={a.n_draft}", "disk": disk, "engine_o_direct": bool(direct == 1),
           "tokens_per_s": m["tokens"] / (m["ms"] * 1e-3), "tau": m["tau"],
           "ssd_to_hbm_gbs": hb / hs / 1e9 if hs else None,
           "ssd_frac_of_disk_read": (hb / hs / 1e9) / disk["read_gbs"] if hs and disk["read_gbs"] else None,
           "ondemand_tokens_per_s": od.metrics["tokens_total"] / od.metrics["gpu_s"],
           "pcie_bytes_per_token": hb / max(1, m["tokens"]),
           "ondemand_bytes_per_token": od.metrics["h2d_expert_bytes"] / max(1, od.metrics["tokens_total"])}
    out["speedup_vs_ondemand"] = out["tokens_per_s"] / out["ondemand_tokens_per_s"]
    return out


def run_b200(a) -> None:
    import torch
    global SHARED_DEVICE
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        # more ranks than visible GPUs (a one-GPU box exercising the N>1 path): ranks share devices, the
        # engines exchange over the C ABI's host transport (gloo all-gather + CUDA IPC), not NCCL
        SHARED_DEVICE = torch.cuda.device_count() < world
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        dist.init_process_group("gloo" if SHARED_DEVICE else "nccl")
    from paper_2604_10152_b200.engine import SWIGLU3, TANH2, ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts

    if a.shape == "c5" and (world < 2 or a.replicas):
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unavailable": "C5 (Mixtral-8x22B shape, 270.6 GB of "
                              "experts) needs expert parallelism over >= 2 GPUs: torchrun --nproc-per-node N bench.py "
                              "--gpus N --shape c5"}), flush=True)
        return
    if a.offload:
        if rank == 0:
            sec = offload_section(a, local, a.batch, a.steps, a.warmup, gammas=(a.gamma,))
            gv = sec["gamma"][str(a.gamma)]
            line = {"metric": METRIC, "value": gv["tokens_per_s"], "unit": "tokens/s", "n_gpus": 1, "steps": a.steps,
                    "warmup": a.warmup, "ms_per_step": gv["ms_per_step"], "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": {"workload": sec["workload"]},
                    "roofline": {"bound": "pcie", "achieved": gv["h2d_gbs"], "peak": sec["pcie_peak_gbs"],
                                 "unit": "GB/s", "frac": gv["h2d_frac_of_measured"], "traffic": None},
                    "offload": sec}
            print(json.dumps(line), flush=True)
        return
    shp = dict(SHAPES[a.shape])
    spec = ModelSpec(**shp, seed=0, gate_skew=a.skew, expert_kind=SWIGLU3 if a.expert == "swiglu3" else TANH2)
    ep = world > 1 and not a.replicas  # N > 1: experts sharded over the GPUs, rows split
    default_sections = world == 1 and a.shape == "c2" and not a.no_sections
    eng = c2_engine(a, spec, local, a.batch, max(a.gamma, 8 if default_sections else a.gamma), rank, world, ep)
    seq_seed = 1000 if ep else 1000 + rank
    prompts = make_prompts(seq_seed, a.batch, 8, spec.vocab)
    cfg = RunCfg(gamma=a.gamma, n_draft=a.n_draft, max_new_tokens=1 << 30, run_seed=0 if ep else rank)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))
    if world > 1:
        # every rank finishes its warm-up before the timed region starts (barrier inside the warm-up
        # region of spec_measure is not possible; warm up here, then measure with warmup=0)
        eng.spec_begin(cfg, prompts)
        for _ in range(a.warmup):
            eng.spec_step()
        eng.spec_end()
        dist.barrier()
    m = spec_measure(eng, stream, cfg, prompts, a.steps, a.warmup if world == 1 else 1, profile=True,
                     clocks=Clocks(local))
    ms, tokens = reduce_over_ranks(m["ms"], m["tokens"], sum_tokens=not ep)
    res = m["res"]
    pk = peaks()
    roof = expert_roofline(m, pk)

    # ---- e2e through the public API (host prompts in, host tokens out; per-phase H2D/D2H inside)
    eng.counters(reset=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    r2 = eng.run_specmoe(RunCfg(gamma=a.gamma, n_draft=a.n_draft, max_new_tokens=a.e2e_tokens,
                                run_seed=0 if ep else rank), prompts)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - w0
    c2 = eng.counters()
    e2e_tokens = r2.metrics["tokens_total"]
    e2e_ms, e2e_tokens = reduce_over_ranks(e2e_s * 1e3, e2e_tokens, sum_tokens=not ep)
    e2e_s = e2e_ms * 1e-3
    phases2 = max(1, r2.metrics["phases"])

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    # the fused MoE launch (k_gemm_tc<SwiGLU, StoreF32>) dominates the step
    dom = m["prof"]["expert_gemm"]
    alg_bytes = m["cnt_prof"]["alg_expert_bytes"]
    roof_kernel = "k_gemm_tc<SwiGLU, StoreF32> (fused MoE up+down: tcgen05 grouped expert GEMM)"
    roof_alg = "distinct (layer, expert) touched per pass x 3*d*f*2 B (swiglu3 bf16)"
    traffic, traffic_src = None, "no committed capture for this configuration"
    if a.shape == "c2" and a.batch == 64 and a.gamma == 4:
        traffic = ncu_traffic(a.gamma, "r04_ncu_fused_moe.json")
        traffic_src = ("ncu --set full, profiles/r04_ncu_fused_moe.json: dram read+write of one draft-pass and one "
                       "verify-pass launch, weighted gamma:1 like the step (committed capture of this kernel)")
    elif a.shape == "c4" and a.batch == 32 and a.gamma == 4:
        traffic = ncu_traffic(a.gamma, "r04_ncu_c4_moe.json")
        traffic_src = "ncu --set full, profiles/r04_ncu_c4_moe.json (committed capture), weighted gamma:1"
    achieved = alg_bytes / (dom["ms"] * 1e-3) / 1e9 if dom["ms"] > 0 else 0.0
    ep_mode = os.environ.get("SMOE_EP_MODE", "p2p")
    exch = ("gate/down-projection epilogues store rows into peer memory over NVLink (fused dispatch/combine)"
            if ep_mode != "a2a" else "NCCL all-to-all dispatch/combine")
    if SHARED_DEVICE:
        exch += f" (TEST MODE: {world} ranks on {torch.cuda.device_count()} GPU(s), host transport; not a multi-GPU number)"
    line = {
        "metric": METRIC, "value": tokens / (ms * 1e-3), "unit": "tokens/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "scaling": "strong" if ep else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init N(0,1/sqrt(d)) weights, synthetic prompts)",
        "config": {"workload": f"{SHAPE_NAMES[a.shape]} spec-decode, {a.expert} experts HBM-resident, "
                               f"B={a.batch}{'' if ep else '/GPU'}{f', experts sharded over {world} GPUs, rows split, {exch}' if ep else ''}, "
                               f"gamma={a.gamma}, N={a.n_draft}, hot_temporal+affinity, greedy",
                   "model": f"{a.shape} L{spec.num_layers} E{spec.experts} K{spec.top_k} d{spec.hidden} f{spec.ffn} "
                            f"V{spec.vocab}",
                   "global_batch": a.batch if ep else a.batch * world, "seq_len": 8,
                   "parallelism": f"ep{world}" if ep else f"replicas{world}",
                   "l2": "inputs larger than L2: every verify pass streams all touched expert weights "
                         "(>= 10 GB) from HBM"},
        "tau": m["tau"],
        "expert_bytes_per_token": {
            "hbm": m["cnt_prof"]["alg_expert_bytes"] * world / max(1, m["tokens_prof"]),  # rank 0's share x G
            "pcie": 0, "pcie_note": "HBM-resident config: no migration (see offload_c3)",
            "ledger_reference_units": res.metrics["bytes_total"] / max(1, res.metrics["tokens_total"])},
        "e2e": {"value": e2e_tokens / e2e_s, "unit": "tokens/s",
                "h2d_bytes_per_step": int(c2["ctl_h2d"] / phases2), "d2h_bytes_per_step": int(c2["ctl_d2h"] / phases2),
                "note": f"run_specmoe via the C ABI, {a.e2e_tokens} new tokens per sequence, host prompts in / host "
                        f"tokens out, per-phase control copies inside"},
        "gpu_launches": int(m["launches"]),
        "roofline": {"bound": "hbm", "kernel": roof_kernel, "achieved": achieved,
                     "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                     "traffic": traffic, "traffic_source": traffic_src,
                     "launches": dom["launches"],
                     "avg_launch_ms": dom["ms"] / max(1, dom["launches"]),
                     "algorithmic_bytes_per_launch": alg_bytes / max(1, dom["launches"]),
                     "share_of_step": dom["ms"] / m["ms_prof"] if m.get("ms_prof") else None,
                     "by_pass": {k: roof[k] for k in ("draft", "verify") if k in roof},
                     "measured_over": "profiled copy of the timed steps (CUDA events around each launch on the engine stream)",
                     "algorithmic_bytes": roof_alg,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if pk.get("_fallback") else ""),
                     # a read-only stream exceeds the copy figure: context for a frac near or above 1
                     "read_stream_peak": {"value": READ_STREAM_GBPS, "frac": achieved / READ_STREAM_GBPS,
                                          "source": "profiles/r04_bw_probe2.txt: tools/bw_probe2.cu, one CTA per SM "
                                                    "streaming 32 KB boxes of a tiled pool into shared memory"}},
        "breakdown_ms": {k: v["ms"] for k, v in m["prof"].items() if v["launches"]},
        "clocks": m["clocks"],
    }
    line["breakdown_ms"].update({"profiled_steps_total": m["ms_prof"], "timed_steps_total": m["ms"]})
    if default_sections:
        for key, fn in (("batch_sweep", lambda: section_sweep(eng, stream, a, spec, pk)),
                        ("ondemand_c2", lambda: section_ondemand(eng, a, spec, a.batch)),
                        ("gamma8_c2", lambda: section_gamma(eng, stream, a, spec, pk, 8, a.batch)),
                        ("c1", lambda: section_c1())):
            try:
                line[key] = fn()
            except Exception as ex:  # reported, never fatal
                line[key] = {"error": str(ex)[:300]}
        od = line["ondemand_c2"]
        if "tokens_per_s" in od:
            od["speculative_vs_ondemand_tokens_per_s"] = line["value"] / od["tokens_per_s"]
            od["speculative_vs_ondemand_expert_bytes_per_token"] = (line["expert_bytes_per_token"]["hbm"] /
                                                                    od["hbm_expert_bytes_per_token"])
    if world == 1:
        eng.close()
    if default_sections:
        for key, kw in (("hot_skew2_c2", dict(shape="c2", B=a.batch, n_draft=a.n_draft, skew=2.0)),
                        ("c4", dict(shape="c4", B=32, n_draft=8)),
                        ("attention_c2", dict(shape="c2", B=a.batch, n_draft=a.n_draft, attention=True))):
            try:
                line[key] = section_shape(a, local, pk=pk, **kw)
            except Exception as ex:
                line[key] = {"error": str(ex)[:300]}
        if "expert_gemm" in line["c4"]:
            line["c4"]["expert_gemm"]["traffic"] = ncu_traffic(a.gamma, "r04_ncu_c4_moe.json")
    if not a.no_offload_section and world == 1:
        try:
            line["offload_c3"] = offload_section(a, local, a.offload_batch, a.offload_steps, 1, gammas=(2, 4, 8))
        except Exception as ex:
            line["offload_c3"] = {"error": str(ex)[:300]}
    if not a.no_offload_section and world == 1 and default_sections:
        try:
            line["offload_ssd"] = section_ssd(a, local)
        except Exception as ex:
            line["offload_ssd"] = {"error": str(ex)[:300]}
    if not a.no_cpu_baseline and world == 1:
        thr = a.cpu_threads or os.cpu_count()
        try:
            line["cpu_baseline"] = cpu_reference(a.shape, a.expert, a.gamma, a.n_draft, thr, tau=line["tau"])
        except Exception as ex:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(a) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    thr = a.cpu_threads or os.cpu_count()
    cb = cpu_reference(a.shape, a.expert, a.gamma, a.n_draft, thr, steps=a.steps, warmup=a.warmup)
    value = statistics.median(cb["step_values"])
    cb = dict(cb, value=value)
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "impl": "reference", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (reference build_model seeded weights, synthetic prompts)",
            "config": {"workload": f"{SHAPE_NAMES[a.shape]} spec-decode, {a.expert}, gamma={a.gamma}, N={a.n_draft}, "
                                   f"reference CPU path (oracle/_ref) on {thr} host threads",
                       "global_batch": thr, "seq_len": 8, "parallelism": f"cpu{thr}"},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = args_parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
