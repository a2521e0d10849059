"""Timeline of the tcgen05 GEMM launches inside real speculative steps (SMOE_TC_TRACE variant build).

    tools/build_variant.sh trace paper_2604_10152_b200/csrc/gemm_tc.cu -DSMOE_TC_TRACE
    SMOE_LIB=build/variants/trace.so python tools/tc_trace.py [B] [gamma]     (on the GPU box)
    python tools/tc_trace.py --analyze gpurun_out/tc_trace.bin                 (anywhere)

Per fused MoE launch: duration, achieved weight GB/s, start ramp (launch start -> a CTA's first full
stage), tail (a CTA's last accumulator -> launch end), and the steady rate between 10% and 90% of
the weight bytes completed.
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")

D, F = 4096, 14336
UP_UNIT = 128 * D * 2  # 128 weight rows x K=d bf16


def run(B, gamma, out):
    from paper_2604_10152_b200 import engine as eng
    from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    spec = ModelSpec(num_layers=32, experts=8, top_k=2, hidden=D, ffn=F, vocab=32000, expert_kind=SWIGLU3)
    e = Engine(spec, weight_type=BF16, max_batch=B, max_gamma=gamma).init_device(0)
    e.build_affinity_device()
    e.spec_begin(RunCfg(gamma=gamma, n_draft=4, max_new_tokens=1 << 30), make_prompts(1000, B, 8, spec.vocab))
    for _ in range(4):
        e.spec_step()
    lib = eng.lib()
    lib.smoe_tc_trace_dump.argtypes = [C.c_char_p]
    rc = lib.smoe_tc_trace_dump(out.encode())
    assert rc == 0, rc


def analyze(path):
    raw = open(path, "rb").read()
    nl, nu, nc = np.frombuffer(raw[:12], np.int32)
    off = 12
    meta = np.frombuffer(raw[off:off + nl * 4 * 4], np.int32).reshape(nl, 4)
    off += nl * 16
    cta = np.frombuffer(raw[off:off + nl * nc * 2 * 8], np.int64).reshape(nl, nc, 2)
    off += nl * nc * 16
    un = np.frombuffer(raw[off:], np.int64).reshape(nl, nu, 6)
    rows = []
    for s in range(nl):
        total, nphase, u0, grid = (int(v) for v in meta[s])
        tag = un[s, :, 0] >> 32
        valid = un[s, :, 1] > 0
        if not valid.any() or grid <= 0:
            continue
        t = tag[valid].max()  # the slot's latest launch (older launches leave stale unit records)
        m = valid & (tag == t)
        ids = np.nonzero(m)[0]
        U = un[s, m]
        t0 = cta[s, :grid, 0].min()
        t1 = cta[s, :grid, 1].max()
        cta_id = (U[:, 0] & 0xFFFFFFFF).astype(int)
        first_full = np.array([U[cta_id == c, 3].min() if (cta_id == c).any() else t1 for c in range(grid)])
        last_done = np.array([U[cta_id == c, 5].max() if (cta_id == c).any() else t0 for c in range(grid)])
        unit_us = (U[:, 4] - U[:, 3]) / 1e3
        up = ids < u0
        kind = "mix/head" if nphase == 1 else ("moe_T>256" if total > 2 * u0 * 1.2 else "moe")
        r = dict(slot=int(s), launch=int(t), kind=kind, units=int(m.sum()), grid=grid,
                 dur_us=float((t1 - t0) / 1e3),
                 ramp_us=float(np.median((first_full - t0) / 1e3)),
                 tail_us=float(np.mean((t1 - last_done) / 1e3)),
                 up_unit_us=float(np.median(unit_us[up])) if up.any() else 0.0,
                 down_unit_us=float(np.median(unit_us[~up])) if (~up).any() else 0.0,
                 n_up=int(up.sum()), n_down=int((~up).sum()),
                 cta_start_spread=float((cta[s, :grid, 0].max() - t0) / 1e3))
        rows.append(r)
    rows.sort(key=lambda r: r["launch"])
    # aggregate per class (moe launches split by their unit count: draft passes touch fewer experts)
    agg = {}
    for r in rows:
        key = (r["kind"], r["n_up"], r["n_down"])
        agg.setdefault(key, []).append(r)
    for key, rs in sorted(agg.items()):
        f = lambda k: round(float(np.mean([x[k] for x in rs])), 1)  # noqa: E731
        print(json.dumps(dict(kind=key[0], n_up=key[1], n_down=key[2], launches=len(rs), dur_us=f("dur_us"),
                              ramp_us=f("ramp_us"), tail_us=f("tail_us"), up_unit_us=f("up_unit_us"),
                              down_unit_us=f("down_unit_us"), cta_start_spread=f("cta_start_spread"))))
    return rows


if __name__ == "__main__":
    if sys.argv[1:2] == ["--analyze"]:
        analyze(sys.argv[2])
    else:
        B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
        g = int(sys.argv[2]) if len(sys.argv) > 2 else 4
        os.makedirs("gpurun_out", exist_ok=True)
        out = f"gpurun_out/tc_trace_b{B}{os.environ.get('TAG', '')}.bin"
        run(B, g, out)
        rows = analyze(out)
        json.dump(rows, open(out.replace(".bin", ".json"), "w"), indent=0)
