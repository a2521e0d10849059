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
NF = 10  # TrUnit fields: cta, claim, tma_done, mma_first, mma_done, epi_done, epi_start, epi_stored, epi_fenced,
# epi_barred
UP_UNIT = 128 * D * 2  # 128 weight rows x K=d bf16


def run(B, gamma, out):
    from paper_2604_10152_b200 import engine as eng
    from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    if os.environ.get("SHAPE") == "c4":  # fine-grained E64 K6 (C4), N=8
        spec = ModelSpec(num_layers=28, experts=64, top_k=6, hidden=2048, ffn=1408, vocab=102400,
                         moe_mask=[0] + [1] * 27, expert_kind=SWIGLU3)
        nd = 8
    else:
        spec = ModelSpec(num_layers=32, experts=8, top_k=2, hidden=D, ffn=F, vocab=32000, expert_kind=SWIGLU3)
        nd = 4
    e = Engine(spec, weight_type=BF16, max_batch=B, max_gamma=gamma).init_device(0)
    e.build_affinity_device()
    e.spec_begin(RunCfg(gamma=gamma, n_draft=nd, max_new_tokens=1 << 30), make_prompts(1000, B, 8, spec.vocab))
    for _ in range(4):
        e.spec_step()
    lib = eng.lib()
    lib.smoe_tc_trace_dump.argtypes = [C.c_char_p]
    rc = lib.smoe_tc_trace_dump(out.encode())
    assert rc == 0, rc
    lib.smoe_rk_trace_dump.argtypes = [C.c_char_p]
    lib.smoe_rk_trace_dump(out.replace(".bin", "_rk.bin").encode())  # row kernels (gate, combine)


def row_kernel_launches(path):
    """Row-kernel launches from the per-block records: kernel id -> [(entry, wait released, end)]."""
    if not os.path.exists(path):
        return {}
    raw = open(path, "rb").read()
    n = int(np.frombuffer(raw[:4], np.int32)[0])
    rec = np.frombuffer(raw[4:4 + n * 56], dtype=np.dtype(
        [("kid", np.int32), ("blk", np.int32), ("t_in", np.int64), ("t_wait", np.int64), ("t_end", np.int64),
         ("t_m", np.int64, (3,))]))
    ga = np.sort(rec[rec["kid"] == 1], order="t_in")
    gl = np.split(ga, np.nonzero(np.diff(ga["t_in"]) > 30_000)[0] + 1) if len(ga) else []
    for label, sel in (("draft", [x for x in gl if len(x) <= 128]), ("verify", [x for x in gl if len(x) > 128])):
        if not sel:
            continue
        # gate anatomy per block (us after its wait released): rms done, GEMV done, selected, end
        g = np.concatenate(sel)
        w = g["t_wait"]
        print(json.dumps({"gate_block_anatomy_us": label, "launches": len(sel), "blocks": int(np.median([len(x) for x in sel])),
            "launch_in_to_last_end": round(float(np.median([(x["t_end"].max() - x["t_in"].min()) / 1e3 for x in sel])), 2),
            "first_wait_to_last_end": round(float(np.median([(x["t_end"].max() - x["t_wait"].min()) / 1e3 for x in sel])), 2), **{
            "rms_done": round(float(np.median((g["t_m"][:, 0] - w) / 1e3)), 2),
            "gemv_done": round(float(np.median((g["t_m"][:, 1] - w) / 1e3)), 2),
            "selected": round(float(np.median((g["t_m"][:, 2] - w) / 1e3)), 2),
            "end": round(float(np.median((g["t_end"] - w) / 1e3)), 2),
            "end_p90": round(float(np.percentile((g["t_end"] - w) / 1e3, 90)), 2),
            "wait_spread_p90": round(float(np.percentile((w - np.min(w)) / 1e3, 90)), 2)}}))
    out = {}
    for kid in np.unique(rec["kid"]):
        r = np.sort(rec[rec["kid"] == kid], order="t_in")
        cut = np.nonzero(np.diff(r["t_in"]) > 30_000)[0] + 1  # launches of one kernel are >= ~250 us apart
        out[int(kid)] = [(int(g["t_in"].min()), int(g["t_wait"].min()), int(g["t_end"].max())) for g in np.split(r, cut)]
    return out


def analyze(path):
    raw = open(path, "rb").read()
    nl, nu, nc = np.frombuffer(raw[:12], np.int32)
    off = 12
    meta = np.frombuffer(raw[off:off + nl * 4 * 4], np.int32).reshape(nl, 4)
    off += nl * 16
    cta = np.frombuffer(raw[off:off + nl * nc * 2 * 8], np.int64).reshape(nl, nc, 2)
    off += nl * nc * 16
    un = np.frombuffer(raw[off:off + nl * nu * NF * 8], np.int64).reshape(nl, nu, NF)
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
        # unit anatomy (us): claim -> producer issued its last stage -> last MMA done -> epilogue done
        epi_us = (U[:, 5] - U[:, 4]) / 1e3
        last = np.zeros(len(U), bool)
        for c in np.unique(cta_id):
            k = np.nonzero(cta_id == c)[0]
            last[k[np.argmax(U[k, 5])]] = True
        anat_x = dict(epi_up=float(np.median(epi_us[up])) if up.any() else 0.0,
                      epi_down=float(np.median(epi_us[~up])) if (~up).any() else 0.0,
                      epi_last=float(np.median(epi_us[last])),
                      mma_first_to_done_last=float(np.median((U[last, 4] - U[last, 3]) / 1e3)))
        anat = dict(claim_to_issued=float(np.median((U[:, 2] - U[:, 1]) / 1e3)),
                    mma_first_to_issued=float(np.median((U[:, 2] - U[:, 3]) / 1e3)),
                    issued_to_mma_done=float(np.median((U[:, 4] - U[:, 2]) / 1e3)),
                    epilogue=float(np.median((U[:, 5] - U[:, 4]) / 1e3)))
        r = dict(slot=int(s), launch=int(t), kind=kind, units=int(m.sum()), grid=grid,
                 dur_us=float((t1 - t0) / 1e3),
                 ramp_us=float(np.median((first_full - t0) / 1e3)),
                 tail_us=float(np.mean((t1 - last_done) / 1e3)),
                 up_unit_us=float(np.median(unit_us[up])) if up.any() else 0.0,
                 down_unit_us=float(np.median(unit_us[~up])) if (~up).any() else 0.0,
                 n_up=int(up.sum()), n_down=int((~up).sum()),
                 cta_start_spread=float((cta[s, :grid, 0].max() - t0) / 1e3),
                 t0=int(t0), t1=int(t1), first_stage=int(first_full.min()), **anat, **anat_x)
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
                              down_unit_us=f("down_unit_us"), cta_start_spread=f("cta_start_spread"),
                              claim_to_issued=f("claim_to_issued"), mma_first_to_issued=f("mma_first_to_issued"),
                              issued_to_mma_done=f("issued_to_mma_done"), epilogue=f("epilogue"),
                              epi_up=f("epi_up"), epi_down=f("epi_down"), epi_last=f("epi_last"))))
    # in-step timeline between consecutive fused MoE launches: the previous MoE launch's end -> the
    # mix launch (start, end) -> this MoE launch's first full weight stage
    gaps = []
    prev = None
    mix = None
    for r in rows:
        if r["kind"] == "mix/head":
            mix = r
            continue
        if prev is not None and mix is not None and mix["t0"] > prev["t1"] - 50_000:
            gaps.append(dict(between_moe_us=(r["first_stage"] - prev["t1"]) / 1e3,
                             mix_start_us=(mix["t0"] - prev["t1"]) / 1e3, mix_end_us=(mix["t1"] - prev["t1"]) / 1e3,
                             moe_launch_us=(r["t0"] - prev["t1"]) / 1e3, moe_dur_us=r["dur_us"]))
        prev, mix = r, None
    rk = row_kernel_launches(path.replace(".bin", "_rk.bin"))
    if rk:
        # per MoE launch: the combine after it and the gate before the next one, relative to its end
        moes = [r for r in rows if r["kind"] != "mix/head"]
        mixes = [r for r in rows if r["kind"] == "mix/head"]
        tl = {"draft": [], "verify": []}
        for a, b in zip(moes, moes[1:]):
            t1 = a["t1"]
            comb = [c for c in rk.get(2, []) if t1 - 100_000 < c[0] and c[2] > t1 and c[2] < b["t0"] + 50_000]
            gate = [c for c in rk.get(1, []) if a["t1"] - 100_000 < c[0] and c[2] < b["first_stage"] and c[2] > t1]
            mix = [m for m in mixes if m["t1"] > t1 and m["t1"] < b["first_stage"]]
            if len(comb) != 1 or len(gate) != 1 or len(mix) != 1:
                continue
            c, g, m = comb[0], gate[0], mix[0]
            us = lambda t: (t - t1) / 1e3  # noqa: E731
            tl["verify" if b["n_up"] > 1000 else "draft"].append(dict(
                combine_in=us(c[0]), combine_waited=us(c[1]), combine_end=us(c[2]),
                mix_start=us(m["t0"]), mix_first_stage=us(m["first_stage"]), mix_end=us(m["t1"]),
                gate_in=us(g[0]), gate_waited=us(g[1]), gate_end=us(g[2]),
                moe_launch=us(b["t0"]), moe_first_stage=us(b["first_stage"]), moe_end=us(b["t1"])))
        for k, v in tl.items():
            if v:
                print(json.dumps({"timeline_after_moe_end_us": k, "n": len(v),
                                  **{f: round(float(np.median([x[f] for x in v])), 2) for f in v[0]}}))
    if gaps:
        print(json.dumps({"between_moe_launches": {k: round(float(np.median([g[k] for g in gaps])), 2) for k in gaps[0]},
                          "n": len(gaps)}))
    return rows


def dump_units(path, rows, dst, per_kind=3):
    """Every unit of a few fused MoE launches per kind (draft / verify by unit count): [cta, claim,
    tma_done, mma_first, mma_done, epi_done] in us from the launch's first CTA start, + unit id."""
    raw = open(path, "rb").read()
    nl, nu, nc = np.frombuffer(raw[:12], np.int32)
    off = 12 + nl * 16
    cta = np.frombuffer(raw[off:off + nl * nc * 2 * 8], np.int64).reshape(nl, nc, 2)
    off += nl * nc * 16
    un = np.frombuffer(raw[off:off + nl * nu * NF * 8], np.int64).reshape(nl, nu, NF)
    off += nl * nu * NF * 8
    dep = np.frombuffer(raw[off:off + nl * nc * 8], np.int64).reshape(nl, nc)
    out, seen = [], {}
    for r in rows:
        if r["kind"] == "mix/head":
            continue
        k = r["n_up"] + r["n_down"]
        if seen.get(k, 0) >= per_kind:
            continue
        seen[k] = seen.get(k, 0) + 1
        s = r["slot"]
        tag = un[s, :, 0] >> 32
        m = (un[s, :, 1] > 0) & (tag == r["launch"])
        t0 = r["t0"]
        ids = np.nonzero(m)[0]
        U = un[s, m]
        units = [[int(U[i, 0] & 0xFFFFFFFF)] + [round((int(U[i, j]) - t0) / 1e3, 2) for j in range(1, 6)] + [int(ids[i])]
                 + [round((int(U[i, j]) - t0) / 1e3, 2) if U[i, j] else None for j in range(6, NF)]
                 for i in range(len(U))]
        ends = [round((int(x) - t0) / 1e3, 2) for x in cta[s, :r["grid"], 1]]
        deps = [round((int(x) - t0) / 1e3, 2) for x in dep[s, :r["grid"]]]
        out.append({"launch": r["launch"], "t0_ns": int(t0), "units_total": k, "dur_us": r["dur_us"], "units": units,
                    "cta_end": ends, "cta_dep_released": deps})
    json.dump(out, open(dst, "w"))


if __name__ == "__main__":
    if sys.argv[1:2] == ["--analyze"]:
        analyze(sys.argv[2])
    else:
        B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
        g = int(sys.argv[2]) if len(sys.argv) > 2 else 4
        os.makedirs("gpurun_out", exist_ok=True)
        out = f"/tmp/tc_trace_b{B}{os.environ.get('TAG', '')}.bin"  # large; only the summary travels back
        run(B, g, out)
        rows = analyze(out)
        json.dump(rows, open("gpurun_out/" + os.path.basename(out).replace(".bin", ".json"), "w"), indent=0)
        dump_units(out, rows, "gpurun_out/" + os.path.basename(out).replace(".bin", "_units.json"))
