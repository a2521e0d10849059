"""Phase timeline of the persistent pass kernel (SMOE_PASS_TRACE variant build of pass_tc.cu).

    tools/build_variant.sh ptrace paper_2604_10152_b200/csrc/pass_tc.cu -DSMOE_PASS_TRACE   (swaps pass_tc.o)
    SMOE_LIB=build/variants/ptrace.so python tools/pass_trace.py B [spec|ondemand]
Per layer: A (mix) from the previous layer's D end to 'A done', B (gate rows), C (expert FFN), D (combine).
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")


def analyze(path, L=32):
    ev = np.fromfile(path, dtype=np.int64).reshape(160, 128, 24)[:148, :L]
    t0 = ev[:, 0, 0][ev[:, 0, 0] > 0].min()
    ev = np.where(ev >= t0, ev - t0, -1).astype(np.float64) / 1e3  # us since the first CTA entered layer 0
    def first(l, k):
        v = ev[:, l, k]
        v = v[v >= 0]
        return float(v.min()) if len(v) else float("nan")
    def last(l, k):
        v = ev[:, l, k]
        v = v[v >= 0]
        return float(v.max()) if len(v) else float("nan")
    rows = []
    prev_d = 0.0
    for l in range(L):
        a_end, b_end, c_end, d_end = first(l, 3), first(l, 1), first(l, 5), last(l, 6)
        rows.append(dict(layer=l, A=round(a_end - prev_d, 1), B=round(b_end - a_end, 1), C=round(c_end - b_end, 1),
                         D=round(d_end - c_end, 1), c_claims_done_spread=round(last(l, 2) - first(l, 2), 1),
                         markD_spread=round(last(l, 7) - first(l, 7), 1)))
        prev_d = d_end
    # inside the B / D rows of one CTA (the first that ran a row of that layer): claim -> resid -> gemv -> select
    # -> dispatch -> fenced; D: claim -> rows done -> fenced
    for l in (1, 2):
        has = np.nonzero(ev[:, l, 8] >= 0)[0]
        if len(has):
            c = has[0]
            s = ev[c, l]
            print(json.dumps(dict(layer=l, cta=int(c), resid=round(s[9] - s[8], 2), gemv=round(s[10] - s[9], 2),
                                  select=round(s[11] - s[10], 2), dispatch=round(s[12] - s[11], 2),
                                  fence_B=round(s[13] - s[12], 2), wait_A_to_claim=round(s[8] - s[3], 2),
                                  D_rows=round(s[14] - s[5], 2), fence_D=round(s[15] - s[14], 2),
                                  D_pos=round(s[16] - s[5], 2), D_bar=round(s[17] - s[16], 2), D_issue=round(s[18] - s[17], 2),
                                  D_fill=round(s[19] - s[18], 2), D_compute=round(s[14] - s[19], 2))))
    tot = {k: round(sum(r[k] for r in rows), 1) for k in ("A", "B", "C", "D")}
    for r in rows[:4] + rows[-2:]:
        print(json.dumps(r))
    print("totals us", json.dumps(tot), "pass us", round(prev_d, 1))


if __name__ == "__main__":
    from paper_2604_10152_b200 import engine as eng
    from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg
    from paper_2604_10152_b200.prompts import make_prompts
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    mode = sys.argv[2] if len(sys.argv) > 2 else "spec"
    spec = ModelSpec(num_layers=32, experts=8, top_k=2, hidden=4096, ffn=14336, vocab=32000, expert_kind=SWIGLU3)
    e = Engine(spec, weight_type=BF16, max_batch=B, max_gamma=4).init_device(0)
    e.build_affinity_device()
    prompts = make_prompts(1000, B, 8, spec.vocab)
    if mode == "spec":
        e.spec_begin(RunCfg(gamma=4, n_draft=4, max_new_tokens=1 << 30), prompts)
        for _ in range(3):
            e.spec_step()
    else:
        e.run_ondemand(RunCfg(gamma=4, n_draft=4, max_new_tokens=4), prompts)
    lib = eng.lib()
    lib.smoe_pass_trace_dump.argtypes = [C.c_char_p]
    out = f"gpurun_out/pass_trace_b{B}_{mode}.bin"
    os.makedirs("gpurun_out", exist_ok=True)
    assert lib.smoe_pass_trace_dump(out.encode()) == 0
    analyze(out)
