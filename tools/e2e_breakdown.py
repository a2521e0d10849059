"""Where an e2e run's wall time goes: spec_begin, each spec_step (host wall, tokens, active rows) and
spec_end, for one bench shape.  usage (GPU box): python tools/e2e_breakdown.py [c2|c4] [batch] [new_tokens]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_10152_b200.engine import SWIGLU3, ModelSpec, RunCfg  # noqa: E402
from paper_2604_10152_b200.prompts import make_prompts  # noqa: E402


def main():
    shape = sys.argv[1] if len(sys.argv) > 1 else "c4"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    new = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    nd = 8 if shape == "c4" else 4

    class A:
        gamma = 4
    spec = ModelSpec(**dict(bench.SHAPES[shape]), seed=0, expert_kind=SWIGLU3)
    eng = bench.c2_engine(A, spec, 0, B, 4)
    prompts = make_prompts(1000, B, 8, spec.vocab)
    cfg = RunCfg(gamma=4, n_draft=nd, max_new_tokens=new)
    for rep in range(2):
        t0 = time.perf_counter()
        eng.spec_begin(cfg, prompts)
        t1 = time.perf_counter()
        steps = []
        while True:
            s0 = time.perf_counter()
            tok, act = eng.spec_step()
            steps.append((time.perf_counter() - s0, tok, act))
            if act == 0:
                break
        t2 = time.perf_counter()
        r = eng.spec_end()
        t3 = time.perf_counter()
        t4 = time.perf_counter()
        r2 = eng.run_specmoe(cfg, prompts)
        t5 = time.perf_counter()
        tot = r.metrics["tokens_total"]
        print(f"rep {rep}: begin {1e3*(t1-t0):.2f} ms, {len(steps)} steps {1e3*(t2-t1):.1f} ms, end {1e3*(t3-t2):.2f} ms;"
              f" tokens {tot} -> {tot/(t3-t0):.0f} tok/s; run_specmoe {1e3*(t5-t4):.1f} ms -> "
              f"{r2.metrics['tokens_total']/(t5-t4):.0f} tok/s")
        if rep == 1:
            for i, (dt, tok, act) in enumerate(steps):
                print(f"  step {i:3d}: {1e3*dt:7.2f} ms tokens {tok:4d} active {act}")
    eng.close()


if __name__ == "__main__":
    main()
