"""Summarise single-launch ncu --set full captures into a profiles/ JSON.

usage: python tools/ncu_summary.py <out.json> <title> <rep>:<label>:<algorithmic_MB> [...]
Per launch: duration, DRAM read/write, traffic over algorithmic bytes, achieved GB/s of the algorithmic
bytes against MEASURED_PEAKS.json, DRAM % of theoretical, tensor-pipe %, SM-active fraction, registers, smem.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, d = rows[0], rows[1], rows[2]
    return {k: (v, uu) for k, v, uu in zip(h, d, u)}


def num(m, k):
    v, u = m[k]
    return float(v.replace(",", "")) * SCALE.get(u, 1.0)


def main():
    out, title = sys.argv[1], sys.argv[2]
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    launches = []
    for spec in sys.argv[3:]:
        rep, label, alg = spec.rsplit(":", 2)
        m = raw(rep)
        t = num(m, "gpu__time_duration.sum")  # us
        rd, wr = num(m, "dram__bytes_read.sum"), num(m, "dram__bytes_write.sum")  # MB
        alg = float(alg)
        launches.append({
            "launch": label, "time_us": round(t, 2), "dram_read_MB": round(rd, 2), "dram_write_MB": round(wr, 2),
            "algorithmic_MB": alg, "traffic_over_algorithmic": round((rd + wr) / alg, 4),
            "achieved_GBps": round(alg / t * 1e3, 1), "peak_GBps": peak, "frac_of_peak": round(alg / t * 1e3 / peak, 4),
            "dram_pct_of_theoretical": round(num(m, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), 2),
            "tensor_pipe_pct": round(num(m, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"), 2),
            "sm_active_frac": round(num(m, "sm__cycles_active.avg") / num(m, "gpc__cycles_elapsed.max"), 3),
            "registers": int(num(m, "launch__registers_per_thread")),
            "smem_KB": round(num(m, "launch__shared_mem_per_block_dynamic") * 1e3, 2) if m["launch__shared_mem_per_block_dynamic"][1] == "Mbyte" else m["launch__shared_mem_per_block_dynamic"][0]})
    json.dump({"title": title, "note": "cold-cache single replayed launch (ncu --set full --clock-control none)",
               "launches": launches}, open(out, "w"), indent=1)
    print(json.dumps(launches, indent=1))


if __name__ == "__main__":
    main()
