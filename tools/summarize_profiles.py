"""Summarise an ncu launch list + an ncu --set full capture of k_gemm_tc into profiles/.

usage: python tools/summarize_profiles.py <launches.csv> <prof.ncu-rep> <round> <title> <d> <f> <E_touched>
"""
import collections
import csv
import json
import subprocess
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, dd = rows[hi], rows[hi + 1:]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg, tot = collections.defaultdict(lambda: [0, 0.0]), 0.0
    for r in dd:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").split("<")[0]
        v = float(r[mi].replace(",", "")) * UNIT[r[ui]]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    return len(dd), tot, agg


def full(path, names, alg):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, data = rows[0], rows[2:]

    def col(n):
        i = h.index(n)
        return [r[i] for r in data]
    res = []
    for i in range(len(data)):
        rd = float(col("dram__bytes_read.sum")[i]) * 1e6
        wr = float(col("dram__bytes_write.sum")[i]) * 1e6
        t = float(col("gpu__time_duration.sum")[i]) * 1e-6
        res.append({"launch": names[i] if i < len(names) else f"launch{i}", "grid": col("Grid Size")[i],
                    "time_us": t * 1e6, "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6,
                    "algorithmic_MB": alg[i] / 1e6, "traffic_over_algorithmic": (rd + wr) / alg[i],
                    "achieved_GBps": alg[i] / t / 1e9,
                    "dram_pct_of_theoretical": float(col("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")[i]),
                    "tensor_pipe_pct": float(col("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")[i]),
                    "registers": int(col("launch__registers_per_thread")[i]),
                    "smem_KB": float(col("launch__shared_mem_per_block_dynamic")[i])})
    return res


def main():
    lpath, rep, rnd, title, d, f, et = sys.argv[1:8]
    d, f, et = int(d), int(f), int(et)
    names = ["mix (dense, K=d)", f"expert up+gate SwiGLU ({et} experts, K=d)", f"expert down ({et} experts, K=f)"]
    alg = [d * d * 2, et * 2 * f * d * 2, et * d * f * 2]
    launches = full(rep, names, alg)
    exp = [l for l in launches if l["launch"].startswith("expert")]
    json.dump({"round": int(rnd), "title": title,
               "note": "cold-cache, serialised replays: compare shares, not absolutes",
               "launches": launches,
               "dram_bytes_per_launch": sum((l["dram_read_MB"] + l["dram_write_MB"]) * 1e6 for l in exp) / len(exp),
               "algorithmic_bytes_per_launch": sum(l["algorithmic_MB"] * 1e6 for l in exp) / len(exp)},
              open("profiles/ncu_expert_gemm.json", "w"), indent=1)
    n, tot, agg = launch_list(lpath)
    with open(f"profiles/r{int(rnd):02d}_summary.md", "w") as fo:
        fo.write(f"# Round {rnd} profile summary: {title}\n\n## Launch list (one speculative step)\n\n")
        fo.write(f"{n} launches, {tot / 1e3:.2f} ms serialised kernel time (cold cache).\n\n")
        fo.write("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|\n")
        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fo.write(f"| {k} | {c} | {t / 1e3:.3f} | {t / tot:.3f} | {t / c:.2f} |\n")
        fo.write("\n## ncu --set full, k_gemm_tc (verify pass)\n\n| launch | grid | us | DRAM MB r+w | algorithmic MB | "
                 "traffic/alg | achieved GB/s | DRAM % theor. | tensor % | regs | smem KB |\n|---|---|---|---|---|---|---|---|---|---|---|\n")
        for l in launches:
            fo.write(f"| {l['launch']} | {l['grid']} | {l['time_us']:.1f} | {l['dram_read_MB'] + l['dram_write_MB']:.1f} | "
                     f"{l['algorithmic_MB']:.1f} | {l['traffic_over_algorithmic']:.4f} | {l['achieved_GBps']:.0f} | "
                     f"{l['dram_pct_of_theoretical']:.1f} | {l['tensor_pipe_pct']:.1f} | {l['registers']} | {l['smem_KB']:.0f} |\n")
    print(open(f"profiles/r{int(rnd):02d}_summary.md").read())


if __name__ == "__main__":
    main()
