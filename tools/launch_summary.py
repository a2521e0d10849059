"""Group an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel into a profiles/ JSON.

usage: python tools/launch_summary.py <launches.csv> <out.json> <title>
"kernels": every launch of the capture (init included); "step_kernels": the launches after the last
weight-init kernel (k_fill_normal* / k_pair_sqdist*), i.e. the speculative steps, with their shares.
"""
import collections
import csv
import json
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, out, title):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, dd = rows[hi], rows[hi + 1:]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = []
    for r in dd:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        seq.append((name, float(r[mi].replace(",", "")) * UNIT[r[ui]]))
    init = [i for i, (n, _) in enumerate(seq) if "k_fill_normal" in n or "k_pair_sqdist" in n]
    first_step = (max(init) + 1) if init else 0

    def group(items):
        agg = collections.defaultdict(lambda: [0, 0.0])
        for n, t in items:
            agg[n][0] += 1
            agg[n][1] += t
        tot = sum(t for _, t in items)
        return {n: {"launches": c, "total_us": round(t, 1), "avg_us": round(t / c, 2), "share": round(t / tot, 4)}
                for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])}, tot
    allk, tot = group(seq)
    stepk, stot = group(seq[first_step:])
    json.dump({"title": title, "launches": len(seq), "total_us": round(tot, 1), "kernels": allk,
               "step_launches": len(seq) - first_step, "step_total_us": round(stot, 1), "step_kernels": stepk},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:4])
