"""Layer-pass timeline of the per-layer path from a tc_trace dump: Mix GEMM and fused MoE launch
windows (first CTA start .. last CTA end) and the gaps between them.
    python tools/tc_gaps.py gpurun_out/tc_trace_b64.bin"""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
nl, nu, nc = np.frombuffer(raw[:12], np.int32)
off = 12
meta = np.frombuffer(raw[off:off + nl * 16], np.int32).reshape(nl, 4)
off += nl * 16
cta = np.frombuffer(raw[off:off + nl * nc * 16], np.int64).reshape(nl, nc, 2)
off += nl * nc * 16
un = np.frombuffer(raw[off:], np.int64).reshape(nl, nu, 6)
ev = []
for s in range(nl):
    total, nphase, u0, grid = (int(v) for v in meta[s])
    if grid <= 0:
        continue
    tag = un[s, :, 0] >> 32
    valid = un[s, :, 1] > 0
    if not valid.any():
        continue
    t = int(tag[valid].max())  # the slot's latest launch (older launches leave stale unit records)
    t0, t1 = cta[s, :grid, 0].min(), cta[s, :grid, 1].max()
    U = un[s, valid & (tag == t)]
    first_full = U[:, 3].min()
    ev.append((t, "moe" if nphase == 2 else "gemm", int(t0), int(t1), int(first_full), int(total)))
ev.sort()
# consecutive (gemm, moe) pairs: gemm = Mix of the layer (or head)
rows = []
for i in range(1, len(ev)):
    a, b = ev[i - 1], ev[i]
    if a[1] == "gemm" and b[1] == "moe" and i >= 2 and ev[i - 2][1] == "moe":
        prev = ev[i - 2]
        rows.append(dict(moe_T=b[5], prev_moe_end_to_mix_start=(a[2] - prev[3]) / 1e3, mix_dur=(a[3] - a[2]) / 1e3,
                         mix_end_to_moe_start=(b[2] - a[3]) / 1e3, moe_start_to_first_full=(b[4] - b[2]) / 1e3,
                         moe_dur=(b[3] - b[2]) / 1e3, prev_moe_end_to_next_moe_first_full=(b[4] - prev[3]) / 1e3))
for key in ("prev_moe_end_to_mix_start", "mix_dur", "mix_end_to_moe_start", "moe_start_to_first_full", "moe_dur",
            "prev_moe_end_to_next_moe_first_full"):
    v = np.array([r[key] for r in rows])
    print(f"{key:40s} median {np.median(v):8.1f} us   mean {v.mean():8.1f}  (n={len(v)})")
