"""Top stalled SASS instructions of an `ncu --page source --csv --print-source sass` export.

  python tools/ncu_src_top.py gpurun_out/x_src.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"total samples {tot}")
agg = {}
for r in data:
    op = r[idx["Source"]].strip().split()[0] if r[idx["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[idx["Source"]].strip().split()[1]
    op = op.split(".")[0]
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    agg[op] = agg.get(op, 0) + s
print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:16]))
data.sort(key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[:n]:
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((int(r[idx[c]] or 0), c) for c in stall_cols), reverse=True)[:3]
    conf = r[idx["L1 Wavefronts Shared Excessive"]]
    print(f"{100*s/tot:5.2f}% {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:60]:60s} "
          + " ".join(f"{c[6:]}={v}" for v, c in top) + (f" smem_excess={conf}" if conf not in ("0", "") else ""))
