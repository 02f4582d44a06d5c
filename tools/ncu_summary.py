"""Summarise an ncu capture (and a launch list) into profiles/.

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --cells 16777216 --levels 4 --tag r01

Writes profiles/ncu_<tag>.json and appends a markdown section to
profiles/README.md; profiles/ncu_summary.json (read by bench.py for the
`traffic` field) is updated with the dominant-kernel numbers.
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_cycles": "sm__cycles_elapsed.avg",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "warp_instructions": "smsp__inst_executed.sum",
    "stall_long_sb": "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "stall_wait": "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "stall_short_sb": "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "stall_no_instruction": "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "stall_not_selected": "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
}

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3,
              "usecond": 1, "msecond": 1e3, "nsecond": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--cells", type=int, required=True, help="lattice cells one launch updates")
    ap.add_argument("--levels", type=int, required=True, help="time levels per launch")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--note", default="")
    ap.add_argument("--secondary", action="store_true",
                    help="not the bench kernel: leave profiles/ncu_summary.json (bench.py's traffic) alone")
    a = ap.parse_args()

    hdr, units, rows = raw(a.rep)
    r = rows[0]
    name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    d = {"kernel": name, "rep": os.path.basename(a.rep)}
    for key, metric in METRICS.items():
        if metric in hdr:
            i = hdr.index(metric)
            v = r[i].replace(",", "")
            try:
                val = float(v) * UNIT_SCALE.get(units[i], 1)
            except ValueError:
                val = v
            d[key] = val
    traffic = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
    alg = 16 * a.cells * a.levels
    d["dram_bytes_per_launch"] = traffic
    d["algorithmic_bytes_per_launch"] = alg
    d["cell_updates_per_launch"] = a.cells * a.levels
    d["dram_bytes_per_cell_update"] = traffic / (a.cells * a.levels)
    if "warp_instructions" in d:
        d["thread_instructions_per_cell_update"] = d["warp_instructions"] * 32 / (a.cells * a.levels)
    if "duration_us" in d:
        d["mcells_per_s_cold"] = a.cells * a.levels / d["duration_us"]

    if a.launches and os.path.exists(a.launches):
        text = open(a.launches).read()
        lines = [l for l in text.splitlines() if l.startswith('"')]
        lrows = list(csv.reader(io.StringIO("\n".join(lines))))
        h = lrows[0]
        ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
        share = {}
        for row in lrows[1:]:
            if row[mi] != "gpu__time_duration.sum":
                continue
            k = row[ki].split("(")[0]
            share.setdefault(k, [0, 0.0])
            share[k][0] += 1
            share[k][1] += float(row[vi].replace(",", ""))
        tot = sum(v[1] for v in share.values()) or 1.0
        d["launch_share"] = {k: {"launches": n, "time_share": round(t / tot, 4)} for k, (n, t) in share.items()}

    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{a.tag}.json"), "w") as f:
        json.dump(d, f, indent=1)
    if not a.secondary:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
            json.dump(d, f, indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
