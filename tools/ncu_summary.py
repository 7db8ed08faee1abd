"""Summarise an `ncu --set full` capture (`ncu -i X.ncu-rep --page raw --csv`)
as a markdown table: per kernel launch the duration, DRAM bytes, DRAM
throughput % of peak, tensor-pipe utilisation, achieved occupancy, issue
activity and the top warp-stall reasons.

  python tools/ncu_summary.py gpurun_out/prof_raw.csv [--labels QKV,attn,O,...] > profiles/r2/ncu_full.md
"""
import argparse
import csv

COLS = [
    ("dur_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("dram_%pk", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("tc_inst_%", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active"),
    ("warps_%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue_%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--labels", default="")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    labels = args.labels.split(",") if args.labels else []
    idx = {h: i for i, h in enumerate(hdr)}
    stall_cols = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), i) for h, i in idx.items()
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    print("| # | kernel | " + " | ".join(c for c, _ in COLS) + " | top stalls (share of samples) |")
    print("|---|---|" + "---|" * len(COLS) + "---|")
    for n, d in enumerate(data):
        name = d[idx["Kernel Name"]]
        short = name.split("(")[0].split("::")[-1].split("<")[0]
        if n < len(labels):
            short = f"{short} ({labels[n]})"
        vals = []
        for _, key in COLS:
            if key not in idx or d[idx[key]] == "":
                vals.append("-")
                continue
            v = float(d[idx[key]].replace(",", ""))
            u = units[idx[key]]
            if key.startswith("dram__bytes"):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
            if key == "gpu__time_duration.sum":
                v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)
            vals.append(f"{v:.1f}" if abs(v) < 1e4 else f"{v:.0f}")
        st = [(h, float(d[i] or 0)) for h, i in stall_cols]
        tot = sum(v for _, v in st) or 1.0
        top = ", ".join(f"{h} {100 * v / tot:.0f}%" for h, v in sorted(st, key=lambda x: -x[1])[:3])
        print(f"| {n} | {short} | " + " | ".join(vals) + f" | {top} |")


if __name__ == "__main__":
    main()
