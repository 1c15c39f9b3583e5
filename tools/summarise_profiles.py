"""Summarise a round's ncu captures (gpurun_out/<R>_*.ncu-rep, <R>_launches.csv)
into tracked files under profiles/: per-kernel key metrics (CSV) and the DRAM
traffic per launch that bench.py reports as roofline.traffic."""
import csv
import io
import json
import os
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, v = rows[0], rows[1], rows[2]
    return {a: (b, u) for a, u, b in zip(h, units, v)}


def main():
    traffic = {}
    summary_rows = []
    for k in ("gnn_kernel", "gnn_cluster_kernel", "gnn_flat_u", "spmv_kernel"):
        rep = os.path.join(OUT, f"{R}_{k}.ncu-rep")
        if not os.path.exists(rep):
            continue
        m = raw(rep)
        row = {"kernel": k}
        for key in KEYS:
            if key in m:
                row[key] = m[key][0]
        summary_rows.append(row)
        rd = float(m["dram__bytes_read.sum"][0].replace(",", "")) * (1e6 if m["dram__bytes_read.sum"][1] == "Mbyte" else 1e9 if m["dram__bytes_read.sum"][1] == "Gbyte" else 1e3 if m["dram__bytes_read.sum"][1] == "Kbyte" else 1)
        wr = float(m["dram__bytes_write.sum"][0].replace(",", "")) * (1e6 if m["dram__bytes_write.sum"][1] == "Mbyte" else 1e9 if m["dram__bytes_write.sum"][1] == "Gbyte" else 1e3 if m["dram__bytes_write.sum"][1] == "Kbyte" else 1)
        traffic[k] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                      "duration": m["gpu__time_duration.sum"]}
    keys = ["kernel"] + KEYS
    with open(os.path.join(PROF, f"{R}_kernel_metrics.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=keys)
        w.writeheader()
        for row in summary_rows:
            w.writerow(row)
    with open(os.path.join(PROF, f"{R}_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    # launch list -> compact CSV
    src = os.path.join(OUT, f"{R}_launches.csv")
    if os.path.exists(src):
        rows = list(csv.reader(open(src)))
        hdr = None
        out = []
        for r in rows:
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d.get("Metric Name") == "gpu__time_duration.sum":
                    out.append([d["ID"], d["Kernel Name"].split("(")[0], d["Grid Size"],
                                d["Block Size"], d["Metric Value"], d["Metric Unit"]])
        with open(os.path.join(PROF, f"{R}_launches.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["id", "kernel", "grid", "block", "gpu_time", "unit"])
            w.writerows(out)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
