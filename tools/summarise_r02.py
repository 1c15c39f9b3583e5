"""Round-2 profile summaries (tracked under profiles/) from the scratch captures in
gpurun_out/: per-kernel launch tables of the PCG iteration at config C and the key
metrics + SASS stall/instruction breakdown of one `ncu --set full` capture of the
GNN kernel."""
import collections
import csv
import io
import json
import os
import statistics as st
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

ALG = {  # algorithmic bytes per launch at config C
    "spmv_kernel": 12 * 6968908 + 20 * 996546,
    "update_kernel": 48 * 996546,
    "pupdate_kernel": 24 * 996546,
    "coarse_gemv_kernel": 8 * 997 * 997 + 16 * 997,
    "prolong_kernel": 36 * 996546 + 16 * 1443638,
}


def launches(csv_name, out_name):
    rows = list(csv.reader(open(os.path.join(OUT, csv_name))))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ci = {n: i for i, n in enumerate(h)}
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        k = r[ci["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "")
        k = k.replace("ddmgnn::", "")
        agg[k][r[ci["Metric Name"]]].append(float(r[ci["Metric Value"]].replace(",", "")))
    with open(os.path.join(PROF, out_name), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "launches", "median_us", "dram_read_MB", "dram_write_MB",
                    "dram_GBps", "algorithmic_MB", "algorithmic_GBps"])
        for k, m in agg.items():
            if "gpu__time_duration.sum" not in m or not any(
                    x in k for x in ("gnn", "spmv", "update", "prolong", "gemv", "glue", "init")):
                continue
            t = st.median(m["gpu__time_duration.sum"])
            rd = st.median(m.get("dram__bytes_read.sum", [0]))
            wr = st.median(m.get("dram__bytes_write.sum", [0]))
            alg = ALG.get(k)
            w.writerow([k, len(m["gpu__time_duration.sum"]), round(t / 1e3, 2), round(rd / 1e6, 2),
                        round(wr / 1e6, 2), round((rd + wr) / t, 0),
                        round(alg / 1e6, 2) if alg else "", round(alg / t, 0) if alg else ""])


def gnn_capture(rep_name, out_name):
    rep = os.path.join(OUT, rep_name)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    raw = dict(zip(rows[0], rows[2]))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__block_size",
            "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    out = {k: raw.get(k) for k in keys}
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    ci = {n: i for i, n in enumerate(h)}
    data = [r for r in rows[2:] if len(r) == len(h)]
    ops = collections.Counter()
    for r in data:
        src = r[ci["Source"]].split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") else src[0]
        ops[op.split(".")[0]] += int(r[ci["Instructions Executed"]] or 0)
    tot = sum(ops.values())
    out["instruction_mix_pct"] = {k: round(100 * v / tot, 1) for k, v in ops.most_common(12)}
    samp = "Warp Stall Sampling (All Samples)"
    total = sum(int(r[ci[samp]] or 0) for r in data)
    stalls = {}
    for c in h:
        if c.startswith("stall_") and "(Not" not in c:
            v = sum(int(r[ci[c]] or 0) for r in data)
            if v:
                stalls[c[6:]] = round(100 * v / total, 1)
    out["stall_samples_pct"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
    out["stall_samples"] = total
    with open(os.path.join(PROF, out_name), "w") as fh:
        json.dump(out, fh, indent=1)
    return out


if __name__ == "__main__":
    if sys.argv[1:] == ["final"]:  # end of round 2: the dataflow kernel (tools/cycle26.sh)
        launches("r02f_pcg_launches.csv", "r02_pcg_iteration_launches_final.csv")
        launches("r02f_bench_launches.csv", "r02_bench_launches_final.csv")
        gnn_capture("r02_gnn_shift.ncu-rep", "r02_gnn_kernel_metrics_shift_barriers.json")
        print(json.dumps(gnn_capture("r02f_gnn.ncu-rep", "r02_gnn_kernel_metrics_dataflow.json"),
                         indent=1))
        sys.exit(0)
    launches("r02_pcg_launches_c3.csv", "r02_pcg_iteration_launches.csv")
    launches("r02_pcg_launches_fused.csv", "r02_pcg_iteration_launches_fused_tail.csv")
    launches("r02_pcg_launches.csv", "r02_pcg_iteration_launches_start.csv")
    print(json.dumps(gnn_capture("r02_gnn_h0.ncu-rep", "r02_gnn_kernel_metrics.json"), indent=1))
    gnn_capture("r02_gnn.ncu-rep", "r02_gnn_kernel_metrics_round_start.json")
