#!/bin/bash
# round-2 cycle 5: GPU tests, measured FP32 FFMA2 peak (with its clock record), bench.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=5 > gpurun_out/c5_pytest.log 2>&1
tail -6 gpurun_out/c5_pytest.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 100 > gpurun_out/c5_fp32_clocks.csv &
SMI=$!
sleep 0.5
./tools/ubench/fp32_peak > gpurun_out/c5_fp32_peak.json
kill $SMI
python - <<'PY'
import json, statistics
rec = json.loads(open("gpurun_out/c5_fp32_peak.json").read())
mhz = [float(l.split(",")[0].split()[0]) for l in open("gpurun_out/c5_fp32_clocks.csv") if l.strip()]
load = [m for m in mhz if m > 500]
rec.update(sm_mhz_median=statistics.median(load) if load else None, sm_mhz_samples=len(mhz),
           clock_lines=open("gpurun_out/c5_fp32_clocks.csv").read().splitlines()[:40])
json.dump(rec, open("gpurun_out/r02_fp32_peak.json", "w"), indent=1)
print(rec["fp32_ffma2_tflops"], rec["sm_mhz_median"])
PY
timeout 1200 python bench.py > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; tail -c 400 gpurun_out/c5_bench.json
