#!/bin/bash
# One GPU verification cycle (run under gpurun): parity tests, bench, optional ncu.
# usage: tools/gpu_cycle.sh TAG [ncu]
TAG=${1:-run}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/${TAG}_pytest.log
python bench.py --steps 10 --warmup 3 --no-pcg --cpu-seconds 2 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
if [ "$2" == "ncu" ]; then
  ncu --set full --clock-control none --import-source on -k regex:gnn_kernel -s 2 -c 1 \
      -o gpurun_out/${TAG}_gnn python tools/profile_apply.py > gpurun_out/${TAG}_ncu.log 2>&1
fi
cat gpurun_out/${TAG}_pytest.log
python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench.json'));print('ms',d['ms_per_step'],'gnn_ms',d['roofline']['gnn_ms'],'frac',d['roofline']['frac'],'spmv',d['roofline_spmv']['ms'])"
