#!/bin/bash
# compute-sanitizer on the dataflow CTA path (config A: 5 subdomains of ~1000 nodes).
mkdir -p gpurun_out
O=gpurun_out/c24_sanitizers.txt; : > $O
echo "## racecheck: pytest tests/test_gpu_parity.py -k config_a (dataflow layer schedule)" >> $O
timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -k config_a -x -q 2>&1 | grep -v Warning | tail -6 >> $O
echo "## memcheck: pytest tests/test_gpu_parity.py -k 'apply or pcg'" >> $O
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -k 'apply or pcg' -x -q 2>&1 | tail -4 >> $O
echo "## synccheck: pytest tests/test_gpu_parity.py -k config_a" >> $O
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -k config_a -x -q 2>&1 | tail -4 >> $O
cat $O
