#!/bin/bash
# round-2 cycle 7: the reference arm as the driver runs it, a default bench line,
# and the BASELINE config E sweep on 1M-node meshes.
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference > gpurun_out/c7_reference.json 2> gpurun_out/c7_reference.err
tail -c 1200 gpurun_out/c7_reference.json; tail -2 gpurun_out/c7_reference.err
timeout 1200 python bench.py > gpurun_out/c7_bench.json 2> gpurun_out/c7_bench.err; tail -c 300 gpurun_out/c7_bench.json
timeout 2400 python tools/sweep.py --min-nodes 1000000 > gpurun_out/r02_sweep_configE.jsonl 2> gpurun_out/c7_sweep.err
wc -l gpurun_out/r02_sweep_configE.jsonl; tail -2 gpurun_out/c7_sweep.err
