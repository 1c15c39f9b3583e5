mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c1_smi.txt
lscpu > gpurun_out/c1_lscpu.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/c1_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
tail -30 gpurun_out/c1_pytest.log
tail -3 gpurun_out/c1_smoke.log
