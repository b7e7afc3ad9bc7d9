nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 300 python scripts/level_costs.py c2 > gpurun_out/levels_c2.log 2>&1; echo lv=$?
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log; cat gpurun_out/levels_c2.log
