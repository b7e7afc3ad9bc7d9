set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "tile or cycles_match or fused or storage or classed or virtual or nccl or random" > gpurun_out/pytest_tile.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_tile.log
MGB_TILE=1 timeout 300 python scripts/level_costs.py c2 > gpurun_out/lc_tile.log 2>&1
cat gpurun_out/lc_tile.log
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-300
