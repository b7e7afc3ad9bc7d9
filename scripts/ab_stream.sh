# A/B: one-column (MGB_STREAM1=1) vs two-column streaming kernel on configs c2 (+ level costs)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for v in 1 0; do
  MGB_STREAM1=$v timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_s$v.log 2>&1; echo "stream1=$v rc=$?"
  tail -1 gpurun_out/bench_s$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["launch_ms"], d["roofline"]["frac"], d["roofline"]["post"]["launch_ms"], d["e2e"]["value"])'
  MGB_STREAM1=$v timeout 300 python scripts/level_costs.py c2 2>&1 | head -3
done
