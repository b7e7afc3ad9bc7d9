# one build->measure iteration: gpu tests, c2 bench summary, level costs, optional ncu of k_stream2
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for cfg in ${CFGS:-c2}; do
  timeout 300 python bench.py --steps 5 --warmup 3 --config $cfg > gpurun_out/bench_$cfg.log 2>&1; echo "bench $cfg rc=$?"
  tail -1 gpurun_out/bench_$cfg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["launch_ms"], d["roofline"]["frac"], d["roofline"]["post"]["launch_ms"], d["e2e"]["value"])'
done
timeout 300 python scripts/level_costs.py c2 2>&1 | head -4
if [ -n "$NCU" ]; then bash scripts/ncu_stream2.sh; fi
