# quick A/B of streaming kernels: bench c2 PRE/POST launch times (+ optional ncu of k_stream2)
for v in ${VARIANTS:-0}; do
  MGB_STREAM1=$v timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_s$v.log 2>&1; echo "stream1=$v rc=$?"
  tail -1 gpurun_out/bench_s$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["launch_ms"], d["roofline"]["frac"], d["roofline"]["post"]["launch_ms"], d["e2e"]["value"])'
done
if [ -n "$NCU" ]; then bash scripts/ncu_stream2.sh; fi
