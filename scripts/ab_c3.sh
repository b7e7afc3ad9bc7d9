# A/B of per-point-plane streaming variants (experiment builds in experiments/) on config 3
for v in ${VARIANTS:-main pf0evh0 pf1evh0 pf0evh1}; do
  if [ "$v" = main ]; then unset MGB_LIB_PATH; else export MGB_LIB_PATH=$PWD/experiments/lib_$v.so; fi
  timeout 600 python bench.py --config ${CFG:-c3} --steps 3 --warmup 3 > gpurun_out/ab_$v.log 2>&1; echo "$v rc=$?"
  tail -1 gpurun_out/ab_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["launch_ms"], d["roofline"]["frac"], d["roofline"]["post"]["launch_ms"], d["roofline"]["post"]["frac"])'
done
