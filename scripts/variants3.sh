# c2 bench with experiment builds (experiments/libmgb_<name>.so): ms/step, level-0 PRE us, POST us;
# with a second argument list after "--", per-level pass times through ab_k3.py instead
for v in "$@"; do
  MGB_LIB_PATH=$PWD/experiments/libmgb_$v.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/var_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/var_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["launch_ms"]*1e3,1), round(d["roofline"]["post"]["launch_ms"]*1e3,1))' 2>&1 | tail -1)"
  MGB_LIB_PATH=$PWD/experiments/libmgb_$v.so timeout 300 python scripts/ab_k3.py c2 0 2>&1 | tail -1
done
