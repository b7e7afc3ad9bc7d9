# tile passes: zero-start stage 1 skipped (default lib) vs computed (experiments/lib_base.so)
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for L in paper_2102_12071_b200/libmgb.so experiments/lib_base.so; do
  echo "== $L"; MGB_LIB_PATH=$PWD/$L timeout 300 python scripts/level_costs.py c2 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
  for cfg in c1 c2; do
    MGB_LIB_PATH=$PWD/$L timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu > gpurun_out/g.log 2>&1
    echo "$L $cfg $(tail -1 gpurun_out/g.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["history_last"])' 2>&1 | tail -1)"
  done
done
done
