# tile side rule: one CTA per SM (default lib) vs two (experiments/lib_base.so); per-level costs and bench c1/c2/c4
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
for L in paper_2102_12071_b200/libmgb.so experiments/lib_base.so; do
  for cfg in c2 c4; do
    echo "== $L $cfg"; MGB_LIB_PATH=$PWD/$L timeout 300 python scripts/level_costs.py $cfg 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
  done
done
for rep in 1 2; do
for L in paper_2102_12071_b200/libmgb.so experiments/lib_base.so; do
  for cfg in c1 c2 c4; do
    MGB_LIB_PATH=$PWD/$L timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu > gpurun_out/g.log 2>&1
    echo "$L $cfg $(tail -1 gpurun_out/g.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["history_last"])' 2>&1 | tail -1)"
  done
done
done
