# c2 bench with experiment builds of libmgb (MGB_LIB_PATH), one line each: ms/step, PRE ms, POST ms
for L in paper_2102_12071_b200/libmgb.so $EXTRA_LIBS; do
  MGB_LIB_PATH=$PWD/$L timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/var.log 2>&1
  echo "$L $(tail -1 gpurun_out/var.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["launch_ms"], d["roofline"]["post"]["launch_ms"])' 2>&1 | tail -1)"
done
