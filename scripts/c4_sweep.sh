# c4 level-0 PRE/POST launch times vs strip width and forced segment length
for tw in 0 64 96 128; do for sg in 0 511 256 128; do
  if [ "$tw" = 0 ]; then unset MGB_S2TW; else export MGB_S2TW=$tw; fi
  if [ "$sg" = 0 ]; then unset MGB_SEG; else export MGB_SEG=$sg; fi
  timeout 300 python bench.py --steps 3 --warmup 3 --config c4 --no-cpu > gpurun_out/c4s.log 2>&1
  echo "tw=$tw seg=$sg $(tail -1 gpurun_out/c4s.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["launch_ms"], d["roofline"]["post"]["launch_ms"])' 2>&1 | tail -1)"
done; done
