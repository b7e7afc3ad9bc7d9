# c2 bench PRE/POST L0 launch times vs forced segment length (MGB_SEG) for the current build
for sg in ${SEGS:-0}; do
  if [ "$sg" = 0 ]; then unset MGB_SEG; else export MGB_SEG=$sg; fi
  timeout 300 python bench.py --steps 3 --warmup 3 > gpurun_out/seg.log 2>&1
  echo "seg=$sg $(tail -1 gpurun_out/seg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["launch_ms"], d["roofline"]["post"]["launch_ms"])' 2>&1 | tail -1)"
done
