# A/B programmatic dependent launch: bench c2 and c1 with and without (MGB_NO_PDL=1)
for v in 1 0; do
  for cfg in c2 c1; do
    MGB_NO_PDL=$v timeout 300 python bench.py --steps 5 --warmup 3 --config $cfg > gpurun_out/pdl.log 2>&1
    echo "no_pdl=$v $cfg $(tail -1 gpurun_out/pdl.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"])' 2>&1 | tail -1)"
  done
done
