# Full GPU check: smoke, GPU parity suite, the default bench line and every config's bench line.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log; tail -2 gpurun_out/smoke.log
for c in c1 c3 c4 c5; do tail -1 gpurun_out/bench_$c.log | cut -c1-400; done
tail -1 gpurun_out/bench_ref.log | cut -c1-300
