# Round-2 full check + profile artefacts: smoke, GPU suite, every config's bench line, the
# reference arm, the c2 launch list and ncu captures (each only after the plain run).
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
  tail -1 gpurun_out/bench_$c.log | cut -c1-300
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python scripts/level_costs.py c2 > gpurun_out/level_costs_c2.log 2>&1; cat gpurun_out/level_costs_c2.log
python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_stream3 -s 4 -c 2 \
    -o gpurun_out/full_c2_s3 python scripts/profile_step.py > gpurun_out/ncu_full_s3.log 2>&1; echo ncu_full_s3=$?
