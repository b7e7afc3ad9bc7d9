set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_stream -s 6 -c 6 \
    -o gpurun_out/sweep python scripts/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench.log; tail -3 gpurun_out/smoke.log
