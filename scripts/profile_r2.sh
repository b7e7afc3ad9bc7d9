# Round-2 profile artefacts for the c2 step: per-level cycle costs, launch list, and ncu
# --set full captures of the level-0 warp-strip passes and the level-1/2 column-pair passes.
python scripts/level_costs.py c2 > gpurun_out/level_costs_c2.log 2>&1; echo level_costs=$?
python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_stream3 -s 4 -c 2 \
    -o gpurun_out/full_c2_s3 python scripts/profile_step.py > gpurun_out/ncu_full_s3.log 2>&1; echo ncu_full_s3=$?
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_stream2 -s 8 -c 4 \
    -o gpurun_out/full_c2_s2 python scripts/profile_step.py > gpurun_out/ncu_full_s2.log 2>&1; echo ncu_full_s2=$?
cat gpurun_out/level_costs_c2.log
