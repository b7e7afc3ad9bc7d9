# Round profile artefacts for the c2 step: launch list (cold-cache, serialised) and one
# ncu --set full capture of the level-0 PRE + POST streaming passes.  Run only after the
# same command has exited 0 without ncu.
python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
# one cycle = launches 0..: capture the first level-0 PRE (norm) of cycle 2 and the level-0 POST
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_stream2 -s 4 -c 4 \
    -o gpurun_out/full_c2 python scripts/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
