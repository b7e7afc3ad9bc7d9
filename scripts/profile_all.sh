# Round profile artefacts: launch lists (cold-cache, serialised) for c2/c3/c4 steps and ncu --set full
# captures of the level-0 streaming passes.  Each config runs once without ncu first.
for c in c2 c3 c4; do
  python scripts/profile_step.py $c > gpurun_out/prof_plain_$c.log 2>&1 || { echo plain_$c failed; continue; }
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$c.csv python scripts/profile_step.py $c > gpurun_out/ncu_launch_$c.log 2>&1; echo launch_$c=$?
done
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_stream2 -s 4 -c 4 \
    -o gpurun_out/full_c2 python scripts/profile_step.py c2 > gpurun_out/ncu_full_c2.log 2>&1; echo full_c2=$?
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_stream -s 0 -c 4 \
    -o gpurun_out/full_c3 python scripts/profile_step.py c3 > gpurun_out/ncu_full_c3.log 2>&1; echo full_c3=$?
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_stream2 -s 0 -c 2 \
    -o gpurun_out/full_c4 python scripts/profile_step.py c4 > gpurun_out/ncu_full_c4.log 2>&1; echo full_c4=$?
