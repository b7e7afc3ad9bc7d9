# c3 profile artefacts: launch list of one step and an ncu --set full capture of the
# level-0 per-point-plane PRE / POST passes (k_stream).  Run after the plain command exits 0.
timeout 600 python scripts/profile_step.py c3 > gpurun_out/prof_plain_c3.log 2>&1 || { echo plain_failed; exit 1; }
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3.csv python scripts/profile_step.py c3 > gpurun_out/ncu_launch_c3.log 2>&1; echo ncu_launch=$?
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k k_stream -s 0 -c 2 \
    -o gpurun_out/full_c3 python scripts/profile_step.py c3 > gpurun_out/ncu_full_c3.log 2>&1; echo ncu_full=$?
python scripts/ncu_summary.py gpurun_out/full_c3.ncu-rep > gpurun_out/ncu_full_c3.txt 2>&1
ncu -i gpurun_out/full_c3.ncu-rep --page raw --csv > gpurun_out/full_c3_raw.csv 2>&1
python scripts/launches.py gpurun_out/launches_c3.csv > gpurun_out/launches_c3_summary.txt 2>&1
head -30 gpurun_out/ncu_full_c3.txt
