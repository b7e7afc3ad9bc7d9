# ncu --set full of the level-0 PRE and POST streaming passes (one cycle of a config-2 step)
K=${K:-k_stream2}
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$K -s 0 -c 2 \
    -o gpurun_out/s2 python scripts/profile_step.py > gpurun_out/ncu_s2.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_s2.log
