mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"onesweep" -s 5 -c 2 -o gpurun_out/prof_sort python tools/profile_frame.py score 2 > gpurun_out/ncu6.log 2>&1; echo ncu6=$?
