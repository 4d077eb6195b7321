mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"project" -s 1 -c 1 -o gpurun_out/prof_proj python tools/profile_frame.py score 2 > gpurun_out/ncu7.log 2>&1; echo ncu7=$?
