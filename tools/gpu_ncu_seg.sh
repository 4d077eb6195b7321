mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"segemit|segcount|expand|project" -s 4 -c 4 -o gpurun_out/prof_seg python tools/profile_frame.py score 2 > gpurun_out/ncu9.log 2>&1; echo ncu9=$?
