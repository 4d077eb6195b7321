mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"emit|project" -s 2 -c 2 -o gpurun_out/prof_score python tools/profile_frame.py score 2 > gpurun_out/ncu4.log 2>&1; echo ncu4=$?
