mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"emit" -s 1 -c 1 -o gpurun_out/prof_emitw python tools/profile_frame.py render 2 > gpurun_out/ncu5.log 2>&1; echo ncu5=$?
