mkdir -p gpurun_out
python tools/profile_train.py 2 > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
ncu --set full --clock-control none --import-source on -k regex:"backward_blend|chain" -s 2 -c 2 -o gpurun_out/prof_bw python tools/profile_train.py 2 > gpurun_out/ncu8.log 2>&1; echo ncu8=$?
