# ncu --set full on emit/project/blend (second frame)
mkdir -p gpurun_out
python tools/profile_frame.py render 3 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"emit|project|blend" -s 3 -c 3 -o gpurun_out/prof_full python tools/profile_frame.py render 3 > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
ls -la gpurun_out/
