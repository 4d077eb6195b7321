mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for k in render score batch; do
  python tools/profile_frame.py $k 2 > /dev/null 2>&1; ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$k.csv python tools/profile_frame.py $k 2 > /dev/null 2>&1
  python tools/launches.py gpurun_out/launches_$k.csv 13 | sed "s/^/$k /"
done
