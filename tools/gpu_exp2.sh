mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in new old; do
  if [ $v = old ]; then RS_NVCC_EXTRA="-DRS_EMIT_PAIRBAL" python -m paper_2403_13806_b200.build > /dev/null; fi
  for k in render score batch; do
    python tools/profile_frame.py $k 2 > /dev/null 2>&1; ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:emit --log-file gpurun_out/exp_${v}_$k.csv python tools/profile_frame.py $k 2 > /dev/null 2>&1
    python tools/launches.py gpurun_out/exp_${v}_$k.csv 2 | head -2 | sed "s/^/$v $k /"
  done
done
python -m paper_2403_13806_b200.build > /dev/null
