mkdir -p gpurun_out
for v in base nocount; do
  if [ $v = nocount ]; then RS_NVCC_EXTRA="-DRS_EXP_NOCOUNT" python -m paper_2403_13806_b200.build --force > /dev/null; fi
  for k in render score; do
    python tools/profile_frame.py $k 2 > /dev/null 2>&1; ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:project --log-file gpurun_out/exp_${v}_$k.csv python tools/profile_frame.py $k 2 > /dev/null 2>&1
    python tools/launches.py gpurun_out/exp_${v}_$k.csv 2 | head -2 | sed "s/^/$v $k /"
  done
done
