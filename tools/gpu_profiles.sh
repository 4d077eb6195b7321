# round profiles: launch lists (render c1, score c2, batch c4) + ncu --set full of one c1 frame, all kernels
mkdir -p gpurun_out
for k in render score batch; do
  python tools/profile_frame.py $k 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$k.csv python tools/profile_frame.py $k 3 > /dev/null 2>&1; echo launches_$k=$?
done
ncu --set full --clock-control none --import-source on -k regex:"rs::|onesweep|blend|emit|project|count|ranges|radix" -s 26 -c 13 -o gpurun_out/prof_frame_c1 python tools/profile_frame.py render 3 > gpurun_out/ncu_frame.log 2>&1; echo full=$?
