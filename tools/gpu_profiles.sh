# round profiles: launch lists (render c1, score c2, batch c4) + ncu --set full of one whole c1 frame
mkdir -p gpurun_out
for k in render score batch; do
  python tools/profile_frame.py $k 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$k.csv python tools/profile_frame.py $k 3 > /dev/null 2>&1; echo launches_$k=$?
done
# the third rendered frame: launches 33..47 of `profile_frame.py render 3` (frame 0 runs twice: pair capacity growth)
ncu --set full --clock-control none --import-source on -s 33 -c 15 -o gpurun_out/prof_frame_c1 python tools/profile_frame.py render 3 > gpurun_out/ncu_frame.log 2>&1; echo full=$?
# one whole configs[2] scoring view (launches 33..47 of `profile_frame.py score 3`)
ncu --set full --clock-control none --import-source on -s 33 -c 15 -o gpurun_out/prof_frame_c2 python tools/profile_frame.py score 3 > gpurun_out/ncu_frame_c2.log 2>&1; echo full_c2=$?
