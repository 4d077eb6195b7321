mkdir -p gpurun_out
python tools/profile_frame.py score 3 > gpurun_out/plain_s.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_score.csv python tools/profile_frame.py score 3 > gpurun_out/ncu1s.log 2>&1; echo ncu1s=$?
