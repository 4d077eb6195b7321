# one GPU call: tests, default bench, scoring bench, launch list + blend/sort ncu captures
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json; tail -2 gpurun_out/bench_default.err
timeout 600 python bench.py --workload score --steps 3 --warmup 1 > gpurun_out/bench_score.json 2> gpurun_out/bench_score.err; cat gpurun_out/bench_score.json
python tools/profile_frame.py render 4 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_render.csv python tools/profile_frame.py render 4 > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
python tools/profile_frame.py score 4 > gpurun_out/plain_s.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_score.csv python tools/profile_frame.py score 4 > gpurun_out/ncu1s.log 2>&1; echo ncu1s=$?
python tools/profile_frame.py render 3 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"blend|onesweep|emit|project" -s 20 -c 10 -o gpurun_out/prof_full python tools/profile_frame.py render 3 > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
