mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_render.json 2> gpurun_out/bench_render.err; tail -3 gpurun_out/bench_render.err
python -c "import json; d=json.load(open('gpurun_out/bench_render.json')); print(d['value'], d['stages_ms'], d['e2e']['value'])"
timeout 600 python bench.py --workload score --steps 3 --warmup 1 > gpurun_out/bench_score.json 2> gpurun_out/bench_score.err; tail -3 gpurun_out/bench_score.err
python -c "import json; d=json.load(open('gpurun_out/bench_score.json')); print(d['value'], d['e2e']['value'], d['kept_at_0.01'])"
python tools/profile_frame.py render 4 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_render.csv python tools/profile_frame.py render 4 > gpurun_out/ncu1.log 2>&1; echo ncu=$?
python tools/profile_frame.py score 3 > gpurun_out/plain_s.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_score.csv python tools/profile_frame.py score 3 > gpurun_out/ncu1s.log 2>&1; echo ncu1s=$?
