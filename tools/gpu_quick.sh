mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/bench_render.json 2> gpurun_out/bench_render.err
python -c "import json; d=json.load(open('gpurun_out/bench_render.json')); print(d['value'], d['stages_ms'], d['e2e']['value'], d['roofline']['frac'])"; tail -3 gpurun_out/bench_render.err
python tools/profile_frame.py render 4 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_render.csv python tools/profile_frame.py render 4 > gpurun_out/ncu1.log 2>&1; echo ncu=$?
