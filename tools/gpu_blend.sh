mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_visibility.py -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python tools/blend_ab.py 20 render 2>&1 | tail -3
python tools/blend_ab.py 10 score 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_render.json 2> gpurun_out/bench_render.err; tail -3 gpurun_out/bench_render.err
python -c "import json; d=json.load(open('gpurun_out/bench_render.json')); print(d['value'], d['stages_ms'], d['e2e']['value'])"
ncu --set full --clock-control none --import-source on -k regex:"blend" -s 1 -c 1 -o gpurun_out/prof_blend python tools/profile_frame.py render 2 > gpurun_out/ncu3.log 2>&1; echo ncu3=$?
