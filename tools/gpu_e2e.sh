mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python tools/e2e_probe.py 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_render.json 2> gpurun_out/bench_render.err; tail -3 gpurun_out/bench_render.err
python -c "import json; d=json.load(open('gpurun_out/bench_render.json')); print(d['value'], d['stages_ms'], d['e2e'])"
