mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t.log 2>&1; grep -v "^frame" gpurun_out/t.log | grep -E "Error|error|assert|passed|failed|FAILED" | head -10
python tools/blend_ab.py 20 render 2>&1 | tail -2
python tools/blend_ab.py 10 score 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_render.json 2> gpurun_out/bench_render.err; tail -2 gpurun_out/bench_render.err
python -c "import json; d=json.load(open('gpurun_out/bench_render.json')); print(d['value'], d['stages_ms'], d['e2e']['value'])"
timeout 600 python bench.py --workload score --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_score.json 2> gpurun_out/bench_score.err; tail -2 gpurun_out/bench_score.err
python -c "import json; d=json.load(open('gpurun_out/bench_score.json')); print(d['value'], d['e2e']['value'])"
