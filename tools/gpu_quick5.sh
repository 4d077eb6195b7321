# tests + render / score / batch bench values (no CPU baseline), expand variants via env
mkdir -p gpurun_out
[ -n "$NOTEST" ] || { timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t.log 2>&1; grep -v "^frame" gpurun_out/t.log | grep -E "Error|error|assert|passed|failed|FAILED" | head -10; }
for w in render score batch; do
  case $w in render) a="--steps 200";; score) a="--steps 3 --warmup 3";; batch) a="--steps 3 --warmup 3";; esac
  timeout 600 python bench.py --workload $w $a --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err || tail -3 gpurun_out/bench_$w.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d.get('stages_ms'), d['e2e']['value'])"
done
