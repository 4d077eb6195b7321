# Per compile-time variant: configs[1] fp32 frames/s + sort / blend stage us (bench --quick) and
# configs[2] scoring views/s (--workload score, 3 passes):
#   bash tools/variant_bench.sh "-DFOO=1" "-DFOO=2" ...   ("" = the default build)
for v in "$@"; do
  RS_NVCC_EXTRA="$v" python -c "from paper_2403_13806_b200.build import build; build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  r=$(timeout 300 python bench.py --quick --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), 'pre', round(d['stages_ms']['preprocess']*1e3,1), 'sort', round(d['stages_ms']['sort']*1e3,1), 'blend', round(d['stages_ms']['blend']*1e3,1))")
  s=$(timeout 300 python bench.py --workload score --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'pre', round(d['stages_ms_per_view']['preprocess']*1e3,1), 'sort', round(d['stages_ms_per_view']['sort']*1e3,1))")
  b=""
  if [ -n "$VB_BATCH" ]; then
    b=$(timeout 400 python bench.py --workload batch --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")
  fi
  echo "== [$v] render fps: $r | score views/s: $s | batch fps: $b"
done
python -c "from paper_2403_13806_b200.build import build; build(force=True)" > /dev/null 2>&1
