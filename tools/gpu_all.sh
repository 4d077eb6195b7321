# every bench workload + the reference arm (render), JSON lines into gpurun_out/
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_render.json 2> gpurun_out/bench_render.err; tail -2 gpurun_out/bench_render.err
timeout 900 python bench.py --workload score > gpurun_out/bench_score.json 2> gpurun_out/bench_score.err; tail -2 gpurun_out/bench_score.err
timeout 900 python bench.py --workload house > gpurun_out/bench_house.json 2> gpurun_out/bench_house.err; tail -2 gpurun_out/bench_house.err
timeout 900 python bench.py --workload batch --warmup 3 > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err; tail -2 gpurun_out/bench_batch.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -2 gpurun_out/bench_ref.err
python smoke_print.py 2>/dev/null; for f in render score house batch ref; do python -c "
import json,sys; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', round(d['value'],1), d['unit'], 'e2e', round(d.get('e2e',{}).get('value',0),1), 'cpu', (d.get('cpu_baseline') or {}).get('value'), d.get('stages_ms'), d.get('fps_unfiltered'), d.get('psnr_filtered_vs_full_db'), d.get('kept_at_0.01'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))"; done
