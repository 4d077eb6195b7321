# one GPU call: tests, then every bench workload (render, score, house, batch)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_render.json 2> gpurun_out/bench_render.err; cut -c1-600 gpurun_out/bench_render.json; tail -3 gpurun_out/bench_render.err
timeout 600 python bench.py --workload score --steps 3 --warmup 1 > gpurun_out/bench_score.json 2> gpurun_out/bench_score.err; cut -c1-300 gpurun_out/bench_score.json; tail -3 gpurun_out/bench_score.err
timeout 900 python bench.py --workload house --steps 100 > gpurun_out/bench_house.json 2> gpurun_out/bench_house.err; cut -c1-300 gpurun_out/bench_house.json; tail -3 gpurun_out/bench_house.err
timeout 900 python bench.py --workload batch --steps 1 --warmup 3 > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err; cut -c1-300 gpurun_out/bench_batch.json; tail -3 gpurun_out/bench_batch.err
