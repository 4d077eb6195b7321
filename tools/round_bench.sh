# Every bench line of the round (render with its fp64 / score / fps_vs_n blocks, score, batch,
# train, house, the reference arm) plus the parity tests, into gpurun_out/final/.
mkdir -p gpurun_out/final
timeout 600 python -m pytest tests/test_gpu_backward.py tests/test_gpu_parity.py -x -q > gpurun_out/final/tests.log 2>&1
timeout 500 python bench.py > gpurun_out/final/render.json 2> gpurun_out/final/render.err
for w in score batch train house; do
  timeout 900 python bench.py --workload $w > gpurun_out/final/$w.json 2> gpurun_out/final/$w.err
done
timeout 400 python bench.py --impl reference > gpurun_out/final/reference.json 2> gpurun_out/final/reference.err
du -sh gpurun_out
