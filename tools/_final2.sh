mkdir -p gpurun_out/final
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q > gpurun_out/final/tests_bwd.log 2>&1
timeout 2700 bash tools/round_profiles.sh round2 > gpurun_out/final/profiles.log 2>&1
du -sh gpurun_out
