# A/B of compile-time variants on the launch lists: bash tools/kernel_variants.sh REGEX "-D..." ...
re=$1; shift
for v in "$@"; do
  RS_NVCC_EXTRA="$v" python -c "from paper_2403_13806_b200.build import build; build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for k in render score; do
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kv_$k.csv python tools/profile_frame.py $k 2 > /dev/null 2>&1
    echo "== $v $k: $(python tools/launches.py gpurun_out/kv_$k.csv 15 | grep -E "$re|total" | awk '{print $1}' | tr '\n' ' ')"
  done
done
python -c "from paper_2403_13806_b200.build import build; build(force=True)" > /dev/null 2>&1
