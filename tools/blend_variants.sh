# blend A/B over compile-time variants: bash tools/blend_variants.sh "-DRS_BLEND_MINB=10" "-DRS_BLEND_UNROLL=2" ...
for v in "$@"; do
  RS_NVCC_EXTRA="$v" python -c "from paper_2403_13806_b200.build import build; build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v: $(python tools/blend_ab.py 20 render fp32 2>&1 | grep 2px) / $(python tools/blend_ab.py 10 score fp32 2>&1 | grep 2px) / $(python tools/blend_ab.py 20 render fp64 2>&1 | grep 2px) / $(python tools/blend_ab.py 10 score fp64 2>&1 | grep 2px)"
done
python -c "from paper_2403_13806_b200.build import build; build(force=True)" > /dev/null 2>&1
