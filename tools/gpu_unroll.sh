for u in 2 3 4; do
  RS_NVCC_EXTRA="-DRS_BLEND_UNROLL=$u" python -m paper_2403_13806_b200.build > /dev/null 2>&1
  echo "U=$u"; python tools/blend_ab.py 20 render 2>&1 | grep 2px; python tools/blend_ab.py 10 score 2>&1 | grep 2px
done
python -m paper_2403_13806_b200.build > /dev/null 2>&1
