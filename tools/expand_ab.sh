# expand A/B: bash tools/expand_ab.sh D,T,W ...  (RS_EXPAND_DENSE=D: ballot walk for chunks averaging
# >= D tiles per segment; RS_EXPAND_MAJOR=T: column-major switch of the transposed walk;
# RS_EXPAND_WAVES=W: resident-CTA waves of the sparse grid)
mkdir -p gpurun_out
[ -n "$NOTEST" ] || timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
for cfg in "$@"; do
 IFS=, read d t w <<< "$cfg"
 for k in render score batch; do
  RS_EXPAND_DENSE=$d RS_EXPAND_MAJOR=$t RS_EXPAND_WAVES=$w ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$k.csv python tools/profile_frame.py $k 2 > /dev/null 2>&1
  echo "d=$d t=$t w=$w $k $(python tools/launches.py gpurun_out/l_$k.csv 15 | grep -E 'chunk_count|expand|total' | awk '{print $1}' | tr '\n' ' ')"
 done
done
