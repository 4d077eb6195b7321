#!/bin/bash
# Per-round ncu evidence (run on the GPU box from the repo root; outputs under gpurun_out/prof):
#   launch lists (gpu__time_duration, serialised, cold) of the bench's default render run and of
#   score / batch frames, and one `ncu --set full` capture of a configs[1] frame (fp32 and fp64)
#   and a configs[2] scoring view, summarised per kernel by tools/ncu_summary.py.
set -u
R=${1:-round2}
O=gpurun_out/prof
P=/tmp/prof_reps  # the reports themselves stay off gpurun_out (too large to bring back)
mkdir -p $O $P
python bench.py --quick --no-cpu-baseline --steps 3 --warmup 3 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/${R}_launches_render_configs1.csv \
    python bench.py --quick --no-cpu-baseline --steps 3 --warmup 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/${R}_launches_render_configs1_fp64.csv \
    python bench.py --quick --no-cpu-baseline --steps 3 --warmup 3 --precision fp64 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/${R}_launches_score_configs2.csv \
    python tools/profile_frame.py score 2 fp32 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/${R}_launches_batch_configs4.csv \
    python tools/profile_frame.py batch 2 fp32 > /dev/null 2>&1
for p in fp32 fp64; do   # two frames: the second one is the warm-workspace frame
  ncu --set full --import-source on --clock-control none -c 40 \
      -o $P/${R}_full_configs1_$p python tools/profile_frame.py render 2 $p > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -c 40 \
    -o $P/${R}_full_configs2_fp32 python tools/profile_frame.py score 2 fp32 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -c 40 \
    -o $P/${R}_full_configs4_fp32 python tools/profile_frame.py batch 2 fp32 > /dev/null 2>&1
# summaries on the box (the reports themselves are too large to bring back)
for f in $P/${R}_full_*.ncu-rep; do
  b=$O/$(basename ${f%.ncu-rep})
  python tools/ncu_summary.py $f $b > $b.txt 2>&1
  python tools/ncu_src.py $f "blend" 1 40 > ${b}_blend_src.txt 2>&1  # skip the first (overflowed) frame's blend
done
python tools/ncu_src.py $P/${R}_full_configs1_fp32.ncu-rep "dsort" 0 30 > $O/${R}_full_configs1_fp32_dsort_src.txt 2>&1
rm -rf $P
ls -la $O
