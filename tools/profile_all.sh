#!/bin/bash
# Runs on the GPU box (under gpurun): plain runs first, then ncu captures into gpurun_out/.
#   1. launch list of the bench command (gpu__time_duration per launch)
#   2. --set full on each hot kernel (c2 u32 fill, c3 u64 fill, c4 f32 fill, c5 fused)
set -u
OUT=gpurun_out
TAG=${1:-r02}
python bench.py --steps 5 --warmup 3 --no-e2e --no-extra > $OUT/plain_bench.log 2>&1 || { echo "plain bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-extra > $OUT/ncu_launches.log 2>&1
for w in c2 c3 c4; do
  python tools/profile_run.py --workload $w --reps 2 > $OUT/plain_$w.log 2>&1 || { echo "plain $w failed"; exit 1; }
  ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 1 -c 1 \
      -o $OUT/${TAG}_prof_$w python tools/profile_run.py --workload $w --reps 2 > $OUT/ncu_$w.log 2>&1
done
python tools/profile_run.py --workload c5 --reps 2 --n 17179869184 > $OUT/plain_c5.log 2>&1 || { echo "plain c5 failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches_c5.csv \
    python bench.py --workload c5 --steps 2 --warmup 3 --no-e2e --no-extra > $OUT/ncu_launches_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 \
    -o $OUT/${TAG}_prof_c5 python tools/profile_run.py --workload c5 --reps 2 --n 17179869184 > $OUT/ncu_c5.log 2>&1
echo done
