bash tools/gpu_suite.sh r02c
python tools/bench_next.py > gpurun_out/r02_bench_next.jsonl 2> gpurun_out/r02_bench_next.err; echo next rc=$?
python tools/profile_run.py --workload c5 --reps 2 --n 17179869184 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o gpurun_out/r02_prof_c5 -f python tools/profile_run.py --workload c5 --reps 2 --n 17179869184 > gpurun_out/ncu_c5.log 2>&1; echo ncu rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c5.csv python bench.py --workload c5 --steps 2 --warmup 3 --no-e2e --no-extra > gpurun_out/ncu_launches_c5.log 2>&1; echo launches rc=$?
