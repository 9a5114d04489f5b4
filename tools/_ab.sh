python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo rc=$?
sleep 20
python bench.py --no-e2e > gpurun_out/r02_bench_rep2.json 2>/dev/null; echo rc=$?
