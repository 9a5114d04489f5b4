#!/bin/bash
# One GPU-box pass: the -m gpu suite, the default bench line, and a 2-rank (gloo, one GPU)
# bench of the multi-rank logic.  Outputs under gpurun_out/ with the tag $1 (e.g. r02).
tag=${1:-r02}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/${tag}_pytest_gpu.log
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/${tag}_bench.err
SQ_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e \
  > gpurun_out/${tag}_bench_2rank_gloo.json 2> gpurun_out/${tag}_bench_2rank.err; echo "2rank rc=$?"
tail -3 gpurun_out/${tag}_bench_2rank.err
