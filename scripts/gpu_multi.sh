#!/bin/bash
# Multi-GPU checks: parity vs the oracle's R-rank emulation, then a weak-scaling bench.
# usage: bash scripts/gpu_multi.sh <ngpu> [particles_per_gpu]
N=${1:-2}
NP=${2:-1e8}
nvidia-smi --query-gpu=index,name,memory.used --format=csv
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1; echo "pytest multi rc=$?"
tail -30 gpurun_out/pytest_multi_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600 \
  bench.py --gpus $N --steps 5 --warmup 3 --particles $NP --no-cpu-baseline > gpurun_out/bench_multi_$N.log 2>&1; echo "bench multi rc=$?"
tail -3 gpurun_out/bench_multi_$N.log
