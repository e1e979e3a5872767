#!/bin/bash
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --particles 1e8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench_small.log
