#!/bin/bash
# One GPU session: build check, smoke, GPU tests, short benches.
# usage: bash scripts/gpu_check.sh [pytest-args]
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
for K in 1 2; do
  timeout 600 python bench.py --particles 1e8 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --rebin-interval $K \
    > gpurun_out/bench_1e8_K$K.log 2>&1; echo "bench K=$K rc=$?"
  tail -3 gpurun_out/bench_1e8_K$K.log
done
if [ -n "$FULL" ]; then
  timeout 900 python bench.py --steps 10 --warmup 3 --rebin-interval 1 > gpurun_out/bench_full_K1.log 2>&1; echo "bench full rc=$?"
  tail -2 gpurun_out/bench_full_K1.log
fi
