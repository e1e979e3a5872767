#!/bin/bash
# parity tests, then the C5 bench at 1e9 for several rebin intervals K
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
for K in ${KS:-1 2 4}; do
  timeout 900 python bench.py --particles ${NP:-1e9} --steps 8 --warmup 3 --rebin-interval $K --no-cpu-baseline --no-e2e > gpurun_out/bench_K$K.log 2>&1
  python -c "import json; j=[json.loads(l) for l in open('gpurun_out/bench_K$K.log') if l.startswith('{')]; j=j[0] if j else None; print('K=$K', {k:j[k] for k in ['ms_per_step','step_kernel_ms','rebin_prep_ms','value','rebins_in_timed_region','fused_rebins']} if j else open('gpurun_out/bench_K$K.log').read()[-400:])"
done
