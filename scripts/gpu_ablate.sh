#!/bin/bash
# Step-kernel ablation on C5 (K=1 fused): which stage costs what.
# Needs the ablation build: make clean && make NVFLAGS_EXTRA=-DST_ABLATION_BUILD (never ship it).
NP=${1:-1e9}
for M in ${MODES:--1 29 27 30 16}; do
  ST_ABLATE=$M timeout 600 python bench.py --particles $NP --steps 4 --warmup 2 --no-cpu-baseline --no-e2e --rebin-interval 1 \
    > gpurun_out/ablate_$M.log 2>&1
  python - "$M" <<'PY'
import json, sys
m = sys.argv[1]
for l in open(f"gpurun_out/ablate_{m}.log"):
    if l.startswith("{"):
        j = json.loads(l)
        print(f"ABLATE {m:>3}: step_kernel {j['step_kernel_ms']:.2f} ms  prep {j['rebin_prep_ms']:.2f} ms  step {j['ms_per_step']:.2f} ms")
        break
else:
    print(f"ABLATE {m}: failed", open(f"gpurun_out/ablate_{m}.log").read()[-300:])
PY
done
