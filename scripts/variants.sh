#!/bin/bash
# A/B of library builds on one box: each build/variants/*.so in turn as the library.
# usage: bash scripts/variants.sh [bench args...]
ARGS=${@:-"--steps 6 --warmup 3 --no-cpu-baseline --no-micro --no-e2e"}
cp paper_2603_26691_b200/lib/libscaletrack.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  cp $v paper_2603_26691_b200/lib/libscaletrack.so
  timeout 600 python bench.py $ARGS > /tmp/v.log 2>&1
  python - "$v" << 'PY'
import json, sys
for l in open("/tmp/v.log"):
    if l.startswith("{"):
        j = json.loads(l); print(f"{sys.argv[1]:40s} {j['ms_per_step']:.3f} ms/step  step_kernel {j['step_kernel_ms']:.3f}  frac {j['roofline']['frac']:.3f}")
        break
else:
    print(sys.argv[1], "FAILED", open("/tmp/v.log").read()[-400:])
PY
done
cp /tmp/lib_orig.so paper_2603_26691_b200/lib/libscaletrack.so
