#!/bin/bash
# A/B of library variants (build/variants/*.so) on one box + the GPU tests of the in-tree build.
# usage: bash scripts/r2_ab.sh <tag> "<bench args>" [test]
TAG=${1:-r2ab}; ARGS=${2:-"--steps 30 --warmup 3 --no-cpu-baseline --no-micro --no-e2e"}
if [ "$3" == "test" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"; grep -E "^FAILED|Error" gpurun_out/${TAG}_pytest.log | head -5
fi
cp paper_2603_26691_b200/lib/libscaletrack.so /tmp/lib_orig.so
for rep in 1 2; do
for v in build/variants/*.so; do
  cp $v paper_2603_26691_b200/lib/libscaletrack.so
  timeout 900 python bench.py $ARGS > gpurun_out/${TAG}_$(basename $v .so)_$rep.log 2>&1
  python - "$v" gpurun_out/${TAG}_$(basename $v .so)_$rep.log << 'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        j = json.loads(l); s = j.get("step_kernel_ms_series", [])
        print(f"{sys.argv[1]:36s} {j['ms_per_step']:.3f} ms/step frac {j['roofline']['frac']:.3f} series first/last 4: {s[:4]} {s[-4:]}")
        break
else:
    print(sys.argv[1], "FAILED", open(sys.argv[2]).read()[-300:])
PY
done; done
cp /tmp/lib_orig.so paper_2603_26691_b200/lib/libscaletrack.so
