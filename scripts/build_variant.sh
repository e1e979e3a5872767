#!/bin/bash
# Build one library variant into build/variants/<name>.so (the in-tree library is untouched).
# usage: bash scripts/build_variant.sh <name> "<-D flags>"
set -e
mkdir -p build/variants
rm -f build/variants/$1.so build/variants/$1_micro.o
make -s LIB=build/variants/$1.so MICRO_O=build/variants/$1_micro.o NVFLAGS_EXTRA="$2" build/variants/$1.so
grep -A2 "k_fs" build/ptxas.log | grep -E "registers" | sort | uniq -c | head -3
