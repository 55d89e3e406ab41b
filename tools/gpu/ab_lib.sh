#!/bin/bash
# A/B of prebuilt libpfbank.so variants under lib_var/<name>/ on one box:
#   bash tools/gpu/ab_lib.sh cfg4 old f0 f1
set -u
cfg=$1; shift
mkdir -p gpurun_out
cp paper_1407_8071_b200/lib/libpfbank.so /tmp/libpfbank.keep.so
for rep in 1 2; do
  for v in "$@"; do
    cp lib_var/$v/libpfbank.so paper_1407_8071_b200/lib/libpfbank.so
    python bench.py --config $cfg --no-cpu-baseline > gpurun_out/ab_${cfg}_${v}_$rep.log 2>&1
  done
done
cp /tmp/libpfbank.keep.so paper_1407_8071_b200/lib/libpfbank.so
