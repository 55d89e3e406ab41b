#!/bin/bash
# Round bench pass (GPU box): every bench.py workload with its CPU baseline,
# the reference arm on the default workload, then the cfg1 sigma = 10 cases.
#   bash tools/bench_all.sh [round-prefix, default r02]
set -u
R=${1:-r02}
out=gpurun_out/bench_$R
mkdir -p $out
for c in cfg4 cfg3 cfg2 cfg2m256 cfg1b cfg1c cfg0 net cfg4apf cfg2apf netapf dbf; do
  python bench.py --config $c > $out/$c.log 2>&1 || echo "FAILED $c" >> $out/failures.txt
done
for c in cfg1b cfg1c; do
  python bench.py --config $c --sigma 10 > $out/${c}_sigma10.log 2>&1 || echo "FAILED $c s10" >> $out/failures.txt
done
python bench.py --impl reference > $out/reference_cfg4.log 2>&1 || echo "FAILED reference" >> $out/failures.txt
echo done
