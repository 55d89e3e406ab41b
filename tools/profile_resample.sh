#!/bin/bash
set -u
out=gpurun_out/prof
mkdir -p $out gpurun_out/bench
for c in cfg1b cfg1c cfg2; do
  python bench.py --config $c > gpurun_out/bench/$c.log 2>&1 || echo "FAILED $c" >> gpurun_out/bench/failures.txt
done
for c in cfg1b cfg1c; do
  python bench.py --config $c --sigma 10 > gpurun_out/bench/${c}_sigma10.log 2>&1 || echo "FAILED $c s10" >> gpurun_out/bench/failures.txt
done
cap() {
  ncu --set full --clock-control none --import-source on -k "regex:$2" -s 2 -c 1 -o $out/$1 \
    python bench.py --config $3 --steps 2 --warmup 2 --no-cpu-baseline --profile > $out/$1.log 2>&1
}
cap resample_bank_cfg1b resample_bank_kernel cfg1b
cap wide2_merge_cfg1c wide2_merge cfg1c
for c in cfg2 cfg1b cfg1c; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 80 --csv --log-file $out/launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile > $out/launches_$c.log 2>&1
done
