#!/bin/bash
# Round profile capture (run on the GPU box after the plain bench has exited 0):
# one `ncu --set full` capture of each workload's dominant kernel plus the
# launch lists (gpu__time_duration, cold-cache, serialised) of every workload.
#   bash tools/profile_all.sh [round-prefix, default r02]
set -u
R=${1:-r02}
out=gpurun_out/prof_$R
mkdir -p $out
cap() {  # name regex config [skip]
  ncu --set full --clock-control none --import-source on -k "regex:$2" -s ${4:-2} -c 1 -o $out/$1 -f \
    python bench.py --config $3 --steps 2 --warmup 3 --no-cpu-baseline --profile \
    > $out/$1.log 2>&1
  # summaries travel back (gpurun_out is capped at 64 MiB); the reports do not
  python tools/ncu_summary.py $out/$1.ncu-rep > $out/${R}_ncu_$1.txt 2>&1
  ncu -i $out/$1.ncu-rep --page raw --csv > $out/${R}_ncu_$1_raw.csv 2>/dev/null
  ncu -i $out/$1.ncu-rep --page source --csv --print-source sass > $out/${R}_ncu_$1_sass.csv 2>/dev/null
  gzip -f $out/${R}_ncu_$1_sass.csv
  rm -f $out/$1.ncu-rep
}
cap fhn_cm_cfg4 fhn_cm_kernel cfg4
cap lorenz_fast_cfg2 lorenz_fast_kernel cfg2
cap resample_bank_cfg1b resample_bank_kernel cfg1b
cap wide2_merge_cfg1c wide2_merge cfg1c
cap fhnnet_fast_net fhnnet_fast_kernel net
cap lorenz_small_cfg0 lorenz_small_kernel cfg0 12  # past the truth simulation's launches
for c in cfg4 cfg3 cfg2 cfg1b cfg1c cfg0 net cfg2apf netapf; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 120 --csv --log-file $out/launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --profile \
    > $out/launches_$c.log 2>&1
done
echo done
