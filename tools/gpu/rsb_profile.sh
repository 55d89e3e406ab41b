#!/bin/bash
# cfg1b bank resampler capture + launch list (r02):  gpurun -- 'bash tools/gpu/rsb_profile.sh'
set -u
R=r02; out=gpurun_out/prof_$R; mkdir -p $out; n=resample_bank_cfg1b
ncu --set full --clock-control none --import-source on -k "regex:resample_bank_kernel" -s 2 -c 1 -o $out/$n -f python bench.py --config cfg1b --steps 2 --warmup 3 --no-cpu-baseline --profile > $out/$n.log 2>&1
python tools/ncu_summary.py $out/$n.ncu-rep > $out/${R}_ncu_$n.txt 2>&1
ncu -i $out/$n.ncu-rep --page source --csv --print-source sass > $out/${R}_ncu_${n}_sass.csv 2>/dev/null
gzip -f $out/${R}_ncu_${n}_sass.csv; rm -f $out/$n.ncu-rep
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv --log-file $out/launches_cfg1b.csv python bench.py --config cfg1b --steps 3 --warmup 3 --no-cpu-baseline --profile > $out/launches_cfg1b.log 2>&1
