set -u
mkdir -p gpurun_out/prof_r02
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest_c0.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_c0.log
python bench.py --config cfg0 > gpurun_out/bench_cfg0.log 2>&1
out=gpurun_out/prof_r02; n=lorenz_small_cfg0
ncu --set full --clock-control none --import-source on -k "regex:lorenz_small_kernel" -s 12 -c 1 -o $out/$n -f python bench.py --config cfg0 --steps 2 --warmup 3 --no-cpu-baseline --profile > $out/$n.log 2>&1
python tools/ncu_summary.py $out/$n.ncu-rep > $out/r02_ncu_$n.txt 2>&1
ncu -i $out/$n.ncu-rep --page source --csv --print-source sass > $out/r02_ncu_${n}_sass.csv 2>/dev/null
gzip -f $out/r02_ncu_${n}_sass.csv; rm -f $out/$n.ncu-rep
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv --log-file $out/launches_cfg0.csv python bench.py --config cfg0 --steps 3 --warmup 3 --no-cpu-baseline --profile > $out/launches_cfg0.log 2>&1
