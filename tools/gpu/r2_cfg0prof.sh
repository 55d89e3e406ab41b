set -u
R=r02; out=gpurun_out/prof_$R; mkdir -p $out
ncu --set full --clock-control none --import-source on -k "regex:lorenz_small_kernel" -s 12 -c 1 -o $out/lorenz_small_cfg0 -f \
    python bench.py --config cfg0 --steps 2 --warmup 3 --no-cpu-baseline --profile > $out/lorenz_small_cfg0.log 2>&1
python tools/ncu_summary.py $out/lorenz_small_cfg0.ncu-rep > $out/${R}_ncu_lorenz_small_cfg0.txt 2>&1
ncu -i $out/lorenz_small_cfg0.ncu-rep --page source --csv --print-source sass > $out/${R}_ncu_lorenz_small_cfg0_sass.csv 2>/dev/null
gzip -f $out/${R}_ncu_lorenz_small_cfg0_sass.csv; rm -f $out/lorenz_small_cfg0.ncu-rep
for c in cfg0 cfg2; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv --log-file $out/launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --profile > $out/launches_$c.log 2>&1
done
python bench.py --config cfg0 --steps 10 --warmup 3 > $out/bench_cfg0.log 2>&1
python bench.py --config cfg3 --steps 10 --warmup 3 > $out/bench_cfg3.log 2>&1
python bench.py --config cfg4apf --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_cfg4apf.log 2>&1
