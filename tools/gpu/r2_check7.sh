set -u
mkdir -p gpurun_out/prof
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -q -p no:cacheprovider -rs -s -k "wide or cfg1 or multinomial or resample" > gpurun_out/r2_gputest7.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest7.log
for c in cfg1c cfg0 cfg3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench7_$c.log 2>&1
  echo "bench rc=$?" >> gpurun_out/r2_bench7_$c.log
done
timeout 600 python bench.py --config cfg1c --sigma 10 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench7_cfg1c_s10.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:wide3_merge" -s 2 -c 1 -o gpurun_out/prof/wide3_merge_r2 -f \
    python bench.py --config cfg1c --steps 2 --warmup 2 --no-cpu-baseline --profile > gpurun_out/prof/wide3_merge_r2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches_cfg1c_r2.csv python bench.py --config cfg1c --steps 3 --warmup 2 --no-cpu-baseline --profile > gpurun_out/prof/launches_cfg1c_r2.log 2>&1
