set -u
mkdir -p gpurun_out/prof
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputest1.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest1.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench1.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench1.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fhn_fast_kernel" -s 2 -c 1 -o gpurun_out/prof/fhn_fast_r2a -f \
    python bench.py --config cfg4 --steps 2 --warmup 2 --no-cpu-baseline --profile > gpurun_out/prof/fhn_fast_r2a.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof/fhn_fast_r2a.log
