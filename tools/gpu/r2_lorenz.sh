set -u
mkdir -p gpurun_out/prof
TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_noise.py -q -p no:cacheprovider -x -k "lorenz" > gpurun_out/r2_lz_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_lz_$TAG.log
for i in 1 2; do timeout 600 python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline --profile >> gpurun_out/r2_lz_$TAG.log 2>&1; done
if [ "${2:-}" = "ncu" ]; then
timeout 900 ncu --set full --clock-control none -k "regex:lorenz_fast" -s 2 -c 1 -o gpurun_out/prof/lz_$TAG -f \
    python bench.py --config cfg2 --steps 2 --warmup 2 --no-cpu-baseline --profile > gpurun_out/prof/lz_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/prof/lz_$TAG.ncu-rep > gpurun_out/prof/lz_$TAG.txt 2>&1
fi
