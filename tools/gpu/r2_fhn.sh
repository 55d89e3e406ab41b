set -u
mkdir -p gpurun_out/prof
TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_noise.py -q -p no:cacheprovider -x -k "fhn" > gpurun_out/r2_fhn_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_fhn_$TAG.log
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --profile >> gpurun_out/r2_fhn_$TAG.log 2>&1
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --profile >> gpurun_out/r2_fhn_$TAG.log 2>&1
if [ "${2:-}" = "ncu" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${3:-fhn_}" -s 2 -c 1 -o gpurun_out/prof/fhn_$TAG -f \
    python bench.py --config cfg4 --steps 2 --warmup 2 --no-cpu-baseline --profile > gpurun_out/prof/fhn_$TAG.log 2>&1
fi
