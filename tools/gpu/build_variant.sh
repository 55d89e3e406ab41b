#!/bin/bash
# Build lib_var/<name>/libpfbank.so with extra nvcc flags (run here, before gpurun), e.g.
#   bash tools/gpu/build_variant.sh p7 -DPF_PHILOX_ROUNDS=7
#   bash tools/gpu/build_variant.sh nosplit -DPF_FHN_SPLIT=-1
#   bash tools/gpu/build_variant.sh p10            # the production build
# then on the GPU box:  bash tools/gpu/ab_lib.sh cfg4 p10 p7   (or tools/gpu/ab_test.sh)
set -eu
name=$1; shift
root=$(cd "$(dirname "$0")/../.." && pwd)
obj=$(mktemp -d)
for f in "$root"/paper_1407_8071_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
    -I"$root/include" -I"$root/paper_1407_8071_b200/csrc" "$@" -c "$f" \
    -o "$obj/$(basename "$f" .cu).o" 2>/dev/null &
done
wait
mkdir -p "$root/lib_var/$name"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/lib_var/$name/libpfbank.so" "$obj"/*.o
rm -rf "$obj"
echo "built lib_var/$name/libpfbank.so ($*)"
