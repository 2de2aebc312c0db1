#!/bin/bash
# usage: scripts/ab_build.sh NAME "EXTRA NVCC FLAGS"
# Builds a variant of the library into ab/NAME/libvsx_b200.so; select it with
# VSX_LIB=ab/NAME/libvsx_b200.so (A/B timing of compile-time variants).
set -e
name="$1"; extra="$2"
root="$(cd "$(dirname "$0")/.." && pwd)"
out="$root/ab/$name"
mkdir -p "$out/obj"
cd "$root/paper_2503_23044_b200/csrc"
objs=()
for f in *.cu; do
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 \
    -diag-suppress 177 $extra -c "$f" -o "$out/obj/${f%.cu}.o" &
  objs+=("$out/obj/${f%.cu}.o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libvsx_b200.so" "${objs[@]}"
echo "built $out/libvsx_b200.so"
