#!/bin/bash
# A/B build of the library from a variant csrc tree:
#   tools/ab_build.sh <name> [elem2 header variant] [extra nvcc flags...]
# copies paper_2404_12703_b200/csrc to abtest/<name>/csrc, overlays the header, builds
# abtest/<name>/libhexdg_b200.so (load it with HEXDG_B200_LIB).
set -e
name=$1; shift
hdr=$1; shift || true
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/abtest/$name
rm -rf "$out"; mkdir -p "$out"
cp -r "$root/paper_2404_12703_b200/csrc" "$out/csrc"
mkdir -p "$out/include"; cp "$root/include/hexdg_b200.h" "$out/include/"
rm -f "$out"/csrc/*.o "$out"/csrc/*.so
if [ -n "$hdr" ] && [ "$hdr" != "-" ]; then b=$(basename "$hdr"); [ -f "$out/csrc/$b" ] || b=elem2.cuh; cp "$hdr" "$out/csrc/$b"; fi
A="-gencode arch=compute_100a,code=sm_100a"
C="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC $A $*"
cd "$out/csrc"
sed -i 's#"../../include/hexdg_b200.h"#"../include/hexdg_b200.h"#' common.cuh
nvcc -c kernels_exact.cu -o ke.o $C -fmad=false &
nvcc -c kernels_fast.cu -o kf.o $C -fmad=true &
nvcc -c api.cu -o api.o $C -fmad=false &
wait
nvcc -shared -o "$out/libhexdg_b200.so" ke.o kf.o api.o $A -lcudart
echo "$out/libhexdg_b200.so"
