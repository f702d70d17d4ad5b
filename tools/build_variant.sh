#!/bin/bash
# Build an experimental variant of the library into _ab/<name>/ (git-ignored,
# travels with gpurun) for A/B timing with tools/ab_*.py:
#   tools/build_variant.sh g4 -DTSM_EPI_GROUPS=4
#   PYTHONPATH=_ab/g4 python tools/ab_epi.py
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
# SRC_ROOT: build another tree (e.g. `git archive HEAD | tar -x -C /tmp/old`)
src=${SRC_ROOT:-$root}
out=$root/_ab/$name
pkg=paper_1910_00932_b200
mkdir -p $out/build
rm -rf $out/$pkg
cp -r $src/$pkg $out/
rm -f $out/$pkg/libtsm_b200.so
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3,-fvisibility=hidden -I$src/include -I$src/$pkg/csrc $*"
pids=()
for f in $src/$pkg/csrc/*.cu; do
  b=$(basename $f .cu)
  $NV -c -o $out/build/$b.o $f & pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/$pkg/libtsm_b200.so $out/build/*.o -Xcompiler -fvisibility=hidden
echo "built $out/$pkg/libtsm_b200.so"
