#!/bin/bash
# Build an alternative copy of the C-ABI library for same-box A/B timing.
#   tools/ab_build.sh NAME [REV]   -> ab_libs/libNAME.so from the working tree's
#   csrc/include, with csrc files taken from git revision REV when given.
# Select it at run time with CS_LIBPATH=ab_libs/libNAME.so.
set -e
NAME=$1; REV=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/ab_$NAME
rm -rf "$T"; mkdir -p "$T/pkg/csrc" "$T/include" "$T/obj" "$ROOT/ab_libs"
cp "$ROOT"/paper_2506_05617_b200/csrc/* "$T/pkg/csrc/"
cp "$ROOT"/include/* "$T/include/"
if [ -n "$REV" ]; then
  for f in $(git -C "$ROOT" ls-tree --name-only "$REV" paper_2506_05617_b200/csrc/); do
    git -C "$ROOT" show "$REV:$f" > "$T/pkg/csrc/$(basename "$f")"
  done
fi
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $CS_AB_FLAGS"
pids=()
for f in $(cd "$T/pkg/csrc" && ls *.cu | sed "s/\.cu$//"); do
  $NV $FL -c "$T/pkg/csrc/$f.cu" -o "$T/obj/$f.o" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p" || { echo "ab_build: a compile failed" >&2; exit 1; }; done
$NV -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$ROOT/ab_libs/lib$NAME.so" "$T"/obj/*.o -lcufft -Xlinker -rpath,/usr/local/cuda/lib64
echo "built ab_libs/lib$NAME.so"
