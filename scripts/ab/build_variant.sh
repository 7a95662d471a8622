#!/bin/bash
# Build libsmoe_b200.so from a git revision (or the working tree: REV=WT) into
# scripts/_bin/libsmoe_<name>.so, with optional extra nvcc flags (e.g. -DSMOE_WAIT_HINT=0),
# for A/B comparisons inside one GPU session: SMOE_LIB=scripts/_bin/libsmoe_<name>.so.
# usage: build_variant.sh REV NAME [nvcc flags...]
set -e
rev=$1; name=$2; shift 2
root=$(cd "$(dirname "$0")/../.." && pwd)
tmp=$(mktemp -d)
if [ "$rev" = WT ]; then
  cp -r "$root/paper_2403_08245_b200" "$root/include" "$tmp/"
else
  git -C "$root" archive "$rev" paper_2403_08245_b200/csrc include | tar -x -C "$tmp"
fi
objs=()
for f in "$tmp"/paper_2403_08245_b200/csrc/*.cu; do
  o="$tmp/$(basename "$f" .cu).o"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I "$tmp/include" "$@" -c "$f" -o "$o" &
  objs+=("$o")
done
wait
mkdir -p "$root/scripts/_bin"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC "${objs[@]}" -o "$root/scripts/_bin/libsmoe_$name.so"
rm -rf "$tmp"
echo "$root/scripts/_bin/libsmoe_$name.so"
