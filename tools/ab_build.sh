#!/bin/bash
# Build libsldg with the files $3.. (default step_fused.cu) of git revision $1 as
# _lib/libsldg_$2.so (the rest of the sources from the working tree), for same-box A/B
# timing: SLDG_LIB_VARIANT=$2.  Revision "-" builds the working tree as is; extra
# nvcc flags (e.g. -DFOO=1) come from $AB_FLAGS.
set -e
cd "$(dirname "$0")/.."
rev=$1; name=$2; shift 2
files=("$@"); [ ${#files[@]} -eq 0 ] && files=(step_fused.cu)
tmp=$(mktemp -d)
cp -r paper_2603_19959_b200/csrc/. "$tmp/"
if [ "$rev" != "-" ]; then
  for f in "${files[@]}"; do git show "$rev:paper_2603_19959_b200/csrc/$f" > "$tmp/$f"; done
fi
objs=()
for f in "$tmp"/*.cu; do
  o="$tmp/$(basename "$f").o"
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    -Xcompiler -O3 --expt-relaxed-constexpr $AB_FLAGS -Iinclude -I"$tmp" -c "$f" -o "$o" 2>/dev/null &
  objs+=("$o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_19959_b200/_lib/libsldg_$name.so "${objs[@]}"
rm -rf "$tmp"
echo built paper_2603_19959_b200/_lib/libsldg_$name.so
