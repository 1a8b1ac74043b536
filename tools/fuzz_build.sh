#!/bin/bash
# Build the schedule-fuzzing variant of libsldg (-DSLDG_FUZZ: pseudo-random sleeps before
# every bulk copy, cp.async, mbarrier wait, pipeline barrier and cluster barrier) as
# paper_2603_19959_b200/_lib/libsldg_fuzz.so; loaded with SLDG_LIB_VARIANT=fuzz by
# tests/test_gpu_schedule_fuzz.py, which requires bit-identical results.
set -e
cd "$(dirname "$0")/.."
out=build/obj_fuzz
mkdir -p "$out"
objs=()
for f in paper_2603_19959_b200/csrc/*.cu; do
  o="$out/$(basename "$f").o"
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    -Xcompiler -O3 --expt-relaxed-constexpr -DSLDG_FUZZ -Iinclude \
    -Ipaper_2603_19959_b200/csrc -c "$f" -o "$o" &
  objs+=("$o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_19959_b200/_lib/libsldg_fuzz.so "${objs[@]}"
echo built paper_2603_19959_b200/_lib/libsldg_fuzz.so
