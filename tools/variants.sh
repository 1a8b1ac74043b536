#!/bin/bash
# Time each prebuilt library variant under build/variants/*.so on the headline
# config (fused-path parity tests + bench kernel time), one after another.
set -u
mkdir -p gpurun_out
cp paper_2603_19959_b200/_lib/libsldg.so /tmp/libsldg.orig.so
for v in build/variants/*.so; do
  cp "$v" paper_2603_19959_b200/_lib/libsldg.so
  t=$(timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pencil_shard.py -q -x -k "fused or pipelined or pencil" 2>&1 | grep -E "^FAILED|passed|failed" | cut -c1-100 | tr "\n" " ")
  j=$(SLDG_FUSED=force timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  k=$(echo "$j" | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),d['clocks']['sm_mhz'])" 2>&1)
  c=$(python tools/chain_time.py 2>&1 | tail -1)
  echo "$(basename $v): tests[$t] step/kernel/mhz: $k $c"
done
cp /tmp/libsldg.orig.so paper_2603_19959_b200/_lib/libsldg.so
