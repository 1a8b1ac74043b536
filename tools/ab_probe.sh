#!/bin/bash
# Same-box A/B of k_step_fused: tools/fused_probe.py alternating the libraries named in
# $@ ("new" = _lib/libsldg.so, anything else = _lib/libsldg_<name>.so) three rounds.
set -u
vs=("$@"); [ ${#vs[@]} -eq 0 ] && vs=(base new)
for r in 1 2 3; do
  for v in "${vs[@]}"; do
    if [ "$v" = new ]; then unset SLDG_LIB_VARIANT; else export SLDG_LIB_VARIANT=$v; fi
    echo "$v $(python tools/fused_probe.py --steps 30 ${PROBE_ARGS:-} 2>&1 | tail -1)"
  done
done
unset SLDG_LIB_VARIANT
