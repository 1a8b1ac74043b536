#!/bin/bash
# Same-box A/B of the AMR step: tools/amr_clocks.py (ms/step + SM clocks) alternating the
# libraries named in $@ ("new" = _lib/libsldg.so) on $AB_CONFIG (default cfg5), 3 rounds.
set -u
vs=("$@"); [ ${#vs[@]} -eq 0 ] && vs=(base new)
for r in 1 2 3; do
  for v in "${vs[@]}"; do
    if [ "$v" = new ]; then unset SLDG_LIB_VARIANT; else export SLDG_LIB_VARIANT=$v; fi
    echo "$v $(python tools/amr_clocks.py --config ${AB_CONFIG:-cfg5} --steps ${AB_STEPS:-6} 2>&1 | tail -1)"
  done
done
unset SLDG_LIB_VARIANT
