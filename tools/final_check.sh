#!/bin/bash
# Round-end evidence on one B200: smoke, pytest -m gpu, bench (both arms), launch list,
# ncu of the field chain.  Outputs gpurun_out/$1_*.
set -u
p=gpurun_out/${1:-final}
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${p}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > ${p}_gpu_tests.log 2>&1
python bench.py > ${p}_bench.json 2> ${p}_bench.err
python bench.py --impl reference > ${p}_reference.json 2> ${p}_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${p}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-amr > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_field_chain -s 10 -c 1 -o ${p}_chain \
  python tools/chain_time.py > /dev/null 2>&1
ncu -i ${p}_chain.ncu-rep --page raw --csv > ${p}_chain_raw.csv 2>&1
rm -f ${p}_chain.ncu-rep
tail -2 ${p}_gpu_tests.log; tail -c 300 ${p}_bench.json; echo; tail -c 200 ${p}_reference.json
