cp paper_2603_19959_b200/_lib/libsldg.so /tmp/o.so
for v in build/variants/*.so; do cp $v paper_2603_19959_b200/_lib/libsldg.so; echo "$(basename $v) $(python tools/chain_time.py 2>&1 | tail -1)"; done
cp /tmp/o.so paper_2603_19959_b200/_lib/libsldg.so
