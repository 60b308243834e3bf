#!/bin/bash
# A/B timing of builds of libsaim.so on the same box, interleaved:
#   tools/ab.sh "configs" rounds lib1.so lib2.so ...   (prints config, build, ms)
CF=$1; N=$2; shift 2
LIB=paper_2501_04971_b200/libsaim.so
cp $LIB /tmp/ab_orig.so
for r in $(seq $N); do
  for v in "$@"; do
    cp $v $LIB
    python tools/bench_all.py --configs $CF --reps 3 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], '$(basename $v)', round(d['seconds']*1e3,2), 'ms', d['counters']['flips'], d['counters']['philox'], d['counters']['uniforms'])"
  done
done
cp /tmp/ab_orig.so $LIB
