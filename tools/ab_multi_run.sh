#!/bin/bash
# Alternate ab/lib0..N-1.so under one command on the GPU box:
# bash tools/ab_multi_run.sh N "python tools/quick_gear.py c5" [rounds]
N=$1; CMD="$2"; R=${3:-3}
LIB=paper_2404_12063_b200/_lib/libvpinn_b200.so
cp $LIB /tmp/lib_default.so
for r in $(seq $R); do
  for i in $(seq 0 $((N-1))); do
    cp ab/lib$i.so $LIB
    echo "$i $($CMD 2>&1 | tail -1 | cut -c1-400)"
  done
done
cp /tmp/lib_default.so $LIB
