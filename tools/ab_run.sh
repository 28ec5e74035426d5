#!/bin/bash
# Alternate ab/libA.so and ab/libB.so under one command on the GPU box:
# bash tools/ab_run.sh "python tools/quick_strong.py" [rounds]
CMD="$1"; R=${2:-3}
LIB=paper_2404_12063_b200/_lib/libvpinn_b200.so
cp $LIB /tmp/lib_default.so
for i in $(seq $R); do
  for v in A B; do
    cp ab/lib$v.so $LIB
    echo "$v $($CMD | cut -c1-160)"
  done
done
cp /tmp/lib_default.so $LIB
