#!/bin/bash
# A/B timing of two compile-time variants of the native library on one box:
# bash tools/ab_build.sh "-DFLAG=0" "-DFLAG=1" [rounds]
A="$1"; B="$2"; R=${3:-3}
LIB=paper_2404_12063_b200/_lib/libvpinn_b200.so
VPINN_EXTRA_NVCC="$A" python -m paper_2404_12063_b200.build_native > /dev/null && cp $LIB /tmp/libA.so
VPINN_EXTRA_NVCC="$B" python -m paper_2404_12063_b200.build_native > /dev/null && cp $LIB /tmp/libB.so
for i in $(seq $R); do
  for v in A B; do
    cp /tmp/lib$v.so $LIB
    echo "$v $(python tools/quick_step.py 30 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_ms"],4), round(d["epoch_flushed_ms"],4))')"
  done
done
python -m paper_2404_12063_b200.build_native --force > /dev/null
