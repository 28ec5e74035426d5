#!/bin/bash
# Build N compile-time variants HERE into ab/lib<i>.so (they travel with the
# snapshot); on the box: bash tools/ab_multi_run.sh N "CMD" [rounds]
# usage: bash tools/ab_multi_local.sh "-DFLAG=0" "-DFLAG=1" ...
set -e
LIB=paper_2404_12063_b200/_lib/libvpinn_b200.so
mkdir -p ab
i=0
for f in "$@"; do
  VPINN_EXTRA_NVCC="$f" python -m paper_2404_12063_b200.build_native > /dev/null && cp $LIB ab/lib$i.so
  echo "ab/lib$i.so: $f"; i=$((i+1))
done
python -m paper_2404_12063_b200.build_native --force > /dev/null
