#!/bin/bash
# Build two compile-time variants HERE (CPU container) into ab/lib{A,B}.so;
# they travel with the snapshot.  On the box: bash tools/ab_run.sh CMD [rounds]
# usage: bash tools/ab_local.sh "-DFLAG=0" "-DFLAG=1"
set -e
LIB=paper_2404_12063_b200/_lib/libvpinn_b200.so
mkdir -p ab
VPINN_EXTRA_NVCC="$1" python -m paper_2404_12063_b200.build_native > /dev/null && cp $LIB ab/libA.so
VPINN_EXTRA_NVCC="$2" python -m paper_2404_12063_b200.build_native > /dev/null && cp $LIB ab/libB.so
python -m paper_2404_12063_b200.build_native --force > /dev/null
echo "built ab/libA.so ($1) ab/libB.so ($2)"
