#!/bin/bash
# phase-clock diagnostics on the GPU box: rebuild with the phase marks compiled
# in, print the per-phase cycle table, then restore the production build.
VPINN_EXTRA_NVCC=-DVPG_PHASE_CLOCK=1 python -m paper_2404_12063_b200.build_native > /dev/null || exit 1
python tools/phase_clock.py "$@"
python -m paper_2404_12063_b200.build_native --force > /dev/null
