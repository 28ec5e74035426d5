#!/bin/bash
# fast GPU iteration: build, GPU parity tests, quick timing.  usage: bash tools/quick_gpu.sh [pytest -k expr]
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/q_build.log 2>&1 || { tail -30 $O/q_build.log; exit 1; }
K=${1:-}
if [ -n "$K" ]; then timeout 600 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -15
else timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15; fi
timeout 300 python tools/quick_step.py 20 2>&1 | tail -3
