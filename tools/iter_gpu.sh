#!/bin/bash
# one iteration on the box: GPU test suite (or -k subset) + C5 / paper-gear epoch timings
# usage: bash tools/iter_gpu.sh TAG [pytest -k expr]
TAG=${1:-it}; K=${2:-}
O=gpurun_out; mkdir -p $O
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $O/${TAG}_t.log 2>&1
else timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_t.log 2>&1; fi
tail -4 $O/${TAG}_t.log
timeout 300 python tools/quick_gear.py c5 paper > $O/${TAG}_g.json 2>&1; tail -2 $O/${TAG}_g.json
