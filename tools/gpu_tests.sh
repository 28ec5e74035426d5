#!/bin/bash
# GPU test pass: build, pytest -m gpu (optional -k expr), smoke.  usage: bash tools/gpu_tests.sh TAG [K-EXPR]
TAG=${1:-t}; K=${2:-}
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/${TAG}_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1 || { tail -30 $O/${TAG}_build.log; exit 1; }
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -q -rA -k "$K" > $O/${TAG}_pytest.log 2>&1
else timeout 1500 python -m pytest tests -m gpu -q -rA > $O/${TAG}_pytest.log 2>&1; fi
echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
tail -3 $O/${TAG}_pytest.log; grep -E "FAILED|ERROR" $O/${TAG}_pytest.log | head -30; tail -2 $O/${TAG}_smoke.log
