#!/bin/bash
# One gpurun call's worth of round evidence: GPU parity tests, smoke, the
# default bench line, the ncu launch list of the bench command and one
# `ncu --set full` capture each of the fused step kernel, the standalone
# contraction and the strong-form kernel.  Everything lands in gpurun_out/ (read back here with
# tools/make_profiles.py).  usage: bash tools/gpu_round.sh [TAG]
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/${TAG}_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > $O/${TAG}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tc2?_step' -s 2 -c 1 \
  -o $O/${TAG}_step -f python tools/profile_step.py 4 > $O/${TAG}_ncu_step.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract -c 1 \
  -o $O/${TAG}_contract -f python tools/profile_step.py 1 > $O/${TAG}_ncu_contract.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sf_step -c 1 \
  -o $O/${TAG}_strong -f python tools/quick_strong.py > $O/${TAG}_ncu_strong.log 2>&1
ls -la $O
