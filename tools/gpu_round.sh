#!/bin/bash
# One gpurun call's worth of round evidence: GPU parity tests, smoke, the
# driver's bench command, the reference arm, the ncu launch list of the bench
# command and one `ncu --set full` capture each of the fused step kernel (C5
# gear, width class 32), its 64-wide class (the paper's [2,50,50,50,1] gear),
# the standalone contraction, the split-path row contraction (C3 40x40), the
# two-output (spatial-eps) step on the C4 disk and the strong-form step.  Everything lands in gpurun_out/ (read back here with
# tools/make_profiles.py).  usage: bash tools/gpu_round.sh [TAG]
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/${TAG}_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > $O/${TAG}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_step -s 2 -c 1 \
  -o $O/${TAG}_step -f python tools/profile_step.py 4 > $O/${TAG}_ncu_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_step -s 2 -c 1 \
  -o $O/${TAG}_h50 -f python tools/profile_h50.py > $O/${TAG}_ncu_h50.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_warp -c 1 \
  -o $O/${TAG}_contract -f python tools/profile_step.py 1 > $O/${TAG}_ncu_contract.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_rowreg -c 2 \
  -o $O/${TAG}_c3rows -f python tools/profile_c3.py 2 > $O/${TAG}_ncu_c3rows.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc2_step -s 2 -c 1 \
  -o $O/${TAG}_spatial -f python tools/profile_spatial.py > $O/${TAG}_ncu_spatial.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sf2_step -s 2 -c 1 \
  -o $O/${TAG}_strong -f python tools/quick_strong2.py > $O/${TAG}_ncu_strong.log 2>&1
ls -la $O | grep $TAG
tail -3 $O/${TAG}_pytest_gpu.log
