VPINN_EXTRA_NVCC=-DVPG_PHASE_CLOCK=1 python -m paper_2404_12063_b200.build_native > /dev/null || exit 1
python tools/phase_clock.py c2_1 > gpurun_out/r02k_phase_c2.txt 2>&1
python tools/phase_clock.py c2_8 > gpurun_out/r02k_phase_c2_8.txt 2>&1
python tools/phase_clock.py > gpurun_out/r02k_phase_gear.txt 2>&1
cat gpurun_out/r02k_phase_c2.txt gpurun_out/r02k_phase_gear.txt
