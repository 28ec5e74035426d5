bash tools/gpu_tests.sh r02i "split or c3 or forward_sine or inverse_eps or q400 or shape_grid or standalone or spill or cuda_core"
python tools/quick_sweeps.py > gpurun_out/r02i_sweeps.json 2>&1; cat gpurun_out/r02i_sweeps.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_rows -c 2 -o gpurun_out/r02i_c3rows -f python tools/profile_c3.py 2 > gpurun_out/r02i_ncu.log 2>&1
tail -3 gpurun_out/r02i_ncu.log
