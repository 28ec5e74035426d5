bash tools/gpu_tests.sh r02n
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sf2_step -s 2 -c 1 -o gpurun_out/r02n_strong -f python tools/quick_strong2.py > gpurun_out/r02n_ncu.log 2>&1
tail -2 gpurun_out/r02n_ncu.log
