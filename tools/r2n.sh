mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_regfile.py -q -x 2>&1 | tail -15 > gpurun_out/gputest_rf.txt
timeout 300 python tools/probes/regfile_timing.py regfile > gpurun_out/rf_timing.txt 2>&1
