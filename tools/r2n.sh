mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_regfile.py -q -x 2>&1 | tail -3 > gpurun_out/gputest_rf.txt
(timeout 300 python tools/probes/regfile_timing.py regfile; FHEGPU_RF_NOREUSE=1 timeout 300 python tools/probes/regfile_timing.py regfile) > gpurun_out/rf_timing.txt 2>&1
cat gpurun_out/gputest_rf.txt
