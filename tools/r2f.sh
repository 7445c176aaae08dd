mkdir -p gpurun_out
(for a in "0 2 1" "0 2 0"; do echo "== $a"; timeout 300 python tools/probes/regfile_debug.py $a; done) > gpurun_out/rf_debug.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_regfile.py -q -x 2>&1 | tail -5 > gpurun_out/gputest_rf.txt
timeout 300 python tools/probes/regfile_timing.py > gpurun_out/rf_timing.txt 2>&1
