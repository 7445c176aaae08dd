mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_regfile.py -q -x 2>&1 | tail -3 > gpurun_out/gputest_rf.txt
timeout 300 python tools/probes/regfile_timing.py regfile > gpurun_out/rf_timing.txt 2>&1
FHEGPU_LIB=$PWD/paper_1611_08769_b200/libfhegpu_trace.so timeout 300 python tools/probes/timeline_regfile.py 40 > gpurun_out/rf_timeline.txt 2>&1
