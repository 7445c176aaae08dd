mkdir -p gpurun_out
FHEGPU_LIB=$PWD/paper_1611_08769_b200/libfhegpu_trace.so timeout 300 python tools/probes/timeline_regfile.py 40 > gpurun_out/rf_timeline.txt 2>&1
FHEGPU_LIB=$PWD/paper_1611_08769_b200/libfhegpu_trace.so timeout 300 python tools/probes/timeline_regfile.py 400 > gpurun_out/rf_timeline2.txt 2>&1
