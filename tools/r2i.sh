mkdir -p gpurun_out
for L in 4 10 14; do FHEGPU_RF_LOOK=$L timeout 300 python tools/probes/regfile_timing.py regfile; done > gpurun_out/rf_timing.txt 2>&1
FHEGPU_RF_DIST=8 timeout 300 python tools/probes/regfile_timing.py regfile >> gpurun_out/rf_timing.txt 2>&1
FHEGPU_RF_BUFFERS=16 timeout 300 python tools/probes/regfile_timing.py regfile >> gpurun_out/rf_timing.txt 2>&1
