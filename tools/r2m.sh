mkdir -p gpurun_out
(echo "lag1 look10"; timeout 300 python tools/probes/regfile_timing.py regfile
 echo "lag1 look14"; FHEGPU_RF_LOOK=14 timeout 300 python tools/probes/regfile_timing.py regfile
 echo "lag1 look6"; FHEGPU_RF_LOOK=6 timeout 300 python tools/probes/regfile_timing.py regfile
 echo "lag4 look10"; FHEGPU_LIB=$PWD/paper_1611_08769_b200/libfhegpu_lag4.so timeout 300 python tools/probes/regfile_timing.py regfile
 echo "lag1 buf 18"; FHEGPU_RF_BUFFERS=18 timeout 300 python tools/probes/regfile_timing.py regfile) > gpurun_out/rf_timing.txt 2>&1
