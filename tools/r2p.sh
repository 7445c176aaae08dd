mkdir -p gpurun_out
RF_LANES=148 RF_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:regfile_tc --launch-skip 1 --launch-count 1 -o gpurun_out/rf_full2 python tools/probes/regfile_timing.py regfile > gpurun_out/rf_ncu.log 2>&1
echo ncu rc=$?
