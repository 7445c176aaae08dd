mkdir -p gpurun_out
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
cat gpurun_out/bench_default.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'resident_tc|level_tc_ws' --launch-skip 1 --launch-count 1 -o gpurun_out/ws_full python tools/ncu_probe.py 131072 > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
# configs[0] warp-dataflow launch: timing vs level launches, per-gate trace (needs a -DFHEGPU_TRACE=1 build at
# paper_1611_08769_b200/libfhegpu_trace.so), full ncu capture of flow_kernel
FLOW_WARM_S=1 python tools/probes/flow_timing.py flow levels > gpurun_out/flow_timing.txt 2>&1; echo flow timing rc=$?
[ -f paper_1611_08769_b200/libfhegpu_trace.so ] && FHEGPU_LIB=$PWD/paper_1611_08769_b200/libfhegpu_trace.so timeout 300 python tools/probes/flow_trace.py > gpurun_out/flow_trace.txt 2>&1; echo flow trace rc=$?
FLOW_WARM_S=0 timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:flow_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/flow_full python tools/probes/flow_timing.py flow > gpurun_out/ncu_flow.log 2>&1; echo flow ncu rc=$?
# configs[4] register-file launch: timing, per-slot role timeline (trace build), full ncu capture (148 lanes = one per CTA)
RF_REPS=3 timeout 300 python tools/probes/regfile_timing.py regfile > gpurun_out/rf_timing.txt 2>&1; echo rf timing rc=$?
[ -f paper_1611_08769_b200/libfhegpu_trace.so ] && FHEGPU_LIB=$PWD/paper_1611_08769_b200/libfhegpu_trace.so timeout 300 python tools/probes/timeline_regfile.py 40 > gpurun_out/rf_timeline.txt 2>&1; echo rf timeline rc=$?
RF_LANES=148 RF_REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:regfile_tc_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/rf_full python tools/probes/regfile_timing.py regfile > gpurun_out/ncu_rf.log 2>&1; echo rf ncu rc=$?
