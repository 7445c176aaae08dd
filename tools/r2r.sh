mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'resident_tc' --launch-skip 1 --launch-count 1 -o gpurun_out/ws_full python tools/ncu_probe.py 131072 > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
python tools/probes/api_timing.py > gpurun_out/api_timing.txt 2>&1
