mkdir -p gpurun_out
timeout 300 python tools/probes/regfile_timing.py > gpurun_out/rf_timing.txt 2>&1
python bench.py --no-fft-single --cpu-seconds 0 > gpurun_out/bench_rf.json 2> gpurun_out/bench_rf.err
