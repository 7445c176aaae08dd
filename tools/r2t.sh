mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_regfile.py -q -x 2>&1 | tail -3
python bench.py --no-fft-single --cpu-seconds 0 --steps 10 > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err; echo rc=$?
