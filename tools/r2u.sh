mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gputest_u.txt
python bench.py --cpu-seconds 0 --sustain-s 0 > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err; echo rc=$?
cat gpurun_out/gputest_u.txt
