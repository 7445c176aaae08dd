mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gputest_q.txt
python bench.py > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
cat gpurun_out/gputest_q.txt
