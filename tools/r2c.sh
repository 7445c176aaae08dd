mkdir -p gpurun_out
python tools/probes/api_timing.py > gpurun_out/api_timing.txt 2>&1
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gputest_c.txt
tail -3 gpurun_out/gputest_c.txt
