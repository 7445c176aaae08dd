mkdir -p gpurun_out
python -m pytest tests/test_gpu_templates.py tests/test_gpu_configs.py -q -k "template or replay or full_range or deps" -x 2>&1 | tail -15 > gpurun_out/gputest_b.txt
python tools/probes/api_timing.py > gpurun_out/api_timing.txt 2>&1
tail -3 gpurun_out/gputest_b.txt
