mkdir -p gpurun_out
python tools/probes/api_timing.py > gpurun_out/api_timing.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_templates.py tests/test_gpu_regfile.py -q 2>&1 | tail -3 > gpurun_out/gputest_s.txt
cat gpurun_out/gputest_s.txt
