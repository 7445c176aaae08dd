mkdir -p gpurun_out
timeout 600 python tools/probes/regfile_synth.py > gpurun_out/rf_synth.txt 2>&1
