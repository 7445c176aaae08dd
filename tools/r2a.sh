mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs 2>&1 | tail -25 > gpurun_out/gputest.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_resident.py 4097 > gpurun_out/racecheck.txt 2>&1; echo race rc=$?
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_resident.py 4097 > gpurun_out/synccheck.txt 2>&1; echo sync rc=$?
tail -3 gpurun_out/gputest.txt
