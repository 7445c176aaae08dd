mkdir -p gpurun_out
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench mma_bench.cu && ./mma_bench peak > ../../gpurun_out/i8_peak.json 2>&1; ./mma_bench peak >> ../../gpurun_out/i8_peak_all.txt 2>&1)
cp gpurun_out/i8_peak.json profiles/i8_peak.json 2>/dev/null
python bench.py > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
