#!/bin/bash
# A/B the lane-resident kernel on cfg1 (XOR + AND): slot order with operand reuse (default),
# dbg bit 20 = no operand reuse; then any ab/*.so given as arguments (same C-ABI).
mkdir -p gpurun_out
P=tools/energy_probe.py
L=${LANES:-131072}
cp paper_1611_08769_b200/libfhegpu.so /tmp/cur.so
for d in 0 1048576; do timeout -s KILL 120 python $P $L 3 $d resident 2>&1 | tail -1; done
for lib in "$@"; do
  echo "== $lib"
  cp "$lib" paper_1611_08769_b200/libfhegpu.so
  timeout -s KILL 120 python $P $L 3 0 resident 2>&1 | tail -1
  cp /tmp/cur.so paper_1611_08769_b200/libfhegpu.so
done
timeout -s KILL 120 python $P $L 3 0 resident 2>&1 | tail -1
