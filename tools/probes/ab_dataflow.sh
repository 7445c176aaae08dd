#!/bin/bash
# A/B tools/dataflow_probe.py across alternative libfhegpu.so builds (restores the original).
cp paper_1611_08769_b200/libfhegpu.so /tmp/libfhegpu_orig.so
for lib in "$@"; do
  cp "$lib" paper_1611_08769_b200/libfhegpu.so
  echo "== $lib"; timeout -s KILL 300 python tools/probes/dataflow_probe.py ${CFG:-cfg3} 2>&1 | grep -E "\(a|\(b|\(c"
done
cp /tmp/libfhegpu_orig.so paper_1611_08769_b200/libfhegpu.so
