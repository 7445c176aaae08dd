#!/bin/bash
# A/B the perf probe against alternative builds of libfhegpu.so (restores the original).
cp paper_1611_08769_b200/libfhegpu.so /tmp/libfhegpu_orig.so
for lib in "$@"; do
  cp "$lib" paper_1611_08769_b200/libfhegpu.so
  echo "== $lib"; timeout -s KILL 120 python tools/probes/perf_probe.py 131072 0 2>&1 | grep lanes=
done
cp /tmp/libfhegpu_orig.so paper_1611_08769_b200/libfhegpu.so
