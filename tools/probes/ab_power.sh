#!/bin/bash
# A/B sustained throughput + power (tools/power_probe.py) across alternative libfhegpu.so builds.
LANES=${LANES:-131072}
cp paper_1611_08769_b200/libfhegpu.so /tmp/libfhegpu_orig.so
for lib in "$@"; do
  cp "$lib" paper_1611_08769_b200/libfhegpu.so
  echo "== $lib"; timeout -s KILL 120 python tools/probes/power_probe.py $LANES 4 2>&1 | tail -1
done
cp /tmp/libfhegpu_orig.so paper_1611_08769_b200/libfhegpu.so
