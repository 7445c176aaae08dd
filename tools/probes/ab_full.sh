#!/bin/bash
# A/B alternative libfhegpu.so builds: kernel parity tests, then sustained throughput
# (tools/power_probe.py) in the tiled (auto) and level schedules.  Restores the original.
LANES=${LANES:-131072}
SECS=${SECS:-4}
mkdir -p gpurun_out
cp paper_1611_08769_b200/libfhegpu.so /tmp/libfhegpu_orig.so
for lib in "$@"; do
  cp "$lib" paper_1611_08769_b200/libfhegpu.so
  echo "== $lib"
  if [ -z "$NOTEST" ]; then
    timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -2
  fi
  for sch in auto levels; do
    timeout -s KILL 120 python tools/probes/power_probe.py $LANES $SECS 0 $sch 2>&1 | tail -1
  done
done
cp /tmp/libfhegpu_orig.so paper_1611_08769_b200/libfhegpu.so
