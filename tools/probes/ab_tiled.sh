#!/bin/bash
# Sweep the tiled schedule's wavefront skew / chunk size across alternative libfhegpu.so builds
# (sustained tools/power_probe.py).  SKEWS / CHUNKS override the grid.  Restores the library.
LANES=${LANES:-131072}
cp paper_1611_08769_b200/libfhegpu.so /tmp/libfhegpu_orig.so
for lib in "$@"; do
  cp "$lib" paper_1611_08769_b200/libfhegpu.so
  for c in ${CHUNKS:-128}; do for k in ${SKEWS:-2 3 4}; do
    echo "== $lib chunk=$c skew=$k"
    FHEGPU_TILE_LANES=$c FHEGPU_TILE_SKEW=$k timeout -s KILL 120 python tools/probes/power_probe.py $LANES 4 0 tiled 2>&1 | tail -1
  done; done
done
cp /tmp/libfhegpu_orig.so paper_1611_08769_b200/libfhegpu.so
