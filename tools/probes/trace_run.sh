#!/bin/bash
# Run tools/timeline.py against a trace build (ab/libfhegpu_trace.so), restoring the library.
cp paper_1611_08769_b200/libfhegpu.so /tmp/libfhegpu_orig.so
cp ab/libfhegpu_trace.so paper_1611_08769_b200/libfhegpu.so
python tools/probes/timeline.py "$@"
cp /tmp/libfhegpu_orig.so paper_1611_08769_b200/libfhegpu.so
