#!/bin/bash
# A/B builds of the strip kernel on the GPU box: staging by cooperative cp.async (default) or
# by per-lane bulk copies (-DSP_ST_BULK).
cd paper_1610_08035_b200/csrc
for v in "" "-DSP_ST_BULK"; do
  touch stream_solve.cu
  make -s -j8 SSFLAGS="$v" 2>&1 | grep -E "error"
  (cd ../.. && timeout 120 python tools/stream_time.py "strip ${v:-cp.async}" && timeout 200 python tools/stream_check.py quick | grep -E "CHECK|worst" && timeout 60 python tools/stream_stamps.py 2>&1 | tail -16 | head -7)
done
