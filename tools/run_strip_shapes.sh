#!/bin/bash
# A/B builds of the strip kernel's b = 3 shape on the GPU box: warps per CTA, blocks per sub-tile.
cd paper_1610_08035_b200/csrc
for v in "8 4" "9 4" "7 4" "4 8"; do
  set -- $v
  touch stream_solve.cu
  make -s -j8 SSFLAGS="-DSP_ST3_NW=$1 -DSP_ST3_MB=$2" 2>&1 | grep -E "error"
  (cd ../.. && timeout 120 python tools/stream_time.py "strip NW=$1 MB=$2" && timeout 200 python tools/stream_check.py quick | grep -E "CHECK|worst")
done
