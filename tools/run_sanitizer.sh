#!/bin/bash
# compute-sanitizer over the b >= 6 paths (settle UB vs miscompile)
for tool in memcheck initcheck racecheck synccheck; do
  compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_team.py > gpurun_out/sanitizer_team_$tool.log 2>&1
  echo "team $tool rc=$?" >> gpurun_out/sanitizer_summary.txt
done
for tool in memcheck initcheck; do
  SPINGP_TEAM=0 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_team.py > gpurun_out/sanitizer_thread_$tool.log 2>&1
  echo "thread-per-chunk $tool rc=$?" >> gpurun_out/sanitizer_summary.txt
done
