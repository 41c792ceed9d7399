#!/bin/bash
# compute-sanitizer evidence: memcheck, racecheck and
# synccheck over short solves; summaries under gpurun_out/.
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py ${1:-all} \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|maxcut|config 1|dense aproj|Error|hazard" gpurun_out/sanitize_$tool.log | head -12
done
