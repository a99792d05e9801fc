#!/bin/bash
# compute-sanitizer over scripts/sanitize_workload.py: every kernel family.
# The second pass forces the steady-state RHS tile pipeline (k_rhs_tp) onto
# the workload's small CH grids with a 3-CTA grid so its ring wraps.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|workload OK|Error|error" gpurun_out/sanitizer_$tool.log | head -5
  SG_CH_RHS_TP=2 SG_CH_RHS_TP_CTAS=3 timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/sanitizer_${tool}_tp.log 2>&1
  echo "$tool (rhs pipeline forced) rc=$?"; grep -E "ERROR SUMMARY|workload OK|Error|error" gpurun_out/sanitizer_${tool}_tp.log | head -5
done
