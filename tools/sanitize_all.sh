#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py with each tool (GPU box):
#   bash tools/sanitize_all.sh OUT.txt
out=${1:-gpurun_out/sanitizer.txt}
: > $out
for tool in memcheck racecheck synccheck initcheck; do
  echo "## $tool" >> $out
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_driver.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|Error|Hazard|Invalid|sanitize driver" | head -40 >> $out
done
cat $out
