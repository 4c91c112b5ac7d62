#!/bin/bash
# compute-sanitizer over the round-2 kernels (tools/sanitize_r2.py).
OUT=gpurun_out/${1:-san2}
mkdir -p "$OUT"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_r2.py > "$OUT/$tool.txt" 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|sanitize cases ok' "$OUT/$tool.txt" | tr '\n' ' ')"
done
