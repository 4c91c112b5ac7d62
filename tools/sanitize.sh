#!/bin/bash
# compute-sanitizer over the small GPU parity cases (every kernel: default TMA-NP copy, LDG,
# TMA bulk ring, exchange rings, pattern fill/verify, failure paths).
OUT=gpurun_out/${1:-san}
mkdir -p "$OUT"
SEL="test_mixed_dtype_gqa_glu_against_oracle and pair0 or test_failure_paths or test_verify_kernel or test_bound_caller or test_identity_resize or test_plan_sized_staging"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_executor.py -q -m gpu -k "$SEL" > "$OUT/$tool.txt" 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' "$OUT/$tool.txt" | tr '\n' ' ')"
done
