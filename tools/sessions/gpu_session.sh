#!/bin/bash
# One GPU session: tests, bench, ncu launch list, ncu full capture of the
# copy kernel on a profiling slice.  Usage (via gpurun):
#   bash tools/gpu_session.sh [tag] [parts...]   parts: tests bench ncu full
set -u
TAG=${1:-r1}
shift || true
PARTS=${*:-"tests bench ncu full"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,memory.free,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu.txt"
for p in $PARTS; do
  case $p in
    tests)
      python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.txt" 2>&1
      timeout 1500 python -m pytest tests -x -q -m gpu > "$OUT/pytest_gpu.txt" 2>&1
      tail -3 "$OUT/pytest_gpu.txt" ;;
    bench)
      timeout 1200 python bench.py --steps 10 --warmup 3 > "$OUT/bench.json" 2> "$OUT/bench.err"
      cat "$OUT/bench.json" ;;
    staged)
      timeout 900 python bench.py --steps 5 --warmup 3 --mode staged --no-e2e --no-cpu-baseline \
        > "$OUT/bench_staged.json" 2> "$OUT/bench_staged.err"
      cat "$OUT/bench_staged.json" ;;
    ref)
      timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
      cat "$OUT/bench_ref.json" ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
        > "$OUT/ncu_launch_bench.txt" 2>&1
      tail -2 "$OUT/ncu_launch_bench.txt" ;;
    full)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rs_copy_kernel -s 3 -c 1 \
        -o "$OUT/prof_copy" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --profile-layers 4 \
        > "$OUT/ncu_full.txt" 2>&1
      tail -2 "$OUT/ncu_full.txt" ;;
  esac
done
