#!/bin/bash
# ncu evidence for profiles/: launch list of the full-size bench (copy kernel
# share of the step) and --set full captures of the copy and exchange kernels
# on a 4-layer slice of the same C2 resize (a full-size replay would have ncu
# save/restore 94 GB per pass).  Parts: launches copy exchange
set -u
OUT=gpurun_out/${1:-prof}
shift || true
PARTS=${*:-"launches copy exchange"}
mkdir -p "$OUT"
for p in $PARTS; do
  case $p in
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
        python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > "$OUT/launch_bench.txt" 2>&1 ;;
    copy)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_copy -s 3 -c 1 \
        -o "$OUT/copy_full" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --profile-layers 4 \
        > "$OUT/copy_full.txt" 2>&1 ;;
    exchange)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_exchange_kernel -s 3 -c 1 \
        -o "$OUT/exchange_full" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --profile-layers 4 \
        --mode staged > "$OUT/exchange_full.txt" 2>&1
      timeout 600 python bench.py --steps 5 --warmup 3 --mode staged --no-e2e --no-cpu-baseline \
        > "$OUT/bench_staged.json" 2> "$OUT/bench_staged.err"
      cat "$OUT/bench_staged.json" ;;
  esac
done
ls -la "$OUT"
