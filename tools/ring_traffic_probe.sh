#!/bin/bash
# DRAM traffic of the STAGED exchange kernel vs ring slot size (C2 4-layer
# slice, L2 policies + discard): does a smaller ring footprint stop the ring
# traffic from reaching DRAM?  One ncu metric pass per slot size.
OUT=gpurun_out/${1:-ringtraffic}
mkdir -p "$OUT"
for kib in 32 64 128 256 1024; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv -k regex:rs_exchange_kernel -s 3 -c 1 --log-file "$OUT/slot${kib}.csv" \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --profile-layers 4 --mode staged \
    --ring-slot-kib $kib > "$OUT/slot${kib}.txt" 2>&1
  echo "slot ${kib} KiB: $(grep -v '^==' "$OUT/slot${kib}.csv" | tail -4 | awk -F'","' '{print $13"="$15}' | tr '\n' ' ')"
done
