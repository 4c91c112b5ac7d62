#!/bin/bash
# Round-2 session r4b: STAGED stream lanes with / without L2 discards of
# drained slots (ncu showed the discards at ~20 % of the lane kernel's L2
# sector lookups); full C2 timings alternated, then ncu L2 sector counters of
# both variants on the 4-layer slice.
OUT=gpurun_out/r4b
mkdir -p $OUT
for rep in 1 2; do
  for d in 0 4; do
    RS_SWEEP_RING_DISCARD=$d RS_SWEEP_STEPS=7 timeout 600 python tools/stream_sweep.py c2 0 2:0:0:0 \
      | sed "s/^{/{\"ring_discard\": $d, \"rep\": $rep, /" >> $OUT/discard_sweep.jsonl 2>> $OUT/sweep.err
  done
done
cat $OUT/discard_sweep.jsonl
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
for d in 0 4; do
  RS_SWEEP_RING_DISCARD=$d RS_SWEEP_STEPS=2 timeout 900 ncu --metrics $M --clock-control none -k regex:rs_stream_lane_kernel \
    -s 2 -c 1 --csv --log-file $OUT/ncu_discard$d.csv python tools/stream_sweep.py c2 4 2:0:0:0 > $OUT/ncu_discard$d.txt 2>&1
done

for d in 0 4; do echo "== discard $d"; grep -v "^==" $OUT/ncu_discard$d.csv | cut -d, -f13-15 | tail -9; done
