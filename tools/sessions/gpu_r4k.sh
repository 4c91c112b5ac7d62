#!/bin/bash
# Round-2 session r4k: STAGED lanes with the spare capacity handed out by
# bytes per lane (water-filling) vs proportional-only (RS_RING_NO_GROW=1),
# alternated on full C2 fused and strict, plus C5 / C5b-16 / C1 fused.
OUT=gpurun_out/r4k
mkdir -p $OUT
for rep in 1 2; do
  for g in 0 1; do
    RS_RING_NO_GROW=$g RS_SWEEP_STEPS=7 timeout 600 python tools/stream_sweep.py c2 0 2:0:0:0 \
      | sed "s/^{/{\"no_grow\": $g, \"rep\": $rep, /" >> $OUT/grow_fused.jsonl 2>> $OUT/err.txt
    RS_RING_NO_GROW=$g timeout 600 python tools/strict_sweep.py c2 0 128:0 \
      | sed "s/^{/{\"no_grow\": $g, \"rep\": $rep, /" >> $OUT/grow_strict.jsonl 2>> $OUT/err.txt
  done
done
for c in "c5 0" "c5b 16" "c1 0" "c4 16"; do
  for g in 0 1; do
    RS_RING_NO_GROW=$g RS_SWEEP_STEPS=7 timeout 600 python tools/stream_sweep.py $c 2:0:0:0 \
      | sed "s/^{/{\"no_grow\": $g, /" >> $OUT/grow_configs.jsonl 2>> $OUT/err.txt
  done
done
cat $OUT/grow_fused.jsonl $OUT/grow_strict.jsonl $OUT/grow_configs.jsonl; tail -3 $OUT/err.txt
