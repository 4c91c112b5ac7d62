#!/bin/bash
# Round-2 session J: full-size C4 (uneven 21/19 stage migration) and C3zb (flat-bucket ZeRO) per state group
# on the device (DIRECT + STAGED, pattern-verified) and full C4 through the windowed host-store path.
OUT=gpurun_out/r2j
mkdir -p $OUT
free -g > $OUT/mem.txt; cat $OUT/mem.txt
timeout 900 python tools/c4_full.py groups 3 c4 > $OUT/c4_groups.jsonl 2> $OUT/c4_groups.err; cat $OUT/c4_groups.jsonl; tail -3 $OUT/c4_groups.err
timeout 900 python tools/c4_full.py groups 3 c3zb > $OUT/c3zb_groups.jsonl 2> $OUT/c3zb_groups.err; cat $OUT/c3zb_groups.jsonl; tail -3 $OUT/c3zb_groups.err
timeout 1200 python tools/c4_full.py window 3 c4 > $OUT/c4_window.jsonl 2> $OUT/c4_window.err; cat $OUT/c4_window.jsonl; tail -3 $OUT/c4_window.err
