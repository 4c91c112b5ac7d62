#!/bin/bash
# Round-2 session r4v: the N>1 bench path with the final code, all processes
# on the one B200 (RS_BENCH_SAME_DEVICE=1): N=2 and N=8 DIRECT lines on a
# C2 8-layer slice (e2e included), N=4 STAGED strict on the same slice.
OUT=gpurun_out/r4v
mkdir -p $OUT
for n in 2 8; do
  RS_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 3 --warmup 3 --profile-layers 8 \
    > $OUT/bench_n$n.json 2> $OUT/bench_n$n.err
  echo "n=$n rc=$?"; head -c 600 $OUT/bench_n$n.json; echo
done
RS_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 3 --warmup 3 --profile-layers 8 \
  --mode staged --strict 1 --no-e2e > $OUT/bench_n4_staged_strict.json 2> $OUT/bench_n4_staged_strict.err
echo "n=4 strict rc=$?"; head -c 600 $OUT/bench_n4_staged_strict.json
