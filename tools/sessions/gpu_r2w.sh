#!/bin/bash
# Round-2 session W: the N>1 bench harness at full size with every process on this one GPU
# (RS_BENCH_SAME_DEVICE=1: CUDA-IPC arenas, .sys handshakes; NOT an NVLink measurement).
OUT=gpurun_out/r2w
mkdir -p $OUT
export RS_BENCH_SAME_DEVICE=1
for n in 2 4 8; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port $((29700+n)) \
    bench.py --gpus $n --steps 5 --warmup 3 > $OUT/bench_n${n}_same_gpu.json 2> $OUT/bench_n${n}.err
  echo "n=$n rc=$?"; python -c "import json; d=json.load(open('$OUT/bench_n${n}_same_gpu.json')); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['bound'], d['correct'], d['e2e']['value'], d['e2e']['ok'])"
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29799 \
  bench.py --gpus 4 --steps 3 --warmup 3 --case c5b --mode staged --profile-layers 8 --no-e2e > $OUT/bench_n4_c5b_staged_relay.json 2> $OUT/bench_c5b.err
echo "c5b rc=$?"; python -c "import json; d=json.load(open('$OUT/bench_n4_c5b_staged_relay.json')); print(d['ms_per_step'], d['config']['relay_routes'], [g['out_GB'] for g in d['roofline']['per_gpu']], d['correct'])"
