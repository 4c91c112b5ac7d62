#!/bin/bash
# Round-2 session r3b: NVSwitch multicast / VMM capability probe on the one visible B200.
OUT=gpurun_out/r3b
mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo.txt 2>&1
nvidia-smi nvlink -s > $OUT/nvlink_status.txt 2>&1
nvidia-smi -q | grep -i -A3 "fabric\|nvlink\|imex" > $OUT/fabric.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/mc_probe.cu -lcuda -o /tmp/mc_probe && timeout 120 /tmp/mc_probe > $OUT/mc_probe.jsonl 2>&1
echo "mc_probe rc=$?" >> $OUT/mc_probe.jsonl
cat $OUT/mc_probe.jsonl; head -20 $OUT/topo.txt; head -30 $OUT/nvlink_status.txt; cat $OUT/fabric.txt | head -30
