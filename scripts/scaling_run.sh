#!/bin/bash
# Weak-scaling lines of the stress headline on one box: N = 1, 2, 4 (one rank per GPU, NCCL),
# 8 instances per GPU, each line as the driver runs it (torchrun for N > 1).
#   bash scripts/scaling_run.sh [out.jsonl]
out=${1:-gpurun_out/scaling.jsonl}
: > $out
ng=$(nvidia-smi -L | wc -l)
for n in 1 2 4 8; do
  [ $n -gt $ng ] && break
  if [ $n -eq 1 ]; then
    python bench.py --steps 3 --warmup 3 --no-configs --no-extras --no-cpu-baseline | tail -1 >> $out
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
      bench.py --gpus $n --steps 3 --warmup 3 --no-configs --no-extras --no-cpu-baseline 2>/dev/null | tail -1 >> $out
  fi
done
