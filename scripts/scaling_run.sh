#!/bin/bash
# Weak-scaling lines of a config (default: the stress headline) on one box: N = 1, 2, 4 (one rank per GPU, NCCL),
# the config's instances per GPU, each line as the driver runs it (torchrun for N > 1).
#   bash scripts/scaling_run.sh [out.jsonl] [config] [steps]
out=${1:-gpurun_out/scaling.jsonl}
cfg=${2:-stress}
steps=${3:-3}
: > $out
ng=$(nvidia-smi -L | wc -l)
for n in 1 2 4 8; do
  [ $n -gt $ng ] && break
  if [ $n -eq 1 ]; then
    python bench.py --config $cfg --steps $steps --warmup 3 --no-configs --no-extras --no-cpu-baseline | tail -1 >> $out
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
      bench.py --config $cfg --gpus $n --steps $steps --warmup 3 --no-configs --no-extras --no-cpu-baseline 2>/dev/null | tail -1 >> $out
  fi
done
