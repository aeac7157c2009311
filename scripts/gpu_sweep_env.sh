#!/bin/bash
# usage: gpu_sweep_env.sh "ENV1=a ENV2=b" "ENV1=c" ...   (quick bench per env setting)
mkdir -p gpurun_out; rm -f gpurun_out/sweep.log
if [ -n "$PYTEST_K" ]; then timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; fi
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --quick ${BENCH_ARGS} > gpurun_out/b.log 2>&1
  echo "$cfg $(grep '^{' gpurun_out/b.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k:round(v['ms_total']/d['steps'],3) for k,v in d['kernels'].items()})") $(grep -v '^{' gpurun_out/b.log | tail -1 | head -c 300)" >> gpurun_out/sweep.log
done
