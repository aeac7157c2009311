#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/sweep.log
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "rounds or churn or hand or edge or full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
GWTF_ROUNDS_GLOBAL=1 timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "rounds or churn" >> gpurun_out/pytest_gpu.log 2>&1; echo "pytest(global) rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in "GWTF_ROUNDS_TPI=32" "GWTF_ROUNDS_TPI=64" "GWTF_ROUNDS_TPI=128" "GWTF_ROUNDS_TPI=64 GWTF_ROUNDS_GLOBAL=1" "GWTF_ROUNDS_TPI=128 GWTF_ROUNDS_GLOBAL=1" "GWTF_ROUNDS_TPI=32 GWTF_ROUNDS_GLOBAL=1"; do
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --quick ${BENCH_ARGS} > gpurun_out/b.log 2>&1
  echo "$cfg $(grep '^{' gpurun_out/b.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k:round(v['ms_total']/d['steps'],3) for k,v in d['kernels'].items()})") $(tail -1 gpurun_out/b.log | head -c 200)" >> gpurun_out/sweep.log
done
