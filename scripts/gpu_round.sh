#!/bin/bash
# Round-end GPU session: parity suite, bench line, ncu launch list + full captures (gpt bench
# kernels and the stress cluster tier).  Outputs under gpurun_out/round/.
O=gpurun_out/round; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 600 python bench.py --steps 2 --warmup 3 --quick > $O/bench_quick.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_gpt.csv \
  python bench.py --steps 2 --warmup 3 --quick > $O/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"rounds_kernel|ssp_kernel" \
  --launch-skip 13 --launch-count 3 -o $O/gpt_full python bench.py --steps 1 --warmup 3 --quick > $O/ncu_gpt_full.log 2>&1
timeout 300 python scripts/stress_probe.py --supply 64 --reps 1 > $O/stress_probe64.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ssp_cluster -c 1 -o $O/stress_full \
  python scripts/stress_probe.py --supply 64 --reps 1 > $O/ncu_stress_full.log 2>&1
ls -la $O
