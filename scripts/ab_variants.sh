#!/bin/bash
# A/B timing of library variants built into variants/<name>/libgwtf.so (testing only):
#   bash scripts/ab_variants.sh [--configs] v0 v1 ...
# gpt bench step (ms, rounds ms, ssp ms); with --configs also llama / churn rounds ms and the
# stress rounds (200 rounds of the 8 stress instances).
cp paper_2509_21221_b200/libgwtf.so /tmp/orig.so
CFG=0; if [ "$1" == "--configs" ]; then CFG=1; shift; fi
for v in "$@"; do
  cp variants/$v/libgwtf.so paper_2509_21221_b200/libgwtf.so
  echo -n "$v gpt "; python bench.py --steps 20 --warmup 3 --quick 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print(round(d['ms_per_step'],3), round(k['rounds_kernel']['ms_total']/20,3), round(k['ssp_kernel']['ms_total']/20,3))"
  if [ $CFG == 1 ]; then
    for c in llama churn; do echo -n "$v "; python scripts/config_probe.py $c 2>&1 | tail -1 | cut -c1-400; done
    echo -n "$v stress "; python scripts/stress_probe.py --supply 64 --reps 1 --rounds 200 2>&1 | tail -1 | cut -c1-300
  fi
done
cp /tmp/orig.so paper_2509_21221_b200/libgwtf.so
