#!/bin/bash
# compute-sanitizer over every kernel family on small configs; logs in gpurun_out/sanitizer/
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for case in "ssp tiny 8" "ssp gpt 4" "ssp_cluster gpt 2" "ssp_cluster stress_s 1" "rounds tiny 8" "rounds gpt 4" \
              "rounds_cluster gpt 2" "rounds_cluster stress_s 1" "warm gpt 4" "churn gpt 4"; do
    set -- $case
    log=gpurun_out/sanitizer/${tool}_$1_$2.log
    timeout 600 $CS --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize.py $1 $2 $3 > $log 2>&1
    echo "$tool $1 $2 rc=$?" | tee -a gpurun_out/sanitizer/summary.txt
  done
done
