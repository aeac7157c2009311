#!/bin/bash
# stress rounds time (stress_step_probe.py rounds) of library variants in variants/<name>/libgwtf.so at the
# cluster sizes given by $CS (default "2 8"); testing only
cp paper_2509_21221_b200/libgwtf.so /tmp/orig.so
for v in "$@"; do
  cp variants/$v/libgwtf.so paper_2509_21221_b200/libgwtf.so
  for c in ${CS:-2 8}; do echo -n "$v C=$c "; GWTF_ROUNDS_CLUSTER_SIZE=$c python scripts/stress_step_probe.py rounds 2>&1 | tail -1; done
done
cp /tmp/orig.so paper_2509_21221_b200/libgwtf.so
