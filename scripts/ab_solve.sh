#!/bin/bash
cp paper_2509_21221_b200/libgwtf.so /tmp/orig.so
# stress cluster-tier solve time (stress_step_probe.py solve) of library variants in variants/<name>/libgwtf.so (testing only)
for v in "$@"; do
  cp variants/$v/libgwtf.so paper_2509_21221_b200/libgwtf.so
  echo -n "$v "; python scripts/stress_step_probe.py solve 2>&1 | tail -1
done
cp /tmp/orig.so paper_2509_21221_b200/libgwtf.so
