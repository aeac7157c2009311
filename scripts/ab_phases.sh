#!/bin/bash
# dev-build phase tables of library variants (variants/<name>/libgwtf.so built with make DEV=1), full-supply stress solve
cp paper_2509_21221_b200/libgwtf.so /tmp/orig.so
for v in "$@"; do
  cp variants/$v/libgwtf.so paper_2509_21221_b200/libgwtf.so
  echo "== $v"; GWTF_DEBUG_FLAGS=16 python scripts/stress_probe.py --supply ${SUPPLY:-4096} --reps 1 2>&1 | tail -15 | cut -c1-200
done
cp /tmp/orig.so paper_2509_21221_b200/libgwtf.so
