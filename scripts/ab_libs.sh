#!/bin/bash
# A/B timing of alternative builds of libbdattn.so (dev helper): each build timed twice, interleaved.
#   bash scripts/ab_libs.sh [config] [script]    (script default: scripts/quick_attn.py)
S=${2:-scripts/quick_attn.py}
for rep in 1 2; do
for L in scripts/libs_tmp/*.so; do
  cp "$L" paper_2512_22234_b200/libbdattn.so
  echo "== $L"
  PYTHONPATH=. timeout 200 python $S ${1:-sdar_8b}
done
done
