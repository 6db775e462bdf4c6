#!/bin/bash
# A/B timing of the builds in one directory (dev helper): bash scripts/ab_dir.sh DIR SCRIPT ARG
for rep in 1 2; do
for L in $1/*.so; do
  cp "$L" paper_2512_22234_b200/libbdattn.so
  echo "== $L"
  PYTHONPATH=. timeout 200 python $2 $3
done
done
