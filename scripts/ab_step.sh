#!/bin/bash
# A/B of alternative builds inside the real step (bench.py, phase times): each build twice, interleaved.
for rep in 1 2; do
for L in scripts/libs_tmp/*.so; do
  cp "$L" paper_2512_22234_b200/libbdattn.so
  echo "== $L"
  timeout 300 python bench.py --steps 8 --warmup 3 --no-e2e --no-configs --no-next --no-cpu-baseline ${BENCH_ARGS} | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'], d['phase_ms'], d['clocks']['sm_mhz'], d['roofline_other']['logprob_fused']['frac'])"
done
done
