#!/bin/bash
# Round-2 evidence run (one gpurun call): bench line, reference arm, ncu launch
# list of the bench command, one ncu --set full capture at the bench shape,
# compute-sanitizer summaries, smoke.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
if [ "${EVIDENCE_NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-next --no-configs > gpurun_out/r02_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"attn_|bwd_|build_map|logprob|zero|token_|group_" -o gpurun_out/r02_full_b16 -f python scripts/profile_step.py sdar_8b 16 > gpurun_out/r02_ncu_full.log 2>&1
fi
for tool in memcheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_tiny.py > gpurun_out/r02_sanitizer_$tool.txt 2>&1
done
grep -h "ERROR SUMMARY\|sanitize run ok" gpurun_out/r02_sanitizer_*.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.txt 2>&1
tail -c 300 gpurun_out/r02_bench.json; cat gpurun_out/r02_smoke.txt
