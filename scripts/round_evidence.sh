set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests.txt
timeout 600 ncu --set full --clock-control none -k regex:"attn_|bwd_|build_map|logprob|zero" -o gpurun_out/full_b16 -f python scripts/profile_step.py sdar_8b 16 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm2sm|lse_combine" -o gpurun_out/lmhead_full -f python scripts/profile_lmhead.py sdar_1_7b > gpurun_out/ncu_lmhead.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"decode_|select_" -c 4 -o gpurun_out/decode_full -f python scripts/bench_decode.py sdar_8b 1 > gpurun_out/ncu_decode.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-next > gpurun_out/launch_bench.log 2>&1
timeout 900 python bench.py --steps 8 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
cat gpurun_out/gpu_tests.txt gpurun_out/smoke.txt; tail -c 600 gpurun_out/bench.json
