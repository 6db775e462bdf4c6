#!/bin/bash
# Round-2: the strong-scaling jobs on one GPU, and the 8-rank head-sharded fig6
# dry run (gloo, all ranks on cuda:0 -- a check of the multi-rank path, not a measurement)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --config rl8 --steps 2 --warmup 3 --no-configs --no-next --no-cpu-baseline > gpurun_out/r02_job_rl8.json 2> gpurun_out/r02_job_rl8.err
timeout 300 python bench.py --config fig6 --steps 10 --warmup 3 --no-configs --no-next --no-cpu-baseline > gpurun_out/r02_job_fig6.json 2> gpurun_out/r02_job_fig6.err
timeout 300 python bench.py --config sdar_8b_strong --steps 5 --warmup 3 --no-configs --no-next --no-cpu-baseline > gpurun_out/r02_job_sdar_8b_strong.json 2> gpurun_out/r02_job_strong.err
BD_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 8 --steps 2 --warmup 3 --config fig6 --dist-backend gloo --no-next --no-cpu-baseline --no-e2e --no-configs > gpurun_out/r02_fig6_8rank_gloo_dryrun.json 2> gpurun_out/r02_fig6_dry.err
for f in gpurun_out/r02_job_*.json gpurun_out/r02_fig6_8rank_gloo_dryrun.json; do echo "$f"; tail -c 200 $f; echo; done
