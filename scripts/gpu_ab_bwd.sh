#!/bin/bash
# dev: parity of the current build's backward, then interleaved A/B timing of scripts/libs_tmp/*.so
cp scripts/libs_tmp/b_ts.so paper_2512_22234_b200/libbdattn.so
timeout 900 python -m pytest tests/test_gpu_attn_bwd.py tests/test_gpu_mask_probe.py tests/test_gpu_varlen.py tests/test_gpu_fullslice.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
tail -3 gpurun_out/ab_pytest.log
bash scripts/ab_libs.sh sdar_8b > gpurun_out/ab_time.log 2>&1
bash scripts/ab_libs.sh sdar_1_7b >> gpurun_out/ab_time.log 2>&1
cat gpurun_out/ab_time.log
