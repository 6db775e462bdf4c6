#!/bin/bash
# dev: parity of the candidate backward (scripts/libs_tmp/b_*.so), then interleaved A/B timing
cp scripts/libs_tmp/b_*.so paper_2512_22234_b200/libbdattn.so
timeout 900 python -m pytest tests/test_gpu_attn_bwd.py tests/test_gpu_mask_probe.py tests/test_gpu_varlen.py tests/test_gpu_graphs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
tail -2 gpurun_out/ab_pytest.log
for c in ${CONFIGS:-sdar_8b sdar_1_7b}; do bash scripts/ab_libs.sh $c; done > gpurun_out/ab_time.log 2>&1
cat gpurun_out/ab_time.log
