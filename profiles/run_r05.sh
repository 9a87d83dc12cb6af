set -x
mkdir -p gpurun_out/r05
timeout 600 python -m pytest tests/test_gpu_group.py -q -x > gpurun_out/r05/pytest_group.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r05/pytest_gpu.log 2>&1
bash bench_tools/group_variants.sh
