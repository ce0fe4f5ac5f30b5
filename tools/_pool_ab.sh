# 3x3 max-pool fast path: exactness tests + per-layer profiles at b64 / b1
set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "maxpool" > gpurun_out/pool_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/pool_tests.log
timeout 300 python tools/profile_convs.py --model resnet50 --batch 64 --sms 148 > gpurun_out/pool_b64.txt 2>&1
timeout 300 python tools/profile_convs.py --model resnet50 --batch 1 --sms 32 > gpurun_out/pool_b1.txt 2>&1
head -1 gpurun_out/pool_b64.txt gpurun_out/pool_b1.txt; grep maxpool gpurun_out/pool_b64.txt gpurun_out/pool_b1.txt; tail -2 gpurun_out/pool_tests.log
