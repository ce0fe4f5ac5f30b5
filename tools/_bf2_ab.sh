# Packed-bf16 residual add + activation in the conv epilogue: numerics, profiles, capacity.
# flat 1x1 tiling rule: numerics, per-layer profiles at b64 / b1, closed-loop capacity at 4x2.
set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_nets_gpu.py tests/test_p3_gpu.py -x -q > gpurun_out/bf_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/bf_tests.log
timeout 300 python tools/profile_convs.py --model resnet50 --batch 64 --sms 148 > gpurun_out/bf_b64.txt 2>&1
timeout 300 python tools/profile_convs.py --model resnet50 --batch 1 --sms 32 > gpurun_out/bf_b1.txt 2>&1
timeout 300 python tools/capacity_probe.py --shapes 4x2_2,4x4_2 --seconds 2 > gpurun_out/bf_capacity.txt 2>&1
head -1 gpurun_out/bf_b64.txt gpurun_out/bf_b1.txt; cat gpurun_out/bf_capacity.txt | tail -4; tail -2 gpurun_out/bf_tests.log
