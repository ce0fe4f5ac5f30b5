# A/B of the flat 1x1 M tiling (DARIS_CONV_FLAT): per-layer ResNet-50 timing at batch 64 (148 SMs)
# and batch 1 (C2 plan, 32 SMs), plus the kernel/network numerics tests.
set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_nets_gpu.py -x -q > gpurun_out/flat_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/flat_tests.log
for f in 1 0; do
  DARIS_CONV_FLAT=$f timeout 300 python tools/profile_convs.py --model resnet50 --batch 64 --sms 148 > gpurun_out/flat${f}_b64.txt 2>&1
  DARIS_CONV_FLAT=$f timeout 300 python tools/profile_convs.py --model resnet50 --batch 1 --sms 32 > gpurun_out/flat${f}_b1.txt 2>&1
done
head -1 gpurun_out/flat1_b64.txt gpurun_out/flat0_b64.txt gpurun_out/flat1_b1.txt gpurun_out/flat0_b1.txt
tail -2 gpurun_out/flat_tests.log
