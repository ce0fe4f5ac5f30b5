# Whole images per M tile for <= 64-pixel maps (DARIS_CONV_IMGS): numerics, b64 profile on/off, b1 profile.
set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_nets_gpu.py tests/test_p3_gpu.py -x -q > gpurun_out/ipt_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ipt_tests.log
for f in 1 0; do
  DARIS_CONV_IMGS=$f timeout 300 python tools/profile_convs.py --model resnet50 --batch 64 --sms 148 > gpurun_out/ipt${f}_b64.txt 2>&1
done
timeout 300 python tools/profile_convs.py --model resnet50 --batch 1 --sms 32 > gpurun_out/ipt_b1.txt 2>&1
head -1 gpurun_out/ipt1_b64.txt gpurun_out/ipt0_b64.txt gpurun_out/ipt_b1.txt; grep 'layer4' gpurun_out/ipt1_b64.txt gpurun_out/ipt0_b64.txt | cut -c1-120; tail -2 gpurun_out/ipt_tests.log
