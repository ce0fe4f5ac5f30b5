# A/B of the conv kernels' register cap (2 vs 3 resident CTAs per SM):
# per-layer times at 24 SMs, conv timeline, closed-loop capacity, GPU tests of the kernels
set -x
mkdir -p gpurun_out
for cap in 96 112; do
  DARIS_NVCC_EXTRA="-DDARIS_CONV_MAXNREG=$cap" python -m paper_2504_08795_b200.build --force > /dev/null
  timeout 300 python tools/profile_convs.py --sms 24 > gpurun_out/regcap_layers_$cap.txt 2>&1
  timeout 300 python tools/timeline_convs.py --sms 24 --dump layer1.1.conv3 > gpurun_out/regcap_timeline_$cap.txt 2>&1
  timeout 300 python tools/capacity_probe.py --shapes 4x2_2,1x16_1,1x1_1 > gpurun_out/regcap_capacity_$cap.jsonl 2>&1
done
python -m paper_2504_08795_b200.build --force > /dev/null
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_nets_gpu.py -q -x -m gpu > gpurun_out/regcap_tests.log 2>&1
tail -2 gpurun_out/regcap_tests.log
