# ncu captures of the ResNet-50 b64 forward on 148 SMs (the batched operating point):
# full set of all 49 conv launches -> raw CSV; details + SASS source of the stem (0) and of
# layer1.1.conv3 (6, 1x1 + residual) to see what bounds the memory-bound layers.
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_" -s 0 -c 49 \
  -o /tmp/b64_convs python tools/one_forward.py --model resnet50 --sms 148 --plan 148 --batch 64 --reps 1 \
  > gpurun_out/r02_ncu_b64.log 2>&1
ncu -i /tmp/b64_convs.ncu-rep --page raw --csv > gpurun_out/r02_ncu_b64_convs_raw.csv 2>> gpurun_out/r02_ncu_b64.log
ncu -i /tmp/b64_convs.ncu-rep --page details --csv > gpurun_out/r02_ncu_b64_convs_details.csv 2>> gpurun_out/r02_ncu_b64.log
for s in 0 6; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"conv_" -s $s -c 1 \
    -o /tmp/b64_src_$s python tools/one_forward.py --model resnet50 --sms 148 --plan 148 --batch 64 --reps 1 \
    > gpurun_out/r02_ncu_b64_src_$s.log 2>&1
  ncu -i /tmp/b64_src_$s.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_ncu_b64_src_$s.csv 2>> gpurun_out/r02_ncu_b64_src_$s.log
done
