# ncu full set of the 49 conv launches of a ResNet-50 b64 forward on 148 SMs after the session-5 changes
set -x
timeout 900 ncu --set full --clock-control none -k regex:"conv_" -s 0 -c 49 \
  -o /tmp/b64_s5 python tools/one_forward.py --model resnet50 --sms 148 --plan 148 --batch 64 --reps 1 \
  > gpurun_out/s5_ncu_b64.log 2>&1
ncu -i /tmp/b64_s5.ncu-rep --page raw --csv > gpurun_out/r02_ncu_full_convs_b64_raw_s5.csv 2>> gpurun_out/s5_ncu_b64.log
ls -la gpurun_out/r02_ncu_full_convs_b64_raw_s5.csv
