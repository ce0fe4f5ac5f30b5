# round-2 ncu evidence (run under gpurun, one GPU): launch list of one ResNet-50 b1 forward at the C2
# plan, full-set captures of the conv kernel (-> bench traffic json) and of the tensor-core linear
# (VGG-16 FC1 at batch 1 on 148 SMs, ResNet-50 head at batch 64), exported to CSV on the box.
set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_ncu_launch_list_forward.csv \
  python tools/one_forward.py --model resnet50 --plan 23 --reps 2 > gpurun_out/r02_ncu_ll.log 2>&1
bash tools/_ncu_r02.sh
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"linear_tc" -c 3 \
  -o /tmp/prof_lin_vgg python tools/one_forward.py --model vgg16 --sms 148 --plan 148 --reps 1 \
  > gpurun_out/r02_ncu_lin.log 2>&1
ncu -i /tmp/prof_lin_vgg.ncu-rep --page raw --csv > gpurun_out/r02_ncu_full_linear_vgg_b1_raw.csv 2>> gpurun_out/r02_ncu_lin.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"linear_tc" -c 1 \
  -o /tmp/prof_lin_r50 python tools/one_forward.py --model resnet50 --sms 148 --plan 148 --batch 64 --reps 1 \
  >> gpurun_out/r02_ncu_lin.log 2>&1
ncu -i /tmp/prof_lin_r50.ncu-rep --page raw --csv > gpurun_out/r02_ncu_full_linear_r50_b64_raw.csv 2>> gpurun_out/r02_ncu_lin.log
ls -la gpurun_out/
