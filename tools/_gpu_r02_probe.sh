timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "linear or avgpool" > gpurun_out/r02_linear_tests2.log 2>&1
timeout 200 python tools/profile_convs.py --model resnet50 --batch 64 --sms 148 > gpurun_out/r02_prof_r50_b64_v3.txt 2>&1
timeout 200 python tools/timeline_convs.py --model resnet50 --sms 24 --json gpurun_out/r02_timeline_24.json > gpurun_out/r02_timeline_24.txt 2>&1
timeout 300 python tools/capacity_probe.py --shapes 4x2_2,4x4_2,1x8_1 --seconds 1.0 > gpurun_out/r02_capacity.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"conv_igemm|linear_tc|avgpool|maxpool|pack_nhwc" \
  --log-file gpurun_out/r02_ncu_launch_list_forward.csv python tools/one_forward.py --model resnet50 --plan 23 --reps 2 > gpurun_out/r02_ncu_ll.log 2>&1
