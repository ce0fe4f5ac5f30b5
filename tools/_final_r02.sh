# Session-5 state: numerics, per-layer profiles (b64 / b1), ncu full set of the b1 forward's convs at the
# C2 plan (-> traffic json for bench.py) and the launch list of one b1 forward.
set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_nets_gpu.py tests/test_p3_gpu.py -x -q > gpurun_out/s5_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s5_tests.log
timeout 300 python tools/profile_convs.py --model resnet50 --batch 64 --sms 148 > gpurun_out/s5_b64.txt 2>&1
timeout 300 python tools/profile_convs.py --model resnet50 --batch 1 --sms 32 > gpurun_out/s5_b1.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_igemm" -s 49 -c 49 \
  -o /tmp/prof_convs python tools/one_forward.py --model resnet50 --plan 32 --reps 2 > gpurun_out/s5_ncu_full.log 2>&1
ncu -i /tmp/prof_convs.ncu-rep --page raw --csv > gpurun_out/r02_ncu_full_convs_raw_s5.csv 2>> gpurun_out/s5_ncu_full.log
python tools/conv_traffic.py gpurun_out/r02_ncu_full_convs_raw_s5.csv --plan 32 \
  --capture r02_ncu_full_convs_raw_s5.csv.gz > gpurun_out/r02_conv_traffic_s5.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_launch_list.csv \
  python tools/one_forward.py --model resnet50 --plan 32 --reps 2 > gpurun_out/s5_launch_list.log 2>&1
head -1 gpurun_out/s5_b64.txt gpurun_out/s5_b1.txt; tail -2 gpurun_out/s5_tests.log; cat gpurun_out/r02_conv_traffic_s5.json
