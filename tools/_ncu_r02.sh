# round-2 ncu captures (run under gpurun): full set of one ResNet-50 b1 forward's 49 conv launches at the
# C2 plan -> raw CSV (+ traffic json for bench.py), and the launch list of a short bench command.
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_igemm" -s 49 -c 49 \
  -o /tmp/prof_convs python tools/one_forward.py --model resnet50 --plan 32 --reps 2 > gpurun_out/r02_ncu_full.log 2>&1
ncu -i /tmp/prof_convs.ncu-rep --page raw --csv > gpurun_out/r02_ncu_full_convs_raw.csv 2>> gpurun_out/r02_ncu_full.log
python tools/conv_traffic.py gpurun_out/r02_ncu_full_convs_raw.csv --plan 32 \
  --capture r02_ncu_full_convs_raw.csv.gz > gpurun_out/r02_conv_traffic.json
cp gpurun_out/r02_conv_traffic.json profiles/r02_conv_traffic.json
