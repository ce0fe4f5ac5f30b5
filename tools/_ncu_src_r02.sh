# source-level (SASS + stall reasons) ncu captures of two b1 conv launches at the C2 plan:
# launch 6 = layer1.1.conv3 (BN=128, residual, 1 K block), launch 16 = layer2.1.conv3 (BN=64, residual)
set -x
for s in 6 16 26; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"conv_igemm" -s $s -c 1 \
    -o /tmp/src_$s python tools/one_forward.py --model resnet50 --plan 23 --reps 1 > gpurun_out/r02_ncu_src_$s.log 2>&1
  ncu -i /tmp/src_$s.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_ncu_src_$s.csv 2>> gpurun_out/r02_ncu_src_$s.log
  ncu -i /tmp/src_$s.ncu-rep --page details --csv > gpurun_out/r02_ncu_details_$s.csv 2>> gpurun_out/r02_ncu_src_$s.log
done
