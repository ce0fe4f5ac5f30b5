# Residual by TMA at batch 1 (DARIS_NO_RES_TMA=1 turns it off): b1 forward at the C2 plan + loaded capacity
set -x
for k in off on; do
  if [ $k = off ]; then export DARIS_NO_RES_TMA=1; else unset DARIS_NO_RES_TMA; fi
  echo "== res_tma $k" >> gpurun_out/s5_rt_b1.txt
  timeout 300 python tools/profile_convs.py --model resnet50 --batch 1 --sms 32 > gpurun_out/s5_rt_b1_$k.txt 2>&1
  head -1 gpurun_out/s5_rt_b1_$k.txt >> gpurun_out/s5_rt_b1.txt
  timeout 300 python tools/capacity_probe.py --shapes 4x2_2,4x4_2 --seconds 3 | grep shape >> gpurun_out/s5_rt_b1.txt 2>&1
done
cat gpurun_out/s5_rt_b1.txt
