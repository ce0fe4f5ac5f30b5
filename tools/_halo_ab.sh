# loaded capacity and 24-SM layer times: halo weight-ring depth 4 (default) / 2, and no halo kernel
mkdir -p gpurun_out
for v in "default" "DARIS_HALO_WS=2" "DARIS_CONV_HALO=0"; do
  for rep in 1 2; do
    env $([ "$v" = default ] || echo "$v") timeout 300 python tools/capacity_probe.py --shapes 4x2_2,1x16_1 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> gpurun_out/halo_ab.jsonl
  done
  env $([ "$v" = default ] || echo "$v") timeout 300 python tools/profile_convs.py --sms 24 > "gpurun_out/halo_ab_layers_$v.txt" 2>&1
done
cat gpurun_out/halo_ab.jsonl
