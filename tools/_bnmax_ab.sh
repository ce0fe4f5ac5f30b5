# loaded capacity vs the widest automatic conv tile (default 128 vs 64)
mkdir -p gpurun_out
for v in default DARIS_CONV_BN_MAX=64; do for rep in 1 2; do
  env $([ "$v" = default ] || echo "$v") timeout 300 python tools/capacity_probe.py --shapes 4x2_2,1x16_1 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> gpurun_out/bnmax_ab.jsonl
done; done
cat gpurun_out/bnmax_ab.jsonl
