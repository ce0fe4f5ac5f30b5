# loaded capacity vs the split-K cap (default plan, at most 2 splits, no split-K)
mkdir -p gpurun_out
for v in default DARIS_SPLITK_MAX=2 DARIS_SPLITK_MAX=1; do for rep in 1 2; do
  env $([ "$v" = default ] || echo "$v") timeout 300 python tools/capacity_probe.py --shapes 4x2_2,1x16_1 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> gpurun_out/splitk_ab.jsonl
done; done
cat gpurun_out/splitk_ab.jsonl
