# loaded capacity vs the per-job planning share (grid sizes), 4x2 OS 2 and 16 jobs
mkdir -p gpurun_out
for p in 18 23 30 36 48; do for rep in 1 2; do
  DARIS_PLAN_SMS=$p timeout 300 python tools/capacity_probe.py --shapes 4x2_2,1x16_1 2>/dev/null | grep '^{' | sed "s/^{/{\"plan_env\": $p, \"rep\": $rep, /" >> gpurun_out/plan_sweep96.jsonl
done; done
cat gpurun_out/plan_sweep96.jsonl
