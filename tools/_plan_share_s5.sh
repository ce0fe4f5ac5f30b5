# Grid planning share after the epilogue diet: closed-loop capacity at 4x2 OS=2 (8 jobs) and 4x4 (16 jobs)
# for plan sizes 24 / 32 (default 1.75 x 148 / 8) / 40 SMs per job.
set -x
for p in 24 40 32; do
  DARIS_PLAN_SMS=$p timeout 300 python tools/capacity_probe.py --shapes 4x2_2 --seconds 3 >> gpurun_out/s5_plan_share.txt 2>&1
done
cat gpurun_out/s5_plan_share.txt | grep shape
