# A/B: BN=64 implicit-GEMM CTAs at 4 per SM (80 regs, 2-stage ring) vs 3 (96 regs, 3-stage ring)
mkdir -p gpurun_out
for v in "-DDARIS_CONV_MAXNREG=96 -DDARIS_BN64_STAGES=3" "-DDARIS_CONV_MAXNREG=80 -DDARIS_BN64_STAGES=2" "-DDARIS_CONV_MAXNREG=96 -DDARIS_BN64_STAGES=2"; do
  DARIS_NVCC_EXTRA="$v" python -m paper_2504_08795_b200.build --force > /dev/null
  DARIS_PRINT_OCC=1 timeout 300 python tools/profile_convs.py --sms 24 2>&1 | grep -v "dyn smem\|carveout" | head -3 | sed "s|^|[$v] |" >> gpurun_out/occ4_ab.txt
  for rep in 1 2; do
    timeout 300 python tools/capacity_probe.py --shapes 4x2_2,1x16_1 2>/dev/null | grep '^{' | sed "s|^{|{\"variant\": \"$v\", \"rep\": $rep, |" >> gpurun_out/occ4_ab.jsonl
  done
done
python -m paper_2504_08795_b200.build --force > /dev/null
cat gpurun_out/occ4_ab.txt
