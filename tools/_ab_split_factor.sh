# A/B: CTAs per planned SM for split-K grids (DARIS_SPLIT_FACTOR), isolated forward + loaded capacity
for f in 1 2 3; do
  echo "== DARIS_SPLIT_FACTOR=$f"
  DARIS_SPLIT_FACTOR=$f timeout 200 python tools/profile_convs.py --model resnet50 --batch 1 --sms 24 | head -1
  DARIS_SPLIT_FACTOR=$f timeout 300 python tools/capacity_probe.py --shapes 4x2_2,4x4_2 --seconds 1.0 | tail -2
done
