set -x
./tools/launch_rate.bin > gpurun_out/launch_rate.txt 2>&1
for part in green soft; do for pdl in 0 1; do for g in 8 2; do
  if [ $part = soft ] && [ $g = 2 ]; then continue; fi
  if [ $pdl = 0 ]; then export DARIS_NO_PDL=1; else unset DARIS_NO_PDL; fi
  DARIS_PART_GROUP=$g timeout 200 python tools/capacity_probe.py --partition $part --shapes 1x1_1,4x2_2,1x16_1 | sed "s/^/{\"group\": $g, \"pdl\": $pdl, /; s/, {/, /" >> gpurun_out/cap3.jsonl
done; done; done
