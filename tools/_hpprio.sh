# A/B on one box: C2 knee with and without high-priority streams for HP stages
for v in 1 0; do
  if [ $v = 1 ]; then export DARIS_HP_STREAM_PRIORITY=1; else unset DARIS_HP_STREAM_PRIORITY; fi
  timeout 600 python bench.py --verbose --no-cpu --no-batching > gpurun_out/bench_hpprio$v.json 2> gpurun_out/bench_hpprio$v.log
done
