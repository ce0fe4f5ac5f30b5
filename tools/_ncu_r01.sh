# round-1 ncu captures (run under gpurun): launch list of the bench command, full set of one forward's convs.
# Reports are exported to CSV on the box and deleted (gpurun copies back <= 64 MiB).
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-batching --no-batched --probe-seconds 0.3 > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_igemm|conv_halo" -s 52 -c 52 \
  -o /tmp/prof_convs python tools/one_forward.py --model resnet50 --plan 23 --reps 2 > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/prof_convs.ncu-rep --page raw --csv > gpurun_out/prof_convs_raw.csv 2>> gpurun_out/ncu_full.log
ls -la gpurun_out/
