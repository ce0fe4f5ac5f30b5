# Session-5 final state: launch list of one b1 forward (first: a clean process), the GPU suite,
# smoke, and the other BASELINE configs (C1, C3 +- stage migration, C4 subset, C5) at the final state.
set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/s5_launch_list.csv python tools/one_forward.py --model resnet50 --plan 32 --reps 2 \
  > gpurun_out/s5_launch_list.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s5_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/s5_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s5_smoke.log
timeout 1500 python tools/configs_gpu.py c1 c3 c5 c4 --c4-cells 2x2_1,4x2_1,4x2_2,4x4_2,8x2_2 > gpurun_out/s5_configs.jsonl 2> gpurun_out/s5_configs.log
echo "configs rc=$?"
tail -2 gpurun_out/s5_gputests.log; tail -2 gpurun_out/s5_smoke.log; wc -l gpurun_out/s5_launch_list.csv
