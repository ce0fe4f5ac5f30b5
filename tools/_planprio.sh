# A/B on one box: C2 knee with per-priority layer planning (HP wider grids)
for cfg in "0 0" "36 18" "48 23" "36 23"; do
  set -- $cfg
  DARIS_PLAN_SMS_HP=$1 DARIS_PLAN_SMS_LP=$2 timeout 600 python bench.py --no-cpu --no-batching --no-batched > gpurun_out/bench_pp_$1_$2.json 2> gpurun_out/bench_pp_$1_$2.log
  python -c "import json;d=json.load(open('gpurun_out/bench_pp_$1_$2.json'));print('hp=$1 lp=$2', d['value'], d['constraints_met'], d['e2e']['value'], d['p99_hp_response_ms'], d['config']['knee_rate_per_task'])"
done
