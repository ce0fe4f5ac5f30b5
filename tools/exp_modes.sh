R=1000,1200,1400
run() { echo "=== $1"; env $2 timeout 150 python tools/diag_knee.py --rates $R --duration 1.5 2>&1 | grep -E "afet|^rate|  HP" ; }
run layers "DARIS_STAGE_MODE=layers"
run layers_split2 "DARIS_STAGE_MODE=layers DARIS_SPLITK_MAX=2"
run layers_split4 "DARIS_STAGE_MODE=layers DARIS_SPLITK_MAX=4"
run persist_g24 "DARIS_STAGE_MODE=persistent DARIS_STAGE_GRID=24"
run persist_g37 "DARIS_STAGE_MODE=persistent DARIS_STAGE_GRID=37"
