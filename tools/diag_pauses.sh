#!/bin/bash
# Environment check for the GPU-wide pauses the executor detects: who else is
# on the GPU, what the driver reports, and the idle freeze pattern.
# Usage (on the GPU box): bash tools/diag_pauses.sh > gpurun_out/<name>.txt 2>&1
set -x
nvidia-smi --query-compute-apps=pid,process_name,used_memory --format=csv
nvidia-smi -q -d PERFORMANCE,CLOCK,POWER,COMPUTE | head -120
ps -eo pid,ppid,etime,comm,args --sort=start_time | head -60
./tools/freeze_probe.bin 10 8 200000
./tools/freeze_probe.bin 10 148 200000
