#!/bin/bash
# Round-end evidence: ncu launch list over bench.py and full-set captures of the per-role kernels.
# Usage: gpurun --timeout 1800 -- bash tools/gpu_profile.sh TAG
set -u
TAG=${1:-prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'attn|select' --launch-skip 35 -c 12 \
    -o $OUT/probe python tools/kernel_probe.py > $OUT/ncu_probe.log 2>&1
echo "probe exit $?"
