#!/bin/bash
# Round-2 evidence: GPU suite, smoke, bench C1 (+cpu baseline) and C2-C4 (C4 with the budget
# sweep), ncu launch list of the C1 bench, ncu --set full of the per-role kernels.
# Usage: gpurun --timeout 3000 -- bash tools/gpu_round3.sh TAG
set -u
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_c1.json 2> $OUT/bench_c1.err; echo "bench exit $?" >> $OUT/bench_c1.err
tail -2 $OUT/bench_c1.err
timeout 600 python bench.py --config c2 --steps 30 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --config c3 --steps 30 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --config c4 --steps 20 --budget 1024,2048,4096,8192 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
for c in c2 c3 c4; do tail -1 $OUT/bench_$c.err | cut -c1-120; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
echo "ncu list exit $?" >> $OUT/ncu_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'attn|select|sparse_lat' --launch-skip 35 -c 12 \
    -o $OUT/probe python tools/kernel_probe.py > $OUT/ncu_probe.log 2>&1; echo "ncu probe exit $?" >> $OUT/ncu_probe.log
for f in ncu_bench ncu_probe; do tail -n 1 $OUT/$f.log; done
